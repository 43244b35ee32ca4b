# Host-buffer entry: per-kernel durations (ncu, serialised) of the x ingress
# and the combine writing y into pinned host memory, over ingress chunk sizes
# and combine CTA widths (GPU box).
for ch in ${CHUNKS:-16384 4096}; do
  echo "chunk=$ch $(DESMOE_INGRESS_CHUNK=$ch ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv python tools/host_entry_loop.py 2>/dev/null | grep x_ingress | tail -4 | awk -F, '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
for ct in ${CTHREADS:-256}; do
  echo "combine_threads=$ct $(DESMOE_COMBINE_THREADS=$ct ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv python tools/host_entry_loop.py 2>/dev/null | grep combine | tail -4 | awk -F, '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
