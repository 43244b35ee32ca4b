# Front-kernel timeline under different cache states (GPU box):
#   F=1024 (315 MB streamed per call) vs F=128 (38 MB: L2 keeps the code),
#   each with and without a 256 MiB L2 flush before the traced call.
for f in ${FFNS:-1024 128}; do
  for fl in flush noflush; do
    extra=""; [ $fl = noflush ] && extra="--no-flush"
    python tools/ffn_trace.py --config ${CFG:-c2} --strategy ${STRAT:-vote} --ffn $f $extra \
        --json gpurun_out/fp_${CFG:-c2}_f${f}_${fl}.json > /dev/null 2>&1
  done
done
python - <<'PY'
import json, glob, os
keys = ["front_wr_issued", "front_tmem_alloced", "front_pdl_waited", "front_setup_synced", "front_setup", "front_x_issued", "front_mma_full0", "front_mma_full_last", "front_mma_done", "front_partials_synced", "front_logits", "front_rowmax",
        "front_activated", "front_selected", "front_v_gathered", "front_ranked", "front_coreset",
        "front_rerouted", "ffn_list_loaded"]
for f in sorted(glob.glob("gpurun_out/fp_*.json")):
    d = json.load(open(f))
    print(os.path.basename(f), " ".join(f"{k[6:] if k.startswith('front_') else k}={d[k][-1] if isinstance(d.get(k), list) else d.get(k)}" for k in keys if k in d))
PY
