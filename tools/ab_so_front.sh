# Same-box A/B of two libdesmoe.so builds (ab/<name>.so): front timeline marks
# (ffn_trace, L2 flushed) and the L2-flushed sweep, alternating builds.
#   SOS="old new" SPECS="c3:64 c3:32" tools/ab_so_front.sh
cp paper_2602_00879_b200/libdesmoe.so ab/_current.so
for r in 1 2; do
  for v in ${SOS:-old new}; do
    cp ab/$v.so paper_2602_00879_b200/libdesmoe.so
    for spec in ${SPECS:-c3:64}; do
      c=${spec%%:*}; b=${spec##*:}
      python tools/ffn_trace.py --config $c --block $b --strategy vote --json gpurun_out/abso_$v.json > /dev/null 2>&1
      python - "$v" $c $b <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/abso_{sys.argv[1]}.json"))
bc = d.get("front_by_cta", {})
mx = lambda k: max(bc[k].values()) if k in bc else None
print(sys.argv[1], sys.argv[2], sys.argv[3], *[f"{k} {mx(k)}" for k in ("rowmax", "activated", "sums_done", "selected", "v_gathered", "ranked")],
      "coreset", mx("coreset"), "rerouted", mx("rerouted"),
      "ffn_counted", d.get("ffn_counted"), "combine_end", d.get("combine_end_us"))
PY
    done
    python tools/sweep.py --configs ${CFGS:-c3} --blocks ${BLOCKS:-32,64} --steps 20 --no-cpu 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('$v sweep', r['config'], r['block'], 'vote', r['vote']['us_per_block'], 'seq3', r['seq3']['us_per_block'], 'vanilla', r['vanilla']['us_per_block'])
"
  done
done
cp ab/_current.so paper_2602_00879_b200/libdesmoe.so
