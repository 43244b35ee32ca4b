# FFN + front timeline summary (run on the GPU box): tools/trace_ffn.sh [config]
for s in vote vanilla; do
  python tools/ffn_trace.py --config ${1:-c2} --strategy $s --json gpurun_out/ffnt_$s.json > gpurun_out/ffnt_$s.log 2>&1
  python - "$s" <<'PY'
import json, sys
s = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ffnt_{s}.json"))
except Exception as e:
    print(s, "failed", open(f"gpurun_out/ffnt_{s}.log").read()[-800:]); sys.exit()
keys = ["front_coreset", "front_exit", "ffn_pdl_released", "ffn_counted", "ffn_gathered",
        "x_ready_seen_us", "first_dequeue_us", "phaseB_first_dequeue_us", "last_unit_done_us",
        "cta_exit_us", "unit_dur_A_us", "unit_dur_B_us", "U"]
print(s, {k: d.get(k) for k in keys})
PY
done
