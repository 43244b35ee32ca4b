# front-kernel timelines (tools/ffn_trace.py) for vote / vanilla, L2 flushed
# and warm; DESMOE_PREWARM variants. Run on the GPU box.
for pw in ${PREWARMS:-0}; do
for s in vote vanilla; do
  DESMOE_PREWARM=$pw python tools/ffn_trace.py --config ${CFG:-c2} --strategy $s --json gpurun_out/tr_${s}_pw$pw.json > /dev/null 2>&1
done; done
python - <<'PY'
import json, os, glob
for f in sorted(glob.glob("gpurun_out/tr_*_pw*.json")):
    d = json.load(open(f))
    print(os.path.basename(f), {k[6:]: v[1] for k, v in d.items() if k.startswith("front_")})
PY
