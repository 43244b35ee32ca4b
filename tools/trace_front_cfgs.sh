for cfg in "c2 32" "c3 32" "c3 64" "c3 256"; do set -- $cfg
python tools/ffn_trace.py --config $1 --block $2 --strategy vote --json gpurun_out/trf_$1_$2.json > /dev/null 2>&1
python - $1 $2 <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/trf_{sys.argv[1]}_{sys.argv[2]}.json"))
print(sys.argv[1], sys.argv[2], {k[6:]: v for k, v in d.items() if k.startswith("front_") and k!="front_by_cta"})
PY
done
