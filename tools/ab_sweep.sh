# Same-box A/B of env settings over the L2-flushed sweep (no CPU column):
#   CFGS=c2,c3 BLOCKS=32,64,256 tools/ab_sweep.sh "" "DESMOE_FFN_FLAGS=4"
for envs in "$@"; do
  env $envs python tools/sweep.py --configs ${CFGS:-c2,c3} --blocks ${BLOCKS:-32,64,128,256} \
      --steps ${STEPS:-20} --no-cpu 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l)
    print('[$envs]', r['config'], r['block'], ' '.join(f\"{s}={r[s]['us_per_block']}/{r[s]['ffn_us']}\" for s in ('vanilla','seq3','vote')))
"
done
