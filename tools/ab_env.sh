# A/B of an environment knob on the bench (GPU box):
#   VAR=DESMOE_FFN_HALF VALS="0 148" REPS=3 bash tools/ab_env.sh
# prints vote / vanilla / flushed µs per block for each value, interleaved.
for r in $(seq ${REPS:-3}); do
  for v in ${VALS}; do
    env ${VAR}=$v timeout 300 python bench.py --no-cpu-baseline --strategies vote,vanilla \
      --steps ${STEPS:-100} --warmup 5 ${EXTRA} 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
s=d['strategies']
print('$VAR=$v', 'vote', d['value'], 'vanilla', s['vanilla']['us_per_block'] if isinstance(s,dict) and 'vanilla' in s else '?', 'flushed', d.get('value_l2_flushed'), d.get('vanilla_l2_flushed'), 'e2e', d['e2e']['value'])
" 2>&1 | tail -1
  done
done
