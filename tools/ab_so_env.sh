# Same-box A/B of (build, env) variants on bench.py (DES-Vote line):
#   VARIANTS="base: new: new:DESMOE_X=1" tools/ab_so_env.sh
cp paper_2602_00879_b200/libdesmoe.so ab/_current.so
for r in 1 2; do
for v in ${VARIANTS:-"base:"}; do
  so=${v%%:*}; ev=${v#*:}
  cp ab/$so.so paper_2602_00879_b200/libdesmoe.so
  env $ev timeout 300 python bench.py --no-cpu-baseline --strategies vote --steps 60 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'vote', d['value'], 'flushed', d['value_l2_flushed'], 'ffn', d['strategies']['vote']['phase_us'], 'e2e', d['e2e']['value'])"
done; done
cp ab/_current.so paper_2602_00879_b200/libdesmoe.so
