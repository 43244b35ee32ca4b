# Same-box A/B of libdesmoe.so builds (ab/<name>.so) on the 24-layer stack
# (tools/stack_bench.py, C3 N=64) and the C2 bench line, alternating builds.
#   SOS="base new" tools/ab_so_stack.sh
cp paper_2602_00879_b200/libdesmoe.so ab/_current.so
for r in 1 2; do
  for v in ${SOS:-base new}; do
    cp ab/$v.so paper_2602_00879_b200/libdesmoe.so
    timeout 600 python tools/stack_bench.py 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v stack', {k: v['us_per_layer'] for k, v in d['strategies'].items()})"
    timeout 300 python bench.py --no-cpu-baseline --strategies vote,vanilla --steps ${STEPS:-60} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v bench vote', d['value'], 'flushed', d['value_l2_flushed'], 'vanilla', d['strategies']['vanilla']['us_per_block'], 'e2e', d['e2e']['value'])"
  done
done
cp ab/_current.so paper_2602_00879_b200/libdesmoe.so
