# Same-box A/B of libdesmoe.so builds (ab/<name>.so) on bench.py (C2 vote +
# vanilla, no CPU baseline) and a C2 FFN trace, alternating builds.
#   SOS="atom red" tools/ab_so_bench.sh
cp paper_2602_00879_b200/libdesmoe.so ab/_current.so
for r in 1 2; do
  for v in ${SOS:-old new}; do
    cp ab/$v.so paper_2602_00879_b200/libdesmoe.so
    timeout 300 python bench.py --no-cpu-baseline --strategies vote,vanilla --steps ${STEPS:-60} \
      --config ${CFG:-c2} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'vote', d['value'], 'flushed', d['value_l2_flushed'], 'vanilla', d['strategies']['vanilla']['us_per_block'], 'ffn', d['strategies']['vote']['phase_us']['expert_ffn'], 'e2e', d['e2e']['value'])"
    python tools/ffn_trace.py --config ${CFG:-c2} --strategy vote --json gpurun_out/abb_$v.json > /dev/null 2>&1
    python -c "
import json; d=json.load(open('gpurun_out/abb_$v.json')); print('$v trace', {k: d.get(k) for k in ['h_ready_waits','phaseA_last_done_us','last_unit_done_us','kernel_span_us','combine_end_us']})"
  done
done
cp ab/_current.so paper_2602_00879_b200/libdesmoe.so
