#!/bin/bash
# One GPU-box pass (run from the repo root under gpurun): GPU tests, bench
# line, ncu launch lists + full captures for C2 and C3.  Usage:
#   tools/gpu_round.sh TAG [tests|bench|ncu|sweep|stack ...]
set -u
TAG=${1:-r02}; shift || true
WHAT=${*:-tests bench ncu}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu_${TAG}.txt 2>&1
for w in $WHAT; do
  case $w in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests_${TAG}.log 2>&1
           echo "tests rc=$?" ;;
    bench) timeout 600 python bench.py > $OUT/bench_c2_${TAG}.json 2> $OUT/bench_c2_${TAG}.err
           echo "bench rc=$?"; tail -c 600 $OUT/bench_c2_${TAG}.json ;;
    bench3) timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/bench_c3_${TAG}.json 2> $OUT/bench_c3_${TAG}.err
           echo "bench3 rc=$?" ;;
    ncu)   for c in c2 c3; do timeout 1500 bash tools/ncu_capture.sh $c $TAG; done
           echo "ncu done" ;;
    sweep) timeout 1500 python tools/sweep.py > $OUT/sweep_${TAG}.json 2> $OUT/sweep_${TAG}.err
           echo "sweep rc=$?" ;;
    stack) timeout 600 python tools/stack_bench.py > $OUT/stack_c3_${TAG}.json 2> $OUT/stack_${TAG}.err
           echo "stack rc=$?" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_${TAG}.log 2>&1
           echo "smoke rc=$?" ;;
    envelope) timeout 600 python tools/envelope_probe.py > $OUT/envelope_${TAG}.json 2> $OUT/envelope_${TAG}.err
           echo "envelope rc=$?" ;;
    ref)   timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_${TAG}.json 2> $OUT/bench_ref_${TAG}.err
           echo "ref rc=$?" ;;
  esac
done
