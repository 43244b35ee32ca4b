#!/bin/bash
# ncu evidence for the DES MoE layer (run on the GPU box from the repo root):
#   1. launch list of the layer's own kernels (device time per launch),
#   2. one --set full capture each of the persistent expert-FFN kernel and the
#      router/routing cluster kernel, DES-Vote strategy of bench.py's workload.
# Usage: tools/ncu_capture.sh [config] [tag]
set -u
CFG=${1:-c2}
TAG=${2:-r01}
OUT=gpurun_out
mkdir -p $OUT
B="python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --strategies vanilla,vote"
# launch order per strategy: warmup 3 + timed 3 + phase warmup 3 + phase timed 3
# = 12 layer calls; vanilla first, so vote's first timed call is call 16.
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:desmoe\|front_kernel\|ffn_persistent\|combine\|route\|coreset\|permute\|tile_gemm \
  --csv --log-file $OUT/launches_${CFG}_${TAG}.csv $B > $OUT/ncu_launches_${CFG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_persistent_kernel \
  -s 15 -c 1 -f -o $OUT/ffn_${CFG}_${TAG} $B > $OUT/ncu_ffn_${CFG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:front_kernel \
  -s 15 -c 1 -f -o $OUT/front_${CFG}_${TAG} $B > $OUT/ncu_front_${CFG}.log 2>&1
# the router GEMM kernel that runs ahead of the front for blocks > 32 tokens
# or pools > 128 experts (C3)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:router_cluster_kernel \
  -s 15 -c 1 -f -o $OUT/router_${CFG}_${TAG} $B > $OUT/ncu_router_${CFG}.log 2>&1
ls -la $OUT
