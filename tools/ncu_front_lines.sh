# Front-kernel warp-state samples per source line (dense sampling) for a few
# shapes (GPU box): gpurun_out/frontsrc_<cfg>_<N>.ncu-rep
set -u
for spec in ${SPECS:-c2:32 c3:32 c3:256}; do
  c=${spec%%:*}; b=${spec##*:}
  timeout 900 ncu --section SourceCounters --section WarpStateStats --section LaunchStats \
    --warp-sampling-interval 0 --clock-control none --import-source on -k regex:front_kernel -s 15 -c 1 -f \
    -o gpurun_out/frontsrc_${c}_${b} python bench.py --config $c --block $b --steps 3 --warmup 3 \
    --no-cpu-baseline --strategies vanilla,vote > gpurun_out/frontsrc_${c}_${b}.log 2>&1
done
