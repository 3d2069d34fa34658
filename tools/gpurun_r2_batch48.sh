# R = 6: 2 producer warps + 21 consumer warps (24 warps, 80 registers) with 21-group blocks, C3
mkdir -p gpurun_out
out=gpurun_out/b48.txt; : > $out
EXTRA_DEFINES="-DSPDNN_MASK_PRODUCERS=2" BENCH_ARGS="--config c3" bash tools/sweep.sh "21:2" "max_groups=21" >> $out 2>&1
BENCH_ARGS="--config c3" bash tools/sweep.sh "20:2" "-" >> $out 2>&1
cat $out
