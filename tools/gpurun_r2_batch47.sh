# mask-loop unroll (quads per iteration) with the R = 6 layout, C3
mkdir -p gpurun_out
out=gpurun_out/b47.txt; : > $out
BENCH_ARGS="--config c3" bash tools/sweep.sh "20:2 20:1 20:3" "-" >> $out 2>&1
cat $out
