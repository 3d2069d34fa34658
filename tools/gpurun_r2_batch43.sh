# R = 6 frees 4 accumulator registers: 22 / 24 consumer warps at 72 registers (spill-free for R = 6), C3
mkdir -p gpurun_out
out=gpurun_out/b43.txt; : > $out
BENCH_ARGS="--config c3" bash tools/sweep.sh "20:2" "-" >> $out 2>&1
BENCH_ARGS="--config c3" bash tools/sweep.sh "22:2" "rows_per_group=6,max_groups=22" >> $out 2>&1
BENCH_ARGS="--config c3" bash tools/sweep.sh "24:2" "rows_per_group=6,max_groups=24 rows_per_group=6,max_groups=24,footprint_cap=184" >> $out 2>&1
cat $out
