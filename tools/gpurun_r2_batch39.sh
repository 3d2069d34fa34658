# rows per group 6 with 20-group blocks (not covered by the earlier R sweeps), C2 and C3
mkdir -p gpurun_out
out=gpurun_out/b39.txt; : > $out
for c in c2 c3; do
  BENCH_ARGS="--config $c" bash tools/sweep.sh "20:2" "- rows_per_group=6 rows_per_group=6,footprint_cap=160 rows_per_group=5,max_groups=24" >> $out 2>&1
done
cat $out
