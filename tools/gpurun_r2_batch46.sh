# 21 consumer warps with 21-group blocks: C1's 147 groups fill 7 entries per tile exactly (8 with 20)
mkdir -p gpurun_out
out=gpurun_out/b46.txt; : > $out
for c in c1 c2 c3; do
  BENCH_ARGS="--config $c" bash tools/sweep.sh "20:2" "-" >> $out 2>&1
  BENCH_ARGS="--config $c" bash tools/sweep.sh "21:2" "max_groups=21,footprint_cap=184 max_groups=21" >> $out 2>&1
done
cat $out
