# consumer-warp count vs groups per block (C < groups desynchronises the warps' epilogues)
mkdir -p gpurun_out
BENCH_ARGS="--config c2" bash tools/sweep.sh "20:2 16:2 18:2 16:1" "- max_groups=24" > gpurun_out/b35.txt 2>&1
cat gpurun_out/b35.txt
