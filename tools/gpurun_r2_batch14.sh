# round 2, batch 14: staging microbenchmark (gather4 vs 2-D tile boxes of
# consecutive rows) and the mask-loop limiter variants
mkdir -p gpurun_out
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench tma_bench.cu -lcuda && timeout 300 ./tma_bench > ../../gpurun_out/b14_tma.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o maskloop maskloop.cu && timeout 300 ./maskloop > ../../gpurun_out/b14_loop.txt 2>&1
cat ../../gpurun_out/b14_tma.txt ../../gpurun_out/b14_loop.txt
