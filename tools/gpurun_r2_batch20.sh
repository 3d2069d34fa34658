mkdir -p gpurun_out
cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o maskloop maskloop.cu && timeout 300 ./maskloop > ../../gpurun_out/b20_loop.txt 2>&1
cat ../../gpurun_out/b20_loop.txt
