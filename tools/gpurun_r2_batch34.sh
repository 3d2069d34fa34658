# source-level stall sampling of a steady C2 layer (which lines of the consumer loop/epilogue stall)
mkdir -p gpurun_out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 200 -c 1 -o gpurun_out/b34_c2_l200 python tools/profile_run.py c2 > gpurun_out/b34_ncu.log 2>&1
ncu -i gpurun_out/b34_c2_l200.ncu-rep --page source --csv --print-source sass > gpurun_out/b34_src_sass.csv 2>&1
ncu -i gpurun_out/b34_c2_l200.ncu-rep --page source --csv --print-source cuda > gpurun_out/b34_src_cuda.csv 2>&1
ncu -i gpurun_out/b34_c2_l200.ncu-rep --page raw --csv > gpurun_out/b34_raw.csv 2>&1
ls -la gpurun_out | tail
