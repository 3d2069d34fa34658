mkdir -p gpurun_out
out=gpurun_out/b23.txt; : > $out
SPDNN_NVCC_DEFINES="-DSPDNN_LTRACE" python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 300 python tools/trace_layers.py c1 >> $out 2>&1
timeout 300 python tools/trace_layers.py c2 >> $out 2>&1
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
