mkdir -p gpurun_out
out=gpurun_out/b18.txt; : > $out
SPDNN_NVCC_DEFINES="-DSPDNN_TRACE" timeout 600 python tools/trace_entries.py c2 --layer 200 >> $out 2>&1
SPDNN_NVCC_DEFINES="-DSPDNN_TRACE -DSPDNN_ABLATE_COMPUTE -DSPDNN_ABLATE_STORE" timeout 600 python tools/trace_entries.py c2 --layer 200 >> $out 2>&1
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
