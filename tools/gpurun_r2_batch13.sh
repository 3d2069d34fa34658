# round 2, batch 13: one steady layer in isolation (C2 layer 200, C3 layer 400)
# with the record loop, the row staging or the output stores removed
mkdir -p gpurun_out
out=gpurun_out/b13.txt; : > $out
for rep in 1 2; do
for d in "" "-DSPDNN_ABLATE_COMPUTE" "-DSPDNN_ABLATE_STAGE" "-DSPDNN_ABLATE_STORE" "-DSPDNN_ABLATE_COMPUTE -DSPDNN_ABLATE_STORE"; do
  SPDNN_NVCC_DEFINES="$d" timeout 600 python tools/layer_ablate.py c2 --layer 200 >> $out 2>/dev/null
  SPDNN_NVCC_DEFINES="$d" timeout 600 python tools/layer_ablate.py c3 --layer 400 --m 31230 >> $out 2>/dev/null
done
done
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
