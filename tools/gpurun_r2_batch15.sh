# round 2, batch 15: cycle accounting of the staging pipeline alone (record
# loop and output stores removed) vs the full kernel, C2 layer 200
mkdir -p gpurun_out
out=gpurun_out/b15.txt; : > $out
for d in "-DSPDNN_PROFILE -DSPDNN_ABLATE_COMPUTE -DSPDNN_ABLATE_STORE" "-DSPDNN_PROFILE -DSPDNN_ABLATE_COMPUTE" "-DSPDNN_PROFILE"; do
  SPDNN_NVCC_DEFINES="$d" timeout 600 python tools/layer_ablate.py c2 --layer 200 >> $out 2>/dev/null
done
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
