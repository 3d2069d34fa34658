# round 2, batch 5: C3 steady layer 400 in isolation, with cycle accounting and ablations
mkdir -p gpurun_out
out=gpurun_out/ablate_c3.txt; : > $out
for d in "" "-DSPDNN_PROFILE" "-DSPDNN_ABLATE_STORE" "-DSPDNN_ABLATE_STAGE" "-DSPDNN_ABLATE_COMPUTE"; do
  SPDNN_NVCC_DEFINES="$d" timeout 600 python tools/layer_ablate.py c3 --layer 400 --m 31230 >> $out 2>&1
done
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
