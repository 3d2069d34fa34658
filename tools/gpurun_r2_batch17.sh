# round 2, batch 17: barrier wait flavour (try_wait / test_wait spin / try_wait with
# a suspend-time hint), full kernel and the staging-only ablation, C2 layer 200
mkdir -p gpurun_out
out=gpurun_out/b17.txt; : > $out
for d in "" "-DSPDNN_WAIT_TEST=1" "-DSPDNN_WAIT_HINT_NS=20" "-DSPDNN_WAIT_HINT_NS=1000"; do
  SPDNN_NVCC_DEFINES="$d" timeout 600 python tools/layer_ablate.py c2 --layer 200 >> $out 2>/dev/null
  SPDNN_NVCC_DEFINES="$d -DSPDNN_ABLATE_COMPUTE -DSPDNN_ABLATE_STORE" timeout 600 python tools/layer_ablate.py c2 --layer 200 >> $out 2>/dev/null
done
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
