# round 2, batch 10: software-pipelined mask loop, L2 prefetch of the next
# item's staged rows, and both, vs the current kernel
mkdir -p gpurun_out
out=gpurun_out/b10.txt; : > $out
run() {  # name defines plan
  SPDNN_NVCC_DEFINES="$2" python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" || { echo "$1 build failed" >> $out; return; }
  for c in c2 c3; do
    timeout 600 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 $3 > gpurun_out/b10_${c}_$1.json 2> gpurun_out/b10_${c}_$1.err
    python -c "import json,sys; d=json.load(open('gpurun_out/b10_${c}_$1.json')); print('$c $1', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1 || tail -3 gpurun_out/b10_${c}_$1.err >> $out
  done
}
run base "" ""
run pipe "-DSPDNN_PIPE_LOOP=1" ""
run l2 "-DSPDNN_L2_PREFETCH=1" ""
run pipel2 "-DSPDNN_PIPE_LOOP=1 -DSPDNN_L2_PREFETCH=1" ""
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b10_tests.log 2>&1; echo "tests (pipe+l2 build) rc=$?" >> $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
