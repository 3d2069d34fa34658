# round 2, batch 27: split survivor layout (whole surviving tiles stay aligned)
mkdir -p gpurun_out
out=gpurun_out/b27.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" >> $out 2>&1 || { echo smoke failed >> $out; cat $out; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parallel.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b27_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -3 gpurun_out/b27_tests.log >> $out
for rep in 1 2; do
for sp in 0 1; do
  for c in c1 c2 c3; do
    SPDNN_SPLIT=$sp timeout 300 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 > gpurun_out/b27.json 2> gpurun_out/b27.err
    python -c "import json,sys; d=json.load(open('gpurun_out/b27.json')); print('$c split=$sp', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), d['config']['survivors'])" >> $out 2>&1 || tail -3 gpurun_out/b27.err >> $out
  done
done
done
cat $out
