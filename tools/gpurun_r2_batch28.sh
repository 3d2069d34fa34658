mkdir -p gpurun_out
out=gpurun_out/b28.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_suite.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b28_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -2 gpurun_out/b28_tests.log >> $out
for c in c1 c2; do
  timeout 300 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 > gpurun_out/b28.json 2> gpurun_out/b28.err
  python -c "import json,sys; d=json.load(open('gpurun_out/b28.json')); print('$c', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1 || tail -3 gpurun_out/b28.err >> $out
done
cat $out
