# round 2, batch 29: row classes (identical rows grouped before the overlap chain)
mkdir -p gpurun_out
out=gpurun_out/b29.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" >> $out 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b29_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -2 gpurun_out/b29_tests.log >> $out
for c in c3 c2 c1; do
  timeout 600 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 > gpurun_out/b29_$c.json 2> gpurun_out/b29_$c.err
  python -c "import json,sys; d=json.load(open('gpurun_out/b29_$c.json')); print('$c', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1 || tail -3 gpurun_out/b29_$c.err >> $out
done
timeout 1200 python bench.py --config c4 --steps 3 --cpu-sample 0 > gpurun_out/b29_c4.json 2> gpurun_out/b29_c4.err
python -c "import json,sys; d=json.load(open('gpurun_out/b29_c4.json')); print('c4', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1 || tail -3 gpurun_out/b29_c4.err >> $out
cat $out
