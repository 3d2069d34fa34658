mkdir -p gpurun_out
out=gpurun_out/b32.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b32_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -2 gpurun_out/b32_tests.log >> $out
for c in c1 c2 c3; do
timeout 600 python bench.py --config $c --cpu-sample 0 --steps 3 > gpurun_out/b32_$c.json 2> gpurun_out/b32_$c.err
python -c "import json; d=json.load(open('gpurun_out/b32_$c.json')); e=d['e2e']; print('$c', round(d['value'],2), 'e2e', round(e['value'],2), {k: round(v['value'],2) for k,v in e['variants'].items()})" >> $out 2>&1 || tail -5 gpurun_out/b32_$c.err >> $out
done
cat $out
