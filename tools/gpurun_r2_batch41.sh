# R = 6 default for large mask layers: GPU suite, default bench; C3 with R = 5 / 4 (20-group blocks)
mkdir -p gpurun_out
out=gpurun_out/b41.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $out 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/b41_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -2 gpurun_out/b41_tests.log >> $out
timeout 600 python bench.py > gpurun_out/b41_c3.json 2> gpurun_out/b41_c3.err
python -c "import json; d=json.load(open('gpurun_out/b41_c3.json')); print('c3 default', round(d['value'],2), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), d.get('parity'))" >> $out 2>&1 || tail -5 gpurun_out/b41_c3.err >> $out
for p in rows_per_group=5 rows_per_group=4; do
  timeout 600 python bench.py --cpu-sample 0 --steps 3 --plan "$p" > gpurun_out/b41.json 2> gpurun_out/b41.err
  python -c "import json; d=json.load(open('gpurun_out/b41.json')); print('c3 [$p]', round(d['value'],2), 'frac', round(d['roofline']['frac'],3))" >> $out 2>&1 || tail -3 gpurun_out/b41.err >> $out
done
cat $out
