# round 2 re-entry: the whole GPU suite, smoke and the default bench on the restored tree
mkdir -p gpurun_out
out=gpurun_out/b33.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $out 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=10 > gpurun_out/b33_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -2 gpurun_out/b33_tests.log >> $out
timeout 600 python bench.py > gpurun_out/b33_c3.json 2> gpurun_out/b33_c3.err
python -c "import json; d=json.load(open('gpurun_out/b33_c3.json')); print('c3', round(d['value'],2), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1 || tail -5 gpurun_out/b33_c3.err >> $out
cat $out
