# header loaded with two 16-byte loads: GPU suite, smoke, default bench (C3) and C1/C2 lines
mkdir -p gpurun_out
out=gpurun_out/b52.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $out 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/b52_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -2 gpurun_out/b52_tests.log >> $out
timeout 600 python bench.py > gpurun_out/b52_c3.json 2> gpurun_out/b52_c3.err
for c in c1 c2; do timeout 300 python bench.py --config $c > gpurun_out/b52_$c.json 2> gpurun_out/b52_$c.err; done
for c in c3 c1 c2; do python -c "import json; d=json.load(open('gpurun_out/b52_$c.json')); print('$c', round(d['value'],2), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1 || tail -5 gpurun_out/b52_$c.err >> $out; done
cat $out
