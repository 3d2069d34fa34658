mkdir -p gpurun_out
out=gpurun_out/b30.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "alternating or reference_nets or pipelined" > gpurun_out/b30_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -2 gpurun_out/b30_tests.log >> $out
timeout 300 python bench.py --config c2 --cpu-sample 0 --steps 3 > gpurun_out/b30_c2.json 2> gpurun_out/b30_c2.err
python -c "import json; d=json.load(open('gpurun_out/b30_c2.json')); print(json.dumps(d['e2e']))" >> $out 2>&1 || tail -5 gpurun_out/b30_c2.err >> $out
cat $out
