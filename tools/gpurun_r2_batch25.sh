# round 2, batch 25: persistent multi-layer chain kernel (grid barrier between layers)
mkdir -p gpurun_out
out=gpurun_out/b25.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" >> $out 2>&1 || { echo smoke failed >> $out; cat $out; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parallel.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b25_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -3 gpurun_out/b25_tests.log >> $out
rm -f gpurun_out/sanitize_summary.txt; bash tools/sanitize.sh; cat gpurun_out/sanitize_summary.txt >> $out
bash tools/gpurun_ab.sh "c1 c2 c3" 1
cat $out gpurun_out/ab.txt
