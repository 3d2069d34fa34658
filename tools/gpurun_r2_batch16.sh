mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b16_tests.log 2>&1; echo "tests rc=$?" > gpurun_out/b16.txt
tail -3 gpurun_out/b16_tests.log >> gpurun_out/b16.txt
bash tools/gpurun_ab.sh "c2 c3 c1" 2
cat gpurun_out/b16.txt
