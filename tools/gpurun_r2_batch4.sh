# round 2, batch 4: exact-count record runs (tail records skipped) + row addressing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_report.py -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/gpu_tests4.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests4.log
timeout 300 python bench.py --config c2 --cpu-sample 0 --steps 10 > gpurun_out/b4_c2.json 2> gpurun_out/b4_c2.err
timeout 400 python bench.py --config c3 --cpu-sample 0 --steps 4 > gpurun_out/b4_c3.json 2> gpurun_out/b4_c3.err
timeout 300 python bench.py --config c1 --cpu-sample 0 --steps 10 > gpurun_out/b4_c1.json 2> gpurun_out/b4_c1.err
bash tools/sanitize.sh
