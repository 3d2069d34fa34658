# round 2, batch 3: the failed multi-rank tests, ncu captures of C1/C3/C4 steady layers,
# the C3 launch list, compute-sanitizer
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parallel.py tests/test_reference_suite.py tests/test_report.py -m gpu -q -p no:cacheprovider -rf > gpurun_out/gpu_tests3.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 400 -c 1 -o gpurun_out/r2_prof_c3_layer400 python tools/profile_run.py c3 > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 60 -c 1 -o gpurun_out/r2_prof_c1_layer60 python tools/profile_run.py c1 > gpurun_out/ncu_c1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/ncu_launch_c3.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 400 -c 1 -o gpurun_out/r2_prof_c4_layer400 python tools/profile_run.py c4 > gpurun_out/ncu_c4.log 2>&1
bash tools/sanitize.sh
ls -la gpurun_out
