mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > gpurun_out/gpu_tests2.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests2.log
for R in 0 5 4; do timeout 300 python bench.py --config c2 --cpu-sample 0 --steps 10 --plan rows_per_group=$R > gpurun_out/b2_c2_R$R.json 2> gpurun_out/b2_c2_R$R.err; done
for R in 0 5; do timeout 400 python bench.py --config c3 --cpu-sample 0 --steps 4 --plan rows_per_group=$R > gpurun_out/b2_c3_R$R.json 2> gpurun_out/b2_c3_R$R.err; done
