# round 2, batch 6: full GPU suite, the default (C3) bench line, every config, the
# reference arm, compute-sanitizer; everything under gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu6.txt
lscpu | head -20 >> gpurun_out/gpu6.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=20 > gpurun_out/gpu_tests6.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests6.log
timeout 600 python bench.py > gpurun_out/b6_c3.json 2> gpurun_out/b6_c3.err
timeout 300 python bench.py --config c1 > gpurun_out/b6_c1.json 2> gpurun_out/b6_c1.err
timeout 300 python bench.py --config c2 > gpurun_out/b6_c2.json 2> gpurun_out/b6_c2.err
timeout 1200 python bench.py --config c4 --steps 3 > gpurun_out/b6_c4.json 2> gpurun_out/b6_c4.err
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/b6_c5.json 2> gpurun_out/b6_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/b6_ref.json 2> gpurun_out/b6_ref.err
bash tools/sanitize.sh
ls -la gpurun_out
