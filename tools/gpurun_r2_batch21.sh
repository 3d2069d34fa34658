# round 2, batch 21: per-layer times (C1, C2), fresh ncu captures of steady
# C1 / C3 layers and the C3 launch list on the current kernel
mkdir -p gpurun_out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b21.txt 2>&1 || { cat gpurun_out/b21.txt; exit 1; }
timeout 300 python bench.py --config c1 --cpu-sample 0 --steps 3 --dump-layers gpurun_out/b21_layers_c1.json > gpurun_out/b21_c1.json 2>/dev/null
timeout 300 python bench.py --config c2 --cpu-sample 0 --steps 3 --dump-layers gpurun_out/b21_layers_c2.json > gpurun_out/b21_c2.json 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 400 -c 1 -o gpurun_out/r2_prof_c3_layer400 python tools/profile_run.py c3 > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 60 -c 1 -o gpurun_out/r2_prof_c1_layer60 python tools/profile_run.py c1 > gpurun_out/ncu_c1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/ncu_launch_c3.log 2>&1
ls -la gpurun_out | tail -12
