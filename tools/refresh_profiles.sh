#!/bin/bash
# Reruns every bench line and ncu capture behind profiles/ (under gpurun, from the repo root);
# outputs go to gpurun_out/, then: python tools/summarize_profiles.py r1 gpurun_out/prof_c2_layer200.ncu-rep gpurun_out/launches_c2.csv c2
set -x
mkdir -p gpurun_out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" >/dev/null
timeout 600 python bench.py > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
timeout 600 python bench.py --config c1 > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err
timeout 900 python bench.py --config c3 --steps 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
timeout 1200 python bench.py --config c4 --steps 2 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --cpu-sample 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 200 -c 1 -o gpurun_out/prof_c2_layer200 python tools/profile_run.py c2 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
