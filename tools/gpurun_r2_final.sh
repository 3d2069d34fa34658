# round 2, final evidence: GPU suite, every bench line, reference arm,
# sanitizers, ncu captures of steady C1/C2/C3/C4 layers and the C3 launch list
mkdir -p gpurun_out
out=gpurun_out/final.txt; : > $out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv >> $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" >> $out 2>&1
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=10 > gpurun_out/final_gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $out; tail -3 gpurun_out/final_gpu_tests.log >> $out
timeout 600 python bench.py > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
timeout 300 python bench.py --config c1 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err
timeout 300 python bench.py --config c2 > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
timeout 1200 python bench.py --config c4 --steps 3 > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
for c in c1 c2 c3 c4; do python -c "import json; d=json.load(open('gpurun_out/final_$c.json')); print('$c', round(d['value'],2), 'TE/s frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1; done
rm -f gpurun_out/sanitize_summary.txt; bash tools/sanitize.sh; cat gpurun_out/sanitize_summary.txt >> $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 400 -c 1 -o gpurun_out/r2_prof_c3_layer400 -f python tools/profile_run.py c3 > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 60 -c 1 -o gpurun_out/r2_prof_c1_layer60 -f python tools/profile_run.py c1 > gpurun_out/ncu_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 200 -c 1 -o gpurun_out/r2_prof_c2_layer200 -f python tools/profile_run.py c2 > gpurun_out/ncu_c2.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 400 -c 1 -o gpurun_out/r2_prof_c4_layer400 -f python tools/profile_run.py c4 > gpurun_out/ncu_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/ncu_launch_c3.log 2>&1
cat $out
