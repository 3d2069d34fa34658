# R = 6 layout: ncu --set full of steady C3/C4 layers, C3 launch list, C4 and C5 bench lines
mkdir -p gpurun_out
out=gpurun_out/b42.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 1200 python bench.py --config c4 --steps 3 > gpurun_out/b42_c4.json 2> gpurun_out/b42_c4.err
python -c "import json; d=json.load(open('gpurun_out/b42_c4.json')); print('c4', round(d['value'],2), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), d.get('parity'))" >> $out 2>&1 || tail -5 gpurun_out/b42_c4.err >> $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 400 -c 1 -o gpurun_out/b42_c3_l400 python tools/profile_run.py c3 > gpurun_out/b42_ncu_c3.log 2>&1; echo "ncu c3 rc=$?" >> $out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 400 -c 1 -o gpurun_out/b42_c4_l400 python tools/profile_run.py c4 > gpurun_out/b42_ncu_c4.log 2>&1; echo "ncu c4 rc=$?" >> $out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b42_launches_c3.csv python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/b42_ncu_launch.log 2>&1; echo "launches rc=$?" >> $out
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/b42_c5.json 2> gpurun_out/b42_c5.err; echo "c5 rc=$?" >> $out
cat $out
