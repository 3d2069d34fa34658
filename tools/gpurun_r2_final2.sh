# round 2, final bench lines after the row-class plan change, and the C3 launch list
mkdir -p gpurun_out
out=gpurun_out/final2.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" >> $out 2>&1
timeout 600 python bench.py > gpurun_out/final2_c3.json 2> gpurun_out/final2_c3.err
timeout 300 python bench.py --config c1 > gpurun_out/final2_c1.json 2> gpurun_out/final2_c1.err
timeout 300 python bench.py --config c2 > gpurun_out/final2_c2.json 2> gpurun_out/final2_c2.err
timeout 1200 python bench.py --config c4 --steps 3 > gpurun_out/final2_c4.json 2> gpurun_out/final2_c4.err
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/final2_c5.json 2> gpurun_out/final2_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/final2_ref.json 2> gpurun_out/final2_ref.err
for c in c1 c2 c3 c4; do python -c "import json; d=json.load(open('gpurun_out/final2_$c.json')); print('$c', round(d['value'],2), 'TE/s frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python bench.py --steps 1 --warmup 0 --cpu-sample 0 > gpurun_out/ncu_launch_c3.log 2>&1
cat $out
