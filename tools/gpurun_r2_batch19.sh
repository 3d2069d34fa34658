# round 2, batch 19: fewer rows per group at the same footprint (2-deep ring,
# more groups per block): less mask padding, more records
mkdir -p gpurun_out
out=gpurun_out/b19.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $out 2>&1 || { echo smoke failed >> $out; cat $out; exit 1; }
for rep in 1 2; do
for plan in "rows_per_group=0" "rows_per_group=5,max_groups=28,record_cap=1024" "rows_per_group=6,max_groups=23,record_cap=880" "rows_per_group=5,max_groups=24,record_cap=900"; do
  for c in c2 c3; do
    timeout 300 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 --plan "$plan" > gpurun_out/b19.json 2> gpurun_out/b19.err
    python -c "import json,sys; d=json.load(open('gpurun_out/b19.json')); print('$c $plan', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3))" >> $out 2>&1 || tail -3 gpurun_out/b19.err >> $out
  done
done
done
cat $out
