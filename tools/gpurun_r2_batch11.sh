# round 2, batch 11: smaller record groups whose blocks fit a 3-deep ring
mkdir -p gpurun_out
out=gpurun_out/b11.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
run() {  # name plan
  for c in c2 c3; do
    timeout 600 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 --plan "$2" > gpurun_out/b11_${c}_$1.json 2> gpurun_out/b11_${c}_$1.err
    python -c "import json,sys; d=json.load(open('gpurun_out/b11_${c}_$1.json')); print('$c $1', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1 || tail -3 gpurun_out/b11_${c}_$1.err >> $out
  done
}
run R5 "rows_per_group=5"
run R4g24 "rows_per_group=4,max_groups=24"
run R6g18 "rows_per_group=6,max_groups=18"
run R7 "rows_per_group=7"
run R5g16 "rows_per_group=5,max_groups=16"
cat $out
