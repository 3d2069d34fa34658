# rows per group 6 vs the cost model's choice (7) on every config
mkdir -p gpurun_out
out=gpurun_out/b40.txt; : > $out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
for c in c1 c3 c4 c2 c3; do
  for p in "" "rows_per_group=6"; do
    st=3; [ $c = c4 ] && st=2
    timeout 900 python bench.py --config $c --cpu-sample 0 --steps $st --warmup 3 --plan "$p" > gpurun_out/b40.json 2> gpurun_out/b40.err
    python -c "import json; d=json.load(open('gpurun_out/b40.json')); print('$c [$p]', round(d['value'],2), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), d.get('parity'))" >> $out 2>&1 || tail -3 gpurun_out/b40.err >> $out
  done
done
cat $out
