# round 2, batch 24: producer lookahead depth (claims kMetaAhead+2 items ahead):
# a shallower queue per CTA should shrink the end-of-layer imbalance
mkdir -p gpurun_out
out=gpurun_out/b24.txt; : > $out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $out 2>&1 || { echo smoke failed >> $out; cat $out; exit 1; }
for rep in 1 2; do
for d in "" "-DSPDNN_META_AHEAD=3 -DSPDNN_FP_AHEAD=2" "-DSPDNN_META_AHEAD=4 -DSPDNN_FP_AHEAD=2"; do
  SPDNN_NVCC_DEFINES="$d" python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
  for c in c1 c2 c3; do
    timeout 300 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 > gpurun_out/b24.json 2> gpurun_out/b24.err
    python -c "import json,sys; d=json.load(open('gpurun_out/b24.json')); print('$c [$d]', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3))" >> $out 2>&1 || tail -3 gpurun_out/b24.err >> $out
  done
done
done
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
