# A/B on one box: gpurun_ab/layer_base.cu vs gpurun_ab/layer_new.cu, alternating
# (usage: bash tools/gpurun_ab.sh "c2 c3" REPS [extra bench args])
mkdir -p gpurun_out
out=gpurun_out/ab.txt; : > $out
CFGS=${1:-"c2 c3"}; REPS=${2:-2}; shift 2
for rep in $(seq $REPS); do
  for v in base new; do
    cp gpurun_ab/layer_$v.cu paper_2007_14152_b200/csrc/layer.cu
    python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" || { echo "$v build failed" >> $out; continue; }
    for c in $CFGS; do
      timeout 600 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 "$@" > gpurun_out/ab_${c}_$v.json 2> gpurun_out/ab_${c}_$v.err
      python -c "import json,sys; d=json.load(open('gpurun_out/ab_${c}_$v.json')); print('$c $v', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1 || tail -3 gpurun_out/ab_${c}_$v.err >> $out
    done
  done
done
cp gpurun_ab/layer_new.cu paper_2007_14152_b200/csrc/layer.cu
cat $out
