# round 2, batch 9: accountant warp (global tile accounting off the slot-release
# path) in three 24/25-warp layouts vs the publisher doing it inline
mkdir -p gpurun_out
out=gpurun_out/b9.txt; : > $out
run() {  # name defines plan
  SPDNN_NVCC_DEFINES="$2" python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" || { echo "$1 build failed" >> $out; return; }
  for c in c2 c3; do
    timeout 600 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 $3 > gpurun_out/b9_${c}_$1.json 2> gpurun_out/b9_${c}_$1.err
    python -c "import json,sys; d=json.load(open('gpurun_out/b9_${c}_$1.json')); print('$c $1', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1 || tail -3 gpurun_out/b9_${c}_$1.err >> $out
  done
}
run base "-DSPDNN_ACCOUNTANT=0" ""
run p2 "-DSPDNN_MASK_PRODUCERS=2" ""
run c19 "-DSPDNN_MASK_CONSUMERS=19" "--plan max_groups=19"
run c19p "-DSPDNN_ACCOUNTANT=0 -DSPDNN_MASK_CONSUMERS=19" "--plan max_groups=19"
run a25 "" ""
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o maskloop maskloop.cu && timeout 300 ./maskloop >> ../../$out 2>&1
cat ../../$out
