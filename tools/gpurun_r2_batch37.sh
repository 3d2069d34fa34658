# consumer cohort offset: half of every SMSP's consumer warps start their first unit N ns late
# (SPDNN_COHORT_NS lived in layer.cu for this run only; removed after it measured no change)
mkdir -p gpurun_out
out=gpurun_out/b37.txt; : > $out
for rep in 1 2; do
for ns in 0 1000 2000 3000; do
  SPDNN_NVCC_DEFINES="-DSPDNN_COHORT_NS=$ns" python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" || { echo "build $ns failed" >> $out; continue; }
  for c in c2 c3; do
    timeout 600 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 > gpurun_out/b37_${c}_$ns.json 2> gpurun_out/b37_${c}_$ns.err
    python -c "import json; d=json.load(open('gpurun_out/b37_${c}_$ns.json')); print('$rep $c ns=$ns', round(d['value'],2), 'frac', round(d['roofline']['frac'],3))" >> $out 2>&1 || tail -3 gpurun_out/b37_${c}_$ns.err >> $out
  done
done
done
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cat $out
