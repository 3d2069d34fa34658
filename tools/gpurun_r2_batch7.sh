# round 2, batch 7: team-mode consumers (SPDNN_TEAMS=2) vs the classic mapping (=1)
mkdir -p gpurun_out
out=gpurun_out/b7.txt; : > $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b7_tests.log 2>&1; echo "tests rc=$?" >> $out
for T in 1 2; do
  for c in c2 c3 c1; do
    SPDNN_TEAMS=$T timeout 600 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 > gpurun_out/b7_${c}_T$T.json 2> gpurun_out/b7_${c}_T$T.err
    python -c "import json,sys; d=json.load(open('gpurun_out/b7_${c}_T$T.json')); print('$c T=$T', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1
  done
done
for T in 1 2; do
  SPDNN_TEAMS=$T SPDNN_NVCC_DEFINES=-DSPDNN_PROFILE timeout 600 python tools/layer_ablate.py c2 --layer 200 >> $out 2>&1
done
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench tma_bench.cu -lcuda && timeout 300 ./tma_bench >> ../../$out 2>&1
cat ../../$out
