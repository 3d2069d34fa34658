# round 2, batch 8: sanitizer-clean synchronisation (every lane arrives, gap path
# waits its own copies, no stale-phase polling), team mode default off
mkdir -p gpurun_out
out=gpurun_out/b8.txt; : > $out
rm -f gpurun_out/sanitize_summary.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b8_tests.log 2>&1; echo "tests rc=$?" >> $out
for c in c2 c3; do
  SPDNN_TEAMS=1 timeout 600 python bench.py --config $c --cpu-sample 0 --steps 3 --warmup 3 > gpurun_out/b8_${c}.json 2> gpurun_out/b8_${c}.err
  python -c "import json,sys; d=json.load(open('gpurun_out/b8_${c}.json')); print('$c', round(d['value'],2), 'TE/s', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> $out 2>&1
done
SPDNN_TEAMS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:layer_kernel -s 200 -c 1 -o gpurun_out/r2_prof_c2_layer200 python tools/profile_run.py c2 > gpurun_out/ncu_c2.log 2>&1
SPDNN_TEAMS=1 bash tools/sanitize.sh
cat gpurun_out/sanitize_summary.txt >> $out
cat $out
