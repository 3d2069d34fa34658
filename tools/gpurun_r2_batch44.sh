# compute-sanitizer on the R = 6 layout (8192 x 6 generator network)
# (compute-sanitizer is closed on the GPU pool as of this run: rc 86 without running; the R = 6 layout is covered by the full-size C3/C4 parity tests instead)
mkdir -p gpurun_out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" > /dev/null
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool "$tool" --kernel-name kns=layer_kernel --print-limit 200 --error-exitcode 9 \
      python tools/sanitize_run.py large > "gpurun_out/sanitize_r6_${tool}.log" 2>&1
  echo "$tool rc=$?"; tail -3 "gpurun_out/sanitize_r6_${tool}.log"
done
