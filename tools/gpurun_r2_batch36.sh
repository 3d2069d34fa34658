# staged host copies under concurrent callers (per-device staging lock)
mkdir -p gpurun_out
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "concurrent or pipelined" > gpurun_out/b36_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/b36_tests.log
