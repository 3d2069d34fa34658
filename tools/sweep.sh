#!/bin/bash
# Kernel-configuration sweep on one GPU (run under gpurun): rebuilds the
# library with each (consumer warps, mask-loop unroll) pair and runs the C2
# bench over a few layout knobs; prints "C U plan TE/s roofline_frac e2e".
# Usage: tools/sweep.sh "20:2 24:1" "footprint_cap=136 footprint_cap=144"
cd "$(dirname "$0")/.."
for cu in $1; do
  c=${cu%%:*}; u=${cu##*:}
  SPDNN_NVCC_DEFINES="-DSPDNN_MASK_CONSUMERS=$c -DSPDNN_MASK_UNROLL=$u ${EXTRA_DEFINES}" \
    python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)" || exit 1
  for p in $2; do
    [ "$p" = "-" ] && p=""
    timeout 400 python bench.py --cpu-sample 0 --steps 5 --warmup 3 --plan "$p" ${BENCH_ARGS} 2>/dev/null \
      | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $u [$p]', round(d['value'],2), round(d['roofline']['frac'],3), round(d['e2e']['value'],2))"
  done
done
python -c "from paper_2007_14152_b200 import _native; _native.build(force=True)"
