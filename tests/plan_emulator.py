"""CPU re-execution of a LayerPlan in the exact order and rounding the CUDA
kernel uses (csrc/layer.cu). Test infrastructure: lets the layout builder be
checked bit-for-bit against the oracle without a GPU. float32 numpy ops are
IEEE single precision with round-to-nearest, like mul.rn / add.rn / fma.rn
with an exact product."""

import numpy as np


def emulate_layer(plan, bias, x):
    """x: (N, M) float32 (column j = feature j). Returns (N, M) F-order out, alive."""
    n, m = x.shape
    out = np.empty((n, m), dtype=np.float32, order="F")
    written = np.zeros(n, dtype=bool)
    R, RW = plan.rows_per_group, plan.record_words
    rec = plan.records.reshape(-1, RW) if plan.num_records else np.zeros((0, RW), np.uint32)
    blocks = plan.blocks.reshape(-1, 8)
    stages = plan.stages.reshape(-1, 4)
    segs = plan.segs.reshape(-1, 2)
    x = np.asarray(x, dtype=np.float32)
    for b in range(plan.num_blocks):
        g0, ng, s0, ns, lo, hi = (int(v) for v in blocks[b][:6])
        seg0 = (lo & 0xffffffff) | (hi << 32)
        acc = np.zeros((ng, R, m), dtype=np.float32)
        for s in range(ns):
            fp_off, fp_cnt, rec_off, rec_cnt = (int(v) for v in stages[s0 + s])
            cols = plan.fp[fp_off:fp_off + fp_cnt]
            for gl in range(ng):
                so, sc = (int(v) for v in segs[seg0 + s * ng + gl])
                for r in rec[rec_off + so: rec_off + so + sc]:
                    slot = int(r[0]) // 256
                    y = x[cols[slot]]
                    ws = r[1:1 + R].view(np.float32)
                    for k in range(R):
                        p = (y * ws[k]).astype(np.float32)
                        acc[gl, k] = acc[gl, k] + p
        for gl in range(ng):
            for k in range(R):
                row = int(plan.rows[(g0 + gl) * R + k])
                if row < 0:
                    continue
                v = (acc[gl, k] + np.float32(bias[row])).astype(np.float32)
                v = np.where(v < 0, np.float32(0), v)
                v = np.where(v > 32, np.float32(32), v)
                out[row] = v
                assert not written[row]
                written[row] = True
    assert written.all() or n == 0
    return out, (out > 0).any(axis=0)
