"""CPU re-execution of a LayerPlan in the exact order and rounding the CUDA
kernel uses (csrc/layer.cu), for both record formats (per-row weights, and
the one-word mask records of uniform-weight layers). Test infrastructure: lets the layout builder be
checked bit-for-bit against the oracle without a GPU. float32 numpy ops are
IEEE single precision with round-to-nearest, like the kernel's fma.rn with
an exact product / add.rn."""

import numpy as np

ROW_BYTES = 512  # SPDNN_STAGED_ROW_BYTES


def r4(x):
    return (x + 3) & ~3


def decode(plan):
    """Yield, per block: (stages, groups) with stages = [(fp list, records)],
    groups = [(rows, [(stage, rel, cnt)])]."""
    R, RW = plan.rows_per_group, plan.record_words
    rec = plan.records.reshape(-1, RW) if plan.num_records else np.zeros((0, RW), np.uint32)
    blocks = plan.blocks.reshape(-1, 8)
    extra = plan.stages.reshape(-1, 4)
    for g0, ng, nst, first_extra, meta_off, fp_cnt, rec_off, rec_cnt in blocks:
        meta = plan.meta
        fp = meta[meta_off:meta_off + fp_cnt]
        seg = meta[meta_off + r4(fp_cnt): meta_off + r4(fp_cnt) + 2 * ng].reshape(-1, 2)
        rows = meta[meta_off + r4(fp_cnt) + 2 * ng: meta_off + r4(fp_cnt) + 2 * ng + R * ng]
        stages = [(fp, rec[rec_off:rec_off + rec_cnt])]
        for s in range(1, nst):
            moff, fc, ro, rc = extra[first_extra + s - 1]
            stages.append((meta[moff:moff + fc], rec[ro:ro + rc]))
        groups = []
        for gl in range(ng):
            segs = [(0, int(seg[gl, 0]), int(seg[gl, 1]))]
            if nst > 1:
                assert ng == 1
                segs += [(s, 0, len(stages[s][1])) for s in range(1, nst)]
            groups.append((rows[gl * R:(gl + 1) * R], segs))
        yield stages, groups


def emulate_layer(plan, bias, x):
    """x: (N, M) float32 (column j = feature j). Returns (N, M) F-order out, alive."""
    n, m = x.shape
    out = np.empty((n, m), dtype=np.float32, order="F")
    written = np.zeros(n, dtype=bool)
    R = plan.rows_per_group
    x = np.asarray(x, dtype=np.float32)
    for stages, groups in decode(plan):
        for rows, segs in groups:
            acc = np.zeros((R, m), dtype=np.float32)
            for s, rel, cnt in segs:
                fp, recs = stages[s]
                for r in recs[rel:rel + cnt]:
                    if plan.uniform:
                        # one word: slot << 24 | row mask << 1; unset bits add nothing
                        word = int(r[0])
                        y = x[fp[word >> 24]]
                        w = np.uint32(plan.weight_bits).view(np.float32)
                        for k in range(R):
                            if word >> (k + 1) & 1:
                                acc[k] = acc[k] + (y * w).astype(np.float32)
                        continue
                    assert int(r[0]) % ROW_BYTES == 0
                    y = x[fp[int(r[0]) // ROW_BYTES]]
                    ws = r[1:1 + R].view(np.float32)
                    for k in range(R):
                        acc[k] = acc[k] + (y * ws[k]).astype(np.float32)
            for k in range(R):
                row = int(rows[k])
                if row < 0:
                    continue
                v = (acc[k] + np.float32(bias[row])).astype(np.float32)
                v = np.where(v < 0, np.float32(0), v)
                v = np.where(v > 32, np.float32(32), v)
                out[row] = v
                assert not written[row]
                written[row] = True
    assert written.all() or n == 0
    return out, (out > 0).any(axis=0)
