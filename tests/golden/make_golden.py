"""Generate the golden fixtures by importing the reference (``spdnn``) itself.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

Outputs (committed, small):
  layers.npz      single-layer known answers: random CSR layers with +/- weights
                  (the reference's conftest.random_layer recipe, tests/conftest.py:35-52),
                  inputs, and the reference's baseline_layer outputs
                  (spdnn/engine.py:93-106 -> kernels.baseline_fused_relu)
  nets.npz        whole-network known answers: 40 small nets in the style of
                  acceptance criterion 1 plus 20 K=32 nets near the survival edge (tests/test_acceptance.py:36-70) run through
                  spdnn.engine.infer(mode="baseline"): categories, per-layer counts,
                  final values
  balance.json    spdnn.parallel.balance_step / imbalance_ratio on 300 count vectors
  digests.json    flagship 1024x120x6000 (tests/test_acceptance.py:30-31) and the
                  config-1 60000-input run: categories + count-sequence sha256
                  (config-1 figures as recorded in BASELINE.md section 3)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_layer(rng, n, max_row_nnz, make_layer_csr):
    rows, cols = [], []
    for r in range(n):
        k = int(rng.integers(0, max_row_nnz + 1))
        if k == 0:
            continue
        c = rng.choice(n, size=min(k, n), replace=False)
        rows.extend([r] * len(c))
        cols.extend(c.tolist())
    vals = rng.uniform(0.01, 1.0, size=len(rows)).astype(np.float32)
    vals *= rng.choice([-1.0, 1.0], size=len(vals)).astype(np.float32)
    return make_layer_csr(n, np.array(rows, np.int64), np.array(cols, np.int64), vals)


def main() -> None:
    sys.path.insert(0, REF)
    import spdnn
    from spdnn import engine, ingest, parallel
    from spdnn.model import InferenceConfig, make_feature_batch, make_layer_csr

    # ---- single layers, +/- weights (generic, non-uniform columns)
    rng = np.random.default_rng(20261017)
    out = {}
    for i in range(24):
        n = int(rng.integers(1, 72))
        m = int(rng.integers(1, 40))
        layer = random_layer(rng, n, min(n, int(rng.integers(1, 20))), make_layer_csr)
        x = rng.uniform(0, 3, (n, m)).astype(np.float32)
        bias = rng.uniform(-0.5, 0.5, n).astype(np.float32)
        y, act = engine.baseline_layer(make_feature_batch(n, x), layer, bias)
        out[f"l{i}_row_ptr"] = layer.row_ptr
        out[f"l{i}_col"] = layer.col_idx
        out[f"l{i}_val"] = layer.values
        out[f"l{i}_x"] = x
        out[f"l{i}_bias"] = bias
        out[f"l{i}_y"] = np.asarray(y)
        out[f"l{i}_active"] = np.asarray(act)
    np.savez_compressed(os.path.join(HERE, "layers.npz"), count=24, **out)

    # ---- small whole networks (criterion-1 style, synthetic generator)
    rng = np.random.default_rng(2024)
    nets = {}
    pruned = 0
    for case in range(60):
        if case < 40:  # criterion-1 recipe (mostly all-dead or all-alive)
            n = int(rng.integers(16, 257))
            L = int(rng.integers(1, 9))
            k = int(rng.integers(2, 17))
            m = int(rng.integers(1, 65))
            bias = -0.3 if case % 2 == 0 else 1.0 / 16.0
            density = float(rng.uniform(0.05, 1.0))
        else:  # K=32, density ~ |bias|: partial survival (finding 4)
            n = int(rng.integers(64, 300))
            L = int(rng.integers(2, 12))
            k = 32
            m = int(rng.integers(40, 200))
            bias = float(rng.choice([-0.3, -0.35, -0.4]))
            density = abs(bias) + float(rng.uniform(-0.02, 0.03))
        mseed, iseed = int(rng.integers(2**31)), int(rng.integers(2**31))
        spec = ingest.GeneratorSpec(neurons=n, layers=L, connections_per_neuron=k,
                                    bias_value=bias, seed=mseed)
        model = ingest.generate_synthetic_network(spec)
        inputs = ingest.generate_synthetic_inputs(n, m, density, seed=iseed)
        res = engine.infer(model, inputs, InferenceConfig(), mode="baseline")
        counts = [o.active_before for o in res.per_layer] + [res.per_layer[-1].active_after]
        nets[f"c{case}_spec"] = np.array([n, L, k, m, mseed, iseed], np.int64)
        nets[f"c{case}_bias"] = np.float64(bias)
        nets[f"c{case}_density"] = np.float64(density)
        nets[f"c{case}_cats"] = res.categories.astype(np.int64)
        nets[f"c{case}_counts"] = np.array(counts, np.int64)
        nets[f"c{case}_final"] = np.asarray(res.final.data)
        pruned += int(len(res.categories) < m)
    np.savez_compressed(os.path.join(HERE, "nets.npz"), count=60, **nets)

    # ---- load balancing
    rng = np.random.default_rng(77)
    cases = []
    for _ in range(300):
        w = int(rng.integers(1, 9))
        counts = rng.integers(0, 60, size=w).tolist()
        cases.append({"counts": counts, "plan": [list(p) for p in parallel.balance_step(counts)],
                      "ratio": parallel.imbalance_ratio(counts)
                      if parallel.imbalance_ratio(counts) != float("inf") else "inf"})
    with open(os.path.join(HERE, "balance.json"), "w") as f:
        json.dump(cases, f)

    # ---- flagship digests (and config-1 from BASELINE.md section 3)
    spec = ingest.GeneratorSpec(neurons=1024, layers=120, connections_per_neuron=32,
                                bias_value=-0.3, seed=1)
    model = ingest.generate_synthetic_network(spec)
    inputs = ingest.generate_synthetic_inputs(1024, 6000, 0.3, seed=2)
    res = engine.infer(model, inputs, InferenceConfig(), mode="optimized")
    counts = np.array([o.active_before for o in res.per_layer] +
                      [res.per_layer[-1].active_after], np.int64)
    digests = {
        "flagship": {
            "neurons": 1024, "layers": 120, "inputs": 6000, "density": 0.3, "bias": -0.3,
            "model_seed": 1, "input_seed": 2,
            "survivors": int(len(res.categories)),
            "categories_sha256": sha(res.categories.astype("<i8")),
            "counts": counts.tolist(),
            "final_sha256": sha(np.asarray(res.final.data, dtype="<f4").T),
            "final_all_32": bool((res.final.data == 32.0).all()),
        },
        "config1": {
            "neurons": 1024, "layers": 120, "inputs": 60000, "density": 0.3, "bias": -0.3,
            "model_seed": 1, "input_seed": 2, "survivors": 30690,
            "categories_sha256":
                "6d66a0839239cdfae536da5841c64d2a7e2b7a2b9fe4ddca8c8ce3d027cf1d9c",
            "counts_sha256":
                "16274d4a0d1460e24669b1b6b8b08b62ecdd12f94aea794da4a58be70afb2279",
            "sum_active": 3855918,
            "inputs_sha256":
                "8736cba3722300e08eb7b17ae9c0a753fa83874e585b99d6025510fc956acc3b",
            "model_cols_sha256":
                "078dcb21c7ee1c3c3e76de8d8e79d304ba477595d5b75ba5d084b06625e3902f",
            "source": "BASELINE.md section 3 (reference run, numpy 2.3.5)",
        },
        "reference_version": spdnn.__version__,
        "numpy": np.__version__,
    }
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(digests, f, indent=1)
    print("wrote fixtures; criterion-1-style nets with pruning:", pruned)


if __name__ == "__main__":
    main()
