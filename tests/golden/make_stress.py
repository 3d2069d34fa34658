"""Generate the skewed-shard (config C5 recipe) fixtures by
running the reference's own ``spdnn.parallel.run_batch_parallel``.

Run in the build container, where /root/reference exists:

    python tests/golden/make_stress.py

Output (committed): stress.json -- per case the spec, the sorted categories,
per-layer (before, after) totals, every BalanceEntry, the CommMatrix and a
sha256 of the final values (category order).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (neurons, layers, workers, columns per shard, bias, threshold)
CASES = [
    (1024, 30, 8, 250, -0.3, 1.25),
    (1024, 30, 8, 250, -0.3, float("inf")),
    (1024, 24, 4, 300, -0.3, 1.25),
    (1024, 24, 3, 301, -0.3, 1.05),
    (512, 20, 5, 97, -0.3, 1.25),
]


def stress_inputs(make_feature_batch, generate_synthetic_inputs, n, workers, cols, bias):
    """Shard s: density |b| + 0.04 - 0.01 s, seed 100 + s."""
    parts = [generate_synthetic_inputs(n, cols, abs(bias) + 0.04 - 0.01 * s, seed=100 + s)
             for s in range(workers)]
    data = np.concatenate([np.asarray(p.data) for p in parts], axis=1)
    return make_feature_batch(n, data)


def main() -> None:
    sys.path.insert(0, REF)
    from spdnn import ingest, parallel
    from spdnn.model import InferenceConfig, make_feature_batch

    out = []
    for n, L, w, cols, bias, thr in CASES:
        model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
            neurons=n, layers=L, connections_per_neuron=32, bias_value=bias, seed=1))
        inputs = stress_inputs(make_feature_batch, ingest.generate_synthetic_inputs,
                               n, w, cols, bias)
        res, comm, bal = parallel.run_batch_parallel(
            model, inputs, InferenceConfig(workers=w, rebalance_threshold=thr))
        final = np.asarray(res.final.data, dtype="<f4").T
        out.append({
            "neurons": n, "layers": L, "workers": w, "columns": cols, "bias": bias,
            "threshold": "inf" if thr == float("inf") else thr,
            "categories": res.categories.astype(int).tolist(),
            "per_layer": [[o.active_before, o.active_after] for o in res.per_layer],
            "entries": [[e.layer, list(e.before_counts), list(e.after_counts), e.moved_rows,
                         bool(e.rebalanced)] for e in bal.entries],
            "comm": comm.matrix.astype(int).tolist(),
            "final_sha256": hashlib.sha256(np.ascontiguousarray(final).tobytes()).hexdigest(),
        })
        print(n, L, w, thr, "survivors", len(res.categories), "rebalances",
              sum(e.rebalanced for e in bal.entries), "moved", comm.total_moved)
    with open(os.path.join(HERE, "stress.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
