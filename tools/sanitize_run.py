"""Small inferences for compute-sanitizer (tools/sanitize.sh): the smoke
network (1024 x 12, 512 inputs at the survival edge), a 2048 x 12
structured network with per-row +/- weights (weight records, exact form) and
an 8192 x 6 generator network (R = 6 groups),
each through the public API and checked against the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [case ...]
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_2007_14152_b200 import InferenceConfig, engine, ingest  # noqa: E402
from paper_2007_14152_b200.model import NetworkModel, make_layer_csr  # noqa: E402


def smoke():
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=12, connections_per_neuron=32, bias_value=-0.3, seed=1))
    inputs = ingest.generate_synthetic_inputs(1024, 512, 0.3, seed=2)
    return model, inputs


def structured():
    """Row-permuted sliding windows (the generator's structure) with random
    +/- weights: union groups with weight records, the exact form."""
    rng = np.random.default_rng(7)
    n, k = 2048, 24
    layers = []
    for _ in range(12):
        off = int(rng.integers(1, n))
        rows = np.repeat(np.arange(n), k)
        base = (np.arange(n) * off) % n
        cols = ((base[:, None] + np.arange(k)[None, :]) % n).reshape(-1)
        vals = rng.uniform(0.02, 0.2, n * k).astype(np.float32)
        vals *= rng.choice([-1.0, 1.0], n * k, p=[0.3, 0.7]).astype(np.float32)
        layers.append(make_layer_csr(n, rows, cols, vals))
    model = NetworkModel(n, tuple(layers), np.full(n, -0.05, np.float32))
    inputs = ingest.generate_synthetic_inputs(n, 300, 0.3, seed=3)
    return model, inputs


def large():
    """8192 x 6 generator network: the R = 6 mask-record layout (>= 8192 rows)."""
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=8192, layers=6, connections_per_neuron=32, bias_value=-0.35, seed=5))
    inputs = ingest.generate_synthetic_inputs(8192, 300, 0.35, seed=6)
    return model, inputs


CASES = {"smoke": smoke, "structured": structured, "large": large}


def main(names):
    for name in names or list(CASES):
        model, inputs = CASES[name]()
        res = engine.infer(model, inputs, InferenceConfig())
        ref = oracle.infer(model, inputs, threads=4)
        ok = (np.array_equal(res.categories, ref.categories) and
              np.array_equal(np.asarray(res.final.data).view(np.uint32),
                             np.asarray(ref.final).view(np.uint32)))
        print(f"{name}: {len(res.categories)}/{inputs.active_count} survive, "
              f"bit-exact {ok}", flush=True)
        if not ok:
            sys.exit(1)


if __name__ == "__main__":
    main(sys.argv[1:])
