"""Full-size parity fixtures for configs C2, C3 and C4 (BASELINE.json configs[1..3]).

TEST INFRASTRUCTURE: the CPU oracle (oracle/spdnn_oracle.c, pinned to the
reference by tests/test_oracle_golden.py) run over the synthetic networks and
60000-input batches that bench.py measures. The GPU tests in
tests/test_gpu_fullsize.py compare the CUDA path with these digests; nothing
here is computed by the GPU.

    python tests/golden/make_fullsize.py [c2] [c3] [c4]   # -> tests/golden/fullsize_<cfg>.json

c2: the whole 60000-input batch through all 480 layers (the reference's
    engine.infer result, spdnn/engine.py:235-290, in BASELINE.md section 3's
    digest form): survivors, sorted-categories sha256, per-layer count
    sequence and its sha256.
c3, c4: a fixed-seed sample of the same 60000-input batch (1024 / 256
    columns) through all 1920 layers. Features never interact
    (spdnn/kernels.py:40-88 computes every column independently), so the full
    batch's survivors restricted to the sample must equal the sample's
    survivors, and the sample run on its own must reproduce these counts and
    final values bit for bit. The network is generated and consumed in
    chunks of layers (C4's CSR is 32 GB).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(neurons=4096, layers=480, bias=-0.35, density=0.35, sample=0),
    "c3": dict(neurons=16384, layers=1920, bias=-0.40, density=0.40, sample=1024),
    "c4": dict(neurons=65536, layers=1920, bias=-0.45, density=0.45, sample=256),
}
INPUTS, MODEL_SEED, INPUT_SEED, SAMPLE_SEED, K = 60000, 1, 2, 20261017, 32


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_columns(cfg) -> np.ndarray:
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(INPUTS, cfg["sample"], replace=False))


def sampled_inputs(cfg, cols) -> np.ndarray:
    """Columns `cols` of generate_synthetic_inputs(N, 60000, density, seed=2)
    without materialising the batch (same row-chunked stream)."""
    n = cfg["neurons"]
    rng = np.random.default_rng(INPUT_SEED)
    out = np.empty((n, len(cols)), np.float32, order="F")
    for r0 in range(0, n, 1024):
        r1 = min(n, r0 + 1024)
        out[r0:r1, :] = rng.random((r1 - r0, INPUTS))[:, cols] < cfg["density"]
    return out


@dataclass
class _Chunk:
    neurons: int
    layers: tuple
    bias: np.ndarray

    @property
    def num_layers(self):
        return len(self.layers)


@dataclass
class _Batch:
    data: np.ndarray
    categories: np.ndarray


def streamed_oracle(cfg, y, cats, chunk=32):
    """The oracle over the generated network, `chunk` layers at a time."""
    from oracle import oracle
    from paper_2007_14152_b200 import ingest
    spec = ingest.GeneratorSpec(neurons=cfg["neurons"], layers=cfg["layers"],
                                connections_per_neuron=K, bias_value=cfg["bias"], seed=MODEL_SEED)
    bias = ingest.synthetic_bias(spec)
    threads = os.cpu_count() or 1
    counts = [len(cats)]
    buf = []

    def flush():
        nonlocal y, cats
        if y.shape[1] == 0:
            counts.extend([0] * len(buf))
            return
        r = oracle.infer(_Chunk(cfg["neurons"], tuple(buf), bias), _Batch(y, cats),
                         threads=threads, want_final=True)
        counts.extend(int(c) for c in r.counts[1:])
        y, cats = r.final, r.categories

    for lay in ingest.iter_synthetic_layers(spec):
        buf.append(lay)
        if len(buf) == chunk:
            flush()
            buf = []
    if buf:
        flush()
    return counts, cats, y


def make(key: str) -> dict:
    cfg = CONFIGS[key]
    t0 = time.time()
    if cfg["sample"] == 0:
        from paper_2007_14152_b200 import ingest
        batch = ingest.generate_synthetic_inputs(cfg["neurons"], INPUTS, cfg["density"],
                                                 seed=INPUT_SEED)
        y, cols = batch.data, np.arange(INPUTS, dtype=np.int64)
    else:
        cols = sample_columns(cfg)
        y = sampled_inputs(cfg, cols)
    counts, cats, final = streamed_oracle(cfg, y, cols.astype(np.int64))
    out = {
        "config": key, "neurons": cfg["neurons"], "layers": cfg["layers"], "bias": cfg["bias"],
        "inputs": INPUTS, "input_density": cfg["density"], "model_seed": MODEL_SEED,
        "input_seed": INPUT_SEED, "connections": K,
        "sample_seed": SAMPLE_SEED if cfg["sample"] else None,
        "sample_columns": int(len(cols)),
        "survivors": int(len(cats)),
        "categories_sha256": sha(np.asarray(cats, np.int64)),
        "counts": counts,
        "counts_sha256": sha(np.asarray(counts, np.int64)),
        "final_sha256": sha(np.asfortranarray(final, np.float32).T) if final is not None else None,
        "generator": "oracle/spdnn_oracle.c via tests/golden/make_fullsize.py",
        "oracle_seconds": round(time.time() - t0, 1),
    }
    if cfg["sample"]:
        out["survivor_categories"] = [int(c) for c in cats]
    return out


def main(argv):
    keys = argv or list(CONFIGS)
    for key in keys:
        d = make(key)
        path = os.path.join(HERE, f"fullsize_{key}.json")
        with open(path, "w") as f:
            json.dump(d, f, indent=1)
        print(key, d["survivors"], d["categories_sha256"][:16], f"{d['oracle_seconds']} s",
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
