"""Full-size parity on BASELINE.json configs[1..3] (C2, C3, C4: the synthetic
networks and 60000-input batches bench.py measures) against digests the CPU
oracle produced (tests/golden/make_fullsize.py -> tests/golden/fullsize_*.json;
the oracle is pinned to the reference by tests/test_oracle_golden.py).

C2: the whole batch -- sorted categories, survivors, every layer's active
count and the final values, bit for bit (the reference's engine.infer
result, spdnn/engine.py:235-290).
C3 / C4: the whole batch runs on the GPU; its survivors restricted to a
fixed-seed sample of 1024 / 256 inputs must equal the oracle's survivors of
that sample (features never interact, spdnn/kernels.py:40-88), and the
sample run alone must reproduce the oracle's per-layer counts and final
values bit for bit.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2007_14152_b200 import InferenceConfig, engine, ingest
from paper_2007_14152_b200.model import make_feature_batch

pytestmark = pytest.mark.gpu


def fixture(key):
    path = os.path.join(GOLDEN, f"fullsize_{key}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_fullsize.py {key})")
    with open(path) as f:
        return json.load(f)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def spec_of(g):
    return ingest.GeneratorSpec(neurons=g["neurons"], layers=g["layers"],
                                connections_per_neuron=g["connections"],
                                bias_value=g["bias"], seed=g["model_seed"])


def sample_columns(g):
    return np.sort(np.random.default_rng(g["sample_seed"]).choice(
        g["inputs"], g["sample_columns"], replace=False))


def counts_of(res):
    return [o.active_before for o in res.per_layer] + [len(res.categories)]


def test_config2_full_batch_digest(cuda_ok):
    g = fixture("c2")
    model = ingest.generate_synthetic_network(spec_of(g))
    inputs = ingest.generate_synthetic_inputs(g["neurons"], g["inputs"], g["input_density"],
                                              seed=g["input_seed"])
    res = engine.infer(model, inputs, InferenceConfig())
    assert len(res.categories) == g["survivors"]
    assert sha(res.categories.astype(np.int64)) == g["categories_sha256"]
    assert counts_of(res) == g["counts"]
    assert sha(np.asarray(res.final.data, np.float32).T) == g["final_sha256"]
    # the Graph Challenge output path (categories only, overlapped upload)
    cats_only = engine.infer(model, inputs, InferenceConfig(), values=False)
    assert sha(cats_only.categories.astype(np.int64)) == g["categories_sha256"]
    assert counts_of(cats_only) == g["counts"]


def _sampled_check(g, run_full, run_sample, data_cols):
    cols = sample_columns(g)
    full_cats = run_full()
    want = np.asarray(g["survivor_categories"], np.int64)
    assert np.intersect1d(full_cats, cols).tolist() == want.tolist()
    sub = make_feature_batch(g["neurons"], data_cols(cols), categories=cols,
                             total_inputs=g["inputs"])
    got = run_sample(sub)
    assert got.categories.tolist() == want.tolist()
    assert counts_of(got) == g["counts"]
    assert sha(np.asarray(got.final.data, np.float32).T) == g["final_sha256"]
    assert 0 < len(want) < len(cols)


@pytest.mark.slow
def test_config3_full_batch_sampled_columns(cuda_ok):
    g = fixture("c3")
    model = ingest.generate_synthetic_network(spec_of(g))
    inputs = ingest.generate_synthetic_inputs(g["neurons"], g["inputs"], g["input_density"],
                                              seed=g["input_seed"])
    prepared = engine.prepare_model(model, InferenceConfig(), "optimized")
    _sampled_check(
        g,
        lambda: engine.infer(model, inputs, InferenceConfig(), prepared=prepared,
                             values=False).categories,
        lambda sub: engine.infer(model, sub, InferenceConfig(), prepared=prepared),
        lambda cols: np.asfortranarray(np.asarray(inputs.data)[:, cols]))


@pytest.mark.slow
def test_config4_full_batch_sampled_columns(cuda_ok):
    """65536 x 1920: the network is generated, planned and uploaded 64 layers
    at a time (DeviceNetwork.from_layers; its host CSR would be 32 GB)."""
    import torch
    g = fixture("c4")
    spec = spec_of(g)
    net = engine.DeviceNetwork.from_layers(ingest.iter_synthetic_layers(spec),
                                           ingest.synthetic_bias(spec), chunk=64)
    n, m = g["neurons"], g["inputs"]
    pinned = torch.empty((m, n), dtype=torch.float32).pin_memory()
    inputs = ingest.generate_synthetic_inputs(n, m, g["input_density"], seed=g["input_seed"],
                                              out=pinned.numpy().T)
    _sampled_check(
        g,
        lambda: engine.infer_device(net, inputs, values=False).categories,
        lambda sub: engine.infer_device(net, sub, values=True),
        lambda cols: np.asfortranarray(np.asarray(inputs.data)[:, cols]))
