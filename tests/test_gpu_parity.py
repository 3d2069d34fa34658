"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle and
the reference fixtures. Integer/category results must be identical and, since
the kernel keeps the reference's per-row ascending fp32 order, values are
checked bit for bit as well (north-star tolerance 1e-4 is the fallback bound
written next to each value check)."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_npz, random_layer
from oracle import oracle
from paper_2007_14152_b200 import engine, ingest
from paper_2007_14152_b200.engine import PlanParams, build_plans
from paper_2007_14152_b200.model import (InferenceConfig, LayerCSR, ModelError, NetworkModel,
                                         make_feature_batch, make_layer_csr)

pytestmark = pytest.mark.gpu
TOL = 1e-4  # north star: final values within 1e-4 absolute


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def same_bits(a, b):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _layer_case(layer, params, rng, m):
    n = layer.neurons
    x = rng.uniform(0, 3, (n, m)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    plan = build_plans([layer], params)[0]
    prep = engine.PreparedLayer(csr=layer, plan=plan)
    y, act = engine.optimized_layer(make_feature_batch(n, x), prep, bias)
    ref, ref_act = oracle.layer(layer, bias, x)
    assert same_bits(y, ref)
    assert np.array_equal(act, ref_act)


PARAMS = [PlanParams(), PlanParams(rows_per_group=1, reorder=False),
          PlanParams(rows_per_group=3), PlanParams(rows_per_group=7, reorder=False),
          PlanParams(rows_per_group=7, footprint_cap=5, record_cap=8, max_groups=3),
          PlanParams(rows_per_group=3, footprint_cap=2, record_cap=2),
          PlanParams(rows_per_group=6), PlanParams(rows_per_group=5),
          PlanParams(rows_per_group=4)]


@pytest.mark.parametrize("pi", range(len(PARAMS)))
def test_layer_random_pm_weights(cuda_ok, pi):
    rng = np.random.default_rng(7 + pi)
    for _ in range(12):
        n = int(rng.integers(1, 90))
        layer = random_layer(rng, n, max_row_nnz=min(n, int(rng.integers(1, 16))))
        _layer_case(layer, PARAMS[pi], rng, m=int(rng.integers(1, 200)))


@pytest.mark.parametrize("pi", range(len(PARAMS)))
def test_layer_synthetic(cuda_ok, pi):
    rng = np.random.default_rng(70 + pi)
    for n, k in ((64, 16), (1024, 32), (4096, 32), (1000, 7)):
        model = ingest.generate_synthetic_network(
            ingest.GeneratorSpec(neurons=n, layers=1, connections_per_neuron=k,
                                 seed=int(rng.integers(1 << 30))))
        _layer_case(model.layers[0], PARAMS[pi], rng, m=int(rng.integers(60, 300)))


def test_layer_reference_fixtures(cuda_ok):
    """Single layers whose expected outputs came from the reference itself."""
    z = load_npz("layers.npz")
    for i in range(int(z["count"])):
        layer = LayerCSR(z[f"l{i}_row_ptr"], z[f"l{i}_col"], z[f"l{i}_val"])
        feats = make_feature_batch(layer.neurons, z[f"l{i}_x"])
        for mode_fn in (lambda: engine.baseline_layer(feats, layer, z[f"l{i}_bias"]),
                        lambda: engine.optimized_layer(
                            feats, engine.prepare_layer(layer, InferenceConfig(), "optimized"),
                            z[f"l{i}_bias"])):
            y, act = mode_fn()
            assert same_bits(y, z[f"l{i}_y"]), i
            assert np.array_equal(act, z[f"l{i}_active"]), i


def test_layer_dense_multistage_rows(cuda_ok):
    rng = np.random.default_rng(6)
    n = 700
    rows = np.repeat(np.arange(5), 600)
    cols = np.concatenate([rng.choice(n, 600, replace=False) for _ in range(5)])
    layer = make_layer_csr(n, rows, cols, rng.uniform(-1, 1, 3000).astype(np.float32))
    for p in (PlanParams(rows_per_group=3), PlanParams(rows_per_group=1, reorder=False)):
        _layer_case(layer, p, rng, m=130)
    # the same pattern with one weight value: mask records, multi-stage blocks
    # whose extra stages are read from global memory (accumulate_global)
    uni = make_layer_csr(n, rows, cols, np.full(3000, 0.0625, np.float32))
    for p in (PlanParams(), PlanParams(rows_per_group=7), PlanParams(rows_per_group=1)):
        plan = build_plans([uni], p)[0]
        assert plan.uniform and len(plan.stages) > 0
        _layer_case(uni, p, rng, m=130)


@pytest.mark.parametrize("mode", ["optimized", "baseline"])
def test_infer_reference_nets(cuda_ok, mode):
    """60 whole networks with reference-produced categories, counts, values."""
    z = load_npz("nets.npz")
    for c in range(int(z["count"])):
        n, L, k, m, mseed, iseed = (int(v) for v in z[f"c{c}_spec"])
        model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
            neurons=n, layers=L, connections_per_neuron=k, bias_value=float(z[f"c{c}_bias"]),
            seed=mseed))
        inputs = ingest.generate_synthetic_inputs(n, m, float(z[f"c{c}_density"]), seed=iseed)
        res = engine.infer(model, inputs, InferenceConfig(), mode=mode)
        counts = [o.active_before for o in res.per_layer] + [res.per_layer[-1].active_after]
        assert np.array_equal(res.categories, z[f"c{c}_cats"]), c
        assert counts == z[f"c{c}_counts"].tolist(), c
        assert same_bits(res.final.data, z[f"c{c}_final"]), c


def test_infer_random_pm_networks_vs_oracle(cuda_ok):
    rng = np.random.default_rng(31)
    for _ in range(8):
        n = int(rng.integers(8, 120))
        L = int(rng.integers(1, 6))
        layers = [random_layer(rng, n, max_row_nnz=min(n, 10)) for _ in range(L)]
        bias = rng.uniform(-0.3, 0.3, n).astype(np.float32)
        model = NetworkModel(neurons=n, layers=layers, bias=bias)
        m = int(rng.integers(1, 300))
        inputs = make_feature_batch(n, rng.uniform(0, 2, (n, m)).astype(np.float32))
        ref = oracle.infer(model, inputs)
        for mode in ("optimized", "baseline"):
            res = engine.infer(model, inputs, InferenceConfig(), mode=mode)
            assert np.array_equal(res.categories, ref.categories)
            assert [o.active_before for o in res.per_layer] == ref.counts[:-1].tolist()
            assert same_bits(res.final.data, ref.final)


def test_flagship_digest(cuda_ok):
    d = json.load(open(os.path.join(GOLDEN, "digests.json")))["flagship"]
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=120, connections_per_neuron=32, bias_value=-0.3, seed=1))
    inputs = ingest.generate_synthetic_inputs(1024, 6000, 0.3, seed=2)
    res = engine.infer(model, inputs, InferenceConfig())
    counts = [o.active_before for o in res.per_layer] + [res.per_layer[-1].active_after]
    assert len(res.categories) == d["survivors"]
    assert sha(res.categories.astype("<i8")) == d["categories_sha256"]
    assert counts == d["counts"]
    assert sha(np.asarray(res.final.data, dtype="<f4").T) == d["final_sha256"]


def test_config1_full_digest(cuda_ok):
    """BASELINE.json config 1 at full size (60000 inputs): exact categories and
    the exact per-layer active-count sequence of the reference."""
    d = json.load(open(os.path.join(GOLDEN, "digests.json")))["config1"]
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=120, connections_per_neuron=32, bias_value=-0.3, seed=1))
    inputs = ingest.generate_synthetic_inputs(1024, 60000, 0.3, seed=2)
    res = engine.infer(model, inputs, InferenceConfig())
    counts = np.array([o.active_before for o in res.per_layer] +
                      [res.per_layer[-1].active_after], np.int64)
    assert len(res.categories) == d["survivors"]
    assert sha(res.categories.astype("<i8")) == d["categories_sha256"]
    assert sha(counts.astype("<i8")) == d["counts_sha256"]
    assert int(counts[:-1].sum()) == d["sum_active"]
    assert (res.final.data == 32.0).all()  # every final value is 32.0


def test_edge_cases(cuda_ok):
    # zero layers: identity (tests/test_engine.py:87-93)
    model = NetworkModel(neurons=4, layers=(), bias=np.zeros(4))
    inputs = make_feature_batch(4, np.ones((4, 3), np.float32))
    res = engine.infer(model, inputs, InferenceConfig())
    assert res.categories.tolist() == [0, 1, 2] and res.per_layer == []
    # all-zero inputs die in layer 0; later layers report zeros (engine.py:265-270)
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=32, layers=5, connections_per_neuron=4, bias_value=-0.3, seed=2))
    res = engine.infer(model, make_feature_batch(32, np.zeros((32, 6), np.float32)),
                       InferenceConfig())
    assert res.categories.tolist() == []
    assert res.per_layer[0].active_before == 6 and res.per_layer[0].active_after == 0
    assert res.per_layer[0].weight_element_reads > 0
    assert all(o.active_before == 0 for o in res.per_layer[1:])
    # one neuron, one feature, m not a multiple of 64, categories carried through
    layer = make_layer_csr(1, np.array([0]), np.array([0]), np.array([2.0], np.float32))
    m1 = NetworkModel(neurons=1, layers=(layer,), bias=np.array([-1.0], np.float32))
    res = engine.infer(m1, make_feature_batch(1, np.array([[3.0, 0.1, 1.0]], np.float32),
                                              categories=[4, 9, 11], total_inputs=12),
                       InferenceConfig())
    assert res.categories.tolist() == [4, 11]
    assert res.final.data[0].tolist() == [5.0, 1.0]
    # wrong-mode prepared structures raise ModelError (tests/test_parallel.py:246-252)
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=64, layers=2, connections_per_neuron=8, seed=1))
    bad = engine.prepare_model(model, InferenceConfig(), "baseline")
    with pytest.raises(ModelError):
        engine.infer(model, ingest.generate_synthetic_inputs(64, 5, 0.5, seed=1),
                     InferenceConfig(), mode="optimized", prepared=bad)


def test_run_layer_step_and_counters(cuda_ok):
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=256, layers=1, connections_per_neuron=32, bias_value=-0.3, seed=5))
    inputs = ingest.generate_synthetic_inputs(256, 100, 0.3, seed=6)
    prep = engine.prepare_model(model, InferenceConfig(), "optimized")[0]
    out = engine.run_layer_step(inputs, prep, model.bias, InferenceConfig(), "optimized")
    ref = oracle.infer(model, inputs)
    assert out.features.categories.tolist() == ref.categories.tolist()
    assert out.weight_element_reads == prep.plan.total_slots * 1  # one 128-feature tile
    assert out.feature_element_reads == prep.plan.num_fp * 100


def _pow2_layer(rng, n, k):
    from paper_2007_14152_b200.model import make_layer_csr
    rows = np.repeat(np.arange(n), k)
    cols = np.concatenate([rng.choice(n, k, replace=False) for _ in range(n)])
    vals = (rng.choice([-1.0, 1.0], n * k) * 2.0 ** rng.integers(-6, 3, n * k)).astype(np.float32)
    return make_layer_csr(n, rows, cols, vals)


def test_fma_form_power_of_two_weights(cuda_ok):
    """+-2^e weights take the one-FFMA2 path; results stay bit-identical."""
    rng = np.random.default_rng(44)
    n = 200
    layers = [_pow2_layer(rng, n, 12) for _ in range(4)]
    model = NetworkModel(neurons=n, layers=layers, bias=np.full(n, -0.05, np.float32))
    prep = engine.prepare_model(model, InferenceConfig(), "optimized")
    assert all(p.plan.pow2 for p in prep)
    inputs = make_feature_batch(n, rng.uniform(0, 1, (n, 150)).astype(np.float32))
    ref = oracle.infer(model, inputs)
    res = engine.infer(model, inputs, InferenceConfig(), prepared=prep)
    assert np.array_equal(res.categories, ref.categories)
    assert same_bits(res.final.data, ref.final)


def test_fma_guard_tiny_inputs_rerun_exact(cuda_ok):
    """Inputs whose products with 2^-4 would be subnormal trip the guard and
    the engine reruns in the exact form: still bit-identical."""
    n = 64
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=n, layers=2, connections_per_neuron=16, bias_value=0.0, seed=3))
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, (n, 70)).astype(np.float32)
    x[::3, ::2] = np.float32(3e-38) * rng.uniform(0.1, 1, x[::3, ::2].shape).astype(np.float32)
    inputs = make_feature_batch(n, x)
    ref = oracle.infer(model, inputs)
    res = engine.infer(model, inputs, InferenceConfig())
    assert np.array_equal(res.categories, ref.categories)
    assert same_bits(res.final.data, ref.final)


def test_nonfinite_inputs_rerun_unpadded(cuda_ok):
    """NaN / inf inputs: zero-weight union slots would spread them; the engine
    reruns with one row per group and matches the reference semantics."""
    n = 96
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=n, layers=3, connections_per_neuron=8, bias_value=-0.1, seed=9))
    rng = np.random.default_rng(9)
    x = rng.uniform(0, 1, (n, 40)).astype(np.float32)
    x[5, 3] = np.nan
    x[17, 9] = np.inf
    inputs = make_feature_batch(n, x)
    ref = oracle.infer(model, inputs)
    res = engine.infer(model, inputs, InferenceConfig())
    assert np.array_equal(res.categories, ref.categories)
    a, b = np.asarray(res.final.data), np.asarray(ref.final)
    assert np.array_equal(np.isnan(a), np.isnan(b))
    ok = ~np.isnan(a)
    assert np.array_equal(a[ok].view(np.uint32), b[ok].view(np.uint32))


def _streaming_case(layers=40, m=1500, bias=-0.3, seed=4):
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=layers, connections_per_neuron=32, bias_value=bias, seed=seed))
    inputs = ingest.generate_synthetic_inputs(1024, m, 0.3, seed=seed + 1)
    return model, inputs


def _spy_streamer(monkeypatch):
    captured = {}
    orig = engine.WeightStreamer

    class Spy(orig):
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            captured["streamer"] = self

    monkeypatch.setattr(engine, "WeightStreamer", Spy)
    return captured


def test_streaming_equals_resident(cuda_ok, monkeypatch):
    """config.streaming (the reference's WeightStreamer path, engine.py:173-282):
    identical categories, values and per-layer counts; at most two layers'
    structures resident; every layer materialized once."""
    model, inputs = _streaming_case()
    eager = engine.infer(model, inputs, InferenceConfig())
    captured = _spy_streamer(monkeypatch)
    streamed = engine.infer(model, inputs, InferenceConfig(streaming=True))
    st = captured["streamer"]
    assert 1 <= st.peak_resident <= 2
    assert st.materialized_count == 40
    assert np.array_equal(streamed.categories, eager.categories)
    assert same_bits(streamed.final.data, eager.final.data)
    assert [(o.active_before, o.active_after) for o in streamed.per_layer] == \
        [(o.active_before, o.active_after) for o in eager.per_layer]
    ref = oracle.infer(model, inputs, threads=4)
    assert streamed.categories.tolist() == ref.categories.tolist()
    with pytest.raises(ModelError):
        engine.infer(model, inputs, InferenceConfig(streaming=True),
                     prepared=engine.prepare_model(model, InferenceConfig(), "optimized"))


def test_streaming_stops_early_on_die_off(cuda_ok, monkeypatch):
    """Every feature dead after a few layers: the streamer is stopped and the
    remaining layers are never materialized (engine.py:265-270)."""
    model, inputs = _streaming_case(layers=300, m=400, bias=-3.0)
    captured = _spy_streamer(monkeypatch)
    res = engine.infer(model, inputs, InferenceConfig(streaming=True))
    assert len(res.categories) == 0
    assert len(res.per_layer) == 300 and res.per_layer[-1].active_before == 0
    assert captured["streamer"].materialized_count < 300
    eager = engine.infer(model, inputs, InferenceConfig())
    assert [(o.active_before, o.active_after) for o in res.per_layer] == \
        [(o.active_before, o.active_after) for o in eager.per_layer]


def test_chunked_device_network_infer_device(cuda_ok):
    """DeviceNetwork.from_layers (plans built and uploaded a chunk of layers at
    a time from a layer iterator) + infer_device == infer on the whole model."""
    spec = ingest.GeneratorSpec(neurons=1024, layers=23, connections_per_neuron=32,
                                bias_value=-0.3, seed=8)
    model = ingest.generate_synthetic_network(spec)
    inputs = ingest.generate_synthetic_inputs(1024, 900, 0.3, seed=9)
    seen = []
    net = engine.DeviceNetwork.from_layers(ingest.iter_synthetic_layers(spec),
                                           ingest.synthetic_bias(spec), chunk=5,
                                           on_chunk=lambda l0, lays: seen.append((l0, len(lays))))
    assert seen == [(0, 5), (5, 5), (10, 5), (15, 5), (20, 3)]
    assert net.num_layers == 23 and len(net.chunks) == 5
    got = engine.infer_device(net, inputs)
    want = engine.infer(model, inputs, InferenceConfig())
    assert got.edges_processed == want.edges_processed
    assert np.array_equal(got.categories, want.categories)
    assert same_bits(got.final.data, want.final.data)
    assert [(o.active_before, o.active_after) for o in got.per_layer] == \
        [(o.active_before, o.active_after) for o in want.per_layer]


def test_pipelined_upload_matches_single_pass(cuda_ok, monkeypatch):
    """A large host batch takes the chunked upload/compute pipeline
    (engine._infer_pipelined), with or without values: same categories,
    per-layer counts and (bit for bit) final values as the one-pass run, and
    the oracle's categories; a NaN input makes it fall back to the guarded
    path with the same answer."""
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=40, connections_per_neuron=32, bias_value=-0.3, seed=3))
    inputs = ingest.generate_synthetic_inputs(1024, 5 * engine.PIPELINE_MIN_FEATURES + 77, 0.3,
                                              seed=5)
    with monkeypatch.context() as mp:
        mp.setattr(engine, "PIPELINE_MIN_FEATURES", 1 << 40)  # one pass
        full = engine.infer(model, inputs, InferenceConfig())
    piped_v = engine.infer(model, inputs, InferenceConfig())
    assert np.array_equal(piped_v.categories, full.categories)
    assert np.array_equal(piped_v.final.categories, full.final.categories)
    assert same_bits(piped_v.final.data, full.final.data)
    # a pageable (numpy) batch goes through the staged host copies
    pageable = make_feature_batch(1024, np.array(inputs.data, order="F"), inputs.categories,
                                  total_inputs=inputs.total_inputs)
    again = engine.infer(model, pageable, InferenceConfig())
    assert same_bits(again.final.data, full.final.data)
    piped = engine.infer(model, inputs, InferenceConfig(), values=False)
    assert piped.final is None
    assert np.array_equal(piped.categories, full.categories)
    assert [(o.active_before, o.active_after) for o in piped.per_layer] == \
        [(o.active_before, o.active_after) for o in full.per_layer]
    pick = np.arange(0, inputs.active_count, 97)
    sub = make_feature_batch(1024, np.asfortranarray(inputs.data[:, pick]), categories=pick,
                             total_inputs=inputs.total_inputs)
    ref = oracle.infer(model, sub, threads=4, want_final=False)
    assert np.intersect1d(piped.categories, pick).tolist() == ref.categories.tolist()
    data = np.asarray(inputs.data).copy()
    data[3, 9000] = np.nan
    poisoned = make_feature_batch(1024, data)
    a = engine.infer(model, poisoned, InferenceConfig(), values=False)
    b = engine.infer(model, poisoned, InferenceConfig())
    assert np.array_equal(a.categories, b.categories)


def test_concurrent_staged_transfers_and_infer(cuda_ok):
    """Pageable host buffers go through one pair of pinned chunks per device
    (engine.h2d_into / d2h_numpy); concurrent callers (the reference's
    concurrent-infer contract, pkg/tests/test_engine.py:264-287) must take
    turns on them: every thread's bytes come back unchanged, and concurrent
    infer calls on staged (pageable, multi-chunk) batches give the
    single-threaded answers bit for bit."""
    import threading
    from concurrent.futures import ThreadPoolExecutor
    import torch

    def roundtrip(seed):
        src = np.random.default_rng(seed).integers(0, 1 << 31, 3 * engine.STAGE_CHUNK // 4 + 12345,
                                                  dtype=np.int32)
        dst = torch.empty(src.shape, dtype=torch.int32, device="cuda")
        for _ in range(3):
            engine.h2d_into(dst, src)
            back = engine.d2h_numpy(dst)
            if not np.array_equal(back, src):
                return False
        return True

    with ThreadPoolExecutor(4) as ex:
        assert all(ex.map(roundtrip, range(8)))

    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=12, connections_per_neuron=32, bias_value=-0.3, seed=21))
    m = 2 * engine.STAGE_CHUNK // (4 * 1024) + 333  # > 2 staging chunks per batch
    batches = []
    for i in range(3):
        b = ingest.generate_synthetic_inputs(1024, m, 0.3, seed=30 + i)
        batches.append(make_feature_batch(1024, np.array(b.data, order="F"), b.categories,
                                          total_inputs=b.total_inputs))
    want = [engine.infer(model, b, InferenceConfig()) for b in batches]
    barrier = threading.Barrier(3)

    def run(i):
        barrier.wait()
        return i, engine.infer(model, batches[i], InferenceConfig())

    with ThreadPoolExecutor(3) as ex:
        for i, got in ex.map(run, range(3)):
            assert np.array_equal(got.categories, want[i].categories)
            assert same_bits(got.final.data, want[i].final.data)
            assert [(o.active_before, o.active_after) for o in got.per_layer] == \
                [(o.active_before, o.active_after) for o in want[i].per_layer]


def test_two_features_per_lane_variant(cuda_ok, monkeypatch):
    """The 64-feature-item kernel variant (FPL = 2, 28 consumer warps) is an
    alternative launch configuration of the same layout: same bits."""
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=30, connections_per_neuron=32, bias_value=-0.3, seed=12))
    inputs = ingest.generate_synthetic_inputs(1024, 700, 0.3, seed=13)
    want = engine.infer(model, inputs, InferenceConfig())
    monkeypatch.setattr(engine, "FEATURES_PER_LANE", 2)
    got = engine.infer(model, inputs, InferenceConfig())
    assert np.array_equal(got.categories, want.categories)
    assert same_bits(got.final.data, want.final.data)
    ref = oracle.infer(model, inputs, threads=4)
    assert got.categories.tolist() == ref.categories.tolist()


def _window_layer(rng, n, k, weights):
    """A row-permuted sliding-window layer (the generator's structure) with
    arbitrary per-entry weights: the union layout groups it with R = 7 but
    must use per-row weight records and the exact arithmetic form."""
    off = int(rng.integers(1, n))
    st = 1
    while np.gcd(st, n) != 1:
        st = int(rng.integers(1, n))
    base = (np.arange(n, dtype=np.int64) * off) % n
    cols = (base[:, None] + np.arange(k, dtype=np.int64)[None, :] * st) % n
    rows = np.repeat(np.arange(n), k)
    return make_layer_csr(n, rows, cols.reshape(-1), weights(rng, n * k))


@pytest.mark.parametrize("kind", ["uniform_negative", "random_pm", "mixed_pow2"])
def test_medium_structured_networks_all_record_formats(cuda_ok, kind):
    """2048 neurons x 12 layers x 2500 inputs with sliding-window structure
    under three weight regimes: one negative value (mask records, FMA form),
    random +-uniform values (weight records, exact form), powers of two of
    mixed sign and exponent (weight records, FMA form). Bit-exact vs oracle."""
    rng = np.random.default_rng({"uniform_negative": 1, "random_pm": 2, "mixed_pow2": 3}[kind])
    wfn = {
        "uniform_negative": lambda r, c: np.full(c, -0.0625, np.float32),
        "random_pm": lambda r, c: (r.uniform(0.01, 0.2, c) * r.choice([-1, 1], c)).astype(np.float32),
        "mixed_pow2": lambda r, c: (np.ldexp(1.0, r.integers(-6, -2, c)) * r.choice([-1, 1], c)).astype(np.float32),
    }[kind]
    n, L = 2048, 12
    layers = [_window_layer(rng, n, 32, wfn) for _ in range(L)]
    bias = np.full(n, 0.05 if kind == "uniform_negative" else -0.1, np.float32)
    model = NetworkModel(neurons=n, layers=layers, bias=bias)
    inputs = make_feature_batch(n, (rng.random((n, 2500)) < 0.3).astype(np.float32))
    prep = engine.prepare_model(model, InferenceConfig(), "optimized")
    if kind == "uniform_negative":
        assert all(p.plan.uniform for p in prep)
    else:
        assert not any(p.plan.uniform for p in prep)
    res = engine.infer(model, inputs, InferenceConfig(), prepared=prep)
    ref = oracle.infer(model, inputs, threads=8)
    assert np.array_equal(res.categories, ref.categories)
    assert [o.active_before for o in res.per_layer] + [len(res.categories)] == ref.counts.tolist()
    assert same_bits(res.final.data, ref.final)
    assert 0 < len(res.categories) or ref.counts[-1] == 0


def test_randomized_structured_networks(cuda_ok):
    """Fuzz over the generator's family (sizes, fan-in, depth, bias, input
    density, batch size, one weight value or per-entry weights): categories,
    per-layer counts and values bit-exact vs the oracle in every case."""
    rng = np.random.default_rng(int(os.environ.get("SPDNN_FUZZ_SEED", "2026")))
    for case in range(int(os.environ.get("SPDNN_FUZZ_CASES", "14"))):
        n = int(rng.choice([97, 257, 1000, 1536, 3000]))
        k = int(min(n, rng.choice([3, 8, 16, 32, 48])))
        L = int(rng.integers(2, 16))
        m = int(rng.integers(1, 2600))
        bias = float(rng.uniform(-0.6, 0.1))
        spec = ingest.GeneratorSpec(neurons=n, layers=L, connections_per_neuron=k,
                                    bias_value=bias, seed=int(rng.integers(1 << 30)))
        model = ingest.generate_synthetic_network(spec)
        if case % 3 == 1:  # per-entry weights (weight records, exact form)
            layers = [make_layer_csr(n, np.repeat(np.arange(n), np.diff(l.row_ptr)), l.col_idx,
                                     rng.uniform(0.02, 0.12, l.nnz).astype(np.float32))
                      for l in model.layers]
            model = NetworkModel(neurons=n, layers=layers, bias=model.bias)
        elif case % 3 == 2:  # another single weight value (mask records)
            w = np.float32(rng.choice([0.125, 0.25, -0.0625, 0.1]))
            layers = [make_layer_csr(n, np.repeat(np.arange(n), np.diff(l.row_ptr)), l.col_idx,
                                     np.full(l.nnz, w, np.float32)) for l in model.layers]
            model = NetworkModel(neurons=n, layers=layers, bias=model.bias)
        x = (rng.random((n, m)) < rng.uniform(0.05, 0.7)).astype(np.float32)
        if case % 4 == 3:
            x *= rng.uniform(0.5, 3.0, (n, m)).astype(np.float32)
        inputs = make_feature_batch(n, x)
        ref = oracle.infer(model, inputs, threads=8)
        res = engine.infer(model, inputs, InferenceConfig())
        msg = f"case {case}: n={n} k={k} L={L} m={m} bias={bias:.3f}"
        assert np.array_equal(res.categories, ref.categories), msg
        assert [o.active_before for o in res.per_layer] + [len(res.categories)] == \
            ref.counts.tolist(), msg
        assert same_bits(res.final.data, ref.final), msg


def test_alternating_models_keep_their_device_networks(cuda_ok):
    """Two prepared models used in turn stay resident (LRU network cache):
    the second call on a model reuses its uploaded layout, and both models'
    results stay bit-exact against the oracle."""
    mk = lambda seed, n: ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=n, layers=6, connections_per_neuron=16, bias_value=-0.2, seed=seed))
    ma, mb = mk(31, 512), mk(32, 256)
    pa = engine.prepare_model(ma, InferenceConfig(), "optimized")
    pb = engine.prepare_model(mb, InferenceConfig(), "optimized")
    ia = ingest.generate_synthetic_inputs(512, 300, 0.3, seed=5)
    ib = ingest.generate_synthetic_inputs(256, 300, 0.3, seed=6)
    net_a = engine.device_network(pa, ma.bias)
    net_b = engine.device_network(pb, mb.bias)
    assert engine.device_network(pa, ma.bias) is net_a
    assert engine.device_network(pb, mb.bias) is net_b
    for model, prep, inputs in ((ma, pa, ia), (mb, pb, ib), (ma, pa, ia)):
        res = engine.infer(model, inputs, InferenceConfig(), prepared=prep)
        ref = oracle.infer(model, inputs, threads=4)
        assert np.array_equal(res.categories, ref.categories)
        assert np.array_equal(np.asarray(res.final.data).view(np.uint32),
                              np.asarray(ref.final).view(np.uint32))
    assert engine.device_network(pa, ma.bias) is net_a
