"""Layout-builder tests (CPU only): the C++ plan is re-executed on the CPU in
the kernel's exact order (tests/plan_emulator.py) and must match the oracle
bit for bit -- generic +/- weights, power-of-two weights, forced
multi-stage blocks, every group size."""

import numpy as np
import pytest

from conftest import random_layer
from oracle import oracle
from plan_emulator import emulate_layer
from paper_2007_14152_b200 import engine, ingest
from paper_2007_14152_b200.engine import PlanParams, build_plans
from paper_2007_14152_b200.model import ModelError, make_layer_csr

PARAMS = [
    PlanParams(),
    PlanParams(rows_per_group=1, reorder=False),
    PlanParams(rows_per_group=3),
    PlanParams(rows_per_group=7, reorder=False),
    PlanParams(rows_per_group=7, footprint_cap=5, record_cap=8, max_groups=3),
    PlanParams(rows_per_group=3, footprint_cap=2, record_cap=2, max_groups=16),
    PlanParams(rows_per_group=1, footprint_cap=1, record_cap=1, max_groups=1),
    PlanParams(rows_per_group=6),
    PlanParams(rows_per_group=5),
    PlanParams(rows_per_group=4, footprint_cap=9, record_cap=12, max_groups=5),
]


def _check(layer, params, rng, m=9):
    n = layer.neurons
    x = rng.uniform(0, 3, (n, m)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    plan = build_plans([layer], params)[0]
    got, act = emulate_layer(plan, bias, x)
    ref, ref_act = oracle.layer(layer, bias, x)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    assert np.array_equal(act, ref_act)
    return plan


@pytest.mark.parametrize("pi", range(len(PARAMS)))
def test_plan_bit_exact_random_layers(pi):
    rng = np.random.default_rng(100 + pi)
    for _ in range(25):
        n = int(rng.integers(1, 60))
        layer = random_layer(rng, n, max_row_nnz=min(n, int(rng.integers(1, 12))))
        _check(layer, PARAMS[pi], rng)


@pytest.mark.parametrize("pi", range(len(PARAMS)))
def test_plan_bit_exact_synthetic_layers(pi):
    rng = np.random.default_rng(200 + pi)
    for _ in range(6):
        n = int(rng.integers(33, 300))
        k = int(rng.integers(2, 33))
        spec = ingest.GeneratorSpec(neurons=n, layers=2, connections_per_neuron=k,
                                    seed=int(rng.integers(1 << 30)))
        model = ingest.generate_synthetic_network(spec)
        for layer in model.layers:
            plan = _check(layer, PARAMS[pi], rng)
            assert plan.pow2 and plan.wexp_min == plan.wexp_max == -4  # all weights 1/16


def test_power_of_two_detection():
    rng = np.random.default_rng(5)
    layer = random_layer(rng, 40, 8, values=0.0625)
    plan = _check(layer, PlanParams(rows_per_group=3), rng)
    assert plan.pow2 and plan.wexp_min == -4
    layer2 = random_layer(rng, 40, 8)
    plan2 = _check(layer2, PlanParams(rows_per_group=3), rng)
    assert not plan2.pow2
    vals = np.array([0.5, -2.0, 0.0, 8.0], np.float32)
    from paper_2007_14152_b200.model import make_layer_csr
    l3 = make_layer_csr(4, np.array([0, 1, 2, 3]), np.array([1, 2, 3, 0]), vals)
    p3 = build_plans([l3], PlanParams())[0]
    assert p3.pow2 and (p3.wexp_min, p3.wexp_max) == (-1, 3)


def test_dense_rows_force_multi_stage():
    rng = np.random.default_rng(6)
    n = 600
    rows = np.repeat(np.arange(3), 500)
    cols = np.concatenate([rng.choice(n, 500, replace=False) for _ in range(3)])
    layer = make_layer_csr(n, rows, cols, rng.uniform(-1, 1, 1500).astype(np.float32))
    plan = _check(layer, PlanParams(rows_per_group=3), rng, m=5)
    extra = plan.stages.reshape(-1, 4)
    assert len(extra) > 0  # some block has several stages
    cap = PlanParams().footprint_cap
    assert extra[:, 1].max() <= cap and plan.max_fp_per_stage <= cap


def test_sliding_window_layers_group_well():
    """Generator layers are row-permuted sliding windows; the overlap ordering
    must find them: ~K+R-1 union columns per group of R rows."""
    model = ingest.generate_synthetic_network(
        ingest.GeneratorSpec(neurons=4096, layers=3, connections_per_neuron=32, seed=1))
    for plan in build_plans(model.layers, PlanParams()):
        assert plan.rows_per_group == 7
        per_group = plan.num_records / (4096 / 7)
        assert per_group < 40.5, per_group
        assert plan.num_fp / 4096 < 1.35


def test_large_mask_layers_group_six_rows():
    """Mask-record layers of >= 8192 rows take R = 6 (measured faster on the
    16384- and 65536-neuron networks): ~K+5 union records per
    group, bit-exact through the emulator; per-row weight records and smaller
    layers keep the cost model's R = 7."""
    rng = np.random.default_rng(23)
    n = 8192
    model = ingest.generate_synthetic_network(
        ingest.GeneratorSpec(neurons=n, layers=2, connections_per_neuron=32, seed=4))
    for layer in model.layers:
        plan = _check(layer, PlanParams(), rng, m=3)
        assert plan.rows_per_group == 6
        assert plan.num_records / (n / 6) < 40.5  # 37 records, runs padded to 4
    small = ingest.generate_synthetic_network(
        ingest.GeneratorSpec(neurons=n - 1, layers=1, connections_per_neuron=32, seed=4))
    assert build_plans(small.layers, PlanParams())[0].rows_per_group == 7
    lay = model.layers[0]
    vals = (rng.uniform(0.01, 0.2, lay.nnz) * rng.choice([-1, 1], lay.nnz)).astype(np.float32)
    weighted = make_layer_csr(n, np.repeat(np.arange(n), 32), lay.col_idx, vals)
    assert build_plans([weighted], PlanParams())[0].rows_per_group == 7


def test_identical_rows_form_classes():
    """Windows shared by thousands of rows (offset/stride ratio with 2-adic
    valuation >= 10 in the generator; each column fans out to > 512 rows):
    identical rows are grouped before the overlap chain, so every row group
    lies inside one class -- R = 7 with (almost) no union padding instead of
    the R = 1 fallback the plain chain produced -- and the layout stays
    bit-exact, including classes mixed with distinct rows."""
    n, k, v = 4096, 32, 10
    r = np.arange(n)
    starts = (r * (1 << v)) % n                    # 2^v rows per window start
    cols = (starts[:, None] + np.arange(k)[None, :]) % n
    layer = make_layer_csr(n, np.repeat(r, k), cols.reshape(-1),
                           np.full(n * k, 0.0625, np.float32))
    plan = build_plans([layer], PlanParams())[0]
    assert plan.rows_per_group == 7
    assert n * k / plan.padded_slots > 0.98
    rng = np.random.default_rng(11)
    _check(layer, PlanParams(), rng, m=4)
    # classes of several sizes next to unique rows
    m_rows = 300
    base = rng.integers(0, 200, m_rows) % 7          # 7 distinct windows, uneven classes
    uniq = np.arange(m_rows) % 3 == 0                 # every third row its own window
    st = np.where(uniq, 40 + np.arange(m_rows), base * 5)
    cl = (st[:, None] + np.arange(6)[None, :]) % m_rows
    mixed = make_layer_csr(m_rows, np.repeat(np.arange(m_rows), 6), cl.reshape(-1),
                           rng.uniform(-1, 1, m_rows * 6).astype(np.float32))
    for p in PARAMS:
        _check(mixed, p, rng)


def test_empty_and_degenerate_layers():
    rng = np.random.default_rng(9)
    empty = make_layer_csr(5, np.empty(0), np.empty(0), np.empty(0, np.float32))
    for p in PARAMS:
        _check(empty, p, rng)
    single = make_layer_csr(1, np.array([0]), np.array([0]), np.array([2.0], np.float32))
    for p in PARAMS:
        _check(single, p, rng)


def test_plan_rejects_bad_params():
    layer = make_layer_csr(4, np.array([0]), np.array([1]), np.array([1.0], np.float32))
    with pytest.raises(ModelError):
        build_plans([layer], PlanParams(rows_per_group=2))
    with pytest.raises(ModelError):
        build_plans([layer], PlanParams(rows_per_group=8))
    with pytest.raises(ModelError):
        build_plans([layer], PlanParams(footprint_cap=0))


def test_prepare_model_modes_and_stats():
    model = ingest.generate_synthetic_network(
        ingest.GeneratorSpec(neurons=256, layers=3, connections_per_neuron=16, seed=3))
    cfg = engine.InferenceConfig()
    opt = engine.prepare_model(model, cfg, "optimized")
    base = engine.prepare_model(model, cfg, "baseline")
    for p in base:
        assert p.plan.rows_per_group == 1 and p.padding.overhead == 0.0
    for p in opt:
        assert p.plan.rows_per_group in (3, 7)
        assert p.padding.padded_slots >= p.padding.nnz
    with pytest.raises(ModelError):
        engine.prepare_model(model, cfg, "fast")


def test_uniform_weight_layers_use_mask_records():
    """All stored weights identical (every Graph Challenge layer): one-word
    mask records, each group's run padded to 4; the same layer with the
    format disabled, with a second weight value, or with an explicit zero
    falls back to per-row weight records. All bit-exact."""
    rng = np.random.default_rng(5)
    spec = ingest.GeneratorSpec(neurons=200, layers=1, connections_per_neuron=12, seed=3)
    layer = ingest.generate_synthetic_network(spec).layers[0]
    for params in (PlanParams(), PlanParams(rows_per_group=3),
                   PlanParams(rows_per_group=1, reorder=False),
                   PlanParams(rows_per_group=7, footprint_cap=5, record_cap=8, max_groups=3)):
        plan = _check(layer, params, rng)
        assert plan.uniform and plan.record_words == 1
        assert plan.weight_bits == 0x3D800000
    plan = _check(layer, PlanParams(uniform_records=False), rng)
    assert not plan.uniform and plan.record_words in (2, 4, 8)
    neg = make_layer_csr(200, np.repeat(np.arange(200), np.diff(layer.row_ptr)),
                         layer.col_idx, np.full(layer.nnz, -0.5, np.float32))
    assert _check(neg, PlanParams(), rng).uniform
    vals = layer.values.copy()
    vals[17] = np.float32(0.125)
    two = make_layer_csr(200, np.repeat(np.arange(200), np.diff(layer.row_ptr)),
                         layer.col_idx, vals)
    assert not _check(two, PlanParams(), rng).uniform
    vals[17] = np.float32(0.0)
    zero = make_layer_csr(200, np.repeat(np.arange(200), np.diff(layer.row_ptr)),
                          layer.col_idx, vals)
    assert not _check(zero, PlanParams(), rng).uniform


def test_default_caps_fit_two_ring_entries_for_every_record_format():
    """The default caps are tuned for one-word mask records; with per-row
    weight records (up to 8 words) the planner shrinks them so a block stage
    still fits half of the kernel's shared memory (two ring entries)."""
    rng = np.random.default_rng(17)
    n, k = 2048, 32
    base = (np.arange(n) * 777) % n
    cols = ((base[:, None] + np.arange(k)[None, :] * 5) % n).reshape(-1)
    rows = np.repeat(np.arange(n), k)
    for vals in (np.full(n * k, 0.0625, np.float32),
                 (rng.uniform(0.01, 0.2, n * k) * rng.choice([-1, 1], n * k)).astype(np.float32)):
        plan = build_plans([make_layer_csr(n, rows, cols, vals)], PlanParams())[0]
        stage = (plan.max_fp_per_stage * 512 + plan.max_records_per_stage * plan.record_words * 4
                 + plan.max_meta_per_block * 4)
        assert stage <= 104 * 1024, (plan.record_words, stage)
        assert plan.rows_per_group == 7
