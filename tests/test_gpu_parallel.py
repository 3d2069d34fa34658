"""GPU batch-parallel runner (parallel.run_batch_parallel, in-process workers
on one device): the reference's parallel test cases (tests/test_parallel.py
of the reference) against the single-worker engine and the oracle."""

import math

import numpy as np
import pytest

from oracle import oracle
from paper_2007_14152_b200 import engine, ingest, parallel
from paper_2007_14152_b200.model import InferenceConfig, ModelError, make_feature_batch

pytestmark = pytest.mark.gpu


def _small(density=0.8, m=40):
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=64, layers=5, connections_per_neuron=16, bias_value=0.0625, seed=31))
    return model, ingest.generate_synthetic_inputs(64, m, density, seed=32)


def _edge(m=400):
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=12, connections_per_neuron=32, bias_value=-0.3, seed=1))
    return model, ingest.generate_synthetic_inputs(1024, m, 0.3, seed=2)


def _check_same(res, single):
    assert np.array_equal(res.categories, single.categories)
    assert np.array_equal(np.asarray(res.final.data).view(np.uint32),
                          np.asarray(single.final.data).view(np.uint32))
    for a, b in zip(res.per_layer, single.per_layer):
        assert (a.active_before, a.active_after) == (b.active_before, b.active_after)


@pytest.mark.parametrize("workers", [1, 2, 3, 5, 8])
def test_worker_count_invariance(cuda_ok, workers):
    for model, inputs in (_small(), _edge()):
        cfg = InferenceConfig(workers=workers, rebalance_threshold=1.1)
        res, comm, bal = parallel.run_batch_parallel(model, inputs, cfg)
        _check_same(res, engine.infer(model, inputs, cfg))
        assert np.trace(comm.matrix) == 0 and comm.total_moved == bal.total_moved


def test_adversarial_die_off_triggers_rebalance(cuda_ok):
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=64, layers=4, connections_per_neuron=32, bias_value=-0.3, seed=3))
    data = np.ones((64, 60), dtype=np.float32)
    data[:, 30:] = 0.0
    inputs = make_feature_batch(64, data)
    res, comm, bal = parallel.run_batch_parallel(model, inputs, InferenceConfig(workers=2))
    _check_same(res, engine.infer(model, inputs, InferenceConfig()))
    assert res.categories.tolist() == oracle.infer(model, inputs).categories.tolist()
    reb = [e for e in bal.entries if e.rebalanced]
    assert reb and all(max(e.after_counts) - min(e.after_counts) <= 1 for e in reb)
    assert comm.matrix[0, 1] == reb[0].moved_rows
    res2, comm2, bal2 = parallel.run_batch_parallel(
        model, inputs, InferenceConfig(workers=2, rebalance_threshold=math.inf))
    assert np.array_equal(res2.categories, res.categories)
    assert not comm2.matrix.any() and not any(e.rebalanced for e in bal2.entries)


def test_skewed_stress_rebalancing(cuda_ok):
    """SURVEY.md 8(d) C5 recipe at small scale: per-shard densities skewed."""
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=24, connections_per_neuron=32, bias_value=-0.3, seed=1))
    parts = [ingest.generate_synthetic_inputs(1024, 300, 0.34 - 0.01 * s, seed=100 + s)
             for s in range(8)]
    inputs = make_feature_batch(1024, np.concatenate([p.data for p in parts], axis=1))
    ref = oracle.infer(model, inputs, threads=8)
    on = parallel.run_batch_parallel(model, inputs, InferenceConfig(workers=8))
    off = parallel.run_batch_parallel(model, inputs,
                                      InferenceConfig(workers=8, rebalance_threshold=math.inf))
    for res, comm, bal in (on, off):
        assert res.categories.tolist() == ref.categories.tolist()
    assert on[1].total_moved > 0 and off[1].total_moved == 0
    worst_on = max(e.imbalance_after for e in on[2].entries if e.before_counts[0] >= 0)
    assert worst_on <= 1.25 or any(e.rebalanced for e in on[2].entries)


def test_latency_hook_sees_typed_messages(cuda_ok):
    model, inputs = _small(m=30)
    seen = []
    cfg = InferenceConfig(workers=3, rebalance_threshold=1.05)
    res, _, _ = parallel.run_batch_parallel(model, inputs, cfg, latency_hook=seen.append)
    assert np.array_equal(res.categories, engine.infer(model, inputs, cfg).categories)
    assert parallel.CountMsg in {type(m) for m in seen}


def test_baseline_mode_and_more_workers_than_features(cuda_ok):
    model, inputs = _small(m=24)
    cfg = InferenceConfig(workers=3)
    res, _, _ = parallel.run_batch_parallel(model, inputs, cfg, mode="baseline")
    _check_same(res, engine.infer(model, inputs, cfg, mode="baseline"))
    model, inputs = _small(m=3)
    res, _, _ = parallel.run_batch_parallel(model, inputs, InferenceConfig(workers=6))
    assert np.array_equal(res.categories, engine.infer(model, inputs, InferenceConfig()).categories)


def test_wrong_mode_prepared_raises(cuda_ok):
    model, inputs = _small(m=12)
    cfg = InferenceConfig(workers=2)
    bad = engine.prepare_model(model, cfg, "baseline")
    with pytest.raises(ModelError):
        parallel.run_batch_parallel(model, inputs, cfg, mode="optimized", prepared=bad)


def _dist_worker_shard_only(rank, world, port, q):
    """Each rank builds the network chunk-wise and holds only its own shard
    (run_batch_parallel_device(shard_only=True), the bench's N > 1 path)."""
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = ingest.GeneratorSpec(neurons=1024, layers=40, connections_per_neuron=32,
                                    bias_value=-0.3, seed=21)
        net = engine.DeviceNetwork.from_layers(ingest.iter_synthetic_layers(spec),
                                               ingest.synthetic_bias(spec), chunk=7)
        lo, hi = parallel.shard_bounds(900, world)[rank]
        shard = ingest.generate_synthetic_inputs(1024, 900, 0.3, seed=22, columns=(lo, hi))
        res, comm, bal = parallel.run_batch_parallel_device(
            net, shard, InferenceConfig(workers=world), values=True, shard_only=True)
        q.put((rank, res.categories.tolist(),
               [(o.active_before, o.active_after) for o in res.per_layer],
               np.asarray(res.final.data).view(np.uint32).tobytes(), res.edges_processed))
    except Exception:  # reported to the parent instead of a queue timeout
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc(), None, None, None))
    finally:
        dist.destroy_process_group()


def test_shard_only_two_ranks_chunk_built(cuda_ok):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker_shard_only, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    errors = [r[1] for r in res if isinstance(r[1], str)]
    assert not errors, errors[0]
    for p in procs:
        assert p.exitcode == 0
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=40, connections_per_neuron=32, bias_value=-0.3, seed=21))
    inputs = ingest.generate_synthetic_inputs(1024, 900, 0.3, seed=22)
    single = engine.infer(model, inputs, InferenceConfig())
    for rank, cats, per_layer, vbits, edges in res:
        assert per_layer == [(o.active_before, o.active_after) for o in single.per_layer]
        assert edges == single.edges_processed
        if rank == 0:  # the merged survivors live on rank 0 (Algorithm 2)
            assert cats == single.categories.tolist()
            assert vbits == np.asarray(single.final.data).view(np.uint32).tobytes()
        else:
            assert set(cats) < set(single.categories.tolist())


def _dist_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)  # one GPU on the test box: ranks share it over gloo
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model, inputs = _edge(m=500)
        data = np.asarray(inputs.data).copy()
        data[:, 250:] *= 0.9  # skew: the second shard thins out faster
        inputs = make_feature_batch(1024, data)
        res, comm, bal = parallel.run_batch_parallel(
            model, inputs, InferenceConfig(workers=world, rebalance_threshold=1.05))
        q.put((rank, res.categories.tolist(),
               [(o.active_before, o.active_after) for o in res.per_layer],
               float(np.asarray(res.final.data, np.float64).sum()), comm.total_moved))
    except Exception:  # reported to the parent instead of a queue timeout
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc(), None, None, None))
    finally:
        dist.destroy_process_group()


def test_distributed_transport_two_ranks(cuda_ok):
    """run_batch_parallel under torch.distributed (2 ranks on the test box's
    single GPU, gloo wire): DistTransport + DeviceShard end to end."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    errors = [r[1] for r in res if isinstance(r[1], str)]
    assert not errors, errors[0]
    for p in procs:
        assert p.exitcode == 0
    model, inputs = _edge(m=500)
    data = np.asarray(inputs.data).copy()
    data[:, 250:] *= 0.9
    inputs = make_feature_batch(1024, data)
    single = engine.infer(model, inputs, InferenceConfig())
    for rank, cats, per_layer, vsum, moved in res:
        assert per_layer == [(o.active_before, o.active_after) for o in single.per_layer]
        if rank == 0:
            assert cats == single.categories.tolist()
            assert vsum == float(np.asarray(single.final.data, np.float64).sum())
        else:
            assert set(cats) < set(single.categories.tolist())
    assert res[0][2] == res[1][2] and res[0][4] == res[1][4]


def test_stress_matches_reference_run_batch_parallel(cuda_ok):
    """Skewed shards (C5 recipe) through DeviceShards + speculative windows:
    categories, per-layer totals, every BalanceEntry, the CommMatrix and the
    final values equal the reference's run_batch_parallel (stress.json)."""
    from test_parallel_host import _check_stress, _stress_cases, _stress_problem
    for case in _stress_cases():
        model, inputs, thr = _stress_problem(case)
        res, comm, bal = parallel.run_batch_parallel(
            model, inputs, InferenceConfig(workers=case["workers"], rebalance_threshold=thr))
        _check_stress(case, [(o.active_before, o.active_after) for o in res.per_layer],
                      comm, bal, res.categories.tolist(), np.asarray(res.final.data).T)


@pytest.mark.parametrize("poison", ["tiny", "nan"])
def test_guard_rewinds_windows(cuda_ok, poison):
    """Inputs that break the FMA form's exactness (subnormal-range values) or
    poison the union padding (NaN): the window is rewound and rerun in the
    exact form / unpadded plans, matching the single-worker engine."""
    model, inputs = _edge(m=300)
    data = np.asarray(inputs.data).copy()
    if poison == "tiny":
        data[:7, 200:220] = np.float32(3e-39)
    else:
        data[5, 150] = np.nan
    inputs = make_feature_batch(1024, data)
    cfg = InferenceConfig(workers=3, rebalance_threshold=1.05)
    res, comm, bal = parallel.run_batch_parallel(model, inputs, cfg)
    single = engine.infer(model, inputs, InferenceConfig())
    assert np.array_equal(res.categories, single.categories)
    assert np.array_equal(np.asarray(res.final.data).view(np.uint32),
                          np.asarray(single.final.data).view(np.uint32))
    ref = oracle.infer(model, inputs)
    assert res.categories.tolist() == ref.categories.tolist()


def test_randomized_batch_parallel_matches_single_worker():
    """Fuzz the in-process batch-parallel runner (2-8 workers, thresholds from
    1.01 (rebalance at any skew) to 4, skewed densities per shard): the merged
    result is the single-worker engine's, bit for bit, and the per-layer
    totals agree."""
    import os
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(int(os.environ.get("SPDNN_FUZZ_SEED", "99")))
    for case in range(int(os.environ.get("SPDNN_FUZZ_CASES", "8"))):
        n = int(rng.choice([256, 1024]))
        w = int(rng.integers(2, 9))
        L = int(rng.integers(3, 25))
        per = int(rng.integers(1, 300))
        model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
            neurons=n, layers=L, connections_per_neuron=min(n, 32),
            bias_value=float(rng.uniform(-0.45, -0.2)), seed=int(rng.integers(1 << 30))))
        dens = rng.uniform(0.15, 0.6, w)
        x = np.concatenate([(rng.random((n, per)) < d).astype(np.float32) for d in dens], axis=1)
        inputs = make_feature_batch(n, x)
        thr = float(rng.choice([1.01, 1.25, 2.0, 4.0]))
        res, comm, bal = parallel.run_batch_parallel(
            model, inputs, InferenceConfig(workers=w, rebalance_threshold=thr))
        single = engine.infer(model, inputs, InferenceConfig())
        msg = f"case {case}: n={n} w={w} L={L} per={per} thr={thr}"
        assert np.array_equal(res.categories, single.categories), msg
        assert [(o.active_before, o.active_after) for o in res.per_layer] == \
            [(o.active_before, o.active_after) for o in single.per_layer], msg
        assert np.array_equal(np.asarray(res.final.data).view(np.uint32),
                              np.asarray(single.final.data).view(np.uint32)), msg
        assert comm.total_moved == sum(e.moved_rows for e in bal.entries)
