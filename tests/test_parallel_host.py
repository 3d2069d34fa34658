"""Batch-parallel host logic on CPU: the balancing rules against the
reference's own outputs (tests/golden/balance.json) and test cases
(spdnn tests/test_parallel.py), and the per-layer exchange loop over a
world-size-2 gloo process group with oracle-backed shards."""

import json
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN
from host_shard import HostShard
from oracle import oracle
from paper_2007_14152_b200 import ingest
from paper_2007_14152_b200.model import ModelError, make_feature_batch
from paper_2007_14152_b200.parallel import (DistTransport, LocalTransport, Partition,
                                            apply_transfers, balance_step, gather_categories,
                                            imbalance_ratio, partition_even,
                                            run_layers_parallel, shard_bounds)


def test_balance_step_matches_reference_outputs():
    cases = json.load(open(os.path.join(GOLDEN, "balance.json")))
    for c in cases:
        assert [list(p) for p in balance_step(c["counts"])] == c["plan"], c["counts"]
        r = imbalance_ratio(c["counts"])
        assert (r == math.inf) if c["ratio"] == "inf" else r == c["ratio"]


def test_balance_step_properties():
    rng = np.random.default_rng(123)
    for _ in range(1000):
        counts = rng.integers(0, 50, size=int(rng.integers(1, 9))).tolist()
        after = list(counts)
        for src, dst, k in balance_step(counts):
            assert k > 0
            after[src] -= k
            after[dst] += k
        assert max(after) - min(after) <= 1 and min(after) >= 0
        moved = sum(k for _, _, k in balance_step(counts))
        assert moved == sum(max(0, b - a) for b, a in zip(counts, after))
    assert balance_step([5, 5, 5]) == []
    assert imbalance_ratio([249, 100]) == 2.49
    assert imbalance_ratio([5, 0]) == math.inf and imbalance_ratio([0, 0]) == 1.0
    with pytest.raises(ModelError):
        imbalance_ratio([-1, 3])


def _batch(n, m, cats=None, total=None):
    data = np.ones((n, m), dtype=np.float32)
    if total is None and cats is not None:
        total = max(cats, default=-1) + 1
    return make_feature_batch(n, data, categories=cats, total_inputs=total)


def test_partition_and_transfers_reference_cases():
    p = partition_even(_batch(2, 10), 3)
    assert p.counts() == [4, 3, 3]
    assert [s.categories.tolist() for s in p.shards] == [[0, 1, 2, 3], [4, 5, 6], [7, 8, 9]]
    assert set(partition_even(_batch(1, 60000), 42).counts()) == {1428, 1429}
    assert shard_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    part = Partition(shards=(_batch(2, 4, cats=[0, 1, 2, 3], total=5),
                             _batch(2, 1, cats=[4], total=5)))
    new, delta = apply_transfers([(0, 1, 2)], part)
    assert new.counts() == [2, 3] and delta[0, 1] == 2
    assert new.shards[0].categories.tolist() == [0, 1]
    assert new.shards[1].categories.tolist() == [2, 3, 4]
    with pytest.raises(ModelError, match="exceeds donor"):
        apply_transfers([(0, 1, 9)], part)
    dup = Partition(shards=(_batch(2, 1, cats=[2]), _batch(2, 1, cats=[2])))
    with pytest.raises(ModelError, match="duplicate"):
        gather_categories(dup)


def _problem():
    # die-off fixture of the reference (tests/test_parallel.py:178-197):
    # the second half of the columns is all zero and dies in layer 0
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=64, layers=4, connections_per_neuron=32, bias_value=-0.3, seed=3))
    data = np.ones((64, 60), dtype=np.float32)
    data[:, 30:] = 0.0
    return model, make_feature_batch(64, data)


def _shards(model, inputs, workers, ranks):
    out = {}
    for r in ranks:
        lo, hi = shard_bounds(inputs.active_count, workers)[r]
        out[r] = HostShard(model, inputs.data[:, lo:hi], inputs.categories[lo:hi])
    return out


def test_local_exchange_loop_rebalances():
    model, inputs = _problem()
    shards = _shards(model, inputs, 2, [0, 1])
    totals, comm, bal, parts = run_layers_parallel(
        model.num_layers, shards, LocalTransport(2, None), 1.25, 2)
    cats = np.sort(torch.cat([p[0] for p in parts]).numpy())
    ref = oracle.infer(model, inputs)
    assert cats.tolist() == ref.categories.tolist()
    assert [b for b, _ in totals] == ref.counts[:-1].tolist()
    rebalanced = [e for e in bal.entries if e.rebalanced]
    assert rebalanced and comm.matrix[0, 1] == rebalanced[0].moved_rows
    assert comm.total_moved == bal.total_moved


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model, inputs = _problem()
        shards = _shards(model, inputs, world, [rank])
        t = DistTransport(None, torch.device("cpu"))
        totals, comm, bal, parts = run_layers_parallel(
            model.num_layers, shards, t, 1.25, world)
        cats = np.sort(torch.cat([p[0] for p in parts]).numpy())
        vals = torch.cat([p[1] for p in parts]).numpy()
        q.put((rank, cats.tolist(), [b for b, _ in totals], comm.matrix.tolist(),
               [e.rebalanced for e in bal.entries], float(vals.sum())))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    model, inputs = _problem()
    ref = oracle.infer(model, inputs)
    for rank, cats, before, matrix, rebalanced, vsum in res:
        assert before == ref.counts[:-1].tolist()
        assert any(rebalanced) and matrix[0][1] > 0
        if rank == 0:  # categories gathered to rank 0 (Algorithm 2)
            assert cats == ref.categories.tolist()
            assert vsum == pytest.approx(float(np.asarray(ref.final).sum()))
        else:          # the other ranks keep their own shard's survivors
            assert 0 < len(cats) < len(ref.categories)
            assert set(cats) <= set(ref.categories.tolist())
    assert res[0][2:5] == res[1][2:5]  # same counts, CommMatrix, decisions everywhere
    assert len(res[0][1]) > len(res[1][1])


# ---------------------------------------------------------------------------
# skewed shards (config C5's recipe) against the reference's own
# run_batch_parallel (tests/golden/stress.json, made by make_stress.py)

def _stress_cases():
    return json.load(open(os.path.join(GOLDEN, "stress.json")))


def _stress_problem(case):
    n, w, cols, bias = case["neurons"], case["workers"], case["columns"], case["bias"]
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=n, layers=case["layers"], connections_per_neuron=32, bias_value=bias, seed=1))
    parts = [ingest.generate_synthetic_inputs(n, cols, abs(bias) + 0.04 - 0.01 * s,
                                              seed=100 + s) for s in range(w)]
    data = np.concatenate([np.asarray(p.data) for p in parts], axis=1)
    thr = math.inf if case["threshold"] == "inf" else case["threshold"]
    return model, make_feature_batch(n, data), thr


def _check_stress(case, totals, comm, bal, cats, final=None):
    assert cats == case["categories"]
    assert [list(t) for t in totals] == case["per_layer"]
    got = [[e.layer, list(e.before_counts), list(e.after_counts), e.moved_rows,
            bool(e.rebalanced)] for e in bal.entries]
    assert got == case["entries"]
    assert comm.matrix.tolist() == case["comm"]
    if final is not None:
        import hashlib
        assert hashlib.sha256(np.ascontiguousarray(final, dtype="<f4").tobytes()
                              ).hexdigest() == case["final_sha256"]


@pytest.mark.parametrize("window", [None, 1, 3])
def test_windowed_loop_matches_reference_stress(window):
    """The speculative-window runner reproduces the reference's per-layer
    decisions exactly (rebalances at the same layers, same plans) whatever
    the window length."""
    for case in _stress_cases():
        model, inputs, thr = _stress_problem(case)
        w = case["workers"]
        shards = _shards(model, inputs, w, list(range(w)))
        totals, comm, bal, parts = run_layers_parallel(
            model.num_layers, shards, LocalTransport(w, None), thr, w, window=window)
        cats = torch.cat([p[0] for p in parts]).numpy()
        vals = torch.cat([p[1] for p in parts]).numpy()
        order = np.argsort(cats, kind="stable")
        _check_stress(case, totals, comm, bal, cats[order].tolist(), vals[order])
        if window is None and bal.total_moved:
            # windows were rewound at the rebalancing layers and regrown after
            assert any(k > 4 for _, k in shards[0].windows)


def _gloo_stress_worker(rank, world, port, q, idx):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = _stress_cases()[idx]
        model, inputs, thr = _stress_problem(case)
        shards = _shards(model, inputs, world, [rank])
        t = DistTransport(None, torch.device("cpu"))
        totals, comm, bal, parts = run_layers_parallel(model.num_layers, shards, t, thr, world)
        cats = torch.cat([p[0] for p in parts]).numpy()
        vals = torch.cat([p[1] for p in parts]).numpy()
        order = np.argsort(cats, kind="stable")
        if rank == 0:
            _check_stress(case, totals, comm, bal, cats[order].tolist(), vals[order])
        else:
            _check_stress(case, totals, comm, bal, case["categories"])
            assert set(cats.tolist()) <= set(case["categories"])
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001 - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_3_stress():
    idx = next(i for i, c in enumerate(_stress_cases()) if c["workers"] == 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_stress_worker, args=(r, 3, port, q, idx))
             for r in range(3)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(3))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == [(0, "ok"), (1, "ok"), (2, "ok")]
