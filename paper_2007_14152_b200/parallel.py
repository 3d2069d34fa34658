"""Batch-parallel inference across GPUs: the drop-in for ``spdnn.parallel``.

The reference (``spdnn/parallel.py``; the paper's Algorithm 2)
replicates the weights, gives every worker a contiguous range of input
features, and after every layer (1) exchanges the per-worker survivor counts
(an allgather), (2) if ``max/min > rebalance_threshold`` plans transfers with a
deterministic greedy rule, (3) moves each donor's highest-category features to
the receivers, and finally (4) gathers and sorts the categories on worker 0.

Here a worker is a GPU: one process per device under ``torch.distributed``
(NCCL over NVLink/NVSwitch for the counts and the feature rows), or -- when no
process group is initialised -- ``config.workers`` logical workers sharing the
current device inside one process (the reference's thread-per-worker layout;
used by the parity tests on one GPU). The host-side rules below are pure
functions and match the reference exactly:

* ``imbalance_ratio``  <- parallel.py:128-139
* ``partition_even``   <- parallel.py:142-158
* ``balance_step``     <- parallel.py:161-193
* ``apply_transfers``  <- parallel.py:196-235
* ``gather_categories``<- parallel.py:238-245
* ``run_batch_parallel`` <- parallel.py:379-454 (per-layer loop :294-376)

The layer step itself is the sm_100a kernel (engine.py / csrc/layer.cu); the
loop needs one device->host read of the survivor count per layer to drive the
exchange, as the reference's barrier does.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from .model import FeatureBatch, InferenceConfig, ModelError, NetworkModel, count_edges

TransferPlan = list  # [(source worker, dest worker, rows)]


# ---------------------------------------------------------------------------
# reports and messages (parallel.py:42-125)

@dataclass(frozen=True)
class Partition:
    shards: tuple

    @property
    def worker_count(self) -> int:
        return len(self.shards)

    def counts(self) -> list:
        return [s.active_count for s in self.shards]


@dataclass
class CommMatrix:
    """W x W counts of feature rows moved between workers while balancing."""

    matrix: np.ndarray

    @classmethod
    def zeros(cls, workers: int) -> "CommMatrix":
        return cls(np.zeros((workers, workers), dtype=np.int64))

    def add(self, delta: np.ndarray) -> None:
        self.matrix += delta

    @property
    def total_moved(self) -> int:
        return int(self.matrix.sum())

    def rows_sent(self) -> np.ndarray:
        return self.matrix.sum(axis=1)

    def rows_received(self) -> np.ndarray:
        return self.matrix.sum(axis=0)


@dataclass(frozen=True)
class BalanceEntry:
    layer: int
    before_counts: tuple
    after_counts: tuple
    imbalance_before: float
    imbalance_after: float
    moved_rows: int
    rebalanced: bool


@dataclass
class BalanceReport:
    entries: list = field(default_factory=list)

    @property
    def total_moved(self) -> int:
        return sum(e.moved_rows for e in self.entries)


@dataclass(frozen=True)
class CountMsg:
    src: int
    layer: int
    count: int


@dataclass(frozen=True)
class RowsMsg:
    src: int
    dst: int
    layer: int
    data: object        # (k, N) feature-major values (device or host tensor)
    categories: object  # (k,) int64


@dataclass(frozen=True)
class GatherMsg:
    src: int
    data: object
    categories: object


LatencyHook = Callable[[object], None]


# ---------------------------------------------------------------------------
# host-side rules

def imbalance_ratio(counts: Sequence[int]) -> float:
    """max/min shard size; empty-vs-nonempty is +inf, all-empty is 1."""
    counts = [int(c) for c in counts]
    if any(c < 0 for c in counts):
        raise ModelError("counts must be nonnegative")
    hi, lo = max(counts), min(counts)
    if hi == 0:
        return 1.0
    if lo == 0:
        return math.inf
    return hi / lo


def shard_bounds(m: int, workers: int) -> list:
    """[lo, hi) column range of each worker: sizes differ by <= 1, the first
    ``m % workers`` shards one larger (parallel.py:142-158)."""
    if workers < 1:
        raise ModelError("workers must be positive")
    base, rem = divmod(m, workers)
    out, start = [], 0
    for w in range(workers):
        size = base + (1 if w < rem else 0)
        out.append((start, start + size))
        start += size
    return out


def partition_even(features: FeatureBatch, workers: int) -> Partition:
    shards = []
    for lo, hi in shard_bounds(features.active_count, workers):
        shards.append(FeatureBatch(neurons=features.neurons,
                                   data=np.asfortranarray(features.data[:, lo:hi]),
                                   categories=features.categories[lo:hi],
                                   total_inputs=features.total_inputs))
    return Partition(shards=tuple(shards))


def balance_step(counts: Sequence[int]) -> TransferPlan:
    """Transfers that leave max - min <= 1 (parallel.py:161-193).

    Targets: the even split, the remainder granted to the currently largest
    shards (ties to the lower index). Then repeatedly pair the largest
    remaining surplus with the largest remaining deficit (ties to the lower
    index). Deterministic.
    """
    counts = [int(c) for c in counts]
    if any(c < 0 for c in counts):
        raise ModelError("counts must be nonnegative")
    w = len(counts)
    if w == 0:
        return []
    base, rem = divmod(sum(counts), w)
    bonus = set(sorted(range(w), key=lambda i: (-counts[i], i))[:rem])
    target = [base + (1 if i in bonus else 0) for i in range(w)]
    surplus = {i: counts[i] - target[i] for i in range(w) if counts[i] > target[i]}
    deficit = {i: target[i] - counts[i] for i in range(w) if counts[i] < target[i]}
    plan: TransferPlan = []
    while surplus:
        d = min(surplus, key=lambda i: (-surplus[i], i))
        r = min(deficit, key=lambda i: (-deficit[i], i))
        k = min(surplus[d], deficit[r])
        plan.append((d, r, k))
        surplus[d] -= k
        deficit[r] -= k
        if surplus[d] == 0:
            del surplus[d]
        if deficit[r] == 0:
            del deficit[r]
    return plan


def apply_transfers(plan: TransferPlan, partition: Partition):
    """Host-side transfer on FeatureBatches (parallel.py:196-235): donors give
    their highest-category columns, in plan order; receivers re-sort."""
    w = partition.worker_count
    datas = [s.data for s in partition.shards]
    cats = [s.categories for s in partition.shards]
    pending = [[] for _ in range(w)]
    delta = np.zeros((w, w), dtype=np.int64)
    for src, dst, k in plan:
        if not (0 <= src < w and 0 <= dst < w) or k < 0:
            raise ModelError("transfer plan does not fit this partition")
        if k > datas[src].shape[1]:
            raise ModelError("transfer plan exceeds donor size")
        if k == 0:
            continue
        cut = datas[src].shape[1] - k
        pending[dst].append((datas[src][:, cut:], cats[src][cut:]))
        datas[src], cats[src] = datas[src][:, :cut], cats[src][:cut]
        delta[src, dst] += k
    shards = []
    for i, shard in enumerate(partition.shards):
        data, cat = datas[i], cats[i]
        if pending[i]:
            data = np.concatenate([data] + [d for d, _ in pending[i]], axis=1)
            cat = np.concatenate([cat] + [c for _, c in pending[i]])
            order = np.argsort(cat, kind="stable")
            data, cat = data[:, order], cat[order]
        shards.append(FeatureBatch(neurons=shard.neurons, data=np.asfortranarray(data),
                                   categories=cat, total_inputs=shard.total_inputs))
    return Partition(shards=tuple(shards)), delta


def gather_categories(partition: Partition) -> list:
    merged = (np.concatenate([s.categories for s in partition.shards])
              if partition.shards else np.empty(0, dtype=np.int64))
    merged = np.sort(merged)
    if merged.size > 1 and (merged[1:] == merged[:-1]).any():
        raise ModelError("duplicate category across shards")
    return [int(c) for c in merged]


# ---------------------------------------------------------------------------
# workers

class DeviceShard:
    """One worker's features on a GPU: the engine's workspace plus the
    operations the exchange needs (count, take highest categories, append)."""

    def __init__(self, net, neurons: int, m_cap: int, num_layers: int):
        from . import engine
        self.engine = engine
        self.net = net
        self.n = neurons
        # receivers append after the columns in use: room for two full shards
        self.ws = engine.Workspace(neurons, 2 * max(m_cap, 1), num_layers,
                                   net.bias.device)
        self.cur = 0     # buffer holding the current active features
        self.m = 0       # active features (host mirror of the device count)
        self.used = 0    # columns of ws.y[cur] in use (appends go after them)

    def load(self, x_rows, categories) -> None:
        """x_rows: (M, N) feature-major host or device tensor."""
        self.engine.stage_inputs(self.ws, x_rows, categories, self.net)
        self.cur, self.m, self.used = 0, int(x_rows.shape[0]), int(x_rows.shape[0])

    def step(self, l: int, fma: bool | None = None) -> None:
        """Enqueue layer l on the current stream (engine.run_layers, one layer)."""
        import ctypes
        from . import _native
        e, ws = self.engine, self.ws
        i, o = self.cur, self.cur ^ 1
        ws.counts[l] = self.m
        ws.counts[l + 1] = 0
        ws.work[l] = 0
        opts = e.run_opts(self.net, fma)
        _native.check(_native.lib().spdnn_layer_forward(
            ctypes.byref(self.net.layer_devs[l]), e._dptr(self.net.bias), e._dptr(ws.y[i]),
            e._dptr(ws.y[o]), ws.ld, e._dptr(ws.a[i]), e._dptr(ws.cat[i]),
            ctypes.c_void_p(ws.counts.data_ptr() + 4 * l), e._dptr(ws.a[o]), e._dptr(ws.cat[o]),
            ctypes.c_void_p(ws.counts.data_ptr() + 4 * (l + 1)), ctypes.byref(ws.scratch),
            ctypes.c_void_p(ws.work.data_ptr() + 4 * l), ctypes.byref(opts),
            e._stream_ptr(e._torch())), "spdnn_layer_forward")
        self.used = self.m  # the output columns 0..m-1 of buffer o
        self.cur = o
        self.pending_layer = l

    def sync_count(self) -> int:
        self.m = int(self.ws.counts[self.pending_layer + 1].item())
        return self.m

    def take_top(self, k: int):
        """Remove the k highest-category active features; returns their values
        ((k, N) feature-major) and categories, highest last."""
        torch = self.engine._torch()
        ws, c = self.ws, self.cur
        cats = ws.cat[c][: self.m]
        top = torch.topk(cats, k, largest=True, sorted=True).indices.flip(0)
        vals = torch.empty((k, self.n), dtype=torch.float32, device=cats.device)
        self.engine._native.check(self.engine._native.lib().spdnn_gather_out(
            self.engine._dptr(ws.y[c]), self.n, ws.ld, self.engine._dptr(ws.a[c]),
            self.engine._dptr(top), k, self.engine._dptr(vals),
            self.engine._stream_ptr(torch)), "spdnn_gather_out")
        sent_cats = cats[top].clone()
        keep = torch.ones(self.m, dtype=torch.bool, device=cats.device)
        keep[top] = False
        a_keep, c_keep = ws.a[c][: self.m][keep], cats[keep]
        self.m -= k
        ws.a[c][: self.m].copy_(a_keep)
        ws.cat[c][: self.m].copy_(c_keep)
        return vals, sent_cats

    def append(self, vals, cats) -> None:
        """Add k features ((k, N) values + categories) after the used columns."""
        torch = self.engine._torch()
        k = int(vals.shape[0])
        if k == 0:
            return
        ws, c = self.ws, self.cur
        base = self.used
        if base + k > ws.ld:
            raise ModelError("shard capacity exceeded while rebalancing")
        vals = vals.to(ws.y[c].device).contiguous()
        ptr = ws.y[c].data_ptr() + 4 * base
        import ctypes
        self.engine._native.check(self.engine._native.lib().spdnn_transpose_in(
            self.engine._dptr(vals), self.n, k, ctypes.c_void_p(ptr), ws.ld, None, 0.0, 3.0e38,
            self.engine._stream_ptr(torch)), "spdnn_transpose_in")
        ws.a[c][self.m: self.m + k] = torch.arange(base, base + k, dtype=torch.int32,
                                                  device=ws.a[c].device)
        ws.cat[c][self.m: self.m + k] = cats.to(ws.cat[c].device)
        self.m += k
        self.used = base + k

    def final(self, values: bool = True):
        """(categories, values (S, N)) of the active features, any order."""
        torch = self.engine._torch()
        ws, c = self.ws, self.cur
        cats = ws.cat[c][: self.m].clone()
        vals = None
        if values:
            vals = torch.empty((self.m, self.n), dtype=torch.float32, device=cats.device)
            self.engine._native.check(self.engine._native.lib().spdnn_gather_out(
                self.engine._dptr(ws.y[c]), self.n, ws.ld, self.engine._dptr(ws.a[c]), None,
                self.m, self.engine._dptr(vals), self.engine._stream_ptr(torch)),
                "spdnn_gather_out")
        return cats, vals


# ---------------------------------------------------------------------------
# transports

class LocalTransport:
    """All workers in this process (the reference's threads; one GPU)."""

    def __init__(self, workers: int, hook: LatencyHook | None):
        self.workers = workers
        self.hook = hook
        self.local = list(range(workers))
        self.root = True

    def allgather_counts(self, layer: int, mine: dict) -> list:
        if self.hook is not None:
            for w in self.local:
                for other in range(self.workers):
                    if other != w:
                        self.hook(CountMsg(src=w, layer=layer, count=mine[w]))
        return [mine[w] for w in range(self.workers)]

    def exchange(self, layer: int, plan: TransferPlan, shards: dict) -> None:
        incoming = {w: [] for w in range(self.workers)}
        for src, dst, k in plan:
            if k == 0:
                continue
            vals, cats = shards[src].take_top(k)
            msg = RowsMsg(src=src, dst=dst, layer=layer, data=vals, categories=cats)
            if self.hook is not None:
                self.hook(msg)
            incoming[dst].append(msg)
        for dst, msgs in incoming.items():
            for msg in msgs:
                shards[dst].append(msg.data, msg.categories)

    def gather(self, shards: dict, values: bool):
        parts = [shards[w].final(values) for w in range(self.workers)]
        if self.hook is not None:
            for w in range(1, self.workers):
                self.hook(GatherMsg(src=w, data=parts[w][1], categories=parts[w][0]))
        return parts


class DistTransport:
    """One worker per process: torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, hook: LatencyHook | None, device):
        import torch.distributed as dist
        self.dist = dist
        self.workers = dist.get_world_size()
        self.rank = dist.get_rank()
        self.local = [self.rank]
        self.root = self.rank == 0
        self.hook = hook
        self.device = device
        # NCCL moves device tensors; gloo (CPU tests, or several ranks sharing
        # one GPU) moves host copies
        self.wire = device if dist.get_backend() == "nccl" else None

    def _wire(self, t):
        return t if self.wire is not None else t.cpu()

    def _empty(self, shape, dtype):
        import torch
        return torch.empty(shape, dtype=dtype,
                           device=self.device if self.wire is not None else "cpu")

    def allgather_counts(self, layer: int, mine: dict) -> list:
        import torch
        t = self._wire(torch.tensor([mine[self.rank]], dtype=torch.int64, device=self.device))
        out = [self._empty(1, torch.int64) for _ in range(self.workers)]
        self.dist.all_gather(out, t)  # NCCL allgather on GPUs (gloo on CPU)
        if self.hook is not None:
            for other in range(self.workers):
                if other != self.rank:
                    self.hook(CountMsg(src=self.rank, layer=layer, count=mine[self.rank]))
        return [int(v.item()) for v in out]

    def exchange(self, layer: int, plan: TransferPlan, shards: dict) -> None:
        import torch
        me = shards[self.rank]
        ops, recv = [], []
        for src, dst, k in plan:
            if k == 0:
                continue
            if src == self.rank:
                vals, cats = me.take_top(k)
                if self.hook is not None:
                    self.hook(RowsMsg(src=src, dst=dst, layer=layer, data=vals, categories=cats))
                ops.append(self.dist.P2POp(self.dist.isend, self._wire(vals.contiguous()), dst))
                ops.append(self.dist.P2POp(self.dist.isend, self._wire(cats.contiguous()), dst))
            elif dst == self.rank:
                vals = self._empty((k, me.n), torch.float32)
                cats = self._empty(k, torch.int64)
                ops.append(self.dist.P2POp(self.dist.irecv, vals, src))
                ops.append(self.dist.P2POp(self.dist.irecv, cats, src))
                recv.append((vals, cats))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        for vals, cats in recv:
            me.append(vals, cats)

    def gather(self, shards: dict, values: bool):
        """Every rank gets every worker's (categories, values)."""
        import torch
        cats, vals = shards[self.rank].final(values)
        counts = self.allgather_counts(-1, {self.rank: int(cats.shape[0])})
        n = shards[self.rank].n
        parts = []
        for w in range(self.workers):
            c = self._wire(cats) if w == self.rank else self._empty(counts[w], torch.int64)
            self.dist.broadcast(c, src=w)
            v = None
            if values:
                v = self._wire(vals) if w == self.rank else self._empty((counts[w], n),
                                                                         torch.float32)
                self.dist.broadcast(v, src=w)
            parts.append((c, v))
        return parts


# ---------------------------------------------------------------------------
# the runner

def run_layers_parallel(num_layers: int, shards: dict, transport, threshold: float,
                        workers: int, step=None, values: bool = True):
    """Per-layer loop of parallel.py:294-376 over any shard/transport pair.

    ``step(shard, l)`` runs layer l on one shard and returns its new count
    (default: the device kernel + one count read). Returns (per-layer
    outcomes as (before_total, after_total) pairs, CommMatrix, BalanceReport,
    gathered parts).
    """
    comm = CommMatrix.zeros(workers)
    balance = BalanceReport()
    totals = []
    before = sum(transport.allgather_counts(-1, {w: shards[w].m for w in transport.local}))
    for l in range(num_layers):
        if before == 0:
            totals.append((0, 0))
            continue
        mine = {}
        for w in transport.local:
            if step is None:
                shards[w].step(l)
        for w in transport.local:
            mine[w] = shards[w].sync_count() if step is None else step(shards[w], l)
        counts = transport.allgather_counts(l, mine)
        totals.append((before, sum(counts)))
        ratio = imbalance_ratio(counts)
        plan = balance_step(counts) if ratio > threshold else []
        if plan:
            transport.exchange(l, plan, shards)
        after = list(counts)
        delta = np.zeros((workers, workers), dtype=np.int64)
        for src, dst, k in plan:
            after[src] -= k
            after[dst] += k
            delta[src, dst] += k
        comm.add(delta)
        balance.entries.append(BalanceEntry(
            layer=l, before_counts=tuple(counts), after_counts=tuple(after),
            imbalance_before=ratio, imbalance_after=imbalance_ratio(after),
            moved_rows=sum(k for _, _, k in plan), rebalanced=bool(plan)))
        before = sum(counts)
        if before == 0:
            totals.extend([(0, 0)] * (num_layers - l - 1))
            break
    parts = transport.gather(shards, values)
    return totals, comm, balance, parts


def run_batch_parallel(model: NetworkModel, inputs: FeatureBatch, config: InferenceConfig,
                       mode: str = "optimized", prepared=None,
                       latency_hook: LatencyHook | None = None, values: bool = True):
    """Inference across ``config.workers`` shards with per-layer balancing
    (parallel.py:379-454). Returns (InferenceResult, CommMatrix, BalanceReport);
    under torch.distributed every rank returns the same merged result."""
    import torch
    from . import engine

    if inputs.neurons != model.neurons:
        raise ModelError("inputs do not match model width")
    if mode not in ("baseline", "optimized"):
        raise ModelError(f"unknown mode {mode!r}")
    if prepared is None:
        prepared = engine.prepare_model(model, config, mode)
    engine._check_prepared(prepared, model, mode)
    distributed = torch.distributed.is_available() and torch.distributed.is_initialized()
    w = torch.distributed.get_world_size() if distributed else config.workers
    if distributed and w != config.workers:
        raise ModelError(f"config.workers={config.workers} but world size is {w}")
    dev = torch.device("cuda", torch.cuda.current_device())
    net = engine.device_network(prepared, model.bias)
    bounds = shard_bounds(inputs.active_count, w)
    m_cap = max((hi - lo for lo, hi in bounds), default=0)
    transport = DistTransport(latency_hook, dev) if distributed else \
        LocalTransport(w, latency_hook)
    shards = {}
    for r in transport.local:
        lo, hi = bounds[r]
        sh = DeviceShard(net, model.neurons, m_cap, model.num_layers)
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(inputs.data)[:, lo:hi].T))
        sh.load(x, torch.from_numpy(np.ascontiguousarray(inputs.categories[lo:hi])))
        shards[r] = sh
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    totals, comm, balance, parts = run_layers_parallel(
        model.num_layers, shards, transport, config.rebalance_threshold, w, values=values)
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    cats = torch.cat([p[0] for p in parts]).cpu().numpy().astype(np.int64)
    order = np.argsort(cats, kind="stable")
    cats = cats[order]
    if cats.size > 1 and (cats[1:] == cats[:-1]).any():
        raise ModelError("duplicate category across shards")
    final = None
    if values:
        vals = torch.cat([p[1] for p in parts]).cpu().numpy()[order]
        final = FeatureBatch(neurons=model.neurons, data=vals.T, categories=cats,
                             total_inputs=inputs.total_inputs)
    per_layer = []
    for l, (before, after) in enumerate(totals):
        if before == 0:
            per_layer.append(engine.LayerOutcome(0, 0, 0, 0))
            continue
        per_layer.append(engine.LayerOutcome(
            active_before=before, active_after=after,
            weight_element_reads=net.total_slots[l] * -(-before // engine.TILE),
            feature_element_reads=net.num_fp[l] * before))
    result = engine.InferenceResult(final=final, categories=cats.copy(), per_layer=per_layer,
                                    elapsed_seconds=elapsed,
                                    edges_processed=inputs.total_inputs * count_edges(model))
    return result, comm, balance
