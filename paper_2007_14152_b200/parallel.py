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

The layer step itself is the sm_100a kernel (engine.py / csrc/layer.cu). The
reference's per-layer barrier becomes a speculative window of layers with one
count allgather and one host read per window (run_layers_parallel), rewound
and replayed up to the layer where the reference would rebalance.
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
    operations the runner and the exchange need.

    Layers run in speculative *windows* (see run_layers_parallel): the state
    at the start of a window stays untouched in its buffer (the checkpoint)
    while the window's layers rotate through two other buffers, so a window
    can be rewound and replayed without copying any feature data. A second,
    speculative window may be enqueued from the first one's (not yet
    checked) final state while the host waits for the first window's counts;
    it rotates through the two buffers that are neither checkpoint.
    """

    BUFFERS = 4
    supports_speculation = True

    def __init__(self, net, neurons: int, m_cap: int, num_layers: int, unpadded=None):
        from . import engine
        self.engine = engine
        self.net = net
        self.n = neurons
        self.num_layers = num_layers
        self.unpadded = unpadded  # () -> DeviceNetwork without zero-weight slots
        # receivers append after the columns in use: room for two full shards
        self.ws = engine.Workspace(neurons, 2 * max(m_cap, 1), num_layers,
                                   net.bias.device, buffers=self.BUFFERS)
        self.cur = 0     # buffer holding the current active features
        self.m = 0       # active features (host mirror of the device count)
        self.used = 0    # columns of ws.y[cur] in use (appends go after them)
        self.fma = None  # None: the network's default form; False: exact form
        self.unpadded_active = False
        self._win = None
        self._spec = None

    def load(self, x_rows, categories) -> None:
        """x_rows: (M, N) feature-major host or device tensor. Resets the
        guard flags (stage_inputs screens the inputs for the FMA form)."""
        self.engine.stage_inputs(self.ws, x_rows, categories, self.net)
        self.cur, self.m, self.used = 0, int(x_rows.shape[0]), int(x_rows.shape[0])
        self.fma = None

    # -- windows ----------------------------------------------------------
    def begin_window(self, l0: int, k: int) -> None:
        """Enqueue layers l0..l0+k-1 from the current state (no host sync)."""
        self._spec = None
        self._win = dict(l0=l0, k=k, start=self.cur, m=self.m, used=self.used)
        self._win["final"] = self._enqueue(l0, k, self.cur, set_m=True, avoid=None)
        self._win["counts"] = self._snapshot(l0, k)

    def begin_speculative(self, l0: int, k: int) -> None:
        """Enqueue layers l0..l0+k-1 from the current window's final state
        before its counts are known (they are produced on the device)."""
        w = self._win
        spec = dict(l0=l0, k=k, start=w["final"])
        spec["final"] = self._enqueue(l0, k, w["final"], set_m=False, avoid=w["start"])
        spec["counts"] = self._snapshot(l0, k)
        self._spec = spec

    def drop_speculative(self) -> None:
        """Forget the speculative window (later work overwrites its buffers)."""
        self._spec = None

    def promote_speculative(self) -> None:
        """After commit(): the speculative window, started from the committed
        state, becomes the current window."""
        spec = self._spec
        assert spec is not None and spec["start"] == self.cur
        spec.update(m=self.m, used=self.used)
        self._win, self._spec = spec, None

    def _enqueue(self, l0: int, k: int, ck: int, set_m: bool, avoid) -> int:
        import ctypes
        from . import _native
        e, ws, net = self.engine, self.ws, self.net
        if set_m:
            ws.counts[l0] = self.m
        ws.counts[l0 + 1: l0 + k + 1].zero_()
        ws.work[l0: l0 + k].zero_()
        opts = e.run_opts(net, self.fma)
        stream = e._stream_ptr(e._torch())
        cnt = ws.counts.data_ptr()
        o1, o2 = [b for b in range(self.BUFFERS) if b != ck and b != avoid][:2]
        _native.check(_native.lib().spdnn_layer_forward(
            ctypes.byref(net.layer_devs[l0]), e._dptr(net.bias), e._dptr(ws.y[ck]),
            e._dptr(ws.y[o1]), ws.ld, e._dptr(ws.a[ck]), e._dptr(ws.cat[ck]),
            ctypes.c_void_p(cnt + 4 * l0), e._dptr(ws.a[o1]), e._dptr(ws.cat[o1]),
            ctypes.c_void_p(cnt + 4 * (l0 + 1)), ctypes.byref(ws.scratch),
            ctypes.c_void_p(ws.work.data_ptr() + 4 * l0), ctypes.byref(opts), stream),
            "spdnn_layer_forward")
        if k > 1:
            # the rest of the window ping-pongs o1 <-> o2 inside one C call
            sc = _native.Scratch(ws.tile_done.data_ptr(), ws.tile_alive.data_ptr(),
                                 ws.work.data_ptr() + 4 * (l0 + 1), ws.guard.data_ptr())
            devs = ctypes.c_void_p(ctypes.addressof(net.layer_devs)
                                   + ctypes.sizeof(_native.LayerDev) * (l0 + 1))
            _native.check(_native.lib().spdnn_infer_layers(
                k - 1, devs, e._dptr(net.bias), e._dptr(ws.y[o1]), e._dptr(ws.y[o2]), ws.ld,
                e._dptr(ws.a[o1]), e._dptr(ws.a[o2]), e._dptr(ws.cat[o1]), e._dptr(ws.cat[o2]),
                ctypes.c_void_p(cnt + 4 * (l0 + 1)), ctypes.byref(sc), ctypes.byref(opts),
                stream), "spdnn_infer_layers")
        return o1 if (k - 1) % 2 == 0 else o2

    def _snapshot(self, l0: int, k: int):
        """The window's counts and the guard word, copied on the stream right
        after its last layer (a later speculative window cannot leak in), and
        an event the transport waits on instead of the whole stream."""
        torch = self.engine._torch()
        t = torch.cat([self.ws.counts[l0 + 1: l0 + k + 1], self.ws.guard]).to(torch.int64)
        ev = torch.cuda.Event()
        ev.record()
        return t, ev

    def window_counts(self):
        """Device int64 [active after each window layer..., guard bits]."""
        return self._win["counts"][0]

    def window_event(self):
        return self._win["counts"][1]

    def rewind(self) -> None:
        """Back to the window's starting state (its buffer was never written)."""
        w = self._win
        self._spec = None
        self.cur, self.m, self.used = w["start"], w["m"], w["used"]

    def replay(self, k: int) -> None:
        """Rewind and run only the first k layers of the window."""
        l0 = self._win["l0"]
        self.rewind()
        self.begin_window(l0, k)

    def commit(self, m_last_in: int, m: int) -> None:
        """Accept the window: its last output becomes the current state. The
        kernel writes a feature's outputs at its input position, so the
        columns in use are those of the last layer's input."""
        self.cur = self._win["final"]
        self.m, self.used = int(m), int(m_last_in)
        self._win = None

    def set_exact(self, unpadded: bool) -> None:
        """Switch to the exact arithmetic form (guard fired); with non-finite
        inputs also to plans without zero-weight union slots."""
        self.fma = False
        if unpadded:
            if self.unpadded is None:
                raise ModelError("non-finite inputs need the unpadded plans")
            self.net = self.unpadded()
            self.unpadded_active = True

    @property
    def uses_fma(self) -> bool:
        return bool(self.engine.run_opts(self.net, self.fma).fma_form)

    def take_top(self, k: int):
        """Remove the k highest-category active features; returns their values
        ((k, N) feature-major) and categories, highest last. Device-side only
        (a stable sort and gathers, no host synchronisation); the kept
        features keep their relative order."""
        torch = self.engine._torch()
        ws, c = self.ws, self.cur
        cats = ws.cat[c][: self.m]
        order = torch.argsort(cats, stable=True)
        top = order[self.m - k:]
        keep = torch.sort(order[: self.m - k]).values
        vals = torch.empty((k, self.n), dtype=torch.float32, device=cats.device)
        self.engine._native.check(self.engine._native.lib().spdnn_gather_out(
            self.engine._dptr(ws.y[c]), self.n, ws.ld, self.engine._dptr(ws.a[c]),
            self.engine._dptr(top), k, self.engine._dptr(vals),
            self.engine._stream_ptr(torch)), "spdnn_gather_out")
        sent_cats = cats[top]
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

_SIDE = {}


def _side_stream(torch):
    """A per-device side stream for the window count reads."""
    dev = torch.cuda.current_device()
    if dev not in _SIDE:
        _SIDE[dev] = torch.cuda.Stream()
    return _SIDE[dev]


class _nullcontext:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False

class LocalTransport:
    """All workers in this process (the reference's threads; one GPU)."""

    def __init__(self, workers: int, hook: LatencyHook | None):
        self.workers = workers
        self.hook = hook
        self.local = list(range(workers))
        self.root = True

    def allgather_counts(self, layer: int, mine: dict, notify: bool = True) -> list:
        if self.hook is not None and notify:
            for w in self.local:
                for other in range(self.workers):
                    if other != w:
                        self.hook(CountMsg(src=w, layer=layer, count=mine[w]))
        return [mine[w] for w in range(self.workers)]

    def allgather_window(self, mine: dict, events: dict | None = None) -> np.ndarray:
        """(workers, k+1) host array of every worker's window counts + guard.
        With `events`, the copy waits for those only (on a side stream), not
        for a speculative window enqueued after them."""
        import torch
        if not events:
            return torch.stack([mine[w] for w in range(self.workers)]).cpu().numpy()
        side = _side_stream(torch)
        for ev in events.values():
            side.wait_event(ev)
        with torch.cuda.stream(side):
            return torch.stack([mine[w] for w in range(self.workers)]).cpu().numpy()

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

    def allgather_counts(self, layer: int, mine: dict, notify: bool = True) -> list:
        """One count per rank to every rank (NCCL allgather on GPUs, gloo on
        CPU). `notify` = False for the exchanges the reference has no message
        for (the initial counts, the gather sizes): the latency hook sees the
        reference's message stream only (parallel.py:306-318)."""
        import torch
        t = self._wire(torch.tensor([mine[self.rank]], dtype=torch.int64, device=self.device))
        out = [self._empty(1, torch.int64) for _ in range(self.workers)]
        self.dist.all_gather(out, t)
        if self.hook is not None and notify:
            for other in range(self.workers):
                if other != self.rank:
                    self.hook(CountMsg(src=self.rank, layer=layer, count=mine[self.rank]))
        return [int(v.item()) for v in out]

    def allgather_window(self, mine: dict, events: dict | None = None) -> np.ndarray:
        """One allgather of the window's counts (device-resident under NCCL)
        and one host read for the whole window. With `events` it runs on a
        side stream that waits for this rank's window only, so a speculative
        window already enqueued keeps the GPU busy meanwhile."""
        import torch
        ctx = None
        if events:
            side = _side_stream(torch)
            for ev in events.values():
                side.wait_event(ev)
            ctx = torch.cuda.stream(side)
        with (ctx if ctx is not None else _nullcontext()):
            t = self._wire(mine[self.rank].contiguous())
            out = [self._empty(t.shape[0], torch.int64) for _ in range(self.workers)]
            self.dist.all_gather(out, t)
            return torch.stack(out).cpu().numpy()

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
        """Algorithm 2's final step (parallel.py:417-433): every
        worker sends its survivors' categories (and values when asked) to
        rank 0, which merges them. Rank 0 returns every worker's part; the
        other ranks return their own part only."""
        import torch
        cats, vals = shards[self.rank].final(values)
        counts = self.allgather_counts(-1, {self.rank: int(cats.shape[0])}, notify=False)
        n = shards[self.rank].n
        if self.rank != 0:
            if self.hook is not None:
                self.hook(GatherMsg(src=self.rank, data=vals, categories=cats))
            ops = []
            if counts[self.rank]:
                ops.append(self.dist.P2POp(self.dist.isend, self._wire(cats.contiguous()), 0))
                if values:
                    ops.append(self.dist.P2POp(self.dist.isend, self._wire(vals.contiguous()), 0))
            if ops:
                for req in self.dist.batch_isend_irecv(ops):
                    req.wait()
            return [(cats, vals)]
        parts = [(self._wire(cats), self._wire(vals) if values else None)]
        ops = []
        for w in range(1, self.workers):
            c = self._empty(counts[w], torch.int64)
            v = self._empty((counts[w], n), torch.float32) if values else None
            if counts[w]:
                ops.append(self.dist.P2POp(self.dist.irecv, c, w))
                if values:
                    ops.append(self.dist.P2POp(self.dist.irecv, v, w))
            parts.append((c, v))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        return parts


# ---------------------------------------------------------------------------
# the runner

WINDOW_MIN = 4
WINDOW_MAX = int(__import__("os").environ.get("SPDNN_WINDOW_MAX", "64"))
# enqueue the next window before reading this one's counts (DeviceShard)
SPECULATE = __import__("os").environ.get("SPDNN_SPECULATE", "1") == "1"


def run_layers_parallel(num_layers: int, shards: dict, transport, threshold: float,
                        workers: int, values: bool = True, window: int | None = None):
    """Per-layer loop of parallel.py:294-376 over any shard/transport pair.

    The reference synchronises every worker after every layer to exchange
    survivor counts. Here the layers run in speculative windows of k layers
    with no host synchronisation inside: each shard enqueues k layers, one
    allgather moves all k counts (plus the arithmetic guard bits), and the
    host then replays the reference's per-layer decisions over them. If layer
    j of the window would have triggered a rebalance (or the all-dead stop),
    every shard rewinds to the window's start and runs only layers ..j, then
    the exchange happens exactly where the reference does it. Windows grow
    from WINDOW_MIN to WINDOW_MAX while no rebalance occurs. The per-layer
    counts, transfer plans, CommMatrix and BalanceReport are therefore those
    of the per-layer loop.

    A guard bit (FMA-form underflow risk or non-finite inputs, see engine)
    on any worker rewinds the window and reruns it in the exact form.

    Returns (per-layer (before_total, after_total) pairs, CommMatrix,
    BalanceReport, gathered parts).
    """
    comm = CommMatrix.zeros(workers)
    balance = BalanceReport()
    totals = []
    hook = transport.hook
    local = transport.local
    before = sum(transport.allgather_counts(-1, {w: shards[w].m for w in local}, notify=False))
    k_max = max(1, window or WINDOW_MAX)
    k_cur = min(WINDOW_MIN, k_max)
    speculate = SPECULATE and all(getattr(shards[w], "supports_speculation", False)
                                  for w in local)
    current = False  # a window (the promoted speculation) is already enqueued
    k = 0
    l = 0
    while l < num_layers:
        if before == 0:
            if current:
                for w in local:
                    shards[w].drop_speculative()
            totals.extend([(0, 0)] * (num_layers - l))
            break
        if not current:
            k = min(k_cur, num_layers - l)
            for w in local:
                shards[w].begin_window(l, k)
        current = False
        # the next window, enqueued from this one's unchecked final state: it
        # keeps the GPU busy while the host waits for this window's counts
        nk = min(2 * k_cur, k_max, num_layers - l - k) if speculate else 0
        if nk > 0:
            for w in local:
                shards[w].begin_speculative(l + k, nk)
        events = {w: shards[w].window_event() for w in local} if speculate else None
        hist = transport.allgather_window({w: shards[w].window_counts() for w in local},
                                          events)
        guard = int(np.bitwise_or.reduce(hist[:, k]))
        unpadded = bool(guard & 2)
        if (guard & 1 and any(shards[w].uses_fma for w in local)) or \
                (unpadded and not all(shards[w].unpadded_active for w in local)):
            for w in local:
                shards[w].rewind()
                shards[w].set_exact(unpadded)
            continue
        accept, plan = k, []
        for j in range(k):
            counts = [int(c) for c in hist[:, j]]
            if sum(counts) == 0:
                accept = j + 1
                break
            if imbalance_ratio(counts) > threshold:
                accept = j + 1
                break
        if accept < k:
            for w in local:
                shards[w].replay(accept)  # drops the speculative window
        for j in range(accept):
            counts = [int(c) for c in hist[:, j]]
            if hook is not None:
                for w in local:
                    for other in range(workers):
                        if other != w:
                            hook(CountMsg(src=w, layer=l + j, count=counts[w]))
            totals.append((before, sum(counts)))
            ratio = imbalance_ratio(counts)
            plan = balance_step(counts) if ratio > threshold else []
            after = list(counts)
            delta = np.zeros((workers, workers), dtype=np.int64)
            for src, dst, n in plan:
                after[src] -= n
                after[dst] += n
                delta[src, dst] += n
            comm.add(delta)
            balance.entries.append(BalanceEntry(
                layer=l + j, before_counts=tuple(counts), after_counts=tuple(after),
                imbalance_before=ratio, imbalance_after=imbalance_ratio(after),
                moved_rows=sum(n for _, _, n in plan), rebalanced=bool(plan)))
            before = sum(counts)
        for w in local:
            last_in = int(hist[w, accept - 2]) if accept > 1 else shards[w].m
            shards[w].commit(last_in, int(hist[w, accept - 1]))
        l += accept
        if plan:
            if nk > 0:
                for w in local:
                    shards[w].drop_speculative()
            transport.exchange(l - 1, plan, shards)
            k_cur = min(WINDOW_MIN, k_max)
        else:
            k_cur = min(2 * k_cur, k_max)
            if nk > 0 and accept == k and sum(int(c) for c in hist[:, k - 1]) > 0:
                for w in local:
                    shards[w].promote_speculative()
                current, k = True, nk
            elif nk > 0:
                for w in local:
                    shards[w].drop_speculative()
    parts = transport.gather(shards, values)
    return totals, comm, balance, parts


def run_batch_parallel(model: NetworkModel, inputs: FeatureBatch, config: InferenceConfig,
                       mode: str = "optimized", prepared=None,
                       latency_hook: LatencyHook | None = None, values: bool = True):
    """Inference across ``config.workers`` shards with per-layer balancing
    (parallel.py:379-454). Returns (InferenceResult, CommMatrix, BalanceReport).
    Under torch.distributed (one worker per rank) the survivors are gathered
    to rank 0 (Algorithm 2): rank 0's result holds the merged,
    sorted categories (and values); every other rank's holds its own shard's
    survivors. Per-layer counts, CommMatrix and BalanceReport are the same on
    every rank.""" 
    from . import engine

    if inputs.neurons != model.neurons:
        raise ModelError("inputs do not match model width")
    if mode not in ("baseline", "optimized"):
        raise ModelError(f"unknown mode {mode!r}")
    if prepared is None:
        prepared = engine.prepare_model(model, config, mode)
    engine._check_prepared(prepared, model, mode)
    net = engine.device_network(prepared, model.bias)
    cache = []

    def unpadded():
        if not cache:
            cache.append(engine.DeviceNetwork(engine._unpadded(prepared, model), model.bias))
        return cache[0]

    return run_batch_parallel_device(net, inputs, config, latency_hook=latency_hook,
                                     values=values, edges_per_input=count_edges(model),
                                     unpadded=unpadded)


def run_batch_parallel_device(net, inputs: FeatureBatch, config: InferenceConfig,
                              latency_hook: LatencyHook | None = None, values: bool = True,
                              edges_per_input: int | None = None, unpadded=None,
                              shard_only: bool = False):
    """run_batch_parallel on a network already resident in HBM (extension, the
    counterpart of engine.infer_device): e.g. one built chunk by chunk with
    DeviceNetwork.from_layers. ``shard_only`` (torch.distributed only): the
    batch is the full 0..total_inputs-1 set and ``inputs`` holds just this
    rank's partition_even shard of it, so no rank materialises the rest."""
    import torch
    from . import engine

    if inputs.neurons != net.neurons:
        raise ModelError("inputs do not match model width")
    distributed = torch.distributed.is_available() and torch.distributed.is_initialized()
    w = torch.distributed.get_world_size() if distributed else config.workers
    if distributed and w != config.workers:
        raise ModelError(f"config.workers={config.workers} but world size is {w}")
    total = inputs.total_inputs
    if shard_only and not distributed:
        raise ModelError("shard_only needs a torch.distributed process group")
    bounds = shard_bounds(total if shard_only else inputs.active_count, w)
    m_cap = max((hi - lo for lo, hi in bounds), default=0)
    transport = DistTransport(latency_hook, net.bias.device) if distributed else \
        LocalTransport(w, latency_hook)
    shards = {}
    data = np.asarray(inputs.data)
    for r in transport.local:
        lo, hi = bounds[r]
        cols = slice(lo, hi)
        if shard_only:
            if inputs.active_count != hi - lo or (hi > lo and (
                    inputs.categories[0] != lo or inputs.categories[-1] != hi - 1)):
                raise ModelError("inputs are not this rank's shard of the batch")
            cols = slice(0, hi - lo)
        sh = DeviceShard(net, net.neurons, m_cap, net.num_layers, unpadded=unpadded)
        x = engine.host_tensor(np.ascontiguousarray(data[:, cols].T))
        sh.load(x, engine.host_tensor(np.ascontiguousarray(inputs.categories[cols])))
        shards[r] = sh
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record()
    totals, comm, balance, parts = run_layers_parallel(
        net.num_layers, shards, transport, config.rebalance_threshold, w, values=values)
    ev1.record()
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
        final = FeatureBatch(neurons=net.neurons, data=vals.T, categories=cats,
                             total_inputs=total)
    per_layer = []
    for l, (before, after) in enumerate(totals):
        if before == 0:
            per_layer.append(engine.LayerOutcome(0, 0, 0, 0))
            continue
        per_layer.append(engine.LayerOutcome(
            active_before=before, active_after=after,
            weight_element_reads=net.total_slots[l] * -(-before // engine.TILE),
            feature_element_reads=net.num_fp[l] * before))
    epi = edges_per_input if edges_per_input is not None else int(sum(net.nnz))
    result = engine.InferenceResult(final=final, categories=cats.copy(), per_layer=per_layer,
                                    elapsed_seconds=elapsed, edges_processed=total * epi,
                                    device_seconds=ev0.elapsed_time(ev1) / 1e3)
    return result, comm, balance
