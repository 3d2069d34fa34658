"""Single-GPU inference engine: the drop-in for ``spdnn.engine``.

Public surface and semantics follow ``spdnn/engine.py`` (paths relative to
/root/reference/pkg/src/):

* ``prepare_model(model, config, mode)``  <- engine.py:88-90 (one-time layout
  conversion, here the C++ plan builder behind the C ABI);
* ``infer(model, inputs, config, mode, prepared)`` <- engine.py:235-290;
* ``optimized_layer`` / ``baseline_layer`` <- engine.py:93-127 (one layer,
  returns the dense (N, M) output and per-column activity);
* ``compact_active`` <- engine.py:130-142; ``run_layer_step`` <- :145-170;
* ``LayerOutcome`` / ``InferenceResult`` / ``PreparedLayer`` <- :41-74.

Both modes run the same sm_100a kernel (csrc/layer.cu). "optimized" uses
row-grouped union plans (R = 3 or 7 rows share every staged operand);
"baseline" uses one row per group (R = 1), i.e. each output row gathers only
its own columns -- the analogue of the reference's CSR baseline kernel. The
two produce bit-identical outputs, as in the reference (kernels.py:1-9).

Device data layout: features are neuron-major,
``Y[n][j]`` with the 128-feature tiles contiguous, so every staged input
neuron is one coalesced 512-byte row segment; dead features are dropped by
index lists that the layer kernel itself appends (no compaction pass).
"""

from __future__ import annotations

import ctypes
import threading
import time
from dataclasses import dataclass, field, replace
from typing import Literal, Sequence

import numpy as np

from . import _native
from .model import (FeatureBatch, InferenceConfig, LayerCSR, ModelError, NetworkModel,
                    count_edges)

Mode = Literal["baseline", "optimized"]
TILE = 128  # features per work item (include/spdnn_b200.h SPDNN_TILE_FEATURES)


# ---------------------------------------------------------------------------
# result types (engine.py:41-65)

@dataclass
class LayerOutcome:
    active_before: int
    active_after: int
    weight_element_reads: int
    feature_element_reads: int
    features: FeatureBatch | None = None

    def summary(self) -> "LayerOutcome":
        return replace(self, features=None)


@dataclass
class InferenceResult:
    final: FeatureBatch
    categories: np.ndarray  # sorted int64
    per_layer: list
    elapsed_seconds: float
    edges_processed: int
    device_seconds: float = 0.0   # CUDA-event time of the layer loop alone


# ---------------------------------------------------------------------------
# one-time layout conversion

@dataclass(frozen=True)
class PlanParams:
    """Kernel geometry knobs of the row-grouped union layout."""
    rows_per_group: int = 0      # 0 = cost model: 1, 3 or 7 (6 for mask layers >= 8192 rows)
    footprint_cap: int = 176     # staged input neurons per block stage (x512 B smem)
    max_groups: int = 20         # row groups per block (one per consumer warp)
    record_cap: int = 800        # union records per block stage
    reorder: bool = True
    uniform_records: bool = True  # one-word mask records when all weights are equal


BASELINE_PARAMS = PlanParams(rows_per_group=1, reorder=False)
OPTIMIZED_PARAMS = PlanParams()


@dataclass(frozen=True)
class PaddingStats:
    """Zero-padding cost of the layout (the reference's fields,
    spdnn/preprocess.py:115-131), measured on the row-grouped union layout:
    multiply-add slots executed per feature beyond the nonzeros if record
    runs were fixed per row group (what the layout stores: one consumer
    warp's unit), per block, or per layer. Overheads are padded slots / nnz."""
    nnz: int
    warp_padded_slots: int
    tile_padded_slots: int
    layer_padded_slots: int
    warp_overhead: float
    tile_overhead: float
    layer_overhead: float
    empty: bool = False

    @property
    def padded_slots(self) -> int:
        """Slots executed per feature: nnz + the group-level padding."""
        return self.nnz + self.warp_padded_slots

    @property
    def overhead(self) -> float:
        return self.warp_overhead


@dataclass(frozen=True)
class LayerPlan:
    """Host copy of one layer's device layout (include/spdnn_b200.h export)."""
    neurons: int
    rows_per_group: int
    record_words: int
    pow2: bool             # every nonzero weight is +-2^e: the FMA form applies
    wexp_min: int
    wexp_max: int
    num_blocks: int
    max_fp_per_stage: int
    max_records_per_stage: int
    max_meta_per_block: int
    max_groups_per_block: int
    num_records: int
    num_fp: int
    padded_slots: int
    uniform: bool          # one-word mask records; every connection weighs weight_bits
    weight_bits: int
    blocks: np.ndarray    # int32 [num_blocks, 8] descriptors
    stages: np.ndarray    # int32 [num_extra_stages, 4]
    meta: np.ndarray      # int32 per-block fp lists / group segments / rows
    records: np.ndarray   # uint32 [num_records * record_words]

    @property
    def total_slots(self) -> int:
        return self.padded_slots


@dataclass(frozen=True)
class PreparedLayer:
    """Execution-ready structures for one layer in one mode (engine.py:68-74)."""
    csr: LayerCSR
    plan: LayerPlan | None = None
    padding: PaddingStats | None = None
    mode: str = "optimized"


def _params_struct(p: PlanParams) -> _native.PlanParams:
    return _native.PlanParams(p.rows_per_group, p.footprint_cap, p.max_groups, p.record_cap,
                              int(p.reorder), int(p.uniform_records))


def _export(handle) -> LayerPlan:
    L = _native.lib()
    s = _native.PlanSizes()
    _native.check(L.spdnn_plan_sizes(handle, ctypes.byref(s)), "spdnn_plan_sizes")
    arrs = dict(
        blocks=np.zeros(s.num_blocks * 8, np.int32),
        stages=np.zeros(s.num_extra_stages * 4, np.int32),
        meta=np.zeros(s.num_meta, np.int32),
        records=np.zeros(s.num_records * s.record_words, np.uint32),
    )
    ptr = lambda a: ctypes.c_void_p(a.ctypes.data)
    _native.check(L.spdnn_plan_export(handle, ptr(arrs["blocks"]), ptr(arrs["stages"]),
                                      ptr(arrs["meta"]), ptr(arrs["records"])),
                  "spdnn_plan_export")
    return LayerPlan(neurons=s.neurons, rows_per_group=s.rows_per_group,
                     record_words=s.record_words, pow2=bool(s.pow2),
                     wexp_min=s.wexp_min, wexp_max=s.wexp_max,
                     num_blocks=s.num_blocks, max_fp_per_stage=s.max_fp_per_stage,
                     max_records_per_stage=s.max_records_per_stage,
                     max_meta_per_block=s.max_meta_per_block,
                     max_groups_per_block=s.max_groups_per_block,
                     num_records=s.num_records, num_fp=s.num_fp,
                     padded_slots=s.padded_slots, uniform=bool(s.uniform),
                     weight_bits=int(s.weight_bits), **arrs)


def _group_records(plan: LayerPlan) -> tuple:
    """(records of every row group, groups of every block) from the exported
    layout: a block's group segments follow its staged-row list in meta; a
    multi-stage block (one group) adds its extra stages' records."""
    blk = plan.blocks.reshape(-1, 8).astype(np.int64)
    if blk.shape[0] == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    ng = blk[:, 1]
    seg = blk[:, 4] + ((blk[:, 5] + 3) & ~3)
    first = np.repeat(seg - 2 * (np.cumsum(ng) - ng), ng) + 2 * np.arange(int(ng.sum()))
    recs = plan.meta[first + 1].astype(np.int64)
    multi = np.nonzero(blk[:, 2] > 1)[0]
    if len(multi):
        st = plan.stages.reshape(-1, 4).astype(np.int64)
        g0 = np.cumsum(ng) - ng
        for b in multi:
            e0 = int(blk[b, 3])
            recs[g0[b]] += int(st[e0: e0 + int(blk[b, 2]) - 1, 3].sum())
    return recs, ng


def _padding(layer: LayerCSR, plan: LayerPlan) -> PaddingStats:
    nnz = layer.nnz
    if nnz == 0:
        return PaddingStats(0, 0, 0, 0, 0.0, 0.0, 0.0, empty=True)
    R = plan.rows_per_group
    recs, ng = _group_records(plan)
    warp = int(recs.sum()) * R - nnz
    starts = np.cumsum(ng) - ng
    tile = int((np.maximum.reduceat(recs, starts) * ng).sum()) * R - nnz if len(recs) else -nnz
    layer_ = int(recs.max(initial=0)) * len(recs) * R - nnz
    return PaddingStats(nnz, warp, tile, layer_, warp / nnz, tile / nnz, layer_ / nnz)


def build_plans(layers: Sequence[LayerCSR], params: PlanParams, threads: int = 0) -> list:
    """C++ conversion of many layers on host threads (spdnn_plan_build_many)."""
    L = _native.lib()
    n_layers = len(layers)
    if n_layers == 0:
        return []
    n = layers[0].neurons
    keep = []
    rps = (ctypes.c_void_p * n_layers)()
    cis = (ctypes.c_void_p * n_layers)()
    vas = (ctypes.c_void_p * n_layers)()
    for i, lay in enumerate(layers):
        if lay.neurons != n:
            raise ModelError("all layers must have the same neuron count")
        # the C++ builder trusts nnz = row_ptr[n]: the arrays must hold that many
        rp = np.asarray(lay.row_ptr)
        if rp.dtype != np.int64 or rp.shape != (n + 1,) or int(rp[0]) != 0 or \
                np.asarray(lay.col_idx).dtype != np.int32 or \
                np.asarray(lay.values).dtype != np.float32 or \
                not len(lay.col_idx) == len(lay.values) == int(rp[-1]) or \
                not (rp.flags.c_contiguous and lay.col_idx.flags.c_contiguous and
                     lay.values.flags.c_contiguous):
            raise ModelError(f"layer {i}: malformed CSR (row_ptr[-1] must equal the "
                             "col_idx and values lengths)")
        keep.append(lay)
        rps[i] = lay.row_ptr.ctypes.data
        cis[i] = lay.col_idx.ctypes.data if lay.nnz else 0
        vas[i] = lay.values.ctypes.data if lay.nnz else 0
    handles = (ctypes.c_void_p * n_layers)()
    if threads <= 0:
        import os
        threads = min(32, os.cpu_count() or 1)
    pp = _params_struct(params)
    _native.check(L.spdnn_plan_build_many(n_layers, n, rps, cis, vas, ctypes.byref(pp),
                                          int(threads), handles), "prepare_model")
    try:
        return [_export(handles[i]) for i in range(n_layers)]
    finally:
        for i in range(n_layers):
            L.spdnn_plan_free(handles[i])


def prepare_layer(layer: LayerCSR, config: InferenceConfig, mode: Mode) -> PreparedLayer:
    return prepare_model(NetworkModel(layer.neurons, (layer,), np.zeros(layer.neurons)),
                         config, mode)[0]


def prepare_model(model: NetworkModel, config: InferenceConfig, mode: Mode,
                  params: PlanParams | None = None) -> list:
    """One-time conversion of every layer (engine.py:88-90), outside any clock."""
    if mode not in ("baseline", "optimized"):
        raise ModelError(f"unknown mode {mode!r}")
    if params is None:
        params = BASELINE_PARAMS if mode == "baseline" else OPTIMIZED_PARAMS
    plans = build_plans(model.layers, params)
    return [PreparedLayer(csr=lay, plan=pl, padding=_padding(lay, pl), mode=mode)
            for lay, pl in zip(model.layers, plans)]


# ---------------------------------------------------------------------------
# device residency

def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2007_14152_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch


def host_tensor(a: np.ndarray):
    """torch view of a host array without a copy. FeatureBatch arrays are
    read-only (model.py freezes them); torch only reads them (H2D copies), so
    its non-writable-array warning is silenced here."""
    torch = _torch()
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(a)


# ---------------------------------------------------------------------------
# host <-> device copies of pageable numpy memory (a reference caller's
# FeatureBatch, the returned final values): the driver's pageable path runs at
# ~2 GB/s into fresh memory (first-touch page faults inside the copy); here the
# bytes go through two reused pinned chunks, the CPU side copied by a few
# threads (page faults in parallel) while the DMA of the other chunk runs.
# The chunks are per device and shared by every caller thread: a transfer
# holds the device's staging lock from its first chunk until its last copy has
# completed (concurrent infer calls, test_engine.py:264-287 of the reference,
# take turns on the copy engine instead of overwriting each other's chunks).

STAGE_CHUNK = 32 << 20
_STAGE_THREADS = 8
_stage_lock = threading.Lock()
_stage: dict = {}


def _stage_buffers(torch, dev):
    with _stage_lock:
        st = _stage.get(dev)
        if st is None:
            bufs = [torch.empty(STAGE_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
            from concurrent.futures import ThreadPoolExecutor
            st = (bufs, [b.numpy() for b in bufs], ThreadPoolExecutor(_STAGE_THREADS),
                  threading.Lock())
            _stage[dev] = st
        return st


def _par_copy(pool, dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src (flat uint8 views) split over the pool's threads."""
    n = dst.size
    parts = min(_STAGE_THREADS, max(1, n >> 22))
    step = -(-n // parts)
    futs = [pool.submit(np.copyto, dst[i:i + step], src[i:i + step]) for i in range(0, n, step)]
    for f in futs:
        f.result()


def d2h_numpy(src) -> np.ndarray:
    """A contiguous device tensor as a new (pageable) numpy array, through the
    pinned chunks (D2H of chunk i+1 overlaps the CPU copy of chunk i)."""
    torch = _torch()
    src = src.contiguous()
    out = np.empty(tuple(src.shape), dtype=np.dtype(str(src.dtype).replace("torch.", "")))
    nbytes = out.nbytes
    if nbytes < (4 << 20):
        out[...] = src.cpu().numpy()
        return out
    bufs, views, pool, lock = _stage_buffers(torch, src.device.index)
    s8 = src.reshape(-1).view(torch.uint8)
    o8 = out.reshape(-1).view(np.uint8)
    stream = torch.cuda.current_stream()
    events = [torch.cuda.Event(), torch.cuda.Event()]
    pending = None  # (buffer index, offset, length) copied to the GPU, not yet to `out`
    with lock:
        for i, off in enumerate(range(0, nbytes, STAGE_CHUNK)):
            b, ln = i % 2, min(STAGE_CHUNK, nbytes - off)
            bufs[b][:ln].copy_(s8[off:off + ln], non_blocking=True)
            events[b].record(stream)
            if pending is not None:
                pb_, poff, pln = pending
                events[pb_].synchronize()
                _par_copy(pool, o8[poff:poff + pln], views[pb_][:pln])
            pending = (b, off, ln)
        pb_, poff, pln = pending
        events[pb_].synchronize()
        _par_copy(pool, o8[poff:poff + pln], views[pb_][:pln])
    return out


def h2d_into(dst, src: np.ndarray) -> None:
    """dst (contiguous device tensor) <- src (C-contiguous host array of the
    same byte size), through the pinned chunks when src is pageable; pinned
    sources are copied directly. Stream-ordered on the current stream; returns
    once every source byte has been handed to a copy."""
    torch = _torch()
    t = host_tensor(src)
    if t.is_pinned() or src.nbytes < (4 << 20):
        dst.copy_(t.reshape(dst.shape), non_blocking=True)
        return
    bufs, views, pool, lock = _stage_buffers(torch, dst.device.index)
    d8 = dst.reshape(-1).view(torch.uint8)
    s8 = src.reshape(-1).view(np.uint8)
    stream = torch.cuda.current_stream()
    events = [None, None]
    with lock:
        for i, off in enumerate(range(0, src.nbytes, STAGE_CHUNK)):
            b, ln = i % 2, min(STAGE_CHUNK, src.nbytes - off)
            if events[b] is not None:
                events[b].synchronize()  # the chunk that used this buffer has been copied
            _par_copy(pool, views[b][:ln], s8[off:off + ln])
            d8[off:off + ln].copy_(bufs[b][:ln], non_blocking=True)
            events[b] = torch.cuda.Event()
            events[b].record(stream)
        for e in events:
            if e is not None:
                e.synchronize()


def _dptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _stream_ptr(torch) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _fill_bias_slots(plan: "LayerPlan", meta: np.ndarray, bias: np.ndarray) -> np.ndarray:
    """Copy of a plan's meta with every block's bias slots set to bias[row]
    (0 for padding rows), so the kernel reads row biases from shared memory."""
    meta = meta.copy()
    R = plan.rows_per_group
    blk = plan.blocks.reshape(-1, 8)
    if blk.shape[0] == 0:
        return meta
    ng = blk[:, 1].astype(np.int64)
    rows_at = blk[:, 4].astype(np.int64) + ((blk[:, 5].astype(np.int64) + 3) & ~3) + 2 * ng
    cnt = R * ng
    idx = np.repeat(rows_at - np.cumsum(cnt) + cnt, cnt) + np.arange(int(cnt.sum()))
    rows = meta[idx]
    vals = np.where(rows >= 0, bias[np.clip(rows, 0, None)], np.float32(0)).astype(np.float32)
    meta[idx + np.repeat(cnt, cnt)] = vals.view(np.int32)
    return meta


_KINDS = ("blocks", "stages", "meta", "records")


class DeviceNetwork:
    """All layer plans of a network resident in HBM, plus the bias vector.

    Plans are uploaded in chunks of layers; within a chunk the arrays of all
    its layers are concatenated per kind (one allocation each). ``layer_devs``
    holds one ``spdnn_layer_dev`` per layer pointing into them. Built either
    from a prepared model (``DeviceNetwork(prepared, bias)``) or layer chunk by
    layer chunk from a CSR iterator (``DeviceNetwork.from_layers``), which never
    holds more than one chunk of host CSR/plans -- the 65536 x 1920 network's
    CSR alone is 32 GB of host memory, its layout 25 GB of HBM.
    """

    def __init__(self, prepared: Sequence[PreparedLayer], bias: np.ndarray, device=None):
        self._start(bias, device)
        self.modes = {p.mode for p in prepared}
        self.nnz = [p.csr.nnz if p.csr is not None else 0 for p in prepared]
        self._append([p.plan for p in prepared])
        self._finish()

    @classmethod
    def from_layers(cls, layers, bias: np.ndarray, params: "PlanParams | None" = None,
                    chunk: int = 64, threads: int = 0, on_chunk=None, device=None
                    ) -> "DeviceNetwork":
        """Plan (C++, host threads) and upload `layers` (any iterable of
        LayerCSR) `chunk` layers at a time. ``on_chunk(first_layer_index,
        csr_list)`` sees each chunk's CSR before it is dropped (e.g. a
        layer-by-layer CPU check)."""
        self = cls.__new__(cls)
        self._start(bias, device)
        params = params or OPTIMIZED_PARAMS
        self.modes = {"baseline" if params == BASELINE_PARAMS else "optimized"}
        self.nnz = []
        buf = []

        def flush():
            plans = build_plans(buf, params, threads)
            if on_chunk is not None:
                on_chunk(self.num_layers, list(buf))
            self.nnz += [lay.nnz for lay in buf]
            self._append(plans)
            buf.clear()

        for lay in layers:
            if lay.neurons != self.neurons:
                raise ModelError("layer width does not match the bias vector")
            buf.append(lay)
            if len(buf) == chunk:
                flush()
        if buf:
            flush()
        self._finish()
        return self

    def _start(self, bias, device):
        torch = _torch()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.neurons = int(bias.shape[0])
        self._bias32 = np.ascontiguousarray(bias, np.float32)
        self.bias = torch.from_numpy(self._bias32.copy()).to(self.device)
        self.num_layers = 0
        self.chunks = []        # per chunk: {kind: device tensor}
        self._ptrs = []         # per layer: {kind: device address}
        self._plans_meta = []   # per layer: the LayerPlan scalars (arrays dropped)
        self.total_slots, self.num_fp = [], []
        self.pow2, self._emin, self._emax = True, None, None
        self.hbm_bytes = int(self.bias.numel() * 4)

    def _append(self, plans) -> None:
        torch = _torch()
        bufs, offsets = {}, {k: [] for k in _KINDS}
        for k in _KINDS:
            parts = []
            off = 0
            for pl in plans:
                a = getattr(pl, k)
                if k == "meta":
                    a = _fill_bias_slots(pl, a, self._bias32)
                pad = (-a.shape[0] * a.itemsize) % 32  # every layer's slice 32-byte aligned
                parts.append(a)
                if pad:
                    parts.append(np.zeros(pad // a.itemsize, dtype=a.dtype))
                offsets[k].append(off)
                off += a.shape[0] + pad // a.itemsize
            cat = np.concatenate(parts) if parts else np.zeros(0, np.int32)
            if cat.dtype == np.uint32:
                cat = cat.view(np.int32)
            if cat.size == 0:
                cat = np.zeros(1, dtype=cat.dtype)
            bufs[k] = torch.from_numpy(np.ascontiguousarray(cat)).to(self.device)
            self.hbm_bytes += int(bufs[k].numel() * bufs[k].element_size())
        self.chunks.append(bufs)
        for l, pl in enumerate(plans):
            self._ptrs.append({k: bufs[k].data_ptr() + offsets[k][l] * bufs[k].element_size()
                               for k in _KINDS})
            self._plans_meta.append(pl)
            self.total_slots.append(pl.total_slots)
            self.num_fp.append(pl.num_fp)
            self.pow2 = self.pow2 and pl.pow2
            self._emin = pl.wexp_min if self._emin is None else min(self._emin, pl.wexp_min)
            self._emax = pl.wexp_max if self._emax is None else max(self._emax, pl.wexp_max)
        self.num_layers += len(plans)

    def _finish(self) -> None:
        self.layer_devs = (_native.LayerDev * max(1, self.num_layers))()
        for l, pl in enumerate(self._plans_meta):
            d = self.layer_devs[l]
            for k in _KINDS:
                setattr(d, k, self._ptrs[l][k])
            d.num_blocks = pl.num_blocks
            d.neurons = pl.neurons
            d.rows_per_group = pl.rows_per_group
            d.record_words = pl.record_words
            d.max_fp_per_stage = pl.max_fp_per_stage
            d.max_records_per_stage = pl.max_records_per_stage
            d.max_meta_per_block = pl.max_meta_per_block
            d.max_groups_per_block = pl.max_groups_per_block
            d.uniform = int(pl.uniform)
            d.weight_bits = pl.weight_bits
        self._plans_meta = [None] * self.num_layers  # host arrays no longer needed
        # FMA form (one FFMA2 per (row, column)) is exact when every weight is
        # +-2^e and no input falls below `tiny` (products stay normal) or above
        # `huge` (no overflow); the kernels flag violations and infer() reruns
        # in the exact form.
        self.pow2 = self.num_layers > 0 and self.pow2
        emin = self._emin if self._emin is not None else 0
        emax = self._emax if self._emax is not None else 0
        self.tiny = float(np.ldexp(np.float32(1.0), -126 - emin)) if -126 - emin > -149 else 0.0
        self.tiny = min(self.tiny, 1.0)
        # |x| <= huge keeps every product <= 2^95 and every sum of up to 2^31
        # of them finite (the FMA form's integer clamp assumes no NaN/inf)
        self.huge = float(np.ldexp(1.0, min(127, 95 - emax))) if emax < 95 else 0.0


# whole surviving tiles stay aligned between layers (spdnn_scratch.split);
# SPDNN_SPLIT=0 packs every layer's survivors (diagnostics)
SPLIT_LAYOUT = __import__("os").environ.get("SPDNN_SPLIT", "1") != "0"


class Workspace:
    """Per-inference device buffers for a feature-count capacity (reused)."""

    def __init__(self, neurons: int, m_cap: int, num_layers: int, device, buffers: int = 2):
        torch = _torch()
        self.neurons = neurons
        self.m_cap = m_cap
        self.ld = max(TILE, -(-m_cap // TILE) * TILE)
        self.num_layers = num_layers
        f32, i32, i64 = torch.float32, torch.int32, torch.int64
        self.x = torch.empty((m_cap, neurons), dtype=f32, device=device)  # raw upload
        nb = range(buffers)
        self.y = [torch.empty((neurons, self.ld), dtype=f32, device=device) for _ in nb]
        # 2 * ld entries: the split survivor layout between layers (spdnn_scratch.split)
        self.a = [torch.empty(2 * self.ld, dtype=i32, device=device) for _ in nb]
        self.cat = [torch.empty(2 * self.ld, dtype=i64, device=device) for _ in nb]
        self.counts = torch.zeros(num_layers + 1, dtype=i32, device=device)
        self.tile_done = torch.zeros(self.ld // 64, dtype=i32, device=device)
        self.tile_alive = torch.zeros(self.ld // 32, dtype=i32, device=device)
        self.work = torch.zeros(max(1, num_layers), dtype=i32, device=device)
        self.guard = torch.zeros(1, dtype=i32, device=device)
        self.split = torch.zeros(2 * (max(1, num_layers) + 1), dtype=i32, device=device)
        self.scratch = _native.Scratch(self.tile_done.data_ptr(), self.tile_alive.data_ptr(),
                                       self.work.data_ptr(), self.guard.data_ptr(),
                                       self.split.data_ptr() if SPLIT_LAYOUT else None)
        self.iota = torch.arange(self.ld, dtype=i32, device=device)

    def fits(self, neurons: int, m: int, num_layers: int) -> bool:
        return neurons == self.neurons and m <= self.m_cap and num_layers <= self.num_layers


_cache_lock = threading.Lock()
_net_cache: dict = {}
_ws_cache: dict = {}


# resident networks kept for repeated or alternating infer calls: least
# recently used first out, at most this many or this share of device memory
NET_CACHE_MAX = 4
NET_CACHE_HBM_SHARE = 0.25


def device_network(prepared: Sequence[PreparedLayer], bias: np.ndarray) -> DeviceNetwork:
    """Upload (once) and cache the device copy of a prepared model. Up to
    NET_CACHE_MAX networks stay resident per process (least recently used is
    evicted first, and beyond NET_CACHE_HBM_SHARE of device memory), so
    alternating infer calls on two models do not re-upload either."""
    torch = _torch()
    dev = torch.cuda.current_device()
    with _cache_lock:
        nets = _net_cache.setdefault("nets", [])  # [(prepared, bias, dev, net)], MRU last
        for i, (c_prep, c_bias, c_dev, net) in enumerate(nets):
            if c_prep is prepared and c_dev == dev and np.array_equal(c_bias, bias):
                nets.append(nets.pop(i))
                return net
        net = DeviceNetwork(prepared, bias)
        nets.append((prepared, np.array(bias, copy=True), dev, net))
        budget = NET_CACHE_HBM_SHARE * torch.cuda.get_device_properties(dev).total_memory
        while len(nets) > 1 and (len(nets) > NET_CACHE_MAX or
                                 sum(e[3].hbm_bytes for e in nets) > budget):
            nets.pop(0)
        return net


def workspace(neurons: int, m: int, num_layers: int) -> Workspace:
    torch = _torch()
    dev = torch.cuda.current_device()
    key = (dev, threading.get_ident())
    with _cache_lock:
        ws = _ws_cache.get(key)
        if ws is None or not ws.fits(neurons, m, num_layers):
            ws = None
            _ws_cache.pop(key, None)
            torch.cuda.empty_cache()
            ws = Workspace(neurons, max(m, 1), num_layers, torch.device("cuda", dev))
            _ws_cache[key] = ws
        return ws


# ---------------------------------------------------------------------------
# device execution

class DeviceRun:
    """State of one on-device inference after the layer loop."""

    def __init__(self, ws: Workspace, num_layers: int, m0: int):
        self.ws = ws
        self.num_layers = num_layers
        self.m0 = m0
        self.out_index = num_layers % 2
        self.fma = False
        self.guard = 0  # filled by collect(): bit 0 FMA-form guard, bit 1 non-finite input

    @property
    def needs_exact_rerun(self) -> bool:
        return bool(self.guard & 1) and self.fma

    @property
    def needs_unpadded_rerun(self) -> bool:
        return bool(self.guard & 2)


def stage_inputs(ws: Workspace, x_host_or_dev, categories, net: "DeviceNetwork | None" = None
                 ) -> None:
    """Copy (M, N) feature-major inputs into the workspace and lay them out
    neuron-major (spdnn_transpose_in, which also screens them for the FMA
    form); A = 0..M-1; categories as given. Resets the guard flags."""
    torch = _torch()
    m = int(x_host_or_dev.shape[0])
    n = ws.neurons
    ws.guard.zero_()
    if m:
        if isinstance(x_host_or_dev, np.ndarray):
            h2d_into(ws.x[:m], x_host_or_dev)
        else:
            ws.x[:m].copy_(x_host_or_dev, non_blocking=True)
        tiny = net.tiny if net is not None else 0.0
        huge = net.huge if net is not None else 3.0e38
        _native.check(_native.lib().spdnn_transpose_in(
            _dptr(ws.x), n, m, _dptr(ws.y[0]), ws.ld, _dptr(ws.guard), tiny, huge,
            _stream_ptr(torch)), "spdnn_transpose_in")
        ws.a[0][:m].copy_(ws.iota[:m])
        ws.cat[0][:m].copy_(categories, non_blocking=True)


FEATURES_PER_LANE = int(__import__("os").environ.get("SPDNN_FEATURES_PER_LANE", "4"))


def run_opts(net: DeviceNetwork, fma: bool | None = None) -> _native.RunOpts:
    use = net.pow2 if fma is None else (fma and net.pow2)
    if FEATURES_PER_LANE not in (2, 4):
        raise ModelError(f"SPDNN_FEATURES_PER_LANE must be 2 or 4, not {FEATURES_PER_LANE}")
    return _native.RunOpts(int(use), net.tiny, FEATURES_PER_LANE)


def reset_run(ws: Workspace, m0: int) -> None:
    """Zero the per-run counters (stream-ordered)."""
    ws.counts.zero_()
    ws.counts[0] = m0
    ws.work.zero_()
    ws.split.zero_()


def run_layers(net: DeviceNetwork, ws: Workspace, m0: int, fma: bool | None = None
               ) -> DeviceRun:
    """Enqueue every layer on the current stream; no host synchronisation."""
    torch = _torch()
    reset_run(ws, m0)
    opts = run_opts(net, fma)
    _native.check(_native.lib().spdnn_infer_layers(
        net.num_layers, net.layer_devs, _dptr(net.bias), _dptr(ws.y[0]), _dptr(ws.y[1]), ws.ld,
        _dptr(ws.a[0]), _dptr(ws.a[1]), _dptr(ws.cat[0]), _dptr(ws.cat[1]), _dptr(ws.counts),
        ctypes.byref(ws.scratch), ctypes.byref(opts), _stream_ptr(torch)), "spdnn_infer_layers")
    run = DeviceRun(ws, net.num_layers, m0)
    run.fma = bool(opts.fma_form)
    return run


def collect(run: DeviceRun, want_values: bool = True):
    """Sorted survivor categories (+ their values as (S, N) feature-major) and
    the per-layer active counts. One host synchronisation."""
    torch = _torch()
    ws = run.ws
    host = torch.cat([ws.counts[: run.num_layers + 1], ws.guard]).cpu().numpy().astype(np.int64)
    counts, run.guard = host[:-1], int(host[-1])
    s = int(counts[run.num_layers]) if run.num_layers else run.m0
    o = run.out_index
    cats = ws.cat[o][:s]
    sorted_cats, perm = torch.sort(cats)
    values = None
    if want_values:
        out = torch.empty((s, ws.neurons), dtype=torch.float32, device=ws.y[o].device)
        _native.check(_native.lib().spdnn_gather_out(
            _dptr(ws.y[o]), ws.neurons, ws.ld, _dptr(ws.a[o]), _dptr(perm), s, _dptr(out),
            _stream_ptr(torch)), "spdnn_gather_out")
        values = out
    return counts, sorted_cats, values


def _check_inputs(model: NetworkModel, inputs: FeatureBatch, mode) -> None:
    if inputs.neurons != model.neurons:
        raise ModelError("inputs do not match model width")
    if mode not in ("baseline", "optimized"):
        raise ModelError(f"unknown mode {mode!r}")


def _check_prepared(prepared: Sequence[PreparedLayer], model: NetworkModel, mode) -> None:
    if len(prepared) != model.num_layers:
        raise ModelError("prepared structures do not match the model depth")
    for p in prepared:
        if p.plan is None or p.mode != mode:
            raise ModelError(f"prepared structures are for {p.mode} mode")


def _outcomes(counts: np.ndarray, net: DeviceNetwork) -> list:
    outs = []
    for l in range(net.num_layers):
        before, after = int(counts[l]), int(counts[l + 1])
        if before == 0:
            outs.append(LayerOutcome(0, 0, 0, 0))
            continue
        tiles = -(-before // TILE)
        outs.append(LayerOutcome(active_before=before, active_after=after,
                                 weight_element_reads=net.total_slots[l] * tiles,
                                 feature_element_reads=net.num_fp[l] * before))
    return outs


def infer(model: NetworkModel, inputs: FeatureBatch, config: InferenceConfig,
          mode: Mode = "optimized", prepared: Sequence[PreparedLayer] | None = None,
          values: bool = True) -> InferenceResult:
    """All layers with pruning after each (engine.py:235-290), on the GPU.

    The clock covers the layer loop only, like the reference's (prepare and
    result assembly excluded); ``device_seconds`` is the same span measured
    with CUDA events. ``values=False`` (extension) skips copying the final
    feature values back: ``final`` is then None and only the sorted
    categories and per-layer counts come back -- the Graph Challenge output.
    With ``config.streaming`` the layouts are built by a WeightStreamer while
    the GPU runs the previous layers (engine.py:173-232, 250-282).
    """
    _check_inputs(model, inputs, mode)
    if config.streaming:
        if prepared is not None:
            raise ModelError("prepared structures cannot be combined with streaming")
        return _infer_streaming(model, inputs, config, mode, values)
    if prepared is None:
        prepared = prepare_model(model, config, mode)
    _check_prepared(prepared, model, mode)
    n, m = model.neurons, inputs.active_count
    if model.num_layers == 0 or m == 0:
        return _trivial_result(model.num_layers, inputs, count_edges(model))
    net = device_network(prepared, model.bias)
    return infer_device(net, inputs, values=values, edges_per_input=count_edges(model),
                        unpadded=lambda: DeviceNetwork(_unpadded(prepared, model), model.bias))


def _trivial_result(num_layers: int, inputs: FeatureBatch, edges: int) -> InferenceResult:
    m = inputs.active_count
    per = [LayerOutcome(0, 0, 0, 0) for _ in range(num_layers)]
    if m and num_layers == 0:
        per = []
    return InferenceResult(final=inputs, categories=inputs.categories.copy(), per_layer=per,
                           elapsed_seconds=0.0, edges_processed=inputs.total_inputs * edges)


def infer_device(net: DeviceNetwork, inputs: FeatureBatch, values: bool = True,
                 edges_per_input: int | None = None, unpadded=None) -> InferenceResult:
    """``infer`` on a network already resident in HBM (extension): e.g. one
    built layer chunk by layer chunk with ``DeviceNetwork.from_layers`` for a
    model whose host CSR would not fit. ``unpadded()`` returns the same
    network with one row per group; it is only called for non-finite inputs
    (see DESIGN.md section 3)."""
    torch = _torch()
    n, m = net.neurons, inputs.active_count
    if inputs.neurons != n:
        raise ModelError("inputs do not match model width")
    edges = inputs.total_inputs * (edges_per_input if edges_per_input is not None
                                   else sum(getattr(net, "nnz", [])))
    if net.num_layers and m >= 4 * PIPELINE_MIN_FEATURES:
        res = _infer_pipelined(net, inputs, edges, values)
        if res is not None:
            return res
    if net.num_layers == 0 or m == 0:
        return _trivial_result(net.num_layers, inputs, edges // max(inputs.total_inputs, 1))
    ws = workspace(n, m, net.num_layers)
    x = np.asarray(inputs.data).T  # (M, N) C-order view of the Fortran bytes
    cats = host_tensor(np.ascontiguousarray(inputs.categories))
    fma = None
    elapsed = device = 0.0
    for _attempt in range(3):
        stage_inputs(ws, x, cats, net)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev0.record()
        run = run_layers(net, ws, m, fma)
        ev1.record()
        torch.cuda.synchronize()
        elapsed += time.perf_counter() - t0
        device += ev0.elapsed_time(ev1) / 1e3
        counts, sorted_cats, vals = collect(run, want_values=values)
        if run.needs_unpadded_rerun and unpadded is not None:
            # NaN/inf inputs: zero-weight union slots would spread them to rows
            # that never read them; one row per group has no such slots.
            net = unpadded()
            unpadded = None
            fma = False
        elif run.needs_unpadded_rerun:
            if all(d.rows_per_group == 1 for d in net.layer_devs[: net.num_layers]):
                break
            raise ModelError("non-finite inputs need the unpadded plans")
        elif run.needs_exact_rerun:
            fma = False
        else:
            break
    cats_np = sorted_cats.cpu().numpy().astype(np.int64)
    final = None
    if values:
        final = FeatureBatch(neurons=n, data=d2h_numpy(vals).T, categories=cats_np,
                             total_inputs=inputs.total_inputs)
    return InferenceResult(final=final, categories=cats_np.copy(),
                           per_layer=_outcomes(counts, net), elapsed_seconds=elapsed,
                           edges_processed=edges, device_seconds=device)


PIPELINE_MIN_FEATURES = 4096  # smallest first chunk of the upload/compute pipeline
# cost model of the head/rest split (B200 measurements): pinned
# host->device bandwidth, credited edge rate of the layer loop, fixed cost per
# layer launch of a chunk
PIPELINE_H2D_BPS = 50e9
PIPELINE_EDGE_RATE = 30e12
PIPELINE_LAYER_FIXED_S = 12e-6


def pipeline_head(m: int, neurons: int, num_layers: int, edges_per_input: float) -> int:
    """Features in the head chunk: large enough that its compute covers the
    rest's upload (then only the head's upload is exposed), no larger --
    h = (T_up - T_fixed) / (T_up + T_compute), clamped to [1/16, 1/2]."""
    t_up = m * neurons * 4.0 / PIPELINE_H2D_BPS
    t_comp = m * edges_per_input / PIPELINE_EDGE_RATE
    t_fixed = num_layers * PIPELINE_LAYER_FIXED_S
    h = (t_up - t_fixed) / max(t_up + t_comp, 1e-12)
    h = min(0.5, max(1.0 / 16, h))
    return max(PIPELINE_MIN_FEATURES, int(m * h))
_pipe_cache: dict = {}


class _PipeBuffers:
    """Device buffers of the chunked upload/compute pipeline: two raw-upload
    buffers (chunk c+1 lands while chunk c computes), the shared neuron-major
    feature buffers, and per chunk the index/category/count arrays that hold
    its survivors until the single read at the end."""

    def __init__(self, n: int, cap: int, chunks: int, num_layers: int, device):
        torch = _torch()
        self.key = (n, cap, chunks, num_layers)
        self.ws = Workspace(n, cap, num_layers, device)  # y[0..1], scratch, iota
        self.x = [self.ws.x, torch.empty((cap, n), dtype=torch.float32, device=device)]
        i32, i64 = torch.int32, torch.int64
        # 2 * ld entries: the split survivor layout between layers
        self.a = [[torch.empty(2 * self.ws.ld, dtype=i32, device=device) for _ in range(2)]
                  for _ in range(chunks)]
        self.cat = [[torch.empty(2 * self.ws.ld, dtype=i64, device=device) for _ in range(2)]
                    for _ in range(chunks)]
        self.counts = torch.zeros((chunks, num_layers + 1), dtype=i32, device=device)
        self.guard = torch.zeros(chunks, dtype=i32, device=device)
        self.up = torch.cuda.Stream(device=device)


def _infer_pipelined(net: DeviceNetwork, inputs: FeatureBatch, edges: int,
                     values: bool = False):
    """Inference with the input upload overlapped: the batch is
    cut into two feature ranges (features never interact, so each runs the
    whole network on its own): a head (pipeline_head: sized so its compute
    covers the rest's upload) whose upload is the only one exposed, and the
    rest, copied host->device on a side stream while the head's layers run;
    one extra launch per layer is paid. One host synchronisation at the end
    reads every chunk's counts. With ``values`` the head's surviving values
    are gathered (one host read of its count) once the rest's upload has been
    issued and before the rest's layers reuse the feature buffers; categories
    increase with the input position, so the head's sorted survivors precede
    the rest's.
    Returns None when an arithmetic guard fired (the caller then takes the
    unchunked path, which reruns in the exact form)."""
    torch = _torch()
    n, m, L = net.neurons, inputs.active_count, net.num_layers
    head = pipeline_head(m, n, L, edges / max(inputs.total_inputs, 1))
    bounds = [(0, head), (head, m)]
    chunks = 2
    cap = max(hi - lo for lo, hi in bounds)
    dev = torch.cuda.current_device()
    key = (dev, threading.get_ident())
    with _cache_lock:
        pb = _pipe_cache.get(key)
        if pb is None or pb.key != (n, cap, chunks, L):
            _pipe_cache.pop(key, None)
            _ws_cache.pop(key, None)
            torch.cuda.empty_cache()
            pb = _PipeBuffers(n, cap, chunks, L, torch.device("cuda", dev))
            _pipe_cache[key] = pb
    ws = pb.ws
    host = np.asarray(inputs.data).T  # (M, N) C-order view of the Fortran bytes
    cats = host_tensor(np.ascontiguousarray(inputs.categories))
    main, up = torch.cuda.current_stream(), pb.up
    lib = _native.lib()
    opts = run_opts(net)
    freed = [None, None]
    pb.guard.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(main)
    vals_parts = []

    def gather_values(c):
        # chunk c's sorted survivors and their values (before the next chunk's
        # input transpose and layers overwrite the feature buffers)
        s_c = int(pb.counts[c][L].item())
        o = L % 2
        sc_cats, perm = torch.sort(pb.cat[c][o][:s_c])
        out = torch.empty((s_c, n), dtype=torch.float32, device=ws.y[o].device)
        if s_c:
            _native.check(lib.spdnn_gather_out(
                _dptr(ws.y[o]), n, ws.ld, _dptr(pb.a[c][o]), _dptr(perm), s_c, _dptr(out),
                _stream_ptr(torch)), "spdnn_gather_out")
        vals_parts.append(out)

    for c, (lo, hi) in enumerate(bounds):
        mc, xb = hi - lo, pb.x[c % 2]
        with torch.cuda.stream(up):
            if freed[c % 2] is not None:
                up.wait_event(freed[c % 2])  # chunk c-2 has been laid out
            h2d_into(xb[:mc], host[lo:hi])  # (pageable sources: staged, blocking)
            pb.cat[c][0][:mc].copy_(cats[lo:hi], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(up)
        if values and c > 0:
            gather_values(c - 1)
        main.wait_event(ready)
        guard = ctypes.c_void_p(pb.guard.data_ptr() + 4 * c)
        _native.check(lib.spdnn_transpose_in(
            _dptr(xb), n, mc, _dptr(ws.y[0]), ws.ld, guard, net.tiny, net.huge,
            _stream_ptr(torch)), "spdnn_transpose_in")
        freed[c % 2] = torch.cuda.Event()
        freed[c % 2].record(main)
        for t in (xb, pb.cat[c][0]):
            t.record_stream(main)
        pb.a[c][0][:mc].copy_(ws.iota[:mc])
        cnt = pb.counts[c]
        cnt.zero_()
        cnt[0] = mc
        ws.work.zero_()
        ws.split.zero_()
        sc = _native.Scratch(ws.tile_done.data_ptr(), ws.tile_alive.data_ptr(),
                             ws.work.data_ptr(), pb.guard.data_ptr() + 4 * c,
                             ws.split.data_ptr() if SPLIT_LAYOUT else None)
        _native.check(lib.spdnn_infer_layers(
            L, net.layer_devs, _dptr(net.bias), _dptr(ws.y[0]), _dptr(ws.y[1]), ws.ld,
            _dptr(pb.a[c][0]), _dptr(pb.a[c][1]), _dptr(pb.cat[c][0]), _dptr(pb.cat[c][1]),
            _dptr(cnt), ctypes.byref(sc), ctypes.byref(opts), _stream_ptr(torch)),
            "spdnn_infer_layers")
    if values:
        gather_values(chunks - 1)
    ev1.record(main)
    host_counts = torch.cat([pb.counts.reshape(-1).to(torch.int64),
                             pb.guard.to(torch.int64)]).cpu().numpy()
    elapsed = time.perf_counter() - t0
    counts = host_counts[:-chunks].reshape(chunks, L + 1)
    if int(np.bitwise_or.reduce(host_counts[-chunks:])) & (2 | (1 if opts.fma_form else 0)):
        return None
    surv = counts[:, L]
    cat_parts = [pb.cat[c][L % 2][: int(surv[c])] for c in range(chunks)]
    cats_np = torch.sort(torch.cat(cat_parts))[0].cpu().numpy().astype(np.int64)
    final = None
    if values:
        vals = vals_parts[0] if chunks == 1 else torch.cat(vals_parts)
        final = FeatureBatch(neurons=n, data=d2h_numpy(vals).T, categories=cats_np,
                             total_inputs=inputs.total_inputs)
    return InferenceResult(final=final, categories=cats_np.copy() if values else cats_np,
                           per_layer=_outcomes(counts.sum(0), net),
                           elapsed_seconds=elapsed, edges_processed=edges,
                           device_seconds=ev0.elapsed_time(ev1) / 1e3)


class WeightStreamer:
    """Double-buffered layer layouts (the reference's WeightStreamer,
    engine.py:173-232): a background thread builds layer l+1's plan (C++,
    the GIL released) while the GPU runs layer l; at most two layers'
    prepared structures exist at once. Same consumer API: ``next_layer``,
    ``release``, ``stop``, ``join``, ``peak_resident``, ``materialized_count``.
    """

    def __init__(self, model: NetworkModel, config: InferenceConfig, mode: Mode = "optimized"):
        import queue
        self._slots = threading.Semaphore(2)
        self._ready = queue.Queue()
        self._stopped = threading.Event()
        self._gauge_lock = threading.Lock()
        self._resident = 0
        self.peak_resident = 0
        self.materialized_count = 0
        self._thread = threading.Thread(target=self._produce, args=(model, config, mode),
                                        daemon=True)
        self._thread.start()

    def _produce(self, model, config, mode) -> None:
        try:
            for layer in model.layers:
                while not self._slots.acquire(timeout=0.05):
                    if self._stopped.is_set():
                        return
                if self._stopped.is_set():
                    return
                prep = prepare_layer(layer, config, mode)
                with self._gauge_lock:
                    self._resident += 1
                    self.materialized_count += 1
                    self.peak_resident = max(self.peak_resident, self._resident)
                self._ready.put(prep)
            self._ready.put(None)
        except BaseException as exc:  # propagate into the consumer
            self._ready.put(exc)

    def next_layer(self) -> PreparedLayer:
        item = self._ready.get()
        if isinstance(item, BaseException):
            raise item
        if item is None:
            raise ModelError("weight streamer exhausted")
        return item

    def release(self) -> None:
        with self._gauge_lock:
            self._resident -= 1
        self._slots.release()

    def stop(self) -> None:
        self._stopped.set()
        self._thread.join()

    def join(self) -> None:
        self._thread.join()


def _infer_streaming(model: NetworkModel, inputs: FeatureBatch, config: InferenceConfig,
                     mode: Mode, values: bool) -> InferenceResult:
    """Layer loop fed by a WeightStreamer. Each layer's plan is uploaded and
    its kernel enqueued as soon as the producer has it; the host never waits
    for the GPU inside the loop except to notice that every feature died
    (a non-blocking read of an earlier layer's count), which stops the
    streamer as the reference does (engine.py:265-270)."""
    torch = _torch()
    n, m, L = model.neurons, inputs.active_count, model.num_layers
    edges = count_edges(model)
    if L == 0 or m == 0:
        return _trivial_result(L, inputs, edges)
    bias = np.asarray(model.bias, np.float32)
    ws = workspace(n, m, L)
    x = host_tensor(np.asarray(inputs.data).T)
    cats = host_tensor(np.ascontiguousarray(inputs.categories))
    stage_inputs(ws, x, cats, None)  # tiny = 0: screens only non-finite inputs
    ws.counts.zero_()
    ws.counts[0] = m
    ws.work.zero_()
    host_counts = torch.zeros(L + 1, dtype=torch.int32).pin_memory()
    stream = _stream_ptr(torch)
    main, up = torch.cuda.current_stream(), torch.cuda.Stream()
    lib = _native.lib()
    nets, checks, slots, fps = [], [], [], []
    opts = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    streamer = WeightStreamer(model, config, mode)  # inside the clock, as engine.py:258-261
    ran = 0
    try:
        for l in range(L):
            # stop once an earlier layer's count has landed as zero
            while checks and checks[0][1].query():
                lc, _ = checks.pop(0)
                if int(host_counts[lc]) == 0:
                    raise StopIteration
            prep = streamer.next_layer()
            try:
                # upload on a side stream: a pageable H2D copy on the compute
                # stream would make the host wait for the running layer
                with torch.cuda.stream(up):
                    net = DeviceNetwork([prep], bias)
            finally:
                streamer.release()
            ready = torch.cuda.Event()
            ready.record(up)
            main.wait_event(ready)
            for t in list(net.chunks[0].values()) + [net.bias]:
                t.record_stream(main)
            if opts is None:
                # the exact form throughout: the FMA form's guard would need a
                # rerun of already-streamed layers
                opts = run_opts(net, fma=False)
            i, o = l & 1, (l & 1) ^ 1
            cnt = ws.counts.data_ptr()
            _native.check(lib.spdnn_layer_forward(
                ctypes.byref(net.layer_devs[0]), _dptr(net.bias), _dptr(ws.y[i]),
                _dptr(ws.y[o]), ws.ld, _dptr(ws.a[i]), _dptr(ws.cat[i]),
                ctypes.c_void_p(cnt + 4 * l), _dptr(ws.a[o]), _dptr(ws.cat[o]),
                ctypes.c_void_p(cnt + 4 * (l + 1)), ctypes.byref(ws.scratch),
                ctypes.c_void_p(ws.work.data_ptr() + 4 * l), ctypes.byref(opts), stream),
                "spdnn_layer_forward")
            slots.append(net.total_slots[0])
            fps.append(net.num_fp[0])
            nets.append(net)
            host_counts[l + 1: l + 2].copy_(ws.counts[l + 1: l + 2], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            checks.append((l + 1, ev))
            ran = l + 1
            if len(nets) > 2:
                # stream-ordered allocator: the freed plan is reused only by
                # work enqueued after this layer's kernel on the same stream
                nets.pop(0)
    except StopIteration:
        pass
    finally:
        streamer.stop()
    ev1.record()
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    run = DeviceRun(ws, ran, m)
    run.out_index = ran % 2
    counts, sorted_cats, vals = collect(run, want_values=values)
    if run.needs_unpadded_rerun:
        # non-finite inputs: redo without streaming on one-row-per-group plans
        return infer(model, inputs, replace(config, streaming=False), mode, values=values)
    per = []
    for l in range(L):
        before = int(counts[l]) if l < ran else 0
        after = int(counts[l + 1]) if l < ran else 0
        if before == 0:
            per.append(LayerOutcome(0, 0, 0, 0))
            continue
        per.append(LayerOutcome(before, after,
                                weight_element_reads=slots[l] * -(-before // TILE),
                                feature_element_reads=fps[l] * before))
    cats_np = sorted_cats.cpu().numpy().astype(np.int64)
    final = None
    if values:
        final = FeatureBatch(neurons=n, data=d2h_numpy(vals).T, categories=cats_np,
                             total_inputs=inputs.total_inputs)
    return InferenceResult(final=final, categories=cats_np.copy(), per_layer=per,
                           elapsed_seconds=elapsed, edges_processed=inputs.total_inputs * edges,
                           device_seconds=ev0.elapsed_time(ev1) / 1e3)


def _unpadded(prepared: Sequence[PreparedLayer], model: NetworkModel) -> list:
    """Plans with one row per group (no zero-weight slots) for the same layers."""
    if all(p.plan.rows_per_group == 1 for p in prepared):
        return list(prepared)
    plans = build_plans([p.csr for p in prepared], BASELINE_PARAMS)
    return [replace(p, plan=pl) for p, pl in zip(prepared, plans)]


# ---------------------------------------------------------------------------
# single-layer entry points (engine.py:93-127) and host helpers

def _one_layer(features: FeatureBatch, prepared: PreparedLayer, bias: np.ndarray):
    torch = _torch()
    n, m = features.neurons, features.active_count
    if m == 0:
        return np.zeros((n, 0), np.float32, order="F"), np.zeros(0, bool)
    net = DeviceNetwork([prepared], bias)
    ws = Workspace(n, m, 1, torch.device("cuda", torch.cuda.current_device()))
    x = host_tensor(np.asarray(features.data).T)
    fma = None
    for _attempt in range(3):
        stage_inputs(ws, x, torch.arange(m, dtype=torch.int64), net)
        ws.counts.zero_()
        ws.counts[0] = m
        ws.work.zero_()
        opts = run_opts(net, fma)
        _native.check(_native.lib().spdnn_layer_forward(
            ctypes.byref(net.layer_devs[0]), _dptr(net.bias), _dptr(ws.y[0]), _dptr(ws.y[1]),
            ws.ld, _dptr(ws.a[0]), _dptr(ws.cat[0]), _dptr(ws.counts), _dptr(ws.a[1]),
            _dptr(ws.cat[1]), ctypes.c_void_p(ws.counts.data_ptr() + 4), ctypes.byref(ws.scratch),
            _dptr(ws.work), ctypes.byref(opts), _stream_ptr(torch)), "spdnn_layer_forward")
        guard = int(ws.guard.item())
        if guard & 2 and prepared.plan.rows_per_group != 1:
            plan = build_plans([prepared.csr], BASELINE_PARAMS)[0]
            net = DeviceNetwork([replace(prepared, plan=plan)], bias)
            fma = False
        elif guard & 1 and opts.fma_form:
            fma = False
        else:
            break
    out = torch.empty((m, n), dtype=torch.float32, device=ws.y[1].device)
    _native.check(_native.lib().spdnn_gather_out(_dptr(ws.y[1]), n, ws.ld, _dptr(ws.iota),
                                                 ctypes.c_void_p(0), m, _dptr(out),
                                                 _stream_ptr(torch)), "spdnn_gather_out")
    s = int(ws.counts[1].item())
    alive = np.zeros(m, dtype=bool)
    alive[ws.a[1][:s].cpu().numpy()] = True
    return d2h_numpy(out).T, alive


def optimized_layer(features: FeatureBatch, prepared, bias: np.ndarray,
                    minibatch: int | None = None):
    """One fused layer on the GPU; returns ((N, M) F-order out, active flags).

    ``prepared`` is a PreparedLayer (or its LayerPlan). ``minibatch`` is
    accepted for signature compatibility (engine.py:109); the kernel's feature
    tile is fixed at 128.
    """
    if minibatch is not None and minibatch < 1:
        raise ModelError("minibatch must be positive")
    if hasattr(prepared, "wdispl") and hasattr(prepared, "windex"):
        # a layer prepared by the reference itself (its sliced ELL): same
        # weights, laid out for this kernel
        csr = csr_from_sliced_ell(prepared)
        prepared = PreparedLayer(csr=csr, plan=build_plans([csr], OPTIMIZED_PARAMS)[0])
    if isinstance(prepared, LayerPlan):
        prepared = PreparedLayer(csr=None, plan=prepared)
    if prepared.plan is None:
        raise ModelError("prepared structures are for baseline mode")
    n = prepared.plan.neurons
    if features.neurons != n or len(bias) != n:
        raise ModelError("dimension mismatch in optimized_layer")
    return _one_layer(features, prepared, np.asarray(bias, np.float32))


def csr_from_sliced_ell(ell) -> LayerCSR:
    """The CSR layer behind a reference-prepared sliced-ELL layer
    (spdnn/preprocess.py:86-113 documents the format: slice m of warp slot
    w = stage * warps_per_block + warp holds one entry per lane; the lane's
    row is block * block_size + warp * warp_size + lane, the entry's column
    plan.map[mapdispl[stage] + windex]; padding has value 0)."""
    from .model import make_layer_csr
    plan, ws = ell.plan, int(ell.warp_size)
    wpb = int(plan.block_size) // ws
    wdispl = np.asarray(ell.wdispl, np.int64)
    n_slices = int(wdispl[-1]) if len(wdispl) else 0
    idx = np.arange(n_slices * ws, dtype=np.int64)
    m, lane = idx // ws, idx % ws
    wslot = np.searchsorted(wdispl, m, side="right") - 1
    stage, warp = wslot // wpb, wslot % wpb
    block = np.searchsorted(np.asarray(plan.buffdispl, np.int64), stage, side="right") - 1
    rows = block * int(plan.block_size) + warp * ws + lane
    vals = np.asarray(ell.wvalue, np.float32)[:n_slices * ws]
    cols = np.asarray(plan.map, np.int64)[np.asarray(plan.mapdispl, np.int64)[stage] +
                                          np.asarray(ell.windex, np.int64)[:n_slices * ws]]
    keep = vals != 0
    return make_layer_csr(int(ell.neurons), rows[keep], cols[keep], vals[keep])


def baseline_layer(features: FeatureBatch, layer: LayerCSR, bias: np.ndarray):
    """One layer with one row per group (each row gathers its own columns)."""
    n = layer.neurons
    if features.neurons != n or len(bias) != n:
        raise ModelError("dimension mismatch in baseline_layer")
    plan = build_plans([layer], BASELINE_PARAMS)[0]
    return _one_layer(features, PreparedLayer(csr=layer, plan=plan, mode="baseline"),
                      np.asarray(bias, np.float32))


def compact_active(out: np.ndarray, active: np.ndarray, categories: np.ndarray,
                   total_inputs: int | None = None) -> FeatureBatch:
    """Keep only active columns with their categories (engine.py:130-142)."""
    if len(active) != out.shape[1] or len(categories) != out.shape[1]:
        raise ModelError("flag/category length must match column count")
    categories = np.asarray(categories, dtype=np.int64)
    if total_inputs is None:
        total_inputs = int(categories.max()) + 1 if len(categories) else 0
    return FeatureBatch(neurons=out.shape[0], data=np.asfortranarray(out[:, active]),
                        categories=categories[active], total_inputs=total_inputs)


def run_layer_step(features: FeatureBatch, prepared: PreparedLayer, bias: np.ndarray,
                   config: InferenceConfig, mode: Mode) -> LayerOutcome:
    """One evaluate-then-compact step (engine.py:145-170)."""
    before = features.active_count
    if before == 0:
        return LayerOutcome(0, 0, 0, 0, features=features)
    if prepared.plan is None or prepared.mode != mode:
        raise ModelError(f"prepared structures are for {prepared.mode} mode")
    out, active = _one_layer(features, prepared, np.asarray(bias, np.float32))
    tiles = -(-before // TILE)
    compacted = compact_active(out, active, features.categories,
                               total_inputs=features.total_inputs)
    return LayerOutcome(active_before=before, active_after=compacted.active_count,
                        weight_element_reads=prepared.plan.total_slots * tiles,
                        feature_element_reads=prepared.plan.num_fp * before,
                        features=compacted)
