"""Run reports in the reference's structured-text schema, with the B200 figures.

The line format is the reference's (``spdnn/report.py:1-120``, schema 1):
``key: value`` scalars, then ``table NAME: <columns>`` ... ``end`` blocks, so
its ``parse_report`` / ``strip_timing`` read these reports unchanged. The
reference's scalars and tables come first, in its order; the B200 figures
are extra scalars after them (a parser keyed by name ignores what it does
not know):

    device_seconds      CUDA-event time of the layer loop
    te_per_second       credited TeraEdges/s (edges_processed / elapsed)
    hbm_bytes           algorithmic HBM bytes, sum over layers of
                        8*N*M_l + 6*nnz_l + 4*N
    roofline_fraction   hbm_bytes / device_seconds / hbm_peak
    hbm_peak_gbs        the peak it is measured against
    imbalance_max_before / imbalance_max_after / rebalances
                        load imbalance of the batch-parallel run

Timing lines (elapsed_seconds, edges_per_second, device_seconds,
te_per_second, roofline_fraction) are the ones a rerun changes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SCHEMA_VERSION = 1
TIMING_KEYS = ("elapsed_seconds", "edges_per_second", "device_seconds", "te_per_second",
               "roofline_fraction")


@dataclass(frozen=True)
class IndexReport:
    """Bytes of the index-bearing layout arrays (the reference's
    CompactIndexReport fields). The B200 layout stores 32-bit record words
    and staged-row lists; nothing is narrowed, so wide == narrow."""
    wide_bytes: int
    narrow_bytes: int
    reduction: float


@dataclass
class RunReport:
    neurons: int
    layers: int
    inputs: int
    mode: str
    workers: int
    minibatch: int
    block_size: int
    warp_size: int
    buffer_capacity: int
    streaming: bool
    rebalance_threshold: float
    elapsed_seconds: float
    edges_processed: int
    weight_element_reads: int
    feature_element_reads: int
    per_layer_active_counts: list
    padding_stats: object
    index_report: IndexReport
    comm_matrix: object | None = None
    balance_report: object | None = None
    verified: bool | None = None
    device_seconds: float = 0.0
    hbm_bytes: int = 0
    hbm_peak_gbs: float = 0.0

    @property
    def edges_per_second(self) -> float:
        return self.edges_processed / self.elapsed_seconds if self.elapsed_seconds else math.inf

    @property
    def te_per_second(self) -> float:
        return self.edges_per_second / 1e12

    @property
    def roofline_fraction(self) -> float:
        if not self.device_seconds or not self.hbm_peak_gbs:
            return 0.0
        return self.hbm_bytes / self.device_seconds / (self.hbm_peak_gbs * 1e9)


def algorithmic_bytes(neurons: int, nnz: list, counts: list) -> int:
    """sum over active layers of 8*N*M_l + 6*nnz_l + 4*N."""
    return int(sum(8 * neurons * before + 6 * z + 4 * neurons
                   for (before, _), z in zip(counts, nnz) if before))


def _combine_padding(stats):
    from .engine import PaddingStats
    nnz = sum(s.nnz for s in stats)
    w = sum(s.warp_padded_slots for s in stats)
    t = sum(s.tile_padded_slots for s in stats)
    l_ = sum(s.layer_padded_slots for s in stats)
    if nnz == 0:
        return PaddingStats(0, w, t, l_, 0.0, 0.0, 0.0, empty=True)
    return PaddingStats(nnz, w, t, l_, w / nnz, t / nnz, l_ / nnz)


def index_report(prepared) -> IndexReport:
    total = 0
    for p in prepared:
        pl = p.plan
        total += 4 * (pl.records.size + pl.meta.size + pl.blocks.size + pl.stages.size)
    return IndexReport(total, total, 0.0)


def build_report(model, inputs, config, mode: str, prepared, result, comm=None, balance=None,
                 verified=None, hbm_peak_gbs: float = 0.0) -> RunReport:
    """A RunReport for one engine.infer / parallel.run_batch_parallel run."""
    counts = [(o.active_before, o.active_after) for o in result.per_layer]
    return RunReport(
        neurons=model.neurons, layers=model.num_layers, inputs=inputs.total_inputs, mode=mode,
        workers=config.workers, minibatch=config.minibatch, block_size=config.block_size,
        warp_size=config.warp_size, buffer_capacity=config.buffer_capacity,
        streaming=config.streaming, rebalance_threshold=config.rebalance_threshold,
        elapsed_seconds=result.elapsed_seconds, edges_processed=result.edges_processed,
        weight_element_reads=sum(o.weight_element_reads for o in result.per_layer),
        feature_element_reads=sum(o.feature_element_reads for o in result.per_layer),
        per_layer_active_counts=counts,
        padding_stats=_combine_padding([p.padding for p in prepared]),
        index_report=index_report(prepared), comm_matrix=comm, balance_report=balance,
        verified=verified, device_seconds=getattr(result, "device_seconds", 0.0),
        hbm_bytes=algorithmic_bytes(model.neurons, [l.nnz for l in model.layers], counts),
        hbm_peak_gbs=hbm_peak_gbs)


def render_report(r: RunReport) -> str:
    lines = [f"spdnn_report: {SCHEMA_VERSION}"]
    for key in ("neurons", "layers", "inputs", "mode", "workers", "minibatch", "block_size",
                "warp_size", "buffer_capacity"):
        lines.append(f"{key}: {getattr(r, key)}")
    lines += [f"streaming: {'on' if r.streaming else 'off'}",
              f"rebalance_threshold: {r.rebalance_threshold!r}",
              f"elapsed_seconds: {r.elapsed_seconds!r}",
              f"edges_processed: {r.edges_processed}",
              f"edges_per_second: {r.edges_per_second!r}",
              f"weight_element_reads: {r.weight_element_reads}",
              f"feature_element_reads: {r.feature_element_reads}",
              f"index_bytes_wide: {r.index_report.wide_bytes}",
              f"index_bytes_narrow: {r.index_report.narrow_bytes}",
              f"index_reduction: {r.index_report.reduction!r}"]
    if r.verified is not None:
        lines.append(f"verified: {'yes' if r.verified else 'no'}")
    # B200 figures
    lines += [f"device_seconds: {r.device_seconds!r}",
              f"te_per_second: {r.te_per_second!r}",
              f"hbm_bytes: {r.hbm_bytes}",
              f"hbm_peak_gbs: {r.hbm_peak_gbs!r}",
              f"roofline_fraction: {r.roofline_fraction!r}"]
    if r.balance_report is not None:
        ent = r.balance_report.entries
        fin = [e for e in ent if np.isfinite(e.imbalance_before)]
        lines += [f"imbalance_max_before: {max((e.imbalance_before for e in fin), default=1.0)!r}",
                  f"imbalance_max_after: "
                  f"{max((e.imbalance_after for e in fin if np.isfinite(e.imbalance_after)), default=1.0)!r}",
                  f"rebalances: {sum(e.rebalanced for e in ent)}"]
    lines.append("table per_layer_active: layer before after")
    lines += [f"  {l} {b} {a}" for l, (b, a) in enumerate(r.per_layer_active_counts)]
    lines.append("end")
    p = r.padding_stats
    lines.append("table padding_stats: nnz warp_padded tile_padded layer_padded"
                 " warp_overhead tile_overhead layer_overhead")
    lines.append(f"  {p.nnz} {p.warp_padded_slots} {p.tile_padded_slots} {p.layer_padded_slots}"
                 f" {p.warp_overhead!r} {p.tile_overhead!r} {p.layer_overhead!r}")
    lines.append("end")
    if r.comm_matrix is not None:
        lines.append("table comm_matrix: rows_sent_by_worker_i_to_worker_j")
        lines += ["  " + " ".join(str(int(v)) for v in row) for row in r.comm_matrix.matrix]
        lines.append("end")
    if r.balance_report is not None:
        lines.append("table balance: layer moved imbalance_before imbalance_after rebalanced"
                     " before_counts after_counts")
        for e in r.balance_report.entries:
            lines.append(f"  {e.layer} {e.moved_rows} {e.imbalance_before!r}"
                         f" {e.imbalance_after!r} {int(e.rebalanced)}"
                         f" {'|'.join(map(str, e.before_counts))}"
                         f" {'|'.join(map(str, e.after_counts))}")
        lines.append("end")
    return "\n".join(lines) + "\n"


@dataclass
class ParsedReport:
    scalars: dict = field(default_factory=dict)
    tables: dict = field(default_factory=dict)

    def number(self, key: str) -> float:
        return float(self.scalars[key])


def parse_report(text: str) -> ParsedReport:
    """Scalars and raw table rows of a rendered report (either package's)."""
    out = ParsedReport()
    rows = None
    for raw in text.splitlines():
        line = raw.rstrip()
        if not line:
            continue
        if rows is not None:
            if line == "end":
                rows = None
            else:
                rows.append(line.split())
            continue
        if line.startswith("table "):
            name = line[len("table "):].split(":", 1)[0]
            rows = out.tables.setdefault(name, [])
            continue
        key, sep, value = line.partition(": ")
        if not sep:
            raise ValueError(f"malformed report line: {line!r}")
        out.scalars[key] = value
    if rows is not None:
        raise ValueError("unterminated table")
    return out


def strip_timing(text: str) -> str:
    """The report without the lines a rerun changes."""
    return "".join(ln + "\n" for ln in text.splitlines()
                   if ln.split(":", 1)[0] not in TIMING_KEYS)
