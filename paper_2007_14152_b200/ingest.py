"""Synthetic Graph-Challenge-style networks and inputs (host data preparation).

This is the boundary data source, not the accelerated path: the bench and the
parity tests need the *same* networks and inputs the reference builds, bit for
bit, on a box where the reference itself is absent. The draw sequence follows
``spdnn/ingest.py:140-180``:

* per layer: ``offset = rng.integers(1, N)``, then a stride redrawn with
  ``rng.integers(1, N)`` until ``gcd(stride, N) == 1``; row ``r`` connects to
  ``{(r*offset + i*stride) mod N : i < K}`` (sorted), every weight 1/16, one
  constant bias;
* inputs: ``rng.random((N, M)) < density`` in row-major draw order.

Inputs are produced in row chunks so the 65536 x 60000 case never builds the
31 GB float64 temporary; the chunked stream equals the one-shot stream
(PCG64 ``random`` fills row-major). Layers can be
streamed one at a time (``iter_synthetic_layers``): the 65536 x 1920 network's
CSR is 32 GB of host memory, its device layout is built chunk by chunk.

The challenge-file loaders (``load_layer_tsv``, ``load_features_tsv``,
``load_truth_categories``) and the binary cache (``write_binary`` /
``read_binary``) follow ``spdnn/ingest.py:56-135,182-270``: same formats,
same 1-based-on-disk convention, same ``IngestError`` cases.
"""

from __future__ import annotations

import io
import math
from dataclasses import dataclass
from typing import BinaryIO, Iterator, Union

import numpy as np

from .model import (FeatureBatch, LayerCSR, ModelError, NetworkModel, make_feature_batch,
                    make_layer_csr)

MODEL_MAGIC = b"SPDN"
FEATURES_MAGIC = b"SPDF"
FORMAT_VERSION = 1


class IngestError(ValueError):
    """Malformed TSV or binary input (``spdnn/ingest.py:33-34``)."""

WEIGHT_VALUE = np.float32(0.0625)


@dataclass(frozen=True)
class GeneratorSpec:
    """Synthetic fixed-fan-in network parameters (``spdnn/ingest.py:37-53``)."""

    neurons: int
    layers: int
    connections_per_neuron: int = 32
    bias_value: float = -0.3
    seed: int = 0
    input_count: int = 0
    input_density: float = 0.3

    def __post_init__(self):
        if self.connections_per_neuron > self.neurons:
            raise ModelError("connections_per_neuron cannot exceed neurons")
        if not 0.0 < self.input_density <= 1.0:
            raise ModelError("input_density must be in (0, 1]")


def layer_parameters(neurons: int, layers: int, seed: int) -> list[tuple[int, int]]:
    """(offset, stride) per layer, drawn exactly as the reference draws them."""
    rng = np.random.default_rng(seed)
    params = []
    for _ in range(layers):
        offset = int(rng.integers(1, neurons)) if neurons > 1 else 0
        stride = 1
        if neurons > 1:
            while True:
                stride = int(rng.integers(1, neurons))
                if math.gcd(stride, neurons) == 1:
                    break
        params.append((offset, stride))
    return params


def synthetic_layer(neurons: int, k: int, offset: int, stride: int) -> LayerCSR:
    """Row r -> sorted {(r*offset + i*stride) mod N}, all weights 1/16."""
    base = (np.arange(neurons, dtype=np.int64) * offset) % neurons
    # base + i*stride < (k + 1) * N: int32 when that fits (sorting 3x faster)
    dt = np.int32 if (k + 1) * neurons < 2 ** 31 else np.int64
    cols = (base.astype(dt)[:, None] + (np.arange(k, dtype=np.int64) * stride).astype(dt)[None, :]) \
        % dt(neurons)
    cols.sort(axis=1)
    return LayerCSR(row_ptr=np.arange(0, neurons * k + 1, k, dtype=np.int64),
                    col_idx=cols.reshape(-1).astype(np.int32),
                    values=np.full(neurons * k, WEIGHT_VALUE, dtype=np.float32))


def iter_synthetic_layers(spec: GeneratorSpec) -> Iterator[LayerCSR]:
    """The layers of ``generate_synthetic_network(spec)``, one at a time."""
    n, k = spec.neurons, spec.connections_per_neuron
    for off, st in layer_parameters(n, spec.layers, spec.seed):
        yield synthetic_layer(n, k, off, st)


def synthetic_bias(spec: GeneratorSpec) -> np.ndarray:
    return np.full(spec.neurons, np.float32(spec.bias_value), dtype=np.float32)


def generate_synthetic_network(spec: GeneratorSpec) -> NetworkModel:
    return NetworkModel(neurons=spec.neurons, layers=tuple(iter_synthetic_layers(spec)),
                        bias=synthetic_bias(spec))


def generate_synthetic_inputs(neurons: int, count: int, density: float, seed: int,
                              chunk_rows: int = 1024, out: np.ndarray | None = None,
                              columns: tuple | None = None) -> FeatureBatch:
    """Bernoulli(density) binary features, (N, M) Fortran fp32, categories 0..M-1.

    Extensions: ``out`` is an (N, M) Fortran float32 array to fill (e.g. the
    numpy view of a pinned host buffer, so a 15.7 GB batch is not copied);
    ``columns=(lo, hi)`` keeps only inputs lo..hi-1 of the same stream (one
    rank's shard; categories lo..hi-1, total_inputs = count)."""
    rng = np.random.default_rng(seed)
    lo, hi = (0, count) if columns is None else (int(columns[0]), int(columns[1]))
    if not 0 <= lo <= hi <= count:
        raise ModelError("columns must satisfy 0 <= lo <= hi <= count")
    if out is not None:
        if out.shape != (neurons, hi - lo) or out.dtype != np.float32 or \
                not out.flags.f_contiguous:
            raise ModelError("out must be an (N, M) Fortran float32 array")
        data = out
    else:
        data = np.empty((neurons, hi - lo), dtype=np.float32, order="F")
    thr = float(density)
    for r0 in range(0, neurons, chunk_rows):
        r1 = min(neurons, r0 + chunk_rows)
        draw = rng.random((r1 - r0, count))
        data[r0:r1, :] = draw[:, lo:hi] < thr
    return FeatureBatch(neurons=neurons, data=data,
                        categories=np.arange(lo, hi, dtype=np.int64), total_inputs=count)


# ---------------------------------------------------------------------------
# challenge TSV files (spdnn/ingest.py:56-135)

def _lines(source: Union[bytes, BinaryIO]) -> io.TextIOBase:
    if isinstance(source, bytes):
        source = io.BytesIO(source)
    return io.TextIOWrapper(source, encoding="ascii")


def _parse_triplet(line: str, lineno: int) -> tuple:
    parts = line.split("\t")
    if len(parts) != 3:
        raise IngestError(f"parse error, line {lineno}: expected 3 tab-separated fields")
    try:
        return int(parts[0]), int(parts[1]), float(parts[2])
    except ValueError:
        raise IngestError(f"parse error, line {lineno}: bad integer or float") from None


def _triplets(source, lo_hi_a, lo_hi_b, what_a: str, what_b: str):
    """(a-1, b-1, value) arrays of the non-blank lines; 1-based range checks
    in line order, as the reference does them."""
    a_s, b_s, v_s = [], [], []
    for lineno, line in enumerate(_lines(source), start=1):
        line = line.strip()
        if not line:
            continue
        a, b, v = _parse_triplet(line, lineno)
        if not 1 <= a <= lo_hi_a:
            raise IngestError(f"{what_a} index out of range, line {lineno}")
        if not 1 <= b <= lo_hi_b:
            raise IngestError(f"{what_b} index out of range, line {lineno}")
        a_s.append(a - 1)
        b_s.append(b - 1)
        v_s.append(v)
    return (np.array(a_s, dtype=np.int64), np.array(b_s, dtype=np.int64),
            np.array(v_s, dtype=np.float32))


def load_layer_tsv(source: Union[bytes, BinaryIO], neurons: int) -> LayerCSR:
    """One weight layer from ``row<TAB>col<TAB>value`` lines (1-indexed); line
    order is free, a repeated (row, col) is an error (ingest.py:67-90)."""
    rows, cols, vals = _triplets(source, neurons, neurons, "row", "column")
    try:
        return make_layer_csr(neurons, rows, cols, vals)
    except ModelError as exc:
        raise IngestError(str(exc)) from None


def load_features_tsv(source: Union[bytes, BinaryIO], neurons: int,
                      max_inputs: int) -> FeatureBatch:
    """Features from ``image<TAB>neuron<TAB>value`` lines (1-indexed) into a
    dense (N, max_inputs) Fortran batch; absent images are zero columns and a
    repeated (image, neuron) keeps the last value (ingest.py:93-111)."""
    img, neu, vals = _triplets(source, max_inputs, neurons, "image", "neuron")
    data = np.zeros((neurons, max_inputs), dtype=np.float32, order="F")
    data[neu, img] = vals  # numpy assigns repeated indices in order: last wins
    return make_feature_batch(neurons, data)


def load_truth_categories(source: Union[bytes, BinaryIO]) -> list:
    """Sorted 0-based categories from one 1-based integer per line;
    duplicates are rejected (ingest.py:114-132)."""
    cats = []
    for lineno, line in enumerate(_lines(source), start=1):
        line = line.strip()
        if not line:
            continue
        try:
            cats.append(int(line))
        except ValueError:
            raise IngestError(f"parse error, line {lineno}: bad integer") from None
    cats.sort()
    for a, b in zip(cats, cats[1:]):
        if a == b:
            raise IngestError(f"duplicate category {a}")
    return [c - 1 for c in cats]


# ---------------------------------------------------------------------------
# binary cache (spdnn/ingest.py:182-270), little-endian:
#   model    "SPDN" | u32 version | u32 N | u32 L | per layer: u64 nnz,
#            u64 row_ptr[N+1], u32 col_idx[nnz], f32 values[nnz] | f32 bias[N]
#   features "SPDF" | u32 version | u32 N | u32 M | u64 nnz |
#            nnz x (u32 image, u32 neuron, f32 value), image-major

_REC = np.dtype([("img", "<u4"), ("neu", "<u4"), ("val", "<f4")])


def _put(out: BinaryIO, arr, dtype: str) -> None:
    out.write(np.ascontiguousarray(arr).astype(dtype).tobytes())


def write_binary(obj: Union[NetworkModel, FeatureBatch], dest: BinaryIO) -> None:
    """Serialize a model or a full input batch (ingest.py:198-224)."""
    if isinstance(obj, NetworkModel):
        dest.write(MODEL_MAGIC)
        _put(dest, np.array([FORMAT_VERSION, obj.neurons, obj.num_layers]), "<u4")
        for layer in obj.layers:
            _put(dest, np.array([layer.nnz]), "<u8")
            _put(dest, layer.row_ptr, "<u8")
            _put(dest, layer.col_idx, "<u4")
            _put(dest, layer.values, "<f4")
        _put(dest, obj.bias, "<f4")
    elif isinstance(obj, FeatureBatch):
        if not np.array_equal(obj.categories, np.arange(obj.total_inputs)):
            raise IngestError("only full input batches can be cached")
        dest.write(FEATURES_MAGIC)
        image_idx, neuron_idx = np.nonzero(obj.data.T)  # image-major record order
        _put(dest, np.array([FORMAT_VERSION, obj.neurons, obj.active_count]), "<u4")
        _put(dest, np.array([len(image_idx)]), "<u8")
        rec = np.empty(len(image_idx), dtype=_REC)
        rec["img"] = image_idx
        rec["neu"] = neuron_idx
        rec["val"] = obj.data[neuron_idx, image_idx]
        dest.write(rec.tobytes())
    else:
        raise TypeError(f"cannot serialize {type(obj).__name__}")


class _Reader:
    def __init__(self, src: BinaryIO):
        self._src = src

    def take(self, nbytes: int) -> bytes:
        buf = self._src.read(nbytes)
        if len(buf) != nbytes:
            raise IngestError("truncated file")
        return buf

    def scalar(self, dtype: str) -> int:
        dt = np.dtype(dtype)
        return int(np.frombuffer(self.take(dt.itemsize), dtype=dt)[0])

    def array(self, count: int, dtype: str) -> np.ndarray:
        dt = np.dtype(dtype)
        return np.frombuffer(self.take(dt.itemsize * count), dtype=dt)


def read_binary(src: BinaryIO, out: np.ndarray | None = None
                ) -> Union[NetworkModel, FeatureBatch]:
    """Read back what write_binary produced, dispatching on the magic
    (ingest.py:242-270). ``out`` (extension, features only): an (N, M)
    Fortran float32 array to scatter the records into -- e.g. a pinned host
    buffer, so the batch can be uploaded without another host copy."""
    rd = _Reader(src)
    magic = rd.take(4)
    if magic not in (MODEL_MAGIC, FEATURES_MAGIC):
        raise IngestError("bad magic")
    version = rd.scalar("<u4")
    if version != FORMAT_VERSION:
        raise IngestError(f"unsupported format version {version}")
    if magic == MODEL_MAGIC:
        n = rd.scalar("<u4")
        num_layers = rd.scalar("<u4")
        layers = []
        for _ in range(num_layers):
            nnz = rd.scalar("<u8")
            row_ptr = rd.array(n + 1, "<u8").astype(np.int64)
            col_idx = rd.array(nnz, "<u4").astype(np.int32)
            values = rd.array(nnz, "<f4").astype(np.float32)
            layers.append(LayerCSR(row_ptr=row_ptr, col_idx=col_idx, values=values))
        bias = rd.array(n, "<f4").astype(np.float32)
        return NetworkModel(neurons=n, layers=tuple(layers), bias=bias)
    n = rd.scalar("<u4")
    m = rd.scalar("<u4")
    nnz = rd.scalar("<u8")
    rec = np.frombuffer(rd.take(_REC.itemsize * nnz), dtype=_REC)
    if out is not None:
        if out.shape != (n, m) or out.dtype != np.float32 or not out.flags.f_contiguous:
            raise IngestError("out must be an (N, M) Fortran float32 array")
        data = out
        data[...] = 0.0
    else:
        data = np.zeros((n, m), dtype=np.float32, order="F")
    if nnz and (int(rec["neu"].max()) >= n or int(rec["img"].max()) >= m):
        raise IngestError("record index out of range")
    data[rec["neu"], rec["img"]] = rec["val"]
    return make_feature_batch(n, data)
