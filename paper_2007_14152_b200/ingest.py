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
# challenge TSV files (formats and IngestError cases of spdnn/ingest.py:56-135)
#
# Parsing is vectorised: the whole text is decoded once, split into lines
# (universal newlines, as a text stream reads them), and the well-formed case
# is converted by numpy's C parser in one call. Only when that fails are the
# lines scanned one by one, to report the first bad line exactly as the
# reference does ("parse error, line N: ...").

def _text_lines(source: Union[bytes, BinaryIO]) -> tuple:
    """(stripped non-blank lines, their 1-based line numbers)."""
    raw = source if isinstance(source, (bytes, bytearray)) else source.read()
    try:
        text = bytes(raw).decode("ascii")
    except UnicodeDecodeError as exc:
        raise IngestError(f"parse error: non-ASCII byte at offset {exc.start}") from None
    lines = text.replace("\r\n", "\n").replace("\r", "\n").split("\n")
    keep = [(i + 1, ln.strip()) for i, ln in enumerate(lines) if ln.strip()]
    return [ln for _, ln in keep], np.array([i for i, _ in keep], dtype=np.int64)


def _first_bad_line(lines, linenos, fields: int, kinds: str) -> None:
    """Raise the reference's message for the first line that does not parse
    as `fields` tab-separated values of `kinds` ('i' int, 'f' float)."""
    for ln, no in zip(lines, linenos.tolist()):
        parts = ln.split("\t") if fields > 1 else [ln]
        if len(parts) != fields:
            raise IngestError(f"parse error, line {no}: expected {fields} tab-separated fields")
        try:
            for part, kind in zip(parts, kinds):
                (int if kind == "i" else float)(part)
        except ValueError:
            what = "bad integer or float" if fields > 1 else "bad integer"
            raise IngestError(f"parse error, line {no}: {what}") from None


def _columns(lines, linenos, fields: int, kinds: str) -> list:
    """The lines as `fields` numpy columns (int64 / float64)."""
    if not lines:
        return [np.zeros(0, np.int64 if k == "i" else np.float64) for k in kinds]
    arr = None
    if all(ln.count("\t") == fields - 1 for ln in lines):
        dt = [(f"c{j}", "<i8" if k == "i" else "<f8") for j, k in enumerate(kinds)]
        try:
            arr = np.loadtxt(io.StringIO("\n".join(lines)), delimiter="\t" if fields > 1 else None,
                             dtype=dt, ndmin=1, comments=None)
        except ValueError:
            arr = None
    if arr is None or arr.shape[0] != len(lines):
        _first_bad_line(lines, linenos, fields, kinds)
        # numpy refused a line Python accepts (e.g. "1_0"): convert per line
        conv = [[(int if k == "i" else float)(x) for x, k in
                 zip(ln.split("\t") if fields > 1 else [ln], kinds)] for ln in lines]
        return [np.array([c[j] for c in conv], np.int64 if k == "i" else np.float64)
                for j, k in enumerate(kinds)]
    return [arr[f"c{j}"] for j in range(fields)]


def _checked_triplets(source, hi_a: int, hi_b: int, what_a: str, what_b: str):
    """(a - 1, b - 1, value) of the non-blank lines; 1-based range checks,
    the first offending line (in line order) reported as the reference does."""
    lines, linenos = _text_lines(source)
    a, b, v = _columns(lines, linenos, 3, "iif")
    bad_a = (a < 1) | (a > hi_a)
    bad_b = (b < 1) | (b > hi_b)
    bad = bad_a | bad_b
    if bad.any():
        j = int(np.argmax(bad))
        what = what_a if bad_a[j] else what_b
        raise IngestError(f"{what} index out of range, line {int(linenos[j])}")
    return a - 1, b - 1, v.astype(np.float32)


def load_layer_tsv(source: Union[bytes, BinaryIO], neurons: int) -> LayerCSR:
    """One weight layer from ``row<TAB>col<TAB>value`` lines (1-indexed); line
    order is free, a repeated (row, col) is an error (ingest.py:67-90)."""
    rows, cols, vals = _checked_triplets(source, neurons, neurons, "row", "column")
    try:
        return make_layer_csr(neurons, rows, cols, vals)
    except ModelError as exc:
        raise IngestError(str(exc)) from None


def load_features_tsv(source: Union[bytes, BinaryIO], neurons: int,
                      max_inputs: int) -> FeatureBatch:
    """Features from ``image<TAB>neuron<TAB>value`` lines (1-indexed) into a
    dense (N, max_inputs) Fortran batch; absent images are zero columns and a
    repeated (image, neuron) keeps the last value (ingest.py:93-111)."""
    img, neu, vals = _checked_triplets(source, max_inputs, neurons, "image", "neuron")
    data = np.zeros((neurons, max_inputs), dtype=np.float32, order="F")
    data[neu, img] = vals  # numpy assigns repeated indices in order: last wins
    return make_feature_batch(neurons, data)


def load_truth_categories(source: Union[bytes, BinaryIO]) -> list:
    """Sorted 0-based categories from one 1-based integer per line;
    duplicates are rejected (ingest.py:114-132)."""
    lines, linenos = _text_lines(source)
    (cats,) = _columns(lines, linenos, 1, "i")
    cats = np.sort(cats)
    dup = np.nonzero(cats[1:] == cats[:-1])[0]
    if dup.size:
        raise IngestError(f"duplicate category {int(cats[dup[0]])}")
    return (cats - 1).tolist()


# ---------------------------------------------------------------------------
# binary cache (byte formats of spdnn/ingest.py:182-270), little-endian:
#   model    "SPDN" | u32 version | u32 N | u32 L | per layer: u64 nnz,
#            u64 row_ptr[N+1], u32 col_idx[nnz], f32 values[nnz] | f32 bias[N]
#   features "SPDF" | u32 version | u32 N | u32 M | u64 nnz |
#            nnz x (u32 image, u32 neuron, f32 value), image-major

_FEATURE_RECORD = np.dtype([("img", "<u4"), ("neu", "<u4"), ("val", "<f4")])


def _model_chunks(model: NetworkModel) -> Iterator[bytes]:
    yield MODEL_MAGIC + np.array([FORMAT_VERSION, model.neurons, model.num_layers],
                                 "<u4").tobytes()
    for layer in model.layers:
        yield np.array([layer.nnz], "<u8").tobytes()
        yield layer.row_ptr.astype("<u8").tobytes()
        yield layer.col_idx.astype("<u4").tobytes()
        yield layer.values.astype("<f4").tobytes()
    yield np.asarray(model.bias).astype("<f4").tobytes()


def _feature_chunks(batch: FeatureBatch) -> Iterator[bytes]:
    if not np.array_equal(batch.categories, np.arange(batch.total_inputs)):
        raise IngestError("only full input batches can be cached")
    dense = np.asarray(batch.data)
    img, neu = np.nonzero(dense.T)  # image-major: all of image 0's nonzeros first
    recs = np.empty(img.shape[0], _FEATURE_RECORD)
    recs["img"], recs["neu"], recs["val"] = img, neu, dense[neu, img]
    yield FEATURES_MAGIC + np.array([FORMAT_VERSION, batch.neurons, batch.active_count],
                                    "<u4").tobytes()
    yield np.array([recs.shape[0]], "<u8").tobytes()
    yield recs.tobytes()


def write_binary(obj: Union[NetworkModel, FeatureBatch], dest: BinaryIO) -> None:
    """Serialize a model or a full input batch (ingest.py:198-224), one
    section at a time (a 65536 x 1920 model is never concatenated in memory)."""
    if isinstance(obj, NetworkModel):
        chunks = _model_chunks(obj)
    elif isinstance(obj, FeatureBatch):
        chunks = _feature_chunks(obj)
    else:
        raise TypeError(f"cannot serialize {type(obj).__name__}")
    for chunk in chunks:
        dest.write(chunk)


def _buffer_of(src: BinaryIO) -> memoryview:
    """The stream's remaining bytes without a copy when it is a regular file
    (memory-mapped) or an in-memory buffer; otherwise read once."""
    if isinstance(src, io.BytesIO):
        return src.getbuffer()[src.tell():]
    try:
        import mmap
        fd = src.fileno()
        start = src.tell()
        mm = mmap.mmap(fd, 0, access=mmap.ACCESS_READ)
        return memoryview(mm)[start:]
    except (AttributeError, OSError, ValueError, io.UnsupportedOperation):
        return memoryview(src.read())


def read_binary(src: BinaryIO, out: np.ndarray | None = None
                ) -> Union[NetworkModel, FeatureBatch]:
    """Read back what write_binary produced, dispatching on the magic
    (ingest.py:242-270). The stream is viewed as one buffer (memory-mapped
    when it is a file) and sliced with np.frombuffer. ``out`` (extension,
    features only): an (N, M) Fortran float32 array to scatter the records
    into -- e.g. a pinned host buffer, so the batch can be uploaded without
    another host copy."""
    buf = _buffer_of(src)
    pos = 0

    def take(dtype: str, count: int = 1) -> np.ndarray:
        nonlocal pos
        dt = np.dtype(dtype)
        end = pos + dt.itemsize * count
        if end > len(buf):
            raise IngestError("truncated file")
        arr = np.frombuffer(buf[pos:end], dtype=dt)
        pos = end
        return arr

    if len(buf) < 4 or bytes(buf[:4]) not in (MODEL_MAGIC, FEATURES_MAGIC):
        raise IngestError("bad magic")
    magic = bytes(buf[:4])
    pos = 4
    version = int(take("<u4")[0])
    if version != FORMAT_VERSION:
        raise IngestError(f"unsupported format version {version}")
    n, count = (int(x) for x in take("<u4", 2))
    if magic == MODEL_MAGIC:
        layers = []
        for _ in range(count):
            nnz = int(take("<u8")[0])
            row_ptr = take("<u8", n + 1).astype(np.int64)
            col_idx = take("<u4", nnz).astype(np.int32)
            values = take("<f4", nnz).astype(np.float32)
            layers.append(LayerCSR(row_ptr=row_ptr, col_idx=col_idx, values=values))
        bias = take("<f4", n).astype(np.float32)
        return NetworkModel(neurons=n, layers=tuple(layers), bias=bias)
    m = count
    recs = take(_FEATURE_RECORD, int(take("<u8")[0]))
    if out is not None:
        if out.shape != (n, m) or out.dtype != np.float32 or not out.flags.f_contiguous:
            raise IngestError("out must be an (N, M) Fortran float32 array")
        data = out
        data[...] = 0.0
    else:
        data = np.zeros((n, m), dtype=np.float32, order="F")
    if recs.size and (int(recs["neu"].max()) >= n or int(recs["img"].max()) >= m):
        raise IngestError("record index out of range")
    data[recs["neu"], recs["img"]] = recs["val"]
    return make_feature_batch(n, data)
