"""Loaders and the binary cache (CPU only), pinned to bytes and parses the
reference's own ingest produced (tests/golden/make_ingest.py), plus the
reference test suite's error cases (tests/test_ingest.py of the reference:
range checks with line numbers, duplicates, truncation, bad magic/version)."""

import io

import numpy as np
import pytest

from conftest import load_npz
from paper_2007_14152_b200 import ingest
from paper_2007_14152_b200.ingest import (GeneratorSpec, IngestError, load_features_tsv,
                                          load_layer_tsv, load_truth_categories, read_binary,
                                          write_binary)
from paper_2007_14152_b200.model import (FeatureBatch, NetworkModel, make_feature_batch,
                                         validate_model)

G = load_npz("ingest.npz")


def _golden_model():
    return ingest.generate_synthetic_network(GeneratorSpec(
        neurons=64, layers=3, connections_per_neuron=8, bias_value=-0.3, seed=5))


def test_write_binary_bytes_equal_reference():
    buf = io.BytesIO()
    write_binary(_golden_model(), buf)
    assert buf.getvalue() == G["model_bin"].tobytes()
    buf = io.BytesIO()
    write_binary(ingest.generate_synthetic_inputs(64, 20, 0.3, seed=6), buf)
    assert buf.getvalue() == G["features_bin"].tobytes()


def test_read_binary_reference_bytes():
    model = read_binary(io.BytesIO(G["model_bin"].tobytes()))
    ref = _golden_model()
    assert isinstance(model, NetworkModel) and model.num_layers == 3
    for a, b in zip(model.layers, ref.layers):
        assert np.array_equal(a.row_ptr, b.row_ptr)
        assert np.array_equal(a.col_idx, b.col_idx)
        assert np.array_equal(a.values, b.values)
    assert validate_model(model) == []
    feats = read_binary(io.BytesIO(G["features_bin"].tobytes()))
    assert isinstance(feats, FeatureBatch)
    want = ingest.generate_synthetic_inputs(64, 20, 0.3, seed=6)
    assert np.array_equal(feats.data, want.data)
    assert feats.categories.tolist() == list(range(20))


def test_read_binary_into_caller_buffer():
    out = np.full((64, 20), 7.0, dtype=np.float32, order="F")
    feats = read_binary(io.BytesIO(G["features_bin"].tobytes()), out=out)
    assert np.shares_memory(feats.data, out)
    assert np.array_equal(out, ingest.generate_synthetic_inputs(64, 20, 0.3, seed=6).data)
    with pytest.raises(IngestError):
        read_binary(io.BytesIO(G["features_bin"].tobytes()), out=np.zeros((64, 20), np.float32))


def test_tsv_loaders_match_reference_parse():
    layer = load_layer_tsv(G["layer_tsv"].tobytes(), 64)
    assert np.array_equal(layer.row_ptr, G["layer_row_ptr"])
    assert np.array_equal(layer.col_idx, G["layer_col_idx"])
    assert np.array_equal(layer.values.view(np.uint32), G["layer_values"].view(np.uint32))
    feats = load_features_tsv(io.BytesIO(G["features_tsv"].tobytes()), 64, 22)
    assert np.array_equal(feats.data, G["features_data"])
    assert not feats.data[:, 20:].any()  # images never listed are zero columns
    assert load_truth_categories(b"5\n2\n\n9\n") == G["truth"].tolist() == [1, 4, 8]


@pytest.mark.parametrize("text,match", [
    (b"3\t1\t1.0\n", "row index out of range, line 1"),
    (b"1\t1\t1.0\n1\t0\t1.0\n", "column index out of range, line 2"),
    (b"1\t1\t1.0\nnot-a-number\t1\t1.0\n", "line 2"),
    (b"1\t1\n", "expected 3 tab-separated fields"),
    (b"1\t1\t1.0\n1\t1\t2.0\n", "duplicate"),
])
def test_layer_tsv_errors(text, match):
    with pytest.raises(IngestError, match=match):
        load_layer_tsv(text, neurons=2)


def test_layer_tsv_order_free_and_empty():
    lines = [b"2\t1\t0.5", b"1\t2\t0.25", b"2\t2\t1.0", b"1\t1\t0.125"]
    a = load_layer_tsv(b"\n".join(lines), neurons=2)
    b = load_layer_tsv(b"\n".join(reversed(lines)) + b"\n\n", neurons=2)
    assert a.row_ptr.tolist() == b.row_ptr.tolist() == [0, 2, 4]
    assert a.col_idx.tolist() == b.col_idx.tolist() == [0, 1, 0, 1]
    assert a.values.tolist() == b.values.tolist() == [0.125, 0.25, 0.5, 1.0]
    empty = load_layer_tsv(b"", neurons=3)
    assert empty.row_ptr.tolist() == [0, 0, 0, 0] and empty.nnz == 0


def test_features_tsv_errors_and_last_value_wins():
    with pytest.raises(IngestError, match="image index out of range, line 1"):
        load_features_tsv(b"3\t1\t1\n", neurons=2, max_inputs=2)
    with pytest.raises(IngestError, match="neuron index out of range, line 2"):
        load_features_tsv(b"1\t1\t1\n1\t5\t1\n", neurons=2, max_inputs=2)
    b = load_features_tsv(b"1\t2\t3.0\n1\t2\t0.5\n", neurons=2, max_inputs=1)
    assert b.data[:, 0].tolist() == [0.0, 0.5]


def test_truth_errors():
    with pytest.raises(IngestError, match="duplicate category 3"):
        load_truth_categories(b"3\n1\n3\n")
    with pytest.raises(IngestError, match="line 2"):
        load_truth_categories(b"1\nx\n")


def test_binary_errors():
    with pytest.raises(IngestError, match="bad magic"):
        read_binary(io.BytesIO(b"XXXX" + bytes(8)))
    bad_version = b"SPDN" + np.array([2, 1, 1], "<u4").tobytes()
    with pytest.raises(IngestError, match="unsupported format version 2"):
        read_binary(io.BytesIO(bad_version))
    with pytest.raises(IngestError, match="truncated"):
        read_binary(io.BytesIO(G["model_bin"].tobytes()[:-3]))
    partial = make_feature_batch(4, np.ones((4, 2), np.float32), categories=[1, 3],
                                 total_inputs=4)
    with pytest.raises(IngestError, match="only full input batches"):
        write_binary(partial, io.BytesIO())
    with pytest.raises(TypeError):
        write_binary(object(), io.BytesIO())


def test_streamed_layers_and_inputs_into_buffer():
    spec = GeneratorSpec(neurons=96, layers=4, connections_per_neuron=6, seed=11)
    whole = ingest.generate_synthetic_network(spec)
    for a, b in zip(whole.layers, ingest.iter_synthetic_layers(spec)):
        assert np.array_equal(a.col_idx, b.col_idx) and np.array_equal(a.values, b.values)
    out = np.empty((96, 33), np.float32, order="F")
    got = ingest.generate_synthetic_inputs(96, 33, 0.4, seed=3, out=out, chunk_rows=7)
    assert np.shares_memory(got.data, out)
    assert np.array_equal(out, ingest.generate_synthetic_inputs(96, 33, 0.4, seed=3).data)


def test_inputs_column_range_is_the_same_stream():
    full = ingest.generate_synthetic_inputs(40, 50, 0.3, seed=4, chunk_rows=9)
    part = ingest.generate_synthetic_inputs(40, 50, 0.3, seed=4, columns=(13, 31))
    assert np.array_equal(part.data, full.data[:, 13:31])
    assert part.categories.tolist() == list(range(13, 31)) and part.total_inputs == 50
