"""Binary-cache and TSV fixtures written by the reference's own ingest
(``spdnn/ingest.py``), so the loaders here are pinned to its byte format.

Run in the build container, where /root/reference exists:

    python tests/golden/make_ingest.py

Output (committed): ingest.npz -- the reference's write_binary bytes for a
small synthetic model and a feature batch, plus the TSV text of one layer and
of the features (challenge conventions, 1-based) and what its loaders return.
"""

from __future__ import annotations

import io
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    from spdnn import ingest

    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=64, layers=3, connections_per_neuron=8, bias_value=-0.3, seed=5))
    feats = ingest.generate_synthetic_inputs(64, 20, 0.3, seed=6)
    mb, fb = io.BytesIO(), io.BytesIO()
    ingest.write_binary(model, mb)
    ingest.write_binary(feats, fb)
    lay = model.layers[1]
    rows = np.repeat(np.arange(64), np.diff(lay.row_ptr))
    order = np.random.default_rng(9).permutation(lay.nnz)  # line order is free
    layer_tsv = "".join(f"{rows[p] + 1}\t{lay.col_idx[p] + 1}\t{float(lay.values[p])!r}\n"
                        for p in order)
    img, neu = np.nonzero(np.asarray(feats.data).T)
    feat_tsv = "".join(f"{i + 1}\t{n + 1}\t1\n" for i, n in zip(img, neu))
    ref_layer = ingest.load_layer_tsv(layer_tsv.encode(), 64)
    ref_feats = ingest.load_features_tsv(feat_tsv.encode(), 64, 22)
    truth = ingest.load_truth_categories(b"5\n2\n\n9\n")
    np.savez_compressed(
        os.path.join(HERE, "ingest.npz"),
        model_bin=np.frombuffer(mb.getvalue(), np.uint8),
        features_bin=np.frombuffer(fb.getvalue(), np.uint8),
        layer_tsv=np.frombuffer(layer_tsv.encode(), np.uint8),
        features_tsv=np.frombuffer(feat_tsv.encode(), np.uint8),
        layer_row_ptr=ref_layer.row_ptr, layer_col_idx=ref_layer.col_idx,
        layer_values=ref_layer.values, features_data=np.asarray(ref_feats.data),
        truth=np.array(truth, np.int64))
    print("model", len(mb.getvalue()), "features", len(fb.getvalue()), "bytes")


if __name__ == "__main__":
    main()
