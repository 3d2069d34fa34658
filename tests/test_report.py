"""Run reports (report.py): the reference's schema plus the B200 figures.
CPU: render/parse round trip, the reference's own parser reads them, timing
lines stripped. GPU: the CLI's report of a real run."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2007_14152_b200 import parallel, report
from paper_2007_14152_b200.engine import PaddingStats


def _fake(balance=True):
    bal = parallel.BalanceReport()
    bal.entries.append(parallel.BalanceEntry(layer=0, before_counts=(8, 2), after_counts=(5, 5),
                                             imbalance_before=4.0, imbalance_after=1.0,
                                             moved_rows=3, rebalanced=True))
    comm = parallel.CommMatrix.zeros(2)
    comm.add(np.array([[0, 3], [0, 0]]))
    return report.RunReport(
        neurons=64, layers=2, inputs=10, mode="optimized", workers=2, minibatch=12,
        block_size=256, warp_size=32, buffer_capacity=1024, streaming=False,
        rebalance_threshold=1.25, elapsed_seconds=0.5, edges_processed=10 * 2 * 64 * 4,
        weight_element_reads=100, feature_element_reads=200,
        per_layer_active_counts=[(10, 10), (10, 7)],
        padding_stats=PaddingStats(512, 100, 120, 130, 100 / 512, 120 / 512, 130 / 512),
        index_report=report.IndexReport(4096, 4096, 0.0), comm_matrix=comm,
        balance_report=bal if balance else None, device_seconds=0.25,
        hbm_bytes=report.algorithmic_bytes(64, [256, 256], [(10, 10), (10, 7)]),
        hbm_peak_gbs=6552.0)


def test_render_parse_roundtrip_and_b200_figures():
    r = _fake()
    text = report.render_report(r)
    p = report.parse_report(text)
    assert p.scalars["spdnn_report"] == "1" and p.number("neurons") == 64
    assert p.number("hbm_bytes") == 2 * (8 * 64 * 10 + 6 * 256 + 4 * 64)
    assert p.number("roofline_fraction") == pytest.approx(r.hbm_bytes / 0.25 / 6552e9)
    assert p.number("te_per_second") == pytest.approx(r.edges_processed / 0.5 / 1e12)
    assert p.number("imbalance_max_before") == 4.0 and p.number("rebalances") == 1
    assert p.tables["per_layer_active"] == [["0", "10", "10"], ["1", "10", "7"]]
    assert p.tables["comm_matrix"] == [["0", "3"], ["0", "0"]]
    stripped = report.strip_timing(text)
    for k in report.TIMING_KEYS:
        assert f"\n{k}:" not in stripped
    assert "hbm_bytes:" in stripped


def test_reference_parser_reads_the_report():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "spdnn")):
        pytest.skip("reference not installed (tools/install_reference.sh)")
    code = ("import sys; sys.path.insert(0, %r); from spdnn.report import parse_report, "
            "strip_timing; t = sys.stdin.read(); p = parse_report(t); "
            "print(p.scalars['neurons'], len(p.tables['per_layer_active']), "
            "p.scalars['roofline_fraction'])" % ref)
    out = subprocess.run([sys.executable, "-c", code], input=report.render_report(_fake()),
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.split()[:2] == ["64", "2"]


@pytest.mark.gpu
def test_cli_run_report(cuda_ok, tmp_path):
    from oracle import oracle
    from paper_2007_14152_b200 import ingest
    cats = tmp_path / "cats.txt"
    out = subprocess.run(
        [sys.executable, "-m", "paper_2007_14152_b200", "run", "--neurons", "1024",
         "--layers", "12", "--inputs", "600", "--bias", "-0.3", "--workers", "2",
         "--categories-out", str(cats)], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    p = report.parse_report(out.stdout)
    model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
        neurons=1024, layers=12, connections_per_neuron=32, bias_value=-0.3, seed=1))
    inputs = ingest.generate_synthetic_inputs(1024, 600, 0.3, seed=2)
    ref = oracle.infer(model, inputs, threads=4, want_final=False)
    assert [int(r[1]) for r in p.tables["per_layer_active"]] == ref.counts[:-1].tolist()
    assert 0 < p.number("roofline_fraction") < 1.5 and p.number("te_per_second") > 0
    assert "balance" in p.tables and "comm_matrix" in p.tables
    assert np.loadtxt(cats, dtype=np.int64, ndmin=1).tolist() == (ref.categories + 1).tolist()
