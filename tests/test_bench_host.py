"""bench.py host-side pieces (CPU only): the config table matches
BASELINE.json's configs, the C5 stress recipe matches the one the reference
fixtures were generated with, and the C5 load model."""

import json
import os

import numpy as np

import bench
from conftest import ROOT
from paper_2007_14152_b200 import ingest, parallel


def test_configs_match_baseline():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        base = json.load(f)
    assert "TeraEdges/s" in base["metric"]
    sizes = [(c["neurons"], c["layers"], c["bias"]) for c in
             (bench.CONFIGS[k] for k in ("c1", "c2", "c3", "c4"))]
    assert sizes == [(1024, 120, -0.3), (4096, 480, -0.35), (16384, 1920, -0.4),
                     (65536, 1920, -0.45)]
    for k, text in zip(("c1", "c2", "c3", "c4"), base["configs"]):
        c = bench.CONFIGS[k]
        assert f"{c['neurons']} neurons" in text and f"{c['layers']} layers" in text
        assert c["density"] == abs(c["bias"]) and c["inputs"] == 60000
    assert bench.CONFIGS["c5"]["stress"] and bench.CONFIGS["c5"]["workers"] == 8


def test_stress_inputs_recipe():
    """Shard s: density |b| + 0.04 - 0.01 s, seed 100 + s,
    the recipe of tests/golden/make_stress.py."""
    cfg = dict(bench.CONFIGS["c5"], neurons=64, inputs=8 * 30)
    got = bench.stress_inputs(cfg)
    for s in range(8):
        want = ingest.generate_synthetic_inputs(64, 30, 0.44 - 0.01 * s, seed=100 + s)
        assert np.array_equal(np.asarray(got.data)[:, 30 * s:30 * (s + 1)], want.data)
    assert got.categories.tolist() == list(range(240))


def test_balance_summary_load_model():
    rep = parallel.BalanceReport()
    mk = lambda layer, b, a, moved: parallel.BalanceEntry(
        layer=layer, before_counts=tuple(b), after_counts=tuple(a),
        imbalance_before=parallel.imbalance_ratio(b), imbalance_after=parallel.imbalance_ratio(a),
        moved_rows=moved, rebalanced=moved > 0)
    rep.entries += [mk(0, [8, 2], [5, 5], 3), mk(1, [4, 4], [4, 4], 0), mk(2, [1, 1], [1, 1], 0)]
    s = bench.balance_summary(rep, [10, 10])
    # layer inputs: [10,10], [5,5], [4,4] -> sum of max == sum of mean
    assert s["time_weighted_max_over_mean"] == 1.0
    assert s["rebalances"] == 1 and s["max_imbalance_before"] == 4.0
    rep2 = parallel.BalanceReport(entries=[mk(0, [8, 2], [8, 2], 0), mk(1, [6, 2], [6, 2], 0)])
    s2 = bench.balance_summary(rep2, [10, 10])
    assert abs(s2["time_weighted_max_over_mean"] - (10 + 8) / (10 + 5)) < 1e-12


def test_relaunch_command():
    """--gpus N without a torchrun environment re-executes the same command
    under torch.distributed.run with N local ranks on 127.0.0.1."""
    env = dict(os.environ)
    try:
        os.environ.pop("WORLD_SIZE", None)
        assert bench.relaunch_command(["--gpus", "1"], 1) is None
        cmd = bench.relaunch_command(["--gpus", "4", "--config", "c3"], 4, port=29555)
        assert cmd[1:3] == ["-m", "torch.distributed.run"]
        assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
        assert "--master-port=29555" in cmd
        assert cmd[-4:] == [os.path.abspath(bench.__file__), "--gpus", "4", "--config", "c3"][-4:]
        os.environ["WORLD_SIZE"] = "4"  # already under torchrun: no relaunch
        assert bench.relaunch_command(["--gpus", "4"], 4) is None
    finally:
        os.environ.clear()
        os.environ.update(env)


def test_gpus2_launch_on_cpu():
    """`bench.py --gpus 2` really starts two ranks (torchrun, world size 2):
    the reference arm runs on rank 0 only, which prints one JSON line with
    n_gpus 2; rank 1 exits 0 without work."""
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
         "--config", "c1", "--steps", "1", "--warmup", "0", "--port-only",
         "--cpu-sample", "16", "--cpu-seconds", "0"],
        capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["value"] > 0
    assert "relaunching" in out.stderr
