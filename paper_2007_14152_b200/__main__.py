"""Command line: ``python -m paper_2007_14152_b200 run|bench ...``.

The reference's ``spdnn run`` / ``spdnn bench`` (spdnn/cli.py:196-336) on the
B200 engine: a synthetic network and batch from the reference's generator
(or a binary cache written by ingest.write_binary), one inference through
engine.infer (or parallel.run_batch_parallel with --workers > 1), and the
run report in the reference's schema with the B200 figures added
(report.py: TE/s, roofline fraction, imbalance). ``--categories-out``
writes the surviving categories 1-based, one per line, as the reference
CLI does (spdnn/cli.py:131-134).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

EXIT_OK, EXIT_ERROR = 0, 1


def _peak_gbs() -> float:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0  # B200_PROFILING.md fallback


def _problem(args):
    from . import ingest
    if args.model:
        with open(args.model, "rb") as f:
            model = ingest.read_binary(f)
    else:
        model = ingest.generate_synthetic_network(ingest.GeneratorSpec(
            neurons=args.neurons, layers=args.layers, connections_per_neuron=args.connections,
            bias_value=args.bias, seed=args.seed))
    if args.features:
        with open(args.features, "rb") as f:
            inputs = ingest.read_binary(f)
    else:
        density = args.density if args.density is not None else abs(args.bias)
        inputs = ingest.generate_synthetic_inputs(model.neurons, args.inputs, density,
                                                  seed=args.seed + 1)
    return model, inputs


def _run_once(args, model, inputs, prepared):
    from . import engine, parallel
    from .model import InferenceConfig
    from .report import build_report
    config = InferenceConfig(workers=args.workers, rebalance_threshold=args.threshold)
    if args.workers > 1:
        res, comm, bal = parallel.run_batch_parallel(model, inputs, config, args.mode,
                                                     prepared=prepared)
    else:
        res = engine.infer(model, inputs, config, args.mode, prepared=prepared)
        comm = bal = None
    return res, build_report(model, inputs, config, args.mode, prepared, res, comm, bal,
                             hbm_peak_gbs=_peak_gbs())


def main(argv=None) -> int:
    from .model import InferenceConfig, ModelError
    from .report import render_report
    ap = argparse.ArgumentParser(prog="python -m paper_2007_14152_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "bench"):
        p = sub.add_parser(name)
        p.add_argument("--neurons", type=int, default=1024)
        p.add_argument("--layers", type=int, default=120)
        p.add_argument("--connections", type=int, default=32)
        p.add_argument("--bias", type=float, default=-0.3)
        p.add_argument("--inputs", type=int, default=60000)
        p.add_argument("--density", type=float, default=None, help="default |bias|")
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--model", default="", help="binary model cache (ingest.write_binary)")
        p.add_argument("--features", default="", help="binary feature cache")
        p.add_argument("--mode", choices=["optimized", "baseline"], default="optimized")
        p.add_argument("--workers", type=int, default=1)
        p.add_argument("--threshold", type=float, default=1.25)
        p.add_argument("--categories-out", default="")
        if name == "bench":
            p.add_argument("--repeat", type=int, default=3)
    args = ap.parse_args(argv)
    try:
        from . import engine
        model, inputs = _problem(args)
        prepared = engine.prepare_model(model, InferenceConfig(), args.mode)
        runs = 1 if args.cmd == "run" else max(1, args.repeat) + 1  # bench: one warm-up
        for _ in range(runs):
            res, rep = _run_once(args, model, inputs, prepared)
    except (ModelError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_ERROR
    sys.stdout.write(render_report(rep))
    if args.categories_out:
        np.savetxt(args.categories_out, np.asarray(res.categories) + 1, fmt="%d")
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
