"""pytest plugin: run the reference's own test suite against the drop-in.

Loaded with ``-p spdnn_alias`` (tests/test_reference_suite.py). It makes
``import spdnn`` resolve to this repo's package for every module on the
hot path the drop-in replaces:

    spdnn.model, spdnn.ingest, spdnn.engine, spdnn.parallel
        -> paper_2007_14152_b200.{model, ingest, engine, parallel}

The reference modules off that path (spdnn.preprocess: the reference's
sliced-ELL builder; spdnn.oracle: its dense oracle; spdnn.report,
spdnn.cli, spdnn.kernels) are loaded from the unmodified reference in
baseline/_ref, and their own ``from .model import ...`` / ``from .engine
import ...`` bind to the drop-in — so the reference CLI and report run on
top of the B200 engine exactly as a user switching packages would get.
"""

from __future__ import annotations

import importlib
import os
import sys
import types

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "spdnn")

REPLACED = ("model", "ingest", "engine", "parallel")
FROM_REFERENCE = ("preprocess", "kernels", "oracle", "report", "cli")


def install() -> types.ModuleType:
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    if not os.path.isdir(REF_PKG):
        raise RuntimeError(f"reference not installed at {REF_PKG} (tools/install_reference.sh)")
    import paper_2007_14152_b200 as drop_in

    pkg = types.ModuleType("spdnn")
    pkg.__path__ = [REF_PKG]
    pkg.__file__ = os.path.join(REF_PKG, "__init__.py")
    pkg.__package__ = "spdnn"
    sys.modules["spdnn"] = pkg
    for name in REPLACED:
        mod = importlib.import_module(f"paper_2007_14152_b200.{name}")
        sys.modules[f"spdnn.{name}"] = mod
        setattr(pkg, name, mod)
    for name in FROM_REFERENCE:
        setattr(pkg, name, importlib.import_module(f"spdnn.{name}"))
    # the reference's top-level re-exports (spdnn/__init__.py:9-63)
    for name in dir(drop_in):
        if not name.startswith("_"):
            setattr(pkg, name, getattr(drop_in, name))
    for mod_name, names in (("preprocess", ("PaddingStats", "SlicedEllLayer", "StagingPlan",
                                            "build_staging_plan", "csr_to_sliced_ell",
                                            "expand_sliced_ell", "narrow_indices",
                                            "padding_stats")),
                            ("oracle", ("reference_infer", "reference_layer"))):
        for n in names:
            if not hasattr(pkg, n):
                setattr(pkg, n, getattr(getattr(pkg, mod_name), n))
    pkg.__version__ = "0.1.0"
    pkg.__drop_in__ = drop_in.__name__
    return pkg


install()
