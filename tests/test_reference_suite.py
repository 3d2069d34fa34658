"""The reference's own test suite (143 tests, /root/reference/pkg/tests,
installed next to the reference in baseline/_ref/tests by
tools/install_reference.sh) run against the drop-in: ``spdnn.model``,
``spdnn.ingest``, ``spdnn.engine`` and ``spdnn.parallel`` resolve to this
package (tests/refsuite/spdnn_alias.py), the reference's off-path modules
(preprocess, oracle, report, cli) are its own and run on top of them.

Every test must pass except the deviations listed in
tests/refsuite/deviations.json, each with its reason.
"""

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

from conftest import ROOT

REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")
DEVIATIONS = os.path.join(ROOT, "tests", "refsuite", "deviations.json")


def run_suite(tmp_path, extra=()):
    xml = tmp_path / "ref.xml"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "refsuite"), ROOT,
                                         env.get("PYTHONPATH", "")])
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-p", "spdnn_alias", "-p", "no:cacheprovider", "-q",
         f"--junitxml={xml}", *extra],
        cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=3000)
    outcomes = {}
    for case in ET.parse(xml).getroot().iter("testcase"):
        name = f"{case.get('classname').split('.')[-1]}::{case.get('name')}"
        bad = [c.tag for c in case if c.tag in ("failure", "error")]
        skipped = any(c.tag == "skipped" for c in case)
        outcomes[name] = "failed" if bad else ("skipped" if skipped else "passed")
    return proc, outcomes


@pytest.mark.gpu
def test_reference_suite_on_drop_in(cuda_ok, tmp_path):
    if not os.path.isdir(REF_TESTS):
        pytest.skip("baseline/_ref/tests missing (tools/install_reference.sh)")
    with open(DEVIATIONS) as f:
        allowed = json.load(f)["deviations"]
    proc, outcomes = run_suite(tmp_path)
    summary = {k: sum(v == k for v in outcomes.values()) for k in ("passed", "failed", "skipped")}
    out_dir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out_dir):
        with open(os.path.join(out_dir, "reference_suite.json"), "w") as f:
            json.dump({"summary": summary, "outcomes": outcomes,
                       "tail": proc.stdout[-6000:]}, f, indent=1)
    assert len(outcomes) >= 143, proc.stdout[-3000:]
    failed = sorted(k for k, v in outcomes.items() if v == "failed")
    unexpected = [k for k in failed if k not in allowed]
    assert not unexpected, (unexpected, proc.stdout[-4000:])


# reference tests that run the engine (a CUDA device) -- the GPU test above
# covers them; every other test of these files runs on the CPU here
_HOST_FILES = ("test_ingest.py", "test_model.py", "test_report.py", "test_preprocess.py",
               "test_parallel.py", "test_oracle.py")
_NEEDS_GPU = ("test_parallel.py::test_single_worker_matches_engine",
              "test_parallel.py::test_worker_count_invariance",
              "test_parallel.py::test_adversarial_die_off_triggers_rebalance",
              "test_parallel.py::test_infinite_threshold_disables_rebalancing",
              "test_parallel.py::test_latency_hook_sees_typed_messages",
              "test_parallel.py::test_baseline_mode_parallel",
              "test_parallel.py::test_more_workers_than_features",
              "test_oracle.py::test_matches_baseline_engine")


def test_reference_host_tests_on_drop_in(tmp_path):
    """The reference's loader, model, report, balancing-rule and oracle tests
    against the drop-in on the CPU (--noconftest: the reference's conftest
    warms its engine, which here needs the GPU)."""
    if not os.path.isdir(REF_TESTS):
        pytest.skip("baseline/_ref/tests missing (tools/install_reference.sh)")
    extra = ["--noconftest", *_HOST_FILES]
    for d in _NEEDS_GPU:
        extra += ["--deselect", d]
    proc, outcomes = run_suite(tmp_path, extra)
    failed = sorted(k for k, v in outcomes.items() if v == "failed")
    assert len(outcomes) >= 80 and not failed, (failed, proc.stdout[-3000:])
