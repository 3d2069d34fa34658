"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
header declares (CPU-only: no device calls)."""

import ctypes
import os
import re
import subprocess

from paper_2007_14152_b200 import _native


def _header_symbols():
    text = open(os.path.join(_native.INCLUDE, "spdnn_b200.h")).read()
    return sorted(set(re.findall(r"\b(spdnn_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    declared = _header_symbols()
    assert set(declared) == set(_native.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.spdnn_version()


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_path_sets_message():
    lib = _native.lib()
    rc = lib.spdnn_plan_sizes(None, None)
    assert rc == _native.SPDNN_EINVAL
    assert b"null" in lib.spdnn_last_error()
