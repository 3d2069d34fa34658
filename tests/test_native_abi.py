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


def _header_struct_fields(name):
    """Field names of `typedef struct name {...} name;` in the header."""
    text = open(os.path.join(_native.INCLUDE, "spdnn_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    body = re.search(r"typedef struct %s(?:_t)?\s*\{(.*?)\}\s*%s;" % (name.rstrip("_t"), name),
                     text, flags=re.S)
    assert body, name
    return [m.group(1) for m in re.finditer(r"[\w\s\*]+?\b(\w+)\s*;", body.group(1))]


def test_ctypes_structs_match_the_header():
    """The Python side's ctypes mirrors of the ABI structs list the header's
    fields in the header's order (a mismatch would shift every later field)."""
    pairs = [("spdnn_plan_params", _native.PlanParams), ("spdnn_plan_sizes_t", _native.PlanSizes),
             ("spdnn_layer_dev", _native.LayerDev), ("spdnn_scratch", _native.Scratch),
             ("spdnn_run_opts", _native.RunOpts)]
    for cname, py in pairs:
        assert _header_struct_fields(cname) == [f[0] for f in py._fields_], cname
