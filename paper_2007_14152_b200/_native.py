"""Loader and ctypes signatures for libspdnn_b200.so (C ABI: include/spdnn_b200.h).

There is no fallback: if the library is missing, was built for another
architecture, or no CUDA device is visible, every device entry point raises.
The CPU oracle under oracle/ is test infrastructure and is never imported
from this package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libspdnn_b200.so")
CSRC = os.path.join(_HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(_HERE), "include")

SOURCES = ["layer.cu", "plan.cpp", "capi.cpp"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3",
              "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared"]

SPDNN_OK, SPDNN_EINVAL, SPDNN_ECUDA, SPDNN_ENOMEM, SPDNN_ERANGE = 0, 1, 2, 3, 4

P = ctypes.c_void_p
i32, i64 = ctypes.c_int32, ctypes.c_int64


class PlanParams(ctypes.Structure):
    _fields_ = [("rows_per_group", i32), ("footprint_cap", i32), ("max_groups", i32),
                ("record_cap", i32), ("reorder", i32), ("uniform_records", i32)]


class PlanSizes(ctypes.Structure):
    _fields_ = [("neurons", i64), ("rows_per_group", i32), ("record_words", i32),
                ("num_blocks", i64), ("num_extra_stages", i64), ("num_groups", i64),
                ("num_meta", i64), ("num_records", i64), ("num_fp", i64), ("nnz", i64),
                ("padded_slots", i64), ("max_fp_per_stage", i32),
                ("max_records_per_stage", i32), ("max_meta_per_block", i32),
                ("max_groups_per_block", i32), ("pow2", i32),
                ("wexp_min", i32), ("wexp_max", i32), ("uniform", i32),
                ("weight_bits", ctypes.c_uint32)]


class LayerDev(ctypes.Structure):
    _fields_ = [("blocks", P), ("stages", P), ("meta", P), ("records", P),
                ("num_blocks", i64), ("neurons", i64), ("rows_per_group", i32),
                ("record_words", i32), ("max_fp_per_stage", i32), ("max_records_per_stage", i32),
                ("max_meta_per_block", i32), ("max_groups_per_block", i32),
                ("uniform", i32), ("weight_bits", ctypes.c_uint32)]


class Scratch(ctypes.Structure):
    _fields_ = [("tile_done", P), ("tile_alive", P), ("work", P), ("guard", P), ("split", P)]


class RunOpts(ctypes.Structure):
    _fields_ = [("fma_form", i32), ("tiny", ctypes.c_float), ("features_per_lane", i32)]


_lib = None
_lock = threading.Lock()


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/ into _lib/libspdnn_b200.so for sm_100a (nvcc, in-tree)."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "common.h"), os.path.join(INCLUDE, "spdnn_b200.h")]
    if not force and os.path.exists(LIB_PATH):
        t = os.path.getmtime(LIB_PATH)
        if all(os.path.getmtime(d) <= t for d in deps):
            return LIB_PATH
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = LIB_PATH + ".tmp"
    # SPDNN_NVCC_DEFINES: extra -D flags for tuning sweeps (e.g.
    # "-DSPDNN_MASK_CONSUMERS=16"); the default build sets none
    extra = os.environ.get("SPDNN_NVCC_DEFINES", "").split()
    cmd = ["nvcc", *NVCC_FLAGS, *extra, "-I", INCLUDE, "-o", tmp, *srcs]
    res = subprocess.run(cmd, capture_output=not verbose, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + (res.stderr or "") + (res.stdout or ""))
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    """The loaded library (built on first use if absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.spdnn_plan_build.argtypes = [i64, P, P, P, ctypes.POINTER(PlanParams), ctypes.POINTER(P)]
        L.spdnn_plan_build_many.argtypes = [i64, i64, P, P, P, ctypes.POINTER(PlanParams), i32, P]
        L.spdnn_plan_sizes.argtypes = [P, ctypes.POINTER(PlanSizes)]
        L.spdnn_plan_export.argtypes = [P, P, P, P, P]
        L.spdnn_plan_free.argtypes = [P]
        L.spdnn_plan_free.restype = None
        L.spdnn_layer_forward.argtypes = [ctypes.POINTER(LayerDev), P, P, P, i64, P, P, P, P, P,
                                          P, ctypes.POINTER(Scratch), P,
                                          ctypes.POINTER(RunOpts), P]
        L.spdnn_infer_layers.argtypes = [i64, P, P, P, P, i64, P, P, P, P, P,
                                         ctypes.POINTER(Scratch), ctypes.POINTER(RunOpts), P]
        L.spdnn_infer_layers_timed.argtypes = [i64, P, P, P, P, i64, P, P, P, P, P,
                                               ctypes.POINTER(Scratch), ctypes.POINTER(RunOpts),
                                               P, P]
        L.spdnn_transpose_in.argtypes = [P, i64, i64, P, i64, P, ctypes.c_float,
                                         ctypes.c_float, P]
        L.spdnn_gather_out.argtypes = [P, i64, i64, P, P, i64, P, P]
        L.spdnn_profile_read.argtypes = [P, i32, i32]
        L.spdnn_profile_read.restype = ctypes.c_int
        L.spdnn_trace_read.argtypes = [P, i32]
        L.spdnn_trace_read.restype = ctypes.c_int
        L.spdnn_ltrace_read.argtypes = [P, i32]
        L.spdnn_ltrace_read.restype = ctypes.c_int
        L.spdnn_last_error.restype = ctypes.c_char_p
        L.spdnn_version.restype = ctypes.c_char_p
        for name in ("spdnn_plan_build", "spdnn_plan_build_many", "spdnn_plan_sizes",
                     "spdnn_plan_export", "spdnn_layer_forward", "spdnn_infer_layers",
                     "spdnn_infer_layers_timed",
                     "spdnn_transpose_in", "spdnn_gather_out"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
        return L


def check(rc: int, what: str) -> None:
    if rc == SPDNN_OK:
        return
    msg = lib().spdnn_last_error().decode(errors="replace")
    if rc == SPDNN_EINVAL:
        from .model import ModelError
        raise ModelError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed (code {rc}): {msg}")


# every symbol include/spdnn_b200.h declares (tests check the exports)
EXPORTED = ("spdnn_plan_build", "spdnn_plan_build_many", "spdnn_plan_sizes",
            "spdnn_plan_export", "spdnn_plan_free", "spdnn_layer_forward",
            "spdnn_infer_layers", "spdnn_infer_layers_timed", "spdnn_transpose_in",
            "spdnn_gather_out",
            "spdnn_layer_occupancy", "spdnn_profile_read", "spdnn_trace_read", "spdnn_ltrace_read",
            "spdnn_last_error",
            "spdnn_version")
