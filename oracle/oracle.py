"""ctypes front-end for the CPU oracle (oracle/spdnn_oracle.c).

TEST INFRASTRUCTURE. Only tests/, ``__graft_entry__.smoke()`` and bench.py's
cpu_baseline / ``--impl reference`` leg may import this module; the product
package never does. See spdnn_oracle.c for the reference lines restated.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "spdnn_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _SO


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        lib.oracle_layer.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, P, P, P, P]
        lib.oracle_layer.restype = None
        lib.oracle_infer.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, P,
                                     ctypes.c_int64, P, ctypes.c_int, P, P, P]
        lib.oracle_infer.restype = None
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def layer(layer_csr, bias: np.ndarray, data: np.ndarray):
    """One layer (kernels.py:21-37 + engine.py:106): returns ((N, M) F-order out, alive)."""
    lib = _load()
    n = layer_csr.neurons
    yin = np.asfortranarray(data, dtype=np.float32)
    m = yin.shape[1]
    out = np.empty((n, m), dtype=np.float32, order="F")
    alive = np.zeros(m, dtype=np.uint8)
    rp = np.ascontiguousarray(layer_csr.row_ptr, np.int64)
    ci = np.ascontiguousarray(layer_csr.col_idx, np.int32)
    va = np.ascontiguousarray(layer_csr.values, np.float32)
    b = np.ascontiguousarray(bias, np.float32)
    lib.oracle_layer(n, m, _ptr(rp), _ptr(ci), _ptr(va), _ptr(b), _ptr(yin), _ptr(out), _ptr(alive))
    return out, alive.astype(bool)


@dataclass
class OracleResult:
    counts: np.ndarray       # int64 [L+1]: active entering each layer, then survivors
    death: np.ndarray        # int32 [M]: layer after which each column died (L = survived)
    categories: np.ndarray   # int64 sorted survivor categories
    final: np.ndarray | None  # (N, S) F-order survivor values, or None


def infer(model, inputs, threads: int = 1, want_final: bool = True) -> OracleResult:
    """Whole-network oracle (engine.py:235-290 semantics, restated per column)."""
    lib = _load()
    n, L = model.neurons, model.num_layers
    y0 = np.asfortranarray(inputs.data, dtype=np.float32)
    m = y0.shape[1]
    keep = []  # hold arrays alive while C reads them
    rps = (ctypes.c_void_p * max(L, 1))()
    cis = (ctypes.c_void_p * max(L, 1))()
    vas = (ctypes.c_void_p * max(L, 1))()
    for l, lay in enumerate(model.layers):
        rp = np.ascontiguousarray(lay.row_ptr, np.int64)
        ci = np.ascontiguousarray(lay.col_idx, np.int32)
        va = np.ascontiguousarray(lay.values, np.float32)
        keep += [rp, ci, va]
        rps[l], cis[l], vas[l] = rp.ctypes.data, ci.ctypes.data, va.ctypes.data
    bias = np.ascontiguousarray(model.bias, np.float32)
    death = np.zeros(m, dtype=np.int32)
    counts = np.zeros(L + 1, dtype=np.int64)
    final = np.empty((n, m), dtype=np.float32, order="F") if want_final else None
    lib.oracle_infer(n, L, rps, cis, vas, _ptr(bias), m, _ptr(y0), int(threads),
                     _ptr(death), _ptr(counts),
                     _ptr(final) if final is not None else ctypes.c_void_p(0))
    alive = death == L
    cats = np.asarray(inputs.categories, dtype=np.int64)[alive]
    fin = np.asfortranarray(final[:, alive]) if final is not None else None
    return OracleResult(counts=counts, death=death, categories=cats, final=fin)
