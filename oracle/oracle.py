"""ctypes binding of oracle/liboob_oracle.so -- TEST INFRASTRUCTURE ONLY.

The CPU restatement of the reference solver (oob_oracle.c).  Importable only
from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs; the
product package never imports this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboob_oracle.so"
SYNTH_LIB = HERE / "liboob_synth.so"

_lib = None


def build(force: bool = False) -> Path:
    synth_src = HERE.parent / "paper_2601_21552_b200" / "csrc" / "synth.cpp"
    stale = (not LIB.exists() or LIB.stat().st_mtime < (HERE / "oob_oracle.cpp").stat().st_mtime
             or not SYNTH_LIB.exists() or SYNTH_LIB.stat().st_mtime < synth_src.stat().st_mtime)
    if force or stale:
        subprocess.check_call(["make", "-s", "-C", str(HERE)])
    return LIB


_synth = None


def synth_lib():
    """The seeded query generator (csrc/synth.cpp) built into oracle/ (no
    engine library involved)."""
    global _synth
    if _synth is None:
        if not SYNTH_LIB.exists():
            build()
        _synth = ctypes.CDLL(str(SYNTH_LIB))
    return _synth


def synth_generate(config: str, n: int, first: int = 0, names: bool = False):
    from paper_2601_21552_b200 import synth
    return synth.generate(config, n, first=first, names=names, lib=synth_lib())


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        vp = ctypes.c_void_p
        L.oracle_solve_batch.argtypes = [vp, ctypes.c_double, ctypes.c_int64, vp, ctypes.c_int]
        L.oracle_propagate_batch.argtypes = [vp, vp, vp, vp]
        L.oracle_check_model_batch.argtypes = [vp, vp, vp]
        L.oracle_side_constraint_count.argtypes = [vp, vp]
        _lib = L
    return _lib


class _Result(ctypes.Structure):
    _fields_ = [("verdict", ctypes.c_void_p), ("model", ctypes.c_void_p),
                ("nodes", ctypes.c_void_p), ("passes", ctypes.c_void_p),
                ("elapsed_s", ctypes.c_void_p)]


def solve_flat(fb, timeout_s=30.0, node_budget=0, threads=1):
    """-> dict of numpy arrays: verdict[n], model[V,2], nodes[n], passes[n], elapsed[n]."""
    n = fb.n
    out = {
        "verdict": np.full(n, -1, dtype=np.int8),
        "model": np.zeros((max(fb.n_vars_total, 1), 2), dtype=np.int64),
        "nodes": np.zeros(n, dtype=np.int64),
        "passes": np.zeros(n, dtype=np.int64),
        "elapsed": np.zeros(n, dtype=np.float64),
    }
    r = _Result(out["verdict"].ctypes.data, out["model"].ctypes.data,
                out["nodes"].ctypes.data, out["passes"].ctypes.data,
                out["elapsed"].ctypes.data)
    cb = fb.as_c()
    lib().oracle_solve_batch(ctypes.byref(cb), float(timeout_s), int(node_budget),
                             ctypes.byref(r), int(threads))
    return out


def propagate_flat(fb):
    V = max(fb.n_vars_total, 1)
    lo = np.zeros((V, 2), dtype=np.int64)
    hi = np.zeros((V, 2), dtype=np.int64)
    st = np.zeros(fb.n, dtype=np.int8)
    cb = fb.as_c()
    lib().oracle_propagate_batch(ctypes.byref(cb), lo.ctypes.data, hi.ctypes.data, st.ctypes.data)
    return lo, hi, st


def check_model_flat(fb, model_words):
    ok = np.zeros(fb.n, dtype=np.int8)
    m = np.ascontiguousarray(model_words, dtype=np.int64)
    cb = fb.as_c()
    lib().oracle_check_model_batch(ctypes.byref(cb), m.ctypes.data, ok.ctypes.data)
    return ok


def side_counts(fb):
    c = np.zeros(fb.n, dtype=np.int64)
    cb = fb.as_c()
    lib().oracle_side_constraint_count(ctypes.byref(cb), c.ctypes.data)
    return c


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
