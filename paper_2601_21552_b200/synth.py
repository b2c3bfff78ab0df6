"""Seeded analyzer-shaped query batches (include/scuba_oob_synth.h) as
FlatBatch objects.  Configs follow SURVEY.md 8(d) / BASELINE.md:

  c3   100K-style stream: M = 2^31-1, input caps 2^3..2^7, 30% buggy  (seed 2601215521)
  c4   mixed 32/64-bit:   M in {2^31-1, 2^59}, caps 2^3..2^10, 3-D    (seed 2601215522)
  c5   adversarial, bug-free (Unsat by construction), caps 2^20        (seed 2601215523)
  c5s  the c5 stream regenerated at caps 2^6, where the reference decides
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .wire import FlatBatch

SEEDS = {"c3": 2601215521, "c4": 2601215522, "c5": 2601215523, "c5s": 2601215523}
CODES = {"c3": 3, "c4": 4, "c5": 5, "c5s": 5}
CAP_LOG2 = {"c5s": 6}
CONFIGS = ("c3", "c4", "c5s")  # (c5 proper: caps 2^20, decided in fast mode only)

AXES = ("TidX", "TidY", "TidZ", "BidX", "BidY", "BidZ",
        "GDimX", "GDimY", "GDimZ", "BDimX", "BDimY", "BDimZ")
TEMPLATES = {1: "linear", 2: "static", 3: "product", 4: "loop", 5: "partition",
             6: "datadep", 7: "rowmajor", 8: "3d"}


def var_name(code: int) -> str:
    if code < 12:
        return "sol" + AXES[code]
    if code == 12:
        return "solOffset"
    if code == 13:
        return "solSize"
    return f"sol_u{code - 14}_v{code - 14}"


class _Out(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "var_begin", "var_lo", "var_hi", "con_begin", "con_rel", "con_lhs", "con_rhs",
        "node_begin", "node_op", "node_a", "node_b", "lit_begin", "lits", "name_code",
        "tmpl")]


def _setup(L):
    if getattr(L, "_synth_ready", False):
        return
    L.oob_synth_caps.argtypes = [ctypes.c_int, ctypes.c_void_p]
    L.oob_synth_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
    L._synth_ready = True


def generate(config: str, n: int, first: int = 0, seed: int | None = None,
             names: bool = True, lib=None) -> FlatBatch:
    """Queries [first, first + n) of the config's stream.  `lib`: a library
    exporting the generator (default: the engine's; bench.py's reference arm
    passes the oracle-side build, oracle/liboob_synth.so, so that arm never
    loads the engine)."""
    L = lib if lib is not None else _lib.lib()
    _setup(L)
    code = CODES[config]
    seed = SEEDS[config] if seed is None else seed
    caps = np.zeros(4, dtype=np.int64)
    L.oob_synth_caps(code, caps.ctypes.data)
    cv, cc, cn, cl = (int(x) for x in caps)
    a = {
        "var_begin": np.zeros(n + 1, np.int64), "var_lo": np.zeros((n * cv, 2), np.int64),
        "var_hi": np.zeros((n * cv, 2), np.int64), "con_begin": np.zeros(n + 1, np.int64),
        "con_rel": np.zeros(n * cc, np.uint8), "con_lhs": np.zeros(n * cc, np.int32),
        "con_rhs": np.zeros(n * cc, np.int32), "node_begin": np.zeros(n + 1, np.int64),
        "node_op": np.zeros(n * cn, np.uint8), "node_a": np.zeros(n * cn, np.int32),
        "node_b": np.zeros(n * cn, np.int32), "lit_begin": np.zeros(n + 1, np.int64),
        "lits": np.zeros((n * cl, 2), np.int64), "name_code": np.zeros(n * cv, np.uint16),
        "tmpl": np.zeros(max(n, 1), np.uint8),
    }
    out = _Out(*[a[f].ctypes.data for f, _ in _Out._fields_])
    rc = L.oob_synth_generate(code, seed, first, n, CAP_LOG2.get(config, 0), ctypes.byref(out))
    if rc != 0:
        raise RuntimeError(f"synthetic generator failed (rc={rc})")
    V, C, N, Lt = (int(a[k][-1]) for k in ("var_begin", "con_begin", "node_begin", "lit_begin"))
    var_names = None
    if names:
        codes = a["name_code"][:V].tolist()
        vb = a["var_begin"].tolist()
        var_names = [[var_name(c) for c in codes[vb[q]:vb[q + 1]]] for q in range(n)]
    fb = FlatBatch(
        a["var_begin"], a["var_lo"][:V].copy(), a["var_hi"][:V].copy(), var_names,
        a["con_begin"], a["con_rel"][:C].copy(), a["con_lhs"][:C].copy(), a["con_rhs"][:C].copy(),
        a["node_begin"], a["node_op"][:N].copy(), a["node_a"][:N].copy(), a["node_b"][:N].copy(),
        a["lit_begin"], a["lits"][:Lt].copy())
    fb.tmpl = a["tmpl"][:n].copy()
    return fb


def generate_json(config: str, n: int, first: int = 0) -> list:
    fb = generate(config, n, first)
    return [fb.query_json(q) for q in range(n)]
