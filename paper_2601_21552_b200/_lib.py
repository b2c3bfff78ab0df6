"""ctypes binding of libscuba_oob.so (include/scuba_oob.h).

There is no CPU fallback: if the shared library is missing, or a batch reaches
search with no CUDA device visible, the call raises.  The library is built
in-tree by `python -m paper_2601_21552_b200.build` (or __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

# several engine kernels run concurrently per device: more hardware work
# queues than the default 8 (effective only before a CUDA context exists);
# 16, not 32: same throughput on B200 (C3/C4 A/B), half the context-creation
# cost (cold corpus analysis 3.1 -> 1.3 s, tools/gpu_connections.sh)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "16")

HERE = Path(__file__).resolve().parent
# (SCUBA_OOB_LIB_PATH: another build of the library, for A/B measurements)
LIB_PATH = Path(os.environ["SCUBA_OOB_LIB_PATH"]) if os.environ.get("SCUBA_OOB_LIB_PATH") else HERE / "libscuba_oob.so"

OOB_OK, OOB_E_INVALID, OOB_E_CUDA, OOB_E_RANGE, OOB_E_NOMEM = 0, 1, 2, 3, 4
UNSAT, SAT, TIMEOUT, ERROR = 0, 1, 2, 3

F_NO_SORT = 1
F_NO_DEMOTE = 2
F_NO_JIT = 4
F_NO_X32 = 8
F_FAST = 16  # fast mode: symbolic Unsat prover in front of the exact emulation
F_CHAIN = 32  # with F_FAST: warp-per-query search with warp-parallel propagation (opt-in)

class EngineError(RuntimeError):
    """The GPU engine could not decide a batch (no device, capacity, range)."""


class oob_options(ctypes.Structure):
    _fields_ = [
        ("timeout_s", ctypes.c_double),
        ("node_budget", ctypes.c_int64),
        ("n_gpus", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("heavy_nodes", ctypes.c_int32),
        ("jit_min", ctypes.c_int32),
    ]


class oob_result(ctypes.Structure):
    _fields_ = [
        ("verdict", ctypes.c_void_p),
        ("model", ctypes.c_void_p),
        ("nodes", ctypes.c_void_p),
        ("passes", ctypes.c_void_p),
        ("elapsed_s", ctypes.c_void_p),
    ]


EXPORTS = (
    "oob_solve_batch",
    "oob_propagate_batch",
    "oob_check_model_batch",
    "oob_side_constraint_count",
    "oob_query_regime",
    "oob_jit_compile",
    "oob_last_error",
    "oob_device_count",
    "oob_version",
    "oob_release",
    "oob_solve_batches",
    "oob_plan_create",
    "oob_plan_run",
    "oob_plan_results",
    "oob_plan_info",
    "oob_plan_destroy",
)

_lib = None


def lib():
    """Load the engine library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA engine first "
            "(python -m paper_2601_21552_b200.build); there is no CPU fallback")
    L = ctypes.CDLL(str(LIB_PATH))
    vp = ctypes.c_void_p
    L.oob_solve_batch.argtypes = [vp, vp, vp]
    L.oob_solve_batch.restype = ctypes.c_int
    L.oob_solve_batches.argtypes = [vp, ctypes.c_int64, vp, vp]
    L.oob_solve_batches.restype = ctypes.c_int
    L.oob_propagate_batch.argtypes = [vp, vp, vp, vp, vp]
    L.oob_propagate_batch.restype = ctypes.c_int
    L.oob_check_model_batch.argtypes = [vp, vp, vp, vp]
    L.oob_check_model_batch.restype = ctypes.c_int
    L.oob_side_constraint_count.argtypes = [vp, vp]
    L.oob_side_constraint_count.restype = ctypes.c_int
    L.oob_jit_compile.argtypes = [vp, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64, vp]
    L.oob_jit_compile.restype = ctypes.c_int
    L.oob_host_bench.argtypes = [vp, vp, vp]
    L.oob_host_bench.restype = ctypes.c_int
    L.oob_query_regime.argtypes = [vp, vp, vp]
    L.oob_query_regime.restype = ctypes.c_int
    L.oob_sweep_run.argtypes = [vp, ctypes.c_int64, ctypes.c_int32, vp, vp]
    L.oob_sweep_run.restype = ctypes.c_int
    L.oob_sweep_replay.argtypes = [vp, ctypes.c_int64, ctypes.c_int32, vp, vp, vp, vp, vp]
    L.oob_sweep_replay.restype = ctypes.c_int
    L.oob_last_error.restype = ctypes.c_char_p
    L.oob_device_count.restype = ctypes.c_int
    L.oob_version.restype = ctypes.c_char_p
    L.oob_release.restype = None
    L.oob_plan_create.argtypes = [vp, vp, vp]
    L.oob_plan_create.restype = ctypes.c_int
    L.oob_plan_run.argtypes = [vp, vp]
    L.oob_plan_run.restype = ctypes.c_int
    L.oob_plan_results.argtypes = [vp, vp]
    L.oob_plan_results.restype = ctypes.c_int
    L.oob_plan_info.argtypes = [vp, vp]
    L.oob_plan_info.restype = ctypes.c_int
    L.oob_plan_destroy.argtypes = [vp]
    L.oob_plan_destroy.restype = None
    _lib = L
    return L


def last_error() -> str:
    return lib().oob_last_error().decode()


def check(rc: int, what: str):
    if rc == OOB_OK:
        return
    msg = last_error()
    if rc == OOB_E_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise EngineError(f"{what} failed (status {rc}): {msg}")


def device_count() -> int:
    return int(lib().oob_device_count())


def release() -> None:
    """Free the pooled device buffers of the solve paths (the stream API keeps
    one set per worker between calls); the next call allocates again."""
    lib().oob_release()


def options(timeout_s=30.0, node_budget=0, n_gpus=0, device=0, flags=0, heavy_nodes=0, jit_min=0):
    o = oob_options()
    o.jit_min = int(jit_min)
    o.timeout_s = float(timeout_s)
    o.node_budget = int(node_budget)
    o.n_gpus = int(n_gpus)
    o.device = int(device)
    o.flags = int(flags)
    o.heavy_nodes = int(heavy_nodes)
    return o


def _result_arrays(fb):
    n = fb.n
    out = {
        "verdict": np.full(n, -1, dtype=np.int8),
        # every row is written by the library (zero unless Sat): no clearing here
        "model": np.empty((max(fb.n_vars_total, 1), 2), dtype=np.int64),
        "nodes": np.zeros(n, dtype=np.int64),
        "passes": np.zeros(n, dtype=np.int64),
        "elapsed": np.zeros(n, dtype=np.float64),
    }
    r = oob_result(out["verdict"].ctypes.data, out["model"].ctypes.data,
                   out["nodes"].ctypes.data, out["passes"].ctypes.data,
                   out["elapsed"].ctypes.data)
    return out, r


def solve_flat(fb, timeout_s=30.0, node_budget=0, n_gpus=0, device=0, flags=0, heavy_nodes=0, jit_min=0):
    """Run oob_solve_batch on a FlatBatch -> dict of numpy result arrays."""
    out, r = _result_arrays(fb)
    cb = fb.as_c()
    o = options(timeout_s, node_budget, n_gpus, device, flags, heavy_nodes, jit_min)
    rc = lib().oob_solve_batch(ctypes.byref(cb), ctypes.byref(o), ctypes.byref(r))
    out["status"] = rc
    out["error"] = last_error() if rc else ""
    return out


def solve_flat_stream(fbs, timeout_s=30.0, node_budget=0, n_gpus=0, device=0, flags=0, heavy_nodes=0,
                      jit_min=0):
    """oob_solve_batches: a list of FlatBatches decided as one pipelined
    stream -> list of result dicts (each exactly solve_flat's)."""
    outs, rs, cbs = [], [], []
    for fb in fbs:
        out, r = _result_arrays(fb)
        outs.append(out)
        rs.append(r)
        cbs.append(fb.as_c())
    if not fbs:
        return []
    ca = (type(cbs[0]) * len(cbs))(*cbs)
    ra = (oob_result * len(rs))(*rs)
    o = options(timeout_s, node_budget, n_gpus, device, flags, heavy_nodes, jit_min)
    rc = lib().oob_solve_batches(ctypes.addressof(ca), len(fbs), ctypes.byref(o), ctypes.addressof(ra))
    err = last_error() if rc else ""
    for out in outs:
        out["status"] = rc
        out["error"] = err
    return outs


def propagate_flat(fb, device=0):
    V = max(fb.n_vars_total, 1)
    lo = np.zeros((V, 2), dtype=np.int64)
    hi = np.zeros((V, 2), dtype=np.int64)
    st = np.zeros(fb.n, dtype=np.int8)
    cb = fb.as_c()
    o = options(device=device, n_gpus=1)
    rc = lib().oob_propagate_batch(ctypes.byref(cb), ctypes.byref(o), lo.ctypes.data,
                                   hi.ctypes.data, st.ctypes.data)
    check(rc, "oob_propagate_batch")
    return lo, hi, st


def check_model_flat(fb, model_words, device=0):
    ok = np.zeros(fb.n, dtype=np.int8)
    m = np.ascontiguousarray(model_words, dtype=np.int64)
    cb = fb.as_c()
    o = options(device=device, n_gpus=1)
    rc = lib().oob_check_model_batch(ctypes.byref(cb), ctypes.byref(o), m.ctypes.data,
                                     ok.ctypes.data)
    check(rc, "oob_check_model_batch")
    return ok


def side_counts(fb):
    c = np.zeros(fb.n, dtype=np.int64)
    cb = fb.as_c()
    check(lib().oob_side_constraint_count(ctypes.byref(cb), c.ctypes.data),
          "oob_side_constraint_count")
    return c


class Plan:
    """oob_plan_*: compile + upload once, run kernels on HBM-resident records."""

    INFO = ("queries", "record_bytes", "result_bytes", "classes", "jobs",
            "launches_per_run", "wide_queries", "compile_us", "h2d_bytes")

    def __init__(self, fb, timeout_s=30.0, node_budget=0, n_gpus=0, device=0, flags=0, heavy_nodes=0,
                 jit_min=0):
        self.fb = fb                     # keeps the batch arrays alive
        self._cb = fb.as_c()
        self._opt = options(timeout_s, node_budget, n_gpus, device, flags, heavy_nodes, jit_min)
        self._p = ctypes.c_void_p()
        check(lib().oob_plan_create(ctypes.byref(self._cb), ctypes.byref(self._opt),
                                    ctypes.byref(self._p)), "oob_plan_create")

    def run(self) -> float:
        ms = ctypes.c_float()
        check(lib().oob_plan_run(self._p, ctypes.byref(ms)), "oob_plan_run")
        return float(ms.value)

    def info(self) -> dict:
        a = np.zeros(len(self.INFO), dtype=np.int64)
        check(lib().oob_plan_info(self._p, a.ctypes.data), "oob_plan_info")
        return dict(zip(self.INFO, (int(x) for x in a)))

    def results(self) -> dict:
        fb = self.fb
        n = fb.n
        out = {
            "verdict": np.full(n, -1, dtype=np.int8),
            "model": np.zeros((max(fb.n_vars_total, 1), 2), dtype=np.int64),
            "nodes": np.zeros(n, dtype=np.int64),
            "passes": np.zeros(n, dtype=np.int64),
            "elapsed": np.zeros(n, dtype=np.float64),
        }
        r = oob_result(out["verdict"].ctypes.data, out["model"].ctypes.data,
                       out["nodes"].ctypes.data, out["passes"].ctypes.data,
                       out["elapsed"].ctypes.data)
        rc = lib().oob_plan_results(self._p, ctypes.byref(r))
        if rc not in (OOB_OK, OOB_E_RANGE):
            check(rc, "oob_plan_results")
        out["status"] = rc
        return out

    def close(self):
        if self._p:
            lib().oob_plan_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def query_regime(fb, timeout_s=30.0):
    """Per-query exact-arithmetic regime chosen by the host compiler
    (0 immediate, 1 int64, 2 int128, 3 256-bit, 4 out of range); host only."""
    out = np.zeros(fb.n, dtype=np.int8)
    cb = fb.as_c()
    o = options(timeout_s)
    check(lib().oob_query_regime(ctypes.byref(cb), ctypes.byref(o), out.ctypes.data), "oob_query_regime")
    return out


def jit_compile(fb, q: int, cap: int = 1 << 22):
    """Generated source of query q's structure class and its NVRTC compile
    time in ms (host only: no device is needed)."""
    buf = ctypes.create_string_buffer(cap)
    ms = ctypes.c_double()
    cb = fb.as_c()
    check(lib().oob_jit_compile(ctypes.byref(cb), int(q), buf, cap, ctypes.byref(ms)), "oob_jit_compile")
    return buf.value.decode(), ms.value


def host_bench(fb, timeout_s=30.0, flags=0):
    """Host pipeline timings without a device: [validate+compile, prepare
    (compile + schedule), pack] in ms (diagnostics)."""
    ms = np.zeros(3, dtype=np.float64)
    cb = fb.as_c()
    o = options(timeout_s, flags=flags)
    check(lib().oob_host_bench(ctypes.byref(cb), ctypes.byref(o), ms.ctypes.data), "oob_host_bench")
    return ms
