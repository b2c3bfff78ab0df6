"""The fast mode's symbolic Unsat prover (csrc/symbolic.cuh), host build
(tests/native/sym_host.cpp, test infrastructure), on CPU.

Soundness: it never refutes a query the reference decides Sat (every golden
record of every set, captured from the reference itself).  Reach: it refutes
every Unsat record of the synthetic sets and the corpus, and every query of
the adversarial C5 stream at caps 2^20 (Unsat by construction).
"""
from __future__ import annotations

import ctypes
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN_SETS, ROOT, load_golden

from paper_2601_21552_b200.wire import flatten

SRC = ROOT / "tests" / "native" / "sym_host.cpp"
LIB = ROOT / "tests" / "native" / "_build" / "libsym_host.so"
DEPS = [SRC, ROOT / "paper_2601_21552_b200" / "csrc" / "symbolic.cuh",
        ROOT / "paper_2601_21552_b200" / "csrc" / "format.h"]


@pytest.fixture(scope="module")
def prover():
    if not LIB.exists() or LIB.stat().st_mtime < max(d.stat().st_mtime for d in DEPS):
        LIB.parent.mkdir(parents=True, exist_ok=True)
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", str(LIB), str(SRC)])
    L = ctypes.CDLL(str(LIB))
    L.sym_host_refute.argtypes = [ctypes.c_void_p, ctypes.c_void_p]

    def refute(fb):
        out = np.zeros(fb.n, dtype=np.int8)
        cb = fb.as_c()
        assert L.sym_host_refute(ctypes.byref(cb), out.ctypes.data) == 0
        return out

    return refute


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_never_refutes_a_reference_sat(prover, name):
    recs = load_golden(name)
    r = prover(flatten(recs))
    sat = np.array([x["verdict"] == "sat" for x in recs])
    assert not (r.astype(bool) & sat).any()
    unsat = np.array([x["verdict"] == "unsat" for x in recs])
    if name.startswith("synth") or name.startswith("corpus"):
        assert r[unsat].all(), f"{name}: {int((~r.astype(bool) & unsat).sum())} Unsat records not refuted"


def test_refutes_c5_proper(prover):
    from paper_2601_21552_b200 import synth
    fb = synth.generate("c5", 2000, names=False)
    assert prover(fb).all()


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_sound_on_streams_vs_oracle(prover, cfg):
    """2000 queries per stream against the C restatement of the reference."""
    from oracle import oracle
    from paper_2601_21552_b200 import synth
    fb = synth.generate(cfg, 2000, first=5000, names=False)
    r = prover(fb).astype(bool)
    v = oracle.solve_flat(fb, 30.0, threads=oracle.cpu_count())["verdict"]
    assert not (r & (v == 1)).any()
    assert r[v == 0].all()


# ---- the engine's own compiled certificates (oob_cert_compile), checked by
# the host build of the device checker (cert.cuh) ---------------------------

def _engine_cert_refutes(fb):
    from paper_2601_21552_b200 import _lib
    L = _lib.lib()
    vp = ctypes.c_void_p
    L.oob_cert_compile.argtypes = [vp, vp, vp, ctypes.c_int64, vp, vp, vp, ctypes.c_int64, vp]
    H = ctypes.CDLL(str(LIB))
    H.sym_host_check_engine_certs.argtypes = [vp] * 7
    n = fb.n
    cap = 1 << 22
    words = np.zeros(cap, dtype=np.uint64)
    nw = np.zeros(1, dtype=np.int64)
    off = np.zeros(n, dtype=np.int64)
    scap = 8 * int(fb.node_op.shape[0]) + 64 * n + 16  # literal slots: one per occurrence in the expanded trees
    slots = np.zeros((scap, 2), dtype=np.int64)
    sb = np.zeros(n + 1, dtype=np.int64)
    cb = fb.as_c()
    o = _lib.options(30.0)
    assert L.oob_cert_compile(ctypes.byref(cb), ctypes.byref(o), words.ctypes.data, cap, nw.ctypes.data,
                              off.ctypes.data, slots.ctypes.data, scap, sb.ctypes.data) == 0, _lib.last_error()
    ref = np.zeros(n, dtype=np.int8)
    why = np.zeros(n, dtype=np.int8)
    H.sym_host_check_engine_certs(ctypes.byref(cb), words.ctypes.data, off.ctypes.data, slots.ctypes.data,
                                  sb.ctypes.data, ref.ctypes.data, why.ctypes.data)
    return ref.astype(bool)


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_engine_certificates_sound(prover, name):
    recs = [r for r in load_golden(name) if r["verdict"] != "timeout"]
    r = _engine_cert_refutes(flatten(recs))
    sat = np.array([x["verdict"] == "sat" for x in recs])
    assert not (r & sat).any()
    if name.startswith("synth"):
        unsat = ~sat
        assert r[unsat].all(), f"{name}: {int((~r & unsat).sum())} Unsat records without a certificate"


@pytest.mark.parametrize("cfg", ["c3", "c4", "c5", "c5s"])
def test_engine_certificates_reach(prover, cfg):
    """Class certificates refute every Unsat query of 4000 per stream (C5
    proper: every query), and no Sat one (C restatement of the reference)."""
    from oracle import oracle
    from paper_2601_21552_b200 import synth
    fb = synth.generate(cfg, 4000, names=False)
    r = _engine_cert_refutes(fb)
    if cfg == "c5":
        assert r.all()
        return
    v = oracle.solve_flat(fb, 30.0, threads=oracle.cpu_count())["verdict"]
    assert not (r & (v == 1)).any()
    assert r[v == 0].all()
