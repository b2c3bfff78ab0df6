"""The Python drop-in API (paper_2601_21552_b200.solver, mirroring
scuba_mini.solver) on the GPU: solve / propagate / check_model with the
reference's own pinned results and the oracle as checker."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import VCODE, load_golden

from oracle import oracle
from paper_2601_21552_b200 import _lib
from paper_2601_21552_b200.solver import (
    BinE, Constraint, Lit, Sat, SolverVar, Timeout, Unsat, VarRef,
    check_model, divisor_side_constraints, propagate, solve, solve_batch, solve_flat,
)
from paper_2601_21552_b200.terms import query_from_json
from paper_2601_21552_b200.wire import flatten, words_to_ints

pytestmark = pytest.mark.gpu


def c(rel, lhs, rhs):
    lhs = Lit(lhs) if isinstance(lhs, int) else lhs
    rhs = Lit(rhs) if isinstance(rhs, int) else rhs
    return Constraint(rel, lhs, rhs)


x, y = VarRef("x"), VarRef("y")


def test_propagate_pinned_results(gpu):
    # test_solver.py:80-107 of the reference
    assert propagate({"x": (0, 100)}, [c("<", x, 5)])["x"] == (0, 4)
    n = propagate({"x": (0, 100), "y": (0, 100)}, [c("=", BinE("+", x, y), 10)])
    assert n["x"] == (0, 10) and n["y"] == (0, 10)
    n = propagate({"x": (0, 10), "y": (0, 10)}, [c("=", BinE("*", x, y), 100)])
    assert n["x"] == (10, 10) and n["y"] == (10, 10)
    assert propagate({"x": (0, 3)}, [c(">", x, 7)]) is None


def test_propagate_batch_matches_oracle(gpu, golden):
    recs = golden["random_solver"] + golden["random_accept"] + golden["corpus_m1048576"]
    fb = flatten(recs)
    lo, hi, st = _lib.propagate_flat(fb)
    olo, ohi, ost = oracle.propagate_flat(fb)
    assert np.array_equal(st, ost)
    ok = st == 1
    for q in np.nonzero(ok)[0]:
        vb, ve = int(fb.var_begin[q]), int(fb.var_begin[q + 1])
        assert np.array_equal(lo[vb:ve], olo[vb:ve]) and np.array_equal(hi[vb:ve], ohi[vb:ve]), q


def test_check_model_matches_oracle(gpu, golden):
    recs = [r for n in ("random_solver", "random_accept", "crafted") for r in golden[n]
            if r["verdict"] == "sat"]
    rng = np.random.default_rng(5)
    fb = flatten(recs)
    model = np.zeros((fb.n_vars_total, 2), dtype=np.int64)
    for q, r in enumerate(recs):
        vb = int(fb.var_begin[q])
        for i, name in enumerate(fb.names(q)):
            v = r["model"][name] + (int(rng.integers(-1, 2)) if q % 3 == 0 else 0)
            model[vb + i] = (v & ((1 << 64) - 1)) - ((1 << 64) if v & (1 << 63) else 0), v >> 64
    got = _lib.check_model_flat(fb, model)
    want = oracle.check_model_flat(fb, model)
    assert np.array_equal(got, want)
    assert got.sum() > 0 and (got == 0).sum() > 0


def test_reference_models_check_with_side_constraints(gpu, golden):
    for r in golden["random_accept"]:
        if r["verdict"] != "sat":
            continue
        vs, cs = query_from_json(r)
        assert check_model(cs + divisor_side_constraints(cs), r["model"])


def test_solve_api_crafted(gpu):
    v = solve([SolverVar("x", 0, 10), SolverVar("y", 0, 10)], [c("=", BinE("*", x, y), 100)])
    assert isinstance(v, Sat) and v.model == {"x": 10, "y": 10}
    assert isinstance(solve([SolverVar("x", 1, 7)], [c("=", BinE("/", Lit(7), x), 2)]), Sat)
    assert solve([SolverVar("x", 1, 7)], [c("=", BinE("/", Lit(7), x), 2)]).model == {"x": 3}
    assert isinstance(solve([SolverVar("x", 0, 0)], [c("=", BinE("/", Lit(4), x), 0)]), Unsat)
    t = solve([SolverVar("x", 0, 3)], [c("<", x, 2)], timeout_s=0.0)
    assert isinstance(t, Timeout) and t.elapsed > 0
    assert isinstance(solve([SolverVar("x", 3, 2)], [], timeout_s=0.0), Unsat)


def test_solve_batch_matches_golden_objects(gpu, golden):
    recs = [r for r in golden["random_accept"]]
    verdicts = solve_batch([query_from_json(r) for r in recs], 20.0)
    for r, v in zip(recs, verdicts):
        if r["verdict"] == "sat":
            assert isinstance(v, Sat) and v.model == r["model"]
        else:
            assert isinstance(v, Unsat)


def test_determinism_across_calls(gpu, golden):
    recs = golden["synth_c3"]
    fb = flatten(recs)
    a = _lib.solve_flat(fb, 30.0)
    b = _lib.solve_flat(fb, 30.0)
    for k in ("verdict", "model", "nodes", "passes"):
        assert np.array_equal(a[k], b[k])
    assert all(int(a["verdict"][q]) == VCODE[r["verdict"]] for q, r in enumerate(recs))


def test_every_model_row_is_written(gpu, golden):
    """oob_solve_batch writes every row of the caller's model array: the Sat
    models (packed on the device, include/scuba_oob.h) and zeros elsewhere --
    the shim hands it an uninitialised buffer."""
    for name in ("synth_c4", "crafted", "corpus_m1048576"):
        recs = golden[name]
        fb = flatten(recs)
        out = _lib.solve_flat(fb, 30.0)
        ref = oracle.solve_flat(fb, 30.0)
        assert np.array_equal(out["verdict"], ref["verdict"]), name
        assert np.array_equal(out["model"], ref["model"]), name  # oracle: zeros unless Sat
        sat = out["verdict"] == 1
        for q in np.flatnonzero(~sat)[:50]:
            vb, ve = int(fb.var_begin[q]), int(fb.var_begin[q + 1])
            assert not out["model"][vb:ve].any(), (name, q)


@pytest.mark.parametrize("flags", [0, _lib.F_FAST])
def test_stream_api_equals_single_calls(gpu, flags):
    """oob_solve_batches (pipelined stream of batches) returns exactly what
    one oob_solve_batch per batch returns."""
    from paper_2601_21552_b200 import synth
    from paper_2601_21552_b200._lib import solve_flat_stream
    fbs = [synth.generate(c, 3000, first=k * 3000, names=False) for k, c in enumerate(("c3", "c4", "c3", "c5s", "c4"))]
    outs = solve_flat_stream(fbs, 30.0, n_gpus=1, flags=flags)
    for fb, o in zip(fbs, outs):
        assert o["status"] == _lib.OOB_OK
        ref = solve_flat(fb, 30.0, n_gpus=1, flags=flags)
        for k in ("verdict", "model", "nodes", "passes"):
            assert np.array_equal(o[k], ref[k]), k
