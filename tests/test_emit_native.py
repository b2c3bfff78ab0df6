"""Native constraint-set construction (paper_2601_21552_b200/emit.py,
csrc/emit_native.cpp) against the reference's own generators
(constraint_gen.py:84-345): every set the reference analyzer asks for over
the whole corpus -- three domain sizes, with and without the underflow check
-- must be EQUAL to the reference's (variables, constraints, check, witness
and __input() leaves, all in order), and the errors must be the same.
CPU only: the reference front end from baseline/_ref or the mounted
reference."""
from __future__ import annotations

import dataclasses
import sys

import pytest

from conftest import reference_available, reference_paths

pytestmark = pytest.mark.skipif(not reference_available(), reason="reference not mounted")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(reference_paths()[0]))
    import scuba_mini.analyzer as An
    import scuba_mini.constraint_gen as CG

    from paper_2601_21552_b200.emit import NativeEmission
    return An, CG, NativeEmission(An)


def _recording(An, em, seen):
    orig_a, orig_l = An.constraint_sets_for_access, An.layout_check_sets

    def rec_a(*a):
        want = orig_a(*a)
        got = em.constraint_sets_for_access(*a)
        seen.append((a, want, got))
        return want

    def rec_l(*a):
        want = orig_l(*a)
        got = em.layout_check_sets(*a)
        seen.append((a, want, got))
        return want

    return rec_a, rec_l, orig_a, orig_l


@pytest.mark.parametrize("m", [2**20, 64, 2**31 - 1])
@pytest.mark.parametrize("underflow", [True, False])
def test_native_sets_equal_reference_on_corpus(ref, m, underflow, monkeypatch):
    An, CG, em = ref
    seen = []
    rec_a, rec_l, _, _ = _recording(An, em, seen)
    monkeypatch.setattr(An, "constraint_sets_for_access", rec_a)
    monkeypatch.setattr(An, "layout_check_sets", rec_l)
    monkeypatch.setattr(An, "solve", lambda v, c, t=30.0: An.Unsat())
    corpus = reference_paths()[1]
    for p in sorted(corpus.glob("*/*.mcu")):
        An.analyze_source(p.read_text(), p.name, An.AnalyzerConfig(max_domain=m, check_underflow=underflow))
    n_sets = 0
    for args, want, got in seen:
        assert got == want, args[5] if len(args) > 6 else "layout"
        sets = [c.cset for c in want] if isinstance(want, list) else want.sets
        got_sets = [c.cset for c in got] if isinstance(got, list) else got.sets
        for w, g in zip(sets, got_sets):
            # the orders the solver depends on: variables, constraints, leaves
            assert [v.name for v in g.variables] == [v.name for v in w.variables]
            assert list(g.witness_leaves.items()) == list(w.witness_leaves.items())
            assert list(g.input_leaves.items()) == list(w.input_leaves.items())
            assert CG.render_constraint_set(g) == CG.render_constraint_set(w)
        n_sets += len(sets)
    assert n_sets >= (100 if underflow else 50)  # 110 queries at the default config (57 upper + layout)


def test_native_errors_match_reference(ref, monkeypatch):
    An, CG, em = ref
    from scuba_mini.expr_trees import BinOp, Const

    seen = []
    rec_a, rec_l, orig_a, _ = _recording(An, em, seen)
    monkeypatch.setattr(An, "constraint_sets_for_access", rec_a)
    monkeypatch.setattr(An, "solve", lambda v, c, t=30.0: An.Unsat())
    corpus = reference_paths()[1]
    prog = sorted(corpus.glob("*/*.mcu"))[0]
    An.analyze_source(prog.read_text(), prog.name, An.AnalyzerConfig())
    args = next(a for a, w, _ in seen if not w.size_unknown)
    access = args[5]
    for bad, text in ((BinOp("<", Const(1), Const(2)), "comparison in arithmetic position"),
                      (BinOp("^", Const(1), Const(2)), "unknown operator '^'"),
                      (BinOp("+", Const(1), 7), "unhandled ET node int")):
        a = list(args)
        a[5] = dataclasses.replace(access, offset_et=bad)
        with pytest.raises(CG.AnalysisError) as w:
            orig_a(*a)
        with pytest.raises(CG.AnalysisError) as g:
            em.constraint_sets_for_access(*a)
        assert str(g.value) == str(w.value) and text in str(g.value)


def test_batched_analysis_uses_native_emission(ref):
    An, CG, _ = ref
    from paper_2601_21552_b200 import emit

    calls = []
    orig = emit.NativeEmission.constraint_sets_for_access

    def spy(self, *a):
        calls.append(1)
        return orig(self, *a)

    emit.NativeEmission.constraint_sets_for_access = spy
    try:
        with emit.native_emission(An):
            assert An.constraint_sets_for_access.__func__ is spy
            prog = sorted(reference_paths()[1].glob("*/*.mcu"))[0]
            An.solve, saved = (lambda v, c, t=30.0: An.Unsat()), An.solve
            try:
                An.analyze_source(prog.read_text(), prog.name, An.AnalyzerConfig())
            finally:
                An.solve = saved
    finally:
        emit.NativeEmission.constraint_sets_for_access = orig
    assert calls
    assert An.constraint_sets_for_access is CG.constraint_sets_for_access  # restored
