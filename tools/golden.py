"""Golden-vector capture from the REAL reference (run in the build container).

Imports the reference package from /root/reference/pkg/src (read-only; never
copied) and records, for every query of every fixture set, the query in the
JSON form of `paper_2601_21552_b200.terms`, the reference verdict and model,
and the reference's own work counters:

  nodes   number of `_search` calls     (solver.py:385)
  passes  number of propagation passes  (one `_Narrower` per pass, solver.py:274)

Those counters pin the *traversal*, not only the answer: an engine that
reproduces them performed the same DFS and the same propagation schedule.

Fixture sets written under tests/golden/:
  corpus_m1048576.jsonl   every solve() call of the analyzer over the 20
                          corpus programs at the default config (110 queries)
  corpus_m64.jsonl        the same at max_domain=64 (acceptance criterion 8)
  corpus_diags.json       analyzer JSON diagnostics per program (default and
                          M=64) + per-access replay_witness outcomes
  random_solver.jsonl     test_solver.random_system, seed 40 x150 and seed 7 x40
  random_accept.jsonl     test_acceptance._random_system, seed 2026 x200
  crafted.jsonl           hand-made edge cases (clamp, traps, negatives, ...)
  synth_<cfg>.jsonl       first queries of the native synthetic generator
                          (tools/golden.py synth ...), when the library is built

Usage:  python tools/golden.py [all|corpus|random|crafted|synth]
"""
from __future__ import annotations

import json
import os
import random
import sys
import time
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
REF_CORPUS = Path("/root/reference/pkg/corpus")
REPO = Path(__file__).resolve().parents[1]
OUT = REPO / "tests" / "golden"

sys.dont_write_bytecode = True
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REF_SRC))

import scuba_mini.solver as S  # noqa: E402  (reference)

from paper_2601_21552_b200.terms import query_to_json, verdict_to_json  # noqa: E402


# ----- counting hooks on the reference solver -------------------------------

class _Counts:
    nodes = 0
    passes = 0


_orig_search = S._search
_OrigNarrower = S._Narrower


def _counting_search(*a, **k):
    _Counts.nodes += 1
    return _orig_search(*a, **k)


class _CountingNarrower(_OrigNarrower):
    def __init__(self, env):
        _Counts.passes += 1
        super().__init__(env)


S._search = _counting_search
S._Narrower = _CountingNarrower


def ref_solve(variables, constraints, timeout_s=30.0):
    """Reference solve() + its counters + wall time."""
    _Counts.nodes = _Counts.passes = 0
    t0 = time.perf_counter()
    v = S.solve(variables, constraints, timeout_s)
    dt = time.perf_counter() - t0
    return v, _Counts.nodes, _Counts.passes, dt


def record(variables, constraints, timeout_s=30.0, **extra):
    v, nodes, passes, dt = ref_solve(variables, constraints, timeout_s)
    rec = {**extra, **query_to_json(variables, constraints),
           "timeout": timeout_s, **verdict_to_json(v),
           "nodes": nodes, "passes": passes, "ref_ms": round(dt * 1e3, 3)}
    return rec


def write_jsonl(name, recs):
    OUT.mkdir(parents=True, exist_ok=True)
    with open(OUT / name, "w") as f:
        for r in recs:
            f.write(json.dumps(r, separators=(",", ":")) + "\n")
    print(f"wrote {name}: {len(recs)} records")


# ----- corpus ---------------------------------------------------------------

def corpus_files():
    return sorted(REF_CORPUS.glob("*/*.mcu"))


def capture_corpus():
    import scuba_mini.analyzer as An
    from scuba_mini.analyzer import AnalyzerConfig, analyze_source
    from scuba_mini.frontend import parse_source
    from scuba_mini.oracle import replay_witness
    from scuba_mini.report import render_json_lines

    diags = {}
    for m in (2**20, 64):
        recs = []
        real = An.solve

        def hook(variables, constraints, timeout_s=30.0):
            rec = record(variables, constraints, timeout_s,
                         prog=hook.prog, idx=hook.idx)
            hook.idx += 1
            recs.append(rec)
            return real(variables, constraints, timeout_s)

        An.solve = hook
        try:
            for p in corpus_files():
                rel = f"{p.parent.name}/{p.name}"
                hook.prog, hook.idx = rel, 0
                src = p.read_text()
                res = analyze_source(src, p.name, AnalyzerConfig(max_domain=m))
                prog_recs = [r for r in recs if r["prog"] == rel]
                program = parse_source(src, p.name)
                replays = []
                for acr in res.access_results:
                    loc = acr.access.location
                    for o in acr.outcomes:
                        if type(o.verdict).__name__ == "Sat":
                            hit, _ = replay_witness(program, o.witness_inputs,
                                                    64, loc.line, loc.column)
                            replays.append({
                                "line": loc.line, "col": loc.column,
                                "check": o.check,
                                "inputs": {str(k): v for k, v in
                                           o.witness_inputs.items()},
                                "replayed": bool(hit)})
                diags.setdefault(rel, {})[f"m{m}"] = {
                    "json": render_json_lines(res.diagnostics),
                    "replays": replays,
                    "n_queries": len(prog_recs),
                }
        finally:
            An.solve = real
        write_jsonl(f"corpus_m{m}.jsonl", recs)
    with open(OUT / "corpus_diags.json", "w") as f:
        json.dump(diags, f, indent=1, sort_keys=True)
    print("wrote corpus_diags.json")


# ----- randomized systems (the reference's own generators) ------------------

def brute_first_model(variables, constraints):
    import itertools
    full = list(constraints) + S.divisor_side_constraints(constraints)
    names = [v.name for v in variables]
    for values in itertools.product(*[range(v.lo, v.hi + 1) for v in variables]):
        model = dict(zip(names, values))
        if S.check_model(full, model):
            return model
    return None


def capture_random():
    sys.path.insert(0, str(REF_TESTS))
    import test_solver as TS        # reference tests, imported (not copied)
    import test_acceptance as TA

    recs = []
    for seed, n in ((40, 150), (7, 40)):
        rng = random.Random(seed)
        for i in range(n):
            vs, cs = TS.random_system(rng)
            r = record(vs, cs, 10.0, gen="test_solver", seed=seed, i=i)
            r["enum"] = brute_first_model(vs, cs)
            recs.append(r)
    write_jsonl("random_solver.jsonl", recs)

    recs = []
    rng = random.Random(2026)
    for i in range(200):
        vs, cs = TA._random_system(rng)
        r = record(vs, cs, 20.0, gen="test_acceptance", seed=2026, i=i)
        r["enum"] = brute_first_model(vs, cs)
        recs.append(r)
    write_jsonl("random_accept.jsonl", recs)


# ----- crafted edge cases ---------------------------------------------------

def crafted_cases():
    L, V, B, C, SV = S.Lit, S.VarRef, S.BinE, S.Constraint, S.SolverVar
    x, y, z = V("x"), V("y"), V("z")
    cases = []

    def add(name, vs, cs, timeout=30.0):
        cases.append((name, vs, cs, timeout))

    # solver tests (test_solver.py:113-189) restated as data
    add("xy100", [SV("x", 0, 10), SV("y", 0, 10)],
        [C("=", B("*", x, y), L(100))])
    add("guarded", [SV("tid", 0, 64), SV("n", 0, 64)],
        [C("<", V("tid"), V("n")), C(">=", V("tid"), V("n"))])
    add("div0", [SV("x", 0, 0)], [C("=", B("/", L(4), x), L(0))])
    add("trunc7", [SV("x", 1, 7)], [C("=", B("/", L(7), x), L(2))])
    add("negoff", [SV("off", -64, 64), SV("n", 1, 8)],
        [C("=", V("off"), B("-", L(0), V("n"))), C("<", V("off"), L(0))])
    add("modcheck", [SV("a", 0, 9), SV("b", 0, 9), SV("d", 1, 9)],
        [C("=", B("%", V("a"), V("d")), L(2)),
         C("<", V("b"), B("/", V("a"), V("d")))])
    # structure edges
    add("empty_vars", [], [])
    add("no_constraints", [SV("x", -3, 5), SV("y", 2, 2)], [])
    add("lit_only_true", [], [C("<", L(1), L(2))])
    add("lit_only_false", [], [C(">", L(1), L(2))])
    add("lo_gt_hi", [SV("x", 5, 4), SV("y", 0, 3)], [C("<", y, L(2))])
    add("lo_gt_hi_t0", [SV("x", 5, 4)], [], 0.0)
    add("timeout0", [SV("x", 0, 3)], [C("<", x, L(2))], 0.0)
    add("timeout_neg", [SV("x", 0, 3)], [C("<", x, L(2))], -1.0)
    # _INF clamp (solver.py:23) -- reference Unsat though mathematically Sat
    add("inf_clamp_gt", [SV("x", 0, 2**62)], [C(">", x, L(10**18 + 5))])
    add("inf_clamp_mul", [SV("x", 0, 2**31), SV("y", 0, 2**31)],
        [C(">=", B("*", x, y), L(2**61))])
    add("inf_edge_ok", [SV("x", 0, 2**62)], [C(">=", x, L(10**18))])
    add("inf_edge_bad", [SV("x", 0, 2**62)], [C(">=", x, L(10**18 + 1))])
    # wide (int128 regime) arithmetic
    add("wide_prod", [SV("a", 0, 2**40), SV("b", 0, 2**40), SV("c", 0, 2**40)],
        [C("=", V("c"), B("/", B("*", V("a"), V("b")), L(2**45))),
         C(">", V("c"), L(1000)), C("<", V("a"), L(2**22))])
    add("wide_neg", [SV("a", -2**50, 2**50), SV("b", -2**50, 2**50)],
        [C("<=", B("*", V("a"), V("b")), L(-(2**55))),
         C(">=", V("a"), L(2**49))])
    add("wide_clamp", [SV("a", -2**50, 2**50), SV("b", -2**50, 2**50)],
        [C("<=", B("*", V("a"), V("b")), L(-(2**95))),
         C(">=", V("a"), L(2**49))])
    # division / modulo semantics with negatives
    add("tdiv_neg", [SV("x", -20, 20), SV("d", -5, 5)],
        [C("=", B("/", x, V("d")), L(-3)), C("=", B("%", x, V("d")), L(-2))])
    add("mod_neg", [SV("x", -9, 9)], [C("=", B("%", x, L(4)), L(-3))])
    add("div_lit0", [SV("x", 0, 9)], [C(">=", B("/", x, L(0)), L(0))])
    add("mod_lit0", [SV("x", 0, 9)], [C(">=", B("%", x, L(0)), L(0))])
    add("div_neg_lit", [SV("x", -9, 9)], [C("=", B("/", x, L(-2)), L(3))])
    add("div_var_side", [SV("x", 0, 30), SV("y", -3, 3)],
        [C("=", B("/", x, y), L(7)), C("=", B("%", x, y), L(1))])
    add("dup_divisors", [SV("x", 0, 30), SV("y", 0, 3), SV("z", 0, 3)],
        [C("=", B("/", x, B("+", y, z)), L(7)),
         C("<", B("%", x, B("+", y, z)), L(2)),
         C(">", B("/", z, y), L(0))])
    # negative domains, floor midpoint on negative sums
    add("neg_mid", [SV("x", -7, -1), SV("y", -6, 3)],
        [C("=", B("+", x, y), L(-9)), C(">", B("*", x, y), L(5))])
    add("neg_mul_skip", [SV("x", -5, 5), SV("y", -5, 5)],
        [C("=", B("*", x, y), L(-12)), C("<", x, y)])
    add("mul_neg_target", [SV("x", 0, 5), SV("y", 0, 5)],
        [C("<", B("*", x, y), L(0))])
    # creeping propagation (bounds move one unit per pass)
    add("creep_small", [SV("a", 0, 300), SV("b", 0, 300)],
        [C("<", V("a"), V("b")), C(">=", V("a"), V("b"))])
    add("creep_cap", [SV("a", 0, 30000), SV("b", 0, 30000)],
        [C("<", V("a"), V("b")), C(">=", V("a"), V("b"))])
    add("creep_cap_sat", [SV("a", 0, 40000), SV("b", 0, 40000), SV("c", 0, 40000)],
        [C("<", V("a"), V("b")), C("<", V("b"), B("+", V("a"), L(2))),
         C("=", V("c"), B("*", V("a"), L(1))), C(">", V("c"), L(39990))])
    # smallest-domain tie-breaks and splitting
    add("ties", [SV("p", 0, 3), SV("q", 0, 3), SV("r", 0, 7)],
        [C("=", B("+", B("*", V("p"), L(4)), V("q")), V("r")),
         C("=", B("%", V("r"), L(3)), L(2)), C(">", V("q"), V("p"))])
    add("big_split", [SV("x", 0, 10**6), SV("y", 0, 10**6)],
        [C("=", B("*", x, y), L(999_983 * 7)), C("<", x, y)])
    # x32-regime proof regressions: narrowing targets that only
    # become real below the root (a `*` side whose lower bound is 0 or
    # negative at the root) must be bounded by the x32 eligibility proof
    add("x32_mul_late", [SV("x", 0, 5), SV("z", 0, 2**24)],
        [C("<=", B("*", x, B("/", z, L(1000))), L(7_000_000)),
         C("=", B("%", x, L(8)), L(3))])
    add("x32_mul_negroot", [SV("b", 0, 5), SV("z", 0, 2**24)],
        [C("<=", B("*", B("-", V("b"), L(1)), B("/", z, L(1000))), L(7_000_000)),
         C("=", B("%", V("b"), L(8)), L(3))])
    add("x32_mul_late_unsat", [SV("x", 0, 5), SV("z", 0, 2**24)],
        [C("<=", B("*", x, B("/", z, L(1000))), L(7_000_000)),
         C("=", B("%", x, L(8)), L(3)), C(">", z, L(2_333_334_000 // 1000))])
    add("x32_add_chain", [SV("x", 0, 6), SV("y", 0, 2**20), SV("z", 0, 2**24)],
        [C("<=", B("+", B("*", x, B("/", z, L(100))), y), L(2**27)),
         C(">", x, L(2)), C(">=", z, B("*", y, L(8)))])
    return cases


def capture_crafted():
    recs = []
    for name, vs, cs, t in crafted_cases():
        r = record(vs, cs, t, name=name)
        if r["verdict"] == "timeout":
            r.pop("nodes"); r.pop("passes")
        recs.append(r)
    write_jsonl("crafted.jsonl", recs)


# ----- synthetic subsamples (needs the built native library) ----------------

def capture_synth(n_per=400):
    from paper_2601_21552_b200 import synth
    from paper_2601_21552_b200.terms import query_from_json
    for cfg in synth.CONFIGS:
        qs = synth.generate_json(cfg, n_per)
        recs = []
        for i, q in enumerate(qs):
            vs, cs = query_from_json(q, S)
            recs.append(record(vs, cs, 30.0, cfg=cfg, i=i))
        write_jsonl(f"synth_{cfg}.jsonl", recs)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "corpus"):
        capture_corpus()
    if what in ("all", "random"):
        capture_random()
    if what in ("all", "crafted"):
        capture_crafted()
    if what in ("synth",):
        capture_synth(int(sys.argv[2]) if len(sys.argv) > 2 else 400)
