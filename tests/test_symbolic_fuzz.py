"""Soundness fuzz of the fast mode's Unsat prover and of the engine's per-class
certificates (CPU: host builds of csrc/symbolic.cuh and csrc/cert.cuh).

Seeded random constraint systems -- all five relations, all five operators,
negative literals and domains, zero and negative divisors, nested products --
are decided by the C restatement of the reference (oracle/); a refutation of a
query the reference decides Sat would be a wrong answer.  Template families
(one random structure, many members that differ only in literal values and
domains) exercise what only certificates have: parameters, folded constants
checked per query, and the guards that decide whether a class certificate
applies to a member.
"""
from __future__ import annotations

import random

import numpy as np
import pytest

from test_symbolic_host import _engine_cert_refutes, prover  # noqa: F401  (fixture)

from oracle import oracle
from paper_2601_21552_b200.wire import flatten

OPS = "+-*/%"
RELS = ("<", "<=", "=", ">=", ">")


def rand_term(rng, names, depth, lits):
    if depth == 0 or rng.random() < 0.35:
        if rng.random() < 0.6:
            return rng.choice(names)
        return lits(rng)
    return [rng.choice(OPS), rand_term(rng, names, depth - 1, lits), rand_term(rng, names, depth - 1, lits)]


def rand_system(rng):
    nv = rng.randrange(1, 6)
    names = [f"x{i}" for i in range(nv)]
    vars_ = []
    for n in names:
        lo = rng.randrange(-20, 20)
        vars_.append([n, lo, lo + rng.randrange(0, 40)])
    lit = lambda r: r.randrange(-5, 13)  # noqa: E731
    cons = [[rng.choice(RELS), rand_term(rng, names, 3, lit), rand_term(rng, names, 3, lit)]
            for _ in range(rng.randrange(1, 6))]
    return {"vars": vars_, "cons": cons}


def shape(t):
    """the term with every literal replaced by a placeholder (structure)"""
    if isinstance(t, list):
        return [t[0], shape(t[1]), shape(t[2])]
    return t if isinstance(t, str) else "#"


def fill(t, rng):
    if isinstance(t, list):
        return [t[0], fill(t[1], rng), fill(t[2], rng)]
    return rng.randrange(-6, 16) if t == "#" else t


def template_family(rng, members):
    base = rand_system(rng)
    cons = [[r, shape(l), shape(h)] for r, l, h in base["cons"]]
    out = []
    for _ in range(members):
        vars_ = []
        for n, _, _ in base["vars"]:
            lo = rng.randrange(-10, 10)
            vars_.append([n, lo, lo + rng.randrange(0, 30)])
        out.append({"vars": vars_, "cons": [[r, fill(l, rng), fill(h, rng)] for r, l, h in cons]})
    return out


def decide(queries):
    fb = flatten(queries)
    v = oracle.solve_flat(fb, 30.0, threads=oracle.cpu_count())["verdict"]
    return fb, v


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_prover_never_refutes_sat_on_random_systems(prover, seed):  # noqa: F811
    rng = random.Random(seed)
    qs = [rand_system(rng) for _ in range(3000)]
    fb, v = decide(qs)
    r = prover(fb).astype(bool)
    assert not (r & (v == 1)).any(), np.nonzero(r & (v == 1))[0][:10]
    assert (v == 1).sum() > 300 and (v == 0).sum() > 300  # both verdicts well represented
    assert r.sum() > 0


@pytest.mark.parametrize("seed", [21, 22])
def test_class_certificates_sound_on_template_families(prover, seed):  # noqa: F811
    rng = random.Random(seed)
    qs = [q for _ in range(80) for q in template_family(rng, 40)]
    fb, v = decide(qs)
    r = _engine_cert_refutes(fb)
    assert not (r & (v == 1)).any(), np.nonzero(r & (v == 1))[0][:10]
    assert r.sum() > 0
