"""The C oracle (CPU restatement of solver.py) against the golden capture of
the real Python reference: verdict, first model, DFS nodes, passes."""
from __future__ import annotations

import pytest

from conftest import GOLDEN_SETS, VCODE, load_golden

from oracle import oracle
from paper_2601_21552_b200.solver import divisor_side_constraints
from paper_2601_21552_b200.terms import query_from_json
from paper_2601_21552_b200.wire import flatten, words_to_ints


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_oracle_matches_reference(name):
    recs = load_golden(name)
    for q, r in enumerate(recs):
        fb = flatten([r])
        out = oracle.solve_flat(fb, r["timeout"])
        assert int(out["verdict"][0]) == VCODE[r["verdict"]], (name, q)
        if r["verdict"] == "timeout":
            continue
        assert int(out["nodes"][0]) == r["nodes"], (name, q)
        assert int(out["passes"][0]) == r["passes"], (name, q)
        if r["verdict"] == "sat":
            model = dict(zip(fb.names(0), words_to_ints(out["model"][: fb.n_vars_total])))
            assert model == r["model"], (name, q)


def test_side_constraints_agree(golden):
    recs = [r for n in ("random_solver", "random_accept", "crafted") for r in golden[n]]
    fb = flatten(recs)
    counts = oracle.side_counts(fb)
    for q, r in enumerate(recs):
        _, cons = query_from_json(r)
        assert len(divisor_side_constraints(cons)) == int(counts[q]), q


def test_models_of_enumeration_sets_check(golden):
    """Every reference model satisfies the oracle's check_model; the first
    enumerated model exists iff the reference says Sat."""
    for name in ("random_solver", "random_accept"):
        for r in golden[name]:
            assert (r["enum"] is not None) == (r["verdict"] == "sat")
