"""The C-ABI library loads and exports every symbol include/*.h declares;
host-side contract checks that need no GPU (immediate verdicts, validation
errors, no CPU fallback)."""
from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, has_gpu

from paper_2601_21552_b200 import _lib
from paper_2601_21552_b200.solver import solve_flat
from paper_2601_21552_b200.wire import flatten


def declared_functions():
    names = []
    for h in sorted((ROOT / "include").glob("*.h")):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names += re.findall(r"^[A-Za-z_][\w \*]*?\b(oob_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert "oob_solve_batch" in names and "oob_plan_run" in names and "oob_synth_generate" in names
    L = _lib.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= set(names)


def test_version_and_device_count():
    assert b"sm_100a" in _lib.lib().oob_version()
    assert _lib.device_count() >= 0


def test_immediate_verdicts_need_no_device():
    # lo > hi => Unsat before search (solver.py:374); timeout <= 0 => Timeout
    fb = flatten([{"vars": [["x", 5, 4], ["y", 0, 3]], "cons": [["<", "y", 2]]}])
    out = solve_flat(fb, 30.0)
    assert out["verdict"][0] == _lib.UNSAT and out["nodes"][0] == 0
    fb = flatten([{"vars": [["x", 0, 3]], "cons": [["<", "x", 2]]}])
    out = solve_flat(fb, 0.0)
    assert out["verdict"][0] == _lib.TIMEOUT and out["elapsed"][0] > 0


def test_malformed_batches_raise_value_error():
    fb = flatten([{"vars": [["x", 0, 3]], "cons": [["<", "x", 2]]}])
    fb.node_op[:] = 9
    with pytest.raises(ValueError, match="unknown operator"):
        solve_flat(fb, 30.0)
    fb = flatten([{"vars": [["x", 0, 3]], "cons": [["<", "x", 2]]}])
    fb.con_rel[:] = 7
    with pytest.raises(ValueError, match="unknown relation"):
        solve_flat(fb, 30.0)
    fb = flatten([{"vars": [["x", 0, 3]], "cons": [["<", "x", 2]]}])
    fb.node_a[fb.node_op == 1] = 5
    with pytest.raises(ValueError, match="undeclared variable"):
        solve_flat(fb, 30.0)


@pytest.mark.skipif(has_gpu(), reason="checks the no-device path")
def test_no_cpu_fallback_without_device():
    fb = flatten([{"vars": [["x", 0, 3]], "cons": [["<", "x", 2]]}])
    with pytest.raises(_lib.EngineError, match="no CPU fallback"):
        solve_flat(fb, 30.0)


def test_side_constraint_count_matches_oracle():
    from oracle import oracle
    from conftest import load_golden
    recs = load_golden("random_solver") + load_golden("crafted")
    fb = flatten(recs)
    assert np.array_equal(_lib.side_counts(fb), oracle.side_counts(fb))


def test_option_flags_match_the_header():
    """The shim's option flags are the header's OOB_F_* values."""
    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "scuba_oob.h").read_text(), flags=re.S)
    hdr = {m[0]: int(m[1]) for m in re.findall(r"\bOOB_F_(\w+)\s*=\s*(\d+)", text)}
    shim = {k[2:]: v for k, v in vars(_lib).items() if re.fullmatch(r"F_[A-Z0-9_]+", k)}
    assert hdr and hdr == shim, (hdr, shim)
