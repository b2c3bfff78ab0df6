"""The native synthetic generator: determinism, slicing, and identity with the
streams the golden capture was taken from (so the GPU box regenerates the
exact queries the Python reference decided)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden

from paper_2601_21552_b200 import synth


@pytest.mark.parametrize("cfg", synth.CONFIGS)
def test_stream_matches_golden(cfg):
    recs = load_golden(f"synth_{cfg}")
    fb = synth.generate(cfg, len(recs))
    for q, r in enumerate(recs):
        j = fb.query_json(q)
        assert j["vars"] == r["vars"] and j["cons"] == r["cons"], (cfg, q)


@pytest.mark.parametrize("cfg", ("c3", "c4", "c5"))
def test_slices_are_independent(cfg):
    a = synth.generate(cfg, 96, first=0)
    b = synth.generate(cfg, 32, first=64)
    for q in range(32):
        assert a.query_json(64 + q) == b.query_json(q)


def test_shapes_are_analyzer_like():
    fb = synth.generate("c3", 500)
    nv = np.diff(fb.var_begin)
    assert nv.min() >= 12 + 1 and nv.max() <= 32
    tm = fb.tmpl // 4
    assert set(np.unique(tm)) == set(range(1, 8))
    # first 12 variables are always the launch geometry (constraint_gen.py:105-107)
    assert fb.names(0)[:12] == ["sol" + a for a in synth.AXES]
