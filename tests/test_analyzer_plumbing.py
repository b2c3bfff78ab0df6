"""Analyzer integration (paper_2601_21552_b200.analyzer) against the real
reference front end (baseline/_ref, or the mounted reference).  The engine
call is stood in by the C oracle so the test runs without a GPU: it checks the
plumbing -- record/replay, flattening of the reference's own objects, verdict
objects of the reference's classes -- reproduces the reference's diagnostics
byte for byte on the whole corpus.  tests/test_gpu_analyzer.py runs the same
analyses with the CUDA engine.
"""
from __future__ import annotations

import json
import sys

import pytest

from conftest import GOLDEN, reference_available, reference_paths

pytestmark = pytest.mark.skipif(not reference_available(), reason="reference not mounted")


@pytest.fixture
def ref(monkeypatch):
    sys.path.insert(0, str(reference_paths()[0]))
    import scuba_mini.analyzer as An
    from oracle import oracle
    from paper_2601_21552_b200 import _lib

    def oracle_engine(fb, timeout_s=30.0, node_budget=0, n_gpus=0, device=0, flags=0, heavy_nodes=0, jit_min=0):
        out = oracle.solve_flat(fb, timeout_s, node_budget)
        out["status"], out["error"] = 0, ""
        return out

    monkeypatch.setattr(_lib, "solve_flat", oracle_engine)
    return An


@pytest.mark.parametrize("m", [2**20, 64])
def test_batched_analysis_reproduces_reference_diagnostics(ref, m):
    from pathlib import Path

    from scuba_mini.analyzer import AnalyzerConfig, analyze_source
    from scuba_mini.report import render_json_lines

    from paper_2601_21552_b200.analyzer import analyze_batched

    want = json.loads((GOLDEN / "corpus_diags.json").read_text())
    corpus = reference_paths()[1]
    total = 0
    for p in sorted(corpus.glob("*/*.mcu")):
        rel = f"{p.parent.name}/{p.name}"
        stats = {}
        res = analyze_batched(ref, analyze_source, p.read_text(), p.name,
                              AnalyzerConfig(max_domain=m), stats=stats)
        assert render_json_lines(res.diagnostics) == want[rel][f"m{m}"]["json"], rel
        assert stats["queries"] == want[rel][f"m{m}"]["n_queries"]
        total += stats["queries"]
    assert total == 110


def test_installed_solve_replaces_reference_binding(ref):
    from scuba_mini.analyzer import analyze_source
    from scuba_mini.report import render_json_lines

    from paper_2601_21552_b200.analyzer import installed

    want = json.loads((GOLDEN / "corpus_diags.json").read_text())
    src = (reference_paths()[1] / "figs/sosfilt_intra.mcu").read_text()
    with installed(ref):
        res = analyze_source(src, "sosfilt_intra.mcu")
    assert render_json_lines(res.diagnostics) == want["figs/sosfilt_intra.mcu"]["m1048576"]["json"]


def test_whole_corpus_in_one_batch(ref):
    """analyze_many: every corpus program's queries in one device batch, the
    diagnostics of each program still the reference's byte for byte."""
    from pathlib import Path

    from scuba_mini.analyzer import AnalyzerConfig, analyze_source
    from scuba_mini.report import render_json_lines

    from paper_2601_21552_b200.analyzer import analyze_many

    want = json.loads((GOLDEN / "corpus_diags.json").read_text())
    progs = sorted(reference_paths()[1].glob("*/*.mcu"))
    jobs = [((p.read_text(), p.name, AnalyzerConfig()), {}) for p in progs]
    stats = {}
    results = analyze_many(ref, analyze_source, jobs, stats=stats)
    assert stats["queries"] == 110 and stats["batches"] == 1
    for p, res in zip(progs, results):
        rel = f"{p.parent.name}/{p.name}"
        assert render_json_lines(res.diagnostics) == want[rel]["m1048576"]["json"], rel
