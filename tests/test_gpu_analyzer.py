"""The reference analyzer driving the CUDA engine (BASELINE config 2, the
20-program corpus): the reference front end runs unchanged (baseline/_ref on
the GPU box), its solver calls are decided on the B200 through the C ABI, and
the diagnostics must be byte-identical to the reference's own run
(tests/golden/corpus_diags.json, captured by tools/golden.py), in canonical
and in fast mode, per program (record/replay), for the whole corpus in one
device batch, and with the solve() binding replaced directly.
"""
from __future__ import annotations

import json
import sys

import pytest

from conftest import GOLDEN, reference_paths

pytestmark = pytest.mark.gpu

PKG, CORPUS = reference_paths()


@pytest.fixture(scope="module")
def ref(gpu):
    if PKG is None:
        pytest.skip("reference package not installed (tools/install_reference.sh)")
    sys.path.insert(0, str(PKG))
    import scuba_mini.analyzer as An
    return An


WANT = json.loads((GOLDEN / "corpus_diags.json").read_text())


@pytest.mark.parametrize("mode", ["canonical", "fast"])
@pytest.mark.parametrize("m", [2**20, 64])
def test_corpus_per_program_on_gpu(ref, m, mode):
    from scuba_mini.analyzer import AnalyzerConfig, analyze_source
    from scuba_mini.report import render_json_lines

    from paper_2601_21552_b200.analyzer import analyze_batched

    total = 0
    progs = sorted(CORPUS.glob("*/*.mcu"))
    assert len(progs) == 20
    for p in progs:
        rel = f"{p.parent.name}/{p.name}"
        stats = {}
        res = analyze_batched(ref, analyze_source, p.read_text(), p.name, AnalyzerConfig(max_domain=m),
                              stats=stats, mode=mode)
        assert render_json_lines(res.diagnostics) == WANT[rel][f"m{m}"]["json"], rel
        total += stats["queries"]
    assert total == 110


@pytest.mark.parametrize("mode", ["canonical", "fast"])
@pytest.mark.parametrize("m", [2**20, 64])
def test_corpus_in_one_device_batch(ref, m, mode):
    from scuba_mini.analyzer import AnalyzerConfig, analyze_source
    from scuba_mini.report import render_json_lines

    from paper_2601_21552_b200.analyzer import analyze_many

    progs = sorted(CORPUS.glob("*/*.mcu"))
    jobs = [((p.read_text(), p.name, AnalyzerConfig(max_domain=m)), {}) for p in progs]
    stats = {}
    results = analyze_many(ref, analyze_source, jobs, stats=stats, mode=mode)
    assert stats["queries"] == 110 and stats["batches"] == 1
    findings = 0
    for p, res in zip(progs, results):
        rel = f"{p.parent.name}/{p.name}"
        out = render_json_lines(res.diagnostics)
        assert out == WANT[rel][f"m{m}"]["json"], rel
        findings += len(res.diagnostics)
        if p.parent.name == "clean":
            assert not res.diagnostics, rel  # zero false alarms on the bug-free programs
    assert findings == 17  # 10 OOB-class (the 10 Sat verdicts) + 7 use-after-free


def test_installed_solve_binding_on_gpu(ref):
    from scuba_mini.analyzer import analyze_source
    from scuba_mini.report import render_json_lines

    from paper_2601_21552_b200.analyzer import installed

    src = (CORPUS / "figs/sosfilt_intra.mcu").read_text()
    for mode in ("canonical", "fast"):
        with installed(ref, mode=mode):
            res = analyze_source(src, "sosfilt_intra.mcu")
        assert render_json_lines(res.diagnostics) == WANT["figs/sosfilt_intra.mcu"]["m1048576"]["json"]
