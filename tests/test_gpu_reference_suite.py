"""The reference's own test suite (200 tests: solver unit and randomized
agreement tests, analyzer, acceptance criteria over the corpus) with every
solve() it makes decided by the CUDA engine (tools/ref_patch_gpu.py binds the
engine into scuba_mini.solver.solve and the analyzer), in both modes."""
from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
SUITE = ROOT / "baseline" / "_ref" / "tests"


@pytest.mark.parametrize("mode", ["canonical", "fast"])
def test_reference_suite_on_the_gpu_engine(gpu, mode):
    if not SUITE.is_dir():
        pytest.skip("reference suite not installed (tools/install_reference.sh)")
    env = dict(os.environ, SCUBA_REF_SUITE_MODE=mode,
               PYTHONPATH=f"{ROOT / 'tools'}:{ROOT / 'baseline' / '_ref'}")
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "ref_patch_gpu", str(SUITE), "-q",
                        "-p", "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    m = re.search(r"(\d+) solve\(\) calls decided by the GPU engine", out)
    assert m and int(m.group(1)) > 1000, out[-2000:]
    assert re.search(r"\b200 passed\b", out), out[-2000:]
