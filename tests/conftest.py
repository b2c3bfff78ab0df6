"""Shared test plumbing: the `gpu` marker, golden fixtures, import paths."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
REF_SRC = Path("/root/reference/pkg/src")
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_SETS = ("corpus_m1048576", "corpus_m64", "crafted", "random_solver", "random_accept",
               "synth_c3", "synth_c4", "synth_c5s")
VCODE = {"unsat": 0, "sat": 1, "timeout": 2}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name: str) -> list:
    with open(GOLDEN / f"{name}.jsonl") as f:
        return [json.loads(line) for line in f]


BASELINE_REF = ROOT / "baseline" / "_ref"  # tools/install_reference.sh (travels to the GPU box)


def reference_paths():
    """(package dir, corpus dir) of the reference: the install under
    baseline/_ref (present on the GPU box), else the mounted source tree
    (build container); (None, None) when neither exists."""
    if (BASELINE_REF / "scuba_mini" / "solver.py").exists() and (BASELINE_REF / "corpus").exists():
        return BASELINE_REF, BASELINE_REF / "corpus"
    if (REF_SRC / "scuba_mini" / "solver.py").exists():
        return REF_SRC, REF_SRC.parent / "corpus"
    return None, None


def reference_available() -> bool:
    return reference_paths()[0] is not None


@pytest.fixture(scope="session")
def golden():
    return {name: load_golden(name) for name in GOLDEN_SETS}


def has_gpu() -> bool:
    try:
        from paper_2601_21552_b200 import _lib
        return _lib.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("GPU test run without a visible CUDA device / engine library")
    return True
