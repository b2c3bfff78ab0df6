"""pytest plugin: the reference's own test suite with the GPU engine bound in
place of its solver -- `scuba_mini.solver.solve` and the analyzer's `solve`
both become the CUDA engine's solve() (reference verdict classes returned),
in the mode named by SCUBA_REF_SUITE_MODE (canonical | fast).
tools/ref_suite_gpu.sh runs it on the GPU box."""
import os
import sys

_here = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(_here, ".."))
sys.path.insert(0, os.path.join(_here, "..", "baseline", "_ref"))
import scuba_mini.analyzer as An  # noqa: E402
import scuba_mini.solver as S  # noqa: E402
from paper_2601_21552_b200 import _lib  # noqa: E402
from paper_2601_21552_b200.analyzer import install  # noqa: E402

if _lib.device_count() < 1:
    raise RuntimeError("ref_patch_gpu: no CUDA device (the engine has no CPU path)")
_mode = os.environ.get("SCUBA_REF_SUITE_MODE", "canonical")
_inner = install(An, mode=_mode)
_calls = [0]


def _gpu(*a, **k):
    _calls[0] += 1
    return _inner(*a, **k)


An.solve = _gpu
S.solve = _gpu


def pytest_sessionfinish(session, exitstatus):
    print(f"\nreference suite: {_calls[0]} solve() calls decided by the GPU engine ({_mode} mode)",
          file=sys.stderr)
print(f"GPU engine bound into scuba_mini.solver.solve and the analyzer ({_mode} mode)", file=sys.stderr)
