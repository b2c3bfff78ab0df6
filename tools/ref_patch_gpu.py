"""pytest plugin: the reference's own test suite with the GPU engine bound in
place of its solver -- `scuba_mini.solver.solve` and the analyzer's `solve`
both become the CUDA engine's solve() (reference verdict classes returned),
`scuba_mini.solver.propagate` the engine's propagate() (its check_model stays
the reference's: the suite uses it to check solve()'s models),
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
# propagate() too (the GPU aux kernel); check_model stays the reference's:
# the suite uses it as the independent checker of solve()'s models
from paper_2601_21552_b200 import solver as _ours  # noqa: E402
_prop_calls = [0]


def _gpu_propagate(domains, constraints, deadline=None):
    _prop_calls[0] += 1
    return _ours.propagate(domains, constraints, deadline)


S.propagate = _gpu_propagate


def pytest_sessionfinish(session, exitstatus):
    print(f"\nreference suite: {_calls[0]} solve() calls decided by the GPU engine ({_mode} mode), "
          f"{_prop_calls[0]} propagate() calls on the GPU", file=sys.stderr)
print(f"GPU engine bound into scuba_mini.solver.solve and the analyzer ({_mode} mode)", file=sys.stderr)
