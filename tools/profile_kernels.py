"""One plan run of a synthetic stream (for an ncu launch list).
usage: python tools/profile_kernels.py [cfg] [n] [mode: fast|canonical] [heavy_nodes]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
mode = sys.argv[3] if len(sys.argv) > 3 else "fast"
heavy = int(sys.argv[4]) if len(sys.argv) > 4 else 0
fb = synth.generate(cfg, n, names=False)
plan = _lib.Plan(fb, 30.0, n_gpus=1, device=0, heavy_nodes=heavy, flags=_lib.F_FAST if mode == "fast" else 0)
print(plan.info(), "ms", plan.run())
if os.environ.get("SCUBA_OOB_TIMELINE"):
    plan.results()
