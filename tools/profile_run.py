"""Per-query device timing dump for kernel analysis (run on the GPU box).

    python tools/profile_run.py [config] [n] [out.npz]
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
dst = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/profile_run.npz"
fb = synth.generate(cfg, n, names=False)
plan = _lib.Plan(fb, 30.0, n_gpus=1, device=0)
info = plan.info()
ms = [plan.run() for _ in range(3)]
res = plan.results()
print("info", info, "kernel ms", ms)
np.savez_compressed(dst, elapsed=res["elapsed"], nodes=res["nodes"], passes=res["passes"],
                    verdict=res["verdict"], tmpl=fb.tmpl, nv=np.diff(fb.var_begin),
                    ncon=np.diff(fb.con_begin), nnode=np.diff(fb.node_begin), ms=np.array(ms))
