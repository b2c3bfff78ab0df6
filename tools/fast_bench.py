"""Fast vs canonical mode on the synthetic configs: plan runs (records
resident in HBM, CUDA-event device time) and verdict agreement.
usage: python tools/fast_bench.py [cfg:n ...]"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

args = sys.argv[1:] or ["c3:100000", "c4:100000", "c5s:100000", "c5:2000"]
for spec in args:
    cfg, n = spec.split(":")
    fb = synth.generate(cfg, int(n), names=False)
    res = {}
    for mode, flags in (("fast", _lib.F_FAST), ("canonical", 0)):
        if cfg == "c5" and mode == "canonical":
            continue
        t = time.perf_counter()
        p = _lib.Plan(fb, 30.0, flags=flags)
        tc = time.perf_counter() - t
        ms = [p.run() for _ in range(6)]
        r = p.results()
        res[mode] = r
        v = r["verdict"]
        print(f"{cfg} n={n} {mode:9s}: plan create {tc:.2f}s, run ms {sorted(ms)[1:4]} "
              f"-> {int(n) / (np.median(ms) * 1e-3) / 1e6:.2f} M q/s; unsat {int((v == 0).sum())} "
              f"sat {int((v == 1).sum())} timeout {int((v == 2).sum())} err {int((v == 3).sum())}", flush=True)
        p.close()
    if len(res) == 2:
        a, b = res["canonical"], res["fast"]
        print(f"  verdicts equal: {np.array_equal(a['verdict'], b['verdict'])}, "
              f"models equal: {np.array_equal(a['model'], b['model'])}", flush=True)
