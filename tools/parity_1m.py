"""Full-batch parity at BASELINE config 4's size: 1M C4 queries decided on the
GPU (fast and canonical) and by the C restatement of the reference on all
host cores; every verdict and model word compared, counters for canonical.
One JSON line (profiles/r02_parity_c4_1m.json)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
fb = synth.generate(cfg, n, names=False)
res = {}
for mode, flags in (("fast", _lib.F_FAST), ("canonical", 0)):
    p = _lib.Plan(fb, 30.0, n_gpus=1, flags=flags)
    ms = p.run()
    res[mode] = (p.results(), ms)
    p.close()
t = time.perf_counter()
ref = oracle.solve_flat(fb, 30.0, threads=oracle.cpu_count())
dt = time.perf_counter() - t
f, c = res["fast"][0], res["canonical"][0]
out = {"config": cfg, "queries": n, "port_seconds": round(dt, 1), "port_threads": oracle.cpu_count(),
       "gpu_ms": {"fast": round(res["fast"][1], 2), "canonical": round(res["canonical"][1], 2)},
       "sat": int((ref["verdict"] == 1).sum()), "unsat": int((ref["verdict"] == 0).sum()),
       "timeout": int((ref["verdict"] == 2).sum()),
       "fast_vs_port": {"verdict_mismatches": int((f["verdict"] != ref["verdict"]).sum()),
                        "model_word_mismatches": int((f["model"] != ref["model"]).any(axis=1).sum())},
       "canonical_vs_port": {"verdict_mismatches": int((c["verdict"] != ref["verdict"]).sum()),
                             "model_word_mismatches": int((c["model"] != ref["model"]).any(axis=1).sum()),
                             "node_mismatches": int((c["nodes"] != ref["nodes"]).sum()),
                             "pass_mismatches": int((c["passes"] != ref["passes"]).sum())}}
print(json.dumps(out), flush=True)
