"""Fast mode with / without the warp-per-query search (chain.cuh), against
canonical mode on the same batches: verdicts, models and node counts must be
identical; prints plan-run times and how many Sat entries the search decided
(their pass counts are the search's rounds).
usage: SCUBA_OOB_CHAIN=0|1 python tools/chain_ab.py (1: OOB_F_CHAIN on) [cfg:n ...]"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

args = sys.argv[1:] or ["c3:100000", "c4:100000", "c5s:100000"]
tag = os.environ.get("SCUBA_OOB_CHAIN", "1")
for spec in args:
    cfg, n = spec.split(":")
    fb = synth.generate(cfg, int(n), names=False)
    p = _lib.Plan(fb, 30.0, flags=0)
    p.run()
    c = p.results()
    p.close()
    p = _lib.Plan(fb, 30.0, flags=_lib.F_FAST | (_lib.F_CHAIN if tag == "1" else 0))
    ms = [p.run() for _ in range(7)]
    f = p.results()
    p.close()
    sat = c["verdict"] == _lib.SAT
    same_v = np.array_equal(c["verdict"], f["verdict"])
    same_m = np.array_equal(c["model"], f["model"])
    same_n = np.array_equal(c["nodes"][sat], f["nodes"][sat])
    by_chain = int((sat & (c["passes"] != f["passes"])).sum())
    print(f"chain={tag} {cfg} n={n}: fast run ms median {np.median(ms):.3f} (sorted {sorted(round(x, 3) for x in ms)}) "
          f"-> {int(n) / (np.median(ms) * 1e-3) / 1e6:.2f} M q/s; identical verdicts {same_v} models {same_m} "
          f"sat nodes {same_n}; sat {int(sat.sum())}, sat with other pass counts {by_chain}", flush=True)
    ch = sat & (c["passes"] != f["passes"])
    if ch.any():
        el = f["elapsed"][ch] * 1e6
        rd = f["passes"][ch]
        print(f"  chain-decided Sat: elapsed us p50 {np.percentile(el, 50):.1f} p99 {np.percentile(el, 99):.1f} "
              f"max {el.max():.1f}; rounds p50 {np.percentile(rd, 50):.0f} max {rd.max()}; "
              f"us/round p50 {np.percentile(el / np.maximum(rd, 1), 50):.2f}; ref passes of those p50 "
              f"{np.percentile(c['passes'][ch], 50):.0f} max {c['passes'][ch].max()}")
        top = np.argsort(-c["passes"] * sat)[:8]
        print("  heaviest canonical Sat (passes, nodes, fast passes):",
              [(int(c['passes'][i]), int(c['nodes'][i]), int(f['passes'][i])) for i in top])
    if not (same_v and same_m and same_n):
        bad = np.nonzero((c["verdict"] != f["verdict"]))[0][:10]
        print("  verdict mismatches at", bad.tolist(), c["verdict"][bad].tolist(), f["verdict"][bad].tolist())
        badn = np.nonzero(sat & (c["nodes"] != f["nodes"]))[0][:10]
        print("  node mismatches at", badn.tolist(), c["nodes"][badn].tolist(), f["nodes"][badn].tolist())
