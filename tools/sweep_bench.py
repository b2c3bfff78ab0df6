"""Throughput of the device exhaustive oracle (csrc/sweep.cu) on the corpus.

For each corpus program and bound B: executions ((B+1)^k tuples), device time
of the sweep kernel (CUDA events), tuples/s, and the reference's Python
brute_force_all time at B = 64 from the golden capture (tools/golden_sweep.py,
build container).  One JSON line per (program, B), then a summary line.

    python tools/sweep_bench.py [B ...]        (default: 64 256 1024)
"""
from __future__ import annotations

import gzip
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_2601_21552_b200 import sweep as S  # noqa: E402


def main():
    bounds = [int(x) for x in sys.argv[1:]] or [64, 256, 1024]
    progs = S.load_programs(ROOT / "tests" / "golden" / "sweep_programs.json.gz")
    expect = json.loads(gzip.decompress((ROOT / "tests" / "golden" / "sweep_expect.json.gz").read_bytes()))
    tot = {b: [0, 0.0, 0.0] for b in bounds}
    for name in sorted(k for k in progs if k.startswith("corpus/")):
        sp = progs[name]
        ref64 = next((s for s in expect[name]["sweeps"] if s["bound"] == 64), None)
        for b in bounds:
            S.sweep_once(sp, b, sp.n_input_sites)  # warm (context, module)
            t0 = time.perf_counter()
            r = S.sweep_once(sp, b, sp.n_input_sites)
            wall = time.perf_counter() - t0
            line = {"program": name, "bound": b, "arity": sp.n_input_sites,
                    "executions": r["executions"], "halted": r["halted"],
                    "device_ms": round(r["device_ms"], 3), "wall_ms": round(1e3 * wall, 3),
                    "tuples_per_s": round(r["executions"] / max(r["device_ms"], 1e-3) * 1e3, 1),
                    "reference_python_s_at_64": ref64["ref_s"] if (ref64 and b == 64) else None}
            tot[b][0] += r["executions"]
            tot[b][1] += r["device_ms"]
            tot[b][2] += wall
            print(json.dumps(line), flush=True)
    ref_total = sum(s["ref_s"] for n, e in expect.items() if n.startswith("corpus/")
                    for s in e["sweeps"] if s["bound"] == 64)
    for b, (n, ms, wall) in tot.items():
        print(json.dumps({"summary": True, "bound": b, "executions": n, "device_ms": round(ms, 3),
                          "wall_ms": round(1e3 * wall, 3),
                          "reference_python_s": round(ref_total, 3) if b == 64 else None}))


if __name__ == "__main__":
    main()
