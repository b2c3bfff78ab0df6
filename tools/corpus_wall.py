"""BASELINE config 2: wall time of analysing the reference's 20-program corpus.

  engine   the reference analyzer (unchanged front end, baseline/_ref) with
           every solver call decided on the GPU: analyze_many (all 110
           queries of the corpus in one device batch) in the given mode;
           "cold" = the first analysis in a fresh process (library load, CUDA
           context, device pools), "warm" = median of later ones
  python   the reference's own analyze_source over the same 20 programs
           (its pure-Python solver), same process, same box

usage: python tools/corpus_wall.py [mode] [--cold-only]  -> one JSON line
"""
from __future__ import annotations

import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    t_proc = time.perf_counter()
    mode = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "fast"
    cold_only = "--cold-only" in sys.argv
    from conftest import reference_paths
    pkg, corpus = reference_paths()
    if pkg is None:
        print(json.dumps({"unavailable": "reference not installed (tools/install_reference.sh)"}))
        return
    sys.path.insert(0, str(pkg))
    import scuba_mini.analyzer as An
    from scuba_mini.analyzer import AnalyzerConfig, analyze_source
    from scuba_mini.report import render_json_lines

    from paper_2601_21552_b200.analyzer import analyze_many

    want = json.loads((ROOT / "tests/golden/corpus_diags.json").read_text())
    progs = sorted(corpus.glob("*/*.mcu"))
    jobs = [((p.read_text(), p.name, AnalyzerConfig()), {}) for p in progs]

    def engine_once():
        t = time.perf_counter()
        res = analyze_many(An, analyze_source, jobs, mode=mode)
        dt = time.perf_counter() - t
        same = all(render_json_lines(r.diagnostics) == want[f"{p.parent.name}/{p.name}"]["m1048576"]["json"]
                   for p, r in zip(progs, res))
        return dt, same

    cold, same = engine_once()
    cold_process = time.perf_counter() - t_proc
    if cold_only:
        print(json.dumps({"cold_s": cold, "cold_process_s": cold_process, "identical": same}))
        return
    warm = []
    for _ in range(5):
        dt, s2 = engine_once()
        warm.append(dt)
        same = same and s2
    py = []
    for _ in range(3):
        t = time.perf_counter()
        for (src, name, cfg), _ in jobs:
            analyze_source(src, name, cfg)
        py.append(time.perf_counter() - t)
    print(json.dumps({
        "programs": len(progs), "queries": 110, "mode": mode, "diagnostics_identical": bool(same),
        "engine_warm_ms": round(1e3 * statistics.median(warm), 2),
        "engine_cold_ms": round(1e3 * cold, 2),
        "engine_cold_process_s": round(cold_process, 3),
        "reference_python_ms": round(1e3 * statistics.median(py), 2),
        "speedup_warm": round(statistics.median(py) / statistics.median(warm), 2),
    }))


if __name__ == "__main__":
    main()
