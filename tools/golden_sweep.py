"""Golden capture for the device exhaustive oracle (run in the build container,
where the reference is mounted; its outputs travel as fixtures).

Imports the reference package from /root/reference/pkg (never copied) and
records, for each program:

  * the program lowered by `paper_2601_21552_b200.sweep.compile_program`
    (the GPU box has no reference front end to parse it);
  * the reference's `brute_force_all(program, B)` (oracle.py:638) at B = 8 and
    B = 64 (when the reference finishes it within the time cap): arity,
    executions, halted executions and violations per (line, column);
  * `replay_witness` (oracle.py:695) on seeded random input tuples at the
    program's access sites: hit, halted, halt reason;
  * for corpus programs: the reference analyzer's per-access flags and Sat
    witness inputs at max_domain = 64 and 1024 (acceptance criterion 8,
    test_acceptance.py:243-278, and the same check at a bound the Python
    sweep cannot reach).

Programs: the 20 corpus files, the reference's own test_oracle.py sources
(imported from the reference test module), seeded variants of the corpus with
their assert caps changed, and 70 seeded synthetic programs
(tools/synth_programs.py) -- sources generated here, regenerated on every run.

Usage:  python tools/golden_sweep.py      -> tests/golden/sweep_programs.json.gz,
                                             tests/golden/sweep_expect.json.gz
"""
from __future__ import annotations

import gzip
import json
import random
import re
import sys
import time
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
REF_CORPUS = Path("/root/reference/pkg/corpus")
REPO = Path(__file__).resolve().parents[1]
OUT = REPO / "tests" / "golden"
TIME_CAP = 20.0  # seconds of reference brute force per (program, bound)


def _sources() -> dict:
    sys.path.insert(0, str(REF_SRC))
    sys.path.insert(0, str(REF_TESTS))
    out = {}
    for p in sorted(REF_CORPUS.glob("*/*.mcu")):
        out["corpus/" + str(p.relative_to(REF_CORPUS))] = p.read_text()
    import test_oracle as T  # the reference's own interpreter tests
    out["test_oracle/INPUT_SRC"] = T.INPUT_SRC
    for i, (src, _inputs, reason) in enumerate(T.HALTS):
        out[f"test_oracle/HALTS_{i}_{reason.replace(' ', '_')}"] = src
    # seeded variants: every assert cap `<= k` / `< k` rescaled
    rng = random.Random(2601215524)
    for name in sorted(k for k in out if k.startswith("corpus/")):
        src = out[name]
        if not re.search(r"assert\([^)]*<=?\s*\d+\)", src):
            continue
        for v in range(2):
            def cap(m):
                k = int(m.group(2))
                return f"{m.group(1)}{max(1, k + rng.choice((-3, -1, 1, 2, 5)))})"
            out[f"variant/{name[7:]}#{v}"] = re.sub(r"(assert\([^)]*<=?\s*)(\d+)\)", cap, src)
    # seeded synthetic programs (tools/synth_programs.py, corpus-shaped templates)
    sys.path.insert(0, str(REPO / "tools"))
    from synth_programs import generate
    out.update(generate(70, 2601215526))
    return out


def _sweep_record(prog, bound):
    from scuba_mini.oracle import brute_force_all
    t0 = time.perf_counter()
    r = brute_force_all(prog, bound)
    dt = time.perf_counter() - t0
    return {"bound": bound, "arity": r.input_arity, "executions": r.executions,
            "halted": r.halted_executions,
            "violations": sorted([l, c, sorted(v)] for (l, c), v in r.violations.items()),
            "ref_s": round(dt, 3)}


def _arity(prog):
    from scuba_mini.oracle import count_input_sites
    return count_input_sites(prog)


def main():
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REF_SRC))
    from paper_2601_21552_b200.sweep import compile_program
    from scuba_mini.frontend import parse_source
    from scuba_mini.oracle import replay_witness
    from scuba_mini.analyzer import AnalyzerConfig, analyze_source
    from scuba_mini.solver import Sat

    programs, expect = {}, {}
    rng = random.Random(2601215525)
    for name, src in _sources().items():
        prog = parse_source(src, name.split("/")[-1])
        sp = compile_program(prog)
        programs[name] = {"source": src, **sp.to_json()}
        rec = {"sweeps": [], "replays": []}
        k = _arity(prog)
        for bound in (8, 64):
            if (bound + 1) ** k > 300_000:
                continue
            rec["sweeps"].append(_sweep_record(prog, bound))
        sites = sp.sites.tolist() or [[1, 1]]
        for _ in range(12):
            line, col = rng.choice(sites)
            vals = {s: rng.randrange(0, 12) for s in range(k) if rng.random() < 0.8}
            default = rng.choice((0, 1, 2, 64))
            hit, tr = replay_witness(prog, vals, default, line, col)
            rec["replays"].append({"inputs": {str(s): v for s, v in vals.items()}, "default": default,
                                   "line": line, "col": col, "hit": bool(hit),
                                   "halted": bool(tr.halted), "halt_reason": tr.halt_reason})
        if name.startswith(("corpus/", "synth/")):
            rec["analyzer"] = {}
            for m in (64, 1024):
                res = analyze_source(src, name.split("/")[-1], AnalyzerConfig(max_domain=m))
                acc = []
                for acr in res.access_results:
                    loc = acr.access.location
                    wits = [{str(s): v for s, v in o.witness_inputs.items()}
                            for o in acr.outcomes
                            if isinstance(o.verdict, Sat) and o.witness_inputs is not None]
                    # the reference's own replay of each witness (default = the bound,
                    # as criterion 8 does): a witness that leaves a data-dependent
                    # input site unpinned may halt on the default
                    reps = [bool(replay_witness(prog, {int(s): v for s, v in w.items()}, m,
                                                loc.line, loc.column)[0]) for w in wits]
                    acc.append({"line": loc.line, "col": loc.column, "flagged": bool(acr.flagged),
                                "witnesses": wits, "witness_replays": reps})
                rec["analyzer"][str(m)] = acc
        expect[name] = rec
        print(name, k, [(s["bound"], s["executions"], s["ref_s"]) for s in rec["sweeps"]], flush=True)
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / "sweep_programs.json.gz").write_bytes(
        gzip.compress(json.dumps(programs, indent=0, sort_keys=True).encode(), 9, mtime=0))
    (OUT / "sweep_expect.json.gz").write_bytes(
        gzip.compress(json.dumps(expect, indent=0, sort_keys=True).encode(), 9, mtime=0))


if __name__ == "__main__":
    main()
