"""Config C5 proper (adversarial, Unsat by construction, input caps 2^20):
the reference times out on this family.  Decides a batch
on the GPU with the reference's 30 s timeout semantics and reports the
verdict mix and wall time, next to the CPU restatement on a few queries
(all host threads, same timeout)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402  (checker / CPU leg only)
from paper_2601_21552_b200 import synth  # noqa: E402
from paper_2601_21552_b200.solver import solve_flat  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
fb = synth.generate("c5", n, names=False)
solve_flat(fb.slice(0, 64), 30.0)  # warm
t = time.perf_counter()
out = solve_flat(fb, 30.0)
dt = time.perf_counter() - t
v = out["verdict"]
print(f"C5 {n} queries on 1 GPU: {dt:.2f} s wall; unsat {int((v == 0).sum())} sat {int((v == 1).sum())} "
      f"timeout {int((v == 2).sum())}; passes median {int(np.median(out['passes']))} max {int(out['passes'].max())}",
      flush=True)
k = 16
t = time.perf_counter()
r = oracle.solve_flat(fb.slice(0, k), 30.0, threads=k)
dt2 = time.perf_counter() - t
rv = r["verdict"]
same = int(((rv == out["verdict"][:k]) | (rv == 2)).sum())
print(f"CPU restatement, first {k} queries on {k} threads: {dt2:.1f} s; unsat {int((rv == 0).sum())} "
      f"timeout {int((rv == 2).sum())}; verdicts equal where the CPU decided: {same}/{k}", flush=True)
