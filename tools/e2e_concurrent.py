"""End-to-end throughput of oob_solve_batch with 1..T host threads submitting
consecutive batches concurrently (the library is reentrant; one batch's host
compile/pack overlaps another's kernels).

    python tools/e2e_concurrent.py [cfg] [n] [steps]
"""
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import synth  # noqa: E402
from paper_2601_21552_b200.solver import solve_flat  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
fbs = [synth.generate(cfg, n, first=i * n, names=False) for i in range(2)]
for fb in fbs:
    solve_flat(fb, 30.0, n_gpus=1, device=0)
ref = [solve_flat(fb, 30.0, n_gpus=1, device=0) for fb in fbs]
for T in (1, 2, 3):
    outs = {}

    def worker(k):
        for s in range(k, steps, T):
            outs[s] = solve_flat(fbs[s % 2], 30.0, n_gpus=1, device=0)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(T)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    dt = time.perf_counter() - t0
    same = all((outs[s]["verdict"] == ref[s % 2]["verdict"]).all() and
               (outs[s]["nodes"] == ref[s % 2]["nodes"]).all() for s in range(steps))
    print(f"{cfg} threads={T}: {steps} batches of {n} in {dt * 1e3:.1f} ms -> {steps * n / dt:,.0f} q/s; identical={same}",
          flush=True)
