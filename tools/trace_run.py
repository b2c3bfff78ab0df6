"""Host-phase trace + kernel timing variants of one synthetic stream (GPU box).

    SCUBA_OOB_TRACE=1 python tools/trace_run.py [config] [n]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402
from paper_2601_21552_b200.solver import solve_flat  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
t = time.perf_counter()
fb = synth.generate(cfg, n, names=False)
print(f"generate {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
for i in range(3):
    t = time.perf_counter()
    solve_flat(fb, 30.0)
    print(f"solve_flat #{i}: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
for heavy in (0, -1, 16, 128):
    for flags in (0, _lib.F_NO_DEMOTE):
        plan = _lib.Plan(fb, 30.0, n_gpus=1, device=0, heavy_nodes=heavy, flags=flags)
        ms = [plan.run() for _ in range(3)]
        print(f"plan heavy={heavy} flags={flags}: info={plan.info()} ms={[round(x, 2) for x in ms]}", flush=True)
        del plan
