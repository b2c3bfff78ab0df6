"""Host phases of oob_solve_batch (SCUBA_OOB_TRACE=1) for one config/mode."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402
from paper_2601_21552_b200.solver import solve_flat  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
flags = _lib.F_FAST if (len(sys.argv) <= 3 or sys.argv[3] == "fast") else 0
fb = synth.generate(cfg, n, names=False)
os.environ.setdefault("SCUBA_OOB_TRACE", "1")  # read once, at the first call
for i in range(4):
    t = time.perf_counter()
    solve_flat(fb, 30.0, n_gpus=1, flags=flags)
    print(f"call {i}: {1e3 * (time.perf_counter() - t):.1f} ms", file=sys.stderr, flush=True)
