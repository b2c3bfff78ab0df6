"""Phase timeline of the stream API (SCUBA_OOB_TRACE=3: each phase's start
time and pool slot) over K different batches, after a warm-up call."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["SCUBA_OOB_TRACE"] = os.environ.get("SCUBA_OOB_TRACE", "3")
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 5
fbs = [synth.generate(cfg, n, first=(i + 1) * n, names=False) for i in range(k)]
_lib.solve_flat_stream([synth.generate(cfg, n, first=(k + 1) * n + 10**8, names=False) for k in range(3)], 30.0, n_gpus=1, flags=_lib.F_FAST)
_lib.solve_flat_stream(fbs, 30.0, n_gpus=1, flags=_lib.F_FAST)
print("=== timed stream", file=sys.stderr, flush=True)
t = time.perf_counter()
_lib.solve_flat_stream(fbs, 30.0, n_gpus=1, flags=_lib.F_FAST)
dt = time.perf_counter() - t
print(f"=== stream {1e3 * dt / k:.1f} ms/batch", file=sys.stderr, flush=True)
