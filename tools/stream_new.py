"""Stream API throughput on NEW batches every repetition (what bench.py's e2e
sees: certificate-cache misses, fresh records), after a warm-up on other
batches.  usage: python tools/stream_new.py [cfg] [n] [k] [reps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 5
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
gen = lambda r, i: synth.generate(cfg, n, first=(r * 16 + i + 1) * n, names=False)  # noqa: E731
for w in range(2):  # (the first call also compiles the classes: the other slots then run without them)
    _lib.solve_flat_stream([gen(98 + w, i) for i in range(3)], 30.0, n_gpus=1, flags=_lib.F_FAST)
print("=== warm done", file=sys.stderr, flush=True)
for r in range(reps):
    fbs = [gen(r, i) for i in range(k)]
    t = time.perf_counter()
    _lib.solve_flat_stream(fbs, 30.0, n_gpus=1, flags=_lib.F_FAST)
    dt = time.perf_counter() - t
    print(f"{cfg} new batches {k} x {n}: stream {1e3 * dt / k:.1f} ms/batch ({k * n / dt / 1e6:.2f} M q/s)", flush=True)
    print(f"=== rep {r} done", file=sys.stderr, flush=True)
