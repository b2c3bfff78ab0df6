"""Stream API vs single calls on K different batches of a stream."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402
from paper_2601_21552_b200._lib import solve_flat_stream  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 6
fbs = [synth.generate(cfg, n, first=(i + 1) * n, names=False) for i in range(k)]
solve_flat_stream([synth.generate(cfg, n, first=(k + 1) * n + 10**8, names=False) for k in range(3)], 30.0, n_gpus=1, flags=_lib.F_FAST)
for rep in range(3):
    t = time.perf_counter()
    solve_flat_stream(fbs, 30.0, n_gpus=1, flags=_lib.F_FAST)
    dt = time.perf_counter() - t
    t = time.perf_counter()
    for fb in fbs:
        _lib.solve_flat(fb, 30.0, n_gpus=1, flags=_lib.F_FAST)
    ds = time.perf_counter() - t
    print(f"{cfg} {k} x {n}: stream {1e3 * dt / k:.1f} ms/batch ({k * n / dt / 1e6:.2f} M q/s); "
          f"single calls {1e3 * ds / k:.1f} ms/batch ({k * n / ds / 1e6:.2f} M q/s)", flush=True)
