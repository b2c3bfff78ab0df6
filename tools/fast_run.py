"""One fast-mode plan, a few runs (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
flags = _lib.F_FAST if (len(sys.argv) <= 4 or sys.argv[4] == "fast") else 0
fb = synth.generate(cfg, n, names=False)
p = _lib.Plan(fb, 30.0, flags=flags)
for _ in range(runs):
    print(f"{p.run():.3f} ms", flush=True)
