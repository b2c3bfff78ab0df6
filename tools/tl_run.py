"""Device timeline of the LAST of a few plan runs (SCUBA_OOB_TIMELINE must be set)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth
cfg = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "canonical"
fb = synth.generate(cfg, 100000, names=False)
p = _lib.Plan(fb, 30.0, flags=_lib.F_FAST if mode == "fast" else 0)
print([round(p.run(), 2) for _ in range(3)], flush=True)
p.results()
