import sys, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth
cfg = sys.argv[1]; jm = int(sys.argv[2])
fb = synth.generate(cfg, 100000, names=False)
kw = dict(flags=_lib.F_NO_JIT) if jm < 0 else dict(jit_min=jm)
p = _lib.Plan(fb, 30.0, **kw)
for i in range(6):
    if i == 1 and os.environ.get("TL1"): os.environ["SCUBA_OOB_TIMELINE"] = ""
    print(i, round(p.run(), 2), flush=True)
