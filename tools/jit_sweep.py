import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth
cfg = sys.argv[1]; n = int(sys.argv[2]); jm = int(sys.argv[3]) if len(sys.argv) > 3 else 0
fb = synth.generate(cfg, n, names=False)
kw = dict(flags=_lib.F_NO_JIT) if jm < 0 else dict(jit_min=jm)
p = _lib.Plan(fb, 30.0, **kw)
ms = [p.run() for _ in range(4)]
print(cfg, n, "jit_min", jm, "ms", [round(x, 2) for x in ms], flush=True)
