import sys, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth
cfg = sys.argv[1]
fb = synth.generate(cfg, 100000, names=False)
for hn in [int(x) for x in sys.argv[2].split(",")]:
    p = _lib.Plan(fb, 30.0, heavy_nodes=hn)
    ms = [p.run() for _ in range(4)]
    print(cfg, "heavy_nodes", hn, "HP", os.environ.get("SCUBA_OOB_HEAVY_PASSES", "256"),
          "maxreg", os.environ.get("SCUBA_OOB_JIT_MAXREG", "-"), [round(x, 2) for x in ms[1:]], flush=True)
    del p
