import sys, time, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import synth
from paper_2601_21552_b200.solver import solve_flat
cfg = sys.argv[1]
fb = synth.generate(cfg, 100000, names=False)
solve_flat(fb, 30.0)
ts = []
for _ in range(5):
    t = time.perf_counter(); solve_flat(fb, 30.0); ts.append(1e3 * (time.perf_counter() - t))
print(cfg, "chunk", os.environ.get("SCUBA_OOB_CHUNK", "default"), "e2e ms", [round(x, 1) for x in ts], flush=True)
