import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import time
from paper_2601_21552_b200 import synth
from paper_2601_21552_b200.solver import solve_flat
fb = synth.generate(sys.argv[1], 100000, names=False)
for _ in range(int(sys.argv[2])):
    t = time.perf_counter(); solve_flat(fb, 30.0); print(round(1e3 * (time.perf_counter() - t), 1), flush=True)
