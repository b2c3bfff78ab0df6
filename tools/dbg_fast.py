import sys, os; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_2601_21552_b200 import _lib, synth
from paper_2601_21552_b200.solver import solve_flat
mode = sys.argv[1]; n = int(sys.argv[2])
fb = synth.generate("c3", n, names=False)
flags = _lib.F_FAST if mode == "fast" else 0
hn = int(sys.argv[3]) if len(sys.argv) > 3 else 0
for i in range(3):
    out = solve_flat(fb, 30.0, flags=flags, heavy_nodes=hn)
    print(mode, i, np.bincount(out["verdict"].astype(np.int64)), flush=True)
