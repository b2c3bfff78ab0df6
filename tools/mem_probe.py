import sys, subprocess
sys.path.insert(0, '.')
from paper_2601_21552_b200 import _lib, synth
from paper_2601_21552_b200.solver import solve_flat
def used():
    out = subprocess.run(["nvidia-smi", "--query-gpu=memory.used", "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout
    return int(out.strip().split()[0])
for cfg in ("c3", "c4"):
    fb = synth.generate(cfg, 100000, names=False)
    p = _lib.Plan(fb, 30.0); p.run()
    print(cfg, "plan MiB used", used(), flush=True)
    solve_flat(fb, 30.0)
    print(cfg, "after solve_flat MiB used", used(), flush=True)
    p.close()
