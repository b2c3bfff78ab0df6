import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import synth
from paper_2601_21552_b200.solver import solve_flat
for cfg in sys.argv[1:]:
    fb = synth.generate(cfg, 100000, names=False)
    print("==", cfg, flush=True)
    solve_flat(fb, 30.0)
