import os, sys
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2601_21552_b200 import _lib, synth
cfg = sys.argv[1]
fb = synth.generate(cfg, 100000, names=False)
p = _lib.Plan(fb, 30.0)
buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda:0")
for i in range(3): p.run()
print(cfg, "no flush", [round(p.run(), 1) for _ in range(4)], flush=True)
r = []
for _ in range(4):
    buf.fill_(1.0); torch.cuda.synchronize(); r.append(round(p.run(), 1))
print(cfg, "flush", r, flush=True)
r = []
for _ in range(4):
    torch.cuda.synchronize(); r.append(round(p.run(), 1))
print(cfg, "sync only", r, flush=True)
