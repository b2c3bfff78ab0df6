"""Host pipeline loop for the sampling profile (tools/host_profile.sh):
oob_host_bench (compile + schedule + pack, no device) over two batches."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
fbs = [synth.generate(cfg, 100000, first=(i + 1) * 100000, names=False) for i in range(2)]
for i in range(iters):
    _lib.host_bench(fbs[i % 2], flags=_lib.F_FAST)
