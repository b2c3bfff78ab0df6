"""One knob setting (env vars set by the caller): median plan-run time of a
synthetic stream.   python tools/knob_run.py <cfg> <n> <label> [heavy_nodes]"""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import _lib, synth  # noqa: E402

cfg, n, label = sys.argv[1], int(sys.argv[2]), sys.argv[3]
hn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
fb = synth.generate(cfg, n, names=False)
p = _lib.Plan(fb, 30.0, heavy_nodes=hn)
for _ in range(3):
    p.run()
ms = [p.run() for _ in range(8)]
r = p.results()
import hashlib  # noqa: E402
h = hashlib.sha1(r["verdict"].tobytes() + r["nodes"].tobytes() + r["passes"].tobytes()).hexdigest()[:10]
print(f"{cfg} {label:28s} median {statistics.median(ms):7.2f} ms  min {min(ms):7.2f}  results {h}  "
      f"{[round(x, 1) for x in ms]}", flush=True)
