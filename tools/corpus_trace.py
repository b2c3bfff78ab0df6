"""Host-phase trace of the corpus batch (config C2: 110 queries), the
latency case of the metric ("corpus wall time")."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_21552_b200.solver import solve_flat  # noqa: E402
from paper_2601_21552_b200.wire import flatten  # noqa: E402

recs = [json.loads(l) for l in open(ROOT / "tests/golden/corpus_m1048576.jsonl")]
fb = flatten(recs)
for i in range(6):
    t = time.perf_counter()
    out = solve_flat(fb, 30.0, n_gpus=1, device=0)
    print(f"corpus solve_flat {1e3 * (time.perf_counter() - t):.3f} ms", file=sys.stderr, flush=True)
