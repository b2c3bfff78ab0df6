"""Cold start of the engine in a fresh process: library load, first call on
the 110 corpus queries (CUDA context, device pools), then a warm call."""
import json
import os
import sys
import time
from pathlib import Path

t0 = time.perf_counter()
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("SCUBA_OOB_TRACE", "1")
from paper_2601_21552_b200 import _lib  # noqa: E402
from paper_2601_21552_b200.solver import solve_flat  # noqa: E402
from paper_2601_21552_b200.wire import flatten  # noqa: E402

root = Path(__file__).resolve().parents[1]
recs = [json.loads(l) for l in open(root / "tests/golden/corpus_m1048576.jsonl")]
fb = flatten(recs)
t1 = time.perf_counter()
_lib.lib()
t2 = time.perf_counter()
n = _lib.device_count()
t3 = time.perf_counter()
mode = sys.argv[1] if len(sys.argv) > 1 else "fast"
flags = _lib.F_FAST if mode == "fast" else 0
solve_flat(fb, 30.0, n_gpus=1, flags=flags)
t4 = time.perf_counter()
solve_flat(fb, 30.0, n_gpus=1, flags=flags)
t5 = time.perf_counter()
print(json.dumps({"imports_s": round(t1 - t0, 3), "lib_load_s": round(t2 - t1, 3), "device_count_s": round(t3 - t2, 3),
                  "first_call_s": round(t4 - t3, 3), "warm_call_s": round(t5 - t4, 4)}), file=sys.stderr)
