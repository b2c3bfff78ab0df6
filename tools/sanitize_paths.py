"""Small batches through every engine path, for compute-sanitizer runs:
canonical (interpreter + run-time compiled classes + frontier + regime
demotion + x32), canonical without demotion, every query through the
frontier, fast mode (certificate kernel), the opt-in warp-per-query search
(OOB_F_CHAIN), and the propagate/check_model aux
kernel.  Verdicts are checked against the C oracle on the way."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("SCUBA_OOB_JIT_MIN", "64")  # small classes compile too
from oracle import oracle  # noqa: E402
from paper_2601_21552_b200 import _lib, synth  # noqa: E402
from paper_2601_21552_b200.solver import solve_flat  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
runs = [("c3", 0, 0), ("c4", 0, 0), ("c4", _lib.F_NO_DEMOTE, 0), ("c3", 0, 1), ("c3", _lib.F_FAST, 0),
        ("c4", _lib.F_FAST, 0), ("c5", _lib.F_FAST, 0), ("c3", _lib.F_FAST | _lib.F_CHAIN, 0),
        ("c4", _lib.F_FAST | _lib.F_CHAIN, 0)]
for cfg, flags, heavy in runs:
    fb = synth.generate(cfg, n if cfg != "c5" else min(n, 200), first=1000, names=False)
    out = solve_flat(fb, 30.0 if cfg != "c5" else 2.0, n_gpus=1, flags=flags, heavy_nodes=heavy)
    assert out["status"] == _lib.OOB_OK, out["error"]
    if cfg != "c5":
        ref = oracle.solve_flat(fb, 30.0, threads=oracle.cpu_count())
        assert np.array_equal(out["verdict"], ref["verdict"]), (cfg, flags, heavy)
    print(cfg, "flags", flags, "heavy", heavy, "verdicts", np.bincount(out["verdict"].astype(np.int64)), flush=True)
lo, hi, st = _lib.propagate_flat(synth.generate("c3", 200, names=False))
print("propagate ok", int(st.sum()), flush=True)
