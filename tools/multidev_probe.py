import os, sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import GOLDEN_SETS, load_golden
from paper_2601_21552_b200 import _lib, synth
from paper_2601_21552_b200.solver import solve_flat
from paper_2601_21552_b200.wire import flatten
recs = [r for n in GOLDEN_SETS for r in load_golden(n) if r["verdict"] != "timeout" and r["timeout"] == 30.0]
batches = {"golden": flatten(recs), "c3": synth.generate("c3", 6000, first=40000, names=False), "c4": synth.generate("c4", 6000, first=40000, names=False)}
for name, fb in batches.items():
    for k in (1, 2, 3, 4, 8):
        os.environ["SCUBA_OOB_VIRTUAL_DEVICES"] = str(k)
        try:
            solve_flat(fb, 30.0, n_gpus=k, flags=_lib.F_FAST)
            print(name, k, "ok", flush=True)
        except Exception as e:
            print(name, k, "FAIL", e, flush=True)
        _lib.lib().oob_release()
