"""GPU parity of the run-time compiled class kernels (jit.cpp, jit_lane.cuh).

Every structure class is forced through NVRTC (jit_min=1) and the results
must equal the golden capture of the Python reference bit for bit: verdicts,
first models, DFS node counts and propagation pass counts -- the compiled
kernels perform the reference's own traversal, exactly like the interpreter.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import VCODE, load_golden

from paper_2601_21552_b200 import _lib
from paper_2601_21552_b200.solver import solve_flat
from paper_2601_21552_b200.wire import flatten, words_to_ints

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("heavy", [0, -1])
@pytest.mark.parametrize("name", ["synth_c3", "synth_c4", "synth_c5s", "corpus_m1048576", "random_solver"])
def test_jit_golden_exact(gpu, name, heavy):
    recs = [r for r in load_golden(name) if r["verdict"] != "timeout" and r["timeout"] >= 1.0]
    fb = flatten(recs)
    out = solve_flat(fb, 30.0, heavy_nodes=heavy, jit_min=1)
    for q, r in enumerate(recs):
        assert int(out["verdict"][q]) == VCODE[r["verdict"]], (name, q)
        assert int(out["nodes"][q]) == r["nodes"], (name, q, "nodes")
        assert int(out["passes"][q]) == r["passes"], (name, q, "passes")
        if r["verdict"] == "sat":
            vb, ve = int(fb.var_begin[q]), int(fb.var_begin[q + 1])
            model = dict(zip(fb.names(q), words_to_ints(out["model"][vb:ve])))
            assert model == r["model"], (name, q)


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_jit_matches_interpreter_on_streams(gpu, cfg):
    from paper_2601_21552_b200 import synth
    fb = synth.generate(cfg, 20000, names=False)
    a = solve_flat(fb, 30.0, flags=_lib.F_NO_JIT)
    b = solve_flat(fb, 30.0, jit_min=64)
    for k in ("verdict", "nodes", "passes", "model"):
        assert np.array_equal(a[k], b[k]), k


def test_jit_plan_runs_match(gpu):
    from paper_2601_21552_b200 import synth
    fb = synth.generate("c3", 5000, names=False)
    p = _lib.Plan(fb, 30.0, jit_min=64)
    for _ in range(2):
        p.run()
    r = p.results()
    ref = solve_flat(fb, 30.0, flags=_lib.F_NO_JIT)
    for k in ("verdict", "nodes", "passes"):
        assert np.array_equal(r[k], ref[k]), k


def test_chunked_pipeline_matches_single_call(gpu, monkeypatch):
    """SCUBA_OOB_CHUNK cuts a large call into concurrently decided chunks;
    results must be identical (queries are independent).  The knob is read
    once per process, so the chunked run happens in a subprocess."""
    import json
    import subprocess
    import sys
    from conftest import ROOT
    code = (
        "import sys, json; sys.path.insert(0, %r)\n"
        "from paper_2601_21552_b200 import synth\n"
        "from paper_2601_21552_b200.solver import solve_flat\n"
        "fb = synth.generate('c3', 30000, names=False)\n"
        "o = solve_flat(fb, 30.0)\n"
        "print(json.dumps([o['verdict'].tolist(), o['nodes'].tolist(), o['passes'].tolist()]))\n" % str(ROOT))
    env = dict(__import__("os").environ, SCUBA_OOB_CHUNK="8000")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True)
    v, nodes, passes = json.loads(out.stdout.strip().splitlines()[-1])
    from paper_2601_21552_b200 import synth
    fb = synth.generate("c3", 30000, names=False)
    ref = solve_flat(fb, 30.0)
    assert v == ref["verdict"].tolist()
    assert nodes == ref["nodes"].tolist()
    assert passes == ref["passes"].tolist()
