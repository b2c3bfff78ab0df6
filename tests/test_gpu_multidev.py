"""The in-call multi-device path on one B200: SCUBA_OOB_VIRTUAL_DEVICES=k
deals a batch over k logical devices (k host threads, k sets of device pools
on the visible GPU) exactly as oob_solve_batch does over k real GPUs; results
must not depend on k (SPEC.md:423 -- calls share nothing; determinism is per
query).  Canonical mode: verdicts, models and node/pass counters; fast mode:
verdicts and models."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN_SETS, load_golden

from paper_2601_21552_b200 import _lib, synth
from paper_2601_21552_b200.solver import solve_flat
from paper_2601_21552_b200.wire import flatten

pytestmark = pytest.mark.gpu


@pytest.fixture
def virtual(monkeypatch):
    def set_k(k):
        monkeypatch.setenv("SCUBA_OOB_VIRTUAL_DEVICES", str(k))
    yield set_k
    _lib.lib().oob_release()


@pytest.mark.parametrize("flags", [0, _lib.F_FAST])
def test_logical_devices_identical(gpu, virtual, flags):
    recs = [r for n in GOLDEN_SETS for r in load_golden(n) if r["verdict"] != "timeout" and r["timeout"] == 30.0]
    batches = [flatten(recs), synth.generate("c3", 6000, first=40000, names=False),
               synth.generate("c4", 6000, first=40000, names=False)]
    for fb in batches:
        base = None
        for k in (1, 2, 3, 4, 8):
            virtual(k)
            out = solve_flat(fb, 30.0, n_gpus=k, flags=flags)
            _lib.lib().oob_release()
            if base is None:
                base = out
                continue
            keys = ("verdict", "model") if flags else ("verdict", "model", "nodes", "passes")
            for key in keys:
                assert np.array_equal(base[key], out[key]), (k, key)
