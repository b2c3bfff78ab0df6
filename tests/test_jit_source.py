"""Run-time specialisation on the host (no GPU): the generated source of a
structure class compiles with NVRTC for sm_100a."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2601_21552_b200 import _lib, synth


@pytest.mark.parametrize("tmpl", [16, 28])
def test_generated_class_compiles(tmpl):
    fb = synth.generate("c3", 400, names=False)
    q = int(np.nonzero(fb.tmpl == tmpl)[0][0])
    src, ms = _lib.jit_compile(fb, q)
    assert "struct Cls" in src and "oob_jit_solve" in src
    n_cons = int(fb.con_begin[q + 1] - fb.con_begin[q])
    assert src.count("static __device__ __forceinline__ bool prop") == n_cons
    assert ms > 0
