"""Build the in-tree CUDA engine (libscuba_oob.so, sm_100a only).

    python -m paper_2601_21552_b200.build

nvcc cross-compiles without a GPU; the .so is written next to this file so it
travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "libscuba_oob.so"


def build(verbose: bool = False) -> Path:
    cmd = ["make", "-C", str(CSRC)]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.check_call(cmd, stdout=None if verbose else subprocess.DEVNULL)
    if not LIB.exists():
        raise RuntimeError(f"build did not produce {LIB}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
