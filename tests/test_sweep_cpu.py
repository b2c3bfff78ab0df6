"""Device exhaustive oracle, CPU side (no GPU): the bytecode compiler and the
interpreter semantics of csrc/sweep_vm.cuh, built for the host by the test
harness tests/native/sweep_host.cpp, against the REFERENCE's own
brute_force_all / replay_witness outputs (tests/golden/sweep_*.json, captured
by tools/golden_sweep.py from /root/reference; oracle.py:638-720).

The GPU run of the same fixtures is tests/test_gpu_sweep.py."""
from __future__ import annotations

import ctypes
import gzip
import json
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REF_SRC, ROOT, reference_available

from paper_2601_21552_b200 import sweep as S

HARNESS_SRC = ROOT / "tests" / "native" / "sweep_host.cpp"
HARNESS = ROOT / "tests" / "native" / "_build" / "libsweep_host.so"


class HostBackend:
    """The host harness behind the same two C-ABI entry points."""

    def __init__(self):
        deps = [HARNESS_SRC, ROOT / "paper_2601_21552_b200" / "csrc" / "sweep_vm.cuh"]
        if not HARNESS.exists() or HARNESS.stat().st_mtime < max(d.stat().st_mtime for d in deps):
            HARNESS.parent.mkdir(parents=True, exist_ok=True)
            subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o",
                                   str(HARNESS), str(HARNESS_SRC)])
        L = ctypes.CDLL(str(HARNESS))
        vp = ctypes.c_void_p
        L.sweep_host_run.argtypes = [vp, ctypes.c_int64, ctypes.c_int32, vp, vp]
        L.sweep_host_replay.argtypes = [vp, ctypes.c_int64, ctypes.c_int32, vp, vp, vp, vp, vp]
        self.oob_sweep_run = L.sweep_host_run
        self.oob_sweep_replay = L.sweep_host_replay


@pytest.fixture(scope="module")
def host():
    return HostBackend()


def load():
    progs = json.loads(gzip.decompress((GOLDEN / "sweep_programs.json.gz").read_bytes()))
    expect = json.loads(gzip.decompress((GOLDEN / "sweep_expect.json.gz").read_bytes()))
    return {k: S.SweepProgram.from_json(v) for k, v in progs.items()}, expect


PROGS, EXPECT = load()


def as_reference(r: S.SweepResult) -> dict:
    return {"arity": r.input_arity, "executions": r.executions, "halted": r.halted_executions,
            "violations": sorted([l, c, sorted(v)] for (l, c), v in r.violations.items())}


def test_opcode_tables_match_the_interpreter():
    hdr = (ROOT / "paper_2601_21552_b200" / "csrc" / "sweep_vm.cuh").read_text()
    body = hdr[hdr.index("enum Op {") + 9: hdr.index("};", hdr.index("enum Op {"))]
    names = [t.strip() for t in body.replace("\n", " ").split(",") if t.strip()]
    assert tuple(names) == S.OPS
    assert S.MAX_SLOTS == 96 and S.MAX_SITES == 64


@pytest.mark.parametrize("name", sorted(PROGS))
def test_sweep_matches_reference_brute_force(host, name):
    for want in EXPECT[name]["sweeps"]:
        got = S.brute_force_all(PROGS[name], want["bound"], backend=host)
        assert as_reference(got) == {k: want[k] for k in ("arity", "executions", "halted", "violations")}


@pytest.mark.parametrize("name", sorted(PROGS))
def test_replay_matches_reference_replay_witness(host, name):
    reqs = [({int(s): v for s, v in r["inputs"].items()}, r["line"], r["col"])
            for r in EXPECT[name]["replays"]]
    defaults = {r["default"] for r in EXPECT[name]["replays"]}
    for d in defaults:
        idx = [i for i, r in enumerate(EXPECT[name]["replays"]) if r["default"] == d]
        out = S.replay_witnesses(PROGS[name], [reqs[i] for i in idx], d, backend=host)
        for i, (hit, tr) in zip(idx, out):
            want = EXPECT[name]["replays"][i]
            assert (hit, tr.halted, tr.halt_reason) == (want["hit"], want["halted"], want["halt_reason"]), (i, want)


@pytest.mark.parametrize("name", sorted(k for k in PROGS if k.startswith(("corpus/", "synth/"))))
def test_criterion_8_on_the_sweep_interpreter(host, name):
    """acceptance criterion 8 (test_acceptance.py:243-278): the analyzer's
    per-access flags at max_domain 64 equal the exhaustive sweep at bound 64,
    and every Sat witness replays."""
    sp = PROGS[name]
    sweep = S.brute_force_all(sp, 64, backend=host)
    oob = {"oob-upper", "oob-underflow"}
    for acc in EXPECT[name]["analyzer"]["64"]:
        site = (acc["line"], acc["col"])
        assert acc["flagged"] == bool(sweep.violations.get(site, set()) & oob), site
        for w, ref_hit in zip(acc["witnesses"], acc["witness_replays"]):
            hit, _ = S.replay_witness(sp, {int(s): v for s, v in w.items()}, 64, *site, backend=host)
            assert hit == ref_hit, (site, w)
            if name.startswith("corpus/"):
                assert hit, (site, w)  # criterion 8: every corpus witness replays


def test_stop_when_violated_and_verdict(host):
    sp = PROGS["test_oracle/INPUT_SRC"]
    assert S.brute_force_verdict(sp, 2, 5, 8, backend=host)
    assert not S.brute_force_verdict(sp, 2, 5, 2, backend=host)
    r = S.brute_force_all(sp, 8, stop_when_violated={(2, 5)}, backend=host)
    assert r.executions == 4 and r.violations == {(2, 5): {"oob-upper"}}  # n = 3 is tuple 3


def test_first_witness_is_the_first_violating_tuple(host):
    sp = PROGS["test_oracle/INPUT_SRC"]
    r = S.brute_force_all(sp, 8, backend=host)
    assert r.first_witness == {(2, 5): (3,)}


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
@pytest.mark.parametrize("name", sorted(PROGS))
def test_compiler_is_deterministic_on_reference_ast(name):
    sys.path.insert(0, str(REF_SRC))
    from scuba_mini.frontend import parse_source
    src = json.loads(gzip.decompress((GOLDEN / "sweep_programs.json.gz").read_bytes()))[name]["source"]
    sp = S.compile_program(parse_source(src, name.split("/")[-1]))
    assert np.array_equal(sp.code, PROGS[name].code)
    assert np.array_equal(sp.sites, PROGS[name].sites)


def test_device_entry_validates_programs_before_touching_a_device():
    """oob_sweep_run checks operands and the value-stack discipline on the
    host first: every fixture program passes (the call then needs a device),
    a program with an unbalanced stack or a bad jump is rejected."""
    from paper_2601_21552_b200 import _lib
    L = _lib.lib()
    no_device = _lib.device_count() == 0

    def rc_of(sp):
        cp, keep = S._cprog(sp)
        ns = max(len(sp.sites), 1)
        lab = np.zeros(ns, dtype=np.uint32)
        first = np.full((ns, 4), -1, dtype=np.int64)
        res = S._CResult()
        res.site_labels, res.site_first_tuple = lab.ctypes.data, first.ctypes.data
        opts = S._copts()
        return L.oob_sweep_run(ctypes.byref(cp), 2, sp.n_input_sites, ctypes.byref(opts), ctypes.byref(res))

    for name, sp in PROGS.items():
        rc = rc_of(sp)
        assert rc != 1, (name, _lib.last_error())  # OOB_E_INVALID
        if no_device:
            assert rc == 2  # OOB_E_CUDA: validation passed, no device here
    sp = PROGS["test_oracle/INPUT_SRC"]
    bad = S.SweepProgram(sp.code.copy(), sp.lits, sp.kernels, sp.kparams, sp.sites, sp.n_slots,
                         sp.n_input_sites)
    bad.code[0] = [S.OP["ST"], 0, 0, 0]  # pops an empty stack
    assert rc_of(bad) == 1 and "stack" in _lib.last_error()
    bad2 = S.SweepProgram(sp.code.copy(), sp.lits, sp.kernels, sp.kparams, sp.sites, sp.n_slots,
                          sp.n_input_sites)
    bad2.code[1] = [S.OP["JMP"], 10 ** 6, 0, 0]
    assert rc_of(bad2) == 1
