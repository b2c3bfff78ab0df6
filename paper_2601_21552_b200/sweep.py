"""Exhaustive program-level oracle on the GPU: brute-force sweeps and witness
replay of MiniCUDA programs.

Reference: /root/reference/pkg/src/scuba_mini/oracle.py -- the AST
interpreter (`_Compiler`, oracle.py:260-580), `brute_force_all`
(oracle.py:638-681), `brute_force_verdict` (oracle.py:684-692) and
`replay_witness` (oracle.py:695-720).  The reference front end parses the
program (unchanged); this module lowers its AST to a flat stack bytecode
(`compile_program`) and hands it to the sm_100a interpreter in
`csrc/sweep.cu` through the C ABI of `include/scuba_oob_sweep.h`: one GPU
thread executes the whole program -- host code, every launched block and
thread in the reference's sequential order -- for one input tuple, so a sweep
over (B+1)^k tuples is one data-parallel launch.

Semantics reproduced (oracle.py:9-24): threads run sequentially (blocks z,y,x
with x fastest, then threads alike); cells start at 0, out-of-bounds reads
yield 0, writes outside the backing storage are discarded; partitions end the
previously created partition of the same storage in the same thread; an
execution halts (its events disregarded) on a failed assert, division by
zero, or a negative allocation size / launch dimension / dynamic shared size
/ scalar argument / stored value.  Integers are int64 on the device; a tuple
whose values leave int64 is reported as an error (never a wrong answer).
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

# ---- bytecode (must match csrc/sweep_vm.cuh) ---------------------------------------
OPS = ("LIT", "LD", "INP", "BLT", "BIN", "RD", "CMP", "ST", "JZ", "JMP", "ASRT",
       "MALLOC", "FREE", "WR", "ATOM", "RET", "XSHM", "ADECL", "PART", "NNEG", "PARG",
       "LAUNCH", "KEND", "END")
OP = {name: i for i, name in enumerate(OPS)}
BINOPS = ("+", "-", "*", "/", "%")
RELS = ("<", "<=", ">", ">=", "==")
ATOMICS = ("atomicAdd", "atomicMin", "atomicMax")
BUILTIN_GROUPS = ("threadIdx", "blockIdx", "blockDim", "gridDim")
AXES = ("x", "y", "z")

# violation labels (oracle.py:44-47) <-> bits
LABELS = ("oob-upper", "oob-underflow", "uaf", "double-free")
# halt reasons (oracle.py:218-539) <-> codes
HALT_REASONS = (None, "negative allocation size", "assert failed", "division by zero",
                "negative stored value", "negative launch dimension",
                "negative dynamic shared size", "negative scalar argument")
H_ALLOC, H_ASSERT, H_DIV0, H_STORE, H_DIM, H_SHM, H_ARG = range(1, 8)
MAX_INPUT_SITES = 5  # oracle.py:41
MAX_SLOTS = 96
MAX_SITES = 64
MAX_KPARAMS = 16

ST_OK, ST_HALT, ST_NEED, ST_ERROR = range(4)
ERRORS = ("none", "integer overflow beyond int64", "arena exhausted", "too many views",
          "too many storages", "value stack overflow", "2-D access to a 1-D view",
          "step limit reached", "malformed program")


class SweepCompileError(ValueError):
    pass


@dataclass
class SweepProgram:
    """Flat, device-ready form of one MiniCUDA program."""
    code: np.ndarray          # int32 [n, 4]: op, a, b, c
    lits: np.ndarray          # int64 [n_lits]
    kernels: np.ndarray       # int32 [n_kernels, 4]: entry pc, n_params, kparam offset, n_shared
    kparams: np.ndarray       # int32 [n_kparams, 2]: slot, kind (0 scalar, 1 pointer)
    sites: np.ndarray         # int32 [n_sites, 2]: line, column of each access/free site
    n_slots: int
    n_input_sites: int        # count_input_sites (oracle.py:621-628)
    filename: str = "<input>"

    def to_json(self) -> dict:
        return {"code": self.code.tolist(), "lits": [int(x) for x in self.lits],
                "kernels": self.kernels.tolist(), "kparams": self.kparams.tolist(),
                "sites": self.sites.tolist(), "n_slots": self.n_slots,
                "n_input_sites": self.n_input_sites, "filename": self.filename}

    @classmethod
    def from_json(cls, d: dict) -> "SweepProgram":
        def arr(x, dt, w):
            a = np.asarray(x, dtype=dt)
            return a.reshape(-1, w) if w else a
        return cls(arr(d["code"], np.int32, 4), arr(d["lits"], np.int64, 0),
                   arr(d["kernels"], np.int32, 4), arr(d["kparams"], np.int32, 2),
                   arr(d["sites"], np.int32, 2), int(d["n_slots"]),
                   int(d["n_input_sites"]), d.get("filename", "<input>"))

    def site_index(self, line: int, column: int) -> int:
        for i, (l, c) in enumerate(self.sites.tolist()):
            if (l, c) == (line, column):
                return i
        return -1


# ---- compiler: reference AST -> bytecode ---------------------------------------------

def _kind(node) -> str:
    return type(node).__name__


class _Compiler:
    """Walks the reference AST (frontend/ast.py) in the interpreter's own
    evaluation order (oracle.py:277-580), emitting postfix expressions and
    jump-based control flow."""

    def __init__(self, program):
        self.code: list[list[int]] = []
        self.lits: list[int] = []
        self.lit_ix: dict[int, int] = {}
        self.sites: list[tuple[int, int]] = []
        self.site_ix: dict[tuple[int, int], int] = {}
        self.n_slots = 0
        self.host_slots: dict[str, int] = {}
        self.program = program
        self.kernel_ix = {k.name: i for i, k in enumerate(program.kernels)}
        self.n_inputs = 0

    # -- helpers
    def emit(self, op: str, a: int = 0, b: int = 0, c: int = 0) -> int:
        self.code.append([OP[op], int(a), int(b), int(c)])
        return len(self.code) - 1

    def lit(self, v: int) -> int:
        v = int(v)
        if not -(1 << 63) <= v < (1 << 63):
            raise SweepCompileError(f"literal {v} does not fit int64")
        if v not in self.lit_ix:
            self.lit_ix[v] = len(self.lits)
            self.lits.append(v)
        return self.lit_ix[v]

    def site(self, loc) -> int:
        key = (int(loc.line), int(loc.column))
        if key not in self.site_ix:
            if len(self.sites) >= MAX_SITES:
                raise SweepCompileError(f"more than {MAX_SITES} access sites")
            self.site_ix[key] = len(self.sites)
            self.sites.append(key)
        return self.site_ix[key]

    def new_slot(self) -> int:
        s = self.n_slots
        self.n_slots += 1
        if self.n_slots > MAX_SLOTS:
            raise SweepCompileError(f"more than {MAX_SLOTS} variables")
        return s

    def slot(self, scope: dict, name: str) -> int:
        if name not in scope:
            scope[name] = self.new_slot()
        return scope[name]

    # -- expressions (oracle.py:277-323)
    def expr(self, e, scope: dict, in_kernel: bool):
        k = _kind(e)
        if k == "IntLit":
            self.emit("LIT", self.lit(e.value))
        elif k == "Ident":
            if e.name not in scope:
                raise SweepCompileError(f"undeclared name {e.name!r}")
            self.emit("LD", scope[e.name])
        elif k == "InputCall":
            if in_kernel:
                raise SweepCompileError("__input() inside a kernel")
            self.emit("INP", e.site)
        elif k == "BuiltinRef":
            if not in_kernel:
                raise SweepCompileError("builtin outside a kernel")
            self.emit("BLT", BUILTIN_GROUPS.index(e.group) * 3 + AXES.index(e.axis))
        elif k == "BinaryOp":
            self.expr(e.left, scope, in_kernel)
            self.expr(e.right, scope, in_kernel)
            self.emit("BIN", BINOPS.index(e.op))
        elif k == "IndexExpr":
            if len(e.indices) not in (1, 2):
                raise SweepCompileError("subscript arity")
            for ix in e.indices:
                self.expr(ix, scope, in_kernel)
            self.emit("RD", self.ptr(scope, e.base), self.site(e.loc), len(e.indices))
        else:
            raise SweepCompileError(f"unhandled expression {k}")

    def ptr(self, scope: dict, name: str) -> int:
        if name not in scope:
            raise SweepCompileError(f"undeclared pointer {name!r}")
        return scope[name]

    def comparison(self, c, scope, in_kernel):
        self.expr(c.left, scope, in_kernel)
        self.expr(c.right, scope, in_kernel)
        self.emit("CMP", RELS.index(c.rel))

    # -- statements (oracle.py:327-508)
    def block(self, stmts, scope, in_kernel):
        for st in stmts:
            self.stmt(st, scope, in_kernel)

    def stmt(self, st, scope: dict, in_kernel: bool):
        k = _kind(st)
        if k == "AssignStmt":
            self.expr(st.value, scope, in_kernel)
            self.emit("ST", self.slot(scope, st.name))
        elif k == "MallocStmt":
            self.expr(st.size, scope, in_kernel)
            self.emit("MALLOC", self.slot(scope, st.name))
        elif k == "FreeStmt":
            self.emit("FREE", self.ptr(scope, st.name), self.site(st.loc))
        elif k == "LaunchStmt":
            self.launch(st, scope)
        elif k == "AssertStmt":
            self.comparison(st.cond, scope, in_kernel)
            self.emit("ASRT")
        elif k == "ForStmt":
            # for i in range(lo, hi): env[var] = i; body   (oracle.py:373-387)
            it, hi = self.new_slot(), self.new_slot()
            self.expr(st.lower, scope, in_kernel)
            self.emit("ST", it)
            self.expr(st.upper, scope, in_kernel)
            self.emit("ST", hi)
            var = self.slot(scope, st.var)
            top = len(self.code)
            self.emit("LD", it)
            self.emit("LD", hi)
            self.emit("CMP", RELS.index("<"))
            jz = self.emit("JZ")
            self.emit("LD", it)
            self.emit("ST", var)
            self.block(st.body, scope, in_kernel)
            self.emit("LD", it)
            self.emit("LIT", self.lit(1))
            self.emit("BIN", BINOPS.index("+"))
            self.emit("ST", it)
            self.emit("JMP", top)
            self.code[jz][1] = len(self.code)
        elif k == "IfStmt":
            self.comparison(st.cond, scope, in_kernel)
            jz = self.emit("JZ")
            self.block(st.then_body, scope, in_kernel)
            if st.else_body:
                jmp = self.emit("JMP")
                self.code[jz][1] = len(self.code)
                self.block(st.else_body, scope, in_kernel)
                self.code[jmp][1] = len(self.code)
            else:
                self.code[jz][1] = len(self.code)
        elif k == "StoreStmt":
            if len(st.indices) not in (1, 2):
                raise SweepCompileError("subscript arity")
            for ix in st.indices:
                self.expr(ix, scope, in_kernel)
            self.expr(st.value, scope, in_kernel)
            self.emit("WR", self.ptr(scope, st.target), self.site(st.loc), len(st.indices))
        elif k == "AtomicStmt":
            self.expr(st.index, scope, in_kernel)
            self.expr(st.value, scope, in_kernel)
            self.emit("ATOM", self.ptr(scope, st.target), self.site(st.loc), ATOMICS.index(st.op))
        elif k == "ReturnStmt":
            if not in_kernel:
                raise SweepCompileError("return in host code")
            self.emit("RET")
        elif k == "ExternSharedDecl":
            self.emit("XSHM", self.slot(scope, st.name), self.shared_decl(st))
        elif k in ("SharedArrayDecl", "LocalArrayDecl"):
            if not in_kernel:
                raise SweepCompileError("array declaration in host code")
            if len(st.dims) not in (1, 2):
                raise SweepCompileError("array arity")
            for d in st.dims:
                self.expr(d, scope, in_kernel)
            shared = k == "SharedArrayDecl"
            decl = self.shared_decl(st) if shared else 0
            self.emit("ADECL", self.slot(scope, st.name), decl, len(st.dims) | (int(shared) << 2))
        elif k == "PartitionStmt":
            self.expr(st.offset, scope, in_kernel)
            base = self.ptr(scope, st.base)
            self.emit("PART", self.slot(scope, st.name), base)
        else:
            raise SweepCompileError(f"unhandled statement {k}")

    def shared_decl(self, st) -> int:
        # block_shared is keyed by the declaration (oracle.py:429-436, :500)
        key = id(st)
        if key not in self.cur_shared:
            self.cur_shared[key] = len(self.cur_shared)
        return self.cur_shared[key]

    def launch(self, st, scope):
        # oracle.py:512-567: grid, block, negativity, shm, args in param order
        kernel = self.program.kernels[self.kernel_ix[st.kernel]]
        for dim in (st.grid, st.block):
            axes = list(dim.axes)
            if len(axes) > 3:
                raise SweepCompileError("more than 3 launch axes")
            for a in axes:
                self.expr(a, scope, False)
            for _ in range(3 - len(axes)):
                self.emit("LIT", self.lit(1))
        self.emit("NNEG", 6, 0, H_DIM)
        if st.shm is not None:
            self.expr(st.shm, scope, False)
        else:
            self.emit("LIT", self.lit(0))
        self.emit("NNEG", 1, 0, H_SHM)
        n = 0
        for param, arg in zip(kernel.params, st.args):
            if param.is_pointer:
                if _kind(arg) != "Ident":
                    raise SweepCompileError("pointer argument must be a bare identifier")
                self.emit("PARG", self.ptr(scope, arg.name))
            else:
                self.expr(arg, scope, False)
                self.emit("NNEG", 1, 0, H_ARG)
            n += 1
        self.emit("LAUNCH", self.kernel_ix[st.kernel], n)

    def compile(self, filename: str) -> SweepProgram:
        prog = self.program
        from_sites = [e.site for e in _walk_inputs(prog.host_main)]
        self.n_inputs = max(from_sites) + 1 if from_sites else 0
        # host code first (pc 0), then each kernel body
        self.cur_shared = {}
        self.block(prog.host_main, self.host_slots, False)
        self.emit("END")
        kernels, kparams = [], []
        for kdef in prog.kernels:
            scope: dict = {}
            self.cur_shared = {}
            off = len(kparams)
            for p in kdef.params:
                kparams.append([self.slot(scope, p.name), int(p.is_pointer)])
            if len(kdef.params) > MAX_KPARAMS:
                raise SweepCompileError(f"more than {MAX_KPARAMS} kernel parameters")
            entry = len(self.code)
            self.block(kdef.body, scope, True)
            self.emit("KEND")
            kernels.append([entry, len(kdef.params), off, 0])
            kernels[-1][3] = len(self.cur_shared)
        return SweepProgram(
            np.asarray(self.code, dtype=np.int32).reshape(-1, 4),
            np.asarray(self.lits, dtype=np.int64),
            np.asarray(kernels, dtype=np.int32).reshape(-1, 4),
            np.asarray(kparams, dtype=np.int32).reshape(-1, 2),
            np.asarray(self.sites, dtype=np.int32).reshape(-1, 2),
            self.n_slots, self.n_inputs, filename)


def _walk_inputs(stmts):
    """InputCall nodes of the host body (count_input_sites, oracle.py:621-628)."""
    def ex(e):
        k = _kind(e)
        if k == "InputCall":
            yield e
        elif k == "BinaryOp":
            yield from ex(e.left)
            yield from ex(e.right)
        elif k == "IndexExpr":
            for i in e.indices:
                yield from ex(i)

    for st in stmts:
        k = _kind(st)
        for attr in ("value", "size", "lower", "upper", "shm", "index", "offset"):
            v = getattr(st, attr, None)
            if v is not None and hasattr(v, "loc") and _kind(v) != "list":
                yield from ex(v)
        if k in ("AssertStmt", "IfStmt"):
            yield from ex(st.cond.left)
            yield from ex(st.cond.right)
        if k == "LaunchStmt":
            for d in (st.grid, st.block):
                for a in d.axes:
                    yield from ex(a)
            for a in st.args:
                yield from ex(a)
        for attr in ("indices", "dims"):
            for v in getattr(st, attr, None) or []:
                yield from ex(v)
        if k == "ForStmt":
            yield from _walk_inputs(st.body)
        elif k == "IfStmt":
            yield from _walk_inputs(st.then_body)
            yield from _walk_inputs(st.else_body or [])


def compile_program(program) -> SweepProgram:
    """Lower a reference `frontend.ast.Program` to a `SweepProgram`."""
    return _Compiler(program).compile(getattr(program, "filename", "<input>"))


def _as_sweep(program) -> SweepProgram:
    return program if isinstance(program, SweepProgram) else compile_program(program)


# ---- C ABI --------------------------------------------------------------------------

class _CProg(ctypes.Structure):
    _fields_ = [("n_code", ctypes.c_int32), ("code", ctypes.c_void_p),
                ("n_lits", ctypes.c_int32), ("lits", ctypes.c_void_p),
                ("n_kernels", ctypes.c_int32), ("kernels", ctypes.c_void_p),
                ("n_kparams", ctypes.c_int32), ("kparams", ctypes.c_void_p),
                ("n_sites", ctypes.c_int32), ("n_slots", ctypes.c_int32),
                ("n_input_sites", ctypes.c_int32)]


class _COpts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("arena_words", ctypes.c_int64),
                ("step_limit", ctypes.c_int64), ("max_threads", ctypes.c_int64)]


class _CResult(ctypes.Structure):
    _fields_ = [("executions", ctypes.c_int64), ("halted", ctypes.c_int64),
                ("errors", ctypes.c_int64), ("need_tuple", ctypes.c_int64),
                ("need_site", ctypes.c_int64), ("error_tuple", ctypes.c_int64),
                ("error_code", ctypes.c_int32), ("arena_words_used", ctypes.c_int64),
                ("site_labels", ctypes.c_void_p), ("site_first_tuple", ctypes.c_void_p),
                ("device_ms", ctypes.c_float)]


def _cprog(sp: SweepProgram):
    keep = [np.ascontiguousarray(sp.code, dtype=np.int32),
            np.ascontiguousarray(sp.lits, dtype=np.int64),
            np.ascontiguousarray(sp.kernels, dtype=np.int32),
            np.ascontiguousarray(sp.kparams, dtype=np.int32)]
    c = _CProg(len(keep[0]), keep[0].ctypes.data, len(keep[1]), keep[1].ctypes.data,
               len(keep[2]), keep[2].ctypes.data, len(keep[3]), keep[3].ctypes.data,
               len(sp.sites), sp.n_slots, sp.n_input_sites)
    return c, keep


def _copts(device=0, arena_words=0, step_limit=0, max_threads=0):
    return _COpts(int(device), int(arena_words), int(step_limit), int(max_threads))


def _labels(mask: int) -> set:
    return {LABELS[i] for i in range(4) if mask >> i & 1}


@dataclass
class SweepResult:
    """Mirror of oracle.SweepResult (oracle.py:625-636) plus, per violated
    site, the first input tuple (itertools.product order) violating it."""
    bound: int
    input_arity: int
    executions: int
    halted_executions: int
    violations: dict = field(default_factory=dict)
    first_witness: dict = field(default_factory=dict)
    device_ms: float = 0.0

    def has_violation(self, line: int, column: int) -> bool:
        return (line, column) in self.violations


def _tuple_of(t: int, bound: int, arity: int) -> tuple:
    out = []
    for _ in range(arity):
        out.append(t % (bound + 1))
        t //= bound + 1
    return tuple(reversed(out))


def _engine(backend):
    """The C-ABI entry points: the CUDA library, or (tests only) an object
    exposing the same two functions."""
    if backend is not None:
        return backend
    from . import _lib
    L = _lib.lib()
    return L


def _check(rc: int, what: str, backend):
    if rc != 0:
        from . import _lib
        _lib.check(rc, what)


def sweep_once(program, bound: int, arity: int, *, device=0, arena_words=0, step_limit=0,
               max_threads=0, backend=None) -> dict:
    """One device sweep over [0, bound]^arity (no arity growth)."""
    sp = _as_sweep(program)
    L = _engine(backend)
    cp, keep = _cprog(sp)
    ns = max(len(sp.sites), 1)
    labels = np.zeros(ns, dtype=np.uint32)
    first = np.full((ns, 4), -1, dtype=np.int64)  # per site and label
    res = _CResult()
    res.site_labels = labels.ctypes.data
    res.site_first_tuple = first.ctypes.data
    opts = _copts(device, arena_words, step_limit, max_threads)
    rc = L.oob_sweep_run(ctypes.byref(cp), int(bound), int(arity), ctypes.byref(opts),
                         ctypes.byref(res))
    _check(rc, "oob_sweep_run", backend)
    del keep
    return {"executions": res.executions, "halted": res.halted, "errors": res.errors,
            "need_tuple": res.need_tuple, "need_site": res.need_site,
            "site_labels": labels[:len(sp.sites)], "site_first": first[:len(sp.sites)],
            "device_ms": float(res.device_ms), "arena_words": res.arena_words_used}


def brute_force_all(program, bound: int, stop_when_violated: Optional[set] = None,
                    **kw) -> SweepResult:
    """Device restatement of oracle.brute_force_all (oracle.py:638-681).

    The arity starts at the number of syntactic input sites and grows when an
    execution consumes more: as in the reference, the FIRST tuple (product
    order) that needs another input decides the new arity.  With
    `stop_when_violated` the reference stops at the first tuple after which
    every listed site has a violation; that only shortens its counts, the
    violations it reports are those of the tuples before the stop."""
    sp = _as_sweep(program)
    arity = sp.n_input_sites
    while True:
        if arity > MAX_INPUT_SITES:
            raise ValueError(f"programs with more than {MAX_INPUT_SITES} input sites "
                             "cannot be brute-forced")
        r = sweep_once(sp, bound, arity, **kw)
        need = r["need_tuple"]
        first = [min([int(x) for x in row if x >= 0], default=-1) for row in r["site_first"]]
        if stop_when_violated is not None:
            idx = [sp.site_index(l, c) for (l, c) in stop_when_violated]
            if all(i >= 0 and first[i] >= 0 for i in idx):
                stop = max(first[i] for i in idx)
                if need < 0 or stop < need:
                    return _result(sp, bound, arity, r, limit=stop)
        if need >= 0:
            arity = max(arity + 1, int(r["need_site"]) + 1)
            continue
        return _result(sp, bound, arity, r)


def _result(sp, bound, arity, r, limit=None) -> SweepResult:
    res = SweepResult(bound, arity, int(r["executions"]), int(r["halted"]),
                      device_ms=r["device_ms"])
    if limit is not None:
        # the reference stopped after tuple `limit` (product order)
        res.executions = limit + 1
        res.halted_executions = None  # not tracked per prefix on the device
    for i, (line, col) in enumerate(sp.sites.tolist()):
        firsts = [int(x) for x in r["site_first"][i]]
        labs = {LABELS[b] for b in range(4)
                if firsts[b] >= 0 and (limit is None or firsts[b] <= limit)}
        if labs:
            res.violations[(line, col)] = labs
            f = min(x for x in firsts if x >= 0)
            res.first_witness[(line, col)] = _tuple_of(f, bound, arity)
    return res


def brute_force_verdict(program, line: int, column: int, bound: int, **kw) -> bool:
    """oracle.brute_force_verdict (oracle.py:684-692)."""
    return brute_force_all(program, bound, stop_when_violated={(line, column)},
                           **kw).has_violation(line, column)


def replay_tuples(program, tuples, *, device=0, arena_words=0, step_limit=0,
                  backend=None) -> dict:
    """Run explicit input tuples (one GPU thread each; all of one length)."""
    sp = _as_sweep(program)
    L = _engine(backend)
    T = np.ascontiguousarray(np.asarray(tuples, dtype=np.int64).reshape(len(tuples), -1))
    n, arity = T.shape
    ns = max(len(sp.sites), 1)
    status = np.zeros(n, dtype=np.int32)
    aux = np.zeros(n, dtype=np.int32)
    labels = np.zeros((n, ns), dtype=np.uint8)
    cp, keep = _cprog(sp)
    opts = _copts(device, arena_words, step_limit, 0)
    rc = L.oob_sweep_replay(ctypes.byref(cp), int(n), int(arity), T.ctypes.data,
                            ctypes.byref(opts), status.ctypes.data, aux.ctypes.data,
                            labels.ctypes.data)
    _check(rc, "oob_sweep_replay", backend)
    del keep
    return {"status": status, "aux": aux, "labels": labels[:, :len(sp.sites)]}


@dataclass
class ReplayTrace:
    """The parts of oracle.ExecutionTrace (oracle.py:81-89) a replay decides:
    halted / halt_reason and the violation labels per (line, column)."""
    halted: bool
    halt_reason: Optional[str]
    violations: dict


def replay_witnesses(program, requests, default_value: int, **kw) -> list:
    """Batched oracle.replay_witness (oracle.py:695-720): requests are
    (input_values: dict site->value, line, column); one device thread each.
    Returns [(hit, ReplayTrace)] in request order."""
    sp = _as_sweep(program)
    base = sp.n_input_sites
    pending = []
    for input_values, line, col in requests:
        arity = max([base] + [s + 1 for s in input_values])
        pending.append([input_values.get(s, default_value) for s in range(arity)])
    out: list = [None] * len(pending)
    todo = list(range(len(pending)))
    while todo:
        by_len: dict = {}
        for i in todo:
            by_len.setdefault(len(pending[i]), []).append(i)
        todo = []
        for arity, idx in by_len.items():
            r = replay_tuples(sp, [pending[i] for i in idx], **kw)
            for j, i in enumerate(idx):
                st, aux = int(r["status"][j]), int(r["aux"][j])
                if st == ST_NEED:
                    pending[i] = pending[i] + [default_value] * (aux + 1 - len(pending[i]))
                    todo.append(i)
                elif st == ST_ERROR:
                    raise RuntimeError(f"sweep replay: {ERRORS[aux]} (request {i})")
                else:
                    viol = {tuple(sp.sites[s].tolist()): _labels(int(m))
                            for s, m in enumerate(r["labels"][j]) if m}
                    halted = st == ST_HALT
                    out[i] = ReplayTrace(halted, HALT_REASONS[aux] if halted else None,
                                         {} if halted else viol)
    res = []
    for (input_values, line, col), tr in zip(requests, out):
        res.append((not tr.halted and (line, col) in tr.violations, tr))
    return res


def replay_witness(program, input_values: dict, default_value: int, line: int, column: int,
                   **kw):
    """oracle.replay_witness (oracle.py:695-720) on the device."""
    return replay_witnesses(program, [(input_values, line, column)], default_value, **kw)[0]


def load_programs(path) -> dict:
    """SweepPrograms from a JSON file (gzip-compressed when it ends in .gz)."""
    import gzip
    raw = open(path, "rb").read()
    if str(path).endswith(".gz"):
        raw = gzip.decompress(raw)
    return {k: SweepProgram.from_json(v) for k, v in json.loads(raw).items()}
