"""Flat wire format of a query batch (the `oob_batch` of include/scuba_oob.h).

`flatten(queries)` turns reference-shaped queries -- `(variables, constraints)`
pairs whose terms are `Lit`/`VarRef`/`BinE` objects (ours or the reference's,
solver.py:32-63) or the compact JSON form of `terms.py` -- into numpy arrays:

  var_begin[n+1]  var_lo/var_hi[V,2]  (int128 as little-endian int64 words)
  con_begin[n+1]  con_rel[C] u8  con_lhs[C] i32  con_rhs[C] i32
  node_begin[n+1] node_op[N] u8  node_a[N] i32  node_b[N] i32
  lit_begin[n+1]  lits[L,2]

Per query the nodes are hash-consed (structurally equal subterms share one
node id), so structural equality -- what the reference's divisor dedup uses
(`e.right not in out`, solver.py:339) -- is node-id equality, and the DAG is
in topological order (children before parents).

Name resolution follows the reference's dict semantics (solver.py:372-374):
the environment is `{v.name: (v.lo, v.hi)}` (last declaration of a name wins),
the branching order is the list order (a repeated name keeps its first
position, which is what the strict `<` tie-break selects), and a query with any
declaration `lo > hi` is Unsat before search -- kept by storing that empty
domain.  A term naming an undeclared variable raises KeyError, an unknown
operator or relation ValueError, as the reference would when evaluating it.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .terms import OPS, RELS

OP_CODE = {"+": 2, "-": 3, "*": 4, "/": 5, "%": 6}
REL_CODE = {r: i for i, r in enumerate(RELS)}
NODE_LIT, NODE_VAR = 0, 1

_I128_MIN = -(1 << 127)
_I128_MAX = (1 << 127) - 1
_M64 = (1 << 64) - 1


def split128(v: int):
    if not (_I128_MIN <= v <= _I128_MAX):
        raise OverflowError(
            f"integer {v} does not fit the engine's 128-bit wire format")
    lo = v & _M64
    hi = v >> 64
    return lo - (1 << 64) if lo >= (1 << 63) else lo, hi


def join128(lo: int, hi: int) -> int:
    return (int(hi) << 64) | (int(lo) & _M64)


def words_to_ints(w: np.ndarray) -> list:
    """[k,2] int64 words -> list of Python ints."""
    if len(w) == 0:
        return []
    lo = w[:, 0].astype(np.uint64).tolist()
    hi = w[:, 1].tolist()
    return [(h << 64) | l for l, h in zip(lo, hi)]


def ints_to_words(vals) -> np.ndarray:
    out = np.empty((len(vals), 2), dtype=np.int64)
    for i, v in enumerate(vals):
        out[i] = split128(int(v))
    return out


class oob_batch(ctypes.Structure):
    _fields_ = [
        ("n_queries", ctypes.c_int64),
        ("var_begin", ctypes.c_void_p),
        ("var_lo", ctypes.c_void_p),
        ("var_hi", ctypes.c_void_p),
        ("con_begin", ctypes.c_void_p),
        ("con_rel", ctypes.c_void_p),
        ("con_lhs", ctypes.c_void_p),
        ("con_rhs", ctypes.c_void_p),
        ("node_begin", ctypes.c_void_p),
        ("node_op", ctypes.c_void_p),
        ("node_a", ctypes.c_void_p),
        ("node_b", ctypes.c_void_p),
        ("lit_begin", ctypes.c_void_p),
        ("lits", ctypes.c_void_p),
    ]


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else 0


@dataclass
class FlatBatch:
    var_begin: np.ndarray
    var_lo: np.ndarray
    var_hi: np.ndarray
    var_names: list          # per query: list of names in var order
    con_begin: np.ndarray
    con_rel: np.ndarray
    con_lhs: np.ndarray
    con_rhs: np.ndarray
    node_begin: np.ndarray
    node_op: np.ndarray
    node_a: np.ndarray
    node_b: np.ndarray
    lit_begin: np.ndarray
    lits: np.ndarray

    @property
    def n(self) -> int:
        return len(self.var_begin) - 1

    @property
    def n_vars_total(self) -> int:
        return int(self.var_begin[-1])

    def as_c(self) -> oob_batch:
        """ctypes view; the FlatBatch must outlive it."""
        b = oob_batch()
        b.n_queries = self.n
        for name, _ in oob_batch._fields_[1:]:
            setattr(b, name, _ptr(getattr(self, name)))
        return b

    def names(self, q: int) -> list:
        if self.var_names is not None:
            return self.var_names[q]
        k = int(self.var_begin[q + 1] - self.var_begin[q])
        return [f"x{i}" for i in range(k)]

    def slice(self, q0: int, q1: int) -> "FlatBatch":
        """Queries [q0, q1) as a new batch (offsets rebased)."""
        def rng(begin, *arrs):
            a, b = int(begin[q0]), int(begin[q1])
            return (begin[q0:q1 + 1] - a,) + tuple(x[a:b] for x in arrs)
        vb, vlo, vhi = rng(self.var_begin, self.var_lo, self.var_hi)
        cb, crel, clhs, crhs = rng(self.con_begin, self.con_rel, self.con_lhs, self.con_rhs)
        nb, nop, na, nbb = rng(self.node_begin, self.node_op, self.node_a, self.node_b)
        lb, lits = rng(self.lit_begin, self.lits)
        names = self.var_names[q0:q1] if self.var_names is not None else None
        return FlatBatch(vb, vlo, vhi, names, cb, crel, clhs, crhs, nb, nop, na, nbb, lb, lits)

    def nbytes(self) -> int:
        return sum(getattr(self, f).nbytes for f in (
            "var_begin", "var_lo", "var_hi", "con_begin", "con_rel", "con_lhs",
            "con_rhs", "node_begin", "node_op", "node_a", "node_b", "lit_begin",
            "lits"))

    # ----- back to terms -----------------------------------------------------

    def query_json(self, q: int) -> dict:
        """The JSON form (terms.py) of query q."""
        vb, ve = int(self.var_begin[q]), int(self.var_begin[q + 1])
        nb = int(self.node_begin[q])
        lb = int(self.lit_begin[q])
        names = self.names(q)
        lo = words_to_ints(self.var_lo[vb:ve])
        hi = words_to_ints(self.var_hi[vb:ve])
        nn = int(self.node_begin[q + 1]) - nb
        lits = words_to_ints(self.lits[lb:int(self.lit_begin[q + 1])])
        ops = self.node_op[nb:nb + nn]
        na = self.node_a[nb:nb + nn]
        nbb = self.node_b[nb:nb + nn]
        memo = {}
        inv_op = {v: k for k, v in OP_CODE.items()}

        def term(i):
            if i in memo:
                return memo[i]
            op = int(ops[i])
            if op == NODE_LIT:
                t = lits[int(na[i])]
            elif op == NODE_VAR:
                t = names[int(na[i])]
            else:
                t = [inv_op[op], term(int(na[i])), term(int(nbb[i]))]
            memo[i] = t
            return t

        cons = []
        for k in range(int(self.con_begin[q]), int(self.con_begin[q + 1])):
            cons.append([RELS[int(self.con_rel[k])], term(int(self.con_lhs[k])),
                         term(int(self.con_rhs[k]))])
        return {"vars": [[n, a, b] for n, a, b in zip(names, lo, hi)], "cons": cons}


class _Builder:
    def __init__(self):
        self.var_begin = [0]
        self.var_lo = []
        self.var_hi = []
        self.var_names = []
        self.con_begin = [0]
        self.con_rel = []
        self.con_lhs = []
        self.con_rhs = []
        self.node_begin = [0]
        self.node_op = []
        self.node_a = []
        self.node_b = []
        self.lit_begin = [0]
        self.lits = []

    def add(self, variables, constraints):
        # --- variables (dict semantics of solver.py:372-374) ---
        index = {}
        names = []
        lo = []
        hi = []
        empty = None
        for v in variables:
            name, vlo, vhi = _var_fields(v)
            if vlo > vhi and empty is None:
                empty = (vlo, vhi)
            if name in index:
                i = index[name]
                lo[i], hi[i] = vlo, vhi       # last declaration wins (dict)
            else:
                index[name] = len(names)
                names.append(name)
                lo.append(vlo)
                hi.append(vhi)
        if empty is not None:                 # Unsat before search (:374)
            lo[0], hi[0] = empty
        # --- nodes, hash-consed ---
        nodes = {}
        lit_index = {}
        n_ops = []
        n_a = []
        n_b = []
        q_lits = []

        def node(key, op, a, b):
            i = nodes.get(key)
            if i is None:
                i = len(n_ops)
                nodes[key] = i
                n_ops.append(op)
                n_a.append(a)
                n_b.append(b)
            return i

        def walk(e):
            kind, payload = _term_kind(e)
            if kind == "L":
                li = lit_index.get(payload)
                if li is None:
                    li = len(q_lits)
                    lit_index[payload] = li
                    q_lits.append(payload)
                return node(("L", payload), NODE_LIT, li, 0)
            if kind == "V":
                if payload not in index:
                    raise KeyError(payload)
                vi = index[payload]
                return node(("V", vi), NODE_VAR, vi, 0)
            op, l, r = payload
            code = OP_CODE.get(op)
            if code is None:
                raise ValueError(f"unknown operator {op!r}")
            li, ri = walk(l), walk(r)
            return node((code, li, ri), code, li, ri)

        rels = []
        lhs = []
        rhs = []
        try:
            for c in constraints:
                rel, l, r = _con_fields(c)
                code = REL_CODE.get(rel)
                if code is None:
                    raise ValueError(f"unknown relation {rel!r}")
                rels.append(code)
                lhs.append(walk(l))
                rhs.append(walk(r))
        except (KeyError, ValueError):
            if empty is None:
                raise
            # an empty domain: Unsat before search (solver.py:374); the
            # reference never evaluates these constraints, so it raises nothing
            rels, lhs, rhs = [], [], []
            n_ops.clear()
            n_a.clear()
            n_b.clear()
            q_lits.clear()
        # --- append ---
        self.var_names.append(names)
        self.var_lo.extend(lo)
        self.var_hi.extend(hi)
        self.var_begin.append(self.var_begin[-1] + len(names))
        self.con_rel.extend(rels)
        self.con_lhs.extend(lhs)
        self.con_rhs.extend(rhs)
        self.con_begin.append(self.con_begin[-1] + len(rels))
        self.node_op.extend(n_ops)
        self.node_a.extend(n_a)
        self.node_b.extend(n_b)
        self.node_begin.append(self.node_begin[-1] + len(n_ops))
        self.lits.extend(q_lits)
        self.lit_begin.append(self.lit_begin[-1] + len(q_lits))

    def finish(self) -> FlatBatch:
        i64 = np.int64
        return FlatBatch(
            var_begin=np.asarray(self.var_begin, dtype=i64),
            var_lo=ints_to_words(self.var_lo),
            var_hi=ints_to_words(self.var_hi),
            var_names=self.var_names,
            con_begin=np.asarray(self.con_begin, dtype=i64),
            con_rel=np.asarray(self.con_rel, dtype=np.uint8),
            con_lhs=np.asarray(self.con_lhs, dtype=np.int32),
            con_rhs=np.asarray(self.con_rhs, dtype=np.int32),
            node_begin=np.asarray(self.node_begin, dtype=i64),
            node_op=np.asarray(self.node_op, dtype=np.uint8),
            node_a=np.asarray(self.node_a, dtype=np.int32),
            node_b=np.asarray(self.node_b, dtype=np.int32),
            lit_begin=np.asarray(self.lit_begin, dtype=i64),
            lits=ints_to_words(self.lits),
        )


def _var_fields(v):
    if isinstance(v, (list, tuple)):
        name, lo, hi = v
    else:
        name, lo, hi = v.name, v.lo, v.hi
    return str(name), int(lo), int(hi)


def _con_fields(c):
    if isinstance(c, (list, tuple)):
        return c[0], c[1], c[2]
    return c.rel, c.lhs, c.rhs


def _term_kind(e):
    """('L', int) | ('V', name) | ('B', (op, left, right)) for objects or JSON."""
    if isinstance(e, bool):
        raise ValueError("boolean is not a term")
    if isinstance(e, int):
        return "L", e
    if isinstance(e, str):
        return "V", e
    if isinstance(e, (list, tuple)):
        return "B", (e[0], e[1], e[2])
    if hasattr(e, "op"):
        return "B", (e.op, e.left, e.right)
    if hasattr(e, "value"):
        return "L", int(e.value)
    if hasattr(e, "name"):
        return "V", e.name
    raise ValueError(f"not a term: {e!r}")


def flatten_py(queries) -> FlatBatch:
    """The interpreted restatement of the wire format (kept as the
    specification the native emitter is tested against)."""
    b = _Builder()
    for q in queries:
        if isinstance(q, dict):
            b.add(q["vars"], q["cons"])
        else:
            b.add(q[0], q[1])
    return b.finish()


def _native():
    try:
        from . import _flatten_native
    except ImportError as e:  # built by paper_2601_21552_b200.build (csrc/Makefile)
        raise ImportError("paper_2601_21552_b200/_flatten_native is not built; run "
                          "python -m paper_2601_21552_b200.build") from e
    return _flatten_native


def flatten(queries) -> FlatBatch:
    """queries: iterable of (variables, constraints) or JSON dicts {vars, cons}.

    Native query emission (csrc/flatten_native.cpp): the Python objects are
    walked through the CPython API, ~20x faster than `flatten_py`, with the
    same arrays, names and errors."""
    if not isinstance(queries, (list, tuple)):
        queries = list(queries)
    f = _native().flatten(queries)
    i64, i32 = np.int64, np.int32

    def arr(buf, dt, w=0):
        a = np.frombuffer(buf, dtype=dt)
        return a.reshape(-1, w) if w else a
    return FlatBatch(
        var_begin=arr(f[0], i64), var_lo=arr(f[1], i64, 2), var_hi=arr(f[2], i64, 2),
        var_names=f[3], con_begin=arr(f[4], i64), con_rel=arr(f[5], np.uint8),
        con_lhs=arr(f[6], i32), con_rhs=arr(f[7], i32), node_begin=arr(f[8], i64),
        node_op=arr(f[9], np.uint8), node_a=arr(f[10], i32), node_b=arr(f[11], i32),
        lit_begin=arr(f[12], i64), lits=arr(f[13], i64, 2))
