"""Prototype of the fast-mode Unsat prover (symbolic bound elimination).

Per query: the constraints become integer polynomial inequalities g >= 0 over
the query's variables plus one atom per distinct division/modulo subterm;
linear equalities with a unit-coefficient variable are eliminated by
substitution; then for a target inequality P >= 0 the prover eliminates
variables one at a time with the other inequalities (P linear in v with a
coefficient a of definite sign on the box, G = R - k*v >= 0 an upper bound
of v: P' = k*P + a*G), and succeeds when the interval upper bound of some P'
is negative.  Every step is sound over the integers in the box, so success
proves Unsat.  Used to shape the device kernel (csrc/fast.cuh)."""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

LIT, VAR, ADD, SUB, MUL, DIV, MOD = range(7)
LT, LE, EQ, GE, GT = range(5)


def padd(p, q, k=1):
    r = dict(p)
    for m, c in q.items():
        r[m] = r.get(m, 0) + k * c
        if r[m] == 0:
            del r[m]
    return r


def pmul(p, q):
    r = {}
    for m1, c1 in p.items():
        for m2, c2 in q.items():
            m = tuple(sorted(m1 + m2))
            r[m] = r.get(m, 0) + c1 * c2
            if r[m] == 0:
                del r[m]
    return r


def pconst(c):
    return {(): c} if c else {}


def ivmul(a, b):
    ps = [a[0] * b[0], a[0] * b[1], a[1] * b[0], a[1] * b[1]]
    return (min(ps), max(ps))


def ivpow(a, e):
    if e == 1:
        return a
    lo, hi = a
    if e % 2 == 0 and lo < 0 < hi:
        return (0, max(lo ** e, hi ** e))
    vals = (lo ** e, hi ** e)
    return (min(vals), max(vals))


def mono_iv(m, box):
    r = (1, 1)
    i = 0
    while i < len(m):
        j = i
        while j < len(m) and m[j] == m[i]:
            j += 1
        r = ivmul(r, ivpow(box[m[i]], j - i))
        i = j
    return r


def peval(p, box):
    lo = hi = 0
    for m, c in p.items():
        a, b = mono_iv(m, box)
        a, b = (c * a, c * b) if c > 0 else (c * b, c * a)
        lo += a
        hi += b
    return lo, hi


def split_var(p, v):
    """p = a*v + s with v not in s; None if p is not linear in v."""
    a, s = {}, {}
    for m, c in p.items():
        n = m.count(v)
        if n == 0:
            s[m] = c
        elif n == 1:
            mm = list(m)
            mm.remove(v)
            a[tuple(mm)] = c
        else:
            return None
    return a, s


class Query:
    def __init__(self, fb, q, box=None):
        vb, ve = int(fb.var_begin[q]), int(fb.var_begin[q + 1])
        nb, ne = int(fb.node_begin[q]), int(fb.node_begin[q + 1])
        lb = int(fb.lit_begin[q])
        cb, ce = int(fb.con_begin[q]), int(fb.con_begin[q + 1])
        from paper_2601_21552_b200.wire import words_to_ints
        lo = words_to_ints(fb.var_lo[vb:ve])
        hi = words_to_ints(fb.var_hi[vb:ve])
        self.nv = ve - vb
        self.box = list(zip(lo, hi)) if box is None else list(box)
        lits = words_to_ints(fb.lits[lb:int(fb.lit_begin[q + 1])]) if fb.lit_begin[q + 1] > lb else []
        ops = fb.node_op[nb:ne]
        na = fb.node_a[nb:ne]
        nbb = fb.node_b[nb:ne]
        self.ineq = []   # polys g >= 0
        self.eqs = []    # polys e == 0
        self.defs = []   # preferred variable to eliminate per equality
        poly = []
        atoms = {}
        for i in range(ne - nb):
            op = int(ops[i])
            if op == LIT:
                poly.append(pconst(lits[int(na[i])]))
            elif op == VAR:
                poly.append({(int(na[i]),): 1})
            elif op == ADD:
                poly.append(padd(poly[na[i]], poly[nbb[i]]))
            elif op == SUB:
                poly.append(padd(poly[na[i]], poly[nbb[i]], -1))
            elif op == MUL:
                poly.append(pmul(poly[na[i]], poly[nbb[i]]))
            else:
                a, b = poly[na[i]], poly[nbb[i]]
                key = (op, tuple(sorted(a.items())), tuple(sorted(b.items())))
                if key not in atoms:
                    atoms[key] = self._atom(op, a, b)
                poly.append(atoms[key])
        rel = fb.con_rel[cb:ce]
        for k in range(ce - cb):
            l = poly[fb.con_lhs[cb + k]]
            r = poly[fb.con_rhs[cb + k]]
            d = padd(r, l, -1)  # r - l
            c = int(rel[k])
            if c == LT:
                self.ineq.append(padd(d, pconst(-1)))
            elif c == LE:
                self.ineq.append(d)
            elif c == EQ:
                # definitions first: `v = expr` eliminates v
                lv = self._bare(l)
                rv = self._bare(r)
                self.eqs.append(d)
                self.defs.append(lv if lv is not None else rv)
            elif c == GE:
                self.ineq.append({m: -x for m, x in d.items()})
            else:
                self.ineq.append(padd({m: -x for m, x in d.items()}, pconst(-1)))

    @staticmethod
    def _bare(p):
        if len(p) == 1:
            (m, c), = p.items()
            if len(m) == 1 and c == 1:
                return m[0]
        return None

    def _atom(self, op, a, b):
        """Fresh variable d for tdiv(a, b) (or a - b*d for tmod)."""
        ia = peval(a, self.box)
        ib = peval(b, self.box)
        d = len(self.box)
        if len(b) == 1 and () in b and b[()] >= 1:
            c = b[()]
            qlo = int(ia[0] / c) if ia[0] >= 0 else -((-ia[0]) // c)
            qhi = int(ia[1] / c) if ia[1] >= 0 else -((-ia[1]) // c)
            self.box.append((qlo, qhi))
            dv = {(d,): 1}
            cd = {(d,): c}
            if ia[0] >= 0:       # c*d <= a <= c*d + c-1
                self.ineq.append(padd(a, cd, -1))
                self.ineq.append(padd(padd(cd, pconst(c - 1)), a, -1))
            elif ia[1] <= 0:     # c*d - (c-1) <= a <= c*d
                self.ineq.append(padd(cd, a, -1))
                self.ineq.append(padd(padd(a, cd, -1), pconst(c - 1)))
            else:
                self.ineq.append(padd(padd(a, cd, -1), pconst(c - 1)))
                self.ineq.append(padd(padd(cd, pconst(c - 1)), a, -1))
            if op == DIV:
                return dv
            return padd(a, cd, -1)
        # opaque: interval of the result only
        if op == DIV:
            cands = []
            for x in ia:
                for y in (max(ib[0], 1), ib[1]):
                    if y >= 1:
                        cands.append(int(x / y) if x >= 0 else -((-x) // y))
            lo, hi = (min(cands + [0]), max(cands + [0]))
        else:
            m = max(abs(ib[0]), abs(ib[1]))
            lo = -(m - 1) if ia[0] < 0 else 0
            hi = (m - 1) if ia[1] > 0 else 0
            lo, hi = min(lo, 0), max(hi, 0)
        self.box.append((lo, hi))
        return {(d,): 1}

    def eliminate_equalities(self):
        changed = True
        while changed:
            changed = False
            for i, e in enumerate(self.eqs):
                pref = self.defs[i]
                cands = sorted(e.items(), key=lambda mc: mc[0] != (pref,))
                for m, c in cands:
                    if len(m) != 1 or abs(c) != 1:
                        continue
                    v = m[0]
                    if any(v in mm for mm in e if mm != m):
                        continue
                    # v = -(e - c*v)/c
                    rest = {mm: x for mm, x in e.items() if mm != m}
                    expr = {mm: -x * c for mm, x in rest.items()}  # c = +-1
                    self._subst(v, expr)
                    lo, hi = self.box[v]
                    self.ineq.append(padd(expr, pconst(-lo)))
                    self.ineq.append(padd(pconst(hi), expr, -1))
                    del self.eqs[i]
                    del self.defs[i]
                    changed = True
                    break
                if changed:
                    break
        for e in self.eqs:
            self.ineq.append(e)
            self.ineq.append({m: -x for m, x in e.items()})
        self.eqs = []
        # drop trivially true (lower bound >= 0) constraints
        self.ineq = [g for g in self.ineq if peval(g, self.box)[0] < 0 or not g]

    def _subst(self, v, expr):
        def sub(p):
            r = {}
            for m, c in p.items():
                n = m.count(v)
                if n == 0:
                    r = padd(r, {m: c})
                    continue
                rest = tuple(x for x in m if x != v)
                t = {rest: c}
                for _ in range(n):
                    t = pmul(t, expr)
                r = padd(r, t)
            return r
        self.ineq = [sub(g) for g in self.ineq]
        self.eqs = [sub(e) for e in self.eqs]

    def tighten(self, rounds=8):
        """Sound bound propagation over the polynomial inequalities: for
        g = k*v + s >= 0 with constant k, k*v >= -max(s).  False on an
        empty box (Unsat)."""
        for _ in range(rounds):
            changed = False
            for g in self.ineq:
                for v in {v for m in g for v in m}:
                    sp = split_var(g, v)
                    if sp is None:
                        continue
                    a, s = sp
                    if len(a) != 1 or () not in a:
                        continue
                    k = a[()]
                    shi = peval(s, self.box)[1]
                    lo, hi = self.box[v]
                    if k > 0:
                        nlo = -(shi // k)          # ceil(-shi / k)
                        if nlo > lo:
                            lo, changed = nlo, True
                    else:
                        nhi = shi // (-k)          # floor(shi / |k|)
                        if nhi < hi:
                            hi, changed = nhi, True
                    if lo > hi:
                        return False
                    self.box[v] = (lo, hi)
            if not changed:
                break
        return True

    def refute(self, depth=4):
        for g in self.ineq:
            if peval(g, self.box)[1] < 0:
                return True
        for t, g in enumerate(self.ineq):
            if self._rec(g, depth, {t}):
                return True
        return False

    def _rec(self, p, depth, used):
        if peval(p, self.box)[1] < 0:
            return True
        if depth == 0:
            return False
        vars_ = sorted({v for m in p for v in m})
        for v in vars_:
            sp = split_var(p, v)
            if sp is None:
                continue
            a, s = sp
            alo, ahi = peval(a, self.box)
            if alo >= 0:
                want = -1
            elif ahi <= 0:
                want = 1
            else:
                continue
            for j, g in enumerate(self.ineq):
                if j in used:
                    continue
                sg = split_var(g, v)
                if sg is None:
                    continue
                ga, gs = sg
                if len(ga) != 1 or () not in ga:
                    continue
                k = ga[()]
                if (k > 0) == (want > 0) and k != 0:
                    # g = k*v + gs, k has the sign we need
                    kk = abs(k)
                    mult = a if want < 0 else {m: -x for m, x in a.items()}
                    p2 = padd({m: kk * x for m, x in p.items()}, pmul(mult, g))
                    if self._rec(p2, depth - 1, used | {j}):
                        return True
        return False


if __name__ == "__main__":
    import numpy as np
    from paper_2601_21552_b200 import synth
    from oracle import oracle
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    fb = synth.generate(cfg, n, names=False)
    lo, hi, st = oracle.propagate_flat(fb)
    from paper_2601_21552_b200.wire import words_to_ints
    ok = fail = root = 0
    fails = []
    for q in range(fb.n):
        if st[q] == 0:
            root += 1
            continue
        vb, ve = int(fb.var_begin[q]), int(fb.var_begin[q + 1])
        box = list(zip(words_to_ints(lo[vb:ve]), words_to_ints(hi[vb:ve])))
        Q = Query(fb, q, box)
        Q.eliminate_equalities()
        if Q.refute():
            ok += 1
        else:
            fail += 1
            fails.append(q)
    print(f"{cfg}: root-refuted {root}, symbolic {ok}, unknown {fail}; tmpl of unknown",
          np.bincount(fb.tmpl[fails]) if fails else [])


def run_declared(cfg, n, first=0):
    import numpy as np
    import time
    from paper_2601_21552_b200 import synth
    fb = synth.generate(cfg, n, first=first, names=False)
    ok = 0
    fails = []
    t = time.perf_counter()
    for q in range(fb.n):
        Q = Query(fb, q)
        Q.eliminate_equalities()
        if Q.refute():
            ok += 1
        else:
            fails.append(q)
    print(f"{cfg} declared domains: symbolic {ok}, unknown {len(fails)} "
          f"({time.perf_counter() - t:.1f} s)")
    return fb, fails
