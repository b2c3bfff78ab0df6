"""Host-side estimate of x32 eligibility after root propagation:
the fraction of synthetic queries / passes whose real values stay below 2^28
while clamp-derived targets stay beyond them (uses the CPU oracle).

    python tools/x32_probe.py
"""
import sys, json, numpy as np, copy
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_21552_b200 import synth
from paper_2601_21552_b200.wire import words_to_ints
from oracle import oracle
INF = 10**18

def term_nodes(t):
    # returns nested tuple representation
    return t

def analyze(q, lo, hi):
    dom = {name: (l, h) for name, l, h in zip([v[0] for v in q["vars"]], lo, hi)}
    Breal = [0]
    for l, h in dom.values(): Breal[0] = max(Breal[0], abs(l), abs(h))
    def fwd(t):
        if isinstance(t, int):
            Breal[0] = max(Breal[0], abs(t)); return (t, t)
        if isinstance(t, str):
            return dom[t]
        op, a, b = t[0], t[1], t[2]
        (l0, l1), (r0, r1) = fwd(a), fwd(b)
        if op == '+': r = (l0 + r0, l1 + r1)
        elif op == '-': r = (l0 - r1, l1 - r0)
        elif op == '*':
            k = [l0*r0, l0*r1, l1*r0, l1*r1]; r = (min(k), max(k))
        else:
            d0, d1 = max(r0, 1), r1
            if d0 > d1: return (0, 0)
            if op == '/':
                def td(x, y): qq = abs(x)//abs(y); return qq if (x<0)==(y<0) else -qq
                k = [td(l0,d0), td(l0,d1), td(l1,d0), td(l1,d1)]; r = (min(k), max(k))
            else:
                m = d1 - 1; r = (0 if l0 >= 0 else max(l0,-m), 0 if l1 <= 0 else min(l1, m))
        Breal[0] = max(Breal[0], abs(r[0]), abs(r[1]))
        return r
    minf = [float('inf')]
    def tgt(t, lo_t, hi_t, lo_inf, hi_inf):
        # lo_inf/hi_inf: magnitude lower bound of the INF-derived target side (None if real)
        if lo_inf is None: Breal[0] = max(Breal[0], abs(lo_t))
        else: minf[0] = min(minf[0], lo_inf)
        if hi_inf is None: Breal[0] = max(Breal[0], abs(hi_t))
        else: minf[0] = min(minf[0], hi_inf)
        if isinstance(t, (int, str)): return
        op, a, b = t[0], t[1], t[2]
        (l0, l1), (r0, r1) = fwd(a), fwd(b)
        F = lambda x: max(abs(x[0]), abs(x[1]))
        if op in '+-':
            fa, fb = F(fwd(a)), F(fwd(b))
            na = lambda v, s: None if v is None else v - s
            if op == '+':
                tgt(a, lo_t - r1, hi_t - r0, na(lo_inf, fb), na(hi_inf, fb))
                tgt(b, lo_t - l1, hi_t - l0, na(lo_inf, fa), na(hi_inf, fa))
            else:
                tgt(a, lo_t + r0, hi_t + r1, na(lo_inf, fb), na(hi_inf, fb))
                tgt(b, l0 - hi_t, l1 - lo_t, na(hi_inf, fa), na(lo_inf, fa))
        elif op == '*':
            if l0 < 0 or r0 < 0: return
            # lower targets: ceil(t0n / ...) real (t0n = max(lo,0), -INF -> 0 -> -INF stays)
            t0n = max(lo_t, 0) if lo_inf is None else 0
            lo_l = -INF if t0n <= 0 else -(-t0n // max(r1,1)); lo_r = -INF if t0n <= 0 else -(-t0n // max(l1,1))
            lli = (INF if t0n <= 0 else None)
            hi_l = hi_t // r0 if r0 > 0 else INF; hi_r = hi_t // l0 if l0 > 0 else INF
            hli = (None if (hi_inf is None and r0 > 0) else ((hi_inf / r0) if (hi_inf is not None and r0 > 0) else INF))
            hri = (None if (hi_inf is None and l0 > 0) else ((hi_inf / l0) if (hi_inf is not None and l0 > 0) else INF))
            tgt(a, lo_l, hi_l, lli, hli); tgt(b, lo_r, hi_r, lli, hri)
        elif op == '/' and isinstance(b, int) and b >= 1:
            c = b
            tgt(a, lo_t * c, hi_t * c + c - 1, None if lo_inf is None else lo_inf * c, None if hi_inf is None else hi_inf * c)
    for rel, lhs, rhs in q["cons"]:
        (l0, l1), (r0, r1) = fwd(lhs), fwd(rhs)
        if rel == '<': tgt(lhs, -INF, r1 - 1, INF, None); tgt(rhs, l0 + 1, INF, None, INF)
        elif rel == '<=': tgt(lhs, -INF, r1, INF, None); tgt(rhs, l0, INF, None, INF)
        elif rel == '=': a0 = max(l0, r0); a1 = min(l1, r1); tgt(lhs, a0, a1, None, None); tgt(rhs, a0, a1, None, None)
        elif rel == '>=': tgt(lhs, r0, INF, None, INF); tgt(rhs, -INF, l1, INF, None)
        else: tgt(lhs, r0 + 1, INF, None, INF); tgt(rhs, -INF, l1 - 1, INF, None)
    return Breal[0], minf[0]

def conv(t):
    if isinstance(t, list):
        return (t[0], conv(t[1]), conv(t[2]))
    return t

for cfg in ("c3", "c4"):
    n = 3000
    fb = synth.generate(cfg, n, names=True)
    r = oracle.solve_flat(fb)
    lo, hi, st = oracle.propagate_flat(fb)
    ok_pass = tot_pass = 0; ok_q = 0
    for q in range(n):
        if st[q] == 0: 
            tot_pass += r["passes"][q]; ok_pass += r["passes"][q]; ok_q += 1; continue
        j = fb.query_json(q)
        j["cons"] = [(c[0], conv(c[1]), conv(c[2])) for c in j["cons"]]
        vb, ve = int(fb.var_begin[q]), int(fb.var_begin[q+1])
        L = words_to_ints(lo[vb:ve]); H = words_to_ints(hi[vb:ve])
        B, mi = analyze(j, L, H)
        ok = B <= 2**28 and mi > 4 * B
        tot_pass += r["passes"][q]
        if ok: ok_pass += r["passes"][q]; ok_q += 1
    print(cfg, "x32-eligible queries %.3f, passes %.3f" % (ok_q / n, ok_pass / tot_pass))
