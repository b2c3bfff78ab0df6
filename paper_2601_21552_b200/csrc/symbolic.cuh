// symbolic.cuh -- the fast mode's Unsat prover (OOB_F_FAST).
//
// The reference decides a query by interval propagation + bisection
// (solver.py:264-280, :385-416).  On wide input domains that procedure creeps:
// `off < n` with `off >= n` moves one bound by one unit per pass, and a
// nonlinear system such as `off = t*w + j, t < h, j < w, off >= h*w` is only
// refuted once the bisection has fixed h and w to single points.  Both are
// one-line arguments for a symbolic prover, and a sound Unsat is always the
// reference's verdict (its propagation only ever removes solutions, check_model
// is exact, so it can never return Sat on a query without integer solutions in
// its root box).  The prover therefore never decides Sat: what it does not
// refute stays with the exact emulation (K1), which returns the reference's
// verdict and first model.
//
// Per query (warp-cooperative, in the frontier phase of the solve kernels):
//  1. build: every constraint `l rel r` becomes an integer polynomial g >= 0
//     (or g = 0) over the query's variables plus one ATOM per distinct
//     division/modulo subterm; a division by a literal c >= 1 gets the exact
//     truncation bounds c*d <= a <= c*d + c-1 (sign-split), a modulo by c is
//     a - c*d, any other division or modulo is an opaque atom with a sound
//     interval;
//  2. eliminate: equalities `v = expr` (v linear with a unit coefficient) are
//     substituted away; v's domain stays as lo <= expr <= hi;
//  3. tighten: bound propagation over the polynomial inequalities
//     (g = k*v + s >= 0, k constant: k*v >= -max(s));
//  4. eliminate by inequalities (lane-parallel over target inequalities): for
//     a target P >= 0 linear in v with coefficient polynomial a of definite
//     sign on the box, and an inequality G = s - k*v >= 0 (k > 0 constant:
//     an upper bound of v), P' = k*P + a*G >= 0 holds at every solution and
//     no longer mentions v; the greedy step takes the move with the smallest
//     interval upper bound (normalised by k); P' with an upper bound < 0 is a
//     contradiction.  Three moves per target.
// Every number is an exact __int128 below 2^120; an operation that would
// leave that range abandons the move (or the query): never a wrong answer.
#pragma once
#include "format.h"
#include "types.h"

namespace oob {
namespace sym {

typedef __int128 i128;
typedef unsigned __int128 u128;

constexpr int MAXV = 96;   // variables + literal parameters + atoms
constexpr int MAXC = 96;   // constraints in the store (<= 64 reach the search)
constexpr int POOL = 1024; // terms of all store constraints (one buffer)
constexpr int MAXT = 48;   // terms of one working polynomial
constexpr int MAXA = 12;   // atoms
constexpr int STK = 16;    // postfix stack depth of one constraint side
constexpr int DEPTH = 3;   // eliminations per target
constexpr int ROUNDS = 8;  // bound-tightening rounds
constexpr int LANES = 32;

enum : int { R_UNKNOWN = 0, R_REFUTED = 1, R_CONTINUE = 2 };

// the larger steps are out-of-line on the device: one copy each per module
// (keeps the run-time compiled class kernels' NVRTC time down)
#if defined(__CUDA_ARCH__)
#define SYM_NI __noinline__
#else
#define SYM_NI
#endif

OOB_HD inline int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __clzll((long long)x);
#else
    return x ? __builtin_clzll(x) : 64;
#endif
}
OOB_HD inline int bits(i128 x) {
    u128 u = x < 0 ? (u128)(-x) : (u128)x;
    uint64_t hi = (uint64_t)(u >> 64), lo = (uint64_t)u;
    return hi ? 128 - clz64(hi) : 64 - clz64(lo);
}
constexpr int LIMB = 120;  // |every stored value| < 2^120
OOB_HD inline bool big(i128 x) { return bits(x) > LIMB; }
OOB_HD inline bool smul(i128 a, i128 b, i128& r) {
    // common case: both factors within int32 -- one 64-bit multiply, exact
    const long long al = (long long)a, bl = (long long)b;
    if ((i128)al == a && (i128)bl == b && al == (long long)(int)al && bl == (long long)(int)bl) {
        r = (i128)(al * bl);
        return true;
    }
    if (a == 0 || b == 0) {
        r = 0;
        return true;
    }
    if (bits(a) + bits(b) > LIMB) return false;
    r = a * b;
    return true;
}
OOB_HD inline bool sadd(i128 a, i128 b, i128& r) {
    r = a + b;  // operands below 2^120: no int128 overflow
    return !big(r);
}
OOB_HD inline i128 imin(i128 a, i128 b) { return a < b ? a : b; }
OOB_HD inline i128 imax(i128 a, i128 b) { return a > b ? a : b; }
OOB_HD inline i128 iabs(i128 a) { return a < 0 ? -a : a; }
// floor(a / b), b > 0
OOB_HD inline i128 fdiv(i128 a, i128 b) {
    i128 q = a / b;
    if ((a % b != 0) && (a < 0)) --q;
    return q;
}
// C truncating division (tdiv, solver.py:94-98), b != 0
OOB_HD inline i128 tdiv(i128 a, i128 b) { return a / b; }

// ---- monomial keys: variable index + 1 per byte, descending from the top ----
OOB_HD inline uint64_t vkey(int v) { return (uint64_t)(v + 1) << 56; }
OOB_HD inline int kcount(uint64_t k, int v) {
    int n = 0;
    const uint64_t b = (uint64_t)(v + 1);
    while (k >> 56) {
        n += (k >> 56) == b;
        k <<= 8;
    }
    return n;
}
OOB_HD inline bool kmul(uint64_t a, uint64_t b, uint64_t& r) {
    r = 0;
    int n = 0;
    while ((a >> 56) || (b >> 56)) {
        if (n == 8) return false;
        uint64_t x = a >> 56, y = b >> 56, t;
        if (x >= y) {
            t = x;
            a <<= 8;
        } else {
            t = y;
            b <<= 8;
        }
        r |= t << (56 - 8 * n);
        ++n;
    }
    return true;
}
// remove one occurrence of variable v
OOB_HD inline uint64_t kremove(uint64_t k, int v) {
    const uint64_t b = (uint64_t)(v + 1);
    uint64_t r = 0;
    int n = 0;
    bool done = false;
    while (k >> 56) {
        uint64_t x = k >> 56;
        k <<= 8;
        if (!done && x == b) {
            done = true;
            continue;
        }
        r |= x << (56 - 8 * n);
        ++n;
    }
    return r;
}

// ---- polynomials: sorted (ascending key) term arrays ------------------------
struct PV {
    uint64_t* k;
    i128* c;
    int n;
    int cap;
};

OOB_HD inline void pclear(PV& p) { p.n = 0; }
// add c * x^k into p (sorted insert, combine, drop zero)
OOB_HD SYM_NI inline bool pins(PV& p, uint64_t k, i128 c) {
    if (c == 0) return true;
    int i = 0;
    while (i < p.n && p.k[i] < k) ++i;
    if (i < p.n && p.k[i] == k) {
        i128 s;
        if (!sadd(p.c[i], c, s)) return false;
        if (s == 0) {
            for (int j = i; j + 1 < p.n; ++j) {
                p.k[j] = p.k[j + 1];
                p.c[j] = p.c[j + 1];
            }
            --p.n;
        } else {
            p.c[i] = s;
        }
        return true;
    }
    if (p.n >= p.cap) return false;
    for (int j = p.n; j > i; --j) {
        p.k[j] = p.k[j - 1];
        p.c[j] = p.c[j - 1];
    }
    p.k[i] = k;
    p.c[i] = c;
    ++p.n;
    return true;
}
OOB_HD inline bool pcopy(const PV& a, PV& o) {
    if (a.n > o.cap) return false;
    for (int i = 0; i < a.n; ++i) {
        o.k[i] = a.k[i];
        o.c[i] = a.c[i];
    }
    o.n = a.n;
    return true;
}
// o = sa*a + sb*b (o must not alias a or b)
OOB_HD SYM_NI inline bool plin(const PV& a, i128 sa, const PV& b, i128 sb, PV& o) {
    int i = 0, j = 0;
    o.n = 0;
    while (i < a.n || j < b.n) {
        uint64_t k;
        i128 c = 0, t;
        if (j >= b.n || (i < a.n && a.k[i] < b.k[j])) {
            k = a.k[i];
            if (!smul(a.c[i], sa, c)) return false;
            ++i;
        } else if (i >= a.n || b.k[j] < a.k[i]) {
            k = b.k[j];
            if (!smul(b.c[j], sb, c)) return false;
            ++j;
        } else {
            k = a.k[i];
            if (!smul(a.c[i], sa, c) || !smul(b.c[j], sb, t) || !sadd(c, t, c)) return false;
            ++i;
            ++j;
        }
        if (c == 0) continue;
        if (o.n >= o.cap) return false;
        o.k[o.n] = k;
        o.c[o.n] = c;
        ++o.n;
    }
    return true;
}
// o += s * a * b
OOB_HD SYM_NI inline bool pmuladd(const PV& a, const PV& b, i128 s, PV& o) {
    for (int i = 0; i < a.n; ++i)
        for (int j = 0; j < b.n; ++j) {
            uint64_t k;
            i128 c;
            if (!kmul(a.k[i], b.k[j], k) || !smul(a.c[i], b.c[j], c) || !smul(c, s, c) || !pins(o, k, c))
                return false;
        }
    return true;
}

// ---- interval evaluation over the box ---------------------------------------
// Box entries [0, np) are literal PARAMETERS (certificate compilation): point
// intervals.  They have the lowest indices, so their bytes are the trailing
// bytes of a key and the terms of one monomial over the other variables are
// adjacent in key order; interval evaluation first collapses each such run to
// one numeric coefficient (exact, as the numeric prover would see it).
struct Box {
    i128* lo;
    i128* hi;
    int np = 0;
};
OOB_HD inline bool ivmul(i128 al, i128 ah, i128 bl, i128 bh, i128& rl, i128& rh) {
    i128 p0, p1, p2, p3;
    if (!smul(al, bl, p0) || !smul(al, bh, p1) || !smul(ah, bl, p2) || !smul(ah, bh, p3)) return false;
    rl = imin(imin(p0, p1), imin(p2, p3));
    rh = imax(imax(p0, p1), imax(p2, p3));
    return true;
}
OOB_HD inline bool ivpow(i128 lo, i128 hi, int e, i128& rl, i128& rh) {
    i128 a = 1, b = 1;
    for (int i = 0; i < e; ++i)
        if (!smul(a, lo, a) || !smul(b, hi, b)) return false;
    if (e % 2 == 0 && lo < 0 && hi > 0) {
        rl = 0;
        rh = imax(a, b);
    } else {
        rl = imin(a, b);
        rh = imax(a, b);
    }
    return true;
}
OOB_HD SYM_NI inline bool mono_iv(uint64_t k, const Box& B, i128& rl, i128& rh) {
    rl = rh = 1;
    while (k >> 56) {
        const int v = (int)(k >> 56) - 1;
        int e = 0;
        while ((k >> 56) == (uint64_t)(v + 1)) {
            ++e;
            k <<= 8;
        }
        i128 pl, ph;
        if (!ivpow(B.lo[v], B.hi[v], e, pl, ph) || !ivmul(rl, rh, pl, ph, rl, rh)) return false;
    }
    return true;
}
// key without its parameter bytes (the trailing bytes with index < np)
OOB_HD inline uint64_t kstrip(uint64_t k, int np, i128& pv_of_key, const Box& B, bool& ok) {
    uint64_t r = 0;
    int n = 0;
    pv_of_key = 1;
    while (k >> 56) {
        const uint64_t x = k >> 56;
        k <<= 8;
        if ((int)x <= np) {
            if (!smul(pv_of_key, B.lo[x - 1], pv_of_key)) ok = false;
        } else {
            r |= x << (56 - 8 * n);
            ++n;
        }
    }
    return r;
}
OOB_HD SYM_NI inline bool peval(const PV& p, const Box& B, i128& lo, i128& hi) {
    lo = hi = 0;
    for (int i = 0; i < p.n;) {
        // one run of terms with the same monomial over the non-parameters
        bool ok = true;
        i128 pv, c = 0, t;
        const uint64_t rk = B.np ? kstrip(p.k[i], B.np, pv, B, ok) : p.k[i];
        if (!B.np) pv = 1;
        if (!ok || !smul(p.c[i], pv, t) || !sadd(c, t, c)) return false;
        ++i;
        while (B.np && i < p.n) {
            const uint64_t rk2 = kstrip(p.k[i], B.np, pv, B, ok);
            if (rk2 != rk) break;
            if (!ok || !smul(p.c[i], pv, t) || !sadd(c, t, c)) return false;
            ++i;
        }
        if (c == 0) continue;
        i128 a, b, x, y;
        if (!mono_iv(rk, B, a, b)) return false;
        if (!smul(c, a, x) || !smul(c, b, y)) return false;
        if (c < 0) {
            i128 u = x;
            x = y;
            y = u;
        }
        if (!sadd(lo, x, lo) || !sadd(hi, y, hi)) return false;
    }
    return true;
}
// p = a*v + s with v absent from s; false if p is not linear in v
OOB_HD SYM_NI inline bool psplit(const PV& p, int v, PV& a, PV& s) {
    a.n = s.n = 0;
    for (int i = 0; i < p.n; ++i) {
        const int n = kcount(p.k[i], v);
        if (n == 0) {
            if (s.n >= s.cap) return false;
            s.k[s.n] = p.k[i];
            s.c[s.n] = p.c[i];
            ++s.n;
        } else if (n == 1) {
            if (!pins(a, kremove(p.k[i], v), p.c[i])) return false;
        } else {
            return false;
        }
    }
    return true;
}
// coefficient of v when p mentions v only in the single term c*v; 0 otherwise
OOB_HD inline i128 unit_coef(const PV& p, int v) {
    const uint64_t kv = vkey(v);
    i128 k = 0;
    for (int i = 0; i < p.n; ++i) {
        if (p.k[i] == kv) k = p.c[i];
        else if (kcount(p.k[i], v)) return 0;
    }
    return k;
}

// g = K*v + s where K involves only literal parameters (box entries
// [p0, p1)) and constants; false when g is not of that form in v (or v is
// absent).  Without parameters K is the constant coefficient of v.
OOB_HD inline bool pcoef(const PV& g, int v, int p0, int p1, PV& K, PV& s) {
    K.n = s.n = 0;
    for (int i = 0; i < g.n; ++i) {
        const int n = kcount(g.k[i], v);
        if (n == 0) {
            if (s.n >= s.cap) return false;
            s.k[s.n] = g.k[i];
            s.c[s.n] = g.c[i];
            ++s.n;
            continue;
        }
        if (n > 1) return false;
        const uint64_t rest = kremove(g.k[i], v);
        for (uint64_t r = rest; r >> 56; r <<= 8) {
            const int u = (int)(r >> 56) - 1;
            if (u < p0 || u >= p1) return false;
        }
        if (!pins(K, rest, g.c[i])) return false;
    }
    return K.n > 0;
}

// ---- the per-query store (global scratch of the warp) -----------------------
struct Store {
    i128 lo[MAXV], hi[MAXV];
    i128 coef[2][POOL];
    uint64_t key[2][POOL];
    int off[MAXC], len[MAXC];
    int8_t is_eq[MAXC];
    int8_t def[MAXC];
    // atoms: dividend / divisor polynomials (dedup) in their own pool
    i128 acoef[MAXA * 2 * 16];
    uint64_t akey[MAXA * 2 * 16];
    int alen[MAXA * 2];
    int8_t aop[MAXA];
    int8_t avar[MAXA];
    int8_t acase[MAXA];   // dividend sign on the build box: 0 >= 0, 1 <= 0, 2 mixed
    int8_t alitdiv[MAXA]; // divisor is a literal >= 1 (constant or parameter)
    int natoms;
    // eliminated variables whose domain became constraints (certificate
    // compilation: those constraints hold for a query only if its domain of
    // the variable lies within the bounds used here -- cert.cuh checks it)
    int nelim;
    int16_t elim_v[MAXC];
    int8_t elim_flags[MAXC];  // 1: lower bound used, 2: upper bound used
    i128 elim_lo[MAXC], elim_hi[MAXC];
    // literal parameters (certificate compilation): box entries 0 .. np-1
    // hold literal slots whose value varies inside the structure class; the
    // query's variables follow (np .. np+nv-1), then the atoms
    int np;
    int nv, nc, cur, used;
    int status;
    // postfix stack while building (one constraint side at a time)
    i128 scoef[STK][MAXT];
    uint64_t skey[STK][MAXT];
    int slen[STK];
};
struct LaneWork {  // per-lane working polynomials of the target search
    i128 c[8][MAXT];
    uint64_t k[8][MAXT];
};

OOB_HD inline PV store_poly(Store& S, int j) {
    PV p;
    p.k = S.key[S.cur] + S.off[j];
    p.c = S.coef[S.cur] + S.off[j];
    p.n = S.len[j];
    p.cap = S.len[j];
    return p;
}
OOB_HD inline PV stk(Store& S, int d) {
    PV p;
    p.k = S.skey[d];
    p.c = S.scoef[d];
    p.n = S.slen[d];
    p.cap = MAXT;
    return p;
}
OOB_HD inline PV work(LaneWork& W, int i) {
    PV p;
    p.k = W.k[i];
    p.c = W.c[i];
    p.n = 0;
    p.cap = MAXT;
    return p;
}
// append polynomial p (times sign) as constraint (eq or ineq)
OOB_HD SYM_NI inline bool add_con(Store& S, const PV& p, i128 sign, i128 add, bool eq, int def) {
    if (S.nc >= MAXC) return false;
    const int o = S.used;
    PV d;
    d.k = S.key[S.cur] + o;
    d.c = S.coef[S.cur] + o;
    d.n = 0;
    d.cap = POOL - o;
    PV k1;
    uint64_t kk = 0;
    i128 cc = add;
    k1.k = &kk;
    k1.c = &cc;
    k1.n = add != 0;
    k1.cap = 1;
    if (!plin(p, sign, k1, 1, d)) return false;
    S.off[S.nc] = o;
    S.len[S.nc] = d.n;
    S.is_eq[S.nc] = eq;
    S.def[S.nc] = (int8_t)def;
    S.used += d.n;
    ++S.nc;
    return true;
}
OOB_HD inline bool poly_eq(const PV& a, const PV& b) {
    if (a.n != b.n) return false;
    for (int i = 0; i < a.n; ++i)
        if (a.k[i] != b.k[i] || a.c[i] != b.c[i]) return false;
    return true;
}
OOB_HD inline PV atom_poly(Store& S, int slot) {
    PV p;
    p.k = S.akey + slot * 16;
    p.c = S.acoef + slot * 16;
    p.n = S.alen[slot];
    p.cap = 16;
    return p;
}

// op(a, b) for DIV/MOD: replaces the stack entry `a` with the atom's polynomial.
// A divisor that is a literal c >= 1 (a constant, or a literal parameter whose
// value is >= 1: certificates guard that) gets the exact truncation bounds.
OOB_HD inline bool lit_divisor(const Store& S, const PV& b) {
    if (b.n != 1) return false;
    if (b.k[0] == 0) return b.c[0] >= 1;
    if (b.c[0] != 1 || (b.k[0] << 8)) return false;
    const int v = (int)(b.k[0] >> 56) - 1;
    return v < S.np && S.lo[v] >= 1;
}
OOB_HD SYM_NI inline bool make_atom(Store& S, int op, PV& a, const PV& b) {
    const bool lit_div = lit_divisor(S, b);
    // dedup: same op, same dividend and divisor
    int at = -1;
    for (int i = 0; i < S.natoms && at < 0; ++i) {
        if (S.aop[i] != op) continue;
        PV x = atom_poly(S, 2 * i), y = atom_poly(S, 2 * i + 1);
        if (poly_eq(x, a) && poly_eq(y, b)) at = i;
    }
    int d;
    if (at >= 0) {
        d = S.avar[at];
    } else {
        if (S.natoms >= MAXA || S.nv >= MAXV || a.n > 16 || b.n > 16) return false;
        at = S.natoms++;
        PV x = atom_poly(S, 2 * at), y = atom_poly(S, 2 * at + 1);
        pcopy(a, x);
        pcopy(b, y);
        S.alen[2 * at] = a.n;
        S.alen[2 * at + 1] = b.n;
        S.aop[at] = (int8_t)op;
        S.alitdiv[at] = lit_div;
        d = S.nv++;
        S.avar[at] = (int8_t)d;
        Box B{S.lo, S.hi, S.np};
        i128 al, ah, bl, bh;
        if (!peval(a, B, al, ah) || !peval(b, B, bl, bh)) return false;
        S.acase[at] = al >= 0 ? 0 : (ah <= 0 ? 1 : 2);
        if (lit_div) {
            const i128 c = bl;  // the literal's value (a point)
            S.lo[d] = tdiv(al, c);
            S.hi[d] = tdiv(ah, c);
            // with t = a - c*d:  0 <= t <= c-1 (a >= 0),  -(c-1) <= t <= 0
            // (a <= 0),  |t| <= c-1 otherwise
            i128 tc[17], uc[17];
            uint64_t tk[17], uk[17];
            PV t{tk, tc, 0, 17}, u{uk, uc, 0, 17}, dv;
            uint64_t kd = vkey(d);
            i128 one = 1;
            dv.k = &kd;
            dv.c = &one;
            dv.n = 1;
            dv.cap = 1;
            if (!pcopy(a, t) || !pmuladd(b, dv, -1, t)) return false;  // t = a - c*d
            if (!pcopy(b, u) || !pins(u, 0, -1)) return false;          // u = c - 1
            i128 wc[40];
            uint64_t wk[40];
            PV w{wk, wc, 0, 40};  // u - t, u + t
            const int cs = S.acase[at];
            if (cs == 0 && !add_con(S, t, 1, 0, false, -1)) return false;
            if (cs == 1 && !add_con(S, t, -1, 0, false, -1)) return false;
            if (cs != 1) {
                if (!plin(u, 1, t, -1, w) || !add_con(S, w, 1, 0, false, -1)) return false;
            }
            if (cs != 0) {
                if (!plin(u, 1, t, 1, w) || !add_con(S, w, 1, 0, false, -1)) return false;
            }
        } else if (op == NODE_DIV) {
            // opaque quotient: |tdiv(a, b)| <= |a|; for a >= 0, b >= 1 the
            // corner quotients
            if (al >= 0 && bl >= 1) {
                S.lo[d] = tdiv(al, bh);
                S.hi[d] = tdiv(ah, bl);
            } else {
                const i128 m = imax(iabs(al), iabs(ah));
                S.lo[d] = -m;
                S.hi[d] = m;
            }
        } else {
            // opaque remainder: sign of the dividend, |r| < |b|, |r| <= |a|
            i128 m = imax(iabs(bl), iabs(bh)) - 1;
            if (m < 0) m = 0;
            m = imin(m, imax(iabs(al), iabs(ah)));
            S.lo[d] = al < 0 ? -m : 0;
            S.hi[d] = ah > 0 ? m : 0;
        }
    }
    // the atom's polynomial replaces the dividend on the stack
    if (S.alitdiv[at] && op == NODE_MOD) {  // a - c*d
        uint64_t kd = vkey(d);
        i128 one = 1;
        PV dv{&kd, &one, 1, 1};
        return pmuladd(b, dv, -1, a);
    }
    a.n = 0;
    return pins(a, vkey(d), 1);
}

// evaluate a postfix constraint side [root - size + 1, root] onto stack slot
// `base` (slots above it are scratch)
template <typename GetLit>
OOB_HD inline bool build_side(Store& S, const uint32_t* code, uint32_t root, int base, GetLit lit,
                              const int16_t* pmap) {
    auto size_of = [&](uint32_t i) -> uint32_t {
        const uint32_t w = code[i];
        return (w & 7u) >= NODE_ADD ? (w >> 3) : 1u;
    };
    const uint32_t start = root + 1 - size_of(root);
    int sp = base;
    for (uint32_t j = start; j <= root; ++j) {
        const uint32_t w = code[j], op = w & 7u, arg = w >> 3;
        if (op == NODE_LIT || op == NODE_VAR) {
            if (sp >= STK) return false;
            PV p = stk(S, sp);
            p.n = 0;
            if (op == NODE_LIT && pmap && pmap[arg] >= 0) {
                if (!pins(p, vkey(pmap[arg]), 1)) return false;
            } else if (op == NODE_LIT) {
                const i128 v = lit(arg);
                if (big(v)) return false;
                if (!pins(p, 0, v)) return false;
            } else {
                if (!pins(p, vkey(S.np + (int)arg), 1)) return false;
            }
            S.slen[sp++] = p.n;
            continue;
        }
        if (sp < base + 2) return false;
        PV a = stk(S, sp - 2), b = stk(S, sp - 1);
        if (op == NODE_ADD || op == NODE_SUB) {
            for (int i = 0; i < b.n; ++i)
                if (!pins(a, b.k[i], op == NODE_ADD ? b.c[i] : -b.c[i])) return false;
        } else if (op == NODE_MUL) {
            // product into the free slot sp, then moved down
            if (sp >= STK) return false;
            PV o = stk(S, sp);
            o.n = 0;
            if (!pmuladd(a, b, 1, o) || !pcopy(o, a)) return false;
        } else if (op == NODE_DIV || op == NODE_MOD) {
            if (!make_atom(S, (int)op, a, b)) return false;
        } else {
            return false;
        }
        S.slen[sp - 2] = a.n;
        --sp;
    }
    return sp == base + 1;
}

OOB_HD inline bool bare_var(const PV& p, int& v) {
    if (p.n == 1 && p.c[0] == 1 && p.k[0] && !(p.k[0] << 8)) {
        v = (int)(p.k[0] >> 56) - 1;
        return true;
    }
    return false;
}

// 1. build the store from the packed query (cons/code of its class, domains
// and literal slots as exact integers)
// pmap (certificate compilation; null: every literal is a number): literal
// slot -> parameter index or -1; pslot: parameter -> literal slot
template <typename GetDom, typename GetLit>
OOB_HD inline bool build(Store& S, const uint32_t* cons, const uint32_t* code, uint32_t nv, uint32_t ncon,
                         GetDom dom, GetLit lit, const int16_t* pmap = nullptr, int np = 0,
                         const int16_t* pslot = nullptr) {
    if (nv + (uint32_t)np > (uint32_t)MAXV) return false;
    S.np = pmap ? np : 0;
    S.nv = S.np + (int)nv;
    S.nelim = 0;
    S.nc = 0;
    S.cur = 0;
    S.used = 0;
    S.natoms = 0;
    for (int p = 0; p < S.np; ++p) {  // a parameter's box is its value
        const i128 x = lit((uint32_t)pslot[p]);
        if (big(x)) return false;
        S.lo[p] = S.hi[p] = x;
    }
    for (uint32_t v = 0; v < nv; ++v) {
        const int b = S.np + (int)v;
        S.lo[b] = dom(2 * v);
        S.hi[b] = dom(2 * v + 1);
        if (big(S.lo[b]) || big(S.hi[b])) return false;
        if (S.lo[b] > S.hi[b]) return false;  // decided before search on the host
    }
    for (uint32_t k = 0; k < ncon; ++k) {
        const uint32_t w = cons[k];
        const uint32_t rel = w & 7u, lr = (w >> 3) & 0x3FFFu, rr = w >> 17;
        // lhs onto slot 0, rhs onto slot 1, d = r - l into slot 2
        if (!build_side(S, code, lr, 0, lit, pmap) || !build_side(S, code, rr, 1, lit, pmap)) return false;
        if (STK < 3) return false;
        PV L = stk(S, 0), R = stk(S, 1), D = stk(S, 2);
        D.n = 0;
        if (!plin(R, 1, L, -1, D)) return false;
        int lv = -1, rv = -1, def = -1;
        if (bare_var(L, lv)) def = lv;
        else if (bare_var(R, rv)) def = rv;
        bool ok;
        switch (rel) {
            case REL_LT: ok = add_con(S, D, 1, -1, false, -1); break;
            case REL_LE: ok = add_con(S, D, 1, 0, false, -1); break;
            case REL_EQ: ok = add_con(S, D, 1, 0, true, def); break;
            case REL_GE: ok = add_con(S, D, -1, 0, false, -1); break;
            default: ok = add_con(S, D, -1, -1, false, -1); break;
        }
        if (!ok) return false;
    }
    return true;
}

// substitute v := expr in every constraint (rebuilds the pool into the other
// buffer); ex[e] = expr^e for e = 1..maxe
OOB_HD SYM_NI inline bool subst_all(Store& S, int v, const PV& expr, PV* work3) {
    const int nb = S.cur ^ 1;
    int used = 0;
    PV pw = work3[0], tmp = work3[1], acc = work3[2];
    for (int j = 0; j < S.nc; ++j) {
        PV g = store_poly(S, j);
        PV o;
        o.k = S.key[nb] + used;
        o.c = S.coef[nb] + used;
        o.n = 0;
        o.cap = POOL - used;
        for (int i = 0; i < g.n; ++i) {
            const int n = kcount(g.k[i], v);
            if (n == 0) {
                if (!pins(o, g.k[i], g.c[i])) return false;
                continue;
            }
            uint64_t rest = g.k[i];
            for (int r = 0; r < n; ++r) rest = kremove(rest, v);
            // acc = c * x^rest * expr^n
            acc.n = 0;
            if (!pins(acc, rest, g.c[i])) return false;
            for (int r = 0; r < n; ++r) {
                tmp.n = 0;
                if (!pmuladd(acc, expr, 1, tmp) || !pcopy(tmp, acc)) return false;
            }
            for (int t = 0; t < acc.n; ++t)
                if (!pins(o, acc.k[t], acc.c[t])) return false;
        }
        S.off[j] = used;
        S.len[j] = o.n;
        used += o.n;
    }
    (void)pw;
    S.cur = nb;
    S.used = used;
    return true;
}

OOB_HD inline void drop_con(Store& S, int j) {
    for (int i = j; i + 1 < S.nc; ++i) {
        S.off[i] = S.off[i + 1];
        S.len[i] = S.len[i + 1];
        S.is_eq[i] = S.is_eq[i + 1];
        S.def[i] = S.def[i + 1];
    }
    --S.nc;
}

// 2. equality elimination; remaining equalities become two inequalities;
// inequalities already true on the box are dropped
OOB_HD SYM_NI inline bool eliminate(Store& S, PV* w) {
    Box B{S.lo, S.hi, S.np};
    for (int guard = 0; guard < MAXC; ++guard) {
        int ej = -1, ev = -1;
        for (int j = 0; j < S.nc && ej < 0; ++j) {
            if (!S.is_eq[j]) continue;
            PV e = store_poly(S, j);
            // the defined variable first, then terms in key order
            for (int pass = 0; pass < 2 && ej < 0; ++pass)
                for (int i = 0; i < e.n && ej < 0; ++i) {
                    const uint64_t k = e.k[i];
                    if (!k || (k << 8)) continue;  // not a single variable
                    const int v = (int)(k >> 56) - 1;
                    if ((pass == 0) != (v == S.def[j])) continue;
                    if (e.c[i] != 1 && e.c[i] != -1) continue;
                    bool elsewhere = false;
                    for (int t = 0; t < e.n; ++t)
                        if (t != i && kcount(e.k[t], v)) elsewhere = true;
                    if (elsewhere) continue;
                    ej = j;
                    ev = v;
                }
        }
        if (ej < 0) break;
        PV e = store_poly(S, ej);
        // v = -(e - c*v) / c = -c * (e - c*v) for c = +-1
        PV ex = w[3];
        ex.n = 0;
        i128 c = 0;
        for (int i = 0; i < e.n; ++i) {
            if (e.k[i] == vkey(ev)) c = e.c[i];
        }
        for (int i = 0; i < e.n; ++i)
            if (e.k[i] != vkey(ev) && !pins(ex, e.k[i], -c * e.c[i])) return false;
        drop_con(S, ej);
        if (!subst_all(S, ev, ex, w)) return false;
        // v's domain as constraints: expr - lo >= 0, hi - expr >= 0 (unless
        // they hold on the whole box)
        i128 elo, ehi;
        const bool ev_ok = peval(ex, B, elo, ehi);
        const bool use_lo = !ev_ok || elo < S.lo[ev], use_hi = !ev_ok || ehi > S.hi[ev];
        if (use_lo && !add_con(S, ex, 1, -S.lo[ev], false, -1)) return false;
        if (use_hi && !add_con(S, ex, -1, S.hi[ev], false, -1)) return false;
        if ((use_lo || use_hi) && S.nelim < MAXC) {
            S.elim_v[S.nelim] = (int16_t)ev;
            S.elim_flags[S.nelim] = (int8_t)((use_lo ? 1 : 0) | (use_hi ? 2 : 0));
            S.elim_lo[S.nelim] = S.lo[ev];
            S.elim_hi[S.nelim] = S.hi[ev];
            ++S.nelim;
        } else if (use_lo || use_hi) {
            return false;
        }
    }
    // remaining equalities -> e >= 0 and -e >= 0
    const int nc0 = S.nc;
    for (int j = 0; j < nc0; ++j) {
        if (!S.is_eq[j]) continue;
        S.is_eq[j] = 0;
        PV e = store_poly(S, j);
        PV cp = w[3];
        if (!pcopy(e, cp)) return false;
        if (!add_con(S, cp, -1, 0, false, -1)) return false;
    }
    // drop inequalities that hold on the whole box (and empty ones)
    for (int j = 0; j < S.nc;) {
        PV g = store_poly(S, j);
        i128 lo, hi;
        if (g.n == 0 || (peval(g, B, lo, hi) && lo >= 0)) drop_con(S, j);
        else ++j;
    }
    return true;
}

// 3. bound propagation; R_REFUTED on an empty box
OOB_HD SYM_NI inline int tighten(Store& S, PV* w) {
    Box B{S.lo, S.hi, S.np};
    for (int r = 0; r < ROUNDS; ++r) {
        bool changed = false;
        for (int j = 0; j < S.nc; ++j) {
            PV g = store_poly(S, j);
            for (int v = 0; v < S.nv; ++v) {
                PV K = w[1], s = w[0];
                if (!pcoef(g, v, 0, S.np, K, s)) continue;
                i128 klo, khi, slo, shi;
                if (!peval(K, B, klo, khi) || klo != khi || klo == 0) continue;
                if (!peval(s, B, slo, shi)) continue;
                const i128 k = klo;
                if (k > 0) {
                    const i128 nlo = -fdiv(shi, k);  // ceil(-shi / k)
                    if (nlo > S.lo[v]) S.lo[v] = nlo, changed = true;
                } else {
                    const i128 nhi = fdiv(shi, -k);
                    if (nhi < S.hi[v]) S.hi[v] = nhi, changed = true;
                }
                if (S.lo[v] > S.hi[v]) return R_REFUTED;
            }
        }
        if (!changed) break;
    }
    for (int j = 0; j < S.nc; ++j) {
        PV g = store_poly(S, j);
        i128 lo, hi;
        if (peval(g, B, lo, hi) && hi < 0) return R_REFUTED;
    }
    return R_CONTINUE;
}

// a/ka < b/kb for ka, kb > 0 (exact when the products fit, else double)
OOB_HD inline bool score_lt(i128 a, i128 ka, i128 b, i128 kb) {
    i128 x, y;
    if (smul(a, kb, x) && smul(b, ka, y)) return x < y;
    return (double)a / (double)ka < (double)b / (double)kb;
}

// 4. greedy elimination from target t; true = contradiction derived.  With
// `rec` (certificate compilation, host) the chosen moves are recorded: the
// constraint index and the multiplier polynomial of every step.
struct Moves {
    int n;
    int j[DEPTH];
    i128 mc[DEPTH][MAXT];  // multipliers
    uint64_t mk[DEPTH][MAXT];
    int mn[DEPTH];
    i128 kc[DEPTH][MAXT];  // the positive factor of the target at each step
    uint64_t kk[DEPTH][MAXT];
    int kn[DEPTH];
    i128 fc[MAXT];         // the final polynomial (upper bound < 0)
    uint64_t fk[MAXT];
    int fn;
};
OOB_HD SYM_NI inline bool greedy_target(Store& S, int t, LaneWork& W, Moves* rec = nullptr) {
    Box B{S.lo, S.hi, S.np};
    PV P = work(W, 0), best = work(W, 1), cand = work(W, 2), A = work(W, 3), Sx = work(W, 4), M = work(W, 5);
    PV K = work(W, 6), T = work(W, 7);
    PV src = store_poly(S, t);
    if (!pcopy(src, P)) return false;
    uint64_t used = 1ull << t;
    if (rec) rec->n = 0;
    for (int step = 0;; ++step) {
        i128 lo, hi;
        if (peval(P, B, lo, hi) && hi < 0) {
            if (rec) {
                rec->fn = P.n;
                for (int i = 0; i < P.n; ++i) rec->fk[i] = P.k[i], rec->fc[i] = P.c[i];
            }
            return true;
        }
        if (step == DEPTH) return false;
        bool have = false;
        i128 best_ub = 0, best_k = 1;
        int best_j = -1, best_v = -1, best_want = 0;
        // distinct variables of P, ascending (parameters are not eliminated)
        for (int v = S.np; v < S.nv; ++v) {
            bool has = false;
            for (int i = 0; i < P.n && !has; ++i) has = kcount(P.k[i], v) != 0;
            if (!has) continue;
            if (!psplit(P, v, A, Sx)) continue;
            i128 alo, ahi;
            if (!peval(A, B, alo, ahi)) continue;
            int want;
            if (alo >= 0) want = -1;
            else if (ahi <= 0) want = 1;
            else continue;
            if (alo == 0 && ahi == 0) continue;
            for (int j = 0; j < S.nc; ++j) {
                if (used >> j & 1ull) continue;
                PV g = store_poly(S, j);
                // g = K*v + s, K a (parametric) constant of the wanted sign
                if (!pcoef(g, v, 0, S.np, K, Sx)) continue;
                i128 klo, khi;
                if (!peval(K, B, klo, khi) || klo != khi || klo == 0) continue;
                if ((klo > 0) != (want > 0)) continue;
                const i128 kk = iabs(klo);
                // cand = |K|*P + mult*g, mult = A (want < 0) or -A
                M.n = 0;
                T.n = 0;
                if (!pmuladd(A, g, want < 0 ? 1 : -1, M)) continue;
                if (!pmuladd(K, P, klo > 0 ? 1 : -1, T)) continue;
                if (!plin(T, 1, M, 1, cand)) continue;
                i128 clo, chi;
                if (!peval(cand, B, clo, chi)) continue;
                if (!have || score_lt(chi, kk, best_ub, best_k)) {
                    have = true;
                    best_ub = chi;
                    best_k = kk;
                    best_j = j;
                    best_v = v;
                    best_want = want;
                    pcopy(cand, best);
                }
            }
        }
        if (!have) return false;
        if (rec) {
            const int m = rec->n++;
            rec->j[m] = best_j;
            psplit(P, best_v, A, Sx);
            rec->mn[m] = A.n;
            for (int i = 0; i < A.n; ++i) {
                rec->mk[m][i] = A.k[i];
                rec->mc[m][i] = best_want < 0 ? A.c[i] : -A.c[i];
            }
            PV g = store_poly(S, best_j);
            pcoef(g, best_v, 0, S.np, K, Sx);
            i128 klo, khi;
            peval(K, B, klo, khi);
            rec->kn[m] = K.n;
            for (int i = 0; i < K.n; ++i) {
                rec->kk[m][i] = K.k[i];
                rec->kc[m][i] = klo > 0 ? K.c[i] : -K.c[i];
            }
        }
        pcopy(best, P);
        used |= 1ull << best_j;
    }
}

// lane 0: steps 1-3 (R_REFUTED / R_UNKNOWN / R_CONTINUE)
template <typename GetDom, typename GetLit>
OOB_HD inline int prepare(Store& S, LaneWork& W, const uint32_t* cons, const uint32_t* code, uint32_t nv,
                          uint32_t ncon, GetDom dom, GetLit lit) {
    if (!build(S, cons, code, nv, ncon, dom, lit)) return R_UNKNOWN;
    PV w[4] = {work(W, 0), work(W, 1), work(W, 2), work(W, 3)};
    if (!eliminate(S, w)) return R_UNKNOWN;
    if (S.nc > 64) return R_UNKNOWN;  // the search's used-set is one 64-bit word
    return tighten(S, w);
}

// host / single-thread form of the whole prover
template <typename GetDom, typename GetLit>
OOB_HD inline bool refute_serial(Store& S, LaneWork& W, const uint32_t* cons, const uint32_t* code, uint32_t nv,
                                 uint32_t ncon, GetDom dom, GetLit lit) {
    const int r = prepare(S, W, cons, code, nv, ncon, dom, lit);
    if (r != R_CONTINUE) return r == R_REFUTED;
    for (int t = 0; t < S.nc; ++t)
        if (greedy_target(S, t, W)) return true;
    return false;
}

}  // namespace sym
}  // namespace oob
