// oob_oracle.cpp -- CPU restatement of the reference solver, for TESTS ONLY.
//
// TEST INFRASTRUCTURE.  This file is the parity checker and the CPU baseline
// ("port") of the B200 engine.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it.  The product
// path (paper_2601_21552_b200) never links, loads or calls it.
//
// It restates /root/reference/pkg/src/scuba_mini/solver.py function by
// function, deliberately in the reference's own shape (recursive evaluation,
// recursive narrowing, recursive DFS with a copied environment per child), so
// that it stays an independent check of the GPU engine, whose structure is
// different (postfix segments, explicit stacks, trail-based backtracking,
// lane-interleaved scratch).
//
// Pinned against the real reference: the tests/golden JSONL files hold the
// Python reference's verdict, first model, DFS node count and propagation pass
// count for the corpus queries, the reference's own randomized test systems,
// crafted edge cases and the synthetic streams (tools/golden.py);
// tests/test_oracle.py checks this file reproduces all four for every record.
//
// Arithmetic: Python ints are unbounded.  Each query runs first on a checked
// __int128; if any operation would overflow, the query is re-run on a
// sign-magnitude multi-limb integer (512-bit capacity, itself checked).  A
// query beyond that gets OOB_ERROR -- never a silently wrong answer.
#include <pthread.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <vector>

#include "../include/scuba_oob.h"

namespace {

using i128 = __int128;
thread_local bool g_ovf = false;  // sticky overflow flag of the current query

// ---------------------------------------------------------------- number types
struct CI {  // checked int128
    i128 v;
    CI(long long x = 0) : v(x) {}
    static CI of(i128 x) { CI c; c.v = x; return c; }
    i128 to128() const { return v; }
};
inline CI operator+(CI a, CI b) { i128 r; if (__builtin_add_overflow(a.v, b.v, &r)) g_ovf = true; return CI::of(r); }
inline CI operator-(CI a, CI b) { i128 r; if (__builtin_sub_overflow(a.v, b.v, &r)) g_ovf = true; return CI::of(r); }
inline CI operator*(CI a, CI b) { i128 r; if (__builtin_mul_overflow(a.v, b.v, &r)) g_ovf = true; return CI::of(r); }
inline CI operator-(CI a) { return CI(0) - a; }
inline bool operator<(CI a, CI b) { return a.v < b.v; }
inline bool operator==(CI a, CI b) { return a.v == b.v; }
// truncating quotient / remainder of magnitudes with signs (C semantics)
inline CI cdiv(CI a, CI b) { return CI::of(a.v / b.v); }
inline CI cmod(CI a, CI b) { return CI::of(a.v % b.v); }

struct Big {  // sign-magnitude, 32-bit limbs, fixed 512-bit capacity
    static const int L = 16;
    bool neg = false;
    int n = 0;  // used limbs (normalized: no leading zero limb)
    uint32_t m[L] = {};
    Big(long long x = 0) { set128(x); }
    static Big of(i128 x) { Big b; b.set128(x); return b; }
    void set128(i128 x) {
        neg = x < 0;
        unsigned __int128 u = neg ? (unsigned __int128)(-(x + 1)) + 1 : (unsigned __int128)x;
        n = 0;
        std::memset(m, 0, sizeof(m));
        while (u) { m[n++] = (uint32_t)u; u >>= 32; }
    }
    void norm() { while (n > 0 && m[n - 1] == 0) n--; if (n == 0) neg = false; }
    i128 to128() const {
        unsigned __int128 u = 0;
        for (int i = std::min(n, 4) - 1; i >= 0; i--) u = (u << 32) | m[i];
        if (n > 4) g_ovf = true;
        return neg ? -(i128)u : (i128)u;
    }
};
int cmp_mag(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; i--)
        if (a.m[i] != b.m[i]) return a.m[i] < b.m[i] ? -1 : 1;
    return 0;
}
Big add_mag(const Big& a, const Big& b) {
    Big r;
    uint64_t c = 0;
    int n = std::max(a.n, b.n);
    for (int i = 0; i < n || c; i++) {
        if (i >= Big::L) { g_ovf = true; break; }
        c += (uint64_t)(i < a.n ? a.m[i] : 0) + (i < b.n ? b.m[i] : 0);
        r.m[i] = (uint32_t)c;
        c >>= 32;
        r.n = i + 1;
    }
    r.norm();
    return r;
}
Big sub_mag(const Big& a, const Big& b) {  // |a| >= |b|
    Big r;
    int64_t br = 0;
    for (int i = 0; i < a.n; i++) {
        int64_t d = (int64_t)a.m[i] - (i < b.n ? b.m[i] : 0) - br;
        br = d < 0;
        r.m[i] = (uint32_t)(d + (br << 32));
    }
    r.n = a.n;
    r.norm();
    return r;
}
Big operator+(const Big& a, const Big& b) {
    if (a.neg == b.neg) { Big r = add_mag(a, b); r.neg = a.neg && r.n; return r; }
    int c = cmp_mag(a, b);
    if (c == 0) return Big(0);
    Big r = c > 0 ? sub_mag(a, b) : sub_mag(b, a);
    r.neg = c > 0 ? a.neg : b.neg;
    r.norm();
    return r;
}
Big operator-(const Big& a) { Big r = a; if (r.n) r.neg = !r.neg; return r; }
Big operator-(const Big& a, const Big& b) { return a + (-b); }
Big operator*(const Big& a, const Big& b) {
    Big r;
    if (!a.n || !b.n) return r;
    if (a.n + b.n > Big::L + 1) { g_ovf = true; return r; }
    uint64_t t[2 * Big::L + 2] = {};
    for (int i = 0; i < a.n; i++) {
        uint64_t c = 0;
        for (int j = 0; j < b.n; j++) {
            uint64_t x = t[i + j] + (uint64_t)a.m[i] * b.m[j] + c;
            t[i + j] = (uint32_t)x;
            c = x >> 32;
        }
        t[i + b.n] += c;
    }
    int n = a.n + b.n;
    for (int i = Big::L; i < n; i++) if (t[i]) g_ovf = true;
    r.n = std::min(n, Big::L);
    for (int i = 0; i < r.n; i++) r.m[i] = (uint32_t)t[i];
    r.neg = a.neg != b.neg;
    r.norm();
    return r;
}
void divmod_mag(const Big& a, const Big& b, Big& q, Big& r) {  // bitwise long division
    q = Big(0);
    r = Big(0);
    for (int bit = a.n * 32 - 1; bit >= 0; bit--) {
        // r = 2r + bit
        uint32_t carry = (a.m[bit / 32] >> (bit % 32)) & 1;
        for (int i = 0; i < Big::L; i++) {
            uint32_t nc = r.m[i] >> 31;
            r.m[i] = (r.m[i] << 1) | carry;
            carry = nc;
        }
        r.n = Big::L;
        r.norm();
        if (cmp_mag(r, b) >= 0) {
            r = sub_mag(r, b);
            q.m[bit / 32] |= 1u << (bit % 32);
        }
    }
    q.n = Big::L;
    q.norm();
}
Big cdiv(const Big& a, const Big& b) {
    Big q, r;
    divmod_mag(a, b, q, r);
    q.neg = (a.neg != b.neg) && q.n;
    return q;
}
Big cmod(const Big& a, const Big& b) {
    Big q, r;
    divmod_mag(a, b, q, r);
    r.neg = a.neg && r.n;
    return r;
}
bool operator<(const Big& a, const Big& b) {
    if (a.neg != b.neg) return a.neg;
    int c = cmp_mag(a, b);
    return a.neg ? c > 0 : c < 0;
}
bool operator==(const Big& a, const Big& b) { return a.neg == b.neg && cmp_mag(a, b) == 0; }

template <class N> bool operator>(const N& a, const N& b) { return b < a; }
template <class N> bool operator<=(const N& a, const N& b) { return !(b < a); }
template <class N> bool operator>=(const N& a, const N& b) { return !(a < b); }
template <class N> bool operator!=(const N& a, const N& b) { return !(a == b); }
template <class N> N nmin(const N& a, const N& b) { return a < b ? a : b; }
template <class N> N nmax(const N& a, const N& b) { return b < a ? a : b; }

// tdiv / tmod: solver.py:94-102 (C truncation) -- cdiv/cmod are exactly that
// Python floor division a // b
template <class N> N fdiv(const N& a, const N& b) {
    N q = cdiv(a, b), r = cmod(a, b);
    if (r != N(0) && ((r < N(0)) != (b < N(0)))) q = q - N(1);
    return q;
}
// _ceil_div: solver.py:105-106  -((-a) // b)
template <class N> N ceil_div(const N& a, const N& b) { return -fdiv(-a, b); }

double now_s() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
i128 from_w(oob_i128 w) { return (i128)(((unsigned __int128)(uint64_t)w.hi << 64) | w.lo); }
oob_i128 to_w(i128 v) { oob_i128 w; w.lo = (uint64_t)v; w.hi = (int64_t)(v >> 64); return w; }

const int LIT_ONE = -1;      // node id of the Lit(1) of side constraints
const int PASS_CAP = 10000;  // _PASS_CAP, solver.py:24

// ------------------------------------------------------------- query view
struct View {
    int nv = 0;
    const uint8_t* op;
    const int32_t* na;
    const int32_t* nb;
    const oob_i128* lit;
    std::vector<uint8_t> rel;
    std::vector<int32_t> lhs, rhs;
    int nuser = 0;
    int opc(int32_t n) const { return n == LIT_ONE ? (int)OOB_NODE_LIT : (int)op[n]; }
    i128 litv(int32_t n) const { return n == LIT_ONE ? 1 : from_w(lit[na[n]]); }
    bool same(int32_t x, int32_t y) const {  // dataclass equality
        if (x == y) return true;
        if (opc(x) != opc(y)) return false;
        if (opc(x) == OOB_NODE_LIT) return litv(x) == litv(y);
        if (opc(x) == OOB_NODE_VAR) return na[x] == na[y];
        return same(na[x], na[y]) && same(nb[x], nb[y]);
    }
    // _collect_divisors: solver.py:334-342
    void collect(int32_t e, std::vector<int32_t>& out) const {
        int o = opc(e);
        if (o < OOB_NODE_ADD) return;
        if (o == OOB_NODE_DIV || o == OOB_NODE_MOD) {
            int32_t R = nb[e];
            if (!(opc(R) == OOB_NODE_LIT && litv(R) >= 1)) {
                bool seen = false;
                for (int32_t d : out) seen = seen || same(d, R);
                if (!seen) out.push_back(R);
            }
        }
        collect(na[e], out);
        collect(nb[e], out);
    }
};

View make_view(const oob_batch* b, int64_t q, bool with_side) {
    View v;
    int64_t vb = b->var_begin[q], cb = b->con_begin[q], nb = b->node_begin[q], lb = b->lit_begin[q];
    v.nv = (int)(b->var_begin[q + 1] - vb);
    v.nuser = (int)(b->con_begin[q + 1] - cb);
    v.op = b->node_op + nb;
    v.na = b->node_a + nb;
    v.nb = b->node_b + nb;
    v.lit = b->lits + lb;
    for (int k = 0; k < v.nuser; k++) {
        v.rel.push_back(b->con_rel[cb + k]);
        v.lhs.push_back(b->con_lhs[cb + k]);
        v.rhs.push_back(b->con_rhs[cb + k]);
    }
    if (with_side) {  // divisor_side_constraints: solver.py:345-357
        std::vector<int32_t> divs;
        for (int k = 0; k < v.nuser; k++) {
            v.collect(v.lhs[k], divs);
            v.collect(v.rhs[k], divs);
        }
        for (int32_t d : divs) {
            if (v.opc(d) == OOB_NODE_LIT) continue;
            v.rel.push_back(OOB_REL_GE);
            v.lhs.push_back(d);
            v.rhs.push_back(LIT_ONE);
        }
    }
    return v;
}

// -------------------------------------------------------------- the solver
template <class N>
struct Solver {
    struct Iv { N lo, hi; };
    const View& c;
    double deadline = 1e300;
    int64_t node_budget = 0;
    int64_t nodes = 0, passes = 0;
    bool timed_out = false;
    explicit Solver(const View& v) : c(v) {}
    N INF() const { return N(1000000000000000000LL); }  // _INF, solver.py:23
    N lit(int32_t e) const { return N::of(c.litv(e)); }

    // _eval_iv: solver.py:112-149
    bool eval_iv(int32_t e, const std::vector<Iv>& env, Iv& out) {
        int op = c.opc(e);
        if (op == OOB_NODE_LIT) { out.lo = out.hi = lit(e); return true; }              // :114-115
        if (op == OOB_NODE_VAR) {                                                        // :116-118
            const Iv& d = env[c.na[e]];
            if (d.lo > d.hi) return false;
            out = d;
            return true;
        }
        Iv l, r;                                                                         // :119-122
        if (!eval_iv(c.na[e], env, l) || !eval_iv(c.nb[e], env, r)) return false;
        switch (op) {
        case OOB_NODE_ADD: out.lo = l.lo + r.lo; out.hi = l.hi + r.hi; return true;      // :126-127
        case OOB_NODE_SUB: out.lo = l.lo - r.hi; out.hi = l.hi - r.lo; return true;      // :128-129
        case OOB_NODE_MUL: {                                                             // :130-132
            N k[4] = {l.lo * r.lo, l.lo * r.hi, l.hi * r.lo, l.hi * r.hi};
            out.lo = nmin(nmin(k[0], k[1]), nmin(k[2], k[3]));
            out.hi = nmax(nmax(k[0], k[1]), nmax(k[2], k[3]));
            return true;
        }
        default: break;
        }
        N d0 = nmax(r.lo, N(1)), d1 = r.hi;                                               // :136-138
        if (d0 > d1) return false;
        if (op == OOB_NODE_DIV) {                                                        // :139-141
            N k[4] = {cdiv(l.lo, d0), cdiv(l.lo, d1), cdiv(l.hi, d0), cdiv(l.hi, d1)};
            out.lo = nmin(nmin(k[0], k[1]), nmin(k[2], k[3]));
            out.hi = nmax(nmax(k[0], k[1]), nmax(k[2], k[3]));
            return true;
        }
        N m = d1 - N(1);                                                                 // :142-148
        if (l.lo >= N(0)) { out.lo = N(0); out.hi = nmin(l.hi, m); return true; }
        if (l.hi <= N(0)) { out.lo = nmax(l.lo, -m); out.hi = N(0); return true; }
        out.lo = nmax(l.lo, -m);
        out.hi = nmin(l.hi, m);
        return true;
    }

    // _Narrower.narrow: solver.py:159-226
    bool narrow(int32_t e, N t0, N t1, std::vector<Iv>& env, bool& changed) {
        if (t0 > t1) return false;                                                       // :161-162
        int op = c.opc(e);
        if (op == OOB_NODE_LIT) { N v = lit(e); return t0 <= v && v <= t1; }             // :163-164
        if (op == OOB_NODE_VAR) {                                                        // :165-173
            Iv& d = env[c.na[e]];
            N nlo = nmax(d.lo, t0), nhi = nmin(d.hi, t1);
            if (nlo > nhi) return false;
            if (nlo != d.lo || nhi != d.hi) { d.lo = nlo; d.hi = nhi; changed = true; }
            return true;
        }
        Iv l, r;                                                                         // :174-177
        if (!eval_iv(c.na[e], env, l) || !eval_iv(c.nb[e], env, r)) return false;
        int32_t L = c.na[e], R = c.nb[e];
        switch (op) {
        case OOB_NODE_ADD:                                                               // :181-185
            return narrow(L, t0 - r.hi, t1 - r.lo, env, changed) &&
                   narrow(R, t0 - l.hi, t1 - l.lo, env, changed);
        case OOB_NODE_SUB:                                                               // :186-190
            return narrow(L, t0 + r.lo, t1 + r.hi, env, changed) &&
                   narrow(R, l.lo - t1, l.hi - t0, env, changed);
        case OOB_NODE_MUL: {                                                             // :191-216
            if (l.lo < N(0) || r.lo < N(0)) return true;
            if (t1 < N(0)) return false;
            N t0n = nmax(t0, N(0));
            int32_t child[2] = {L, R};
            N olo[2] = {r.lo, l.lo}, ohi[2] = {r.hi, l.hi};
            for (int k = 0; k < 2; k++) {
                N lo_req = -INF(), hi_req = INF();
                if (t0n > N(0)) {
                    if (ohi[k] == N(0)) return false;
                    lo_req = ceil_div(t0n, ohi[k]);
                }
                if (olo[k] > N(0)) hi_req = fdiv(t1, olo[k]);
                if (!narrow(child[k], lo_req, hi_req, env, changed)) return false;
            }
            return true;
        }
        case OOB_NODE_DIV:                                                               // :217-223
            if (c.opc(R) == OOB_NODE_LIT && lit(R) >= N(1)) {
                N cc = lit(R);
                N lo_req = t0 > N(0) ? t0 * cc : t0 * cc - (cc - N(1));
                N hi_req = t1 >= N(0) ? t1 * cc + (cc - N(1)) : t1 * cc;
                return narrow(L, lo_req, hi_req, env, changed);
            }
            return true;
        default:                                                                         // % :224-225
            return true;
        }
    }

    // _propagate_constraint: solver.py:229-261
    bool propagate_constraint(size_t k, std::vector<Iv>& env, bool& changed) {
        Iv l, r;
        if (!eval_iv(c.lhs[k], env, l) || !eval_iv(c.rhs[k], env, r)) return false;
        int32_t A = c.lhs[k], B = c.rhs[k];
        switch (c.rel[k]) {
        case OOB_REL_LT:
            return narrow(A, -INF(), r.hi - N(1), env, changed) && narrow(B, l.lo + N(1), INF(), env, changed);
        case OOB_REL_LE:
            return narrow(A, -INF(), r.hi, env, changed) && narrow(B, l.lo, INF(), env, changed);
        case OOB_REL_EQ: {
            N lo = nmax(l.lo, r.lo), hi = nmin(l.hi, r.hi);
            return narrow(A, lo, hi, env, changed) && narrow(B, lo, hi, env, changed);
        }
        case OOB_REL_GE:
            return narrow(A, r.lo, INF(), env, changed) && narrow(B, -INF(), l.hi, env, changed);
        default:
            return narrow(A, r.lo + N(1), INF(), env, changed) && narrow(B, -INF(), l.hi - N(1), env, changed);
        }
    }

    // propagate: solver.py:264-280 (env updated in place)
    bool propagate(std::vector<Iv>& env, bool check_deadline) {
        for (int pass = 0; pass < PASS_CAP; pass++) {
            if (check_deadline && now_s() > deadline) { timed_out = true; return false; }
            passes++;
            bool changed = false;
            for (size_t k = 0; k < c.rel.size(); k++)
                if (!propagate_constraint(k, env, changed)) return false;
            if (!changed) break;
        }
        return true;
    }

    // _eval_exact / check_model: solver.py:286-328
    bool eval_exact(int32_t e, const std::vector<N>& model, N& out) {
        int op = c.opc(e);
        if (op == OOB_NODE_LIT) { out = lit(e); return true; }
        if (op == OOB_NODE_VAR) { out = model[c.na[e]]; return true; }
        N a, b;
        if (!eval_exact(c.na[e], model, a) || !eval_exact(c.nb[e], model, b)) return false;
        switch (op) {
        case OOB_NODE_ADD: out = a + b; return true;
        case OOB_NODE_SUB: out = a - b; return true;
        case OOB_NODE_MUL: out = a * b; return true;
        default: break;
        }
        if (b == N(0)) return false;                                                     // :301-302
        out = op == OOB_NODE_DIV ? cdiv(a, b) : cmod(a, b);
        return true;
    }
    bool check_model(const std::vector<N>& model) {
        for (size_t k = 0; k < c.rel.size(); k++) {
            N a, b;
            if (!eval_exact(c.lhs[k], model, a) || !eval_exact(c.rhs[k], model, b)) return false;
            bool ok;
            switch (c.rel[k]) {
            case OOB_REL_LT: ok = a < b; break;
            case OOB_REL_LE: ok = a <= b; break;
            case OOB_REL_EQ: ok = a == b; break;
            case OOB_REL_GE: ok = a >= b; break;
            default: ok = a > b; break;
            }
            if (!ok) return false;
        }
        return true;
    }

    // _search: solver.py:385-416 (recursive, child = copy of the narrowed env)
    bool search(std::vector<Iv> env, std::vector<N>& model) {
        if (now_s() > deadline || (node_budget > 0 && nodes >= node_budget)) {        // :391-392
            timed_out = true;
            return false;
        }
        nodes++;
        if (!propagate(env, true) || g_ovf) return false;                               // :393-395
        int pick = -1;                                                                   // :397-404
        N pick_size(0);
        for (int v = 0; v < c.nv; v++) {
            if (env[v].lo < env[v].hi) {
                N size = env[v].hi - env[v].lo + N(1);
                if (pick < 0 || size < pick_size) { pick = v; pick_size = size; }
            }
        }
        if (pick < 0) {                                                                  // :405-407
            model.assign(c.nv, N(0));
            for (int v = 0; v < c.nv; v++) model[v] = env[v].lo;
            return check_model(model);
        }
        N lo = env[pick].lo, hi = env[pick].hi;                                          // :408-415
        N mid = fdiv(lo + hi, N(2));
        std::vector<Iv> child = env;
        child[pick].lo = lo;
        child[pick].hi = mid;
        if (search(child, model)) return true;
        if (timed_out || g_ovf) return false;
        child = env;
        child[pick].lo = mid + N(1);
        child[pick].hi = hi;
        return search(child, model);
    }
};

// solve: solver.py:363-382
template <class N>
int8_t solve_with(const oob_batch* b, int64_t q, double start, double timeout_s, int64_t budget,
                  oob_result* out) {
    View v = make_view(b, q, true);
    Solver<N> s(v);
    s.deadline = start + timeout_s;
    s.node_budget = budget;
    int64_t vb = b->var_begin[q];
    std::vector<typename Solver<N>::Iv> env(v.nv);
    for (int i = 0; i < v.nv; i++) {
        env[i].lo = N::of(from_w(b->var_lo[vb + i]));
        env[i].hi = N::of(from_w(b->var_hi[vb + i]));
    }
    std::vector<N> model;
    bool found = s.search(env, model);
    int8_t verdict = g_ovf ? OOB_ERROR : s.timed_out ? OOB_TIMEOUT : found ? OOB_SAT : OOB_UNSAT;
    if (verdict == OOB_SAT && out->model)
        for (int i = 0; i < v.nv; i++) out->model[vb + i] = to_w(model[i].to128());
    if (out->nodes) out->nodes[q] = s.nodes;
    if (out->passes) out->passes[q] = s.passes;
    return verdict;
}

void solve_one(const oob_batch* b, int64_t q, double timeout_s, int64_t budget, oob_result* out) {
    double start = now_s();
    int64_t vb = b->var_begin[q], ve = b->var_begin[q + 1];
    bool empty = false;
    for (int64_t i = vb; i < ve; i++) empty = empty || from_w(b->var_lo[i]) > from_w(b->var_hi[i]);
    int8_t verdict;
    if (empty) {
        verdict = OOB_UNSAT;                               // :374-375
        if (out->nodes) out->nodes[q] = 0;
        if (out->passes) out->passes[q] = 0;
    } else if (!(timeout_s > 0)) {
        verdict = OOB_TIMEOUT;                             // deadline already passed at :391
        if (out->nodes) out->nodes[q] = 0;
        if (out->passes) out->passes[q] = 0;
    } else {
        g_ovf = false;
        verdict = solve_with<CI>(b, q, start, timeout_s, budget, out);
        if (verdict == OOB_ERROR) {                        // int128 overflowed: exact wide re-run
            g_ovf = false;
            verdict = solve_with<Big>(b, q, start, timeout_s, budget, out);
        }
    }
    out->verdict[q] = verdict;
    if (out->elapsed_s) out->elapsed_s[q] = now_s() - start;
}

struct Job {
    const oob_batch* b;
    double timeout_s;
    int64_t budget;
    oob_result* out;
    std::atomic<long long> next{0};
};

void* worker(void* arg) {
    Job* j = (Job*)arg;
    for (;;) {
        long long q = j->next.fetch_add(1);
        if (q >= j->b->n_queries) break;
        solve_one(j->b, q, j->timeout_s, j->budget, j->out);
    }
    return nullptr;
}

template <class N>
int8_t propagate_with(const oob_batch* b, int64_t q, oob_i128* out_lo, oob_i128* out_hi) {
    View v = make_view(b, q, false);
    Solver<N> s(v);
    int64_t vb = b->var_begin[q];
    std::vector<typename Solver<N>::Iv> env(v.nv);
    for (int i = 0; i < v.nv; i++) {
        env[i].lo = N::of(from_w(b->var_lo[vb + i]));
        env[i].hi = N::of(from_w(b->var_hi[vb + i]));
    }
    bool ok = s.propagate(env, false);
    for (int i = 0; i < v.nv; i++) {
        out_lo[vb + i] = to_w(env[i].lo.to128());
        out_hi[vb + i] = to_w(env[i].hi.to128());
    }
    return g_ovf ? -1 : (int8_t)ok;
}

template <class N>
int8_t check_with(const oob_batch* b, int64_t q, const oob_i128* model) {
    View v = make_view(b, q, false);
    Solver<N> s(v);
    int64_t vb = b->var_begin[q];
    std::vector<N> m(v.nv);
    for (int i = 0; i < v.nv; i++) m[i] = N::of(from_w(model[vb + i]));
    bool ok = s.check_model(m);
    return g_ovf ? -1 : (int8_t)ok;
}

}  // namespace

extern "C" {

int oracle_solve_batch(const oob_batch* b, double timeout_s, int64_t node_budget, oob_result* out,
                       int n_threads) {
    Job j;
    j.b = b;
    j.timeout_s = timeout_s;
    j.budget = node_budget;
    j.out = out;
    if (n_threads <= 1) {
        worker(&j);
        return 0;
    }
    std::vector<pthread_t> th(n_threads);
    for (int i = 0; i < n_threads; i++) pthread_create(&th[i], nullptr, worker, &j);
    for (int i = 0; i < n_threads; i++) pthread_join(th[i], nullptr);
    return 0;
}

// propagate(domains, constraints) as the public API: no side constraints, no deadline
int oracle_propagate_batch(const oob_batch* b, oob_i128* out_lo, oob_i128* out_hi, int8_t* status) {
    for (int64_t q = 0; q < b->n_queries; q++) {
        g_ovf = false;
        status[q] = propagate_with<CI>(b, q, out_lo, out_hi);
        if (status[q] < 0) {
            g_ovf = false;
            status[q] = propagate_with<Big>(b, q, out_lo, out_hi);
        }
    }
    return 0;
}

int oracle_check_model_batch(const oob_batch* b, const oob_i128* model, int8_t* ok) {
    for (int64_t q = 0; q < b->n_queries; q++) {
        g_ovf = false;
        ok[q] = check_with<CI>(b, q, model);
        if (ok[q] < 0) {
            g_ovf = false;
            ok[q] = check_with<Big>(b, q, model);
        }
    }
    return 0;
}

int oracle_side_constraint_count(const oob_batch* b, int64_t* counts) {
    for (int64_t q = 0; q < b->n_queries; q++) {
        View v = make_view(b, q, true);
        counts[q] = (int64_t)v.rel.size() - v.nuser;
    }
    return 0;
}

}  // extern "C"
