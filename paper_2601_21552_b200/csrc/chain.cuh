// chain.cuh -- fast mode (OOB_F_FAST), warp-per-query kernels of the int64
// job's open own entries (after the certificate kernels, before the root
// kernel):
//   oob_enum_kernel   K3, on by default: exhaustive enumeration of declared
//                     boxes of at most SCUBA_OOB_ENUM_MAX points (bottom of
//                     this file);
//   oob_chain_kernel  opt-in (OOB_F_CHAIN): the reference's DFS with
//                     warp-parallel propagation, below.
//
// The exact emulation (engine.cuh) runs a query's propagation passes in ONE
// lane: a pass visits the constraints in order (solver.py:271-277), so a Sat
// query with a long propagation chain (C3: 11-15 DFS nodes, 200-400 passes)
// costs 10-20 us per pass of dependent single-lane work and bounds the step.
// Here the 32 lanes of a warp share one query: in a ROUND every lane applies
// its constraints (k = lane, lane + 32, ...) to the round's snapshot of the
// domains, and the narrowed domains are met (shared-memory atomicMax/Min on
// the bounds) into the next snapshot -- a Jacobi iteration of the reference's
// per-constraint narrowing operators f_c (_propagate_constraint, :229-261).
//
// Why the result is the reference's (the DFS tree -- node count, branching
// variables, first model -- is then the reference's too):
//  * each f_c is reductive and, for the entries admitted below, monotone in
//    the domains (forward intervals, narrowing targets and the contradiction
//    tests only tighten as domains shrink).  The one constant that can break
//    monotonicity is the `_INF` upper target of a product's operand when the
//    other operand's lower bound is 0 (:206-213): it is vacuous -- so the
//    rule is monotone -- when every product operand's upper bound is <= _INF
//    at the entry's declared domains (forward intervals only shrink below),
//    which is checked per entry before the search (else the entry is left to
//    the exact emulation);
//  * so the reference's Gauss-Seidel sweep and this Jacobi iteration both
//    descend to the greatest common fixpoint F below the node's domains, and
//    after i passes the sweep is at least as narrow as the iteration after i
//    rounds (induction with monotonicity).  If the iteration reaches F (a
//    round that changes nothing) or a contradiction within i <= _PASS_CAP
//    rounds, the reference's propagate() returned that same F / None within
//    its pass cap.  Otherwise the entry is left to the exact emulation.
// Nodes: the reference's; passes: the rounds of this kernel (fast mode
// reports the reference's node counts but not its pass counts for these).
//
// An entry whose search exceeds the node or depth budget is left untouched
// (resume word 0): the exact emulation then runs it from its root.
#pragma once
#include "engine.cuh"
#include "format.h"

namespace oob {
namespace chain {

constexpr int WARPS = 4;            // warps per block
constexpr uint32_t MAXV = 64;       // variables per query (more: left to the exact path)
constexpr uint32_t DEPTH = 64;      // DFS frames per warp (global scratch)
constexpr int OVN = 16;             // per-constraint overlay of narrowed variables
constexpr int VST = 36;             // forward-evaluation value stack (tree depth <= 32)
constexpr int NST = 40;             // narrowing stack
using ll = long long;
using A = Arith<ll>;

__device__ __forceinline__ uint32_t op_of(uint32_t w) { return w & 7u; }
__device__ __forceinline__ uint32_t arg_of(uint32_t w) { return w >> 3; }

struct Query {
    const uint32_t* cons;
    const uint32_t* code;
    const ll* lit;
    uint32_t nv, ncon, ncode;
    __device__ __forceinline__ uint32_t size_of(uint32_t i) const {
        const uint32_t w = __ldg(code + i);
        return op_of(w) >= NODE_ADD ? arg_of(w) : 1u;
    }
};

// the variables one lane's constraint narrowed so far (the reference mutates
// the environment in place inside a constraint, :165-173)
struct Overlay {
    uint32_t var[OVN];
    ll lo[OVN], hi[OVN];
    int n;
    bool full;
    __device__ __forceinline__ int find(uint32_t v) const {
        for (int e = 0; e < n; ++e)
            if (var[e] == v) return e;
        return -1;
    }
};

struct Ctx {
    const Query& q;
    const ll* cur_lo;  // round snapshot (shared memory)
    const ll* cur_hi;
    Overlay& ov;
    __device__ __forceinline__ void get(uint32_t v, ll& lo, ll& hi) const {
        const int e = ov.find(v);
        if (e >= 0) {
            lo = ov.lo[e];
            hi = ov.hi[e];
        } else {
            lo = cur_lo[v];
            hi = cur_hi[v];
        }
    }

    // _eval_iv over the postfix subtree rooted at `root` (:112-149)
    __device__ bool eval(uint32_t root, ll& out_lo, ll& out_hi) const {
        ll s_lo[VST], s_hi[VST];
        int sp = 0;
        const uint32_t start = root + 1 - q.size_of(root);
        for (uint32_t j = start; j <= root; ++j) {
            const uint32_t w = __ldg(q.code + j);
            const uint32_t op = op_of(w);
            ll lo, hi;
            if (op < NODE_ADD && sp == VST) {
                ov.full = true;  // deeper than the value stack: exact path
                return false;
            }
            if (op == NODE_LIT) {
                lo = hi = q.lit[arg_of(w)];
            } else if (op == NODE_VAR) {
                get(arg_of(w), lo, hi);
                if (lo > hi) return false;
            } else {
                const ll r0 = s_lo[sp - 1], r1 = s_hi[sp - 1];
                const ll l0 = s_lo[sp - 2], l1 = s_hi[sp - 2];
                sp -= 2;
                if (op == NODE_ADD) {
                    lo = l0 + r0;
                    hi = l1 + r1;
                } else if (op == NODE_SUB) {
                    lo = l0 - r1;
                    hi = l1 - r0;
                } else if (op == NODE_MUL) {
                    const ll k0 = l0 * r0, k1 = l0 * r1, k2 = l1 * r0, k3 = l1 * r1;
                    lo = A::mn(A::mn(k0, k1), A::mn(k2, k3));
                    hi = A::mx(A::mx(k0, k1), A::mx(k2, k3));
                } else {
                    const ll d0 = A::mx(r0, 1ll), d1 = r1;
                    if (d0 > d1) return false;
                    if (op == NODE_DIV) {
                        const ll k0 = l0 / d0, k1 = l0 / d1, k2 = l1 / d0, k3 = l1 / d1;
                        lo = A::mn(A::mn(k0, k1), A::mn(k2, k3));
                        hi = A::mx(A::mx(k0, k1), A::mx(k2, k3));
                    } else {  // NODE_MOD
                        const ll m = d1 - 1;
                        if (l0 >= 0) {
                            lo = 0;
                            hi = A::mn(l1, m);
                        } else if (l1 <= 0) {
                            lo = A::mx(l0, -m);
                            hi = 0;
                        } else {
                            lo = A::mx(l0, -m);
                            hi = A::mn(l1, m);
                        }
                    }
                }
            }
            s_lo[sp] = lo;
            s_hi[sp] = hi;
            ++sp;
        }
        out_lo = s_lo[0];
        out_hi = s_hi[0];
        return true;
    }

    // _Narrower.narrow (:159-226), pre-order with the children's targets
    // computed from their intervals before either is narrowed (the
    // reference's stale-sibling order: its `l`, `r` are evaluated on entry)
    __device__ bool narrow2(uint32_t n0, ll a0, ll b0, uint32_t n1, ll a1, ll b1) {
        uint32_t st_n[NST];
        ll st_a[NST], st_b[NST];
        int sp = 0;
        st_n[sp] = n1; st_a[sp] = a1; st_b[sp] = b1; ++sp;  // popped second
        st_n[sp] = n0; st_a[sp] = a0; st_b[sp] = b0; ++sp;
        while (sp > 0) {
            --sp;
            const uint32_t i = st_n[sp];
            const ll a = st_a[sp], b = st_b[sp];
            if (a > b) return false;                                   // :161-162
            const uint32_t w = __ldg(q.code + i);
            const uint32_t op = op_of(w);
            if (op == NODE_LIT) {                                      // :163-164
                const ll v = q.lit[arg_of(w)];
                if (!(a <= v && v <= b)) return false;
                continue;
            }
            if (op == NODE_VAR) {                                      // :165-173
                const uint32_t v = arg_of(w);
                ll lo, hi;
                get(v, lo, hi);
                const ll nlo = A::mx(lo, a), nhi = A::mn(hi, b);
                if (nlo > nhi) return false;
                if (nlo != lo || nhi != hi) {
                    int e = ov.find(v);
                    if (e < 0) {
                        if (ov.n == OVN) {
                            ov.full = true;
                            return false;
                        }
                        e = ov.n++;
                        ov.var[e] = v;
                    }
                    ov.lo[e] = nlo;
                    ov.hi[e] = nhi;
                }
                continue;
            }
            const uint32_t R = i - 1;                                  // :174-177
            const uint32_t L = R - q.size_of(R);
            ll l0, l1, r0, r1;
            if (!eval(L, l0, l1) || !eval(R, r0, r1)) return false;
            if (sp + 2 > NST) {
                ov.full = true;
                return false;
            }
            if (op == NODE_ADD) {                                      // :181-185
                st_n[sp] = R; st_a[sp] = a - l1; st_b[sp] = b - l0; ++sp;
                st_n[sp] = L; st_a[sp] = a - r1; st_b[sp] = b - r0; ++sp;
            } else if (op == NODE_SUB) {                               // :186-190
                st_n[sp] = R; st_a[sp] = l0 - b; st_b[sp] = l1 - a; ++sp;
                st_n[sp] = L; st_a[sp] = a + r0; st_b[sp] = b + r1; ++sp;
            } else if (op == NODE_MUL) {                               // :191-216
                if (l0 < 0 || r0 < 0) continue;
                if (b < 0) return false;
                const ll t0n = A::mx(a, 0ll);
                ll lo_l = -A::inf(), hi_l = A::inf(), lo_r = -A::inf(), hi_r = A::inf();
                if (t0n > 0) {
                    if (r1 == 0 || l1 == 0) return false;
                    lo_l = A::ceil_div(t0n, r1);
                    lo_r = A::ceil_div(t0n, l1);
                }
                if (r0 > 0) hi_l = A::fdiv(b, r0);
                if (l0 > 0) hi_r = A::fdiv(b, l0);
                st_n[sp] = R; st_a[sp] = lo_r; st_b[sp] = hi_r; ++sp;
                st_n[sp] = L; st_a[sp] = lo_l; st_b[sp] = hi_l; ++sp;
            } else if (op == NODE_DIV) {                               // :217-223
                const uint32_t rw = __ldg(q.code + R);
                if (op_of(rw) == NODE_LIT) {
                    const ll c = q.lit[arg_of(rw)];
                    if (c >= 1) {
                        st_n[sp] = L;
                        st_a[sp] = a > 0 ? a * c : a * c - (c - 1);
                        st_b[sp] = b >= 0 ? b * c + (c - 1) : b * c;
                        ++sp;
                    }
                }
            }
            // NODE_MOD: forward-only (:224-225)
        }
        return true;
    }

    // _propagate_constraint (:229-261); false = contradiction
    __device__ bool constraint(uint32_t k) {
        const uint32_t w = __ldg(q.cons + k);
        const uint32_t rel = w & 7u, lr = (w >> 3) & 0x3FFFu, rr = w >> 17;
        ll l0, l1, r0, r1;
        if (!eval(lr, l0, l1) || !eval(rr, r0, r1)) return false;
        ll a0, a1, b0, b1;
        switch (rel) {
        case REL_LT: a0 = -A::inf(); a1 = r1 - 1; b0 = l0 + 1; b1 = A::inf(); break;
        case REL_LE: a0 = -A::inf(); a1 = r1; b0 = l0; b1 = A::inf(); break;
        case REL_EQ: a0 = b0 = A::mx(l0, r0); a1 = b1 = A::mn(l1, r1); break;
        case REL_GE: a0 = r0; a1 = A::inf(); b0 = -A::inf(); b1 = l1; break;
        default:     a0 = r0 + 1; a1 = A::inf(); b0 = -A::inf(); b1 = l1 - 1; break;
        }
        return narrow2(lr, a0, a1, rr, b0, b1);
    }

    // _eval_exact at the point cur_lo (:286-328): every value is a singleton
    __device__ bool exact(uint32_t k) {
        const uint32_t w = __ldg(q.cons + k);
        const uint32_t rel = w & 7u, lr = (w >> 3) & 0x3FFFu, rr = w >> 17;
        ll v[2];
        const uint32_t roots[2] = {lr, rr};
        for (int s = 0; s < 2; ++s) {
            ll st[VST];
            int sp = 0;
            const uint32_t root = roots[s];
            for (uint32_t j = root + 1 - q.size_of(root); j <= root; ++j) {
                const uint32_t ww = __ldg(q.code + j);
                const uint32_t op = op_of(ww);
                if (op < NODE_ADD && sp == VST) {  // unreachable (host: depth <= 30); callers treat as unknown
                    ov.full = true;
                    return false;
                }
                if (op == NODE_LIT) {
                    st[sp++] = q.lit[arg_of(ww)];
                } else if (op == NODE_VAR) {
                    st[sp++] = cur_lo[arg_of(ww)];
                } else {
                    const ll y = st[--sp], x = st[--sp];
                    ll r;
                    if (op == NODE_ADD) r = x + y;
                    else if (op == NODE_SUB) r = x - y;
                    else if (op == NODE_MUL) r = x * y;
                    else {
                        if (y == 0) return false;  // trapping division falsifies (:301-302)
                        r = op == NODE_DIV ? x / y : x % y;
                    }
                    st[sp++] = r;
                }
            }
            v[s] = st[0];
        }
        switch (rel) {
        case REL_LT: return v[0] < v[1];
        case REL_LE: return v[0] <= v[1];
        case REL_EQ: return v[0] == v[1];
        case REL_GE: return v[0] >= v[1];
        default: return v[0] > v[1];
        }
    }
};

}  // namespace chain

// One warp per open own entry of the int64 job (fast mode, before the root
// kernel): decided entries get their verdict, model, nodes and the resume
// word RES_SKIP (no later kernel touches them); the rest stay as they were.
__global__ void __launch_bounds__(chain::WARPS * 32) oob_chain_kernel(LaunchArgs a) {
    using namespace chain;
    __shared__ ll s_lo[WARPS][MAXV], s_hi[WARPS][MAXV], s_nlo[WARPS][MAXV], s_nhi[WARPS][MAXV];
    __shared__ uint32_t s_entry[WARPS];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * WARPS + wib;
    ll* cur_lo = s_lo[wib];
    ll* cur_hi = s_hi[wib];
    ll* nx_lo = s_nlo[wib];
    ll* nx_hi = s_nhi[wib];
    ll* frames = a.chain_frames + (size_t)gw * DEPTH * 2 * MAXV;
    const uint32_t node_cap =
        a.node_budget > 0 ? (uint32_t)min((long long)a.chain_nodes, (long long)a.node_budget) : a.chain_nodes;
    const int64_t round_cap = a.chain_rounds;
    for (;;) {
        if (lane == 0) s_entry[wib] = atomicAdd(a.next, 1u);
        __syncwarp();
        const uint32_t qi = s_entry[wib];
        __syncwarp();
        if (qi >= a.chain_n) break;
        if (__ldcg(a.resume + qi) != 0u) continue;  // refuted by a certificate
        const QDesc d = a.qdesc[qi];
        Query q;
        q.nv = d.nv_ncon & 0xFFFFu;
        q.ncon = d.nv_ncon >> 16;
        q.ncode = d.ncode_nlit & 0xFFFFu;
        if (q.nv == 0 || q.nv > MAXV || q.ncon == 0) continue;
        q.cons = a.code + d.code_off;
        q.code = q.cons + q.ncon;
        const ll* src = reinterpret_cast<const ll*>(a.data + d.data_off);
        q.lit = src + 2 * q.nv;
        const uint64_t t_start = global_ns();
        for (uint32_t v = lane; v < q.nv; v += 32) {
            cur_lo[v] = src[2 * v];
            cur_hi[v] = src[2 * v + 1];
        }
        __syncwarp();
        // admission: every product operand's upper bound <= _INF at the
        // declared domains (the Jacobi iteration's monotonicity, see above)
        bool bad = false;
        {
            Overlay ov;
            ov.n = 0;
            ov.full = false;
            Ctx c{q, cur_lo, cur_hi, ov};
            for (uint32_t j = lane; j < q.ncode; j += 32) {
                if (op_of(__ldg(q.code + j)) != NODE_MUL) continue;
                const uint32_t R = j - 1, L = R - q.size_of(R);
                ll l0, l1, r0, r1;
                if (!c.eval(L, l0, l1) || !c.eval(R, r0, r1) || l1 > A::inf() || r1 > A::inf()) bad = true;
            }
        }
        if (__any_sync(0xFFFFFFFFu, bad)) continue;
        uint32_t depth = 0, nodes = 0;
        uint64_t stage = 0;  // bit f: frame f's upper half is being searched
        int64_t rounds_total = 0;
        int outcome = -1;    // 1 Sat, 0 Unsat, -1 left to the exact path
        for (;;) {
            // ----- one _search node (:385-416) -------------------------------
            if (++nodes > node_cap) break;
            int pr = -1;  // 1 fixpoint, 0 contradiction, -1 over the pass cap
            for (int round = 0; round < PASS_CAP; ++round) {
                if (++rounds_total > round_cap) break;  // search budget: exact path
                for (uint32_t v = lane; v < q.nv; v += 32) {
                    nx_lo[v] = cur_lo[v];
                    nx_hi[v] = cur_hi[v];
                }
                __syncwarp();
                bool dead = false, changed = false, full = false;
                Overlay ov;
                Ctx c{q, cur_lo, cur_hi, ov};
                for (uint32_t k = lane; k < q.ncon && !dead; k += 32) {
                    ov.n = 0;
                    ov.full = false;
                    if (!c.constraint(k)) {
                        dead = true;
                        full = ov.full;
                        break;
                    }
                    for (int e = 0; e < ov.n; ++e) {
                        const uint32_t v = ov.var[e];
                        if (ov.lo[e] != cur_lo[v]) atomicMax(nx_lo + v, ov.lo[e]);
                        if (ov.hi[e] != cur_hi[v]) atomicMin(nx_hi + v, ov.hi[e]);
                        changed = true;
                    }
                }
                __syncwarp();
                if (__any_sync(0xFFFFFFFFu, full)) {
                    pr = -2;
                    break;
                }
                if (__any_sync(0xFFFFFFFFu, dead)) {
                    pr = 0;
                    break;
                }
                if (!__any_sync(0xFFFFFFFFu, changed)) {
                    pr = 1;
                    break;
                }
                bool empty = false;
                for (uint32_t v = lane; v < q.nv; v += 32) {
                    cur_lo[v] = nx_lo[v];
                    cur_hi[v] = nx_hi[v];
                    empty |= nx_lo[v] > nx_hi[v];
                }
                __syncwarp();
                if (__any_sync(0xFFFFFFFFu, empty)) {
                    pr = 0;
                    break;
                }
            }
            if (pr < 0) break;  // overlay / stack capacity or pass cap: exact path
            bool backtrack = pr == 0;
            if (!backtrack) {
                // smallest unresolved domain, ties to the first declared (:397-404)
                uint64_t best = ~0ull;
                uint32_t bv = 0xFFFFFFFFu;
                for (uint32_t v = lane; v < q.nv; v += 32) {
                    if (cur_lo[v] < cur_hi[v]) {
                        const uint64_t size = (uint64_t)cur_hi[v] - (uint64_t)cur_lo[v];
                        if (size < best) {
                            best = size;
                            bv = v;
                        }
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const uint64_t ob = __shfl_xor_sync(0xFFFFFFFFu, best, o);
                    const uint32_t ov2 = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
                    if (ob < best || (ob == best && ov2 < bv)) {
                        best = ob;
                        bv = ov2;
                    }
                }
                if (bv == 0xFFFFFFFFu) {  // a leaf: check_model (:405-407)
                    Overlay ov;
                    ov.n = 0;
                    Ctx c{q, cur_lo, cur_hi, ov};
                    bool ok = true;
                    ov.full = false;
                    for (uint32_t k = lane; k < q.ncon && ok; k += 32) ok = c.exact(k);
                    if (__any_sync(0xFFFFFFFFu, ov.full)) break;  // (unreachable) exact path
                    if (__all_sync(0xFFFFFFFFu, ok)) {
                        outcome = 1;
                        break;
                    }
                    backtrack = true;
                } else {
                    if (depth == DEPTH) break;
                    ll* f = frames + (size_t)depth * 2 * MAXV;
                    for (uint32_t v = lane; v < q.nv; v += 32) {
                        f[2 * v] = cur_lo[v];
                        f[2 * v + 1] = cur_hi[v];
                    }
                    stage &= ~(1ull << depth);
                    ++depth;
                    __syncwarp();
                    if (lane == 0) {  // lower half first, floor midpoint (:408-415)
                        const ll lo = cur_lo[bv], hi = cur_hi[bv];
                        cur_hi[bv] = (lo >> 1) + (hi >> 1) + (lo & hi & 1);
                    }
                    __syncwarp();
                    continue;
                }
            }
            // ----- backtrack: the upper half of the deepest open frame --------
            bool resumed = false;
            while (depth > 0) {
                const uint32_t fi = depth - 1;
                if (stage & (1ull << fi)) {
                    stage &= ~(1ull << fi);
                    --depth;
                    continue;
                }
                stage |= 1ull << fi;
                const ll* f = frames + (size_t)fi * 2 * MAXV;
                uint64_t best = ~0ull;
                uint32_t bv = 0xFFFFFFFFu;
                for (uint32_t v = lane; v < q.nv; v += 32) {
                    cur_lo[v] = f[2 * v];
                    cur_hi[v] = f[2 * v + 1];
                    if (f[2 * v] < f[2 * v + 1]) {
                        const uint64_t size = (uint64_t)f[2 * v + 1] - (uint64_t)f[2 * v];
                        if (size < best) {
                            best = size;
                            bv = v;
                        }
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const uint64_t ob = __shfl_xor_sync(0xFFFFFFFFu, best, o);
                    const uint32_t ov2 = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
                    if (ob < best || (ob == best && ov2 < bv)) {
                        best = ob;
                        bv = ov2;
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    const ll lo = cur_lo[bv], hi = cur_hi[bv];
                    cur_lo[bv] = (lo >> 1) + (hi >> 1) + (lo & hi & 1) + 1;
                }
                __syncwarp();
                resumed = true;
                break;
            }
            if (!resumed) {  // the whole tree is exhausted
                outcome = 0;
                break;
            }
        }
        __syncwarp();
        if (outcome < 0) continue;
        if (outcome == 1) {
            int64_t* m = a.model + 2 * d.out_v;
            for (uint32_t v = lane; v < q.nv; v += 32) store_i128(m + 2 * v, cur_lo[v]);
        }
        if (lane == 0) {
            a.verdict[qi] = (int8_t)(outcome == 1 ? VERDICT_SAT : VERDICT_UNSAT);
            a.err[qi] = (int8_t)ERR_NONE;
            a.nodes[qi] = nodes;
            a.passes[qi] = rounds_total;
            a.elapsed[qi] = (float)((double)(global_ns() - t_start) * 1e-9);
            a.resume[qi] = RES_SKIP;
            if (a.fast_stats) atomicAdd(a.fast_stats + 5, 1ull);
        }
        __syncwarp();
    }
}

}  // namespace oob

namespace oob {

// Fast mode, K3: exhaustive enumeration of the small boxes.  An own entry of
// the int64 job that no certificate refuted and whose declared box holds at
// most a.enum_max points is enumerated point by point (lanes stride over the
// mixed-radix point index; each lane evaluates every constraint exactly at
// its point, _eval_exact / check_model :286-328, divisor side constraints
// included).  The reference only ever answers Sat with a point of the box
// that passes check_model (:405-407), so a box without such a point is the
// reference's Unsat: decided here (nodes/passes 0, like a certificate
// refutation).  The first satisfying point any lane meets (warp ballot) ends
// the enumeration and leaves the entry to the exact emulation, which finds
// the reference's first model.  int64 arithmetic is exact here: the job's
// bound proof covers every value of the box.
__global__ void __launch_bounds__(chain::WARPS * 32) oob_enum_kernel(LaunchArgs a) {
    using namespace chain;
    __shared__ ll s_lo[WARPS][MAXV];
    __shared__ uint64_t s_size[WARPS][MAXV];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t nwarps = gridDim.x * WARPS;
    // 32 consecutive entries per warp and step: each lane screens one (open,
    // box within enum_max), then the warp enumerates the admitted ones
    for (uint32_t base = (blockIdx.x * WARPS + wib) * 32u; base < a.enum_n; base += nwarps * 32u) {
        const uint32_t qi = base + lane;
        bool cand = false;
        if (qi < a.enum_n && __ldcg(a.resume + qi) == 0u) {
            const QDesc d = a.qdesc[qi];
            const uint32_t nv = d.nv_ncon & 0xFFFFu;
            if (nv > 0 && nv <= MAXV && (d.nv_ncon >> 16) > 0) {
                const ll* src = reinterpret_cast<const ll*>(a.data + d.data_off);
                uint64_t box = 1;
                cand = true;
                for (uint32_t v = 0; v < nv && cand; ++v) {
                    const ll lo = src[2 * v], hi = src[2 * v + 1];
                    const uint64_t sz = hi >= lo ? (uint64_t)hi - (uint64_t)lo + 1 : 0;
                    if (sz == 0 || sz > a.enum_max || box * sz > a.enum_max) cand = false;
                    else box *= sz;
                }
            }
        }
        uint32_t todo = __ballot_sync(0xFFFFFFFFu, cand);
        while (todo) {
            const uint32_t e = base + (uint32_t)(__ffs(todo) - 1);
            todo &= todo - 1;
            const QDesc d = a.qdesc[e];
            Query q;
            q.nv = d.nv_ncon & 0xFFFFu;
            q.ncon = d.nv_ncon >> 16;
            q.ncode = d.ncode_nlit & 0xFFFFu;
            q.cons = a.code + d.code_off;
            q.code = q.cons + q.ncon;
            const ll* src = reinterpret_cast<const ll*>(a.data + d.data_off);
            q.lit = src + 2 * q.nv;
            uint64_t box = 1;
            for (uint32_t v = lane; v < q.nv; v += 32) {
                s_lo[wib][v] = src[2 * v];
                s_size[wib][v] = (uint64_t)src[2 * v + 1] - (uint64_t)src[2 * v] + 1;
            }
            __syncwarp();
            for (uint32_t v = 0; v < q.nv; ++v) box *= s_size[wib][v];
            ll pt[MAXV];
            Overlay ov;
            ov.n = 0;
            ov.full = false;
            Ctx c{q, pt, pt, ov};
            bool found = false;
            for (uint64_t b0 = 0; b0 < box && !found; b0 += 32) {
                const uint64_t idx = b0 + lane;
                bool ok = false;
                if (idx < box) {
                    uint64_t r = idx;
                    for (uint32_t v = 0; v < q.nv; ++v) {  // variable 0 varies slowest
                        const uint32_t w = q.nv - 1 - v;
                        const uint64_t sz = s_size[wib][w];
                        pt[w] = s_lo[wib][w] + (ll)(r % sz);
                        r /= sz;
                    }
                    ok = true;
                    for (uint32_t k = 0; k < q.ncon && ok; ++k) ok = c.exact(k);
                    ok = ok || ov.full;  // (unreachable) an unevaluated point counts as found
                }
                found = __any_sync(0xFFFFFFFFu, ok);
            }
            if (!found && lane == 0) {
                a.verdict[e] = (int8_t)VERDICT_UNSAT;
                a.err[e] = (int8_t)ERR_NONE;
                a.nodes[e] = 0;
                a.passes[e] = 0;
                a.elapsed[e] = 0.f;
                a.resume[e] = RES_SKIP;
            }
            __syncwarp();
        }
    }
}

}  // namespace oob
