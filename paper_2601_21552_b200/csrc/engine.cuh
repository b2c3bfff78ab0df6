// engine.cuh -- device-side exact emulation of the reference solver
// (/root/reference/pkg/src/scuba_mini/solver.py:112-416) for sm_100a.
//
// One lane owns one query at a time.  Everything a lane touches repeatedly
// lives in a per-warp scratch slab laid out [index][32 lanes] (lane-minor), so
// when the lanes of a warp run instances of one structure class in lockstep
// (kernels.cu schedules whole warps per class and advances all lanes one
// propagation pass at a time) every scratch access of the warp is one
// coalesced line per word and every code word is a broadcast load.
//
// Exactness: the host proves, per query, a bound B on the magnitude of every
// intermediate value the reference algorithm can produce (forward intervals at
// the declared domains, narrowing targets including the 10**18 clamp, exact
// model evaluation); the query then runs on int64, __int128 or the 256-bit
// type of wide.cuh, on which plain two's-complement arithmetic is exact.
//
// Constraint skipping (exact): a constraint whose last propagation changed
// nothing and none of whose variables changed since is skipped -- running it
// again would change nothing and succeed, because narrowing is a function of
// the current domains only.  Per lane a "clean" bit per constraint is kept;
// a domain change of variable v clears the bits of every constraint that
// mentions v (per-class membership masks).  Pass counts, node counts, the
// order of every effective narrowing and hence verdicts and models are those
// of the reference.  A DFS child starts from its parent's clean mask minus
// the constraints of the split variable.
#pragma once
#include "types.h"

#include "format.h"
#include "wide.cuh"

namespace oob {

// C truncating division / remainder (tdiv / tmod, solver.py:94-102); the
// 128-bit software routine is skipped when both operands fit in 64 bits
template <typename T>
__device__ __forceinline__ T cdiv(T a, T b) { return a / b; }
template <typename T>
__device__ __forceinline__ T cmod(T a, T b) { return a % b; }
__device__ __forceinline__ bool fits64(__int128 v) { return v == (__int128)(long long)v; }
// int64: the 32-bit hardware path when both operands lie in [-(2^31-1), 2^31-1]
// (no INT32_MIN, so no overflow), the 64-bit software routine otherwise
__device__ __forceinline__ bool fits31(long long v) { return (unsigned long long)v + 0x7FFFFFFFull <= 0xFFFFFFFEull; }
// (one out-of-line copy each: every inlined division site would otherwise
// carry ~25 instructions of the 32-bit path and blow the instruction cache)
__device__ __noinline__ long long cdiv_ll(long long a, long long b) {
    if (fits31(a) && fits31(b)) return (long long)((int)a / (int)b);
    return a / b;
}
__device__ __noinline__ long long cmod_ll(long long a, long long b) {
    if (fits31(a) && fits31(b)) return (long long)((int)a % (int)b);
    return a % b;
}
template <>
__device__ __forceinline__ long long cdiv<long long>(long long a, long long b) { return cdiv_ll(a, b); }
template <>
__device__ __forceinline__ long long cmod<long long>(long long a, long long b) { return cmod_ll(a, b); }
template <>
__device__ __forceinline__ __int128 cdiv<__int128>(__int128 a, __int128 b) {
    if (fits64(a) && fits64(b) && !((long long)a == (-9223372036854775807LL - 1) && (long long)b == -1))
        return (__int128)cdiv<long long>((long long)a, (long long)b);
    return a / b;
}
template <>
__device__ __forceinline__ __int128 cmod<__int128>(__int128 a, __int128 b) {
    if (fits64(a) && fits64(b) && !((long long)a == (-9223372036854775807LL - 1) && (long long)b == -1))
        return (__int128)cmod<long long>((long long)a, (long long)b);
    return a % b;
}

// The x32 regime (int32 values): narrowing targets derived from
// the reference's +-10**18 clamp are carried as +-2^30 ("beyond range") while
// every real value is below 2^28 (device proof Lane::fit_x32).  A target
// computed from an out-of-range one is renormalised to +-2^30, and a division
// or multiplication of one stays out of range -- exactly how the reference's
// huge finite values behave against values below 2^28.
template <typename T>
struct Ext {
    static constexpr bool X32 = false;
    __device__ static inline T sat(T x) { return x; }
    __device__ static inline bool big_hi(T) { return false; }
    __device__ static inline bool big_lo(T) { return false; }
};
template <>
struct Ext<int> {
    static constexpr bool X32 = true;
    static constexpr int INF = 1 << 30, HALF = 1 << 29;
    __device__ static inline int sat(int x) { return x >= HALF ? INF : (x <= -HALF ? -INF : x); }
    __device__ static inline bool big_hi(int x) { return x >= HALF; }
    __device__ static inline bool big_lo(int x) { return x <= -HALF; }
};

template <typename T>
struct Arith {
    __device__ static inline T inf() {  // _INF = 10**18 (solver.py:23); x32: 2^30 (out of range)
        if constexpr (Ext<T>::X32) return T(1 << 30);
        else return T(1000000000000000000LL);
    }
    __device__ static inline T mn(T a, T b) { return a < b ? a : b; }
    __device__ static inline T mx(T a, T b) { return a > b ? a : b; }
    // Python floor division a // b (C division truncates: that is tdiv, solver.py:94)
    __device__ static inline T fdiv(T a, T b) {
        T q = cdiv(a, b);
        T r = a - q * b;
        return (r != T(0) && ((r < T(0)) != (b < T(0)))) ? q - T(1) : q;
    }
    // _ceil_div (solver.py:105-106): -((-a) // b)
    __device__ static inline T ceil_div(T a, T b) { return -fdiv(-a, b); }
};

// model / domain output in the caller's int128 wire format (values are
// within the declared domains, which the wire format bounds to 128 bits)
__device__ __forceinline__ void store_i128(int64_t* out, int v) {
    out[0] = v;
    out[1] = v < 0 ? -1 : 0;
}
__device__ __forceinline__ void store_i128(int64_t* out, long long v) {
    out[0] = v;
    out[1] = v < 0 ? -1 : 0;
}
__device__ __forceinline__ void store_i128(int64_t* out, __int128 v) {
    out[0] = (int64_t)(uint64_t)v;
    out[1] = (int64_t)(v >> 64);
}
__device__ __forceinline__ void store_i128(int64_t* out, const i256& v) {
    out[0] = (int64_t)v.w[0];
    out[1] = (int64_t)v.w[1];
}

// value conversions between the regimes (the caller has proven the value fits)
template <typename T>
__device__ __forceinline__ T from_i128(__int128 v) { return (T)v; }
template <>
__device__ __forceinline__ i256 from_i128<i256>(__int128 v) { return i256::from128(v); }
__device__ __forceinline__ long long low64(int v) { return v; }
__device__ __forceinline__ long long low64(long long v) { return v; }
__device__ __forceinline__ long long low64(__int128 v) { return (long long)v; }
__device__ __forceinline__ long long low64(const i256& v) { return (long long)v.w[0]; }
__device__ __forceinline__ __int128 low128(int v) { return v; }
__device__ __forceinline__ __int128 low128(long long v) { return v; }
__device__ __forceinline__ __int128 low128(__int128 v) { return v; }
__device__ __forceinline__ __int128 low128(const i256& v) { return v.low128(); }

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

extern __shared__ __align__(16) unsigned char oob_smem[];

// The interpreting lane: one query's search state, driven by the class's code
// words.  lockstep_phase / frontier_phase (phases.cuh) drive any lane type
// with this interface; jit_lane.cuh provides the compiled counterpart.
template <typename TT>
struct Lane {
    using T = TT;
    using A = Arith<T>;
    // lane-minor scratch views (element i of this lane is p[i * 32])
    T* env_lo;
    T* env_hi;
    T* val_lo;
    T* val_hi;
    T* lit;
    T* fr_mid;
    T* fr_hi;
    T* tr_lo;
    T* tr_hi;
    uint32_t* stamp;
    uint32_t* fr_pick;
    uint32_t* fr_mark;
    uint32_t* fr_clean;  // 4 words per frame
    uint32_t* tr_var;
    uint32_t* st_n;          // narrowing stack (shared memory when it fits)
    T* st_0;
    T* st_1;
    uint32_t st_cap;
    const SlabGeom* g;
    // current query (class-uniform within a warp)
    const uint32_t* cons;    // ncon constraint words
    const uint32_t* code;    // ncode node words
    const uint32_t* member;  // 4 words per variable: constraints mentioning it
    uint32_t nv, ncon, ncode, nlit;
    uint32_t vbase;          // first node of the constraint being processed
    bool skip;               // constraint skipping enabled (ncon <= 128)
    // search state
    uint32_t depth, trail_len, seg;
    uint64_t clean0, clean1; // clean bit per constraint (0..63, 64..127)
    bool dirty;     // a variable changed since the current constraint's top-level eval
    bool changed;   // the current pass changed a domain (_Narrower.changed)
    int err;

    __device__ __forceinline__ T& E(T* p, uint32_t i) const { return p[(size_t)i * 32]; }
    // forward-interval cache of the current constraint's nodes (indexed from
    // the constraint's first node, so it only needs max-constraint-size slots)
    __device__ __forceinline__ T& VL(uint32_t j) const { return val_lo[(size_t)(j - vbase) * 32]; }
    __device__ __forceinline__ T& VH(uint32_t j) const { return val_hi[(size_t)(j - vbase) * 32]; }
    __device__ __forceinline__ uint32_t& U(uint32_t* p, uint32_t i) const { return p[(size_t)i * 32]; }

    __device__ __forceinline__ static uint32_t op_of(uint32_t w) { return w & 7u; }
    __device__ __forceinline__ static uint32_t arg_of(uint32_t w) { return w >> 3; }
    __device__ __forceinline__ uint32_t size_of(uint32_t i) const {
        uint32_t w = __ldg(code + i);
        return op_of(w) >= NODE_ADD ? arg_of(w) : 1u;
    }

    __device__ __forceinline__ bool is_clean(uint32_t k) const {
        if (!skip) return false;
        return k < 64 ? ((clean0 >> k) & 1ull) : ((clean1 >> (k - 64)) & 1ull);
    }
    __device__ __forceinline__ void set_clean(uint32_t k) {
        if (k < 64) clean0 |= 1ull << k;
        else if (k < 128) clean1 |= 1ull << (k - 64);
    }
    __device__ __forceinline__ void touch(uint32_t v) {
        const uint32_t* m = member + 4 * v;
        clean0 &= ~(((uint64_t)__ldg(m + 1) << 32) | __ldg(m));
        clean1 &= ~(((uint64_t)__ldg(m + 3) << 32) | __ldg(m + 2));
    }

    // ----- _eval_iv over a postfix range (solver.py:112-149) ------------------
    // Computes val[j] for every node of the subtree rooted at `root`; false if
    // any node of it has no non-trapping value (the reference's None).
    __device__ bool eval_subtree(uint32_t root) {
        uint32_t start = root + 1 - size_of(root);
        for (uint32_t j = start; j <= root; ++j) {
            uint32_t w = __ldg(code + j);
            uint32_t op = op_of(w);
            T lo, hi;
            if (op == NODE_LIT) {
                lo = hi = E(lit, arg_of(w));
            } else if (op == NODE_VAR) {
                lo = E(env_lo, arg_of(w));
                hi = E(env_hi, arg_of(w));
                if (lo > hi) return false;
            } else {
                uint32_t R = j - 1;
                uint32_t L = R - size_of(R);
                T l0 = VL(L), l1 = VH(L), r0 = VL(R), r1 = VH(R);
                if (op == NODE_ADD) {
                    lo = l0 + r0;
                    hi = l1 + r1;
                } else if (op == NODE_SUB) {
                    lo = l0 - r1;
                    hi = l1 - r0;
                } else if (op == NODE_MUL) {
                    T k0 = l0 * r0, k1 = l0 * r1, k2 = l1 * r0, k3 = l1 * r1;
                    lo = A::mn(A::mn(k0, k1), A::mn(k2, k3));
                    hi = A::mx(A::mx(k0, k1), A::mx(k2, k3));
                } else {
                    T d0 = A::mx(r0, T(1)), d1 = r1;
                    if (d0 > d1) return false;
                    if (op == NODE_DIV) {
                        T k0 = cdiv(l0, d0), k1 = cdiv(l0, d1), k2 = cdiv(l1, d0), k3 = cdiv(l1, d1);
                        lo = A::mn(A::mn(k0, k1), A::mn(k2, k3));
                        hi = A::mx(A::mx(k0, k1), A::mx(k2, k3));
                    } else {  // NODE_MOD
                        T m = d1 - T(1);
                        if (l0 >= T(0)) {
                            lo = T(0);
                            hi = A::mn(l1, m);
                        } else if (l1 <= T(0)) {
                            lo = A::mx(l0, -m);
                            hi = T(0);
                        } else {
                            lo = A::mx(l0, -m);
                            hi = A::mn(l1, m);
                        }
                    }
                }
            }
            VL(j) = lo;
            VH(j) = hi;
        }
        return true;
    }

    // ----- domain update with trail logging -----------------------------------
    __device__ __forceinline__ bool set_dom(uint32_t v, T lo, T hi) {
        if (depth > 0 && U(stamp, v) != seg) {
            if (trail_len >= g->trail_cap) {
                err = ERR_TRAIL;
                return false;
            }
            U(tr_var, trail_len) = v;
            E(tr_lo, trail_len) = E(env_lo, v);
            E(tr_hi, trail_len) = E(env_hi, v);
            ++trail_len;
            U(stamp, v) = seg;
        }
        E(env_lo, v) = lo;
        E(env_hi, v) = hi;
        touch(v);
        return true;
    }

    // ----- _Narrower.narrow (solver.py:159-226), explicit pre-order stack ------
    // The pre-order stack lives in lane-minor shared memory (st_*), sized by
    // the host to the deepest term of the job (st_cap entries).
    __device__ bool narrow(uint32_t root, T t0, T t1) {
        const int NS = (int)st_cap;
        int sp = 1;
        U(st_n, 0) = root;
        E(st_0, 0) = t0;
        E(st_1, 0) = t1;
        while (sp > 0) {
            --sp;
            uint32_t i = U(st_n, sp);
            T a = E(st_0, sp), b = E(st_1, sp);
            if (a > b) return false;                                   // :161-162
            uint32_t w = __ldg(code + i);
            uint32_t op = op_of(w);
            if (op == NODE_LIT) {                                      // :163-164
                T v = E(lit, arg_of(w));
                if (!(a <= v && v <= b)) return false;
                continue;
            }
            if (op == NODE_VAR) {                                      // :165-173
                uint32_t v = arg_of(w);
                T lo = E(env_lo, v), hi = E(env_hi, v);
                T nlo = A::mx(lo, a), nhi = A::mn(hi, b);
                if (nlo > nhi) return false;
                if (nlo != lo || nhi != hi) {
                    if (!set_dom(v, nlo, nhi)) return false;
                    changed = true;
                    dirty = true;
                }
                continue;
            }
            uint32_t R = i - 1;                                        // :174-177
            uint32_t L = R - size_of(R);
            if (dirty) {
                if (!eval_subtree(L) || !eval_subtree(R)) return false;
            }
            T l0 = VL(L), l1 = VH(L), r0 = VL(R), r1 = VH(R);
            if (sp + 2 > NS) {
                err = ERR_STACK;
                return false;
            }
            using X = Ext<T>;
            if (op == NODE_ADD) {                                      // :181-185
                U(st_n, sp) = R; E(st_0, sp) = X::sat(a - l1); E(st_1, sp) = X::sat(b - l0); ++sp;
                U(st_n, sp) = L; E(st_0, sp) = X::sat(a - r1); E(st_1, sp) = X::sat(b - r0); ++sp;
            } else if (op == NODE_SUB) {                               // :186-190
                U(st_n, sp) = R; E(st_0, sp) = X::sat(l0 - b); E(st_1, sp) = X::sat(l1 - a); ++sp;
                U(st_n, sp) = L; E(st_0, sp) = X::sat(a + r0); E(st_1, sp) = X::sat(b + r1); ++sp;
            } else if (op == NODE_MUL) {                               // :191-216
                if (l0 < T(0) || r0 < T(0)) continue;
                if (b < T(0)) return false;
                T t0n = A::mx(a, T(0));
                T lo_l = -A::inf(), hi_l = A::inf(), lo_r = -A::inf(), hi_r = A::inf();
                if (t0n > T(0)) {
                    if (r1 == T(0) || l1 == T(0)) return false;
                    lo_l = A::ceil_div(t0n, r1);
                    lo_r = A::ceil_div(t0n, l1);
                }
                if (r0 > T(0)) hi_l = X::big_hi(b) ? A::inf() : A::fdiv(b, r0);
                if (l0 > T(0)) hi_r = X::big_hi(b) ? A::inf() : A::fdiv(b, l0);
                U(st_n, sp) = R; E(st_0, sp) = lo_r; E(st_1, sp) = hi_r; ++sp;
                U(st_n, sp) = L; E(st_0, sp) = lo_l; E(st_1, sp) = hi_l; ++sp;
            } else if (op == NODE_DIV) {                               // :217-223
                uint32_t rw = __ldg(code + R);
                if (op_of(rw) == NODE_LIT) {
                    T c = E(lit, arg_of(rw));
                    if (c >= T(1)) {
                        T lo_req = X::big_lo(a) ? -A::inf() : (a > T(0) ? a * c : a * c - (c - T(1)));
                        T hi_req = X::big_hi(b) ? A::inf() : (b >= T(0) ? b * c + (c - T(1)) : b * c);
                        U(st_n, sp) = L; E(st_0, sp) = lo_req; E(st_1, sp) = hi_req; ++sp;
                    }
                }
            }
            // NODE_MOD: forward-only (:224-225)
        }
        return true;
    }

    // ----- leaf fast path: both sides are a variable or a literal ---------------
    // (most analyzer constraints: geometry ranges, launch equations, bindings,
    // asserts).  Same semantics as the general path below, without the
    // forward-interval cache or the narrowing stack.
    __device__ __forceinline__ bool narrow_leaf(uint32_t w, T a, T b) {
        if (a > b) return false;                                       // :161-162
        if (op_of(w) == NODE_LIT) {                                    // :163-164
            T v = E(lit, arg_of(w));
            return a <= v && v <= b;
        }
        uint32_t v = arg_of(w);                                        // :165-173
        T lo = E(env_lo, v), hi = E(env_hi, v);
        T nlo = A::mx(lo, a), nhi = A::mn(hi, b);
        if (nlo > nhi) return false;
        if (nlo != lo || nhi != hi) {
            if (!set_dom(v, nlo, nhi)) return false;
            changed = true;
        }
        return true;
    }

    __device__ __forceinline__ bool propagate_leaves(uint32_t rel, uint32_t lw, uint32_t rw) {
        T l0, l1, r0, r1;
        if (op_of(lw) == NODE_LIT) {
            l0 = l1 = E(lit, arg_of(lw));
        } else {
            l0 = E(env_lo, arg_of(lw));
            l1 = E(env_hi, arg_of(lw));
            if (l0 > l1) return false;
        }
        if (op_of(rw) == NODE_LIT) {
            r0 = r1 = E(lit, arg_of(rw));
        } else {
            r0 = E(env_lo, arg_of(rw));
            r1 = E(env_hi, arg_of(rw));
            if (r0 > r1) return false;
        }
        T a0, a1, b0, b1;
        switch (rel) {
        case REL_LT: a0 = -A::inf(); a1 = r1 - T(1); b0 = l0 + T(1); b1 = A::inf(); break;
        case REL_LE: a0 = -A::inf(); a1 = r1; b0 = l0; b1 = A::inf(); break;
        case REL_EQ: a0 = b0 = A::mx(l0, r0); a1 = b1 = A::mn(l1, r1); break;
        case REL_GE: a0 = r0; a1 = A::inf(); b0 = -A::inf(); b1 = l1; break;
        default:     a0 = r0 + T(1); a1 = A::inf(); b0 = -A::inf(); b1 = l1 - T(1); break;
        }
        return narrow_leaf(lw, a0, a1) && narrow_leaf(rw, b0, b1);
    }

    // ----- _propagate_constraint (solver.py:229-261) ---------------------------
    __device__ bool propagate_constraint(uint32_t k) {
        uint32_t w = __ldg(cons + k);
        uint32_t rel = w & 7u;
        uint32_t lr = (w >> 3) & 0x3FFFu;
        uint32_t rr = w >> 17;
        {
            uint32_t lw = __ldg(code + lr), rw = __ldg(code + rr);
            if (op_of(lw) < NODE_ADD && op_of(rw) < NODE_ADD) return propagate_leaves(rel, lw, rw);
        }
        vbase = lr + 1 - size_of(lr);
        dirty = false;
        if (!eval_subtree(lr) || !eval_subtree(rr)) return false;
        T l0 = VL(lr), l1 = VH(lr), r0 = VL(rr), r1 = VH(rr);
        T a0, a1, b0, b1;
        switch (rel) {
        case REL_LT: a0 = -A::inf(); a1 = r1 - T(1); b0 = l0 + T(1); b1 = A::inf(); break;
        case REL_LE: a0 = -A::inf(); a1 = r1; b0 = l0; b1 = A::inf(); break;
        case REL_EQ: a0 = b0 = A::mx(l0, r0); a1 = b1 = A::mn(l1, r1); break;
        case REL_GE: a0 = r0; a1 = A::inf(); b0 = -A::inf(); b1 = l1; break;
        default:     a0 = r0 + T(1); a1 = A::inf(); b0 = -A::inf(); b1 = l1 - T(1); break;
        }
        return narrow(lr, a0, a1) && narrow(rr, b0, b1);
    }

    // lowest constraint index >= k that is not clean (ncon if none)
    __device__ __forceinline__ uint32_t next_dirty(uint32_t k) const {
        if (!skip) return k < ncon ? k : ncon;
        uint64_t d0 = ~clean0, d1 = ~clean1;
        if (k < 64) {
            uint64_t m = d0 & (~0ull << k);
            if (m) return min((uint32_t)__ffsll((long long)m) - 1, ncon);
            k = 64;
        }
        if (k < 128) {
            uint64_t m = d1 & (~0ull << (k - 64));
            if (m) return min(64u + (uint32_t)__ffsll((long long)m) - 1, ncon);
        }
        return ncon;
    }

    // one (dirty) constraint inside a pass; false = contradiction
    __device__ __forceinline__ bool pass_constraint(uint32_t k) {
        bool before = changed;
        changed = false;
        bool ok = propagate_constraint(k);
        if (ok && !changed && skip) set_clean(k);
        changed = changed || before;
        return ok;
    }

    // ----- propagate (solver.py:264-280), in place (aux kernel) ----------------
    // returns 1 ok, 0 contradiction, -2 error
    __device__ int propagate(int64_t& passes) {
        for (int pass = 0; pass < PASS_CAP; ++pass) {
            ++passes;
            changed = false;
            for (uint32_t k = next_dirty(0); k < ncon; k = next_dirty(k + 1)) {
                if (!pass_constraint(k)) return err ? -2 : 0;
            }
            if (!changed) break;
        }
        return 1;
    }

    // ----- _eval_exact / check_model (solver.py:286-328) ----------------------
    // Exact evaluation of every constraint at the point env_lo (val_lo holds
    // the node values).  Division/modulo by zero falsifies (:301-302).
    __device__ bool check_point(const T* point) {
        for (uint32_t k = 0; k < ncon; ++k) {
            uint32_t w = __ldg(cons + k);
            uint32_t rel = w & 7u;
            uint32_t lr = (w >> 3) & 0x3FFFu;
            uint32_t rr = w >> 17;
            vbase = lr + 1 - size_of(lr);
            T vv[2];
            uint32_t roots[2] = {lr, rr};
            for (int s = 0; s < 2; ++s) {
                uint32_t root = roots[s];
                uint32_t start = root + 1 - size_of(root);
                for (uint32_t j = start; j <= root; ++j) {
                    uint32_t cw = __ldg(code + j);
                    uint32_t op = op_of(cw);
                    T x;
                    if (op == NODE_LIT) {
                        x = E(lit, arg_of(cw));
                    } else if (op == NODE_VAR) {
                        x = point[(size_t)arg_of(cw) * 32];
                    } else {
                        uint32_t R = j - 1;
                        uint32_t L = R - size_of(R);
                        T a = VL(L), b = VL(R);
                        if (op == NODE_ADD) x = a + b;
                        else if (op == NODE_SUB) x = a - b;
                        else if (op == NODE_MUL) x = a * b;
                        else {
                            if (b == T(0)) return false;
                            x = op == NODE_DIV ? cdiv(a, b) : cmod(a, b);
                        }
                    }
                    VL(j) = x;
                }
                vv[s] = VL(root);
            }
            T a = vv[0], b = vv[1];
            bool ok;
            switch (rel) {
            case REL_LT: ok = a < b; break;
            case REL_LE: ok = a <= b; break;
            case REL_EQ: ok = a == b; break;
            case REL_GE: ok = a >= b; break;
            default: ok = a > b; break;
            }
            if (!ok) return false;
        }
        return true;
    }

    // ----- the lane interface used by the scheduling phases (phases.cuh) -------
    __device__ __forceinline__ T get_lo(uint32_t v) const { return E(env_lo, v); }
    __device__ __forceinline__ T get_hi(uint32_t v) const { return E(env_hi, v); }
    __device__ __forceinline__ void put_env(uint32_t v, T lo, T hi) {
        E(env_lo, v) = lo;
        E(env_hi, v) = hi;
    }
    __device__ __forceinline__ uint32_t nvars() const { return nv; }
    // whole domain vectors: (lo, hi) pairs in / out, model = the lower bounds
    __device__ __forceinline__ void load_env(const T* env) {
        for (uint32_t v = 0; v < nv; ++v) put_env(v, env[2 * v], env[2 * v + 1]);
    }
    __device__ __forceinline__ void store_env(T* env) const {
        for (uint32_t v = 0; v < nv; ++v) {
            env[2 * v] = get_lo(v);
            env[2 * v + 1] = get_hi(v);
        }
    }
    __device__ __forceinline__ void store_model(int64_t* m) const {
        for (uint32_t v = 0; v < nv; ++v) store_i128(m + 2 * v, get_lo(v));
    }
    __device__ __forceinline__ bool check_env() { return check_point(env_lo); }
    // One propagation pass of every lane with run set, warp-synchronously: the
    // warp visits, in order, every constraint that is dirty in at least one
    // lane (clean ones would change nothing), so constraint k's code words are
    // warp-uniform.  Returns true if this lane's pass hit a contradiction.
    __device__ __forceinline__ bool pass_sync(bool run) {
        bool dead = false;
        for (uint32_t k = 0;;) {
            uint32_t mine = (run && !dead) ? next_dirty(k) : 0xFFFFu;
            if (mine >= ncon) mine = 0xFFFFu;  // lanes may be on different classes
            uint32_t kk = __reduce_min_sync(0xffffffffu, mine);
            if (kk == 0xFFFFu) break;
            if (mine == kk && !pass_constraint(kk)) dead = true;
            k = kk + 1;
        }
        return dead;
    }

    // per-warp scratch binding (host-computed SlabGeom)
    __device__ void bind(const LaunchArgs& a, uint32_t warp, uint32_t lane) {
        const SlabGeom& gg = a.g;
        T* sT = reinterpret_cast<T*>(a.slab_T) + (size_t)warp * gg.slab_T_words + lane;
        uint32_t* sU = a.slab_u32 + (size_t)warp * gg.slab_u32_words + lane;
        if (gg.smem_per_warp) {  // hot state on chip, lane-minor (conflict-free in lockstep)
            T* s = reinterpret_cast<T*>(oob_smem + (threadIdx.x >> 5) * gg.smem_per_warp) + lane;
            env_lo = s + gg.o_s_env_lo;
            env_hi = s + gg.o_s_env_hi;
            val_lo = s + gg.o_s_val_lo;
            val_hi = s + gg.o_s_val_hi;
            lit = sT + gg.o_lit;
            st_0 = s + gg.o_s_st0;
            st_1 = s + gg.o_s_st1;
            st_n = reinterpret_cast<uint32_t*>(oob_smem + (threadIdx.x >> 5) * gg.smem_per_warp + gg.o_s_stn_bytes) +
                   lane;
        } else {
            env_lo = sT + gg.o_env_lo;
            env_hi = sT + gg.o_env_hi;
            val_lo = sT + gg.o_val_lo;
            val_hi = sT + gg.o_val_hi;
            lit = sT + gg.o_lit;
            st_0 = sT + gg.o_st0;
            st_1 = sT + gg.o_st1;
            st_n = sU + gg.o_stn;
        }
        st_cap = gg.st_cap;
        fr_mid = sT + gg.o_fr_mid;
        fr_hi = sT + gg.o_fr_hi;
        tr_lo = sT + gg.o_tr_lo;
        tr_hi = sT + gg.o_tr_hi;
        stamp = sU + gg.o_stamp;
        fr_pick = sU + gg.o_fr_pick;
        fr_mark = sU + gg.o_fr_mark;
        fr_clean = sU + gg.o_fr_clean;
        tr_var = sU + gg.o_tr_var;
        g = &a.g;
        seg = 0;
    }

    __device__ __forceinline__ void set_class(const LaunchArgs& a, const ClassDesc& c) {
        nv = c.nv_ncon & 0xFFFFu;
        ncon = c.nv_ncon >> 16;
        ncode = c.ncode_nlit & 0xFFFFu;
        nlit = c.ncode_nlit >> 16;
        cons = a.code + c.code_off;
        code = cons + ncon;
        member = code + ncode;
        skip = ncon <= 128;
    }

    // stage a query's domains and literal slots into lane-minor scratch
    __device__ __forceinline__ void load(const LaunchArgs& a, const QDesc& d) { load_from(a.data, d); }
    // current domains + literals in the job's data layout (hand-off at the root)
    __device__ __forceinline__ void save_state(int64_t* base, const QDesc& d) const {
        T* dst = reinterpret_cast<T*>(base + d.data_off);
        for (uint32_t v = 0; v < nv; ++v) {
            dst[2 * v] = E(env_lo, v);
            dst[2 * v + 1] = E(env_hi, v);
        }
        for (uint32_t i = 0; i < nlit; ++i) dst[2 * nv + i] = E(lit, i);
    }
    __device__ __forceinline__ void load_from(const int64_t* base, const QDesc& d) {
        const T* src = reinterpret_cast<const T*>(base + d.data_off);
        for (uint32_t v = 0; v < nv; ++v) {
            E(env_lo, v) = src[2 * v];
            E(env_hi, v) = src[2 * v + 1];
            U(stamp, v) = 0xFFFFFFFFu;
        }
        for (uint32_t i = 0; i < nlit; ++i) E(lit, i) = src[2 * nv + i];
        err = ERR_NONE;
        depth = 0;
        trail_len = 0;
        clean0 = 0;
        clean1 = 0;
    }

    // ----- regime demotion (root kernel) ----------------------------------------
    // The host proves its regime bound at the DECLARED domains (host.cpp
    // prove_bound).  Domains only shrink below the current node, and forward
    // intervals, narrowing targets and exact values are inclusion-monotone, so
    // the same proof restated at the CURRENT domains bounds every value the
    // rest of the search can produce.  Returns the narrowest regime that
    // holds: 0 int64, 1 int128, 2 neither.
    __device__ static T tabs(T x) { return x < T(0) ? -x : x; }
    __device__ int fit_regime() {
        T B = T(0), D = T(0);
        for (uint32_t v = 0; v < nv; ++v) D = A::mx(D, A::mx(tabs(E(env_lo, v)), tabs(E(env_hi, v))));
        for (uint32_t i = 0; i < nlit; ++i) B = A::mx(B, tabs(E(lit, i)));
        const T INF = A::inf();
        for (uint32_t k = 0; k < ncon; ++k) {
            uint32_t w = __ldg(cons + k);
            uint32_t rel = w & 7u, lr = (w >> 3) & 0x3FFFu, rr = w >> 17;
            uint32_t start = lr + 1 - size_of(lr);
            vbase = start;
            // forward intervals F; "no value" (the reference's None) is lo > hi
            for (uint32_t j = start; j <= rr; ++j) {
                uint32_t cw = __ldg(code + j), op = op_of(cw);
                T lo, hi;
                if (op == NODE_LIT) {
                    lo = hi = E(lit, arg_of(cw));
                } else if (op == NODE_VAR) {
                    lo = E(env_lo, arg_of(cw));
                    hi = E(env_hi, arg_of(cw));
                } else {
                    uint32_t R = j - 1, L = R - size_of(R);
                    T l0 = VL(L), l1 = VH(L), r0 = VL(R), r1 = VH(R);
                    lo = T(1);
                    hi = T(0);
                    if (l0 <= l1 && r0 <= r1) {
                        if (op == NODE_ADD) { lo = l0 + r0; hi = l1 + r1; }
                        else if (op == NODE_SUB) { lo = l0 - r1; hi = l1 - r0; }
                        else if (op == NODE_MUL) {
                            T k0 = l0 * r0, k1 = l0 * r1, k2 = l1 * r0, k3 = l1 * r1;
                            lo = A::mn(A::mn(k0, k1), A::mn(k2, k3));
                            hi = A::mx(A::mx(k0, k1), A::mx(k2, k3));
                        } else {
                            T d0 = A::mx(r0, T(1)), d1 = r1;
                            if (d0 <= d1) {
                                if (op == NODE_DIV) {
                                    T k0 = cdiv(l0, d0), k1 = cdiv(l0, d1), k2 = cdiv(l1, d0), k3 = cdiv(l1, d1);
                                    lo = A::mn(A::mn(k0, k1), A::mn(k2, k3));
                                    hi = A::mx(A::mx(k0, k1), A::mx(k2, k3));
                                } else {
                                    T m = d1 - T(1);
                                    lo = l0 >= T(0) ? T(0) : A::mx(l0, -m);
                                    hi = l1 <= T(0) ? T(0) : A::mn(l1, m);
                                }
                            }
                        }
                    }
                }
                VL(j) = lo;
                VH(j) = hi;
                if (lo <= hi) B = A::mx(B, A::mx(tabs(lo), tabs(hi)));
            }
            // narrowing targets, top-down from both roots
            auto fmag = [&](uint32_t j) -> T {
                T lo = VL(j), hi = VH(j);
                return lo <= hi ? A::mx(tabs(lo), tabs(hi)) : T(0);
            };
            T fl = fmag(lr), fr = fmag(rr), tl, tr;
            if (rel == REL_LT || rel == REL_GT) {
                tl = A::mx(INF, fr + T(1));
                tr = A::mx(INF, fl + T(1));
            } else if (rel == REL_LE || rel == REL_GE) {
                tl = A::mx(INF, fr);
                tr = A::mx(INF, fl);
            } else {
                tl = tr = A::mn(fl, fr);
            }
            int sp = 0;
            U(st_n, sp) = lr; E(st_0, sp) = tl; ++sp;
            U(st_n, sp) = rr; E(st_0, sp) = tr; ++sp;
            while (sp > 0) {
                --sp;
                uint32_t i = U(st_n, sp);
                T t = E(st_0, sp);
                B = A::mx(B, t);
                uint32_t cw = __ldg(code + i), op = op_of(cw);
                if (op < NODE_ADD) continue;
                uint32_t R = i - 1, L = R - size_of(R);
                if (sp + 2 > (int)st_cap) return 2;
                if (op == NODE_ADD || op == NODE_SUB) {
                    U(st_n, sp) = L; E(st_0, sp) = t + fmag(R); ++sp;
                    U(st_n, sp) = R; E(st_0, sp) = t + fmag(L); ++sp;
                } else if (op == NODE_MUL) {
                    U(st_n, sp) = L; E(st_0, sp) = A::mx(t, INF); ++sp;
                    U(st_n, sp) = R; E(st_0, sp) = A::mx(t, INF); ++sp;
                } else if (op == NODE_DIV) {
                    uint32_t rw = __ldg(code + R);
                    if (op_of(rw) == NODE_LIT) {
                        T c = E(lit, arg_of(rw));
                        if (c >= T(1)) { U(st_n, sp) = L; E(st_0, sp) = t * c + c; ++sp; }
                    }
                }
            }
            // exact-value magnitudes G (reuse VL: children precede parents)
            for (uint32_t j = start; j <= rr; ++j) {
                uint32_t cw = __ldg(code + j), op = op_of(cw);
                T g;
                if (op == NODE_LIT) g = tabs(E(lit, arg_of(cw)));
                else if (op == NODE_VAR) g = A::mx(tabs(E(env_lo, arg_of(cw))), tabs(E(env_hi, arg_of(cw))));
                else {
                    uint32_t R = j - 1, L = R - size_of(R);
                    T gl = VL(L), gr = VL(R);
                    if (op == NODE_ADD || op == NODE_SUB) g = gl + gr;
                    else if (op == NODE_MUL) g = gl * gr;
                    else if (op == NODE_DIV) g = gl;
                    else g = A::mn(gl, gr);
                }
                VL(j) = g;
                B = A::mx(B, g);
            }
        }
        if (B <= T(0x7FFFFFFFFFFFFFFFLL) && D <= T((long long)((1ull << 62) - 1))) return 0;
        const __int128 one = 1;
        if (B <= from_i128<T>((__int128)(~((unsigned __int128)0) >> 1)) && D <= from_i128<T>((one << 126) - 1))
            return 1;
        return 2;
    }

    // ----- x32 eligibility (int64 root kernel) -----------------------------------
    // Proof, at the current domains D0, that int32 reproduces the reference on
    // EVERY node of the subtree below (domains only shrink there, so every
    // forward interval at a descendant lies inside its interval at D0).  Each
    // narrowing target is tracked as the SET of values it can take at any
    // descendant: a real part (an interval, every value exact in int32) and a
    // far part (values derived from the 10**18 clamp; a lower bound on their
    // magnitude; lower targets are only ever far-negative, upper targets
    // far-positive).  The rules follow _Narrower.narrow (solver.py:159-226)
    // with the children's intervals ranging over their D0 intervals -- in
    // particular `*` is assumed to narrow whenever some descendant could make
    // both sides non-negative, `other_lo` may be 0 (clamp) or any value up to
    // its D0 maximum (real quotient), and far magnitudes shrink by the largest
    // divisor.  Eligible when every real value (domains, literals, forward
    // intervals, exact values, real targets) is below 2^28 and every far
    // value exceeds 2 B + 2, so Ext<int>'s +-2^30 stands in for it in every
    // comparison.  Doubles: real bounds are widened and far bounds shrunk by
    // a relative 1e-9 plus 1 (the margins are many orders larger).
    struct X32Tg {
        double rlo, rhi;  // real part (valid when rl)
        double fm;        // far part: magnitude lower bound (valid when fr)
        bool rl, fr;
    };
    struct X32Pair {
        X32Tg a, b;
    };
    __device__ bool fit_x32() {
        double B = 0.0, minf = 1e300;
        auto ad = [](T x) { return x < T(0) ? -(double)x : (double)x; };
        for (uint32_t v = 0; v < nv; ++v) B = fmax(B, fmax(ad(E(env_lo, v)), ad(E(env_hi, v))));
        for (uint32_t i = 0; i < nlit; ++i) B = fmax(B, ad(E(lit, i)));
        const double INFD = 1e18;
        auto up = [](double x) { return x + fabs(x) * 1e-9 + 1.0; };    // round a bound outward (up)
        auto dn = [](double x) { return x - fabs(x) * 1e-9 - 1.0; };    // ... (down)
        auto real = [&](double lo, double hi) { X32Tg t; t.rlo = dn(lo); t.rhi = up(hi); t.rl = true; t.fr = false; t.fm = 0; return t; };
        auto far = [](double m) { X32Tg t; t.rlo = t.rhi = 0; t.rl = false; t.fr = true; t.fm = m; return t; };
        auto none = []() { X32Tg t; t.rlo = t.rhi = t.fm = 0; t.rl = t.fr = false; return t; };
        auto join = [](X32Tg a, const X32Tg& b) {
            if (b.rl) {
                if (a.rl) { a.rlo = fmin(a.rlo, b.rlo); a.rhi = fmax(a.rhi, b.rhi); }
                else { a.rlo = b.rlo; a.rhi = b.rhi; a.rl = true; }
            }
            if (b.fr) { a.fm = a.fr ? fmin(a.fm, b.fm) : b.fm; a.fr = true; }
            return a;
        };
        constexpr int SMAX = 24;
        uint32_t sn[SMAX];
        X32Tg slo[SMAX], shi[SMAX];
        for (uint32_t k = 0; k < ncon; ++k) {
            uint32_t w = __ldg(cons + k);
            uint32_t rel = w & 7u, lr = (w >> 3) & 0x3FFFu, rr = w >> 17;
            uint32_t start = lr + 1 - size_of(lr);
            vbase = start;
            // forward intervals at D0 (exact in T)
            for (uint32_t j = start; j <= rr; ++j) {
                uint32_t cw = __ldg(code + j), op = op_of(cw);
                T lo, hi;
                if (op == NODE_LIT) {
                    lo = hi = E(lit, arg_of(cw));
                } else if (op == NODE_VAR) {
                    lo = E(env_lo, arg_of(cw));
                    hi = E(env_hi, arg_of(cw));
                } else {
                    uint32_t R = j - 1, L = R - size_of(R);
                    T l0 = VL(L), l1 = VH(L), r0 = VL(R), r1 = VH(R);
                    lo = T(1);
                    hi = T(0);
                    if (l0 <= l1 && r0 <= r1) {
                        if (op == NODE_ADD) { lo = l0 + r0; hi = l1 + r1; }
                        else if (op == NODE_SUB) { lo = l0 - r1; hi = l1 - r0; }
                        else if (op == NODE_MUL) {
                            T k0 = l0 * r0, k1 = l0 * r1, k2 = l1 * r0, k3 = l1 * r1;
                            lo = A::mn(A::mn(k0, k1), A::mn(k2, k3));
                            hi = A::mx(A::mx(k0, k1), A::mx(k2, k3));
                        } else {
                            T d0 = A::mx(r0, T(1)), d1 = r1;
                            if (d0 <= d1) {
                                if (op == NODE_DIV) {
                                    T k0 = cdiv(l0, d0), k1 = cdiv(l0, d1), k2 = cdiv(l1, d0), k3 = cdiv(l1, d1);
                                    lo = A::mn(A::mn(k0, k1), A::mn(k2, k3));
                                    hi = A::mx(A::mx(k0, k1), A::mx(k2, k3));
                                } else {
                                    T m = d1 - T(1);
                                    lo = l0 >= T(0) ? T(0) : A::mx(l0, -m);
                                    hi = l1 <= T(0) ? T(0) : A::mn(l1, m);
                                }
                            }
                        }
                    }
                }
                VL(j) = lo;
                VH(j) = hi;
                if (lo <= hi) B = fmax(B, fmax(ad(lo), ad(hi)));
            }
            auto defined = [&](uint32_t j) { return VL(j) <= VH(j); };
            auto F = [&](uint32_t j) -> double { return fmax(ad(VL(j)), ad(VH(j))); };
            // exact values are bounded by the magnitude recurrence
            {
                double g[64];
                uint32_t n = rr + 1 - start;
                if (n > 64) return false;
                for (uint32_t j = start; j <= rr; ++j) {
                    uint32_t cw = __ldg(code + j), op = op_of(cw);
                    double x;
                    if (op == NODE_LIT) x = ad(E(lit, arg_of(cw)));
                    else if (op == NODE_VAR) x = fmax(ad(E(env_lo, arg_of(cw))), ad(E(env_hi, arg_of(cw))));
                    else {
                        uint32_t R = j - 1, L = R - size_of(R);
                        double gl = g[L - start], gr = g[R - start];
                        x = op == NODE_ADD || op == NODE_SUB ? gl + gr : op == NODE_MUL ? gl * gr
                            : op == NODE_DIV ? gl : fmin(gl, gr);
                    }
                    g[j - start] = x;
                    B = fmax(B, x);
                }
            }
            // a constraint with an empty side fails before any narrowing, at D0
            // and (inclusion) at every descendant
            if (!defined(lr) || !defined(rr)) continue;
            const double L0 = (double)VL(lr), L1 = (double)VH(lr), R0 = (double)VL(rr), R1 = (double)VH(rr);
            int sp = 0;
            auto push = [&](uint32_t node, const X32Tg& lo, const X32Tg& hi) {
                sn[sp] = node;
                slo[sp] = lo;
                shi[sp] = hi;
                ++sp;
            };
            // root targets (solver.py:240-259); l0, l1 range over [L0, L1] etc.
            switch (rel) {
            case REL_LT: push(lr, far(INFD), real(R0 - 1, R1 - 1)); push(rr, real(L0 + 1, L1 + 1), far(INFD)); break;
            case REL_LE: push(lr, far(INFD), real(R0, R1)); push(rr, real(L0, L1), far(INFD)); break;
            case REL_EQ: {
                X32Tg lo = real(fmax(L0, R0), fmax(L1, R1)), hi = real(fmin(L0, R0), fmin(L1, R1));
                push(lr, lo, hi);
                push(rr, lo, hi);
                break;
            }
            case REL_GE: push(lr, real(R0, R1), far(INFD)); push(rr, far(INFD), real(L0, L1)); break;
            default:     push(lr, real(R0 + 1, R1 + 1), far(INFD)); push(rr, far(INFD), real(L0 - 1, L1 - 1)); break;
            }
            while (sp > 0) {
                --sp;
                const uint32_t i = sn[sp];
                const X32Tg lo = slo[sp], hi = shi[sp];
                if (lo.rl) B = fmax(B, fmax(fabs(lo.rlo), fabs(lo.rhi)));
                if (hi.rl) B = fmax(B, fmax(fabs(hi.rlo), fabs(hi.rhi)));
                if (lo.fr) minf = fmin(minf, lo.fm);
                if (hi.fr) minf = fmin(minf, hi.fm);
                uint32_t cw = __ldg(code + i), op = op_of(cw);
                if (op < NODE_ADD) continue;
                uint32_t R = i - 1, L = R - size_of(R);
                if (!defined(L) || !defined(R)) continue;  // _eval_iv None: contradiction, no narrowing
                if (sp + 2 > SMAX) return false;
                const double cl0 = (double)VL(L), cl1 = (double)VH(L), cr0 = (double)VL(R), cr1 = (double)VH(R);
                const double fL = F(L), fR = F(R);
                // target - [x0, x1] (sibling interval), far magnitudes shrink by its magnitude
                auto shift = [&](X32Tg t, double x0, double x1, double fx) {
                    if (t.rl) { t.rlo = dn(t.rlo - x1); t.rhi = up(t.rhi - x0); }
                    if (t.fr) t.fm = dn(t.fm - fx);
                    return t;
                };
                if (op == NODE_ADD) {  // (t0 - r1, t1 - r0) / (t0 - l1, t1 - l0)
                    push(R, shift(lo, cl0, cl1, fL), shift(hi, cl0, cl1, fL));
                    push(L, shift(lo, cr0, cr1, fR), shift(hi, cr0, cr1, fR));
                } else if (op == NODE_SUB) {
                    // right: (l0 - t1, l1 - t0); a far upper becomes a far lower and vice versa
                    auto neg = [&](X32Tg t) {  // [l0, l1] - t
                        X32Tg o = t;
                        if (t.rl) { o.rlo = dn(cl0 - t.rhi); o.rhi = up(cl1 - t.rlo); }
                        if (t.fr) o.fm = dn(t.fm - fL);
                        return o;
                    };
                    push(R, neg(hi), neg(lo));
                    // left: (t0 + r0, t1 + r1)
                    push(L, shift(lo, -cr1, -cr0, fR), shift(hi, -cr1, -cr0, fR));
                } else if (op == NODE_MUL) {
                    // narrows only when l0 >= 0 and r0 >= 0 at the node: possible
                    // at some descendant iff both D0 maxima are >= 0
                    if (cl1 < 0 || cr1 < 0) continue;
                    auto side = [&](double o0, double o1) {  // other side's interval (clipped to >= 0)
                        o0 = fmax(o0, 0.0);
                        X32Tg nlo = none(), nhi = none();
                        // lo_req: -INF when t0n = max(t0, 0) <= 0, else ceil(t0n / other_hi), other_hi in [1, o1]
                        if (lo.fr || (lo.rl && lo.rlo <= 0)) nlo = join(nlo, far(INFD));
                        if (lo.rl && lo.rhi > 0 && o1 >= 1) nlo = join(nlo, real(fmax(lo.rlo, 1.0) / o1, lo.rhi));
                        // hi_req: INF when other_lo = 0, else t1 // other_lo, other_lo in [max(o0, 1), o1]
                        if (o0 <= 0) nhi = join(nhi, far(INFD));
                        if (o1 >= 1) {
                            if (hi.rl && hi.rhi >= 0) nhi = join(nhi, real(fmax(hi.rlo, 0.0) / o1, hi.rhi));
                            if (hi.fr) nhi = join(nhi, far(dn(hi.fm / o1)));
                        }
                        return X32Pair{nlo, nhi};
                    };
                    auto pl = side(cr0, cr1), pr = side(cl0, cl1);
                    push(R, pr.a, pr.b);
                    push(L, pl.a, pl.b);
                } else if (op == NODE_DIV) {
                    uint32_t rw = __ldg(code + R);
                    if (op_of(rw) == NODE_LIT) {
                        const T cc = E(lit, arg_of(rw));
                        if (cc >= T(1)) {
                            const double c = (double)cc;
                            auto sc = [&](X32Tg t) {  // t * c (+- (c - 1))
                                if (t.rl) { t.rlo = dn(t.rlo * c - (c - 1.0)); t.rhi = up(t.rhi * c + (c - 1.0)); }
                                if (t.fr) t.fm = dn(t.fm);  // |t * c +- (c - 1)| >= |t|
                                return t;
                            };
                            push(L, sc(lo), sc(hi));
                        }
                    }
                }
            }
        }
        const double LIM = 268435456.0;  // 2^28
        return B < LIM && minf > 2.0 * B + 2.0;
    }

    __device__ void undo_to(uint32_t mark) {
        while (trail_len > mark) {
            --trail_len;
            uint32_t v = U(tr_var, trail_len);
            E(env_lo, v) = E(tr_lo, trail_len);
            E(env_hi, v) = E(tr_hi, trail_len);
        }
    }

    // ----- DFS steps of _search (solver.py:397-415) ---------------------------
    // smallest unresolved domain, ties by declaration order (:397-404); -1: leaf
    __device__ int pick_var() const {
        int pick = -1;
        T best = T(0);
        for (uint32_t v = 0; v < nv; ++v) {
            T lo = E(env_lo, v), hi = E(env_hi, v);
            if (lo < hi) {
                T size = hi - lo + T(1);
                if (pick < 0 || size < best) {
                    pick = (int)v;
                    best = size;
                }
            }
        }
        return pick;
    }

    // push a frame and enter the lower half (:408-413); false on capacity error
    __device__ bool split(uint32_t pick) {
        if (depth >= g->depth_cap) {
            err = ERR_DEPTH;
            return false;
        }
        T lo = E(env_lo, pick), hi = E(env_hi, pick);
        T mid = (lo + hi) >> 1;  // floor((lo + hi) / 2) in two's complement
        U(fr_pick, depth) = pick;
        U(fr_mark, depth) = trail_len;
        E(fr_mid, depth) = mid;
        E(fr_hi, depth) = hi;
        uint32_t* c = fr_clean + (size_t)depth * 4 * 32;
        c[0] = (uint32_t)clean0;
        c[32] = (uint32_t)(clean0 >> 32);
        c[64] = (uint32_t)clean1;
        c[96] = (uint32_t)(clean1 >> 32);
        ++depth;
        ++seg;
        return set_dom(pick, lo, mid);
    }

    // after a dead node: enter the next upper half (:414-416).  Returns 1 if a
    // new node is ready, 0 if the search space is exhausted (Unsat), -1 error.
    __device__ int backtrack() {
        for (;;) {
            if (depth == 0) return 0;
            uint32_t f = depth - 1;
            uint32_t pk = U(fr_pick, f);
            undo_to(U(fr_mark, f));
            if (!(pk & 0x80000000u)) {
                U(fr_pick, f) = pk | 0x80000000u;
                uint32_t* c = fr_clean + (size_t)f * 4 * 32;
                clean0 = ((uint64_t)c[32] << 32) | c[0];
                clean1 = ((uint64_t)c[96] << 32) | c[64];
                ++seg;
                return set_dom(pk, E(fr_mid, f) + T(1), E(fr_hi, f)) ? 1 : -1;
            }
            depth = f;
        }
    }
};

}  // namespace oob
