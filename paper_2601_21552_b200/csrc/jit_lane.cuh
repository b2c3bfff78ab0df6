// jit_lane.cuh -- the compiled lane: one structure class specialised at run
// time (jit.cpp generates the class struct C and compiles it with NVRTC).
//
// The interpreting Lane<T> (engine.cuh) walks the class's code words and keeps
// domains and forward intervals in lane-minor shared memory.  JitLane<C>
// executes the SAME algorithm (solver.py:112-416, the identical narrowing
// order, 10**18 clamp, pass structure and constraint skipping) but the
// structure is compile-time: every term node is straight-line register code,
// domains and literals live in registers, and only the DFS frames and the
// trail (dynamically indexed) stay in the per-warp global slab.
//
// C (generated) provides
//   NV, NCON, NLIT                  variables, constraints (<= 128), literals
//   M0(v), M1(v)                    membership masks: constraints 0-63 / 64-127
//                                   that mention variable v
//   template <class L> static bool prop(L&, k)      one constraint (a4-a6)
//   template <class L> static void pass(L&, bool&)  one pass over the dirty
//                                                   constraints (a3)
//   template <class L> static bool check(L&)        check_model at env lo (a7)
#pragma once
#include "phases.cuh"

namespace oob {

template <class C>
struct JitLane {
    using T = typename C::T;  // long long (int64 regime) or int (x32 regime)
    using A = Arith<T>;
    static constexpr uint32_t NV = C::NV;
    static constexpr uint32_t NL = C::NLIT > 0 ? C::NLIT : 1;

    T lo[NV], hi[NV];
    T lit[NL];
    // per-warp global slab, lane-minor (element i of this lane is p[i * 32])
    T *fr_mid, *fr_hi, *tr_lo, *tr_hi;
    uint32_t *fr_pick, *fr_mark, *fr_clean, *tr_var, *stamp;
    const uint32_t* member;  // the class's membership words (dynamic-index touch)
    uint32_t trail_cap, depth_cap;
    uint32_t depth, trail_len, seg;
    uint64_t clean0, clean1;
    bool dirty, changed;
    int err;

    // ----- lane interface (phases.cuh) ------------------------------------------
    __device__ __forceinline__ void bind(const LaunchArgs& a, uint32_t warp, uint32_t lane) {
        const SlabGeom& g = a.g;
        T* sT = reinterpret_cast<T*>(a.slab_T) + (size_t)warp * g.slab_T_words + lane;
        uint32_t* sU = a.slab_u32 + (size_t)warp * g.slab_u32_words + lane;
        fr_mid = sT + g.o_fr_mid;
        fr_hi = sT + g.o_fr_hi;
        tr_lo = sT + g.o_tr_lo;
        tr_hi = sT + g.o_tr_hi;
        fr_pick = sU + g.o_fr_pick;
        fr_mark = sU + g.o_fr_mark;
        fr_clean = sU + g.o_fr_clean;
        tr_var = sU + g.o_tr_var;
        stamp = sU + g.o_stamp;
        member = a.code + a.classes[0].code_off + C::NCON + C::NCODE;
        trail_cap = g.trail_cap;
        depth_cap = g.depth_cap;
        seg = 0;
        depth = trail_len = 0;
        clean0 = clean1 = 0;
        err = ERR_NONE;
        changed = dirty = false;
    }
    __device__ __forceinline__ void set_class(const LaunchArgs&, const ClassDesc&) {}
    __device__ __forceinline__ void load(const LaunchArgs& a, const QDesc& d) { load_from(a.data, d); }
    __device__ __forceinline__ void save_state(int64_t* base, const QDesc& d) const {
        T* dst = reinterpret_cast<T*>(base + d.data_off);
#pragma unroll
        for (uint32_t v = 0; v < NV; ++v) {
            dst[2 * v] = lo[v];
            dst[2 * v + 1] = hi[v];
        }
#pragma unroll
        for (uint32_t i = 0; i < C::NLIT; ++i) dst[2 * NV + i] = lit[i];
    }
    __device__ __forceinline__ void load_from(const int64_t* base, const QDesc& d) {
        const T* src = reinterpret_cast<const T*>(base + d.data_off);
#pragma unroll
        for (uint32_t v = 0; v < NV; ++v) {
            lo[v] = src[2 * v];
            hi[v] = src[2 * v + 1];
            stamp[(size_t)v * 32] = 0xFFFFFFFFu;
        }
#pragma unroll
        for (uint32_t i = 0; i < C::NLIT; ++i) lit[i] = src[2 * NV + i];
        err = ERR_NONE;
        depth = 0;
        trail_len = 0;
        clean0 = clean1 = 0;
    }
    __device__ __forceinline__ uint32_t nvars() const { return NV; }
    __device__ __forceinline__ T get_lo(uint32_t v) const {
        T r = lo[0];
#pragma unroll
        for (uint32_t i = 1; i < NV; ++i)
            if (v == i) r = lo[i];
        return r;
    }
    __device__ __forceinline__ T get_hi(uint32_t v) const {
        T r = hi[0];
#pragma unroll
        for (uint32_t i = 1; i < NV; ++i)
            if (v == i) r = hi[i];
        return r;
    }
    __device__ __forceinline__ void put_env(uint32_t v, T l, T h) {
#pragma unroll
        for (uint32_t i = 0; i < NV; ++i)
            if (v == i) {
                lo[i] = l;
                hi[i] = h;
            }
    }
    // whole domain vectors, constant indices (no select chains)
    __device__ __forceinline__ void load_env(const T* env) {
#pragma unroll
        for (uint32_t v = 0; v < NV; ++v) {
            lo[v] = env[2 * v];
            hi[v] = env[2 * v + 1];
        }
    }
    __device__ __forceinline__ void store_env(T* env) const {
#pragma unroll
        for (uint32_t v = 0; v < NV; ++v) {
            env[2 * v] = lo[v];
            env[2 * v + 1] = hi[v];
        }
    }
    __device__ __forceinline__ void store_model(int64_t* m) const {
#pragma unroll
        for (uint32_t v = 0; v < NV; ++v) store_i128(m + 2 * v, lo[v]);
    }
    __device__ __forceinline__ bool pass_sync(bool run) {
        bool dead = false;
        if (run) C::pass(*this, dead);
        return dead;
    }
    __device__ __forceinline__ bool check_env() { return C::check(*this); }

    // ----- constraint skipping (engine.cuh header) ----------------------------
    __device__ __forceinline__ bool is_clean(uint32_t k) const {
        return k < 64 ? ((clean0 >> k) & 1ull) : ((clean1 >> (k - 64)) & 1ull);
    }
    __device__ __forceinline__ void set_clean(uint32_t k) {
        if (k < 64) clean0 |= 1ull << k;
        else clean1 |= 1ull << (k - 64);
    }
    // one (dirty) constraint inside a pass; false = contradiction
    template <class P>
    __device__ __forceinline__ bool pass_constraint(uint32_t k, P prop) {
        bool before = changed;
        changed = false;
        bool ok = prop();
        if (ok && !changed) set_clean(k);
        changed = changed || before;
        return ok;
    }

    // ----- domain updates --------------------------------------------------------
    // trail entry for variable v (its domain before the first change in this
    // DFS segment); false on capacity overflow
    __device__ __forceinline__ bool trail(uint32_t v, T ol, T oh) {
        if (depth > 0 && stamp[(size_t)v * 32] != seg) {
            if (trail_len >= trail_cap) {
                err = ERR_TRAIL;
                return false;
            }
            tr_var[(size_t)trail_len * 32] = v;
            tr_lo[(size_t)trail_len * 32] = ol;
            tr_hi[(size_t)trail_len * 32] = oh;
            ++trail_len;
            stamp[(size_t)v * 32] = seg;
        }
        return true;
    }
    // i is a compile-time constant after inlining (narrowing sites)
    __device__ __forceinline__ bool set_dom_i(uint32_t i, T l, T h) {
        if (!trail(i, lo[i], hi[i])) return false;
        lo[i] = l;
        hi[i] = h;
        clean0 &= ~C::M0(i);
        clean1 &= ~C::M1(i);
        return true;
    }
    // v dynamic (DFS split / backtrack / frontier child): one select chain per
    // access instead of an unrolled copy of set_dom_i per variable
    __device__ __forceinline__ bool set_dom(uint32_t v, T l, T h) {
        if (!trail(v, get_lo(v), get_hi(v))) return false;
        put_env(v, l, h);
        const uint32_t* m = member + 4 * v;
        clean0 &= ~(((uint64_t)__ldg(m + 1) << 32) | __ldg(m));
        clean1 &= ~(((uint64_t)__ldg(m + 3) << 32) | __ldg(m + 2));
        return true;
    }
    // _Narrower.narrow on a VarRef (solver.py:165-173)
    __device__ __forceinline__ bool narrow_var(uint32_t i, T a, T b) {
        T l = lo[i], h = hi[i];
        T nl = A::mx(l, a), nh = A::mn(h, b);
        if (nl > nh) return false;
        if (nl != l || nh != h) {
            if (!set_dom_i(i, nl, nh)) return false;
            changed = true;
            dirty = true;
        }
        return true;
    }
    // leaf fast path (both constraint sides are a variable or a literal)
    __device__ __forceinline__ bool narrow_leaf_var(uint32_t i, T a, T b) {
        if (a > b) return false;
        T l = lo[i], h = hi[i];
        T nl = A::mx(l, a), nh = A::mn(h, b);
        if (nl > nh) return false;
        if (nl != l || nh != h) {
            if (!set_dom_i(i, nl, nh)) return false;
            changed = true;
        }
        return true;
    }

    // ----- DFS (solver.py:397-415) -------------------------------------------
    __device__ __forceinline__ int pick_var() const {
        int pick = -1;
        T best = 0;
#pragma unroll
        for (uint32_t v = 0; v < NV; ++v) {
            if (lo[v] < hi[v]) {
                T size = hi[v] - lo[v] + 1;
                if (pick < 0 || size < best) {
                    pick = (int)v;
                    best = size;
                }
            }
        }
        return pick;
    }
    __device__ __forceinline__ bool split(uint32_t pick) {
        if (depth >= depth_cap) {
            err = ERR_DEPTH;
            return false;
        }
        T l = get_lo(pick), h = get_hi(pick);
        T mid = (l + h) >> 1;  // floor((lo + hi) / 2)
        fr_pick[(size_t)depth * 32] = pick;
        fr_mark[(size_t)depth * 32] = trail_len;
        fr_mid[(size_t)depth * 32] = mid;
        fr_hi[(size_t)depth * 32] = h;
        uint32_t* c = fr_clean + (size_t)depth * 4 * 32;
        c[0] = (uint32_t)clean0;
        c[32] = (uint32_t)(clean0 >> 32);
        c[64] = (uint32_t)clean1;
        c[96] = (uint32_t)(clean1 >> 32);
        ++depth;
        ++seg;
        return set_dom(pick, l, mid);
    }
    __device__ __forceinline__ void undo_to(uint32_t mark) {
        while (trail_len > mark) {
            --trail_len;
            uint32_t v = tr_var[(size_t)trail_len * 32];
            put_env(v, tr_lo[(size_t)trail_len * 32], tr_hi[(size_t)trail_len * 32]);
        }
    }
    __device__ __forceinline__ int backtrack() {
        for (;;) {
            if (depth == 0) return 0;
            uint32_t f = depth - 1;
            uint32_t pk = fr_pick[(size_t)f * 32];
            undo_to(fr_mark[(size_t)f * 32]);
            if (!(pk & 0x80000000u)) {
                fr_pick[(size_t)f * 32] = pk | 0x80000000u;
                uint32_t* c = fr_clean + (size_t)f * 4 * 32;
                clean0 = ((uint64_t)c[32] << 32) | c[0];
                clean1 = ((uint64_t)c[96] << 32) | c[64];
                ++seg;
                return set_dom(pk, fr_mid[(size_t)f * 32] + 1, fr_hi[(size_t)f * 32]) ? 1 : -1;
            }
            depth = f;
        }
    }
};

// The compiled solve kernel of class C: lockstep phase over the class's queue,
// then the frontier phase over the class's heavy list.
template <class C>
__device__ __forceinline__ void jit_solve(const LaunchArgs& a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    JitLane<C> L;
    const uint32_t slot = claim_slab(a, warp, lane);
    L.bind(a, slot, lane);
    lockstep_phase(a, L, warp, lane);
    frontier_phase(a, L, warp, lane);
    release_slab(a, slot, lane);
}

}  // namespace oob
