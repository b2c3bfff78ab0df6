// phases.cuh -- the scheduling phases of the solve kernels, generic over the
// lane type (the interpreting Lane<T> of engine.cuh or a compiled JitLane of
// jit_lane.cuh).  A lane type provides: T, set_class, load, get_lo/get_hi,
// put_env, load_env/store_env/store_model (whole domain vectors), nvars,
// pass_sync, check_env, pick_var, split, set_dom, backtrack,
// and the fields changed, err, depth, clean0, clean1.
#pragma once
#include "engine.cuh"
#include "frontier.cuh"
#include "symbolic.cuh"

namespace oob {

enum : int { PH_IDLE = 0, PH_NODE = 1, PH_PASS = 2, PH_DONE = 3, PH_POST = 4 };

// Phase 1 of the solve kernel: lockstep class queues (returns when the warp's
// lanes are idle and every class queue is drained).
template <typename LaneT>
__device__ __forceinline__ void lockstep_phase(const LaunchArgs& a, LaneT& L, uint32_t warp, uint32_t lane) {
    const unsigned FULL = 0xffffffffu;
    const unsigned lt_mask = (1u << lane) - 1u;

    if (lane == 0) atomicAdd(a.heavy_count + 2, 1u);  // a producer of this launch's heavy list
    uint32_t c = a.warp_class ? a.warp_class[warp] : 0u;  // the warp's current class queue (warp-uniform)
    if (c == NO_CLASS) return;
    ClassDesc cd = a.classes[c];
    L.set_class(a, cd);
    bool drained = false;             // every class queue is empty

    int phase = PH_IDLE;
    uint32_t qi = 0;
    int64_t nodes = 0, passes = 0;
    int pin = 0;
    int verdict = VERDICT_UNSAT;
    uint64_t t0 = 0, deadline = 0;

    for (;;) {
        // ---- refill idle lanes from the warp's class queue; when it runs dry
        // move the queue on to the next class with work (lanes still busy keep
        // their own class: every lane carries its own code pointers) ----
        unsigned idle = __ballot_sync(FULL, phase == PH_IDLE);
        while (idle && !drained) {
            uint32_t base = 0;
            int leader = __ffs(idle) - 1;
            if ((int)lane == leader) base = atomicAdd(a.class_next + c, (uint32_t)__popc(idle));
            base = __shfl_sync(FULL, base, leader);
            if (phase == PH_IDLE) {
                uint32_t q = base + __popc(idle & lt_mask);
                if (q < cd.q_end) {
                    const uint32_t rs = a.resume ? a.resume[q] : 0u;
                    if (rs != RES_SKIP) {
                        qi = q;
                        L.set_class(a, cd);
                        const QDesc d = a.qdesc[qi];
                        L.load(a, d);
                        if (rs & RES_ROOT) {  // demoted: resume the root node (format.h)
                            nodes = 1;
                            passes = rs & RES_PASSES;
                            pin = (int)passes;
                            t0 = a.heavy_t0[qi];
                            phase = (rs & RES_FIX) ? PH_POST : PH_PASS;
                        } else {
                            nodes = passes = 0;
                            t0 = global_ns();
                            phase = PH_NODE;
                        }
                        deadline = a.timeout_ns ? t0 + a.timeout_ns : 0;
                        if (a.timeline) a.timeline[4 * (size_t)qi] = t0;
                    }
                }
            }
            idle = __ballot_sync(FULL, phase == PH_IDLE);
            if (idle && *(volatile uint32_t*)(a.class_next + c) >= cd.q_end) {
                // class c is exhausted: find the next class with work
                bool found = false;
                for (uint32_t s = 1; s <= a.n_classes && !found; ++s) {
                    uint32_t c2 = (c + s) % a.n_classes;
                    if (*(volatile uint32_t*)(a.class_next + c2) < a.classes[c2].q_end) {
                        c = c2;
                        found = true;
                    }
                }
                if (found) cd = a.classes[c];
                else drained = true;
            }
        }
        unsigned active = __ballot_sync(FULL, phase != PH_IDLE);
        if (!active) break;

        // ---- node start (_search, solver.py:391-393) ----
        // (fast mode: only while some frontier warp of this launch waits for
        // an entry -- a queue behind busy frontier warps is slower than
        // staying here; the check repeats every pass)
        if ((phase == PH_NODE || phase == PH_PASS) && a.heavy_nodes &&
            ((phase == PH_NODE && nodes >= a.heavy_nodes) || (a.heavy_passes && passes >= a.heavy_passes)) &&
            (!a.handoff_gate ||
             ((volatile uint32_t*)a.heavy_count)[4] > ((volatile uint32_t*)a.heavy_count)[0] -
                                                          ((volatile uint32_t*)a.heavy_count)[1])) {
            // a heavy search (many nodes, or a long propagation chain): hand
            // it to the warp-cooperative frontier phase, which restarts it
            // from the root in a warp of its own (so a long chain no longer
            // shares its warp's steps with 31 other queries); the list entry
            // is published after the start time it carries
            if (phase == PH_PASS && nodes == 1 && a.handoff) {
                // still at the root node, between two passes (the last one
                // changed something): the frontier resumes here instead of
                // redoing these passes (the same resume as regime demotion)
                L.save_state(a.handoff, a.qdesc[qi]);
                a.resume[qi] = RES_ROOT | RES_HANDOFF | passes;
            }
            uint32_t slot = atomicAdd(a.heavy_count, 1u);
            a.heavy_t0[qi] = t0;
            if (a.timeline) a.timeline[4 * (size_t)qi + 1] = global_ns();
            __threadfence();
            *(volatile uint32_t*)(a.heavy_list + slot) = qi + 1u;
            phase = PH_IDLE;
        }
        if (phase == PH_NODE) {
            if ((deadline && global_ns() > deadline) || (a.node_budget > 0 && nodes >= a.node_budget)) {
                verdict = VERDICT_TIMEOUT;
                phase = PH_DONE;
            } else {
                ++nodes;
                pin = 0;
                phase = PH_PASS;
            }
        }
        // ---- pass start (propagate, solver.py:271-274) ----
        const bool in_pass = (phase == PH_PASS);
        bool dead = false;
        if (in_pass) {
            if (deadline && global_ns() > deadline) {
                verdict = VERDICT_TIMEOUT;
                phase = PH_DONE;
            } else {
                ++passes;
                ++pin;
                L.changed = false;
            }
        }
        // a resumed root node whose last pass (in the root kernel) changed
        // nothing: only the pass-end step remains
        const bool post = (phase == PH_POST);
        if (post) {
            L.changed = false;
            phase = PH_PASS;
        }
        const bool run = (phase == PH_PASS) && !post;
        // ---- the pass: constraint loop (solver.py:275-277) ----
        dead = L.pass_sync(run);
        if (a.stats) {  // [4] warp steps x 32 [5] lanes in a pass
            unsigned r = __ballot_sync(FULL, run);
            if (lane == 0) {
                atomicAdd(a.stats + 4, 32ull);
                atomicAdd(a.stats + 5, (unsigned long long)__popc(r));
            }
        }
        // ---- pass end ----
        if (run || post) {
            if (dead) {
                if (L.err) {
                    verdict = VERDICT_ERROR;
                    phase = PH_DONE;
                } else {
                    int r = L.backtrack();
                    if (r <= 0) {
                        verdict = r == 0 ? VERDICT_UNSAT : VERDICT_ERROR;
                        phase = PH_DONE;
                    } else {
                        phase = PH_NODE;
                    }
                }
            } else if (L.changed && pin < PASS_CAP) {
                // another pass of this node
            } else {
                int pick = L.pick_var();
                if (pick < 0) {                                        // leaf (:405-407)
                    if (L.check_env()) {
                        verdict = VERDICT_SAT;
                        phase = PH_DONE;
                    } else {
                        int r = L.backtrack();
                        if (r <= 0) {
                            verdict = r == 0 ? VERDICT_UNSAT : VERDICT_ERROR;
                            phase = PH_DONE;
                        } else {
                            phase = PH_NODE;
                        }
                    }
                } else if (L.split((uint32_t)pick)) {                 // (:408-413)
                    phase = PH_NODE;
                } else {
                    verdict = VERDICT_ERROR;
                    phase = PH_DONE;
                }
            }
        }
        // ---- finished lanes publish their result and go idle ----
        if (phase == PH_DONE) {
            const QDesc d = a.qdesc[qi];
            a.verdict[qi] = (int8_t)verdict;
            a.err[qi] = (int8_t)L.err;
            a.nodes[qi] = nodes;
            a.passes[qi] = passes;
            a.elapsed[qi] = (float)((double)(global_ns() - t0) * 1e-9);
            if (a.timeline) a.timeline[4 * (size_t)qi + 3] = global_ns();
            if (verdict == VERDICT_SAT) {
                int64_t* m = a.model + 2 * d.out_v;
                L.store_model(m);
            }
            phase = PH_IDLE;
        }
    }
}

// Phase 2 of the solve kernel: heavy queries, one warp per query, lanes
// expand the leftmost pending nodes (frontier.cuh).  A warp whose lockstep
// phase is over serves the heavy list; when the list is empty it waits while
// warps of the same launch are still in their lockstep phase (they may hand
// off more: a warp of creeping chains hands off 32 at once, and a lone
// producer would then serve them one after another) -- only warps that have
// STARTED count, so no warp ever waits on a block that is not resident -- and
// exits once every started producer is done (or after frontier_wait_us).  An entry
// appended after that comes from a warp still in its lockstep phase, which
// serves the list itself afterwards, so every entry is taken.
// first free region of the job's pool (bitmap, starting at a warp-dependent
// word to spread contention); spins while all are held
__device__ __forceinline__ uint32_t claim_region(uint32_t* bitmap, uint32_t n, uint32_t warp) {
    const uint32_t words = (n + 31) >> 5;
    uint32_t w = (warp * 2654435761u) % words;
    for (uint32_t tries = 0;; tries++) {
        const uint32_t valid = (w == words - 1 && (n & 31)) ? ((1u << (n & 31)) - 1u) : 0xffffffffu;
        uint32_t freeb = ~*(volatile uint32_t*)(bitmap + w) & valid;
        while (freeb) {
            const uint32_t b = __ffs(freeb) - 1;
            const uint32_t old = atomicOr(bitmap + w, 1u << b);
            if (!(old & (1u << b))) {
                __threadfence();
                return w * 32 + b;
            }
            freeb = ~old & valid;
        }
        w = (w + 1) % words;
        if (tries % words == words - 1) __nanosleep(2000);
    }
}

// slab of a SOLVE-kernel warp: from the job's pool, held for the warp's life
__device__ __forceinline__ uint32_t claim_slab(const LaunchArgs& a, uint32_t warp, uint32_t lane) {
    if (!a.slab_bitmap) return warp;
    uint32_t slot = 0;
    if (lane == 0) slot = claim_region(a.slab_bitmap, a.slab_nslots, warp);
    return __shfl_sync(0xffffffffu, slot, 0);
}
__device__ __forceinline__ void release_slab(const LaunchArgs& a, uint32_t slot, uint32_t lane) {
    __syncwarp();
    if (a.slab_bitmap && lane == 0) {
        __threadfence();
        atomicAnd(a.slab_bitmap + (slot >> 5), ~(1u << (slot & 31)));
    }
}

// exact values of a job's value type for the symbolic prover (the 256-bit
// regime stays with the exact emulation)
template <typename T>
struct SymVal {
    static constexpr bool ok = false;
    __device__ static sym::i128 get(const T&) { return 0; }
};
template <>
struct SymVal<int> {
    static constexpr bool ok = true;
    __device__ static sym::i128 get(const int& x) { return x; }
};
template <>
struct SymVal<long long> {
    static constexpr bool ok = true;
    __device__ static sym::i128 get(const long long& x) { return x; }
};
template <>
struct SymVal<__int128> {
    static constexpr bool ok = true;
    __device__ static sym::i128 get(const __int128& x) { return x; }
};

// fast mode: the warp tries to refute query d symbolically (symbolic.cuh);
// lane 0 builds the store, the lanes then search from one target each.  The
// warp's frontier region is the scratch (the frontier re-initialises what it
// uses).  src: the query's domains + literal slots in the job's layout.
template <typename T>
__device__ __noinline__ bool sym_refute_warp(const LaunchArgs& a, const QDesc& d, const T* src,
                                             unsigned char* region, uint32_t lane) {
    if (!SymVal<T>::ok) return false;
    const unsigned FULL = 0xffffffffu;
    sym::Store& S = *reinterpret_cast<sym::Store*>(region);
    sym::LaneWork* W = reinterpret_cast<sym::LaneWork*>(region + sizeof(sym::Store));
    const uint32_t nv = d.nv_ncon & 0xFFFFu, ncon = d.nv_ncon >> 16;
    const uint32_t* cons = a.code + d.code_off;
    const uint32_t* code = cons + ncon;
    int r = sym::R_UNKNOWN;
    const long long c0 = clock64();
    if (lane == 0) {
        auto dom = [&](uint32_t i) -> sym::i128 { return SymVal<T>::get(src[i]); };
        auto lit = [&](uint32_t i) -> sym::i128 { return SymVal<T>::get(src[2 * nv + i]); };
        r = sym::prepare(S, W[0], cons, code, nv, ncon, dom, lit);
    }
    r = __shfl_sync(FULL, r, 0);
    __syncwarp();
    const long long c1 = clock64();
    if (a.fast_stats && lane == 0) atomicAdd(a.fast_stats + 2, (unsigned long long)(c1 - c0));
    if (r != sym::R_CONTINUE) return r == sym::R_REFUTED;
    const int nc = S.nc;
    bool refuted = false;  // warp-uniform
    for (int t0 = 0; t0 < nc && !refuted; t0 += 32) {
        const int t = t0 + (int)lane;
        const bool found = t < nc && sym::greedy_target(S, t, W[lane]);
        refuted = __any_sync(FULL, found);
    }
    if (a.fast_stats && lane == 0) atomicAdd(a.fast_stats + 3, (unsigned long long)(clock64() - c1));
    return refuted;
}

template <typename LaneT>
__device__ __forceinline__ void frontier_phase(const LaunchArgs& a, LaneT& L, uint32_t warp, uint32_t lane) {
    const unsigned FULL = 0xffffffffu;
    volatile uint32_t* ctl = a.heavy_count;  // [0] listed [1] claimed [2] lockstep started [3] lockstep done
                                             // [4] frontier warps waiting for an entry
    if (!a.frontier_only && lane == 0) {
        __threadfence();
        atomicAdd(a.heavy_count + 3, 1u);
    }
    if (!a.heavy_nodes) return;
    const uint64_t WAIT_NS = 1000ull * a.frontier_wait_us;  // bound on waiting for producers
    uint64_t idle_since = 0;
    FrontierRegion<typename LaneT::T> R;  // scratch region, claimed per heavy query
    for (;;) {
        int idx = -1;
        if (lane == 0) {
            bool waiting = false;
            for (;;) {
                const uint32_t done = ctl[3], started = ctl[2];
                __threadfence();
                const uint32_t listed = ctl[0], claimed = ctl[1];
                if (claimed < listed) {
                    if (atomicCAS(a.heavy_count + 1, claimed, claimed + 1) == claimed) {
                        idx = (int)claimed;
                        idle_since = 0;
                        break;
                    }
                    continue;
                }
                if (done >= started || !WAIT_NS) break;  // no producer of this launch left
                if (!waiting) {
                    waiting = true;
                    atomicAdd(a.heavy_count + 4, 1u);
                }
                const uint64_t now = global_ns();
                if (!idle_since) idle_since = now;
                else if (now - idle_since > WAIT_NS) break;
                __nanosleep(4000);
            }
            if (waiting) atomicSub(a.heavy_count + 4, 1u);
        }
        idx = __shfl_sync(FULL, idx, 0);
        if (idx < 0) break;
        uint32_t e = 0;
        if (lane == 0)
            while ((e = *(volatile uint32_t*)(a.heavy_list + idx)) == 0u) __nanosleep(100);
        e = __shfl_sync(FULL, e, 0);
        __threadfence();
        const uint32_t qi = e - 1u;
        if (a.timeline && lane == 0) a.timeline[4 * (size_t)qi + 2] = global_ns();
        const QDesc d = a.qdesc[qi];
        ClassDesc cd;
        cd.code_off = d.code_off;
        cd.nv_ncon = d.nv_ncon;
        cd.ncode_nlit = d.ncode_nlit;
        L.set_class(a, cd);
        const uint32_t rs0 = a.resume ? a.resume[qi] : 0u;
        if ((rs0 & RES_HANDOFF) && a.handoff) L.load_from(a.handoff, d);
        else L.load(a, d);
        // a scratch region of the job's pool, held for this query only (every
        // query re-initialises what it uses); a waiter always gets one in the
        // end because holders release theirs without waiting on anything
        uint32_t region = 0;
        if (lane == 0) region = claim_region(a.fr_bitmap, a.fr_nregions, warp);
        region = __shfl_sync(FULL, region, 0);
        unsigned char* rbase = (unsigned char*)a.fr_region + (size_t)region * a.fr_region_bytes;
#if !defined(OOB_JIT)  // (the run-time compiled classes never run the frontier prover)
        if (a.fast) {
            typedef typename LaneT::T VT;
            const VT* src = reinterpret_cast<const VT*>(((rs0 & RES_HANDOFF) && a.handoff ? a.handoff : a.data) +
                                                        d.data_off);
            const bool refuted = sym_refute_warp<VT>(a, d, src, rbase, lane);
            if (lane == 0 && a.fast_stats) {
                atomicAdd(a.fast_stats, 1ull);
                if (refuted) atomicAdd(a.fast_stats + 1, 1ull);
            }
            if (refuted) {
                if (lane == 0) {
                    a.verdict[qi] = (int8_t)VERDICT_UNSAT;
                    a.err[qi] = 0;
                    a.nodes[qi] = 0;
                    a.passes[qi] = 0;
                    a.elapsed[qi] = (float)((double)(global_ns() - a.heavy_t0[qi]) * 1e-9);
                    if (a.timeline) a.timeline[4 * (size_t)qi + 3] = global_ns();
                    __threadfence();
                    atomicAnd(a.fr_bitmap + (region >> 5), ~(1u << (region & 31)));
                }
                __syncwarp();
                continue;
            }
        }
#endif
        R.bind(rbase, a.g.maxv, a.fr_ecap, a.fr_ucap, a.fr_logcap);
        frontier_query(L, a, R, qi, lane);
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAnd(a.fr_bitmap + (region >> 5), ~(1u << (region & 31)));
        }
    }
}

}  // namespace oob
