// kernels.cu -- sm_100a kernels of the OOB-query engine.
//
//   oob_lockstep_kernel<T>  K1: exact solve() emulation (solver.py:363-416)
//                           with K4 (check_model at every leaf, :405-407)
//                           fused in.
//   oob_aux_kernel<T>       one root propagate() (solver.py:264-280) or one
//                           check_model() (solver.py:319-328) per query.
//
// Scheduling of K1 (persistent grid, a multiple of the 148 SMs):
//   * the host groups queries by STRUCTURE CLASS (identical constraint/term
//     shapes, different domains and literals) and gives every class a work
//     queue; each warp is assigned a starting class in proportion to the
//     class sizes and moves to the next non-empty class when its own drains;
//   * all 32 lanes of a warp run instances of ONE class and advance together
//     one propagation pass per step: the constraint loop inside a pass is
//     uniform, so constraint k's code words are broadcast loads and every
//     lane-minor scratch access is coalesced;
//   * between passes each lane independently starts a node, splits, leaves a
//     model, backtracks or finishes; a finished lane immediately takes the
//     next query of the warp's class (no lane waits for a whole tile).
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.cuh"
#include "format.h"
#include "frontier.cuh"
#include "wide.cuh"

namespace oob {

constexpr int THREADS = 64;  // 2 warps per block: fine-grained shared-memory packing

extern __shared__ __align__(16) unsigned char oob_smem[];

template <typename T>
__device__ __forceinline__ void bind_scratch(Lane<T>& L, const LaunchArgs& a, uint32_t warp, uint32_t lane) {
    const SlabGeom& g = a.g;
    T* sT = reinterpret_cast<T*>(a.slab_T) + (size_t)warp * g.slab_T_words + lane;
    uint32_t* sU = a.slab_u32 + (size_t)warp * g.slab_u32_words + lane;
    if (g.smem_per_warp) {  // hot state on chip, lane-minor (conflict-free in lockstep)
        T* s = reinterpret_cast<T*>(oob_smem + (threadIdx.x >> 5) * g.smem_per_warp) + lane;
        L.env_lo = s + g.o_s_env_lo;
        L.env_hi = s + g.o_s_env_hi;
        L.val_lo = s + g.o_s_val_lo;
        L.val_hi = s + g.o_s_val_hi;
        L.lit = sT + g.o_lit;
        L.st_0 = s + g.o_s_st0;
        L.st_1 = s + g.o_s_st1;
        L.st_n = reinterpret_cast<uint32_t*>(oob_smem + (threadIdx.x >> 5) * g.smem_per_warp + g.o_s_stn_bytes) + lane;
    } else {
        L.env_lo = sT + g.o_env_lo;
        L.env_hi = sT + g.o_env_hi;
        L.val_lo = sT + g.o_val_lo;
        L.val_hi = sT + g.o_val_hi;
        L.lit = sT + g.o_lit;
        L.st_0 = sT + g.o_st0;
        L.st_1 = sT + g.o_st1;
        L.st_n = sU + g.o_stn;
    }
    L.st_cap = g.st_cap;
    L.fr_mid = sT + g.o_fr_mid;
    L.fr_hi = sT + g.o_fr_hi;
    L.tr_lo = sT + g.o_tr_lo;
    L.tr_hi = sT + g.o_tr_hi;
    L.stamp = sU + g.o_stamp;
    L.fr_pick = sU + g.o_fr_pick;
    L.fr_mark = sU + g.o_fr_mark;
    L.fr_clean = sU + g.o_fr_clean;
    L.tr_var = sU + g.o_tr_var;
    L.g = &a.g;
    L.seg = 0;
}

template <typename T>
__device__ __forceinline__ void bind_class(Lane<T>& L, const LaunchArgs& a, const ClassDesc& c) {
    L.nv = c.nv_ncon & 0xFFFFu;
    L.ncon = c.nv_ncon >> 16;
    L.ncode = c.ncode_nlit & 0xFFFFu;
    L.nlit = c.ncode_nlit >> 16;
    L.cons = a.code + c.code_off;
    L.code = L.cons + L.ncon;
    L.member = L.code + L.ncode;
    L.skip = L.ncon <= 128;
}

// stage a query's domains and literal slots into lane-minor scratch
template <typename T>
__device__ __forceinline__ void load_query(Lane<T>& L, const LaunchArgs& a, const QDesc& d) {
    const T* src = reinterpret_cast<const T*>(a.data + d.data_off);
    for (uint32_t v = 0; v < L.nv; ++v) {
        L.E(L.env_lo, v) = src[2 * v];
        L.E(L.env_hi, v) = src[2 * v + 1];
        L.U(L.stamp, v) = 0xFFFFFFFFu;
    }
    for (uint32_t i = 0; i < L.nlit; ++i) L.E(L.lit, i) = src[2 * L.nv + i];
    L.err = ERR_NONE;
    L.depth = 0;
    L.trail_len = 0;
    L.clean0 = 0;
    L.clean1 = 0;
}

enum : int { PH_IDLE = 0, PH_NODE = 1, PH_PASS = 2, PH_DONE = 3, PH_POST = 4 };

// Phase 1 of the solve kernel: lockstep class queues (returns when the warp's
// lanes are idle and every class queue is drained).
template <typename T>
__device__ __forceinline__ void lockstep_phase(const LaunchArgs& a, Lane<T>& L, uint32_t warp, uint32_t lane) {
    const unsigned FULL = 0xffffffffu;
    const unsigned lt_mask = (1u << lane) - 1u;

    uint32_t c = a.warp_class[warp];  // the warp's current class queue (warp-uniform)
    ClassDesc cd = a.classes[c];
    bind_class(L, a, cd);
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
                        bind_class(L, a, cd);
                        const QDesc d = a.qdesc[qi];
                        load_query(L, a, d);
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
        if (phase == PH_NODE && a.heavy_nodes && nodes >= a.heavy_nodes) {
            // a heavy search: hand it to the warp-cooperative frontier phase
            // (which restarts it from the root with 32 lanes); the list entry
            // is published after the start time it carries
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
        // ---- the pass: class-uniform constraint loop (solver.py:275-277) ----
        // The warp visits, in order, every constraint that is dirty in at
        // least one lane (clean ones would change nothing, engine.cuh).
        for (uint32_t k = 0;;) {
            uint32_t mine = (run && !dead) ? L.next_dirty(k) : 0xFFFFu;
            if (mine >= L.ncon) mine = 0xFFFFu;  // lanes may be on different classes
            uint32_t kk = __reduce_min_sync(FULL, mine);
            if (kk == 0xFFFFu) break;
            if (mine == kk && !L.pass_constraint(kk)) dead = true;
            k = kk + 1;
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
                    if (L.check_point(L.env_lo)) {
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
                for (uint32_t v = 0; v < L.nv; ++v) store_i128(m + 2 * v, L.E(L.env_lo, v));
            }
            phase = PH_IDLE;
        }
    }
}

// Phase 2 of the solve kernel: heavy queries, one warp per query, lanes
// expand the leftmost pending nodes (frontier.cuh).  A warp whose lockstep
// phase is over serves the heavy list until it finds nothing left to claim,
// then exits (it never spins: an idle resident warp would keep the SMs from
// the other regimes' kernels).  An entry appended later comes from a warp
// still in its lockstep phase, which serves the list itself afterwards, so
// every entry is taken.
template <typename T>
__device__ __forceinline__ void frontier_phase(const LaunchArgs& a, Lane<T>& L, uint32_t warp, uint32_t lane) {
    const unsigned FULL = 0xffffffffu;
    volatile uint32_t* ctl = a.heavy_count;  // [0] listed [1] claimed
    if (!a.heavy_nodes) return;
    FrontierRegion<T> R;  // one scratch region per warp of the grid
    R.bind((unsigned char*)a.fr_region + (size_t)warp * a.fr_region_bytes, a.g.maxv, a.fr_ecap, a.fr_ucap,
           a.fr_logcap);
    for (;;) {
        int idx = -1;
        if (lane == 0) {
            for (;;) {
                const uint32_t listed = ctl[0], claimed = ctl[1];
                if (claimed >= listed) break;
                if (atomicCAS(a.heavy_count + 1, claimed, claimed + 1) == claimed) {
                    idx = (int)claimed;
                    break;
                }
            }
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
        bind_class(L, a, cd);
        load_query(L, a, d);
        frontier_query(L, a, R, qi, lane);
    }
}

// K1 + K4: the solve kernel (persistent; lockstep phase, then frontier phase)
template <typename T>
__global__ void __launch_bounds__(THREADS) oob_solve_kernel(LaunchArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    Lane<T> L;
    bind_scratch(L, a, warp, lane);
    lockstep_phase(a, L, warp, lane);
    frontier_phase(a, L, warp, lane);
}

// Root phase of the wide regimes (format.h, "regime demotion"): one lane per
// query runs the root node's propagate() passes (solver.py:264-280 under
// _search's first call, :393) in the query's proven regime; after passes 1,
// 2, 4, ... and at the fixpoint it restates the bound proof at the narrowed
// domains (Lane::fit_regime) and, if a narrower regime holds, hands the
// query's state to that regime's shadow entry.  A contradiction at the root
// is the final verdict (Unsat after one node).  Queries that neither die nor
// demote within ROOT_MAX_PASSES are left to this regime's lockstep kernel,
// which restarts them from the declared domains.
template <typename T, int SELF>
__global__ void __launch_bounds__(THREADS) oob_root_kernel(LaunchArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    Lane<T> L;
    bind_scratch(L, a, warp, lane);
    for (uint32_t qi = blockIdx.x * blockDim.x + threadIdx.x; qi < a.n; qi += gridDim.x * blockDim.x) {
        if (a.resume[qi] != 0u) continue;  // a shadow of a wider job's query
        const QDesc d = a.qdesc[qi];
        ClassDesc cd;
        cd.code_off = d.code_off;
        cd.nv_ncon = d.nv_ncon;
        cd.ncode_nlit = d.ncode_nlit;
        bind_class(L, a, cd);
        load_query(L, a, d);
        const uint64_t t0 = global_ns();
        const uint64_t deadline = a.timeout_ns ? t0 + a.timeout_ns : 0;
        uint32_t passes = 0;
        bool dead = false, fix = false, expired = false;
        int target = -1;
        while (passes < ROOT_MAX_PASSES) {
            if (deadline && global_ns() > deadline) {
                expired = true;
                break;
            }
            ++passes;
            L.changed = false;
            for (uint32_t k = L.next_dirty(0); k < L.ncon; k = L.next_dirty(k + 1)) {
                if (!L.pass_constraint(k)) {
                    dead = true;
                    break;
                }
            }
            if (dead) break;
            fix = !L.changed;
            if (fix || (passes & (passes - 1)) == 0) {
                int r = L.fit_regime();
                if (r < SELF && a.dem[r].slot) {
                    target = r;
                    break;
                }
            }
            if (fix) break;
        }
        if (expired || L.err) continue;  // the lockstep kernel redoes it and reports
        if (dead) {                      // Unsat after the root node (solver.py:393-394)
            a.verdict[qi] = (int8_t)VERDICT_UNSAT;
            a.err[qi] = (int8_t)ERR_NONE;
            a.nodes[qi] = 1;
            a.passes[qi] = passes;
            a.elapsed[qi] = (float)((double)(global_ns() - t0) * 1e-9);
            if (a.timeline) {
                a.timeline[4 * (size_t)qi] = t0;
                a.timeline[4 * (size_t)qi + 3] = global_ns();
            }
            a.resume[qi] = RES_SKIP;
            continue;
        }
        if (target < 0) continue;
        const DemoteTarget& tg = a.dem[target];
        const uint32_t s = tg.slot[qi];
        int64_t* dst = tg.data + tg.qdesc[s].data_off;
        if (target == 0) {
            for (uint32_t v = 0; v < L.nv; ++v) {
                dst[2 * v] = low64(L.E(L.env_lo, v));
                dst[2 * v + 1] = low64(L.E(L.env_hi, v));
            }
            for (uint32_t i = 0; i < L.nlit; ++i) dst[2 * L.nv + i] = low64(L.E(L.lit, i));
        } else {
            auto put = [&](uint32_t at, __int128 x) {
                dst[2 * at] = (int64_t)(uint64_t)x;
                dst[2 * at + 1] = (int64_t)(x >> 64);
            };
            for (uint32_t v = 0; v < L.nv; ++v) {
                put(2 * v, low128(L.E(L.env_lo, v)));
                put(2 * v + 1, low128(L.E(L.env_hi, v)));
            }
            for (uint32_t i = 0; i < L.nlit; ++i) put(2 * L.nv + i, low128(L.E(L.lit, i)));
        }
        tg.t0[s] = t0;
        __threadfence();
        tg.resume[s] = RES_ROOT | (fix ? RES_FIX : 0u) | passes;
        a.resume[qi] = RES_SKIP;
    }
}

// propagate() / check_model() batches: one query per lane, no search
template <typename T>
__global__ void __launch_bounds__(THREADS) oob_aux_kernel(LaunchArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    Lane<T> L;
    bind_scratch(L, a, warp, lane);
    for (uint32_t qi = blockIdx.x * blockDim.x + threadIdx.x; qi < a.n; qi += gridDim.x * blockDim.x) {
        (void)warp;
        const QDesc d = a.qdesc[qi];
        ClassDesc cd;
        cd.code_off = d.code_off;
        cd.nv_ncon = d.nv_ncon;
        cd.ncode_nlit = d.ncode_nlit;
        bind_class(L, a, cd);
        load_query(L, a, d);
        int64_t passes = 0;
        int verdict;
        if (a.mode == MODE_PROPAGATE) {
            int pr = L.propagate(passes);
            verdict = pr == 1 ? VERDICT_SAT : (pr == 0 ? VERDICT_UNSAT : VERDICT_ERROR);
        } else {
            verdict = L.check_point(L.env_lo) ? VERDICT_SAT : VERDICT_UNSAT;
        }
        a.verdict[qi] = (int8_t)verdict;
        a.err[qi] = (int8_t)L.err;
        a.nodes[qi] = 0;
        a.passes[qi] = passes;
        a.elapsed[qi] = 0.f;
        if (a.mode == MODE_PROPAGATE) {
            int64_t* m = a.model + 4 * d.out_v;
            for (uint32_t v = 0; v < L.nv; ++v) {
                store_i128(m + 4 * v, L.E(L.env_lo, v));
                store_i128(m + 4 * v + 2, L.E(L.env_hi, v));
            }
        }
    }
}

template <typename T>
static const void* kernel_ptr(int mode) {
    return mode == MODE_SOLVE ? (const void*)oob_solve_kernel<T> : (const void*)oob_aux_kernel<T>;
}

template <typename T>
static cudaError_t launch_impl(const LaunchArgs& a, int blocks, int fblocks, cudaStream_t s) {
    size_t smem = (size_t)a.g.smem_per_warp * (THREADS / 32);
    (void)fblocks;
    if (a.mode == MODE_SOLVE) {
        oob_solve_kernel<T><<<blocks, THREADS, smem, s>>>(a);
    } else {
        oob_aux_kernel<T><<<blocks, THREADS, smem, s>>>(a);
    }
    return cudaGetLastError();
}

template <typename T>
static cudaError_t occupancy_impl(int mode, size_t smem, int* blocks_per_sm) {
    const void* fn = kernel_ptr<T>(mode);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, THREADS, smem);
}

// root phase of a wide job (wide = 1 or 2)
cudaError_t launch_root(const LaunchArgs& a, int wide, int blocks, cudaStream_t s) {
    size_t smem = (size_t)a.g.smem_per_warp * (THREADS / 32);
    if (wide == 2) {
        cudaFuncSetAttribute((const void*)oob_root_kernel<i256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        oob_root_kernel<i256, 2><<<blocks, THREADS, smem, s>>>(a);
    } else {
        cudaFuncSetAttribute((const void*)oob_root_kernel<__int128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        oob_root_kernel<__int128, 1><<<blocks, THREADS, smem, s>>>(a);
    }
    return cudaGetLastError();
}

// wide: 0 = int64, 1 = __int128, 2 = 256-bit regime
cudaError_t launch_solve(const LaunchArgs& a, int wide, int blocks, int fblocks, cudaStream_t s) {
    if (wide == 2) return launch_impl<i256>(a, blocks, fblocks, s);
    return wide ? launch_impl<__int128>(a, blocks, fblocks, s) : launch_impl<long long>(a, blocks, fblocks, s);
}

// resident blocks per SM of the kernel for `mode` with `smem` dynamic bytes per block
cudaError_t kernel_occupancy(int wide, int mode, size_t smem, int* blocks_per_sm) {
    if (wide == 2) return occupancy_impl<i256>(mode, smem, blocks_per_sm);
    return wide ? occupancy_impl<__int128>(mode, smem, blocks_per_sm)
                : occupancy_impl<long long>(mode, smem, blocks_per_sm);
}

}  // namespace oob
