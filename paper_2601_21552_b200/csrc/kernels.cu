// kernels.cu -- sm_100a kernels of the OOB-query engine.
//
//   oob_solve_kernel<T>   K1: exact solve() emulation (solver.py:363-416) with
//                         K4 (check_model at every leaf, solver.py:405-407)
//                         fused in; MODE_PROPAGATE runs one root propagate()
//                         (solver.py:264-280), MODE_CHECK one check_model()
//                         (solver.py:319-328).
//
// Scheduling: a persistent grid (a multiple of the 148 SMs) whose warps pull
// tiles of 32 consecutive scheduled queries from one atomic counter; lane i of
// a warp owns query tile*32+i.  The host schedule is sorted by structure class
// so a tile is normally 32 instances of one class and its lanes walk the same
// code words in lockstep (broadcast loads, coalesced lane-minor scratch).
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.cuh"
#include "format.h"
#include "wide.cuh"

namespace oob {

// model / domain output in the caller's int128 wire format (values are
// within the declared domains, which the wire format bounds to 128 bits)
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

template <typename T>
__global__ void __launch_bounds__(128) oob_solve_kernel(LaunchArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const SlabGeom& g = a.g;

    Lane<T> L;
    T* sT = reinterpret_cast<T*>(a.slab_T) + (size_t)warp * g.slab_T_words + lane;
    uint32_t* sU = a.slab_u32 + (size_t)warp * g.slab_u32_words + lane;
    L.env_lo = sT + g.o_env_lo;
    L.env_hi = sT + g.o_env_hi;
    L.val_lo = sT + g.o_val_lo;
    L.val_hi = sT + g.o_val_hi;
    L.lit = sT + g.o_lit;
    L.fr_mid = sT + g.o_fr_mid;
    L.fr_hi = sT + g.o_fr_hi;
    L.tr_lo = sT + g.o_tr_lo;
    L.tr_hi = sT + g.o_tr_hi;
    L.stamp = sU + g.o_stamp;
    L.fr_pick = sU + g.o_fr_pick;
    L.fr_mark = sU + g.o_fr_mark;
    L.tr_var = sU + g.o_tr_var;
    L.g = &g;
    L.seg = 0;

    for (;;) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(a.next, 32u);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= a.n) break;
        const uint32_t qi = base + lane;
        if (qi >= a.n) continue;

        const QDesc d = a.qdesc[qi];
        L.nv = d.nv_ncon & 0xFFFFu;
        L.ncon = d.nv_ncon >> 16;
        L.ncode = d.ncode_nlit & 0xFFFFu;
        L.nlit = d.ncode_nlit >> 16;
        L.cons = a.code + d.code_off;
        L.code = L.cons + L.ncon;
        L.err = ERR_NONE;
        L.depth = 0;
        L.trail_len = 0;

        // stage this query's domains and literal slots into lane-minor scratch
        const T* src = reinterpret_cast<const T*>(a.data + d.data_off);
        for (uint32_t v = 0; v < L.nv; ++v) {
            L.E(L.env_lo, v) = src[2 * v];
            L.E(L.env_hi, v) = src[2 * v + 1];
            L.U(L.stamp, v) = 0xFFFFFFFFu;
        }
        for (uint32_t i = 0; i < L.nlit; ++i) L.E(L.lit, i) = src[2 * L.nv + i];

        const uint64_t t_start = global_ns();
        int64_t nodes = 0, passes = 0;
        int verdict;
        if (a.mode == MODE_SOLVE) {
            uint64_t deadline = a.timeout_ns ? t_start + a.timeout_ns : 0;
            verdict = L.search(nodes, passes, deadline, a.node_budget);
        } else if (a.mode == MODE_PROPAGATE) {
            int pr = L.propagate(passes, 0);
            verdict = pr == 1 ? VERDICT_SAT : (pr == 0 ? VERDICT_UNSAT : VERDICT_ERROR);
        } else {
            verdict = L.check_point(L.env_lo) ? VERDICT_SAT : VERDICT_UNSAT;
        }
        const uint64_t t_end = global_ns();

        a.verdict[qi] = (int8_t)verdict;
        a.err[qi] = (int8_t)L.err;
        if (a.nodes) a.nodes[qi] = nodes;
        if (a.passes) a.passes[qi] = passes;
        if (a.elapsed) a.elapsed[qi] = (float)((double)(t_end - t_start) * 1e-9);
        const bool write_lo = (a.mode == MODE_SOLVE && verdict == VERDICT_SAT);
        const bool write_both = (a.mode == MODE_PROPAGATE);
        if (write_lo || write_both) {
            int64_t* m = a.model + 2 * d.out_v * (write_both ? 2 : 1);
            for (uint32_t v = 0; v < L.nv; ++v) {
                if (write_both) {
                    store_i128(m + 4 * v, L.E(L.env_lo, v));
                    store_i128(m + 4 * v + 2, L.E(L.env_hi, v));
                } else {
                    store_i128(m + 2 * v, L.E(L.env_lo, v));
                }
            }
        }
    }
}

// explicit instantiations + launchers (called from host.cpp)
template <typename T>
static cudaError_t launch_impl(const LaunchArgs& a, int blocks, cudaStream_t s) {
    oob_solve_kernel<T><<<blocks, 128, 0, s>>>(a);
    return cudaGetLastError();
}

// wide: 0 = int64, 1 = __int128, 2 = 256-bit regime
cudaError_t launch_solve(const LaunchArgs& a, int wide, int blocks, cudaStream_t s) {
    if (wide == 2) return launch_impl<i256>(a, blocks, s);
    return wide ? launch_impl<__int128>(a, blocks, s) : launch_impl<long long>(a, blocks, s);
}

}  // namespace oob
