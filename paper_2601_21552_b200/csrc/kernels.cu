#include <algorithm>
#include <map>
#include <mutex>
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

#include "cert.cuh"
#include "chain.cuh"
#include "engine.cuh"
#include "format.h"
#include "frontier.cuh"
#include "phases.cuh"
#include "wide.cuh"

namespace oob {

constexpr int THREADS = 64;  // 2 warps per block: fine-grained shared-memory packing

// K1 + K4: the solve kernel (persistent; lockstep phase, then frontier phase)
template <typename T>
__global__ void __maxnreg__(128) oob_solve_kernel(LaunchArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    Lane<T> L;
    const uint32_t slot = claim_slab(a, warp, lane);
    L.bind(a, slot, lane);
    if (!a.frontier_only) lockstep_phase(a, L, warp, lane);
    frontier_phase(a, L, warp, lane);
    release_slab(a, slot, lane);
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
    L.bind(a, warp, lane);
    // domains + literal slots of the lane's query into a data block of width w
    auto store_state = [&](int64_t* dst, int w) {
        if (w == 2) {  // x32: packed int32 values
            int32_t* d32 = reinterpret_cast<int32_t*>(dst);
            for (uint32_t v = 0; v < L.nv; ++v) {
                d32[2 * v] = (int32_t)low64(L.E(L.env_lo, v));
                d32[2 * v + 1] = (int32_t)low64(L.E(L.env_hi, v));
            }
            for (uint32_t i = 0; i < L.nlit; ++i) d32[2 * L.nv + i] = (int32_t)low64(L.E(L.lit, i));
        } else if (w == 0) {
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
    };
    for (uint32_t qi = blockIdx.x * blockDim.x + threadIdx.x; qi < a.n; qi += gridDim.x * blockDim.x) {
        // own fresh entries, and (int128 job) shadows the 256-bit root phase
        // resumed here: their root propagation continues in this narrower
        // width until it fits int64 (a 256-bit query typically fits int128
        // after one pass and int64 only after the asserts have propagated)
        const uint32_t rs = a.resume[qi];
        if (rs == RES_SKIP || (rs != 0u && SELF == 2)) continue;
        // a shadow at its fixpoint: the wider phase already proved it cannot
        // narrow further except int64 -> x32, which only this job checks
        if (rs != 0u && (rs & RES_FIX) && SELF != 0) continue;
        const bool from_shadow = rs != 0u;
        const QDesc d = a.qdesc[qi];
        ClassDesc cd;
        cd.code_off = d.code_off;
        cd.nv_ncon = d.nv_ncon;
        cd.ncode_nlit = d.ncode_nlit;
        L.set_class(a, cd);
        L.load(a, d);
        const uint64_t t0 = from_shadow ? a.heavy_t0[qi] : global_ns();
        const uint64_t deadline = a.timeout_ns ? t0 + a.timeout_ns : 0;
        uint32_t passes = from_shadow ? (rs & RES_PASSES) : 0u;
        bool dead = false, fix = from_shadow && (rs & RES_FIX), expired = false;
        int target = -1;
        if constexpr (SELF == 0) {
            if (fix && a.dem[2].slot && L.fit_x32()) target = 2;
        }
        // the int64 root phase only probes for x32 (long root propagations
        // continue in the int64 job); the wide ones run until they fit int64
        const uint32_t max_passes = SELF == 0 ? ROOT_MAX_PASSES_X32 : ROOT_MAX_PASSES;
        while (!fix && passes < max_passes) {
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
                if constexpr (SELF == 0) {  // int64 -> x32
                    if (a.dem[2].slot && L.fit_x32()) {
                        target = 2;
                        break;
                    }
                } else {
                    int r = L.fit_regime();
                    if (r < SELF && a.dem[r].slot) {
                        target = r;
                        break;
                    }
                }
            }
            if (fix) break;
        }
        if (expired || L.err) {  // the lockstep kernel redoes it and reports
            if (from_shadow) a.resume[qi] = rs;
            continue;
        }
        if (dead) {  // Unsat after the root node (solver.py:393-394)
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
        if (target < 0) {
            if (from_shadow) {  // continue from here in this job (the shadow block is ours to rewrite)
                store_state(const_cast<int64_t*>(a.data) + d.data_off, SELF == 0 ? 0 : 1);
                __threadfence();
                a.resume[qi] = RES_ROOT | (fix ? RES_FIX : 0u) | passes;
            }
            continue;
        }
        const DemoteTarget& tg = a.dem[target];
        const uint32_t s = tg.slot[qi];
        store_state(tg.data + tg.qdesc[s].data_off, target);
        tg.t0[s] = t0;
        __threadfence();
        tg.resume[s] = RES_ROOT | (fix ? RES_FIX : 0u) | passes;
        a.resume[qi] = RES_SKIP;
    }
}

// exact value of a job's element for the certificate check (a 256-bit value
// beyond int128 becomes 2^126: "too big", which every check treats as unknown)
__device__ __forceinline__ sym::i128 cert_value(long long x) { return x; }
__device__ __forceinline__ sym::i128 cert_value(__int128 x) { return x; }
__device__ __forceinline__ sym::i128 cert_value(const i256& x) {
    const __int128 lo = x.low128();
    const uint64_t s = lo < 0 ? ~0ull : 0ull;
    return (x.w[2] == s && x.w[3] == s) ? lo : ((sym::i128)1 << 126);
}

// Fast mode (OOB_F_FAST): the Unsat certificates of each entry's structure
// class (cert.cuh), checked numerically before the root and solve kernels; a
// refuted entry is decided Unsat and never searched.  Two launches: every
// entry's first certificate (the one from the class's widest member, which
// refutes most entries), then one thread per (entry, later certificate) pair
// for the entries still open -- so an entry no certificate refutes (a Sat
// query) costs two certificates of latency instead of all of them in
// sequence.  Entries are class-major, so a warp's lanes share a certificate.
template <typename T>
__global__ void __launch_bounds__(128) oob_cert_kernel(LaunchArgs a, uint32_t k0, uint32_t k1) {
    cert::BoxV B;
    const uint64_t items = (uint64_t)a.n * (k1 - k0);
    for (uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
         it += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t kk = (uint32_t)(it / a.n), qi = (uint32_t)(it - (uint64_t)kk * a.n);
        const uint32_t k = k0 + kk;
        const uint32_t r0 = __ldcg(a.resume + qi);
        if (r0 == RES_SKIP) continue;  // a shadow, or refuted by another certificate already
        // the entry's class: the last class starting at or before qi
        uint32_t lo = 0, hi = a.cert_nclasses;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (a.cert_classes[mid].q_begin <= qi) lo = mid;
            else hi = mid;
        }
        const uint32_t off = a.cert_classes[lo].cert;
        if (off == NO_CERT) continue;
        const uint64_t* c = a.certs + off;
        const uint64_t ncerts = *c++;
        if (k >= ncerts) continue;
        for (uint32_t s = 0; s < k; s++) c += 1 + c[0];  // [length][words] per certificate
        ++c;
        const QDesc d = a.qdesc[qi];
        const uint32_t nv = d.nv_ncon & 0xFFFFu;
        const T* src = reinterpret_cast<const T*>(a.data + d.data_off);
        auto dom = [&](uint32_t i) -> sym::i128 { return cert_value(src[i]); };
        auto lit = [&](uint32_t i) -> sym::i128 { return cert_value(src[2 * nv + i]); };
        if (cert::cert_check(c, dom, lit, B) != cert::C_REFUTED) continue;
        if (atomicCAS(a.resume + qi, r0, RES_SKIP) != r0) continue;  // another certificate was first
        a.verdict[qi] = (int8_t)VERDICT_UNSAT;
        a.err[qi] = (int8_t)ERR_NONE;
        a.nodes[qi] = 0;
        a.passes[qi] = 0;
        a.elapsed[qi] = 0.f;
        if (a.fast_stats) atomicAdd(a.fast_stats + 4, 1ull);
    }
}

// Device-side records (SOLVE): every own entry's domains and literal slots,
// written in its job's width (VW int64 words per value: 1 int64, 2 int128,
// 4 256-bit, sign-extended) from the caller's raw values, narrowed to int64
// by the host (a call with a value beyond int64 keeps the host fill) and
// uploaded once per call; the host only writes the entry's offsets {raw var
// offset, raw literal offset, literal-source table offset} (shadows:
// UINT32_MAX).  One thread per entry; the padding is zeroed as the host did.
struct RawWord {
    int64_t v;
};
template <int VW>
__global__ void __launch_bounds__(256) oob_expand_kernel(const QDesc* __restrict__ qd, uint32_t n,
                                                         const uint4* __restrict__ rawoff,
                                                         const RawWord* __restrict__ vlo,
                                                         const RawWord* __restrict__ vhi,
                                                         const RawWord* __restrict__ lits,
                                                         const int32_t* __restrict__ litsrc, int64_t* data,
                                                         uint32_t align) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint4 ro = rawoff[i];
        if (ro.x == 0xFFFFFFFFu) continue;  // a shadow: written by the root phases
        const QDesc d = qd[i];
        const uint32_t nv = d.nv_ncon & 0xFFFFu, nlit = d.ncode_nlit >> 16;
        int64_t* out = data + d.data_off;
        auto put = [&](int64_t x) {
            out[0] = x;
            if (VW >= 2) out[1] = x < 0 ? -1 : 0;
            if (VW == 4) out[2] = out[3] = x < 0 ? -1 : 0;
            out += VW;
        };
        for (uint32_t v = 0; v < nv; v++) {
            put(vlo[ro.x + v].v);
            put(vhi[ro.x + v].v);
        }
        for (uint32_t s = 0; s < nlit; s++) {
            const int32_t src = litsrc[ro.z + s];
            put(src < 0 ? 1 : lits[ro.y + src].v);
        }
        const uint64_t words = (uint64_t)(2 * nv + nlit) * VW;
        const uint64_t dsz = (words + align - 1) / align * align;
        for (uint64_t k = words; k < dsz; k++) data[d.data_off + k] = 0;
    }
}

cudaError_t launch_expand(int wide, const QDesc* qd, uint32_t n, const void* rawoff, const void* vlo, const void* vhi,
                          const void* lits, const int32_t* litsrc, int64_t* data, int sms, cudaStream_t s) {
    const int blocks = (int)std::max<uint32_t>(1, std::min<uint32_t>((n + 255) / 256, (uint32_t)sms * 8));
    const uint4* ro = (const uint4*)rawoff;
    const RawWord *a = (const RawWord*)vlo, *b = (const RawWord*)vhi, *l = (const RawWord*)lits;
    if (wide == 0) oob_expand_kernel<1><<<blocks, 256, 0, s>>>(qd, n, ro, a, b, l, litsrc, data, 2);
    else if (wide == 1) oob_expand_kernel<2><<<blocks, 256, 0, s>>>(qd, n, ro, a, b, l, litsrc, data, 2);
    else if (wide == 2) oob_expand_kernel<4><<<blocks, 256, 0, s>>>(qd, n, ro, a, b, l, litsrc, data, 4);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// propagate() / check_model() batches: one query per lane, no search
template <typename T>
__global__ void __launch_bounds__(THREADS) oob_aux_kernel(LaunchArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    Lane<T> L;
    L.bind(a, warp, lane);
    for (uint32_t qi = blockIdx.x * blockDim.x + threadIdx.x; qi < a.n; qi += gridDim.x * blockDim.x) {
        (void)warp;
        const QDesc d = a.qdesc[qi];
        ClassDesc cd;
        cd.code_off = d.code_off;
        cd.nv_ncon = d.nv_ncon;
        cd.ncode_nlit = d.ncode_nlit;
        L.set_class(a, cd);
        L.load(a, d);
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

// The dynamic shared memory limit of a kernel is a per-function attribute
// of the device: several host threads staging jobs on one device (logical
// devices, the stream API's workers) must never LOWER it under another's
// launch, so it only ever grows (per function and device).
cudaError_t grow_smem_limit(const void* fn, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> set;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = set[{fn, dev}];
    if (smem <= cur && cur) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max(smem, cur));
    if (e == cudaSuccess) cur = std::max(smem, cur);
    return e;
}

template <typename T>
static cudaError_t occupancy_impl(int mode, size_t smem, int* blocks_per_sm) {
    const void* fn = kernel_ptr<T>(mode);
    cudaError_t e = grow_smem_limit(fn, smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, THREADS, smem);
}

// root phase of job `wide` (0 int64 -> x32, 1 int128, 2 256-bit)
cudaError_t launch_root(const LaunchArgs& a, int wide, int blocks, cudaStream_t s) {
    size_t smem = (size_t)a.g.smem_per_warp * (THREADS / 32);
    if (wide == 0) {
        grow_smem_limit((const void*)oob_root_kernel<long long, 0>, smem);
        oob_root_kernel<long long, 0><<<blocks, THREADS, smem, s>>>(a);
    } else if (wide == 2) {
        grow_smem_limit((const void*)oob_root_kernel<i256, 2>, smem);
        oob_root_kernel<i256, 2><<<blocks, THREADS, smem, s>>>(a);
    } else {
        grow_smem_limit((const void*)oob_root_kernel<__int128, 1>, smem);
        oob_root_kernel<__int128, 1><<<blocks, THREADS, smem, s>>>(a);
    }
    return cudaGetLastError();
}

// fast mode certificate check of job `wide` (0 int64, 1 int128, 2 256-bit)
// certificates [k0, k1) of every entry: one thread per (entry, certificate)
cudaError_t launch_chain(const LaunchArgs& a, int blocks, cudaStream_t s) {
    oob_chain_kernel<<<blocks, chain::WARPS * 32, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_enum(const LaunchArgs& a, int blocks, cudaStream_t s) {
    oob_enum_kernel<<<blocks, chain::WARPS * 32, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_cert(const LaunchArgs& a, int wide, uint32_t k0, uint32_t k1, int sms, cudaStream_t s) {
    const uint64_t items = (uint64_t)a.n * (k1 - k0);
    const int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>((items + 127) / 128, (uint64_t)sms * 16));
    if (wide == 0) oob_cert_kernel<long long><<<blocks, 128, 0, s>>>(a, k0, k1);
    else if (wide == 1) oob_cert_kernel<__int128><<<blocks, 128, 0, s>>>(a, k0, k1);
    else if (wide == 2) oob_cert_kernel<i256><<<blocks, 128, 0, s>>>(a, k0, k1);
    return cudaGetLastError();
}

// wide: 0 = int64, 1 = __int128, 2 = 256-bit, 3 = x32 regime
cudaError_t launch_solve(const LaunchArgs& a, int wide, int blocks, int fblocks, cudaStream_t s) {
    if (wide == 3) return launch_impl<int>(a, blocks, fblocks, s);
    if (wide == 2) return launch_impl<i256>(a, blocks, fblocks, s);
    return wide ? launch_impl<__int128>(a, blocks, fblocks, s) : launch_impl<long long>(a, blocks, fblocks, s);
}

// SOLVE fetch: the models of Sat entries only, packed (an entry's model slot
// is written by the search only when it ends Sat; the rest of the model
// buffer is never read by the host) -- sat_off[i] is entry i's offset in vars
__global__ void oob_gather_sat_kernel(const int8_t* __restrict__ verdict, const QDesc* __restrict__ qd,
                                      const int64_t* __restrict__ model, uint32_t n,
                                      unsigned long long* counter, uint32_t* sat_off, int64_t* compact) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (verdict[i] != VERDICT_SAT) continue;
        const uint32_t nv = qd[i].nv_ncon & 0xffffu;
        const unsigned long long off = atomicAdd(counter, (unsigned long long)nv);
        sat_off[i] = (uint32_t)off;
        const int64_t* src = model + 2 * qd[i].out_v;
        int64_t* dst = compact + 2 * off;
        for (uint32_t k = 0; k < 2 * nv; k++) dst[k] = src[k];
    }
}

cudaError_t launch_gather_sat(const int8_t* verdict, const QDesc* qd, const int64_t* model, uint32_t n,
                              unsigned long long* counter, uint32_t* sat_off, int64_t* compact, int sms,
                              cudaStream_t s) {
    const uint32_t blocks = std::max(1u, std::min<uint32_t>((n + 255) / 256, (uint32_t)sms * 4));
    oob_gather_sat_kernel<<<blocks, 256, 0, s>>>(verdict, qd, model, n, counter, sat_off, compact);
    return cudaGetLastError();
}

// resident blocks per SM of the kernel for `mode` with `smem` dynamic bytes per block
cudaError_t kernel_occupancy(int wide, int mode, size_t smem, int* blocks_per_sm) {
    if (wide == 3) return occupancy_impl<int>(mode, smem, blocks_per_sm);
    if (wide == 2) return occupancy_impl<i256>(mode, smem, blocks_per_sm);
    return wide ? occupancy_impl<__int128>(mode, smem, blocks_per_sm)
                : occupancy_impl<long long>(mode, smem, blocks_per_sm);
}

}  // namespace oob
