// sweep.cu -- device exhaustive oracle (include/scuba_oob_sweep.h).
//
// One thread per input tuple runs the whole MiniCUDA program through the
// bytecode interpreter of sweep_vm.cuh.  Grid: a persistent grid (SM count x
// resident blocks) strides over the tuple space warp by warp, so every lane of
// a warp works on consecutive tuples of product order and the warp's results
// are reduced with ballots before touching global memory: halted counts with
// one atomicAdd per warp, violations as (site, label) bits OR-reduced over
// the warp, and the first violating tuple per (site, label) as the lowest
// lane of the ballot (one atomicMin per warp and label bit).  The per-tuple
// cell arena is lane-interleaved in HBM (cell w of thread g at w*T + g).
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/scuba_oob.h"
#include "../../include/scuba_oob_sweep.h"
#include "sweep_vm.cuh"

int oob_internal_fail(int code, const std::string& msg);  // host.cpp

namespace {

constexpr int BLOCK = 128;

struct Dev {
    int64_t total, bound;
    int arity, mode;  // mode 0: enumerate [0,bound]^arity; 1: explicit tuples
    const int64_t* tuples;
    unsigned long long* counters;  // [0] halted, [1] errors, [2] need key, [3] error key, [4] arena peak
    uint32_t* site_labels;
    unsigned long long* site_first;  // [n_sites * 4]
    int32_t* t_status;
    int32_t* t_aux;
    uint8_t* t_labels;
};

__global__ void __launch_bounds__(BLOCK) oob_sweep_kernel(sweep::Prog P, Dev D, int64_t* arena,
                                                          int64_t words) {
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    sweep::Arena A{arena + g, nthreads, words};
    sweep::Machine m;
    int64_t in[sweep::MAX_INPUTS];
    const int nw = (P.n_sites * 4 + 31) / 32;
    int64_t peak = 0;
    for (int64_t wbase = g - lane; wbase < D.total; wbase += nthreads) {
        const int64_t t = wbase + lane;
        const bool valid = t < D.total;
        sweep::Out o{sweep::S_OK, 0};
        if (valid) {
            if (D.mode == 0) {
                int64_t r = t;
                for (int i = D.arity - 1; i >= 0; i--) {
                    in[i] = r % (D.bound + 1);
                    r /= D.bound + 1;
                }
            } else {
                for (int i = 0; i < D.arity; i++) in[i] = D.tuples[t * D.arity + i];
            }
            o = sweep::run(P, in, D.arity, A, m);
            peak = max(peak, m.arena_peak);
        }
        const bool ok = valid && o.status == sweep::S_OK;
        if (D.mode == 1) {
            if (valid) {
                D.t_status[t] = o.status;
                D.t_aux[t] = o.aux;
                for (int s = 0; s < P.n_sites; s++) {
                    uint32_t bits = ok ? (m.labels[(s * 4) >> 5] >> ((s * 4) & 31)) & 15u : 0u;
                    D.t_labels[t * P.n_sites + s] = (uint8_t)bits;
                }
            }
            continue;
        }
        const unsigned halted = __ballot_sync(FULL, valid && o.status == sweep::S_HALT);
        if (halted && lane == 0) atomicAdd(&D.counters[0], (unsigned long long)__popc(halted));
        const unsigned err = __ballot_sync(FULL, valid && o.status == sweep::S_ERROR);
        if (err) {
            if (lane == 0) atomicAdd(&D.counters[1], (unsigned long long)__popc(err));
            if (lane == __ffs(err) - 1)
                atomicMin(&D.counters[3], ((unsigned long long)t << 8) | (unsigned)o.aux);
        }
        const unsigned need = __ballot_sync(FULL, valid && o.status == sweep::S_NEED);
        if (need && lane == __ffs(need) - 1)
            atomicMin(&D.counters[2], ((unsigned long long)t << 8) | (unsigned)o.aux);
        for (int w = 0; w < nw; w++) {
            const uint32_t mine = ok ? m.labels[w] : 0u;
            uint32_t any = __reduce_or_sync(FULL, mine);
            while (any) {
                const int bit = __ffs(any) - 1;
                any &= any - 1;
                const unsigned who = __ballot_sync(FULL, (mine >> bit) & 1u);
                if (lane == __ffs(who) - 1) {
                    const int sl = w * 32 + bit;  // site * 4 + label
                    atomicOr(&D.site_labels[sl >> 2], 1u << (sl & 3));
                    atomicMin(&D.site_first[sl], (unsigned long long)t);
                }
            }
        }
    }
    if (peak) atomicMax(&D.counters[4], (unsigned long long)peak);
}

#define SCK(x)                                                                                   \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            return oob_internal_fail(OOB_E_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)

// device buffers pooled per device across calls (a sweep is often tiny: the
// allocation of a fresh arena would dominate it); grown on demand
struct PoolBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        bytes = std::max<size_t>(bytes, 256);
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
};

struct SweepPool {
    std::mutex mu;
    PoolBuf code, lits, kern, kpar, counters, slab, sfirst, tup, tst, taux, tlab, arena;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
};

SweepPool& pool_of(int dev) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<SweepPool>> pools;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)pools.size() <= dev) pools.resize(dev + 1);
    if (!pools[dev]) pools[dev].reset(new SweepPool());
    return *pools[dev];
}

int validate(const oob_sweep_program* pr, int32_t arity) {
    if (!pr || !pr->code || pr->n_code <= 0) return oob_internal_fail(OOB_E_INVALID, "sweep: empty program");
    if (arity < 0 || arity > sweep::MAX_INPUTS)
        return oob_internal_fail(OOB_E_INVALID, "sweep: arity out of range");
    if (pr->n_sites < 0 || pr->n_sites > sweep::MAX_SITES)
        return oob_internal_fail(OOB_E_INVALID, "sweep: too many access sites");
    if (pr->n_slots < 0 || pr->n_slots > sweep::MAX_SLOTS)
        return oob_internal_fail(OOB_E_INVALID, "sweep: too many variables");
    for (int i = 0; i < pr->n_code; i++) {
        const int32_t* c = pr->code + 4 * i;
        if (c[0] < 0 || c[0] > sweep::END)
            return oob_internal_fail(OOB_E_INVALID, "sweep: bad opcode at " + std::to_string(i));
        if ((c[0] == sweep::LIT && (c[1] < 0 || c[1] >= pr->n_lits)) ||
            ((c[0] == sweep::JZ || c[0] == sweep::JMP) && (c[1] < 0 || c[1] >= pr->n_code)) ||
            ((c[0] == sweep::LD || c[0] == sweep::ST || c[0] == sweep::MALLOC || c[0] == sweep::FREE ||
              c[0] == sweep::RD || c[0] == sweep::WR || c[0] == sweep::ATOM || c[0] == sweep::XSHM ||
              c[0] == sweep::ADECL || c[0] == sweep::PART || c[0] == sweep::PARG) &&
             (c[1] < 0 || c[1] >= pr->n_slots)) ||
            ((c[0] == sweep::RD || c[0] == sweep::WR || c[0] == sweep::ATOM || c[0] == sweep::FREE) &&
             (c[2] < 0 || c[2] >= pr->n_sites)) ||
            (c[0] == sweep::LAUNCH && (c[1] < 0 || c[1] >= pr->n_kernels)))
            return oob_internal_fail(OOB_E_INVALID, "sweep: bad operand at " + std::to_string(i));
    }
    // stack discipline: every reachable pc has one value-stack depth, never
    // negative nor above the device stack (the interpreter does not re-check)
    std::vector<int> depth(pr->n_code, -1);
    std::vector<int> work;
    auto reach = [&](int pc, int d) -> bool {
        if (pc < 0 || pc >= pr->n_code || d < 0 || d > sweep::MAX_STACK) return false;
        if (depth[pc] == -1) {
            depth[pc] = d;
            work.push_back(pc);
            return true;
        }
        return depth[pc] == d;
    };
    bool ok = reach(0, 0);
    for (int k = 0; k < pr->n_kernels && ok; k++) ok = reach(pr->kernels[4 * k], 0);
    while (ok && !work.empty()) {
        const int pc = work.back();
        work.pop_back();
        const int32_t* c = pr->code + 4 * pc;
        const int d = depth[pc];
        int nd = d, need = 0;
        switch (c[0]) {
        case sweep::LIT: case sweep::LD: case sweep::INP: case sweep::BLT: case sweep::PARG: nd = d + 1; break;
        case sweep::BIN: case sweep::CMP: need = 2; nd = d - 1; break;
        case sweep::RD: need = c[3]; nd = d - c[3] + 1; break;
        case sweep::ST: case sweep::JZ: case sweep::ASRT: case sweep::MALLOC: case sweep::PART: need = 1; nd = d - 1; break;
        case sweep::WR: need = c[3] + 1; nd = d - need; break;
        case sweep::ATOM: need = 2; nd = d - 2; break;
        case sweep::ADECL: need = c[3] & 3; nd = d - need; break;
        case sweep::NNEG: need = c[1]; break;
        case sweep::LAUNCH:
            need = 7 + c[2];
            nd = d - need;
            if (c[2] < 0 || c[2] > pr->kernels[4 * c[1] + 1]) ok = false;
            break;
        default: break;
        }
        if (d < need || (c[0] == sweep::RD && c[3] != 1 && c[3] != 2) ||
            (c[0] == sweep::WR && c[3] != 1 && c[3] != 2)) {
            ok = false;
            break;
        }
        if (c[0] == sweep::RET || c[0] == sweep::KEND || c[0] == sweep::END) continue;
        if (c[0] == sweep::JMP) {
            ok = reach(c[1], nd);
            continue;
        }
        if (c[0] == sweep::JZ) ok = reach(c[1], nd);
        if (ok) ok = reach(pc + 1, nd);
    }
    if (!ok) return oob_internal_fail(OOB_E_INVALID, "sweep: malformed program (value stack discipline)");
    return OOB_OK;
}

// Shared driver of both entry points.
int drive(const oob_sweep_program* pr, Dev D, int64_t n_out_tuples, const int64_t* tuples,
          const oob_sweep_options* opt, oob_sweep_result* out, int32_t* status, int32_t* aux,
          uint8_t* labels) {
    const int dev = opt ? opt->device : 0;
    SCK(cudaSetDevice(dev));
    int sms = 0;  // (cudaGetDeviceProperties costs milliseconds per call)
    SCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int ns = std::max(pr->n_sites, 1);

    SweepPool& pool = pool_of(dev);
    std::lock_guard<std::mutex> lk(pool.mu);
    PoolBuf &code = pool.code, &lits = pool.lits, &kern = pool.kern, &kpar = pool.kpar, &counters = pool.counters,
            &slab = pool.slab, &sfirst = pool.sfirst, &tup = pool.tup, &tst = pool.tst, &taux = pool.taux,
            &tlab = pool.tlab;
    SCK(code.ensure(sizeof(int32_t) * 4 * pr->n_code));
    SCK(cudaMemcpy(code.p, pr->code, sizeof(int32_t) * 4 * pr->n_code, cudaMemcpyHostToDevice));
    SCK(lits.ensure(sizeof(int64_t) * std::max(pr->n_lits, 1)));
    if (pr->n_lits)
        SCK(cudaMemcpy(lits.p, pr->lits, sizeof(int64_t) * pr->n_lits, cudaMemcpyHostToDevice));
    SCK(kern.ensure(sizeof(int32_t) * 4 * std::max(pr->n_kernels, 1)));
    if (pr->n_kernels)
        SCK(cudaMemcpy(kern.p, pr->kernels, sizeof(int32_t) * 4 * pr->n_kernels, cudaMemcpyHostToDevice));
    SCK(kpar.ensure(sizeof(int32_t) * 2 * std::max(pr->n_kparams, 1)));
    if (pr->n_kparams)
        SCK(cudaMemcpy(kpar.p, pr->kparams, sizeof(int32_t) * 2 * pr->n_kparams, cudaMemcpyHostToDevice));
    SCK(counters.ensure(sizeof(unsigned long long) * 8));
    SCK(slab.ensure(sizeof(uint32_t) * ns));
    SCK(sfirst.ensure(sizeof(unsigned long long) * 4 * ns));
    if (D.mode == 1) {
        SCK(tup.ensure(sizeof(int64_t) * std::max<int64_t>(n_out_tuples * D.arity, 1)));
        if (n_out_tuples * D.arity)
            SCK(cudaMemcpy(tup.p, tuples, sizeof(int64_t) * n_out_tuples * D.arity, cudaMemcpyHostToDevice));
        SCK(tst.ensure(sizeof(int32_t) * std::max<int64_t>(n_out_tuples, 1)));
        SCK(taux.ensure(sizeof(int32_t) * std::max<int64_t>(n_out_tuples, 1)));
        SCK(tlab.ensure(std::max<int64_t>(n_out_tuples * ns, 1)));
    }
    sweep::Prog P{(const int32_t*)code.p, (const int64_t*)lits.p, (const int32_t*)kern.p,
                  (const int32_t*)kpar.p, pr->n_code, pr->n_sites, pr->n_slots, pr->n_kernels,
                  (opt && opt->step_limit > 0) ? opt->step_limit : (int64_t)1 << 40};
    D.tuples = (const int64_t*)tup.p;
    D.counters = (unsigned long long*)counters.p;
    D.site_labels = (uint32_t*)slab.p;
    D.site_first = (unsigned long long*)sfirst.p;
    D.t_status = (int32_t*)tst.p;
    D.t_aux = (int32_t*)taux.p;
    D.t_labels = (uint8_t*)tlab.p;

    static int occ = 0;  // the same kernel and block on every device of the box
    if (!occ) SCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, oob_sweep_kernel, BLOCK, 0));
    occ = std::max(occ, 1);
    int64_t want_blocks = (D.total + BLOCK - 1) / BLOCK;
    int64_t blocks = std::min<int64_t>(want_blocks, (int64_t)sms * occ);
    if (opt && opt->max_threads > 0) blocks = std::min<int64_t>(blocks, std::max<int64_t>(opt->max_threads / BLOCK, 1));
    blocks = std::max<int64_t>(blocks, 1);
    int64_t words = (opt && opt->arena_words > 0) ? opt->arena_words : 512;
    const int64_t budget = (int64_t)8 << 30;  // arena bytes
    const int64_t max_words = (int64_t)1 << 26;
    if (!pool.e0) {
        SCK(cudaEventCreate(&pool.e0));
        SCK(cudaEventCreate(&pool.e1));
    }
    cudaEvent_t e0 = pool.e0, e1 = pool.e1;
    float ms = 0.f;
    unsigned long long host_c[8];
    for (;;) {
        while (blocks > 1 && blocks * BLOCK * words * 8 > budget) blocks = (blocks + 1) / 2;
        PoolBuf& arena = pool.arena;
        SCK(arena.ensure((size_t)blocks * BLOCK * words * 8));
        unsigned long long init_c[8] = {0, 0, ~0ull, ~0ull, 0, 0, 0, 0};
        SCK(cudaMemcpy(counters.p, init_c, sizeof(init_c), cudaMemcpyHostToDevice));
        SCK(cudaMemset(slab.p, 0, sizeof(uint32_t) * ns));
        SCK(cudaMemset(sfirst.p, 0xff, sizeof(unsigned long long) * 4 * ns));
        SCK(cudaEventRecord(e0));
        oob_sweep_kernel<<<(unsigned)blocks, BLOCK>>>(P, D, (int64_t*)arena.p, words);
        SCK(cudaGetLastError());
        SCK(cudaEventRecord(e1));
        SCK(cudaEventSynchronize(e1));
        SCK(cudaEventElapsedTime(&ms, e0, e1));
        SCK(cudaMemcpy(host_c, counters.p, sizeof(host_c), cudaMemcpyDeviceToHost));
        bool arena_short = false;
        int64_t first_err = -1;
        int err_code = 0;
        if (D.mode == 0) {
            if (host_c[1]) {
                first_err = (int64_t)(host_c[3] >> 8);
                err_code = (int)(host_c[3] & 255);
                arena_short = err_code == sweep::E_ARENA;
            }
        } else {
            std::vector<int32_t> st(n_out_tuples), ax(n_out_tuples);
            SCK(cudaMemcpy(st.data(), tst.p, sizeof(int32_t) * n_out_tuples, cudaMemcpyDeviceToHost));
            SCK(cudaMemcpy(ax.data(), taux.p, sizeof(int32_t) * n_out_tuples, cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < n_out_tuples; i++)
                if (st[i] == sweep::S_ERROR && ax[i] == sweep::E_ARENA) arena_short = true;
            if (!arena_short) {
                std::copy(st.begin(), st.end(), status);
                std::copy(ax.begin(), ax.end(), aux);
                std::vector<uint8_t> lb(n_out_tuples * ns);
                if (n_out_tuples)
                    SCK(cudaMemcpy(lb.data(), tlab.p, n_out_tuples * ns, cudaMemcpyDeviceToHost));
                for (int64_t i = 0; i < n_out_tuples; i++)
                    std::copy(lb.begin() + i * ns, lb.begin() + i * ns + pr->n_sites, labels + i * pr->n_sites);
            }
        }
        if (arena_short && words < max_words) {
            words *= 4;
            continue;
        }
        if (D.mode == 0) {
            out->executions = D.total;
            out->halted = (int64_t)host_c[0];
            out->errors = (int64_t)host_c[1];
            out->need_tuple = host_c[2] == ~0ull ? -1 : (int64_t)(host_c[2] >> 8);
            out->need_site = host_c[2] == ~0ull ? -1 : (int64_t)(host_c[2] & 255);
            out->error_tuple = first_err;
            out->error_code = err_code;
            out->arena_words_used = (int64_t)host_c[4];
            out->device_ms = ms;
            std::vector<uint32_t> lab(ns);
            std::vector<unsigned long long> fst(4 * ns);
            SCK(cudaMemcpy(lab.data(), slab.p, sizeof(uint32_t) * ns, cudaMemcpyDeviceToHost));
            SCK(cudaMemcpy(fst.data(), sfirst.p, sizeof(unsigned long long) * 4 * ns, cudaMemcpyDeviceToHost));
            for (int s = 0; s < pr->n_sites; s++) {
                if (out->site_labels) out->site_labels[s] = lab[s];
                for (int l = 0; l < 4; l++)
                    if (out->site_first_tuple)
                        out->site_first_tuple[4 * s + l] = fst[4 * s + l] == ~0ull ? -1 : (int64_t)fst[4 * s + l];
            }
            if (host_c[1]) {
                static const char* names[] = {"none", "integer overflow beyond int64", "arena exhausted",
                                              "too many views", "too many storages", "value stack overflow",
                                              "2-D access to a 1-D view", "step limit reached",
                                              "malformed program"};
                return oob_internal_fail(
                    OOB_ERROR, "sweep: " + std::to_string(host_c[1]) + " tuple(s) not executable exactly (first: tuple " +
                                   std::to_string(first_err) + ", " + names[std::min(err_code, 8)] + ")");
            }
        }
        break;
    }
    return OOB_OK;
}

}  // namespace

extern "C" int oob_sweep_run(const oob_sweep_program* prog, int64_t bound, int32_t arity,
                             const oob_sweep_options* opt, oob_sweep_result* out) {
    int rc = validate(prog, arity);
    if (rc) return rc;
    if (!out) return oob_internal_fail(OOB_E_INVALID, "sweep: null result");
    if (bound < 0) return oob_internal_fail(OOB_E_INVALID, "sweep: negative bound");
    // (bound+1)^arity must fit 55 bits (tuple index << 8 in the 64-bit keys)
    __int128 total = 1;
    for (int i = 0; i < arity; i++) {
        total *= (__int128)bound + 1;
        if (total >= ((__int128)1 << 55)) return oob_internal_fail(OOB_E_INVALID, "sweep: tuple space too large");
    }
    Dev D{};
    D.total = (int64_t)total;
    D.bound = bound;
    D.arity = arity;
    D.mode = 0;
    return drive(prog, D, 0, nullptr, opt, out, nullptr, nullptr, nullptr);
}

extern "C" int oob_sweep_replay(const oob_sweep_program* prog, int64_t n, int32_t arity,
                                const int64_t* tuples, const oob_sweep_options* opt, int32_t* status,
                                int32_t* aux, uint8_t* labels) {
    int rc = validate(prog, arity);
    if (rc) return rc;
    if (n < 0 || (n > 0 && (!tuples || !status || !aux || !labels)))
        return oob_internal_fail(OOB_E_INVALID, "sweep: bad replay buffers");
    if (n == 0) return OOB_OK;
    Dev D{};
    D.total = n;
    D.arity = arity;
    D.mode = 1;
    return drive(prog, D, n, tuples, opt, nullptr, status, aux, labels);
}
