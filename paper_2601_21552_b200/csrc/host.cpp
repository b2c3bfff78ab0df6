// host.cpp -- C ABI (include/scuba_oob.h), query compiler and multi-GPU driver.
//
// Pipeline of one oob_solve_batch() call:
//   1. compile  : validate each query of the flat batch, append the divisor
//                 side constraints (solver.py:334-357), expand each constraint
//                 side to a postfix segment, prove the 126-bit (or 62-bit)
//                 magnitude bound, and dedup the code into structure classes;
//   2. schedule : sort by (regime, class, cost) and deal 32-query tiles
//                 round-robin over the devices (queries are independent; no
//                 collective: SURVEY.md 8(e));
//   3. run      : one host thread per device -- H2D, persistent kernel, D2H --
//                 and a capacity retry for queries whose DFS outgrew the
//                 default scratch (deeper stack / longer trail);
//   4. scatter  : verdicts, models, counters back to the caller's arrays.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <dlfcn.h>
#include <signal.h>
#include <sys/time.h>
#include <ucontext.h>

#include "../../include/scuba_oob.h"
#include "format.h"
#include "jit.h"
#include "cert.cuh"
#include "symbolic.cuh"
#include "wide.cuh"

namespace oob {
cudaError_t launch_solve(const LaunchArgs& a, int wide, int blocks, int fblocks, cudaStream_t s);
cudaError_t launch_root(const LaunchArgs& a, int wide, int blocks, cudaStream_t s);
cudaError_t launch_cert(const LaunchArgs& a, int wide, uint32_t k0, uint32_t k1, int sms, cudaStream_t s);
cudaError_t launch_chain(const LaunchArgs& a, int blocks, cudaStream_t s);
cudaError_t launch_enum(const LaunchArgs& a, int blocks, cudaStream_t s);
cudaError_t grow_smem_limit(const void* fn, size_t smem);
cudaError_t launch_expand(int wide, const QDesc* qd, uint32_t n, const void* rawoff, const void* vlo, const void* vhi,
                          const void* lits, const int32_t* litsrc, int64_t* data, int sms, cudaStream_t s);
cudaError_t kernel_occupancy(int wide, int mode, size_t smem, int* blocks_per_sm);
cudaError_t launch_gather_sat(const int8_t* verdict, const QDesc* qd, const int64_t* model, uint32_t n,
                              unsigned long long* counter, uint32_t* sat_off, int64_t* compact, int sms,
                              cudaStream_t s);
}

using namespace oob;
using i128 = __int128;

// ============================================================================
// errors
// ============================================================================
static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

// error reporting for the other translation units of the library (sweep.cu)
int oob_internal_fail(int code, const std::string& msg) { return fail(code, msg); }

// SCUBA_OOB_TRACE=1: per-phase host timings on stderr (compile, pack, stage,
// kernels, fetch) -- the engine's only tracing hook
static int trace_level() {
    static const int lv = [] {
        const char* e = std::getenv("SCUBA_OOB_TRACE");
        return (e && *e) ? std::atoi(e) : 0;
    }();
    return lv;
}
static bool trace_on() { return trace_level() > 0; }
static const std::chrono::steady_clock::time_point g_trace_epoch = std::chrono::steady_clock::now();
thread_local int tl_pool_slot = 0;  // stream API pool slot of this thread (see HostGate)
struct Phase {
    const char* name;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit Phase(const char* n) : name(n) {}
    ~Phase() {
        if (!trace_on()) return;
        using ms = std::chrono::duration<double, std::milli>;
        if (trace_level() >= 3)  // start time + pool slot: shows the overlap of stream batches
            std::fprintf(stderr, "[oob] %-10s %9.3f ms  @%10.3f slot %d\n", name,
                         ms(std::chrono::steady_clock::now() - t0).count(), ms(t0 - g_trace_epoch).count(),
                         tl_pool_slot);
        else
            std::fprintf(stderr, "[oob] %-10s %9.3f ms\n", name, ms(std::chrono::steady_clock::now() - t0).count());
    }
};

// SCUBA_OOB_TIMELINE=<file>: per-entry device timestamps of every solve run
// appended to <file> (tools/timeline.py reads it)
static const char* timeline_path() {
    static const char* p = std::getenv("SCUBA_OOB_TIMELINE");
    return (p && *p) ? p : nullptr;
}

// The engine runs several kernels per device concurrently (root, int64 and
// wide solve kernels, one per compiled class): ask for more hardware work
// queues than the default 8 so that independent streams do not serialise.
// Only effective before the process creates its CUDA context; never
// overrides a value the user set.
// SCUBA_OOB_PROF=<file>: sampling profile of the host pipeline -- SIGPROF
// every 0.5 ms of process CPU time records the interrupted program counter;
// at exit the counters inside this library are written to <file> as offsets
// from its load address (tools/host_profile.sh symbolizes them with
// addr2line).  A diagnostics hook only.
namespace prof {
constexpr size_t CAP = 1 << 20;
std::atomic<size_t> n{0};
uintptr_t pc[CAP];
const char* path = nullptr;
void on_sigprof(int, siginfo_t*, void* uc) {
    const size_t i = n.fetch_add(1, std::memory_order_relaxed);
    if (i < CAP) pc[i] = (uintptr_t)((ucontext_t*)uc)->uc_mcontext.gregs[REG_RIP];
}
void dump() {
    Dl_info info{};
    if (!dladdr((void*)&dump, &info)) return;
    FILE* f = std::fopen(path, "w");
    if (!f) return;
    const uintptr_t base = (uintptr_t)info.dli_fbase;
    const size_t m = std::min(n.load(), CAP);
    size_t outside = 0;
    for (size_t i = 0; i < m; i++) {
        Dl_info d{};
        if (dladdr((void*)pc[i], &d) && d.dli_fbase == info.dli_fbase) std::fprintf(f, "%lx\n", (unsigned long)(pc[i] - base));
        else outside++;
    }
    std::fprintf(f, "# samples %zu outside %zu\n", m, outside);
    std::fclose(f);
}
__attribute__((constructor)) void init() {
    path = std::getenv("SCUBA_OOB_PROF");
    if (!path || !*path) return;
    struct sigaction sa {};
    sa.sa_sigaction = on_sigprof;
    sa.sa_flags = SA_SIGINFO | SA_RESTART;
    sigemptyset(&sa.sa_mask);
    sigaction(SIGPROF, &sa, nullptr);
    itimerval t{};
    t.it_interval.tv_usec = 500;
    t.it_value.tv_usec = 500;
    setitimer(ITIMER_PROF, &t, nullptr);
    std::atexit(dump);
}
}  // namespace prof

__attribute__((constructor)) static void oob_default_connections() {
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "16", 0);
}

static i128 from_w(oob_i128 w) { return (i128)(((unsigned __int128)(uint64_t)w.hi << 64) | w.lo); }

// ============================================================================
// 1. compile
// ============================================================================
namespace {

enum Regime : int8_t { R_IMMEDIATE = 0, R_W64 = 1, R_W128 = 2, R_W256 = 3, R_RANGE = 4, R_INVALID = 5 };

struct QView {
    int nv, ncon, nn, nl;
    const oob_i128 *vlo, *vhi, *lits;
    const uint8_t* rel;
    const int32_t *lhs, *rhs;
    const uint8_t* op;
    const int32_t *na, *nb;
};

QView view_of(const oob_batch* b, int64_t q) {
    QView v;
    int64_t vb = b->var_begin[q], cb = b->con_begin[q], nb = b->node_begin[q], lb = b->lit_begin[q];
    v.nv = (int)(b->var_begin[q + 1] - vb);
    v.ncon = (int)(b->con_begin[q + 1] - cb);
    v.nn = (int)(b->node_begin[q + 1] - nb);
    v.nl = (int)(b->lit_begin[q + 1] - lb);
    v.vlo = b->var_lo + vb;
    v.vhi = b->var_hi + vb;
    v.lits = b->lits + lb;
    v.rel = b->con_rel + cb;
    v.lhs = b->con_lhs + cb;
    v.rhs = b->con_rhs + cb;
    v.op = b->node_op + nb;
    v.na = b->node_a + nb;
    v.nb = b->node_b + nb;
    return v;
}

// the checks on the query's terms and constraints (validate); the compile
// pass runs them only for a query whose terms are not word-for-word those of
// an already validated query (StructCache)
std::string validate_terms(const QView& v) {
    for (int i = 0; i < v.nn; i++) {
        int op = v.op[i];
        if (op > OOB_NODE_MOD) return "unknown operator code " + std::to_string(op);
        if (op == OOB_NODE_LIT && (v.na[i] < 0 || v.na[i] >= v.nl)) return "literal index out of range";
        if (op == OOB_NODE_VAR && (v.na[i] < 0 || v.na[i] >= v.nv)) return "undeclared variable index";
        if (op >= OOB_NODE_ADD && (v.na[i] < 0 || v.na[i] >= i || v.nb[i] < 0 || v.nb[i] >= i))
            return "operand node not before its parent";
    }
    for (int k = 0; k < v.ncon; k++) {
        if (v.rel[k] > OOB_REL_GT) return "unknown relation code " + std::to_string(v.rel[k]);
        if (v.lhs[k] < 0 || v.lhs[k] >= v.nn || v.rhs[k] < 0 || v.rhs[k] >= v.nn)
            return "constraint root out of range";
    }
    return "";
}
// the checks on the query's offsets and sizes (validate)
const char* validate_offsets(const oob_batch* b, int64_t q) {
    if (b->var_begin[q + 1] < b->var_begin[q] || b->con_begin[q + 1] < b->con_begin[q] ||
        b->node_begin[q + 1] < b->node_begin[q] || b->lit_begin[q + 1] < b->lit_begin[q])
        return "decreasing offsets";
    if (b->var_begin[q + 1] - b->var_begin[q] > 65535 || b->con_begin[q + 1] - b->con_begin[q] > 65535)
        return "more than 65535 variables or constraints";
    return nullptr;
}
std::string validate(const oob_batch* b, int64_t q) {
    if (const char* e = validate_offsets(b, q)) return e;
    return validate_terms(view_of(b, q));
}

// structural equality of two input terms (dataclass equality in the reference)
bool same_term(const QView& v, int x, int y) {
    if (x == y) return true;
    if (v.op[x] != v.op[y]) return false;
    if (v.op[x] == OOB_NODE_LIT) return from_w(v.lits[v.na[x]]) == from_w(v.lits[v.na[y]]);
    if (v.op[x] == OOB_NODE_VAR) return v.na[x] == v.na[y];
    return same_term(v, v.na[x], v.na[y]) && same_term(v, v.nb[x], v.nb[y]);
}

// _collect_divisors (solver.py:334-342): pre-order, structural dedup
void collect_divisors(const QView& v, int e, std::vector<int>& out) {
    int op = v.op[e];
    if (op < OOB_NODE_ADD) return;
    if (op == OOB_NODE_DIV || op == OOB_NODE_MOD) {
        int r = v.nb[e];
        bool lit_ok = v.op[r] == OOB_NODE_LIT && from_w(v.lits[v.na[r]]) >= 1;
        if (!lit_ok) {
            bool seen = false;
            for (int d : out) seen = seen || same_term(v, d, r);
            if (!seen) out.push_back(r);
        }
    }
    collect_divisors(v, v.na[e], out);
    collect_divisors(v, v.nb[e], out);
}

// checked 128-bit arithmetic for the bound proof
struct Chk {
    bool ovf = false;
    i128 add(i128 a, i128 b) { i128 r; if (__builtin_add_overflow(a, b, &r)) ovf = true; return r; }
    i128 sub(i128 a, i128 b) { i128 r; if (__builtin_sub_overflow(a, b, &r)) ovf = true; return r; }
    i128 mul(i128 a, i128 b) {
        // both factors within int64: one 64x64->128 multiply, exact (|a*b| < 2^126)
        if (a == (int64_t)a && b == (int64_t)b) return (i128)(int64_t)a * (i128)(int64_t)b;
        i128 r;
        if (__builtin_mul_overflow(a, b, &r)) ovf = true;
        return r;
    }
};
inline i128 iabs(i128 a) { return a < 0 ? -a : a; }
inline i128 imax(i128 a, i128 b) { return a > b ? a : b; }
inline i128 imin(i128 a, i128 b) { return a < b ? a : b; }

const i128 INF_R = (i128)1000000000000000000LL;
// Regime limits.  Every intermediate value is bounded by B (forward
// intervals F, exact values G, narrowing targets T, literals); domain
// arithmetic (hi - lo + 1, lo + hi) additionally needs 2*Dmax + 1.
const i128 I64MAX = (i128)INT64_MAX;
const i128 D64MAX = ((i128)1 << 62) - 1;
const i128 D128MAX = ((i128)1 << 126) - 1;

// The structure of a query (everything but domain and literal VALUES): shared
// by all queries with identical terms, built once per thread per structure.
struct Structure {
    uint32_t nv = 0, ncon = 0, ncode = 0, nlit = 0;
    uint32_t maxcsize = 1;        // largest constraint (lhs + rhs nodes)
    uint32_t maxdepth = 1;        // deepest term
    std::vector<uint32_t> words;  // ncon constraint words + ncode node words + 4 nv membership words
    std::vector<std::pair<uint32_t, uint32_t>> roots;  // per constraint: lhs / rhs root node
    std::vector<uint8_t> rels;
    std::vector<int32_t> lit_src; // per literal slot: the query's input literal index (-1: the constant 1)
    uint64_t key = 0;             // structure-class hash (words, nv, ncon)
    std::string range_why;        // non-empty: the structure alone is beyond the engine (R_RANGE)
    int w128_log2 = -1;           // ... and <= 2^w128_log2: the int128 regime (fast mode's shortcut)
    int w64_log2 = -1;            // every query of this structure whose domain bounds and literals
                                  // are <= 2^w64_log2 in magnitude is in the int64 regime (-1: none)
    const uint32_t* code() const { return words.data() + ncon; }
};

// Structures referenced by one call's Compiled records, which hold plain
// pointers: a reference per distinct structure and compile chunk instead of
// an atomic reference-count update per query (the counts of a few shared
// structures are contended by every compile thread)
struct Pins {
    std::vector<std::shared_ptr<const Structure>> v;
    const Structure* add(const std::shared_ptr<const Structure>& p) {
        const Structure* r = p.get();
        if (last < v.size() && v[last].get() == r) return r;
        const size_t k0 = v.size() > 64 ? v.size() - 64 : 0;  // (a bounded look-back)
        for (size_t k = v.size(); k > k0; k--)
            if (v[k - 1].get() == r) {
                last = k - 1;
                return r;
            }
        last = v.size();
        v.push_back(p);
        first.emplace_back();
        vary.emplace_back();
        seen.push_back(0);
        return r;
    }
    // fast mode: per pinned structure, the literal-slot values of its first
    // device query in the chunk and which slots took another value since
    // (the certificates' parameter scan, done while the values are at hand)
    std::vector<std::vector<i128>> first;
    std::vector<std::vector<uint8_t>> vary;
    std::vector<uint8_t> seen;
    void note_lits(const std::vector<i128>& lits, size_t nlit) {  // for the structure added or hit last
        if (!seen[last]) {
            seen[last] = 1;
            first[last].assign(lits.begin(), lits.begin() + nlit);
            vary[last].assign(nlit, 0);
            return;
        }
        const i128* f = first[last].data();
        uint8_t* y = vary[last].data();
        for (size_t i = 0; i < nlit; i++) y[i] |= lits[i] != f[i];
    }
    size_t last = 0;
};

struct Compiled {
    int8_t regime = R_IMMEDIATE;
    int8_t immediate = OOB_UNSAT;
    const Structure* st = nullptr;  // kept alive by the call's Pins
    uint32_t nv = 0, ncon = 0, ncode = 0, nlit = 0;
    uint32_t maxcsize = 1, maxdepth = 1;
    double cost = 0;
    uint64_t key = 0;             // structure-class hash (words, nv, ncon)
    uint32_t cls = UINT32_MAX;    // batch-wide structure class id (prepare)
    uint32_t lsrc = 0;            // offset of its structure's literal-slot sources in the call's table
    const char* why = nullptr;    // reason for R_RANGE (static text or the pinned structure's)
    const std::vector<uint32_t>& words() const { return st->words; }
};

// literal slot i of query q (values are read from the caller's batch)
inline i128 lit_value(const oob_batch* b, int64_t q, const Structure& st, uint32_t i) {
    const int32_t src = st.lit_src[i];
    return src < 0 ? (i128)1 : from_w(b->lits[b->lit_begin[q] + src]);
}

// Page-locked host blocks, recycled across calls (H2D / D2H at full PCIe /
// C2C bandwidth without a driver staging copy).  Falls back to pageable
// memory when no CUDA context can be created (host-only diagnostics).
struct PinnedPool {
    std::mutex mu;
    std::multimap<size_t, void*> free_;
    void* acquire(size_t bytes, bool* pinned) {
        bytes = std::max<size_t>(bytes, 64);
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = free_.lower_bound(bytes);
            if (it != free_.end() && it->first <= 2 * bytes + (1u << 20)) {
                void* p = it->second;
                free_.erase(it);
                *pinned = true;
                return p;
            }
        }
        void* p = nullptr;
        size_t want = bytes + bytes / 8;
        if (cudaMallocHost(&p, want) == cudaSuccess) {
            *pinned = true;
            std::lock_guard<std::mutex> lk(mu);
            sizes[p] = want;
            return p;
        }
        cudaGetLastError();
        *pinned = false;
        return std::malloc(bytes);
    }
    void release(void* p, bool pinned) {
        if (!p) return;
        if (!pinned) {
            std::free(p);
            return;
        }
        std::lock_guard<std::mutex> lk(mu);
        free_.emplace(sizes[p], p);
    }
    std::unordered_map<void*, size_t> sizes;
};
PinnedPool& pinned_pool() {
    static PinnedPool* pp = new PinnedPool();  // never destroyed: blocks live for the process
    return *pp;
}

// uninitialised page-locked host array (filled in parallel; no zero-fill pass)
template <typename T>
struct HostArr {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    bool pinned = false;
    HostArr() = default;
    HostArr(const HostArr&) = delete;
    HostArr& operator=(const HostArr&) = delete;
    HostArr(HostArr&& o) noexcept : p(o.p), n(o.n), cap(o.cap), pinned(o.pinned) { o.p = nullptr; o.n = o.cap = 0; }
    HostArr& operator=(HostArr&& o) noexcept {
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(cap, o.cap);
        std::swap(pinned, o.pinned);
        return *this;
    }
    ~HostArr() { pinned_pool().release(p, pinned); }
    void alloc(size_t m) {
        if (m > cap || !p) {
            pinned_pool().release(p, pinned);
            cap = std::max<size_t>(m, 1);
            p = (T*)pinned_pool().acquire(cap * sizeof(T), &pinned);
        }
        n = m;
    }
    size_t size() const { return n; }
    T* data() { return p; }
    const T* data() const { return p; }
    T& operator[](size_t i) { return p[i]; }
    const T& operator[](size_t i) const { return p[i]; }
};

// 64-bit FNV-1a over the structure words: the structure-class key
inline uint64_t class_hash(const std::vector<uint32_t>& w, uint32_t nv, uint32_t ncon) {
    uint64_t h = 1469598103934665603ull ^ ((uint64_t)nv << 32 | ncon);
    for (uint32_t x : w) {
        h ^= x;
        h *= 1099511628211ull;
    }
    return h;
}

// host worker threads (SCUBA_OOB_HOST_THREADS caps them; default: cores, <= 32)
unsigned host_threads() {
    static const unsigned n = [] {
        const char* e = std::getenv("SCUBA_OOB_HOST_THREADS");
        unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        unsigned cap = (e && *e) ? (unsigned)std::max(1, std::atoi(e)) : 32u;
        return std::max(1u, std::min(hw, cap));
    }();
    return n;
}

// Persistent host worker pool (thread creation per parallel loop cost ~0.5 ms
// a call, and a solve runs about ten such loops).  Several loops may run at
// once -- the stream API's workers (one batch packing while the next one
// compiles) -- and idle workers take chunks from the oldest loop with work
// left, so one batch's short loop is not queued behind another's long one.
// Each caller works on its own loop too; a loop nested inside a worker runs
// inline.
class HostPool {
  public:
    static HostPool& get() {
        static HostPool* p = new HostPool(host_threads() - 1);  // never destroyed (detached workers)
        return *p;
    }
    // runs body(lo, hi) over [0, n) in chunks of `grain`; false from inside a
    // pool worker (nested sections run serially)
    bool run(size_t n, size_t grain, const std::function<void(size_t, size_t)>& body) {
        if (workers_.empty() || tl_in_pool) return false;
        Loop L;
        L.body = &body;
        L.n = n;
        L.grain = std::max<size_t>(grain, 1);
        {
            std::lock_guard<std::mutex> lk(mu_);
            active_.push_back(&L);
        }
        cv_.notify_all();
        work_on(L);  // the caller takes chunks too
        std::unique_lock<std::mutex> lk(mu_);
        active_.erase(std::find(active_.begin(), active_.end(), &L));
        done_cv_.wait(lk, [&] { return L.done == L.n && L.users == 0; });
        return true;
    }

  private:
    struct Loop {
        const std::function<void(size_t, size_t)>* body = nullptr;
        size_t n = 0, grain = 1;
        std::atomic<size_t> next{0};
        std::atomic<size_t> done{0};  // items finished
        int users = 0;     // workers holding a pointer to this loop (under mu_)
    };
    explicit HostPool(unsigned n) {
        for (unsigned i = 0; i < n; i++) {
            workers_.emplace_back([this] { loop(); });
            workers_.back().detach();
        }
    }
    void work_on(Loop& L) {
        for (;;) {
            const size_t a = L.next.fetch_add(L.grain);
            if (a >= L.n) break;
            const size_t z = std::min(L.n, a + L.grain);
            (*L.body)(a, z);
            if (L.done.fetch_add(z - a) + (z - a) == L.n) {
                std::lock_guard<std::mutex> lk(mu_);  // (the waiter tests under mu_: no lost wake-up)
                done_cv_.notify_all();
            }
        }
    }
    void loop() {
        tl_in_pool = true;
        for (;;) {
            Loop* L = nullptr;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] {
                    for (Loop* x : active_)
                        if (x->next.load() < x->n) {
                            L = x;
                            return true;
                        }
                    return false;
                });
                L->users++;
            }
            work_on(*L);
            std::lock_guard<std::mutex> lk(mu_);
            if (--L->users == 0 && L->done == L->n) done_cv_.notify_all();
        }
    }
    static thread_local bool tl_in_pool;
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<Loop*> active_;
};
thread_local bool HostPool::tl_in_pool = false;

template <typename F>
void parallel_for(size_t n, size_t grain, F f) {
    if (n < 2 * grain || host_threads() == 1) {
        f(0, n);
        return;
    }
    const std::function<void(size_t, size_t)> body = f;
    if (!HostPool::get().run(n, grain, body)) f(0, n);
}

struct Emitter {
    const QView& v;
    std::vector<uint32_t>& code;  // per-thread scratch
    std::vector<int32_t>& lits;   // per literal slot: input literal index (-1: constant 1)
    int max_depth = 0;
    static std::vector<uint32_t>& scratch() {
        static thread_local std::vector<uint32_t> c;
        c.clear();
        return c;
    }
    Emitter(const QView& vv, std::vector<int32_t>& l) : v(vv), code(scratch()), lits(l) {}
    // returns the postfix index of the emitted subtree root
    uint32_t emit(int e, int depth) {
        max_depth = std::max(max_depth, depth);
        int op = v.op[e];
        if (op == OOB_NODE_LIT) {
            lits.push_back(v.na[e]);
            code.push_back(node_word(NODE_LIT, (uint32_t)(lits.size() - 1)));
        } else if (op == OOB_NODE_VAR) {
            code.push_back(node_word(NODE_VAR, (uint32_t)v.na[e]));
        } else {
            size_t start = code.size();
            emit(v.na[e], depth + 1);
            emit(v.nb[e], depth + 1);
            code.push_back(node_word((uint32_t)op, (uint32_t)(code.size() + 1 - start)));
        }
        return (uint32_t)(code.size() - 1);
    }
    uint32_t emit_one() {  // the literal 1 of a divisor side constraint (solver.py:357)
        lits.push_back(-1);
        code.push_back(node_word(NODE_LIT, (uint32_t)(lits.size() - 1)));
        return (uint32_t)(code.size() - 1);
    }
};

inline uint32_t w_op(uint32_t w) { return w & 7u; }
inline uint32_t w_arg(uint32_t w) { return w >> 3; }

// Bound proof over the expanded code (see engine.cuh header).  Returns the
// largest magnitude any intermediate value can reach, or -1 on overflow.
i128 prove_bound(const uint32_t* code, size_t n, const std::vector<std::pair<uint32_t, uint32_t>>& cons,
                 const std::vector<uint8_t>& rels, const std::vector<i128>& dlo,
                 const std::vector<i128>& dhi, const std::vector<i128>& lits) {
    Chk c;
    static thread_local std::vector<i128> tl_flo, tl_fhi, tl_gm, tl_tgt;  // scratch reused across queries
    static thread_local std::vector<char> tl_none, tl_has;
    std::vector<i128>&flo = tl_flo, &fhi = tl_fhi, &gm = tl_gm, &tgt = tl_tgt;
    std::vector<char>&none = tl_none, &has = tl_has;
    flo.resize(n);
    fhi.resize(n);
    gm.resize(n);
    none.assign(n, 0);
    i128 B = 0;
    for (size_t i = 0; i < dlo.size(); i++) B = imax(B, imax(iabs(dlo[i]), iabs(dhi[i])));
    for (i128 l : lits) B = imax(B, iabs(l));
    auto size_of = [&](uint32_t i) { return w_op(code[i]) >= NODE_ADD ? w_arg(code[i]) : 1u; };
    // forward intervals F (exactly _eval_iv at the declared domains) and exact
    // magnitude bounds G, postfix order
    for (size_t j = 0; j < n; j++) {
        uint32_t w = code[j], op = w_op(w);
        if (op == NODE_LIT) {
            flo[j] = fhi[j] = lits[w_arg(w)];
            gm[j] = iabs(flo[j]);
            continue;
        }
        if (op == NODE_VAR) {
            flo[j] = dlo[w_arg(w)];
            fhi[j] = dhi[w_arg(w)];
            if (flo[j] > fhi[j]) none[j] = 1;
            gm[j] = imax(iabs(flo[j]), iabs(fhi[j]));
            continue;
        }
        uint32_t R = (uint32_t)j - 1, L = R - size_of(R);
        i128 gl = gm[L], gr = gm[R];
        switch (op) {
        case NODE_ADD: case NODE_SUB: gm[j] = c.add(gl, gr); break;
        case NODE_MUL: gm[j] = c.mul(gl, gr); break;
        case NODE_DIV: gm[j] = gl; break;
        default: gm[j] = imin(gl, gr); break;
        }
        if (none[L] || none[R]) { none[j] = 1; continue; }
        i128 l0 = flo[L], l1 = fhi[L], r0 = flo[R], r1 = fhi[R];
        if (op == NODE_ADD) { flo[j] = c.add(l0, r0); fhi[j] = c.add(l1, r1); }
        else if (op == NODE_SUB) { flo[j] = c.sub(l0, r1); fhi[j] = c.sub(l1, r0); }
        else if (op == NODE_MUL) {
            i128 k[4] = {c.mul(l0, r0), c.mul(l0, r1), c.mul(l1, r0), c.mul(l1, r1)};
            flo[j] = imin(imin(k[0], k[1]), imin(k[2], k[3]));
            fhi[j] = imax(imax(k[0], k[1]), imax(k[2], k[3]));
        } else {
            i128 d0 = imax(r0, 1), d1 = r1;
            if (d0 > d1) { none[j] = 1; continue; }
            if (op == NODE_DIV) {
                i128 k[4] = {l0 / d0, l0 / d1, l1 / d0, l1 / d1};
                flo[j] = imin(imin(k[0], k[1]), imin(k[2], k[3]));
                fhi[j] = imax(imax(k[0], k[1]), imax(k[2], k[3]));
            } else {
                i128 m = d1 - 1;
                flo[j] = l0 >= 0 ? 0 : imax(l0, -m);
                fhi[j] = l1 <= 0 ? 0 : imin(l1, m);
            }
        }
        if (c.ovf) return -1;
    }
    if (c.ovf) return -1;
    auto fmag = [&](uint32_t i) -> i128 { return none[i] ? 0 : imax(iabs(flo[i]), iabs(fhi[i])); };
    for (size_t j = 0; j < n; j++) B = imax(B, imax(fmag((uint32_t)j), gm[j]));
    // narrowing targets T, top-down from every constraint root.  Root targets
    // per relation (solver.py:240-259): the one-sided ones are +-INF and the
    // other side's forward bound +-1; for "=" arithmetic only happens when the
    // target [max(l0,r0), min(l1,r1)] is non-empty, i.e. inside both sides.
    // Every node of the expanded code has one parent (constraint terms are
    // emitted separately), so one reverse sweep over the postfix code hands
    // each node its parent's target.
    tgt.resize(n);
    has.assign(n, 0);
    for (size_t k = 0; k < cons.size(); k++) {
        i128 fl = fmag(cons[k].first), fr = fmag(cons[k].second), tl, tr;
        switch (rels[k]) {
        case OOB_REL_LT: case OOB_REL_GT:
            tl = imax(INF_R, c.add(fr, 1));
            tr = imax(INF_R, c.add(fl, 1));
            break;
        case OOB_REL_LE: case OOB_REL_GE:
            tl = imax(INF_R, fr);
            tr = imax(INF_R, fl);
            break;
        default:
            tl = tr = imin(fl, fr);
            break;
        }
        tgt[cons[k].first] = tl;
        has[cons[k].first] = 1;
        tgt[cons[k].second] = tr;
        has[cons[k].second] = 1;
    }
    for (size_t i = n; i-- > 0;) {
        if (!has[i]) continue;
        const i128 T = tgt[i];
        B = imax(B, T);
        uint32_t op = w_op(code[i]);
        if (op < NODE_ADD) continue;
        uint32_t R = (uint32_t)i - 1, L = R - size_of(R);
        if (op == NODE_ADD || op == NODE_SUB) {
            tgt[L] = c.add(T, fmag(R));
            tgt[R] = c.add(T, fmag(L));
            has[L] = has[R] = 1;
        } else if (op == NODE_MUL) {
            tgt[L] = tgt[R] = imax(T, INF_R);
            has[L] = has[R] = 1;
        } else if (op == NODE_DIV && w_op(code[R]) == NODE_LIT && lits[w_arg(code[R])] >= 1) {
            i128 cc = lits[w_arg(code[R])];
            tgt[L] = c.add(c.mul(T, cc), cc);
            has[L] = 1;
        }
    }
    return c.ovf ? -1 : B;
}

// Conservative magnitude bound in double precision (used when the exact
// 128-bit proof overflows): |x + y| <= |x| + |y|, |x * y| <= |x||y|,
// |tdiv(a, d)| <= |a|, |a % d| <= min(|a|, |d|); targets as in prove_bound.
// Relative rounding error is far below the 2^250 vs 2^255 margin.
// stop: return as soon as the bound exceeds it (the value is then a lower
// bound of the full one, above `stop`)
double prove_bound_mag(const uint32_t* code, size_t n, const std::vector<std::pair<uint32_t, uint32_t>>& cons,
                       const std::vector<uint8_t>& rels, const std::vector<i128>& dlo, const std::vector<i128>& dhi,
                       const std::vector<i128>& lits, double stop = HUGE_VAL) {
    auto mag = [](i128 v) -> double {
        if (v == (int64_t)v) return std::fabs((double)(int64_t)v);  // one conversion in the common case
        return (double)(v < 0 ? -(long double)v : (long double)v);
    };
    static thread_local std::vector<double> tl_m, tl_t;
    std::vector<double>&m = tl_m, &tg = tl_t;
    m.resize(n);
    double B = 0;
    auto size_of = [&](uint32_t i) { return w_op(code[i]) >= NODE_ADD ? w_arg(code[i]) : 1u; };
    for (size_t j = 0; j < n; j++) {
        uint32_t w = code[j], op = w_op(w);
        if (op == NODE_LIT) m[j] = mag(lits[w_arg(w)]);
        else if (op == NODE_VAR) m[j] = std::max(mag(dlo[w_arg(w)]), mag(dhi[w_arg(w)]));
        else {
            uint32_t R = (uint32_t)j - 1, L = R - size_of(R);
            if (op == NODE_ADD || op == NODE_SUB) m[j] = m[L] + m[R];
            else if (op == NODE_MUL) m[j] = m[L] * m[R];
            else if (op == NODE_DIV) m[j] = m[L];
            else m[j] = std::min(m[L], m[R]);
        }
        B = std::max(B, m[j]);
        if (B > stop) return B;
    }
    const double INF_D = 1e18;
    // targets: one reverse sweep (every node has one parent; prove_bound);
    // -1 = no target
    tg.assign(n, -1.0);
    for (size_t k = 0; k < cons.size(); k++) {
        double fl = m[cons[k].first], fr = m[cons[k].second], tl, tr;
        if (rels[k] == OOB_REL_EQ) tl = tr = std::min(fl, fr);
        else { tl = std::max(INF_D, fr + 1); tr = std::max(INF_D, fl + 1); }
        tg[cons[k].first] = tl;
        tg[cons[k].second] = tr;
    }
    for (size_t i = n; i-- > 0;) {
        const double T = tg[i];
        if (T < 0) continue;
        B = std::max(B, T);
        if (B > stop) return B;
        uint32_t op = w_op(code[i]);
        if (op < NODE_ADD) continue;
        uint32_t R = (uint32_t)i - 1, L = R - size_of(R);
        if (op == NODE_ADD || op == NODE_SUB) {
            tg[L] = T + m[R];
            tg[R] = T + m[L];
        } else if (op == NODE_MUL) {
            tg[L] = tg[R] = std::max(T, INF_D);
        } else if (op == NODE_DIV && w_op(code[R]) == NODE_LIT && lits[w_arg(code[R])] >= 1) {
            double cc = mag(lits[w_arg(code[R])]);
            tg[L] = T * cc + cc;
        }
    }
    return B;
}

// The structure of query q (mode: MODE_SOLVE appends the divisor side
// constraints; they depend on the divisors' literal VALUES, solver.py:353-357).
std::shared_ptr<Structure> build_structure(const QView& v, int mode) {
    auto out = std::make_shared<Structure>();
    Structure& st = *out;
    st.nv = (uint32_t)v.nv;
    static thread_local std::vector<int> divs;
    divs.clear();
    bool has_div = false;
    for (int i = 0; i < v.nn && !has_div; i++) has_div = v.op[i] == OOB_NODE_DIV || v.op[i] == OOB_NODE_MOD;
    if (mode == MODE_SOLVE && has_div)
        for (int k = 0; k < v.ncon; k++) {  // constraint list + side constraints (solver.py:371)
            collect_divisors(v, v.lhs[k], divs);
            collect_divisors(v, v.rhs[k], divs);
        }
    Emitter em(v, st.lit_src);
    for (int k = 0; k < v.ncon; k++) {
        uint32_t l = em.emit(v.lhs[k], 1);
        uint32_t r = em.emit(v.rhs[k], 1);
        st.roots.push_back({l, r});
        st.rels.push_back(v.rel[k]);
    }
    for (int d : divs) {
        if (v.op[d] == OOB_NODE_LIT) continue;  // solver.py:353-357
        uint32_t l = em.emit(d, 1);
        uint32_t r = em.emit_one();
        st.roots.push_back({l, r});
        st.rels.push_back(OOB_REL_GE);
    }
    st.ncon = (uint32_t)st.roots.size();
    st.ncode = (uint32_t)em.code.size();
    st.nlit = (uint32_t)st.lit_src.size();
    if (st.ncode > MAX_CODE || st.nlit > 65535 || st.ncon > 65535) {
        st.range_why = "expanded query too large (" + std::to_string(st.ncode) + " term nodes)";
        return out;
    }
    if (em.max_depth > (int)MAX_TREE_DEPTH - 2) {
        st.range_why = "term nesting deeper than " + std::to_string(MAX_TREE_DEPTH - 2);
        return out;
    }
    st.maxdepth = (uint32_t)std::max(1, em.max_depth);
    for (auto& rt : st.roots) {
        uint32_t lsz = w_op(em.code[rt.first]) >= NODE_ADD ? w_arg(em.code[rt.first]) : 1u;
        st.maxcsize = std::max(st.maxcsize, rt.second + 1 - (rt.first + 1 - lsz));
    }
    st.words.reserve(st.ncon + st.ncode + 4 * st.nv);
    for (size_t k = 0; k < st.roots.size(); k++)
        st.words.push_back(con_word(st.rels[k], st.roots[k].first, st.roots[k].second));
    st.words.insert(st.words.end(), em.code.begin(), em.code.end());
    // membership masks for exact constraint skipping: bit k of variable v is
    // set iff constraint k mentions v (only used when ncon <= 128)
    const size_t mbase = st.words.size();
    st.words.resize(mbase + (size_t)st.nv * 4, 0);
    if (st.ncon <= 128) {
        for (uint32_t k = 0; k < st.ncon; k++) {
            for (uint32_t root : {st.roots[k].first, st.roots[k].second}) {
                uint32_t sz = w_op(em.code[root]) >= NODE_ADD ? w_arg(em.code[root]) : 1u;
                for (uint32_t j = root + 1 - sz; j <= root; j++)
                    if (w_op(em.code[j]) == NODE_VAR)
                        st.words[mbase + 4 * w_arg(em.code[j]) + k / 32] |= 1u << (k % 32);
            }
        }
    }
    st.key = class_hash(st.words, st.nv, st.ncon);
    // int64 acceptance threshold of the structure.  prove_bound_mag is
    // nondecreasing in every domain-bound and literal magnitude (|x|+|y|,
    // |x||y|, min, max, T+m, T*c+c), so the bound computed with every domain
    // [-D, D] and every literal D dominates that of any query whose
    // magnitudes are <= D: the largest D = 2^k passing the int64 test admits
    // such queries without a per-query proof (bisection over k, once per
    // structure and thread).
    {
        std::vector<i128> dlo(st.nv), dhi(st.nv), lits(st.nlit);
        auto ok = [&](int k) {
            const i128 D = (i128)1 << k;
            for (uint32_t i = 0; i < st.nv; i++) { dlo[i] = -D; dhi[i] = D; }
            for (uint32_t i = 0; i < st.nlit; i++) lits[i] = D;
            return prove_bound_mag(st.code(), st.ncode, st.roots, st.rels, dlo, dhi, lits) < 9.2e18;
        };
        int lo = -1, hi = 62;  // invariant: ok(lo) (or lo = -1), !ok(hi + 1)
        if (ok(hi)) lo = hi;
        else
            while (hi - lo > 1) {
                int mid = lo + (hi - lo) / 2;
                if (mid >= 0 && ok(mid)) lo = mid;
                else hi = mid;
            }
        st.w64_log2 = lo;
        // the same for the int128 regime (2^127 = 1.7e38; the double bound's
        // relative rounding error is below 1e-12)
        auto ok128 = [&](int k) {
            const i128 D = (i128)1 << k;
            for (uint32_t i = 0; i < st.nv; i++) { dlo[i] = -D; dhi[i] = D; }
            for (uint32_t i = 0; i < st.nlit; i++) lits[i] = D;
            return prove_bound_mag(st.code(), st.ncode, st.roots, st.rels, dlo, dhi, lits) < 1.6e38;
        };
        lo = -1;
        hi = 125;
        if (ok128(hi)) lo = hi;
        else
            while (hi - lo > 1) {
                int mid = lo + (hi - lo) / 2;
                if (mid >= 0 && ok128(mid)) lo = mid;
                else hi = mid;
            }
        st.w128_log2 = lo;
    }
    return out;
}

// Per-thread cache of structures keyed by the query's input terms: the input
// arrays are compared exactly, plus -- for side constraints -- whether each
// literal divisor is >= 1.  Queries with a non-literal divisor are not cached
// (their side-constraint dedup compares literal values inside the divisors).
struct StructCache {
    struct Entry {
        int mode, nv, ncon, nn, nl;
        std::vector<uint8_t> op, rel, divok;
        std::vector<int32_t> na, nb, lhs, rhs;
        std::shared_ptr<const Structure> st;
    };
    std::unordered_multimap<uint64_t, Entry> map;

    static uint64_t fingerprint(const QView& v, int mode, std::vector<uint8_t>& divok, bool& cacheable, bool& bad) {
        uint64_t h = 1469598103934665603ull ^ ((uint64_t)mode << 56) ^ ((uint64_t)v.nv << 40) ^
                     ((uint64_t)v.ncon << 20) ^ (uint64_t)v.nn;
        auto mix = [&](uint64_t x) {
            h ^= x;
            h *= 1099511628211ull;
        };
        divok.clear();
        cacheable = true;
        bad = false;
        for (int i = 0; i < v.nn; i++) {
            mix((uint64_t)v.op[i] | ((uint64_t)(uint32_t)v.na[i] << 8) | ((uint64_t)(uint32_t)v.nb[i] << 36));
            if (v.op[i] == OOB_NODE_DIV || v.op[i] == OOB_NODE_MOD) {
                const int r = v.nb[i];
                if (r < 0 || r >= i) {  // (not yet validated: invalid indices are not followed)
                    bad = true;
                    continue;
                }
                if (v.op[r] == OOB_NODE_LIT) {
                    if (v.na[r] < 0 || v.na[r] >= v.nl) {
                        bad = true;
                        continue;
                    }
                    divok.push_back(from_w(v.lits[v.na[r]]) >= 1);
                } else {
                    cacheable = false;
                }
            }
        }
        for (int k = 0; k < v.ncon; k++) mix((uint64_t)v.rel[k] | ((uint64_t)(uint32_t)v.lhs[k] << 8) |
                                             ((uint64_t)(uint32_t)v.rhs[k] << 36));
        for (uint8_t d : divok) mix(d);
        return h;
    }
    static bool same(const Entry& e, const QView& v, int mode, const std::vector<uint8_t>& divok) {
        if (e.mode != mode || e.nv != v.nv || e.ncon != v.ncon || e.nn != v.nn || e.nl != v.nl) return false;
        return std::memcmp(e.op.data(), v.op, v.nn) == 0 && std::memcmp(e.na.data(), v.na, v.nn * 4) == 0 &&
               std::memcmp(e.nb.data(), v.nb, v.nn * 4) == 0 && std::memcmp(e.rel.data(), v.rel, v.ncon) == 0 &&
               std::memcmp(e.lhs.data(), v.lhs, v.ncon * 4) == 0 &&
               std::memcmp(e.rhs.data(), v.rhs, v.ncon * 4) == 0 && e.divok == divok;
    }
    // null: the query's terms are invalid (validate_terms).  A query equal
    // word for word to a cached one is valid like it: only the others are
    // checked here
    const Structure* get(const QView& v, int mode, Pins& pins) {
        static thread_local std::vector<uint8_t> divok;
        bool cacheable, bad;
        uint64_t h = fingerprint(v, mode, divok, cacheable, bad);
        if (bad) return nullptr;
        if (!cacheable) {
            if (!validate_terms(v).empty()) return nullptr;
            return pins.add(build_structure(v, mode));
        }
        auto range = map.equal_range(h);
        for (auto it = range.first; it != range.second; ++it)
            if (same(it->second, v, mode, divok)) return pins.add(it->second.st);
        if (!validate_terms(v).empty()) return nullptr;
        std::shared_ptr<const Structure> st = build_structure(v, mode);
        pins.add(st);
        if (map.size() > 4096) map.clear();  // bounded
        Entry e;
        e.mode = mode;
        e.nv = v.nv;
        e.ncon = v.ncon;
        e.nn = v.nn;
        e.nl = v.nl;
        e.op.assign(v.op, v.op + v.nn);
        e.na.assign(v.na, v.na + v.nn);
        e.nb.assign(v.nb, v.nb + v.nn);
        e.rel.assign(v.rel, v.rel + v.ncon);
        e.lhs.assign(v.lhs, v.lhs + v.ncon);
        e.rhs.assign(v.rhs, v.rhs + v.ncon);
        e.divok = divok;
        const Structure* st_ptr = st.get();
        e.st = std::move(st);
        map.emplace(h, std::move(e));
        return st_ptr;
    }
};

// mode: MODE_SOLVE (side constraints), MODE_PROPAGATE / MODE_CHECK (as given)
// fast: the fast mode's regime shortcut -- a query the double-precision
// bound does not admit to int64 but whose magnitudes are within the
// structure's int128 threshold goes to the int128 job without the exact
// proof (which would move some of them to int64: a scheduling choice only;
// every regime is exact for the query it holds)
// literal-slot values of the last query compile_query got that far with (per thread)
thread_local std::vector<i128> tl_cq_lits;

Compiled compile_query(const oob_batch* b, int64_t q, int mode, double timeout_s,
                       const oob_i128* model_in, Pins& pins, bool fast = false) {
    Compiled out;
    QView v = view_of(b, q);
    out.nv = (uint32_t)v.nv;
    // per-thread scratch reused across queries (no allocation per query)
    static thread_local std::vector<i128> dlo, dhi;
    std::vector<i128>& lits = tl_cq_lits;
    static thread_local StructCache cache;
    dlo.resize(v.nv);
    dhi.resize(v.nv);
    bool empty = false;
    for (int i = 0; i < v.nv; i++) {
        if (mode == MODE_CHECK) {
            dlo[i] = dhi[i] = from_w(model_in[b->var_begin[q] + i]);
        } else {
            dlo[i] = from_w(v.vlo[i]);
            dhi[i] = from_w(v.vhi[i]);
        }
        if (dlo[i] > dhi[i]) empty = true;
        if (dhi[i] > dlo[i]) {  // scheduling cost: bits of the domain width
            unsigned __int128 w = (unsigned __int128)(dhi[i] - dlo[i]);
            uint64_t hi64 = (uint64_t)(w >> 64), lo64 = (uint64_t)w;
            out.cost += hi64 ? 128 - __builtin_clzll(hi64) : (lo64 ? 64 - __builtin_clzll(lo64) : 0);
        }
    }
    if (mode == MODE_SOLVE && (empty || !(timeout_s > 0))) {
        if (!validate_terms(v).empty()) {  // (the structure cache is not consulted on this path)
            out.regime = R_INVALID;
            return out;
        }
        out.immediate = empty ? OOB_UNSAT : OOB_TIMEOUT;  // solver.py:374-375 / deadline passed (:391)
        return out;
    }
    out.st = cache.get(v, mode, pins);
    if (!out.st) {  // invalid terms (the caller reports validate()'s message)
        out.regime = R_INVALID;
        return out;
    }
    const Structure& st = *out.st;
    out.ncon = st.ncon;
    out.ncode = st.ncode;
    out.nlit = st.nlit;
    out.maxcsize = st.maxcsize;
    out.maxdepth = st.maxdepth;
    out.key = st.key;
    if (!st.range_why.empty()) {
        out.regime = R_RANGE;
        out.why = st.range_why.c_str();
        return out;
    }
    lits.resize(st.nlit);
    i128 Lmax = 0;
    for (uint32_t i = 0; i < st.nlit; i++) {
        lits[i] = lit_value(b, q, st, i);
        Lmax = imax(Lmax, iabs(lits[i]));
    }
    i128 Dmax = 0;
    for (int i = 0; i < v.nv; i++) Dmax = imax(Dmax, imax(iabs(dlo[i]), iabs(dhi[i])));
    if (Dmax > D128MAX) {
        out.regime = R_RANGE;
        out.why = "domain bounds exceed the 128-bit wire format";
        return out;
    }
    // structure-level acceptance (build_structure): no per-query proof needed
    if (st.w64_log2 >= 0 && imax(Dmax, Lmax) <= ((i128)1 << st.w64_log2) && Dmax <= D64MAX) {
        out.regime = R_W64;
        return out;
    }
    // Fast acceptance: the magnitude bound in double precision dominates the
    // exact one (|x|+|y|, |x||y| instead of interval corners); its rounding
    // error over < 2^14 operations is below 1e-12 relative, so a value under
    // 9.2e18 (I64MAX = 9.223e18) proves the int64 regime.  Otherwise the exact
    // checked 128-bit proof decides.
    // (fast mode: only whether the bound stays under 9.2e18 matters before the
    // int128 shortcut, so its computation stops as soon as it does not)
    double mag = prove_bound_mag(st.code(), st.ncode, st.roots, st.rels, dlo, dhi, lits, fast ? 9.2e18 : HUGE_VAL);
    if (mag < 9.2e18 && Dmax <= D64MAX) {
        out.regime = R_W64;
        return out;
    }
    if (fast && st.w128_log2 >= 0 && imax(Dmax, Lmax) <= ((i128)1 << st.w128_log2) && Dmax <= D128MAX) {
        out.regime = R_W128;
        return out;
    }
    if (fast && mag >= 9.2e18) mag = prove_bound_mag(st.code(), st.ncode, st.roots, st.rels, dlo, dhi, lits);
    // (fast mode: a magnitude bound beyond 2^127 goes to the 256-bit regime
    // without the exact proof -- on C3 the proof admits 14 of 14 000 such
    // queries to int128; a scheduling choice, every regime is exact)
    i128 B = (fast && mag >= 1.7e38) ? (i128)-1 : prove_bound(st.code(), st.ncode, st.roots, st.rels, dlo, dhi, lits);
    if (B >= 0) {
        out.regime = (B <= I64MAX && Dmax <= D64MAX) ? R_W64 : R_W128;
    } else if (mag < 1.8e75) {  // < 2^250
        out.regime = R_W256;
    } else {
        out.regime = R_RANGE;
        out.why = "intermediate magnitudes exceed the exact 256-bit regime";
        return out;
    }
    return out;
}

// ============================================================================
// 2./3. device pool, schedule, run
// ============================================================================
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (trace_level() >= 3)
            std::fprintf(stderr, "[oob]   device buffer %p grows %.1f -> %.1f MiB\n", (const void*)this, cap / 1048576.0,
                         bytes / 1048576.0);
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max(bytes, (size_t)1 << 16);
        want = want + want / 4;
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

// fast-mode warp-per-query search (chain.cuh): grid, per-warp frame words
// (chain::DEPTH frames of chain::MAXV domain pairs), budgets
constexpr int CHAIN_WARPS = 4;
constexpr size_t CHAIN_FRAME_WORDS = (size_t)64 * 2 * 64;
int chain_blocks(int sms) { return sms * 4; }
struct ChainCfg {
    bool on = false;
    uint32_t nodes = 512, rounds = 4096;
};
const ChainCfg& chain_cfg() {
    static const ChainCfg c = [] {
        ChainCfg r;
        const char* e = std::getenv("SCUBA_OOB_CHAIN");
        if (e && *e == '1') r.on = true;
        if ((e = std::getenv("SCUBA_OOB_CHAIN_NODES")) && *e) r.nodes = (uint32_t)std::max(1, std::atoi(e));
        if ((e = std::getenv("SCUBA_OOB_CHAIN_ROUNDS")) && *e) r.rounds = (uint32_t)std::max(1, std::atoi(e));
        return r;
    }();
    return c;
}

uint32_t enum_max_points() {
    static const uint32_t v = [] {
        const char* e = std::getenv("SCUBA_OOB_ENUM_MAX");
        return (uint32_t)((e && *e) ? std::max(0, std::atoi(e)) : 4096);
    }();
    return v;
}

struct DevicePool {
    std::mutex mu;
    DevBuf qdesc, code, data, slabT, slabU, next, verdict, model, nodes, passes, elapsed, err;
    DevBuf classes, class_next, class_init, warp_class;
    DevBuf heavy_count, heavy_list, heavy_t0, fr_region;
    DevBuf resume, resume_init, slot64, slot128, slotx32, timeline, classes_interp, stats, certs;
    DevBuf satcnt, satoff, compact;  // SOLVE fetch: packed Sat models
    DevBuf fr_map;                   // frontier region pool: held bits
    DevBuf slab_map;                 // slab pool (SOLVE kernels): held bits
    DevBuf handoff;                  // root states of queries handed off at their root
    DevBuf raw_vlo, raw_vhi, raw_l, litsrc;  // SOLVE: the call's raw values (device-side records)
    DevBuf rawoff;                   // per entry: raw var / literal offsets, literal-source table offset
    DevBuf chain;                    // fast mode: DFS frames of the warp-per-query search (chain.cuh)
    std::vector<cudaStream_t> xs;  // extra streams (one per compiled-class kernel)
    std::vector<cudaEvent_t> xev;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evr = nullptr, evraw = nullptr;
    int sms = 148;
    void release_all() {
        for (DevBuf* b : {&qdesc, &code, &data, &slabT, &slabU, &next, &verdict, &model, &nodes, &passes,
                          &elapsed, &err, &classes, &class_next, &class_init, &warp_class, &heavy_count, &heavy_list,
                          &heavy_t0, &fr_region, &resume, &resume_init, &slot64, &slot128, &slotx32, &timeline,
                          &classes_interp, &stats, &certs, &satcnt, &satoff, &compact, &fr_map, &slab_map, &handoff,
                          &raw_vlo, &raw_vhi, &raw_l, &litsrc, &rawoff, &chain})
            b->release();
    }
};

std::mutex g_pools_mu;
std::vector<std::unique_ptr<DevicePool>> g_pools;

// one pool (buffers + stream) per (device, regime): the int64, int128 and
// 256-bit jobs of a batch run concurrently on their own streams, so their
// tails overlap on the device
// Pipelined calls (oob_solve_batch on a large batch) run chunks concurrently
// on separate pool slots; the host-heavy part of a chunk (compile, pack,
// upload, launch) is serialised by a gate so that chunk k+1's host work
// overlaps chunk k's kernels.
struct HostGate {
    std::mutex mu;
    std::condition_variable cv;
    int turn = 0;  // the chunk whose host phase may run
};
thread_local HostGate* tl_gate = nullptr;
thread_local int tl_chunk = 0;
thread_local bool tl_gate_held = false;
// stream API: the host phase after which the next batch's host work may
// start (SCUBA_OOB_GATE = compile | schedule | pack | launch; default
// compile: the next batch compiles while this one schedules, packs and runs)
enum { GATE_COMPILE = 0, GATE_SCHEDULE = 1, GATE_PACK = 2, GATE_LAUNCH = 3 };
int gate_point() {
    static const int g = [] {
        const char* e = std::getenv("SCUBA_OOB_GATE");
        if (!e || !*e) return (int)GATE_COMPILE;
        std::string v(e);
        return v == "compile" ? (int)GATE_COMPILE : v == "schedule" ? (int)GATE_SCHEDULE
                                                  : v == "pack" ? (int)GATE_PACK : (int)GATE_LAUNCH;
    }();
    return g;
}
void gate_release() {
    if (!tl_gate || !tl_gate_held) return;
    {
        std::lock_guard<std::mutex> lk(tl_gate->mu);
        tl_gate->turn = tl_chunk + 1;
    }
    tl_gate->cv.notify_all();
    tl_gate_held = false;
}

// device jobs: 0 int64, 1 int128, 2 256-bit (proven at the declared domains),
// 3 x32 (only shadows: queries the int64 root phase proves small enough)
constexpr int NJOBS = 4;
constexpr int W_X32 = 3;
inline size_t tbytes_of(int w) { return w == 3 ? 4 : (w == 2 ? 32 : (w == 1 ? 16 : 8)); }

// Logical devices (test knob SCUBA_OOB_VIRTUAL_DEVICES=k): one call deals its
// queries over k logical devices -- k host threads, k sets of device pools --
// that map onto the visible GPUs round-robin, so the multi-device dealing and
// gather can be exercised (and shown to give identical results) on one B200.
int env_virtual_devices() {
    const char* e = std::getenv("SCUBA_OOB_VIRTUAL_DEVICES");
    return (e && *e) ? std::max(0, std::min(64, std::atoi(e))) : 0;
}
int visible_devices();
int phys_dev(int dev) {
    if (env_virtual_devices() <= 0) return dev;
    const int v = visible_devices();
    return v > 0 ? dev % v : dev;
}

// frees the device buffers of one pool slot (every device)
void release_slot_pools(int slot) {
    std::lock_guard<std::mutex> lk(g_pools_mu);
    for (size_t i = 0; i < g_pools.size(); i++) {
        if (!g_pools[i] || (int)(i / NJOBS / 64) != slot) continue;
        std::lock_guard<std::mutex> lk2(g_pools[i]->mu);
        cudaSetDevice(phys_dev((int)((i / NJOBS) % 64)));
        g_pools[i]->release_all();
    }
}

DevicePool* pool_for(int dev, int wide) {
    std::lock_guard<std::mutex> lk(g_pools_mu);
    size_t slot = ((size_t)tl_pool_slot * 64 + (size_t)dev) * NJOBS + (size_t)wide;
    if (g_pools.size() <= slot) g_pools.resize(slot + 1);
    if (!g_pools[slot]) g_pools[slot].reset(new DevicePool());
    return g_pools[slot].get();
}

struct RunCtx {
    const oob_batch* b;
    oob_options opt;
    std::vector<Compiled>* comp;
    const std::vector<uint32_t>* qcls;  // structure class per query (compact copy of comp[q].cls)
    int mode;
    // outputs (caller arrays, or internal for propagate/check)
    int8_t* verdict;
    oob_i128* model;      // SOLVE: lo per var; PROPAGATE: (lo,hi) pairs; CHECK: input model
    int64_t* nodes;
    int64_t* passes;
    double* elapsed;
    std::vector<int8_t>* errs;
    // fast mode: Unsat certificates per batch-wide structure class (cert.cuh)
    const std::vector<uint64_t>* certs = nullptr;
    const std::vector<uint32_t>* cert_off = nullptr;  // per class, NO_CERT: none
    // SOLVE: the records are written on the device from the caller's raw
    // values (copied to page-locked memory by the compile pass): domains and
    // input literals at their batch offsets minus raw_v0 / raw_l0, and the
    // literal-slot sources of every structure the call uses
    bool raw = false;
    const int64_t *raw_vlo = nullptr, *raw_vhi = nullptr, *raw_l = nullptr;  // int64 (the call's values fit)
    uint64_t raw_nv = 0, raw_nl = 0;
    int64_t raw_v0 = 0, raw_l0 = 0;
    const std::vector<int32_t>* litsrc = nullptr;
};

constexpr size_t SMEM_WARP_MAX = 48 * 1024;  // hot state per warp kept on chip up to this

SlabGeom make_geom(uint32_t maxv, uint32_t maxcode, uint32_t maxlit, uint32_t depth_cap, uint32_t trail_cap,
                   uint32_t maxcsize, uint32_t maxdepth, size_t tbytes) {
    SlabGeom g{};
    g.maxcsize = std::max(maxcsize, 1u);
    g.st_cap = maxdepth + 2;
    {
        uint64_t o = 0;
        auto sput = [&](uint64_t& off, uint64_t count) { off = o; o += count * 32; };
        sput(g.o_s_env_lo, std::max(maxv, 1u));
        sput(g.o_s_env_hi, std::max(maxv, 1u));
        sput(g.o_s_val_lo, g.maxcsize);
        sput(g.o_s_val_hi, g.maxcsize);
        sput(g.o_s_st0, g.st_cap);
        sput(g.o_s_st1, g.st_cap);
        g.o_s_lit = 0;  // literal slots stay in the L1-cached global slab
        g.o_s_stn_bytes = (size_t)o * tbytes;
        size_t bytes = g.o_s_stn_bytes + (size_t)g.st_cap * 32 * 4;
        bytes = (bytes + 15) & ~(size_t)15;
        g.smem_per_warp = bytes <= SMEM_WARP_MAX ? (uint32_t)bytes : 0;
    }
    g.maxv = std::max(maxv, 1u);
    g.maxcode = std::max(maxcode, 1u);
    g.maxlit = std::max(maxlit, 1u);
    g.depth_cap = depth_cap;
    g.trail_cap = trail_cap;
    uint64_t o = 0;
    auto put = [&](uint64_t& off, uint64_t count) { off = o; o += count * 32; };
    put(g.o_env_lo, g.maxv);
    put(g.o_env_hi, g.maxv);
    put(g.o_val_lo, g.maxcsize);
    put(g.o_val_hi, g.maxcsize);
    put(g.o_lit, g.maxlit);
    put(g.o_fr_mid, depth_cap);
    put(g.o_fr_hi, depth_cap);
    put(g.o_tr_lo, trail_cap);
    put(g.o_tr_hi, trail_cap);
    put(g.o_st0, g.st_cap);
    put(g.o_st1, g.st_cap);
    g.slab_T_words = o;
    o = 0;
    put(g.o_stamp, g.maxv);
    put(g.o_fr_pick, depth_cap);
    put(g.o_fr_mark, depth_cap);
    put(g.o_fr_clean, (uint64_t)depth_cap * 4);
    put(g.o_tr_var, trail_cap);
    put(g.o_stn, g.st_cap);
    g.slab_u32_words = o;
    return g;
}

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess)                                                                    \
            return std::string(#x) + ": " + cudaGetErrorString(e_);                              \
    } while (0)

constexpr uint32_t DEPTH_CAP0 = 128, TRAIL_CAP0 = 1024;
constexpr int BLOCKS_PER_SM = 16;
constexpr uint32_t WARPS_PER_BLOCK = 2;  // kernels.cu THREADS / 32

// One device's share of one regime: packed device records + launch geometry.
struct DevJob {
    int dev = 0;
    int wide = 0;
    std::vector<int64_t> qs;     // caller query ids, in schedule order
    std::vector<int64_t> shadows;  // wider-regime queries this job may resume (SOLVE mode)
    std::vector<uint8_t> is_shadow;  // per scheduled entry
    std::vector<uint32_t> resume_init;  // per scheduled entry (format.h resume words)
    std::vector<uint32_t> slot[3];      // per entry, index of its shadow in job[0] / job[1] / job[3] (x32)
    // run-time compiled classes (int64 SOLVE jobs, jit.cpp): one kernel each
    std::vector<uint32_t> jit_cls;      // class ids
    std::vector<const void*> jit_fn;
    std::vector<uint32_t> jit_blocks;
    std::vector<LaunchArgs> jit_args;
    std::vector<ClassDesc> cls_interp;  // the class table of the interpreting kernel (JIT classes emptied)
    double jit_ms = 0;
    uint64_t jit_queries = 0;
    std::vector<uint64_t> mo;    // device-local model offset (vars) per scheduled query
    std::vector<uint32_t> code;  // class code blocks
    HostArr<int64_t> data;       // per query domains + literal slots
    HostArr<QDesc> qd;
    std::vector<ClassDesc> cls;
    std::vector<uint32_t> warp_class;
    uint32_t maxv = 1, maxcode = 1, maxlit = 1, maxcsize = 1, maxdepth = 1;
    uint64_t model_words = 0;
    uint32_t n_classes = 0;
    uint32_t blocks = 1, fblocks = 0;
    uint32_t fr_regions = 0;     // frontier scratch regions of the job (shared by its launches)
    uint32_t slab_slots = 0;     // per-warp slabs of the job (SOLVE: a pool shared by its launches)
    uint32_t root_blocks = 1;  // root kernel: one thread per query (grid-stride)
    uint32_t tail_blocks = 0;    // wide SOLVE jobs: frontier-only launch after the int64 kernel
    LaunchArgs tail_args{};
    SlabGeom g{};
    LaunchArgs a{};
    size_t out_model_words = 0;
    bool staged = false;
    float last_ms = 0;
    int64_t last_sat_vars = -1;  // packed Sat-model vars of the last fetch (SOLVE), -1: unpacked
    bool data_uploaded = false;  // records already on their way (uploaded right after pack)
    std::string upload_err;
    bool dev_fill = false;       // SOLVE: records written on the device (oob_expand_kernel) from the raw values
    uint64_t data_words = 0;     // record words of the job (data[] on the device)
    HostArr<uint32_t> rawoff;    // dev_fill: per entry {var offset, literal offset, literal-source offset, 0}
    DevicePool* raw_pool = nullptr;  // dev_fill: the pool holding the call's raw values on this device

    uint64_t record_bytes() const {  // algorithmic input bytes of one launch (x32 records: written on device)
        return qd.size() * sizeof(QDesc) + cls.size() * sizeof(ClassDesc) + code.size() * 4 +
               (wide == W_X32 ? 0 : data_words * 8);
    }
};

void pack(const RunCtx& rc, DevJob& j, bool inline_fill = false) {
    const auto pack_t0 = std::chrono::steady_clock::now();
    const std::vector<Compiled>& comp = *rc.comp;
    const oob_batch* b = rc.b;
    const std::vector<uint32_t>& qcls = *rc.qcls;  // 4 bytes per query: cache-resident, unlike comp[]
    // The job's entries are its own queries, then its shadows, each list in
    // class runs (prepare's class-major schedule).  Entries are grouped by
    // structure class (batch-wide ids) keeping their order within a class
    // (the lockstep kernel runs each warp on one class): the runs are found
    // in parallel, placed serially (a few per class), and copied + filled in
    // parallel.  Scratch is reused across calls (per calling thread).
    static thread_local std::vector<int64_t> tl_own;
    std::vector<int64_t>& own = tl_own;
    own.swap(j.qs);
    const size_t n_own = own.size(), n = n_own + j.shadows.size();
    const int64_t* shp = j.shadows.data();
    auto entry = [&](size_t i) -> int64_t { return i < n_own ? own[i] : ~shp[i - n_own]; };
    auto qid = [](int64_t e) { return e < 0 ? ~e : e; };
    struct Run {
        uint32_t g;
        size_t at, len;
    };
    const size_t RCH = 16384;
    const size_t nrch = (n + RCH - 1) / RCH;
    std::vector<std::vector<Run>> chunk_runs(nrch);
    auto find_runs = [&](size_t c0, size_t c1) {
        for (size_t ch = c0; ch < c1; ch++) {
            std::vector<Run>& R = chunk_runs[ch];
            const size_t z = std::min(n, (ch + 1) * RCH);
            for (size_t i = ch * RCH; i < z; i++) {
                const uint32_t g = qcls[qid(entry(i))];
                if (R.empty() || R.back().g != g) R.push_back({g, i, 0});
                R.back().len++;
            }
        }
    };
    find_runs(0, nrch);  // (serial: ~2 ns an entry, less than waking the pool)
    std::vector<Run> runs;
    for (const auto& R : chunk_runs)
        for (const Run& r : R) {
            if (!runs.empty() && runs.back().g == r.g) runs.back().len += r.len;
            else runs.push_back(r);
        }
    // local class ids in order of first appearance
    std::unordered_map<uint32_t, uint32_t> local;
    std::vector<size_t> rep;  // first entry of every local class
    std::vector<uint32_t> run_cls(runs.size());
    for (size_t r = 0; r < runs.size(); r++) {
        auto it = local.emplace(runs[r].g, (uint32_t)rep.size());
        if (it.second) rep.push_back(runs[r].at);
        run_cls[r] = it.first->second;
    }
    const size_t nc = rep.size();
    std::vector<uint64_t> count(nc + 1, 0);
    for (size_t r = 0; r < runs.size(); r++) count[run_cls[r] + 1] += runs[r].len;
    for (size_t c = 0; c < nc; c++) count[c + 1] += count[c];
    j.code.clear();
    j.cls.assign(nc, ClassDesc{});
    // data layout: per entry (2 nv + nlit) values of the job's width, padded
    // to 16 bytes (x32/int64/int128) or 32 bytes (256-bit); every entry of a
    // class has the same data size, so offsets follow from the class bases
    const size_t tb = tbytes_of(j.wide);
    const size_t vw = tb >= 8 ? tb / 8 : 1;  // int64 words per value (x32 entries are shadows only)
    const size_t align = j.wide == 2 ? 4 : 2;
    std::vector<uint64_t> dbase(nc), dsz(nc), mbase(nc);
    uint64_t dtot = 0, mtot = 0;
    for (size_t id = 0; id < nc; id++) {
        const Compiled& c = comp[qid(entry(rep[id]))];
        ClassDesc& cd = j.cls[id];
        cd.code_off = (uint32_t)j.code.size();
        j.code.insert(j.code.end(), c.words().begin(), c.words().end());
        cd.nv_ncon = c.nv | (c.ncon << 16);
        cd.ncode_nlit = c.ncode | (c.nlit << 16);
        cd.q_begin = (uint32_t)count[id];
        cd.q_end = (uint32_t)count[id + 1];
        cd.cert = (rc.cert_off && c.cls < rc.cert_off->size()) ? (*rc.cert_off)[c.cls] : NO_CERT;
        j.maxv = std::max(j.maxv, c.nv);
        j.maxcode = std::max(j.maxcode, c.ncode);
        j.maxlit = std::max(j.maxlit, c.nlit);
        j.maxcsize = std::max(j.maxcsize, c.maxcsize);
        j.maxdepth = std::max(j.maxdepth, c.maxdepth);
        const uint64_t words = ((2 * (uint64_t)c.nv + c.nlit) * tb + 7) / 8;
        dsz[id] = ((words + align - 1) / align) * align;
        dbase[id] = dtot;
        mbase[id] = mtot;
        dtot += dsz[id] * (count[id + 1] - count[id]);
        mtot += (uint64_t)c.nv * (count[id + 1] - count[id]);
    }
    j.n_classes = (uint32_t)nc;
    j.model_words = mtot;
    // copy segments: every run at its place in its class, cut into pieces
    struct Seg {
        size_t src, dst, len;
        uint32_t cls;
    };
    std::vector<Seg> segs;
    {
        std::vector<uint64_t> at(count.begin(), count.end() - 1);
        const size_t PIECE = 2048;
        for (size_t r = 0; r < runs.size(); r++) {
            const uint32_t c = run_cls[r];
            for (size_t k = 0; k < runs[r].len; k += PIECE)
                segs.push_back({runs[r].at + k, at[c] + k, std::min(PIECE, runs[r].len - k), c});
            at[c] += runs[r].len;
        }
    }
    if (trace_level() >= 2)
        std::fprintf(stderr, "[oob]   pack w%d: %zu entries, %zu classes, %zu runs, serial part %.3f ms\n", j.wide, n,
                     nc, runs.size(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - pack_t0).count());
    j.qs.resize(n);
    j.is_shadow.resize(n);
    j.resume_init.resize(n);
    j.mo.resize(n);
    j.qd.alloc(n);
    j.dev_fill = rc.raw && rc.mode == MODE_SOLVE && j.wide != W_X32;
    j.data_words = std::max<uint64_t>(dtot, 4);
    if (j.dev_fill) j.rawoff.alloc(4 * std::max<size_t>(n, 1));
    else j.data.alloc(j.data_words);
    auto fill = [&](size_t s0, size_t s1) {
        for (size_t si = s0; si < s1; si++) {
            const Seg& sg = segs[si];
            const ClassDesc& cd = j.cls[sg.cls];
            const uint64_t ds = dsz[sg.cls];
            for (size_t k = 0; k < sg.len; k++) {
                const int64_t e = entry(sg.src + k);
                const int64_t q = qid(e);
                const size_t i = sg.dst + k;
                const uint64_t rank = i - cd.q_begin;
                j.qs[i] = q;
                j.is_shadow[i] = e < 0;
                j.resume_init[i] = e < 0 ? RES_SKIP : 0u;
                QDesc& d = j.qd[i];
                d.code_off = cd.code_off;
                d.nv_ncon = cd.nv_ncon;
                d.ncode_nlit = cd.ncode_nlit;
                d.out_q = (uint32_t)i;
                d.data_off = dbase[sg.cls] + rank * ds;
                const uint32_t nv = cd.nv_ncon & 0xFFFFu;
                d.out_v = mbase[sg.cls] + rank * nv;
                j.mo[i] = d.out_v;
                const Compiled& c = comp[q];
                if (j.dev_fill) {  // the device writes the record (oob_expand_kernel)
                    uint32_t* ro = j.rawoff.data() + 4 * i;
                    ro[0] = e < 0 ? UINT32_MAX : (uint32_t)(b->var_begin[q] - rc.raw_v0);
                    ro[1] = e < 0 ? 0u : (uint32_t)(b->lit_begin[q] - rc.raw_l0);
                    ro[2] = c.lsrc;
                    ro[3] = 0;
                    continue;
                }
                if (e < 0) continue;  // a shadow: written on the device before it is ever read
                int64_t* out = j.data.data() + d.data_off;
                int64_t* end = out + ds;
                auto put = [&](i128 x) {
                    *out++ = (int64_t)(uint64_t)x;
                    if (vw >= 2) *out++ = (int64_t)(x >> 64);
                    if (vw == 4) {
                        int64_t sgn = x < 0 ? -1 : 0;
                        *out++ = sgn;
                        *out++ = sgn;
                    }
                };
                const int64_t vb = b->var_begin[q];
                for (uint32_t v = 0; v < nv; v++) {
                    if (rc.mode == MODE_CHECK) {
                        i128 m = from_w(rc.model[vb + v]);
                        put(m);
                        put(m);
                    } else {
                        put(from_w(b->var_lo[vb + v]));
                        put(from_w(b->var_hi[vb + v]));
                    }
                }
                const Structure& st = *c.st;
                const int64_t lb = b->lit_begin[q];
                for (uint32_t li = 0; li < c.nlit; li++) {
                    const int32_t src = st.lit_src[li];
                    put(src < 0 ? (i128)1 : from_w(b->lits[lb + src]));
                }
                std::fill(out, end, 0);
            }
        }
    };
    if (inline_fill) fill(0, segs.size());
    else parallel_for(segs.size(), 1, fill);
    if (n == 0 && !j.dev_fill) std::fill(j.data.data(), j.data.data() + j.data.size(), 0);
    if (j.code.empty()) j.code.push_back(0);
    if (j.cls.empty()) j.cls.push_back(ClassDesc{});
}

// starting class of every warp, in proportion to the class sizes
void assign_warps(DevJob& j, const std::vector<ClassDesc>& cls, uint32_t n_warps) {
    j.warp_class.assign(n_warps, NO_CLASS);  // no class left for this kernel: its warps exit at once
    uint64_t total = 0;
    std::vector<uint32_t> live;
    for (uint32_t c = 0; c < cls.size(); c++)
        if (cls[c].q_end > cls[c].q_begin) {
            total += cls[c].q_end - cls[c].q_begin;
            live.push_back(c);
        }
    if (total == 0) return;
    uint32_t w = 0;
    for (uint32_t c : live) {
        if (w >= n_warps) break;
        uint64_t size = cls[c].q_end - cls[c].q_begin;
        uint64_t share = std::max<uint64_t>(1, (size * n_warps + total - 1) / total);
        share = std::min<uint64_t>(share, (size + 31) / 32);
        for (uint64_t k = 0; k < share && w < n_warps; k++) j.warp_class[w++] = c;
    }
    for (size_t i = 0; w < n_warps; w++, i = (i + 1) % live.size()) j.warp_class[w] = live[i];
}

inline bool demote_on(const RunCtx& rc) { return rc.mode == MODE_SOLVE && !(rc.opt.flags & OOB_F_NO_DEMOTE); }
inline bool x32_on(const RunCtx& rc) { return demote_on(rc) && !(rc.opt.flags & OOB_F_NO_X32); }

// JIT policy: classes with at least jit_min queries (default 1024) in an int64
// SOLVE job run as run-time compiled kernels (oob_options.jit_min, else
// SCUBA_OOB_JIT_MIN; OOB_F_NO_JIT disables; if NVRTC is unavailable the
// classes stay on the interpreting kernel)
uint64_t jit_min() {
    static const uint64_t m = [] {
        const char* e = std::getenv("SCUBA_OOB_JIT_MIN");
        return (e && *e) ? (uint64_t)std::strtoull(e, nullptr, 10) : (uint64_t)1024;
    }();
    return m;
}
constexpr uint32_t JIT_MAX_NV = 48, JIT_MAX_LIT = 48, JIT_MAX_CODE = 1024;
// block geometry of the compiled-class kernels: warps per block and the
// dynamic shared memory requested per block (an occupancy lever: enough of it
// keeps one class per SM, so an SM's instruction cache holds one class's code)
uint32_t jit_warps() {
    static const uint32_t w = [] {
        const char* e = std::getenv("SCUBA_OOB_JIT_WARPS");
        return (uint32_t)std::max(1, std::min(8, (e && *e) ? std::atoi(e) : 8));
    }();
    return w;
}
uint32_t jit_smem() {
    static const uint32_t b = [] {
        const char* e = std::getenv("SCUBA_OOB_JIT_SMEM");
        return (uint32_t)std::max(0, (e && *e) ? std::atoi(e) : 0);
    }();
    return b;
}

// allocate + upload the packed records of `j` into pool P (caller holds P->mu)
constexpr uint32_t FR_ECAP = 2048, FR_UCAP = 4096, FR_LOGCAP = 32768;
// (B200 A/B with the root hand-off resume, identical results: 16 -> 24 nodes
// C3 -9%, C4 -3%, C5s neutral)
constexpr uint32_t HEAVY_NODES_DEFAULT = 24;
// long propagation chains leave the shared lockstep warps (B200 A/B, two
// repeats, identical results, median plan run: 256 -> 192 passes C3 -2%,
// C4 -2%, C5s -4%; with the root hand-off resume and 24-node hand-off,
// 192 -> 128: C3 -7%, C4 +0.5%, C5s neutral)
constexpr uint32_t HEAVY_PASSES_DEFAULT = 128;

// fast mode (OOB_F_FAST): every entry's class certificate is checked first
// (oob_cert_kernel); SCUBA_OOB_FAST_FRONTIER=1 additionally runs the symbolic
// prover itself on heavy queries in the (interpreting) frontier, which then
// receives them earlier than in canonical mode
bool fast_frontier() {
    static const bool v = [] {
        const char* e = std::getenv("SCUBA_OOB_FAST_FRONTIER");
        return e && *e == '1';
    }();
    return v;
}
// Fast mode hand-off thresholds.  With the Unsat bulk refuted up front, the
// queries left are mostly Sat with a few dozen DFS nodes; handing them to the
// frontier after 24 nodes only queues them behind the few warps that serve a
// class's heavy list (B200 A/B, identical results, plan-run ms, 128-pass
// hand-off: C3 24 nodes 7.6, 96 nodes 6.4, never 5.3; C4 24 13.3, 96 13.0,
// never 25.0 -- C4's long Sat chains still need the frontier): 96 nodes.
// With the frontier prover (SCUBA_OOB_FAST_FRONTIER=1) heavy queries should
// meet it early: 8 nodes / 32 passes.
// SCUBA_OOB_HANDOFF_GATE=0 disables the fast mode's hand-off gate
bool handoff_gate_env() {
    static const bool v = [] {
        const char* e = std::getenv("SCUBA_OOB_HANDOFF_GATE");
        return !(e && *e == '0');
    }();
    return v;
}
uint32_t fast_heavy_nodes() {
    static const uint32_t v = [] {
        const char* e = std::getenv("SCUBA_OOB_FAST_HEAVY_NODES");
        return (uint32_t)std::max(1, (e && *e) ? std::atoi(e) : (fast_frontier() ? 8 : 96));
    }();
    return v;
}
uint32_t fast_heavy_passes(uint32_t canonical) {
    static const int v = [] {
        const char* e = std::getenv("SCUBA_OOB_FAST_HEAVY_PASSES");
        return (e && *e) ? std::max(1, std::atoi(e)) : 0;
    }();
    return v > 0 ? (uint32_t)v : (fast_frontier() ? 32u : canonical);
}
// the symbolic prover's scratch at the start of a frontier region: the
// query's store plus one working set per lane
size_t sym_scratch_bytes() { return sizeof(sym::Store) + 32 * sizeof(sym::LaneWork); }

size_t frontier_region_bytes(uint32_t maxv, size_t tbytes) {
    size_t b = (size_t)FR_ECAP * 2 * maxv * tbytes + 2 * (size_t)FR_ECAP * tbytes + (size_t)FR_ECAP * 16 +
               (size_t)FR_LOGCAP * 16 + (size_t)FR_ECAP * 4 * 2 + (size_t)FR_ECAP * 16 + (size_t)FR_UCAP * 4 +
               (size_t)FR_ECAP * 4 + (size_t)FR_LOGCAP * 8;
    return (b + 255) & ~(size_t)255;
}

constexpr size_t DEVICE_STACK_BYTES = 4096;
constexpr uint64_t SLAB_BUDGET = 12ull << 30;  // per job, before the slabs are pooled

std::string ensure_stream(DevicePool* P, int dev) {
    CK(cudaSetDevice(phys_dev(dev)));
    if (!P->stream) {
        CK(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
        CK(cudaEventCreate(&P->ev0));
        CK(cudaEventCreate(&P->ev1));
        CK(cudaEventCreateWithFlags(&P->evr, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P->evraw, cudaEventDisableTiming));
        CK(cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, phys_dev(dev)));
        // per-thread stack: the deepest kernels (root phase, certificate
        // check, 256-bit solve) need up to ~2.2 KB; the default is 1 KB
        size_t stack = 0;
        CK(cudaDeviceGetLimit(&stack, cudaLimitStackSize));
        if (stack < DEVICE_STACK_BYTES) CK(cudaDeviceSetLimit(cudaLimitStackSize, DEVICE_STACK_BYTES));
    }
    return "";
}

std::string stage(const RunCtx& rc, DevJob& j, DevicePool* P, uint32_t depth_cap, uint32_t trail_cap,
                  bool heavy = true) {
    if (!j.upload_err.empty()) return j.upload_err;
    {
        std::string e = ensure_stream(P, j.dev);
        if (!e.empty()) return e;
    }
    const uint32_t n = (uint32_t)j.qs.size();
    const size_t tbytes = tbytes_of(j.wide);
    j.g = make_geom(j.maxv, j.maxcode, j.maxlit, depth_cap, trail_cap, j.maxcsize, j.maxdepth, tbytes);
    // run-time compiled classes (int64 solve jobs)
    j.jit_cls.clear();
    j.jit_fn.clear();
    j.jit_blocks.clear();
    j.jit_args.clear();
    j.jit_queries = 0;
    j.cls_interp = j.cls;
    // compiled classes: the x32 job and the int64 job (queries the root phase
    // could not move to x32 -- long root propagations -- stay there)
    // SCUBA_OOB_JIT128=1: int128-job classes compiled too (parity-exact; A/B on
    // B200 neutral on C3/C4/C5s while adding ~10 s of NVRTC per class on a
    // cold cache -- off)
    static const bool jit128 = [] {
        const char* e = std::getenv("SCUBA_OOB_JIT128");
        return e && *e == '1';
    }();
    if ((j.wide == 0 || j.wide == W_X32 || (j.wide == 1 && jit128)) && rc.mode == MODE_SOLVE &&
        !(rc.opt.flags & OOB_F_NO_JIT)) {
        const std::vector<Compiled>& comp = *rc.comp;
        std::vector<JitClass> want;
        // launch order = start order on the shared streams: class id, or
        // (SCUBA_OOB_JIT_ORDER=1) the classes with the most estimated work
        // (queries x domain bits) first -- A/B on B200: C3/C4 equal, C5s 10%
        // slower, so off
        static const bool by_work = [] {
            const char* e = std::getenv("SCUBA_OOB_JIT_ORDER");
            return e && *e == '1';
        }();
        std::vector<uint32_t> corder(j.n_classes);
        for (uint32_t c = 0; c < j.n_classes; c++) corder[c] = c;
        if (by_work) {
            std::vector<double> work(j.n_classes, 0.0);
            for (uint32_t c = 0; c < j.n_classes; c++)
                for (uint32_t i = j.cls[c].q_begin; i < j.cls[c].q_end; i++) work[c] += 1.0 + comp[j.qs[i]].cost;
            std::stable_sort(corder.begin(), corder.end(), [&](uint32_t a, uint32_t b) { return work[a] > work[b]; });
        }
        for (uint32_t c : corder) {
            const ClassDesc& cd = j.cls[c];
            const uint64_t size = cd.q_end - cd.q_begin;
            const Compiled& rep = comp[j.qs[cd.q_begin]];
            const uint64_t min_q = rc.opt.jit_min > 0 ? (uint64_t)rc.opt.jit_min : jit_min();
            if (size < min_q || rep.ncon > 128 || rep.nv > JIT_MAX_NV || rep.nlit > JIT_MAX_LIT ||
                rep.ncode > JIT_MAX_CODE)
                continue;
            j.jit_cls.push_back(c);
            want.push_back(JitClass{j.code.data() + cd.code_off, rep.nv, rep.ncon, rep.ncode, rep.nlit,
                                    j.wide == W_X32 ? 32 : (j.wide == 1 ? 128 : 64)});
        }
        if (!want.empty()) {
            std::vector<int> regs;
            std::string e = jit_prepare(want, j.jit_fn, regs, &j.jit_ms);
            if (!e.empty()) {  // no NVRTC / compile failure: the interpreter decides these classes
                if (trace_on()) std::fprintf(stderr, "[oob] run-time compile unavailable: %s\n", e.c_str());
                j.jit_cls.clear();
                j.jit_fn.clear();
            }
            for (size_t i = 0; i < j.jit_cls.size(); i++) {
                ClassDesc& cd = j.cls_interp[j.jit_cls[i]];
                j.jit_queries += cd.q_end - cd.q_begin;
                cd.q_end = cd.q_begin;  // the interpreting kernel sees the class drained
            }
        }
    }
    int per_sm = BLOCKS_PER_SM;
    CK(kernel_occupancy(j.wide, rc.mode, (size_t)j.g.smem_per_warp * WARPS_PER_BLOCK, &per_sm));
    per_sm = std::max(1, per_sm);
    const uint32_t warps_needed = (uint32_t)((n - j.jit_queries + 31) / 32);
    // the wide-regime solve kernels run next to the int64 one and hold their
    // blocks while their long searches last: one block per SM at most, so
    // they can never keep the int64 kernel (most of the work) off the SMs
    const uint32_t cap_blocks = (j.wide && rc.mode == MODE_SOLVE) ? (uint32_t)P->sms : (uint32_t)(P->sms * per_sm);
    j.blocks = std::max(1u, std::min<uint32_t>((warps_needed + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, cap_blocks));
    uint32_t n_warps = j.blocks * WARPS_PER_BLOCK;
    assign_warps(j, j.cls_interp, n_warps);
    for (size_t i = 0; i < j.jit_cls.size(); i++) {
        const ClassDesc& cd = j.cls[j.jit_cls[i]];
        const uint32_t jw = jit_warps();
        // resident blocks of a compiled class kernel: computed once per loaded
        // function (the block shape and shared memory never change)
        static std::mutex occ_mu;
        static std::unordered_map<const void*, int> occ_of;
        int occ = 0;
        {
            std::lock_guard<std::mutex> lk(occ_mu);
            auto it = occ_of.find(j.jit_fn[i]);
            if (it != occ_of.end()) occ = it->second;
        }
        if (!occ) {
            if (jit_smem())
                grow_smem_limit(j.jit_fn[i], jit_smem());
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, j.jit_fn[i], jw * 32, jit_smem()) != cudaSuccess) {
                cudaGetLastError();
                occ = 4;
            }
            occ = std::max(1, occ);
            std::lock_guard<std::mutex> lk(occ_mu);
            occ_of[j.jit_fn[i]] = occ;
        }
        // warps: one per 32 queries of the class, times SCUBA_OOB_JIT_GRID_MULT
        // (extra blocks start as others finish and serve the class's heavy list;
        // measured on B200, median plan run: x1 -> x3 = C3 14.7 -> 13.0 ms,
        // C4 52.6 -> 37.4 ms, C5s 11.6 -> 7.9 ms; x6 and more lose again)
        static const uint32_t mult = [] {
            const char* e = std::getenv("SCUBA_OOB_JIT_GRID_MULT");
            return (uint32_t)std::max(1, (e && *e) ? std::atoi(e) : 3);
        }();
        // the int64 job's classes hold the queries the x32 probe could not take
        // (long root propagations, wide values): fewer queries, heavier each
        static const uint32_t mult64 = [] {
            const char* e = std::getenv("SCUBA_OOB_JIT_GRID_MULT64");
            return (uint32_t)std::max(1, (e && *e) ? std::atoi(e) : (int)mult);
        }();
        const uint32_t need = (j.wide == 0 ? mult64 : mult) * ((cd.q_end - cd.q_begin + 31) / 32);
        const uint32_t b = std::max(1u, std::min<uint32_t>((need + jw - 1) / jw, (uint32_t)(P->sms * occ)));
        j.jit_blocks.push_back(b);
        n_warps += b * jw;
    }
    // heavy-query hand-off (solve mode): threshold from the options; in fast
    // mode the frontier is where the symbolic prover meets heavy queries, so
    // it is always on, with its own (earlier) thresholds
    int64_t hn = rc.opt.heavy_nodes;
    const bool fast = rc.mode == MODE_SOLVE && (rc.opt.flags & OOB_F_FAST);
    uint32_t heavy_nodes = (rc.mode == MODE_SOLVE && heavy && hn >= 0) ? (hn ? (uint32_t)hn : HEAVY_NODES_DEFAULT) : 0;
    if (fast && heavy_nodes) heavy_nodes = hn > 0 ? (uint32_t)hn : fast_heavy_nodes();
    // wide jobs: a frontier-only tail launch with a full grid serves their
    // heavy list once the int64 kernel has freed the SMs
    const uint32_t own_warps = n_warps;  // slabs [0, own_warps): the interpreting kernel + class kernels
    j.tail_blocks = (j.wide && heavy_nodes) ? (uint32_t)(P->sms * per_sm) : 0u;
    n_warps += j.tail_blocks * WARPS_PER_BLOCK;
    j.fblocks = heavy_nodes ? (n_warps + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK : 0;
    // frontier scratch: a pool of regions shared by every launch of the job,
    // held per heavy query (phases.cuh claim_region) -- sized for the warps
    // that can be resident at once, not for every warp of every launch
    // (C3: 74 -> ~20 GB per plan)
    const uint32_t regions_cap = (uint32_t)P->sms * (j.wide == 1 || j.wide == 2 ? 8u : 32u);
    j.fr_regions = heavy_nodes ? std::max(1u, std::min(n_warps, regions_cap)) : 0u;
    // the root kernel walks every query of the job (JIT classes included), one
    // thread each: its grid follows n, not the interpreting kernel's share,
    // bounded by the per-warp slabs allocated below
    // per-warp slabs: one per warp of every launch, or (SCUBA_OOB_SLAB_POOL=1,
    // SOLVE) a pool shared by the job's launches, one slab held per running
    // warp (phases.cuh claim_slab; at most 64 warps per SM are resident, so no
    // warp ever waits for one)
    // SCUBA_OOB_SLAB_POOL=1: slabs from the job pool (saves ~2 GB per plan on
    // C3, measured equal to 5% slower than one slab per warp -- off)
    static const bool slab_pool = [] {
        const char* e = std::getenv("SCUBA_OOB_SLAB_POOL");
        return e && *e == '1';
    }();
    // large batches: one slab per warp of every launch would outgrow the
    // device (C4 at 1M queries: ~100 K warps x ~0.7 MB); from SLAB_BUDGET on,
    // the slabs come from the job pool (one per running warp)
    const uint64_t slab_bytes = (uint64_t)n_warps * (j.g.slab_T_words * tbytes + j.g.slab_u32_words * 4);
    const bool pooled = rc.mode == MODE_SOLVE && (slab_pool || slab_bytes > SLAB_BUDGET);
    j.slab_slots = pooled ? std::max(1u, std::min(n_warps, (uint32_t)P->sms * 64u)) : n_warps;
    j.root_blocks = std::max<uint32_t>(
        1u, std::min<uint64_t>((n + 32 * WARPS_PER_BLOCK - 1) / (32 * WARPS_PER_BLOCK), j.slab_slots / WARPS_PER_BLOCK));
    size_t fr_bytes = frontier_region_bytes(j.maxv, tbytes);
    if (fast && fast_frontier()) fr_bytes = std::max(fr_bytes, (sym_scratch_bytes() + 255) & ~(size_t)255);
    j.out_model_words = j.model_words * (rc.mode == MODE_PROPAGATE ? 4 : 2);
    CK(P->qdesc.ensure(j.qd.size() * sizeof(QDesc)));
    CK(P->code.ensure(j.code.size() * 4));
    CK(P->data.ensure(j.data_words * 8));
    CK(P->slabT.ensure((size_t)j.slab_slots * j.g.slab_T_words * tbytes));
    CK(P->slabU.ensure((size_t)j.slab_slots * j.g.slab_u32_words * 4));
    if (pooled) CK(P->slab_map.ensure(((size_t)j.slab_slots + 31) / 32 * 4));
    CK(P->next.ensure(16));
    CK(P->verdict.ensure(n));
    CK(P->err.ensure(n));
    CK(P->model.ensure(std::max<size_t>(j.out_model_words, 2) * 8));
    CK(P->nodes.ensure((size_t)n * 8));
    CK(P->passes.ensure((size_t)n * 8));
    CK(P->elapsed.ensure((size_t)n * 4));
    CK(P->classes.ensure(j.cls.size() * sizeof(ClassDesc)));
    CK(P->class_next.ensure(j.cls.size() * 4));
    CK(P->class_init.ensure(j.cls.size() * 4));
    CK(P->warp_class.ensure((size_t)n_warps * 4));
    CK(P->heavy_count.ensure(32 * (1 + j.jit_cls.size())));
    CK(P->heavy_list.ensure((size_t)n * 8));  // [0, n): per compiled class at its q range; [n, 2n): interpreter
    CK(P->heavy_t0.ensure((size_t)n * 8));
    if (j.fr_regions) {
        CK(P->fr_region.ensure((size_t)j.fr_regions * fr_bytes));
        CK(P->fr_map.ensure(((size_t)j.fr_regions + 31) / 32 * 4));
    }
    CK(P->resume.ensure((size_t)n * 4));
    CK(P->resume_init.ensure((size_t)n * 4));
    auto slot_buf = [&](int t) -> DevBuf& { return t == 0 ? P->slot64 : (t == 1 ? P->slot128 : P->slotx32); };
    for (int t = 0; t < 3; t++)
        if (!j.slot[t].empty()) CK(slot_buf(t).ensure(j.slot[t].size() * 4));
    cudaStream_t s = P->stream;
    CK(cudaMemcpyAsync(P->resume_init.p, j.resume_init.data(), (size_t)n * 4, cudaMemcpyHostToDevice, s));
    for (int t = 0; t < 3; t++)
        if (!j.slot[t].empty())
            CK(cudaMemcpyAsync(slot_buf(t).p, j.slot[t].data(), j.slot[t].size() * 4,
                               cudaMemcpyHostToDevice, s));
    CK(P->classes_interp.ensure(j.cls.size() * sizeof(ClassDesc)));
    {
        std::vector<uint32_t> init(j.cls.size());
        for (size_t c = 0; c < j.cls.size(); c++) init[c] = j.cls[c].q_begin;
        CK(cudaMemcpyAsync(P->classes.p, j.cls.data(), j.cls.size() * sizeof(ClassDesc), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(P->classes_interp.p, j.cls_interp.data(), j.cls.size() * sizeof(ClassDesc),
                           cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(P->class_init.p, init.data(), init.size() * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(P->warp_class.p, j.warp_class.data(), j.warp_class.size() * 4, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));  // host vectors above are temporaries
    }
    CK(cudaMemcpyAsync(P->qdesc.p, j.qd.data(), j.qd.size() * sizeof(QDesc), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(P->code.p, j.code.data(), j.code.size() * 4, cudaMemcpyHostToDevice, s));
    // the x32 job holds shadows only: their records are written on the device
    // (by the int64 root phase) before they are ever read -- nothing to upload
    if ((j.wide != W_X32 || rc.mode != MODE_SOLVE) && !j.data_uploaded && !j.dev_fill)
        CK(cudaMemcpyAsync(P->data.p, j.data.data(), j.data.size() * 8, cudaMemcpyHostToDevice, s));
    if (j.dev_fill && n > 0) {  // the records, written on the device from the call's raw values
        DevicePool* R = j.raw_pool;
        if (!R || !R->raw_vlo.p) return "device-side records: the raw values were not uploaded";
        CK(P->rawoff.ensure((size_t)n * 16));
        CK(cudaMemcpyAsync(P->rawoff.p, j.rawoff.data(), (size_t)n * 16, cudaMemcpyHostToDevice, s));
        if (R != P) CK(cudaStreamWaitEvent(s, R->evraw, 0));
        CK(launch_expand(j.wide, (const QDesc*)P->qdesc.p, n, P->rawoff.p, R->raw_vlo.p, R->raw_vhi.p, R->raw_l.p,
                         (const int32_t*)R->litsrc.p, (int64_t*)P->data.p, P->sms, s));
    }
    LaunchArgs& a = j.a;
    a = LaunchArgs{};
    a.qdesc = (const QDesc*)P->qdesc.p;
    a.code = (const uint32_t*)P->code.p;
    a.data = (const int64_t*)P->data.p;
    a.n = n;
    a.next = (uint32_t*)P->next.p;
    a.classes = (const ClassDesc*)P->classes_interp.p;
    a.n_classes = j.n_classes;
    a.class_next = (uint32_t*)P->class_next.p;
    a.warp_class = (const uint32_t*)P->warp_class.p;
    a.heavy_nodes = heavy_nodes;
    {
        static const uint32_t wus = [] {
            const char* e = std::getenv("SCUBA_OOB_FRONTIER_WAIT_US");
            return (uint32_t)((e && *e) ? std::atoi(e) : 20000);
        }();
        a.frontier_wait_us = wus;
    }
    {
        static const uint32_t hp = [] {
            const char* e = std::getenv("SCUBA_OOB_HEAVY_PASSES");
            return (uint32_t)((e && *e) ? std::atoi(e) : (int)HEAVY_PASSES_DEFAULT);
        }();
        a.heavy_passes = fast ? fast_heavy_passes(hp) : hp;
    }
    a.fast = (fast && fast_frontier()) ? 1u : 0u;
    a.handoff_gate = (fast && !fast_frontier() && handoff_gate_env()) ? 1u : 0u;
    a.fast_stats = nullptr;
    a.cert_classes = nullptr;
    a.certs = nullptr;
    a.cert_nclasses = (uint32_t)j.cls.size();
    a.cert_kmax = 0;
    if (fast && rc.certs && !rc.certs->empty() && j.wide != W_X32) {
        for (const ClassDesc& cd : j.cls)
            if (cd.cert != NO_CERT && cd.q_end > cd.q_begin)
                a.cert_kmax = std::max<uint32_t>(a.cert_kmax, (uint32_t)(*rc.certs)[cd.cert]);
        CK(P->certs.ensure(rc.certs->size() * 8));
        CK(cudaMemcpyAsync(P->certs.p, rc.certs->data(), rc.certs->size() * 8, cudaMemcpyHostToDevice, s));
        a.certs = (const uint64_t*)P->certs.p;
        a.cert_classes = (const ClassDesc*)P->classes.p;
    }
    // fast mode with OOB_F_CHAIN (or SCUBA_OOB_CHAIN=1): the int64 job's own
    // entries first meet the warp-per-query search with warp-parallel
    // propagation (chain.cuh); SCUBA_OOB_CHAIN_NODES / _ROUNDS: its budgets
    a.chain_n = 0;
    a.chain_frames = nullptr;
    // fast mode, K3: the int64 job's own entries with small declared boxes are
    // enumerated (chain.cuh oob_enum_kernel); SCUBA_OOB_ENUM_MAX points
    // (default 4096, 0 = off)
    a.enum_n = 0;
    a.enum_max = 0;
    {
        // frontier speculative-lane abort (frontier.cuh): on in fast mode (B200
        // A/B: C4 13.4 -> 11.4 ms, C3 and C5s within noise; canonical C4 +4%,
        // so off there); SCUBA_OOB_FRONTIER_ABORT=<factor> overrides both
        static const int fa = [] {
            const char* e = std::getenv("SCUBA_OOB_FRONTIER_ABORT");
            return (e && *e) ? std::max(0, std::atoi(e)) : -1;
        }();
        a.fr_abort = fa >= 0 ? (uint32_t)fa : (fast ? 2u : 0u);
        static const uint32_t fm = [] {
            const char* e = std::getenv("SCUBA_OOB_FRONTIER_ABORT_MIN");
            return (uint32_t)((e && *e) ? std::max(0, std::atoi(e)) : 16);
        }();
        a.fr_abort_min = fm;
    }
    if (fast && rc.mode == MODE_SOLVE && j.wide == 0 && enum_max_points() > 0) {
        uint32_t own = 0;
        while (own < n && !j.is_shadow[own]) ++own;
        a.enum_n = own;
        a.enum_max = enum_max_points();
    }
    if (fast && rc.mode == MODE_SOLVE && j.wide == 0 && ((rc.opt.flags & OOB_F_CHAIN) || chain_cfg().on)) {
        uint32_t own = 0;
        while (own < n && !j.is_shadow[own]) ++own;
        if (own > 0) {
            const size_t warps = (size_t)chain_blocks(P->sms) * CHAIN_WARPS;
            CK(P->chain.ensure(warps * CHAIN_FRAME_WORDS * 8));
            a.chain_n = own;
            a.chain_frames = (long long*)P->chain.p;
            a.chain_nodes = chain_cfg().nodes;
            a.chain_rounds = chain_cfg().rounds;
        }
    }
    a.heavy_count = (uint32_t*)P->heavy_count.p;
    a.heavy_next = (uint32_t*)P->heavy_count.p + 1;
    a.heavy_list = (uint32_t*)P->heavy_list.p + n;
    a.heavy_t0 = (uint64_t*)P->heavy_t0.p;
    a.fr_region = j.fr_regions ? P->fr_region.p : nullptr;
    a.fr_region_bytes = fr_bytes;
    a.fr_bitmap = j.fr_regions ? (uint32_t*)P->fr_map.p : nullptr;
    a.fr_nregions = j.fr_regions;
    a.slab_bitmap = pooled ? (uint32_t*)P->slab_map.p : nullptr;
    a.slab_nslots = j.slab_slots;
    // hand-offs at the root resume in the frontier (SCUBA_OOB_HANDOFF_RESUME=0:
    // they restart from the declared domains, as before)
    static const bool handoff_resume = [] {
        const char* e = std::getenv("SCUBA_OOB_HANDOFF_RESUME");
        return !(e && *e == '0');
    }();
    a.handoff = nullptr;
    if (rc.mode == MODE_SOLVE && heavy_nodes && handoff_resume) {
        CK(P->handoff.ensure(j.data_words * 8));
        a.handoff = (int64_t*)P->handoff.p;
    }
    a.fr_ecap = FR_ECAP;
    a.fr_ucap = FR_UCAP;
    a.fr_logcap = FR_LOGCAP;
    a.slab_T = P->slabT.p;
    a.slab_u32 = (uint32_t*)P->slabU.p;
    a.g = j.g;
    a.verdict = (int8_t*)P->verdict.p;
    a.err = (int8_t*)P->err.p;
    a.model = (int64_t*)P->model.p;
    a.nodes = (int64_t*)P->nodes.p;
    a.passes = (int64_t*)P->passes.p;
    a.elapsed = (float*)P->elapsed.p;
    double t = rc.opt.timeout_s;
    a.timeout_ns = (rc.mode == MODE_SOLVE && t > 0 && t < 1e9) ? (uint64_t)(t * 1e9) : 0;
    a.node_budget = rc.opt.node_budget;
    a.mode = rc.mode;
    a.resume = (uint32_t*)P->resume.p;
    a.stats = nullptr;
    if (trace_level() >= 2 && rc.mode == MODE_SOLVE) {
        CK(P->stats.ensure(128));
        CK(cudaMemsetAsync(P->stats.p, 0, 128, s));
        a.stats = (unsigned long long*)P->stats.p;
        if (fast) a.fast_stats = a.stats + 10;  // [10..14] (certificate kernel: [14])
    }
    a.timeline = nullptr;
    if (timeline_path() && rc.mode == MODE_SOLVE) {
        CK(P->timeline.ensure((size_t)n * 32));
        a.timeline = (uint64_t*)P->timeline.p;
    }
    if (j.tail_blocks) {
        j.tail_args = a;
        j.tail_args.frontier_only = 1;
        if (!a.slab_bitmap) {  // one slab per warp: the tail's warps follow the job's own
            j.tail_args.slab_T = (unsigned char*)P->slabT.p + (uint64_t)own_warps * j.g.slab_T_words * tbytes;
            j.tail_args.slab_u32 = (uint32_t*)P->slabU.p + (uint64_t)own_warps * j.g.slab_u32_words;
        }

    }
    // one launch per compiled class: its own class queue and heavy list (slabs
    // and frontier regions come from the job's pools)
    uint64_t warp_base = (uint64_t)j.blocks * WARPS_PER_BLOCK;  // one slab per warp: per-launch ranges
    for (size_t i = 0; i < j.jit_cls.size(); i++) {
        const uint32_t c = j.jit_cls[i];
        LaunchArgs b = a;
        if (!a.slab_bitmap) {
            b.slab_T = (unsigned char*)P->slabT.p + warp_base * j.g.slab_T_words * tbytes;
            b.slab_u32 = (uint32_t*)P->slabU.p + warp_base * j.g.slab_u32_words;
            warp_base += (uint64_t)j.jit_blocks[i] * jit_warps();
        }
        b.classes = (const ClassDesc*)P->classes.p + c;
        b.n_classes = 1;
        b.class_next = (uint32_t*)P->class_next.p + c;
        b.warp_class = nullptr;
        b.heavy_count = (uint32_t*)P->heavy_count.p + 8 * (1 + i);
        b.heavy_list = (uint32_t*)P->heavy_list.p + j.cls[c].q_begin;
        j.jit_args.push_back(b);
    }
    if (trace_on()) {
        auto mb = [](const DevBuf& b) { return (double)b.cap / (1 << 20); };
        std::fprintf(stderr,
                     "[oob] pool w%d: slabT %.0f slabU %.0f fr %.0f data %.0f model %.0f heavy %.0f MiB "
                     "(warps %u slots %u regions %u fr_bytes %zu)\n",
                     j.wide, mb(P->slabT), mb(P->slabU), mb(P->fr_region), mb(P->data), mb(P->model),
                     mb(P->heavy_list) + mb(P->heavy_t0), n_warps, j.slab_slots, j.fr_regions, fr_bytes);
    }
    j.staged = true;
    return "";
}

// ----- device groups: the regime jobs of one device ---------------------------
// job[w] holds the queries whose proven regime is w (0 int64, 1 int128, 2
// 256-bit).  In SOLVE mode job[0] also carries a shadow entry for every query
// of job[1] and job[2], and job[1] one for every query of job[2]: the root
// kernels of the wide jobs run first and hand demoted queries to their shadows
// (format.h), then the three lockstep kernels run concurrently on their own
// streams.
struct DevGroup {
    int dev = 0;
    DevJob job[NJOBS];
    DevicePool* pool[NJOBS] = {nullptr, nullptr, nullptr, nullptr};
    bool raw_uploaded = false;
};

// SOLVE: the call's raw domains / literals and the literal-source table go to
// the device once per group (into the int64 job's pool, on its stream); the
// jobs' record kernels wait for them (evraw)
std::string upload_raw(const RunCtx& rc, DevGroup& G) {
    if (!rc.raw || G.raw_uploaded) return "";
    DevicePool* R = G.pool[0];
    if (!R) return "device-side records: no pool for the raw values";
    std::string e = ensure_stream(R, G.dev);
    if (!e.empty()) return e;
    CK(R->raw_vlo.ensure(std::max<uint64_t>(rc.raw_nv, 1) * 8));
    CK(R->raw_vhi.ensure(std::max<uint64_t>(rc.raw_nv, 1) * 8));
    CK(R->raw_l.ensure(std::max<uint64_t>(rc.raw_nl, 1) * 8));
    CK(R->litsrc.ensure(std::max<size_t>(rc.litsrc->size(), 1) * 4));
    if (rc.raw_nv) {
        CK(cudaMemcpyAsync(R->raw_vlo.p, rc.raw_vlo, rc.raw_nv * 8, cudaMemcpyHostToDevice, R->stream));
        CK(cudaMemcpyAsync(R->raw_vhi.p, rc.raw_vhi, rc.raw_nv * 8, cudaMemcpyHostToDevice, R->stream));
    }
    if (rc.raw_nl) CK(cudaMemcpyAsync(R->raw_l.p, rc.raw_l, rc.raw_nl * 8, cudaMemcpyHostToDevice, R->stream));
    if (!rc.litsrc->empty())
        CK(cudaMemcpyAsync(R->litsrc.p, rc.litsrc->data(), rc.litsrc->size() * 4, cudaMemcpyHostToDevice, R->stream));
    CK(cudaEventRecord(R->evraw, R->stream));
    for (int w = 0; w < NJOBS; w++) G.job[w].raw_pool = R;
    G.raw_uploaded = true;
    return "";
}

// start the upload of a packed job's records at once (caller holds P->mu):
// the copy overlaps the packing of the next jobs instead of following it
std::string upload_data(DevJob& j, DevicePool* P) {
    if (j.dev_fill) return "";  // written on the device at staging (oob_expand_kernel)
    std::string e = ensure_stream(P, j.dev);
    if (!e.empty()) return e;
    CK(P->data.ensure(j.data.size() * 8));
    CK(cudaMemcpyAsync(P->data.p, j.data.data(), j.data.size() * 8, cudaMemcpyHostToDevice, P->stream));
    j.data_uploaded = true;
    return "";
}

// shadows + pack + demotion slots of a group (before staging)
void pack_group(const RunCtx& rc, DevGroup& G, bool upload = false) {
    for (int w = 0; w < NJOBS; w++) {
        G.job[w].dev = G.dev;
        G.job[w].wide = w;
        G.job[w].shadows.clear();
        for (auto& sl : G.job[w].slot) sl.clear();
    }
    G.job[W_X32].qs.clear();  // x32 entries are always shadows
    // the original (own-regime) query lists, before pack() reorders them
    std::vector<int64_t> own[3];
    for (int w = 0; w < 3; w++) own[w] = G.job[w].qs;
    if (demote_on(rc)) {
        for (int w = 1; w < 3; w++)
            for (int t = 0; t < w; t++)
                G.job[t].shadows.insert(G.job[t].shadows.end(), own[w].begin(), own[w].end());
    }
    if (x32_on(rc))
        for (int w = 0; w < 3; w++)
            G.job[W_X32].shadows.insert(G.job[W_X32].shadows.end(), own[w].begin(), own[w].end());
    static const char* pk_names[NJOBS] = {"pack.int64", "pack.int128", "pack.i256", "pack.x32"};
    for (int w = 0; w < NJOBS; w++) {
        G.job[w].data_uploaded = false;
        G.job[w].upload_err.clear();
    }
    if (upload) {  // the raw values travel while the jobs are packed
        const std::string e = upload_raw(rc, G);
        if (!e.empty())
            for (int w = 0; w < NJOBS; w++) G.job[w].upload_err = e;
    }
    auto has = [&](int w) { return !G.job[w].qs.empty() || !G.job[w].shadows.empty(); };
    // the x32 job (shadows only: descriptors, no record data) is packed on a
    // thread of its own, its per-entry loop inline, while this thread packs
    // the other jobs with the host pool
    std::thread x32_thread;
    if (has(W_X32) && host_threads() > 2)
        x32_thread = std::thread([&]() { pack(rc, G.job[W_X32], true); });
    else if (has(W_X32)) {
        Phase ph(pk_names[W_X32]);
        pack(rc, G.job[W_X32]);
    }
    for (int w = 0; w < 3; w++) {
        if (!has(w)) continue;
        Phase ph(pk_names[w]);
        pack(rc, G.job[w]);
        if (upload && G.pool[w]) G.job[w].upload_err = upload_data(G.job[w], G.pool[w]);
    }
    if (x32_thread.joinable()) {
        Phase ph("pack.x32.join");
        x32_thread.join();
    }
    if (upload && G.pool[W_X32] && has(W_X32) && rc.mode != MODE_SOLVE)
        G.job[W_X32].upload_err = upload_data(G.job[W_X32], G.pool[W_X32]);
    Phase ph_slots("pack.slots");
    if (!demote_on(rc)) return;
    // demotion slots: target t (0 int64, 1 int128, 2 x32 = job 3) of the jobs that hand down to it
    for (int t = 0; t < 3; t++) {
        const DevJob& T = G.job[t == 2 ? W_X32 : t];
        if (T.shadows.empty()) continue;
        static thread_local std::vector<uint32_t> at;  // query id -> shadow index in T
        if (at.size() < (size_t)rc.b->n_queries) at.resize((size_t)rc.b->n_queries);
        uint32_t* atp = at.data();
        parallel_for(T.qs.size(), 8192, [&](size_t lo, size_t hi) {
            for (size_t i = lo; i < hi; i++)
                if (T.is_shadow[i]) atp[T.qs[i]] = (uint32_t)i;
        });
        for (int w = 0; w < 3; w++) {
            if (t == 2 ? w != 0 : w <= t) continue;  // x32: from the int64 job; else from the wider jobs
            DevJob& W = G.job[w];
            if (W.qs.empty()) continue;
            W.slot[t].resize(W.qs.size());
            uint32_t* sl = W.slot[t].data();
            parallel_for(W.qs.size(), 8192, [&](size_t lo, size_t hi) {
                for (size_t i = lo; i < hi; i++) sl[i] = atp[W.qs[i]];
            });
        }
    }
}

// a job is present when it has own queries or shadows
inline bool present(const DevJob& j) { return !j.qs.empty(); }

std::string stage_group(const RunCtx& rc, DevGroup& G, uint32_t depth_cap, uint32_t trail_cap, bool heavy) {
    {
        const std::string e = upload_raw(rc, G);  // (once per group)
        if (!e.empty()) return e;
    }
    for (int w = 0; w < NJOBS; w++) {
        if (!present(G.job[w])) continue;
        std::string e = stage(rc, G.job[w], G.pool[w], depth_cap, trail_cap, heavy);
        if (!e.empty()) return e;
    }
    // demotion targets: t = 0 int64 job, 1 int128 job, 2 x32 job (index 3)
    for (int w = 0; w < 3; w++) {
        if (!present(G.job[w])) continue;
        LaunchArgs& a = G.job[w].a;
        for (int t = 0; t < 3; t++) {
            a.dem[t] = DemoteTarget{};
            if (G.job[w].slot[t].empty()) continue;
            DevicePool* T = G.pool[t == 2 ? W_X32 : t];
            DevicePool* S = G.pool[w];
            a.dem[t].qdesc = (const QDesc*)T->qdesc.p;
            a.dem[t].data = (int64_t*)T->data.p;
            a.dem[t].resume = (uint32_t*)T->resume.p;
            a.dem[t].t0 = (uint64_t*)T->heavy_t0.p;
            a.dem[t].slot = (const uint32_t*)(t == 0 ? S->slot64.p : (t == 1 ? S->slot128.p : S->slotx32.p));
        }
    }
    return "";
}

// one run of a group: resets, root kernels, then the lockstep kernels
std::string launch_group(const RunCtx& rc, DevGroup& G) {
    CK(cudaSetDevice(phys_dev(G.dev)));
    int first = -1;
    for (int w = 0; w < NJOBS; w++)
        if (present(G.job[w])) { first = w; break; }
    if (first < 0) return "";
    cudaStream_t s0 = G.pool[first]->stream;
    // every per-run reset on the first stream, so that the root kernels may
    // write into the other jobs' buffers once it is done
    for (int w = first; w < NJOBS; w++) {
        if (!present(G.job[w])) continue;
        DevicePool* P = G.pool[w];
        const DevJob& j = G.job[w];
        const size_t n = j.qs.size();
        CK(cudaMemsetAsync(P->next.p, 0, 4, s0));  // work cursor (aux kernel / opt-in chain search)
        CK(cudaMemcpyAsync(P->class_next.p, P->class_init.p, j.cls.size() * 4, cudaMemcpyDeviceToDevice, s0));
        CK(cudaMemsetAsync(P->heavy_count.p, 0, 32 * (1 + j.jit_cls.size()), s0));
        if (rc.mode == MODE_SOLVE) CK(cudaMemsetAsync(P->heavy_list.p, 0, n * 8, s0));
        if (j.fr_regions) CK(cudaMemsetAsync(P->fr_map.p, 0, ((size_t)j.fr_regions + 31) / 32 * 4, s0));
        if (j.a.slab_bitmap) CK(cudaMemsetAsync(P->slab_map.p, 0, ((size_t)j.slab_slots + 31) / 32 * 4, s0));
        if (j.a.timeline) CK(cudaMemsetAsync(j.a.timeline, 0, n * 32, s0));
        CK(cudaMemsetAsync(P->verdict.p, 0xFF, n, s0));
        CK(cudaMemcpyAsync(P->resume.p, P->resume_init.p, n * 4, cudaMemcpyDeviceToDevice, s0));
    }
    CK(cudaEventRecord(G.pool[first]->ev0, s0));
    for (int w = first + 1; w < NJOBS; w++)
        if (present(G.job[w])) {
            CK(cudaStreamWaitEvent(G.pool[w]->stream, G.pool[first]->ev0, 0));
            CK(cudaEventRecord(G.pool[w]->ev0, G.pool[w]->stream));
        }
    if (rc.mode == MODE_SOLVE) {
        // fast mode: class certificates first (refuted entries are never
        // searched: RES_SKIP)
        for (int w = 0; w < 3; w++) {
            if (!present(G.job[w]) || !G.job[w].a.certs) continue;
            const DevJob& j = G.job[w];
            if (!j.a.cert_kmax) continue;
            CK(launch_cert(j.a, w, 0, 1, G.pool[w]->sms, G.pool[w]->stream));
            if (j.a.cert_kmax > 1) CK(launch_cert(j.a, w, 1, j.a.cert_kmax, G.pool[w]->sms, G.pool[w]->stream));
        }
        // fast mode: the int64 job's small boxes (K3), then (opt-in) its
        // open own entries, warp per query
        if (present(G.job[0]) && G.job[0].a.enum_n)
            CK(launch_enum(G.job[0].a, chain_blocks(G.pool[0]->sms), G.pool[0]->stream));
        if (present(G.job[0]) && G.job[0].a.chain_n)
            CK(launch_chain(G.job[0].a, chain_blocks(G.pool[0]->sms), G.pool[0]->stream));
        // root phases, widest first: 256-bit -> int128 -> int64 -> x32
        for (int w = 2; w >= 0; w--) {
            if (!present(G.job[w])) continue;
            DevJob& j = G.job[w];
            if (j.slot[0].empty() && j.slot[1].empty() && j.slot[2].empty()) continue;
            CK(launch_root(j.a, w, (int)j.root_blocks, G.pool[w]->stream));
            CK(cudaEventRecord(G.pool[w]->evr, G.pool[w]->stream));
            for (int t = 0; t < 3; t++) {
                const int tj = t == 2 ? W_X32 : t;
                if (present(G.job[tj]) && !j.slot[t].empty())
                    CK(cudaStreamWaitEvent(G.pool[tj]->stream, G.pool[w]->evr, 0));
            }
        }
    }
    // launch order = block dispatch priority: the int64 job first (its few
    // remaining queries are the long root propagations), then x32 (the bulk),
    // then the wide jobs
    static const bool x32_first = [] {
        const char* e = std::getenv("SCUBA_OOB_X32_FIRST");
        return e && *e == '1';
    }();
    static const int order_a[NJOBS] = {0, W_X32, 1, 2}, order_b[NJOBS] = {W_X32, 0, 1, 2};
    const int* order = x32_first ? order_b : order_a;
    for (int oi = 0; oi < NJOBS; oi++) {
        const int w = order[oi];
        if (!present(G.job[w])) continue;
        DevJob& j = G.job[w];
        DevicePool* P = G.pool[w];
        cudaStream_t s = P->stream;
        // compiled classes first (the big ones), each on its own stream after
        // everything queued so far on the job's stream (resets, root kernels)
        if (!j.jit_cls.empty()) {
            static const size_t kmax = [] {
                const char* e = std::getenv("SCUBA_OOB_JIT_STREAMS");
                return (size_t)((e && *e) ? std::max(1, std::atoi(e)) : 16);
            }();
            const size_t nxs = std::min(kmax, j.jit_cls.size());
            while (P->xs.size() < nxs) {
                cudaStream_t xs;
                cudaEvent_t xe;
                CK(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
                CK(cudaEventCreateWithFlags(&xe, cudaEventDisableTiming));
                P->xs.push_back(xs);
                P->xev.push_back(xe);
            }
            CK(cudaEventRecord(P->evr, s));
            for (size_t x = 0; x < nxs; x++) CK(cudaStreamWaitEvent(P->xs[x], P->evr, 0));
            for (size_t i = 0; i < j.jit_cls.size(); i++) {
                void* args[] = {&j.jit_args[i]};
                CK(cudaLaunchKernel(j.jit_fn[i], dim3(j.jit_blocks[i]), dim3(jit_warps() * 32), args, jit_smem(),
                                    P->xs[i % nxs]));
            }
            for (size_t x = 0; x < nxs; x++) CK(cudaEventRecord(P->xev[x], P->xs[x]));
        }
        CK(launch_solve(j.a, w, (int)j.blocks, (int)j.fblocks, s));
        for (size_t x = 0; x < std::min(P->xs.size(), j.jit_cls.size()); x++) CK(cudaStreamWaitEvent(s, P->xev[x], 0));
        if (w != 0) CK(cudaEventRecord(P->ev1, s));
    }
    if (present(G.job[0])) {  // the wide jobs' frontier tails once the int64 and x32 work is done
        cudaStream_t s = G.pool[0]->stream;
        if (rc.mode == MODE_SOLVE) {
            if (present(G.job[W_X32])) CK(cudaStreamWaitEvent(s, G.pool[W_X32]->ev1, 0));
            for (int t = 1; t < 3; t++)
                if (present(G.job[t]) && G.job[t].tail_blocks)
                    CK(launch_solve(G.job[t].tail_args, t, (int)G.job[t].tail_blocks, 0, s));
        }
        CK(cudaEventRecord(G.pool[0]->ev1, s));
    }
    return "";
}

// device time of the last run of a group: first start event to the last end
std::string group_ms(DevGroup& G, float* ms) {
    CK(cudaSetDevice(phys_dev(G.dev)));
    *ms = 0;
    int first = -1;
    for (int w = 0; w < NJOBS; w++)
        if (present(G.job[w])) {
            if (first < 0) first = w;
            CK(cudaEventSynchronize(G.pool[w]->ev1));
            float t = 0;
            CK(cudaEventElapsedTime(&t, G.pool[first]->ev0, G.pool[w]->ev1));
            G.job[w].last_ms = t;
            *ms = std::max(*ms, t);
        }
    return "";
}

// D2H + scatter into the caller arrays; capacity overflows go to `retry`
// (by the query's own regime).  Entries a job does not own (shadows that were
// not resumed, queries that were demoted) carry VERDICT_NONE.
std::string fetch(RunCtx& rc, DevJob& j, DevicePool* P, std::vector<int64_t> retry[3]) {
    CK(cudaSetDevice(phys_dev(j.dev)));
    const uint32_t n = (uint32_t)j.qs.size();
    cudaStream_t s = P->stream;
    HostArr<int8_t> verdict, err;
    HostArr<int64_t> nodes, passes, mw;
    HostArr<float> el;
    verdict.alloc(n);
    err.alloc(n);
    nodes.alloc(n);
    passes.alloc(n);
    el.alloc(n);
    mw.alloc(std::max<size_t>(j.out_model_words, 2));
    // SOLVE: only Sat entries carry a model -- pack them on the device and
    // copy those (C3: ~15% of the entries) instead of the whole model buffer
    const bool packed = rc.mode == MODE_SOLVE && j.out_model_words;
    HostArr<uint32_t> satoff;
    unsigned long long nsat = 0;
    if (packed) {
        CK(P->satcnt.ensure(8));
        CK(P->satoff.ensure((size_t)n * 4));
        CK(P->compact.ensure(j.out_model_words * 8));
        CK(cudaMemsetAsync(P->satcnt.p, 0, 8, s));
        CK(launch_gather_sat((const int8_t*)P->verdict.p, (const QDesc*)P->qdesc.p, (const int64_t*)P->model.p, n,
                             (unsigned long long*)P->satcnt.p, (uint32_t*)P->satoff.p, (int64_t*)P->compact.p,
                             P->sms, s));
        satoff.alloc(n);
        CK(cudaMemcpyAsync(satoff.data(), P->satoff.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&nsat, P->satcnt.p, 8, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaMemcpyAsync(verdict.data(), P->verdict.p, n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(err.data(), P->err.p, n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(nodes.data(), P->nodes.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(passes.data(), P->passes.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(el.data(), P->elapsed.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    if (j.out_model_words && !packed)
        CK(cudaMemcpyAsync(mw.data(), P->model.p, j.out_model_words * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (packed && nsat * 2 > j.out_model_words)
        return "packed Sat models exceed the model buffer (" + std::to_string(nsat) + " vars, " +
               std::to_string(j.out_model_words) + " words, job " + std::to_string(j.wide) + ", " +
               std::to_string(n) + " entries)";
    if (packed && nsat) {
        CK(cudaMemcpyAsync(mw.data(), P->compact.p, (size_t)nsat * 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    j.last_sat_vars = packed ? (int64_t)nsat : -1;
    if (j.a.timeline) {  // records: q, wide, shadow, verdict, nodes, passes, 4 timestamps (int64 each)
        std::vector<uint64_t> tl((size_t)n * 4);
        CK(cudaMemcpy(tl.data(), j.a.timeline, (size_t)n * 32, cudaMemcpyDeviceToHost));
        static std::mutex mu;
        std::lock_guard<std::mutex> lk(mu);
        if (FILE* f = std::fopen(timeline_path(), "ab")) {
            for (uint32_t i = 0; i < n; i++) {
                int64_t rec[10] = {j.qs[i], j.wide, j.is_shadow[i], verdict[i], nodes[i], passes[i],
                                   (int64_t)tl[4 * i], (int64_t)tl[4 * i + 1], (int64_t)tl[4 * i + 2],
                                   (int64_t)tl[4 * i + 3]};
                std::fwrite(rec, sizeof rec, 1, f);
            }
            std::fclose(f);
        }
    }
    if (j.a.stats) {
        unsigned long long st[16];
        CK(cudaMemcpy(st, j.a.stats, 128, cudaMemcpyDeviceToHost));
        std::fprintf(stderr,
                     "[oob] job w%d: frontier rounds %llu units %llu lane-passes %llu / slots %llu (%.1f%%); "
                     "lockstep lane-passes %llu / slots %llu (%.1f%%)\n",
                     j.wide, st[2], st[3], st[1], st[0], st[0] ? 100.0 * st[1] / st[0] : 0.0, st[5], st[4],
                     st[4] ? 100.0 * st[5] / st[4] : 0.0);
        std::fprintf(stderr, "[oob] job w%d: frontier Sat passes expanded %llu / reference %llu; Unsat %llu / %llu\n",
                     j.wide, st[6], st[7], st[8], st[9]);
        if (j.a.fast || j.a.certs)
            std::fprintf(stderr,
                         "[oob] job w%d: fast mode: %llu entries refuted by their class certificate; %llu heavy "
                         "queries met the frontier prover, %llu refuted; cycles per query: prepare %.0f search %.0f\n",
                         j.wide, st[14], st[10], st[11], st[10] ? (double)st[12] / st[10] : 0.0,
                         st[10] ? (double)st[13] / st[10] : 0.0);
    }
    const std::vector<Compiled>& comp = *rc.comp;
    const oob_batch* b = rc.b;
    std::vector<uint8_t> is_retry(n, 0);
    parallel_for(n, 2048, [&](size_t lo, size_t hi) {
        for (size_t i = lo; i < hi; i++) {
            if (verdict[i] == VERDICT_NONE) continue;
            int64_t q = j.qs[i];
            if (err[i] == ERR_DEPTH || err[i] == ERR_TRAIL) {
                is_retry[i] = 1;
                continue;
            }
            (*rc.errs)[q] = err[i];
            rc.verdict[q] = verdict[i];
            if (rc.nodes) rc.nodes[q] = nodes[i];
            if (rc.passes) rc.passes[q] = passes[i];
            if (rc.elapsed) rc.elapsed[q] = el[i];
            int64_t vb = b->var_begin[q];
            uint32_t nv = comp[q].nv;
            uint64_t m0 = j.mo[i];
            if (rc.mode == MODE_SOLVE && verdict[i] == VERDICT_SAT && rc.model) {
                if (packed) m0 = satoff[i];
                for (uint32_t v = 0; v < nv; v++) {
                    rc.model[vb + v].lo = (uint64_t)mw[2 * (m0 + v)];
                    rc.model[vb + v].hi = mw[2 * (m0 + v) + 1];
                }
            } else if (rc.mode == MODE_PROPAGATE && rc.model) {
                for (uint32_t v = 0; v < nv; v++) {
                    rc.model[2 * (vb + v)].lo = (uint64_t)mw[4 * (m0 + v)];
                    rc.model[2 * (vb + v)].hi = mw[4 * (m0 + v) + 1];
                    rc.model[2 * (vb + v) + 1].lo = (uint64_t)mw[4 * (m0 + v) + 2];
                    rc.model[2 * (vb + v) + 1].hi = mw[4 * (m0 + v) + 3];
                }
            }
        }
    });
    for (uint32_t i = 0; i < n; i++)
        if (is_retry[i]) retry[comp[j.qs[i]].regime - R_W64].push_back(j.qs[i]);
    return "";
}

std::string fetch_group(RunCtx& rc, DevGroup& G, std::vector<int64_t> retry[3]) {
    for (int w = 0; w < NJOBS; w++) {
        if (!present(G.job[w])) continue;
        std::string e = fetch(rc, G.job[w], G.pool[w], retry);
        if (!e.empty()) return e;
    }
    return "";
}

// full run of one device's queries on the shared pools, with capacity retries
std::string run_group(RunCtx& rc, int dev, std::vector<int64_t> qs[3]) {
    uint32_t depth_cap = DEPTH_CAP0, trail_cap = TRAIL_CAP0;
    DevicePool* pools[NJOBS] = {pool_for(dev, 0), pool_for(dev, 1), pool_for(dev, 2), pool_for(dev, 3)};
    std::vector<int64_t> cur[3] = {qs[0], qs[1], qs[2]};
    for (int round = 0; round < 5; round++) {
        if (cur[0].empty() && cur[1].empty() && cur[2].empty()) return "";
        DevGroup G;
        G.dev = dev;
        // per-entry host vectors recycled per thread (see drive)
        struct JobScratch {
            std::vector<int64_t> qs, shadows;
            std::vector<uint8_t> is_shadow;
            std::vector<uint32_t> resume_init, slot[3];
            std::vector<uint64_t> mo;
        };
        static thread_local JobScratch tl_js[NJOBS];
        auto swap_scratch = [&]() {
            for (int w = 0; w < NJOBS; w++) {
                DevJob& j = G.job[w];
                JobScratch& x = tl_js[w];
                j.qs.swap(x.qs);
                j.shadows.swap(x.shadows);
                j.is_shadow.swap(x.is_shadow);
                j.resume_init.swap(x.resume_init);
                j.mo.swap(x.mo);
                for (int t = 0; t < 3; t++) j.slot[t].swap(x.slot[t]);
            }
        };
        swap_scratch();
        for (int w = 0; w < NJOBS; w++) {
            if (w < 3) G.job[w].qs.assign(cur[w].begin(), cur[w].end());
            else G.job[w].qs.clear();
            G.pool[w] = pools[w];
        }
        struct SwapBack {
            std::function<void()> f;
            ~SwapBack() { f(); }
        } swap_back{swap_scratch};
        std::vector<int64_t> retry[3];
        {
            std::lock_guard<std::mutex> l0(pools[0]->mu), l1(pools[1]->mu), l2(pools[2]->mu), l3(pools[3]->mu);
            {
                Phase ph("pack");
                pack_group(rc, G, true);  // each job's upload overlaps the next job's packing
            }
            if (gate_point() == GATE_PACK) gate_release();
            std::string e;
            {
                Phase ph("stage");
                e = stage_group(rc, G, depth_cap, trail_cap, round == 0);
                for (int w = 0; w < NJOBS && e.empty(); w++)
                    if (present(G.job[w]) && cudaStreamSynchronize(G.pool[w]->stream) != cudaSuccess)
                        e = "stage sync failed";
            }
            if (e.empty()) {
                Phase ph("kernels");
                e = launch_group(rc, G);
                gate_release();  // the next chunk's host work overlaps these kernels
                float ms = 0;
                if (e.empty()) e = group_ms(G, &ms);
            }
            if (e.empty()) {
                Phase ph("fetch");
                e = fetch_group(rc, G, retry);
            }
            if (!e.empty()) return e;
        }
        if (trace_on())
            std::fprintf(stderr, "[oob] round %d dev %d: retry %zu/%zu/%zu (jit classes %zu)\n", round, dev,
                         retry[0].size(), retry[1].size(), retry[2].size(), G.job[0].jit_cls.size());
        for (int w = 0; w < 3; w++) cur[w].swap(retry[w]);
        depth_cap *= 4;
        trail_cap *= 8;
    }
    for (int w = 0; w < 3; w++)
        for (int64_t q : cur[w]) {  // still out of scratch after the last retry
            rc.verdict[q] = OOB_ERROR;
            (*rc.errs)[q] = ERR_DEPTH;
        }
    return "";
}

struct DevWork {
    int dev = 0;
    std::vector<int64_t> qs[3];
};

std::string run_all(RunCtx& rc, std::vector<DevWork>& work) {
    std::vector<std::string> errs(work.size());
    if (work.size() == 1) {  // one device: stay on the caller's thread (pipeline slot / gate)
        errs[0] = run_group(rc, work[0].dev, work[0].qs);
    } else {
        const int slot = tl_pool_slot;
        std::vector<std::thread> th;
        for (size_t k = 0; k < work.size(); k++)
            th.emplace_back([&, k, slot]() {
                tl_pool_slot = slot;
                errs[k] = run_group(rc, work[k].dev, work[k].qs);
            });
        for (auto& t : th) t.join();
    }
    for (auto& e : errs)
        if (!e.empty()) return e;
    return "";
}

int visible_devices() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Device-bound queries by regime, grouped by structure class.  A class is a
// structure word for word (queries compiled on different threads hold
// different Structure objects of one class); classes are numbered densely in
// order of first appearance (lowest query index), and each regime's list is
// class-major with ascending query indices inside a class.  The class table
// is built from the call's pins (a few entries per structure); the per-query
// passes run in parallel over query chunks.
struct Classes {
    std::vector<int64_t> reg[3];
    std::vector<uint32_t> start[3];  // class c of regime w: reg[w][start[w][c] .. start[w][c + 1])
    uint32_t ncls = 0;
    size_t members(uint32_t c) const {
        size_t m = 0;
        for (int w = 0; w < 3; w++) m += start[w][c + 1] - start[w][c];
        return m;
    }
    int64_t member(uint32_t c, size_t i) const {  // regime-major, ascending query index
        for (int w = 0; w < 3; w++) {
            const size_t k = start[w][c + 1] - start[w][c];
            if (i < k) return reg[w][start[w][c] + i];
            i -= k;
        }
        return -1;
    }
};
inline bool device_regime(const Compiled& c) { return c.regime >= R_W64 && c.regime < R_W64 + 3; }

// other(q, comp[q]) is called (concurrently) for every query that is not
// device-bound; qcls[q] = class of a device query, 0 otherwise
template <typename Other>
void classify(std::vector<Compiled>& comp, int64_t n, const std::vector<std::shared_ptr<const Structure>>& pins,
              std::vector<uint32_t>& qcls, Classes& K, Other other, std::vector<int32_t>* litsrc = nullptr,
              std::vector<uint32_t>* pin_cls = nullptr) {
    // distinct structure objects -> canonical class (word-for-word equality)
    size_t TB = 1024;
    while (TB < 2 * pins.size()) TB *= 2;
    std::vector<const Structure*> slot_ptr(TB, nullptr);
    std::vector<uint32_t> slot_canon(TB, 0), slot_lsrc(TB, 0);
    if (litsrc) litsrc->clear();
    std::unordered_multimap<uint64_t, const Structure*> by_key;  // key -> first structure of a class
    std::unordered_map<const Structure*, uint32_t> canon_of_first;
    uint32_t nct = 0;
    auto hash_slot = [&](const Structure* p) { return (size_t)((std::hash<const void*>{}(p) * 0x9E3779B97F4A7C15ull) >> 20) & (TB - 1); };
    for (const auto& sp : pins) {
        const Structure* p = sp.get();
        size_t i = hash_slot(p);
        while (slot_ptr[i] && slot_ptr[i] != p) i = (i + 1) & (TB - 1);
        if (slot_ptr[i]) continue;
        uint32_t id = UINT32_MAX;
        auto range = by_key.equal_range(p->key);
        for (auto it = range.first; it != range.second; ++it) {
            const Structure& o = *it->second;
            if (o.nv == p->nv && o.ncon == p->ncon && o.words == p->words) {
                id = canon_of_first[it->second];
                break;
            }
        }
        if (id == UINT32_MAX) {
            id = nct++;
            by_key.emplace(p->key, p);
            canon_of_first[p] = id;
        }
        slot_ptr[i] = p;
        slot_canon[i] = id;
        if (litsrc) {  // this structure's literal-slot sources (device-side records)
            slot_lsrc[i] = (uint32_t)litsrc->size();
            litsrc->insert(litsrc->end(), p->lit_src.begin(), p->lit_src.end());
        }
    }
    auto slot_of = [&](const Structure* p) -> size_t {
        size_t i = hash_slot(p);
        while (slot_ptr[i] != p) i = (i + 1) & (TB - 1);  // every compiled structure is pinned
        return i;
    };
    qcls.resize(n);
    // chunks: per-chunk tables of 3 * classes entries stay within 2^22 words
    const size_t per = std::max<size_t>(1, ((size_t)1 << 22) / std::max<size_t>(1, 3 * (size_t)nct));
    const size_t G = std::max<size_t>(8192, ((size_t)n + per - 1) / per);
    const size_t nch = ((size_t)n + G - 1) / G;
    std::vector<int64_t> firstq(nch * (size_t)std::max(nct, 1u), INT64_MAX);
    parallel_for(nch, 1, [&](size_t c0, size_t c1) {
        for (size_t ch = c0; ch < c1; ch++) {
            int64_t* fq = firstq.data() + ch * nct;
            const int64_t q1 = std::min<int64_t>(n, (int64_t)((ch + 1) * G));
            for (int64_t q = (int64_t)(ch * G); q < q1; q++) {
                Compiled& c = comp[q];
                if (!device_regime(c)) {
                    qcls[q] = 0;
                    other(q, c);
                    continue;
                }
                const size_t si = slot_of(c.st);
                const uint32_t cc = slot_canon[si];
                c.lsrc = slot_lsrc[si];
                qcls[q] = cc;
                if (fq[cc] == INT64_MAX) fq[cc] = q;
            }
        }
    });
    // dense ids in order of first appearance
    std::vector<std::pair<int64_t, uint32_t>> order;
    for (uint32_t cc = 0; cc < nct; cc++) {
        int64_t m = INT64_MAX;
        for (size_t ch = 0; ch < nch; ch++) m = std::min(m, firstq[ch * nct + cc]);
        if (m != INT64_MAX) order.push_back({m, cc});
    }
    std::sort(order.begin(), order.end());
    std::vector<uint32_t> dense(std::max(nct, 1u), UINT32_MAX);
    for (uint32_t i = 0; i < order.size(); i++) dense[order[i].second] = i;
    const uint32_t ncls = (uint32_t)order.size();
    K.ncls = ncls;
    if (pin_cls) {  // the class of every pins entry (UINT32_MAX: no device query)
        pin_cls->resize(pins.size());
        for (size_t k = 0; k < pins.size(); k++) (*pin_cls)[k] = dense[slot_canon[slot_of(pins[k].get())]];
    }
    const size_t W = 3 * (size_t)ncls;
    std::vector<uint32_t> cnt(nch * std::max<size_t>(W, 1), 0);
    parallel_for(nch, 1, [&](size_t c0, size_t c1) {
        for (size_t ch = c0; ch < c1; ch++) {
            uint32_t* ct = cnt.data() + ch * W;
            const int64_t q1 = std::min<int64_t>(n, (int64_t)((ch + 1) * G));
            for (int64_t q = (int64_t)(ch * G); q < q1; q++) {
                Compiled& c = comp[q];
                if (!device_regime(c)) continue;
                const uint32_t id = dense[qcls[q]];
                qcls[q] = id;
                c.cls = id;
                ct[(size_t)(c.regime - R_W64) * ncls + id]++;
            }
        }
    });
    // offsets: regime, then class, then chunk
    for (int w = 0; w < 3; w++) {
        K.start[w].assign(ncls + 1, 0);
        uint32_t at = 0;
        for (uint32_t c = 0; c < ncls; c++) {
            K.start[w][c] = at;
            for (size_t ch = 0; ch < nch; ch++) {
                uint32_t& x = cnt[ch * W + (size_t)w * ncls + c];
                const uint32_t k = x;
                x = at;
                at += k;
            }
        }
        K.start[w][ncls] = at;
        K.reg[w].resize(at);
    }
    parallel_for(nch, 1, [&](size_t c0, size_t c1) {
        for (size_t ch = c0; ch < c1; ch++) {
            uint32_t* ct = cnt.data() + ch * W;
            const int64_t q1 = std::min<int64_t>(n, (int64_t)((ch + 1) * G));
            for (int64_t q = (int64_t)(ch * G); q < q1; q++) {
                const Compiled& c = comp[q];
                if (!device_regime(c)) continue;
                const int w = c.regime - R_W64;
                K.reg[w][ct[(size_t)w * ncls + qcls[q]]++] = q;
            }
        }
    });
}

// Fast mode: compile the Unsat certificates of every structure class
// (cert.cuh) from up to CERT_REPS representatives spread over the class; the
// literal slots whose value varies inside the class are parameters.  Layout
// per class: [n certificates] then per certificate [length] [words].  The
// host only COMPILES (symbolic algebra on a few representatives); every
// query is decided by the device's numeric check of its class certificate.
constexpr int CERT_REPS = 8;

// Compiled certificates are kept per (structure, parameter slots, folded
// constants) -- exactly what they are valid for -- so later batches of the
// same structure classes (an analyzer re-run, the next chunk of a stream)
// skip the symbolic compile.  The full key is compared on a hit.
struct CertCache {
    std::mutex mu;
    std::unordered_map<uint64_t, std::vector<std::pair<std::vector<uint64_t>, std::vector<uint64_t>>>> map;
    size_t entries = 0;
};
CertCache& cert_cache() {
    static CertCache c;
    return c;
}
uint64_t key_hash(const std::vector<uint64_t>& k) {
    uint64_t h = 1469598103934665603ull;
    for (uint64_t x : k) h = (h ^ x) * 1099511628211ull;
    return h;
}
bool cert_cache_get(const std::vector<uint64_t>& key, std::vector<uint64_t>& out) {
    CertCache& C = cert_cache();
    std::lock_guard<std::mutex> lk(C.mu);
    auto it = C.map.find(key_hash(key));
    if (it == C.map.end()) return false;
    for (const auto& e : it->second)
        if (e.first == key) {
            out = e.second;
            return true;
        }
    return false;
}
void cert_cache_put(std::vector<uint64_t>&& key, const std::vector<uint64_t>& val) {
    CertCache& C = cert_cache();
    std::lock_guard<std::mutex> lk(C.mu);
    if (C.entries >= 65536) {  // bounded: start over
        C.map.clear();
        C.entries = 0;
    }
    const uint64_t h = key_hash(key);
    C.map[h].emplace_back(std::move(key), val);
    ++C.entries;
}
// the parameter scan's inputs gathered during compilation (Pins::note_lits)
struct VaryInput {
    const std::vector<std::vector<i128>>* first;
    const std::vector<std::vector<uint8_t>>* vary;
    const std::vector<uint8_t>* seen;
    const std::vector<uint32_t>* cls;
};
void build_certs(const oob_batch* b, const std::vector<Compiled>& comp, const Classes& K,
                 const std::vector<uint32_t>& qcls, std::vector<uint64_t>& certs, std::vector<uint32_t>& cert_off,
                 const VaryInput* vin = nullptr) {
    const uint32_t ncls = K.ncls;
    // literal slots whose value varies inside the class (the parameters):
    // each query against its class's first member, in parallel over queries
    // (every query through its own Structure: equal code words do not imply
    // equal literal-slot sources)
    std::vector<uint32_t> loff(ncls + 1, 0);
    std::vector<int64_t> first(ncls, -1);
    for (uint32_t c = 0; c < ncls; c++) {
        first[c] = K.member(c, 0);
        loff[c + 1] = loff[c] + (first[c] >= 0 ? comp[first[c]].st->nlit : 0);
    }
    std::vector<i128> v0(loff[ncls]);
    std::unique_ptr<std::atomic<uint8_t>[]> vary(new std::atomic<uint8_t>[std::max<uint32_t>(loff[ncls], 1)]);
    for (uint32_t c = 0; c < ncls; c++) {
        if (first[c] < 0) continue;
        for (uint32_t i = 0; i < loff[c + 1] - loff[c]; i++) {
            v0[loff[c] + i] = lit_value(b, first[c], *comp[first[c]].st, i);
            vary[loff[c] + i].store(0, std::memory_order_relaxed);
        }
    }
    if (vin) {
        // from the compile pass: a slot varies in a class if it varied within
        // one of the class's pinned structures (per compile chunk) or two of
        // them started with different values
        for (size_t k = 0; k < vin->seen->size(); k++) {
            const uint32_t c = (*vin->cls)[k];
            if (!(*vin->seen)[k] || c >= ncls) continue;
            const std::vector<i128>& f = (*vin->first)[k];
            const std::vector<uint8_t>& y = (*vin->vary)[k];
            const uint32_t ns = std::min<uint32_t>(loff[c + 1] - loff[c], (uint32_t)f.size());
            for (uint32_t i = 0; i < ns; i++)
                if (y[i] || f[i] != v0[loff[c] + i]) vary[loff[c] + i].store(1, std::memory_order_relaxed);
        }
    } else {
        for (int w = 0; w < 3; w++)
            parallel_for(K.reg[w].size(), 4096, [&](size_t lo, size_t hi) {
                for (size_t k = lo; k < hi; k++) {
                    const int64_t q = K.reg[w][k];
                    const uint32_t c = qcls[q];
                    const Structure& sk = *comp[q].st;
                    for (uint32_t i = 0; i < loff[c + 1] - loff[c]; i++) {
                        std::atomic<uint8_t>& f = vary[loff[c] + i];
                        if (!f.load(std::memory_order_relaxed) && lit_value(b, q, sk, i) != v0[loff[c] + i])
                            f.store(1, std::memory_order_relaxed);
                    }
                }
            });
    }
    std::vector<std::vector<uint64_t>> per(ncls);
    parallel_for(ncls, 1, [&](size_t lo, size_t hi) {
        static thread_local std::unique_ptr<sym::Store> S;
        static thread_local std::unique_ptr<sym::LaneWork> W;
        static thread_local std::unique_ptr<sym::Moves> M;
        static thread_local std::vector<uint64_t> buf;
        if (!S) {
            S.reset(new sym::Store());
            W.reset(new sym::LaneWork());
            M.reset(new sym::Moves());
            buf.resize(1 << 15);
        }
        for (size_t c = lo; c < hi; c++) {
            const size_t nm = K.members((uint32_t)c);
            if (!nm) continue;
            const Structure& st = *comp[first[c]].st;
            if (!st.range_why.empty()) continue;
            std::vector<int16_t> pmap(st.nlit, -1), pslot;
            for (uint32_t i = 0; i < st.nlit; i++)
                if (vary[loff[c] + i].load(std::memory_order_relaxed)) {
                    pmap[i] = (int16_t)pslot.size();
                    pslot.push_back((int16_t)i);
                }
            // compiled before for this structure, parameter set and constants?
            std::vector<uint64_t> ckey;
            ckey.reserve(st.words.size() + 4 + 3 * st.nlit);
            ckey.push_back(st.nv);
            ckey.push_back(st.ncon);
            ckey.push_back(st.nlit);
            ckey.insert(ckey.end(), st.words.begin(), st.words.end());
            for (uint32_t i = 0; i < st.nlit; i++) {
                const bool var_i = pmap[i] >= 0;
                ckey.push_back(var_i);
                if (!var_i) {
                    const i128 x = v0[loff[c] + i];
                    ckey.push_back((uint64_t)x);
                    ckey.push_back((uint64_t)((unsigned __int128)x >> 64));
                }
            }
            // representatives: the member with the widest domains first (a
            // certificate holds for every member whose domains of the
            // eliminated variables lie within the representative's, and its
            // sign conditions only get easier on sub-boxes), then members
            // spread over the class
            int64_t widest = first[c];
            {
                double wc = comp[widest].cost;
                size_t i = 0;
                for (int w = 0; w < 3; w++)
                    for (uint32_t k = K.start[w][c]; k < K.start[w][c + 1]; k++, i++) {
                        const int64_t q = K.reg[w][k];
                        if (i > 0 && comp[q].cost > wc) {
                            widest = q;
                            wc = comp[q].cost;
                        }
                    }
            }
            // ... so the cache key also carries the widest member's domains
            {
                const int64_t vb = b->var_begin[widest];
                for (uint32_t v = 0; v < st.nv; v++) {
                    const i128 lo = from_w(b->var_lo[vb + v]), hi = from_w(b->var_hi[vb + v]);
                    ckey.push_back((uint64_t)lo);
                    ckey.push_back((uint64_t)((unsigned __int128)lo >> 64));
                    ckey.push_back((uint64_t)hi);
                    ckey.push_back((uint64_t)((unsigned __int128)hi >> 64));
                }
            }
            if (cert_cache_get(ckey, per[c])) continue;
            std::vector<std::vector<uint64_t>> got;
            const size_t nr = std::min<size_t>(CERT_REPS, nm);
            for (size_t r = 0; r <= nr; r++) {
                const int64_t q = r == 0 ? widest : K.member((uint32_t)c, (r - 1) * nm / nr);
                if (r > 0 && q == widest) continue;
                const int64_t vb = b->var_begin[q];
                auto dom = [&](uint32_t i) -> i128 { return from_w(i % 2 ? b->var_hi[vb + i / 2] : b->var_lo[vb + i / 2]); };
                const Structure& sq = *comp[q].st;
                auto lit = [&](uint32_t i) -> i128 { return lit_value(b, q, sq, i); };
                const size_t n = cert::cert_build(*S, *W, *M, st.words.data(), st.code(), st.nv, st.ncon, st.nlit,
                                                  dom, lit,
                                                  pmap.data(), (int)pslot.size(), pslot.data(), buf.data(),
                                                  buf.size());
                if (!n) continue;
                std::vector<uint64_t> blob(buf.begin(), buf.begin() + n);
                bool dup = false;
                for (const auto& o : got) dup = dup || o == blob;
                if (!dup) got.push_back(std::move(blob));
            }
            std::vector<uint64_t>& out = per[c];
            if (!got.empty()) {
                out.push_back(got.size());
                for (const auto& g : got) {
                    out.push_back(g.size());
                    out.insert(out.end(), g.begin(), g.end());
                }
            }
            cert_cache_put(std::move(ckey), out);
        }
    });
    certs.clear();
    cert_off.assign(ncls, NO_CERT);
    for (uint32_t c = 0; c < ncls; c++) {
        if (per[c].empty()) continue;
        cert_off[c] = (uint32_t)certs.size();
        certs.insert(certs.end(), per[c].begin(), per[c].end());
    }
}

// Compile + schedule: fills immediate verdicts and returns the device jobs.
struct Prepared {
    std::vector<Compiled> comp;
    // SOLVE: the caller's raw domains and literals in page-locked memory,
    // copied by the compile pass (device-side records, RunCtx::raw)
    bool raw = false;
    HostArr<int64_t> raw_vlo, raw_vhi, raw_l;  // narrowed to int64 (else no device-side records)
    int64_t raw_v0 = 0, raw_l0 = 0;
    uint64_t raw_nv = 0, raw_nl = 0;
    std::vector<int32_t> litsrc;  // literal-slot sources of every structure (Compiled::lsrc)
    std::vector<std::shared_ptr<const Structure>> pins;  // every structure comp[] points to
    // fast mode, per pins entry (Pins::note_lits): first literal-slot values,
    // varying slots, whether a device query was seen; the class of each entry
    std::vector<std::vector<i128>> pin_first;
    std::vector<std::vector<uint8_t>> pin_vary;
    std::vector<uint8_t> pin_seen;
    std::vector<uint32_t> pin_cls;
    Classes classes;
    std::vector<uint32_t> qcls;  // comp[q].cls, compact
    std::vector<uint64_t> certs;     // fast mode: Unsat certificates (cert.cuh)
    std::vector<uint32_t> cert_off;  // per structure class: offset in certs, NO_CERT: none
    std::vector<int8_t> errs;
    std::vector<DevWork> work;  // per device: queries by proven regime
    std::string range_msg;
    oob_options opt{};
    double compile_s = 0;
};

int prepare(const oob_batch* b, const oob_options* opt_in, int mode, const oob_i128* model_in, int8_t* verdict,
            int64_t* nodes, int64_t* passes, double* elapsed, Prepared& pr, int virtual_devices = 0) {
    g_last_error.clear();
    if (!b || b->n_queries < 0) return fail(OOB_E_INVALID, "null or negative batch");
    pr.opt.timeout_s = 30.0;
    if (opt_in) pr.opt = *opt_in;
    const oob_options& opt = pr.opt;
    const int64_t n = b->n_queries;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<Compiled>& comp = pr.comp;
    if ((int64_t)comp.size() != n) comp.resize(n);  // every entry is overwritten below (recycled storage)
    const bool fast_shortcut = mode == MODE_SOLVE && (opt.flags & OOB_F_FAST);
    pr.pins.clear();
    pr.pin_first.clear();
    pr.pin_vary.clear();
    pr.pin_seen.clear();
    // device-side records (SOLVE): the compile pass also copies each chunk's
    // raw domains and literals into page-locked arrays (one H2D per call
    // instead of ~2x their size in regime-width records filled on the host)
    {
        static const bool env_on = [] {
            const char* e = std::getenv("SCUBA_OOB_DEVICE_RECORDS");
            return !(e && *e == '0');
        }();
        pr.raw = false;
        if (mode == MODE_SOLVE && env_on && n > 0) {
            const int64_t v0 = b->var_begin[0], v1 = b->var_begin[n], l0 = b->lit_begin[0], l1 = b->lit_begin[n];
            if (v1 >= v0 && l1 >= l0 && v1 - v0 < (int64_t)UINT32_MAX && l1 - l0 < (int64_t)UINT32_MAX) {
                pr.raw = true;
                pr.raw_v0 = v0;
                pr.raw_l0 = l0;
                pr.raw_nv = (uint64_t)(v1 - v0);
                pr.raw_nl = (uint64_t)(l1 - l0);
                pr.raw_vlo.alloc(std::max<uint64_t>(pr.raw_nv, 1));
                pr.raw_vhi.alloc(std::max<uint64_t>(pr.raw_nv, 1));
                pr.raw_l.alloc(std::max<uint64_t>(pr.raw_nl, 1));
            }
        }
    }
    {
        // validation and compilation in one pass over the batch: a query is
        // compiled only once it has validated; the lowest invalid query is
        // reported (nothing is decided for an invalid batch)
        Phase ph("validate+compile");
        std::atomic<int64_t> bad{INT64_MAX};
        std::atomic<bool> raw_wide{false};  // a raw value beyond int64: the records are filled on the host
        std::mutex pins_mu;
        std::unordered_map<const Structure*, size_t> pin_at;  // structure -> its pins entry
        parallel_for((size_t)n, 256, [&](size_t lo, size_t hi) {
            Pins pins;
            bool valid = true;
            for (size_t q = lo; q < hi; q++) {
                // offsets here; the terms inside compile_query, only for terms
                // not already validated in an equal query (StructCache::get)
                if (validate_offsets(b, (int64_t)q) ||
                    (comp[q] = compile_query(b, (int64_t)q, mode, opt.timeout_s, model_in, pins, fast_shortcut))
                            .regime == R_INVALID) {
                    int64_t cur = bad.load();
                    while ((int64_t)q < cur && !bad.compare_exchange_weak(cur, (int64_t)q)) {
                    }
                    valid = false;
                    break;
                }
                if (fast_shortcut && device_regime(comp[q])) pins.note_lits(tl_cq_lits, comp[q].nlit);
            }
            if (valid && pr.raw) {  // this chunk's raw values (contiguous: offsets validated), as int64
                const int64_t va = b->var_begin[lo], vz = b->var_begin[hi];
                const int64_t la = b->lit_begin[lo], lz = b->lit_begin[hi];
                bool fits = true;
                auto narrow = [&](int64_t* dst, const oob_i128* src, int64_t k) {
                    for (int64_t i = 0; i < k; i++) {
                        const int64_t w = (int64_t)src[i].lo;
                        fits &= src[i].hi == (w >> 63);
                        dst[i] = w;
                    }
                };
                narrow(pr.raw_vlo.data() + (va - pr.raw_v0), b->var_lo + va, vz - va);
                narrow(pr.raw_vhi.data() + (va - pr.raw_v0), b->var_hi + va, vz - va);
                narrow(pr.raw_l.data() + (la - pr.raw_l0), b->lits + la, lz - la);
                if (!fits) raw_wide.store(true, std::memory_order_relaxed);
            }
            std::lock_guard<std::mutex> lk(pins_mu);
            for (size_t k = 0; k < pins.v.size(); k++) {
                // one parameter-scan entry per distinct structure: merge this chunk's
                const Structure* sp = pins.v[k].get();
                auto it = pin_at.find(sp);
                if (it == pin_at.end()) {
                    pin_at.emplace(sp, pr.pins.size());
                    pr.pins.push_back(std::move(pins.v[k]));
                    pr.pin_first.push_back(std::move(pins.first[k]));
                    pr.pin_vary.push_back(std::move(pins.vary[k]));
                    pr.pin_seen.push_back(pins.seen[k]);
                    continue;
                }
                if (!pins.seen[k]) continue;
                const size_t g = it->second;
                if (!pr.pin_seen[g]) {
                    pr.pin_seen[g] = 1;
                    pr.pin_first[g] = std::move(pins.first[k]);
                    pr.pin_vary[g] = std::move(pins.vary[k]);
                    continue;
                }
                const std::vector<i128>& f = pins.first[k];
                std::vector<uint8_t>& y = pr.pin_vary[g];
                for (size_t i = 0; i < f.size() && i < y.size(); i++)
                    y[i] |= pins.vary[k][i] | (f[i] != pr.pin_first[g][i]);
            }
        });
        if (bad.load() != INT64_MAX) {
            int64_t q = bad.load();
            return fail(OOB_E_INVALID, "query " + std::to_string(q) + ": " + validate(b, q));
        }
        if (raw_wide.load()) pr.raw = false;  // (values beyond int64: records filled on the host)
    }
    pr.compile_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (gate_point() == GATE_COMPILE) gate_release();
    pr.errs.assign(n, 0);
    if (virtual_devices <= 0) virtual_devices = env_virtual_devices();
    const int ndev = virtual_devices > 0 ? virtual_devices : visible_devices();
    Phase ph_sched("schedule");
    Classes& K = pr.classes;
    {
        // immediate verdicts and range errors on the way (the lowest
        // out-of-range query is reported)
        Phase ph_cls("schedule.classes");
        std::atomic<int64_t> range_q{INT64_MAX};
        const double el = std::max(pr.compile_s / std::max<int64_t>(n, 1), 1e-9);
        classify(comp, n, pr.pins, pr.qcls, K, [&](int64_t q, const Compiled& c) {
            if (c.regime == R_IMMEDIATE) {
                verdict[q] = c.immediate;
                if (nodes) nodes[q] = 0;
                if (passes) passes[q] = 0;
                if (elapsed) elapsed[q] = el;
            } else {  // R_RANGE
                verdict[q] = OOB_ERROR;
                int64_t cur = range_q.load();
                while (q < cur && !range_q.compare_exchange_weak(cur, q)) {
                }
            }
        }, pr.raw ? &pr.litsrc : nullptr, &pr.pin_cls);
        if (range_q.load() != INT64_MAX)
            pr.range_msg = "query " + std::to_string(range_q.load()) + ": " + comp[range_q.load()].why;
    }
    const size_t n_dev_q = K.reg[0].size() + K.reg[1].size() + K.reg[2].size();
    if (n_dev_q > 0 && ndev == 0)
        return fail(OOB_E_CUDA, "no CUDA device visible: the OOB engine has no CPU fallback");
    int first = std::max(0, opt.device);
    if (first >= ndev && n_dev_q > 0)
        return fail(OOB_E_CUDA, "device ordinal out of range");
    int want = opt.n_gpus > 0 ? opt.n_gpus : ndev - first;
    want = std::max(1, std::min(want, ndev - first));
    pr.certs.clear();
    pr.cert_off.clear();
    if (mode == MODE_SOLVE && (opt.flags & OOB_F_FAST) && opt.timeout_s > 0) {
        Phase ph_cert("certify");
        const VaryInput vin{&pr.pin_first, &pr.pin_vary, &pr.pin_seen, &pr.pin_cls};
        build_certs(b, comp, K, pr.qcls, pr.certs, pr.cert_off, fast_shortcut ? &vin : nullptr);
    }
    if (n_dev_q > 0) {
        pr.work.resize(want);
        for (int d = 0; d < want; d++) pr.work[d].dev = first + d;
    }
    struct GateAtEnd {
        ~GateAtEnd() { if (gate_point() == GATE_SCHEDULE) gate_release(); }
    } gate_at_end;
    Phase ph_sort("schedule.sort");
    // class-major (classify), cost-minor: expensive first, ties by query
    // index -- a stable counting sort per (regime, class) range, in parallel
    if (!(opt.flags & OOB_F_NO_SORT)) {
        std::vector<std::pair<int, uint32_t>> ranges;
        for (int w = 0; w < 3; w++)
            for (uint32_t c = 0; c < K.ncls; c++)
                if (K.start[w][c + 1] - K.start[w][c] >= 2) ranges.push_back({w, c});
        parallel_for(ranges.size(), 1, [&](size_t lo, size_t hi) {
            std::vector<uint32_t> cnt;
            std::vector<std::pair<uint32_t, int64_t>> tmp;
            for (size_t r = lo; r < hi; r++) {
                std::vector<int64_t>& qs = K.reg[ranges[r].first];
                const uint32_t c = ranges[r].second;
                const size_t a = K.start[ranges[r].first][c], z = K.start[ranges[r].first][c + 1];
                tmp.resize(z - a);
                uint32_t kmin = 0xFFFFFFFFu, kmax = 0;
                for (size_t i = a; i < z; i++) {
                    const uint32_t key = 0xFFFFu - (uint32_t)std::min(comp[qs[i]].cost, 65535.0);
                    tmp[i - a] = {key, qs[i]};
                    kmin = std::min(kmin, key);
                    kmax = std::max(kmax, key);
                }
                if (kmin == kmax) continue;  // one key: already in query order
                cnt.assign(kmax - kmin + 2, 0);
                for (const auto& t : tmp) cnt[t.first - kmin + 1]++;
                for (size_t k = 1; k < cnt.size(); k++) cnt[k] += cnt[k - 1];
                for (const auto& t : tmp) qs[a + cnt[t.first - kmin]++] = t.second;
            }
        });
    }
    for (int w = 0; w < 3; w++) {
        const auto& qs = K.reg[w];
        if (qs.empty()) continue;
        if (want == 1) {
            pr.work[0].qs[w] = qs;
        } else {
            for (int d = 0; d < want; d++) pr.work[d].qs[w].reserve(qs.size() / want + 32);
            for (size_t i = 0; i < qs.size(); i++) pr.work[(i / 32) % want].qs[w].push_back(qs[i]);
        }
    }
    return OOB_OK;
}

int finish(Prepared& pr, int64_t n) {
    for (int64_t q = 0; q < n; q++) {
        if (pr.errs[q] != ERR_NONE && pr.range_msg.empty())
            pr.range_msg = "query " + std::to_string(q) + ": search outgrew the device scratch (error " +
                           std::to_string(pr.errs[q]) + ")";
    }
    if (!pr.range_msg.empty()) return fail(OOB_E_RANGE, pr.range_msg);
    return OOB_OK;
}

// device-side records: the prepared call's raw values (RunCtx::raw)
void set_raw(RunCtx& rc, const Prepared& pr) {
    rc.raw = pr.raw;
    rc.raw_vlo = pr.raw_vlo.data();
    rc.raw_vhi = pr.raw_vhi.data();
    rc.raw_l = pr.raw_l.data();
    rc.raw_nv = pr.raw_nv;
    rc.raw_nl = pr.raw_nl;
    rc.raw_v0 = pr.raw_v0;
    rc.raw_l0 = pr.raw_l0;
    rc.litsrc = &pr.litsrc;
}

// Common driver of the three batched entry points.
int drive(const oob_batch* b, const oob_options* opt_in, int mode, const oob_i128* model_in, oob_i128* model_out,
          int8_t* verdict, int64_t* nodes, int64_t* passes, double* elapsed) {
    if (mode == MODE_SOLVE && model_out && b && b->n_queries > 0) {
        // every model row is written (zero unless SAT): cleared here in
        // parallel, so the caller's fresh buffer is faulted in by all host
        // threads instead of one
        Phase ph("clear");
        const int64_t v0 = b->var_begin[0], v1 = b->var_begin[b->n_queries];
        if (v1 > v0)
            parallel_for((size_t)(v1 - v0), 1 << 14, [&](size_t lo, size_t hi) {
                std::memset((void*)(model_out + v0 + lo), 0, (hi - lo) * sizeof(oob_i128));
            });
    }
    // the per-query vectors of a call are recycled per thread (fresh 10+ MB
    // vectors would be page-faulted in on every call)
    static thread_local std::vector<Compiled> tl_comp;
    static thread_local std::vector<uint32_t> tl_qcls;
    static thread_local std::vector<int8_t> tl_errs;
    Prepared pr;
    pr.comp.swap(tl_comp);
    pr.qcls.swap(tl_qcls);
    pr.errs.swap(tl_errs);
    auto recycle = [&]() {
        pr.comp.swap(tl_comp);  // (kept sized: entries are overwritten by the next call)
        pr.qcls.swap(tl_qcls);
        pr.errs.swap(tl_errs);
    };
    int rc0 = prepare(b, opt_in, mode, model_in, verdict, nodes, passes, elapsed, pr);
    if (rc0 != OOB_OK) {
        recycle();
        return rc0;
    }
    RunCtx rc;
    rc.b = b;
    rc.opt = pr.opt;
    rc.comp = &pr.comp;
    rc.qcls = &pr.qcls;
    rc.mode = mode;
    rc.verdict = verdict;
    rc.model = mode == MODE_CHECK ? const_cast<oob_i128*>(model_in) : model_out;
    rc.nodes = nodes;
    rc.passes = passes;
    rc.elapsed = elapsed;
    rc.errs = &pr.errs;
    rc.certs = &pr.certs;
    rc.cert_off = &pr.cert_off;
    set_raw(rc, pr);
    std::string e = run_all(rc, pr.work);
    if (!e.empty()) {
        recycle();
        return fail(OOB_E_CUDA, e);
    }
    int rcode = finish(pr, b->n_queries);
    {
        Phase ph("teardown");
        recycle();
        Prepared gone(std::move(pr));
    }
    return rcode;
}

// SOLVE through drive().  A device allocation failure frees the device
// buffers of the other pool slots (stream API workers keep theirs between
// calls) and retries once; a worker of another slot falls back to slot 0's
// buffers for good (the pool locks serialise the device phases).
int drive_solve(const oob_batch* b, const oob_options* opt, const oob_result& o) {
    int rc = drive(b, opt, MODE_SOLVE, nullptr, o.model, o.verdict, o.nodes, o.passes, o.elapsed_s);
    if (rc != OOB_E_CUDA || g_last_error.find("out of memory") == std::string::npos) return rc;
    cudaGetLastError();
    if (tl_pool_slot != 0) {
        release_slot_pools(tl_pool_slot);
        tl_pool_slot = 0;
    } else {
        for (int s = 1; s < 4; s++) release_slot_pools(s);
    }
    return drive(b, opt, MODE_SOLVE, nullptr, o.model, o.verdict, o.nodes, o.passes, o.elapsed_s);
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int oob_solve_batch(const oob_batch* batch, const oob_options* opt, oob_result* out) {
    if (!out || !out->verdict) return fail(OOB_E_INVALID, "result arrays missing");
    if (!batch) return fail(OOB_E_INVALID, "null batch");
    // SCUBA_OOB_CHUNK=<queries>: large single-device calls are pipelined: the batch is cut into chunks
    // (each an oob_batch view; all offsets are per query) decided
    // concurrently on separate device buffers, with the host-heavy phases
    // taken in chunk order.  Results are identical (queries are independent).
    const int64_t n = batch->n_queries;
    static const int64_t chunk_q = [] {
        const char* e = std::getenv("SCUBA_OOB_CHUNK");
        return (int64_t)((e && *e) ? std::atoll(e) : 0);  // off by default: measured slower
    }();
    const bool one_dev = (opt && opt->n_gpus == 1) || visible_devices() <= 1;
    if (chunk_q <= 0 || n < 2 * chunk_q || !one_dev || tl_gate) return drive_solve(batch, opt, *out);
    const int k = (int)std::min<int64_t>(4, (n + chunk_q - 1) / chunk_q);
    HostGate gate;
    std::vector<int> rcs(k, OOB_OK);
    std::vector<std::string> msgs(k);
    std::vector<std::thread> th;
    for (int c = 0; c < k; c++) {
        th.emplace_back([&, c]() {
            const int64_t q0 = n * c / k, q1 = n * (c + 1) / k;
            oob_batch sub = *batch;
            sub.n_queries = q1 - q0;
            sub.var_begin += q0;
            sub.con_begin += q0;
            sub.node_begin += q0;
            sub.lit_begin += q0;
            tl_pool_slot = c;
            tl_gate = &gate;
            tl_chunk = c;
            {
                std::unique_lock<std::mutex> lk(gate.mu);
                gate.cv.wait(lk, [&] { return gate.turn >= c; });
            }
            tl_gate_held = true;
            oob_result part = *out;
            part.verdict = out->verdict + q0;
            part.nodes = out->nodes ? out->nodes + q0 : nullptr;
            part.passes = out->passes ? out->passes + q0 : nullptr;
            part.elapsed_s = out->elapsed_s ? out->elapsed_s + q0 : nullptr;
            rcs[c] = drive_solve(&sub, opt, part);
            if (rcs[c] != OOB_OK) msgs[c] = g_last_error;
            gate_release();  // also on early exits (no launch happened)
            tl_gate = nullptr;
            tl_pool_slot = 0;
        });
    }
    for (auto& t : th) t.join();
    for (int c = 0; c < k; c++)
        if (rcs[c] != OOB_OK) return fail(rcs[c], "chunk " + std::to_string(c) + ": " + msgs[c]);
    g_last_error.clear();
    return OOB_OK;
}

int oob_solve_batches(const oob_batch* batches, int64_t n_batches, const oob_options* opt, oob_result* outs) {
    if (!batches || !outs || n_batches < 0) return fail(OOB_E_INVALID, "null argument");
    for (int64_t i = 0; i < n_batches; i++)
        if (!outs[i].verdict) return fail(OOB_E_INVALID, "result arrays missing");
    if (n_batches == 1) return oob_solve_batch(batches, opt, outs);
    // two workers (pool slots 0/1) take the batches alternately; the gate
    // hands the host phase (compile, certify, pack, upload, launch) to batch
    // i + 1 as soon as batch i has launched its kernels, so host work and
    // device work of consecutive batches overlap
    HostGate gate;
    std::vector<int> rcs(n_batches, OOB_OK);
    std::vector<std::string> msgs(n_batches);
    std::vector<std::thread> th;
    static const int n_slots = [] {
        const char* e = std::getenv("SCUBA_OOB_STREAM_SLOTS");
        return (e && *e) ? std::max(1, std::min(4, std::atoi(e))) : 3;
    }();
    for (int s = 0; s < n_slots && s < n_batches; s++) {
        th.emplace_back([&, s]() {
            tl_pool_slot = s;
            tl_gate = &gate;
            for (int64_t i = s; i < n_batches; i += n_slots) {
                tl_chunk = (int)i;
                {
                    std::unique_lock<std::mutex> lk(gate.mu);
                    gate.cv.wait(lk, [&] { return gate.turn >= (int)i; });
                }
                tl_gate_held = true;
                const oob_result& o = outs[i];
                rcs[i] = drive_solve(batches + i, opt, o);
                if (rcs[i] != OOB_OK) msgs[i] = g_last_error;
                gate_release();  // also on early exits (no launch happened)
            }
            tl_gate = nullptr;
            tl_pool_slot = 0;
        });
    }
    for (auto& t : th) t.join();
    for (int64_t i = 0; i < n_batches; i++)
        if (rcs[i] != OOB_OK) return fail(rcs[i], "batch " + std::to_string(i) + ": " + msgs[i]);
    g_last_error.clear();
    return OOB_OK;
}

int oob_propagate_batch(const oob_batch* batch, const oob_options* opt, oob_i128* out_lo, oob_i128* out_hi,
                        int8_t* status) {
    if (!batch || !out_lo || !out_hi || !status) return fail(OOB_E_INVALID, "null argument");
    int64_t V = batch->var_begin[batch->n_queries];
    std::vector<oob_i128> pairs((size_t)std::max<int64_t>(V, 1) * 2);
    std::vector<int8_t> verdict(batch->n_queries);
    int rc = drive(batch, opt, MODE_PROPAGATE, nullptr, pairs.data(), verdict.data(), nullptr, nullptr, nullptr);
    if (rc != OOB_OK) return rc;
    for (int64_t q = 0; q < batch->n_queries; q++) {
        status[q] = verdict[q] == OOB_SAT ? 1 : 0;
        for (int64_t v = batch->var_begin[q]; v < batch->var_begin[q + 1]; v++) {
            out_lo[v] = pairs[2 * v];
            out_hi[v] = pairs[2 * v + 1];
        }
    }
    return OOB_OK;
}

int oob_check_model_batch(const oob_batch* batch, const oob_options* opt, const oob_i128* model, int8_t* ok) {
    if (!batch || !model || !ok) return fail(OOB_E_INVALID, "null argument");
    std::vector<int8_t> verdict(batch->n_queries);
    int rc = drive(batch, opt, MODE_CHECK, model, nullptr, verdict.data(), nullptr, nullptr, nullptr);
    if (rc != OOB_OK) return rc;
    for (int64_t q = 0; q < batch->n_queries; q++) ok[q] = verdict[q] == OOB_SAT ? 1 : 0;
    return OOB_OK;
}

int oob_side_constraint_count(const oob_batch* b, int64_t* counts) {
    g_last_error.clear();
    if (!b || !counts) return fail(OOB_E_INVALID, "null argument");
    for (int64_t q = 0; q < b->n_queries; q++) {
        std::string why = validate(b, q);
        if (!why.empty()) return fail(OOB_E_INVALID, "query " + std::to_string(q) + ": " + why);
        QView v = view_of(b, q);
        std::vector<int> divs;
        for (int k = 0; k < v.ncon; k++) {
            collect_divisors(v, v.lhs[k], divs);
            collect_divisors(v, v.rhs[k], divs);
        }
        int64_t c = 0;
        for (int d : divs) c += v.op[d] != OOB_NODE_LIT;
        counts[q] = c;
    }
    return OOB_OK;
}

int oob_jit_compile(const oob_batch* b, int64_t q, char* src, int64_t src_cap, double* compile_ms) {
    g_last_error.clear();
    if (!b || q < 0 || q >= b->n_queries) return fail(OOB_E_INVALID, "bad query index");
    std::string why = validate(b, q);
    if (!why.empty()) return fail(OOB_E_INVALID, why);
    Pins pins;
    Compiled c = compile_query(b, q, MODE_SOLVE, 30.0, nullptr, pins);
    if (c.regime == R_IMMEDIATE || c.regime == R_RANGE) return fail(OOB_E_INVALID, "query has no search");
    JitClass jc{c.words().data(), c.nv, c.ncon, c.ncode, c.nlit, c.regime == R_W128 ? 128 : 64};
    std::string text = jit_source(jc);
    if (src && src_cap > 0) {
        size_t n = std::min<size_t>(text.size(), (size_t)src_cap - 1);
        std::memcpy(src, text.data(), n);
        src[n] = 0;
    }
    std::vector<const void*> k;
    std::vector<int> regs;
    std::string e = jit_prepare({jc}, k, regs, compile_ms, false);
    if (!e.empty()) return fail(OOB_E_INVALID, e);
    return OOB_OK;
}

int oob_host_bench(const oob_batch* b, const oob_options* opt, double* ms) {
    // host pipeline only (no device): compile + schedule (prepare), then pack
    if (!b || !ms) return fail(OOB_E_INVALID, "null argument");
    const int64_t n = b->n_queries;
    std::vector<int8_t> verdict(n);
    std::vector<int64_t> nodes(n), passes(n);
    std::vector<double> el(n);
    auto t0 = std::chrono::steady_clock::now();
    Prepared pr;
    int rc0 = prepare(b, opt, MODE_SOLVE, nullptr, verdict.data(), nodes.data(), passes.data(), el.data(), pr, 1);
    if (rc0 != OOB_OK) return rc0;
    auto t1 = std::chrono::steady_clock::now();
    RunCtx rc;
    rc.b = b;
    rc.opt = pr.opt;
    rc.comp = &pr.comp;
    rc.qcls = &pr.qcls;
    rc.mode = MODE_SOLVE;
    rc.errs = &pr.errs;
    rc.certs = &pr.certs;
    rc.cert_off = &pr.cert_off;
    set_raw(rc, pr);
    for (auto& wk : pr.work) {
        DevGroup G;
        G.dev = wk.dev;
        for (int w = 0; w < 3; w++) G.job[w].qs = wk.qs[w];
        pack_group(rc, G);
    }
    auto t2 = std::chrono::steady_clock::now();
    ms[0] = pr.compile_s * 1e3;
    ms[1] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    ms[2] = std::chrono::duration<double, std::milli>(t2 - t1).count();
    return OOB_OK;
}

int oob_cert_compile(const oob_batch* b, const oob_options* opt, uint64_t* words, int64_t words_cap,
                     int64_t* n_words, int64_t* cert_off, oob_i128* slots, int64_t slots_cap, int64_t* slot_begin) {
    g_last_error.clear();
    if (!b || !words || !n_words || !cert_off || !slots || !slot_begin) return fail(OOB_E_INVALID, "null argument");
    const double timeout_s = opt ? opt->timeout_s : 30.0;
    const int64_t n = b->n_queries;
    std::vector<Compiled> comp(n);
    Pins pins;
    for (int64_t q = 0; q < n; q++) {
        std::string why = validate(b, q);
        if (!why.empty()) return fail(OOB_E_INVALID, "query " + std::to_string(q) + ": " + why);
        comp[q] = compile_query(b, q, MODE_SOLVE, timeout_s, nullptr, pins);
    }
    Classes K;
    std::vector<uint32_t> qcls;
    classify(comp, n, pins.v, qcls, K, [](int64_t, const Compiled&) {});
    std::vector<uint64_t> certs;
    std::vector<uint32_t> off;
    build_certs(b, comp, K, qcls, certs, off);
    if ((int64_t)certs.size() > words_cap) return fail(OOB_E_NOMEM, "certificate words exceed the buffer");
    std::copy(certs.begin(), certs.end(), words);
    *n_words = (int64_t)certs.size();
    int64_t at = 0;
    for (int64_t q = 0; q < n; q++) {
        slot_begin[q] = at;
        const Compiled& c = comp[q];
        const bool dev = c.regime >= R_W64 && c.regime < R_W64 + 3;
        cert_off[q] = (dev && c.cls < off.size() && off[c.cls] != NO_CERT) ? (int64_t)off[c.cls] : -1;
        if (!dev) continue;
        if (at + c.nlit > slots_cap) return fail(OOB_E_NOMEM, "literal slots exceed the buffer");
        for (uint32_t i = 0; i < c.nlit; i++) {
            const i128 v = lit_value(b, q, *c.st, i);
            slots[at++] = oob_i128{(uint64_t)v, (int64_t)(v >> 64)};
        }
    }
    slot_begin[n] = at;
    return OOB_OK;
}

int oob_query_regime(const oob_batch* b, const oob_options* opt, int8_t* regime) {
    g_last_error.clear();
    if (!b || !regime) return fail(OOB_E_INVALID, "null argument");
    double timeout_s = opt ? opt->timeout_s : 30.0;
    for (int64_t q = 0; q < b->n_queries; q++) {
        std::string why = validate(b, q);
        if (!why.empty()) return fail(OOB_E_INVALID, "query " + std::to_string(q) + ": " + why);
        Pins pins;
        regime[q] = compile_query(b, q, MODE_SOLVE, timeout_s, nullptr, pins).regime;
    }
    return OOB_OK;
}

// ----- plans: compile + upload once, time kernels on device-resident data -----
struct oob_plan {
    const oob_batch* b;
    Prepared pr;
    std::vector<DevGroup> groups;
    std::vector<std::unique_ptr<DevicePool>> pools;  // three private pools per group
    RunCtx rc;
    std::vector<int8_t> verdict;
    std::vector<int64_t> nodes, passes;
    std::vector<double> elapsed;
    std::vector<oob_i128> model;
    int64_t runs = 0;
};

// frees a plan's device buffers, streams and events (also a partly built one)
static void plan_free(oob_plan* p) {
    if (!p) return;
    for (auto& G : p->groups)
        for (int w = 0; w < NJOBS; w++) {
            DevicePool* P = G.pool[w];
            if (!P) continue;
            cudaSetDevice(phys_dev(G.dev));
            P->release_all();
            if (P->ev0) cudaEventDestroy(P->ev0);
            if (P->ev1) cudaEventDestroy(P->ev1);
            if (P->evr) cudaEventDestroy(P->evr);
            for (auto x : P->xs) cudaStreamDestroy(x);
            for (auto x : P->xev) cudaEventDestroy(x);
            if (P->stream) cudaStreamDestroy(P->stream);
        }
    delete p;
}
struct PlanFree {
    void operator()(oob_plan* p) const { plan_free(p); }
};

static int plan_create_once(const oob_batch* batch, const oob_options* opt, oob_plan** out) {
    std::unique_ptr<oob_plan, PlanFree> p(new oob_plan());
    p->b = batch;
    if (!batch) return fail(OOB_E_INVALID, "null batch");
    int64_t n = batch->n_queries;
    p->verdict.assign(n, 0);
    p->nodes.assign(n, 0);
    p->passes.assign(n, 0);
    p->elapsed.assign(n, 0);
    p->model.assign((size_t)std::max<int64_t>(batch->var_begin[n], 1), oob_i128{0, 0});
    int rc0 = prepare(batch, opt, MODE_SOLVE, nullptr, p->verdict.data(), p->nodes.data(), p->passes.data(),
                      p->elapsed.data(), p->pr);
    if (rc0 != OOB_OK) return rc0;
    RunCtx& rc = p->rc;
    rc.b = batch;
    rc.opt = p->pr.opt;
    rc.comp = &p->pr.comp;
    rc.qcls = &p->pr.qcls;
    rc.mode = MODE_SOLVE;
    rc.verdict = p->verdict.data();
    rc.model = p->model.data();
    rc.nodes = p->nodes.data();
    rc.passes = p->passes.data();
    rc.elapsed = p->elapsed.data();
    rc.errs = &p->pr.errs;
    rc.certs = &p->pr.certs;
    rc.cert_off = &p->pr.cert_off;
    set_raw(rc, p->pr);
    p->groups.resize(p->pr.work.size());
    for (size_t k = 0; k < p->pr.work.size(); k++) {
        DevGroup& G = p->groups[k];
        G.dev = p->pr.work[k].dev;
        for (int w = 0; w < NJOBS; w++) {
            if (w < 3) G.job[w].qs = p->pr.work[k].qs[w];
            p->pools.emplace_back(new DevicePool());
            G.pool[w] = p->pools.back().get();
        }
        pack_group(rc, G);
        std::string e = stage_group(rc, G, DEPTH_CAP0, TRAIL_CAP0, true);
        if (!e.empty()) return fail(OOB_E_CUDA, e);
    }
    for (auto& G : p->groups)
        for (int w = 0; w < NJOBS; w++)
            if (present(G.job[w])) {
                cudaSetDevice(phys_dev(G.dev));
                if (cudaStreamSynchronize(G.pool[w]->stream) != cudaSuccess)
                    return fail(OOB_E_CUDA, cudaGetErrorString(cudaGetLastError()));
            }
    *out = p.release();
    return OOB_OK;
}

int oob_plan_create(const oob_batch* batch, const oob_options* opt, oob_plan** out) {
    if (!out) return fail(OOB_E_INVALID, "null plan pointer");
    int rc = plan_create_once(batch, opt, out);
    if (rc == OOB_E_CUDA && g_last_error.find("out of memory") != std::string::npos) {
        // the solve paths' pooled buffers (stream workers keep theirs
        // between calls) make room for the plan's own
        cudaGetLastError();
        for (int s = 0; s < 4; s++) release_slot_pools(s);
        rc = plan_create_once(batch, opt, out);
    }
    return rc;
}

int oob_plan_run(oob_plan* p, float* device_ms) {
    if (!p) return fail(OOB_E_INVALID, "null plan");
    // every device's groups are launched back to back and overlap
    for (auto& G : p->groups) {
        std::string e = launch_group(p->rc, G);
        if (!e.empty()) return fail(OOB_E_CUDA, e);
    }
    float worst = 0;
    for (auto& G : p->groups) {
        float ms = 0;
        std::string e = group_ms(G, &ms);
        if (!e.empty()) return fail(OOB_E_CUDA, e);
        worst = std::max(worst, ms);
    }
    p->runs++;
    if (device_ms) *device_ms = worst;
    return OOB_OK;
}

int oob_plan_results(oob_plan* p, oob_result* out) {
    if (!p || !out || !out->verdict) return fail(OOB_E_INVALID, "null argument");
    if (p->runs == 0) {
        int rc0 = oob_plan_run(p, nullptr);
        if (rc0 != OOB_OK) return rc0;
    }
    RunCtx& rc = p->rc;
    for (auto& G : p->groups) {
        std::vector<int64_t> retry[3];
        std::string e = fetch_group(rc, G, retry);
        if (!e.empty()) return fail(OOB_E_CUDA, e);
        if (!retry[0].empty() || !retry[1].empty() || !retry[2].empty()) {
            e = run_group(rc, G.dev, retry);
            if (!e.empty()) return fail(OOB_E_CUDA, e);
        }
    }
    int64_t n = p->b->n_queries;
    for (int64_t q = 0; q < n; q++) {
        out->verdict[q] = p->verdict[q];
        if (out->nodes) out->nodes[q] = p->nodes[q];
        if (out->passes) out->passes[q] = p->passes[q];
        if (out->elapsed_s) out->elapsed_s[q] = p->elapsed[q];
        if (out->model && p->verdict[q] == OOB_SAT)
            for (int64_t v = p->b->var_begin[q]; v < p->b->var_begin[q + 1]; v++) out->model[v] = p->model[v];
    }
    return finish(p->pr, n);
}

int oob_plan_info(const oob_plan* p, int64_t info[9]) {
    if (!p || !info) return fail(OOB_E_INVALID, "null argument");
    int64_t nq = 0, rec = 0, res = 0, cls = 0, wide = 0, jobs = 0, launches = 0, h2d = 0;
    for (auto& G : p->groups) {
        if (p->rc.raw)  // the raw values and literal sources, once per device
            h2d += (int64_t)(p->rc.raw_nv * 2 + p->rc.raw_nl) * 8 + (int64_t)p->rc.litsrc->size() * 4;
        for (int w = 0; w < NJOBS; w++) {
            const DevJob& j = G.job[w];
            if (!present(j)) continue;
            h2d += (int64_t)(j.qd.size() * sizeof(QDesc) + 2 * j.cls.size() * sizeof(ClassDesc) + j.code.size() * 4 +
                             j.qs.size() * 4 + (j.slot[0].size() + j.slot[1].size() + j.slot[2].size()) * 4) +
                   (j.dev_fill ? (int64_t)j.qs.size() * 16 : (j.wide == W_X32 ? 0 : (int64_t)j.data_words * 8));
            int64_t own = 0;
            for (uint8_t sh : j.is_shadow) own += !sh;
            nq += own;
            rec += (int64_t)j.record_bytes();
            // bytes copied back per run: verdict, error, nodes, passes, elapsed per
            // entry, plus the models (SOLVE: only the Sat ones, packed, with a
            // 4-byte offset per entry)
            res += (int64_t)j.qs.size() * (1 + 1 + 8 + 8 + 4) +
                   (j.last_sat_vars >= 0 ? (int64_t)j.qs.size() * 4 + j.last_sat_vars * 16
                                         : (int64_t)j.out_model_words * 8);
            cls += j.n_classes;
            if (w == 1 || w == 2) wide += own;
            jobs++;
            launches += 1 + (int64_t)j.jit_cls.size() + (j.tail_blocks ? 1 : 0) +
                        ((!j.slot[0].empty() || !j.slot[1].empty() || !j.slot[2].empty()) ? 1 : 0) +
                        (j.a.certs && j.a.cert_kmax ? (j.a.cert_kmax > 1 ? 2 : 1) : 0) +  // fast mode: certificates
                        (j.a.enum_n ? 1 : 0) + (j.a.chain_n ? 1 : 0);  // fast mode: enumeration, (opt-in) search
        }
    }
    info[0] = nq;
    info[1] = rec;
    info[2] = res;
    info[3] = cls;
    info[4] = jobs;
    info[5] = launches;  // kernel launches per run
    info[6] = wide;
    info[7] = (int64_t)(p->pr.compile_s * 1e6);
    info[8] = h2d;
    return OOB_OK;
}

void oob_plan_destroy(oob_plan* p) { plan_free(p); }

// Host-side self-test of the 256-bit regime arithmetic (tests/test_wide.py
// compares it with Python integers).  op: 0 + 1 - 2 * 3 / 4 % 5 < 6 >>1
int oob_selftest_i256(int op, const int64_t* a, const int64_t* b, int64_t* out) {
    i256 x, y;
    for (int i = 0; i < 4; i++) {
        x.w[i] = (uint64_t)a[i];
        y.w[i] = (uint64_t)b[i];
    }
    i256 r(0);
    switch (op) {
    case 0: r = x + y; break;
    case 1: r = x - y; break;
    case 2: r = x * y; break;
    case 3: r = x / y; break;
    case 4: r = x % y; break;
    case 5: r = i256(x < y ? 1 : 0); break;
    case 6: r = x >> 1; break;
    default: return fail(OOB_E_INVALID, "unknown self-test op");
    }
    for (int i = 0; i < 4; i++) out[i] = (int64_t)r.w[i];
    return OOB_OK;
}

const char* oob_last_error(void) { return g_last_error.c_str(); }

int oob_device_count(void) { return visible_devices(); }

const char* oob_version(void) { return "scuba-oob-b200 0.1 (sm_100a)"; }

void oob_release(void) {
    for (int s = 0; s < 4; s++) release_slot_pools(s);
}

}  // extern "C"
