// sweep_vm.cuh -- interpreter of the MiniCUDA sweep bytecode (sweep.py),
// one input tuple per thread.  Restates the reference's AST interpreter
// (/root/reference/pkg/src/scuba_mini/oracle.py:160-580) over a flat program:
//
//  * the whole execution of one tuple -- host statements, and for every
//    launch each block (z, y, x; x fastest) and each thread of it in the same
//    order (oracle.py:555-567) -- runs sequentially in one thread;
//  * memory: a per-thread arena of int64 cells.  Host allocations and
//    per-thread local arrays grow from the bottom (released at thread end),
//    block-shared storages from the top (released at block end).  Cells start
//    at 0 (oracle.py:13); reads outside the backing storage yield 0, writes
//    there are discarded (oracle.py:181-203);
//  * views: (storage, start, end, row_len).  A partition ends the previous
//    partition of the same storage created by the same thread (oracle.py:446-455);
//  * violations are recorded per access site as label bits and only kept
//    when the execution does not halt (oracle.py:660-667).
//
// Compiled for the device (csrc/sweep.cu) and, for CPU unit tests only, for
// the host (tests/native/sweep_host.cpp); SW_HD marks the shared code.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define SW_HD __host__ __device__ __forceinline__
#else
#define SW_HD inline
#endif

namespace sweep {

enum Op {
    LIT, LD, INP, BLT, BIN, RD, CMP, ST, JZ, JMP, ASRT, MALLOC, FREE, WR, ATOM, RET,
    XSHM, ADECL, PART, NNEG, PARG, LAUNCH, KEND, END
};
enum Status { S_OK = 0, S_HALT = 1, S_NEED = 2, S_ERROR = 3 };
enum Err {
    E_NONE = 0, E_OVERFLOW, E_ARENA, E_VIEWS, E_STORAGES, E_STACK, E_ROWLEN, E_STEPS, E_PROGRAM
};
enum Halt { H_ALLOC = 1, H_ASSERT, H_DIV0, H_STORE, H_DIM, H_SHM, H_ARG };
enum Label { L_UPPER = 1, L_UNDER = 2, L_UAF = 4, L_DFREE = 8 };

constexpr int MAX_SLOTS = 96;
constexpr int MAX_VIEWS = 64;
constexpr int MAX_STOR = 32;
constexpr int MAX_STACK = 32;
constexpr int MAX_SITES = 64;
constexpr int MAX_SHARED = 8;
constexpr int MAX_KPARAMS = 16;
constexpr int MAX_INPUTS = 8;
constexpr int LABEL_WORDS = MAX_SITES * 4 / 32;

struct Prog {
    const int32_t* code;    // [n_code][4]
    const int64_t* lits;
    const int32_t* kernels; // [n_kernels][4]: entry, n_params, kparam offset, n_shared
    const int32_t* kparams; // [n][2]: slot, kind
    int32_t n_code, n_sites, n_slots, n_kernels;
    int64_t step_limit;
};

// cell w of this thread lives at base[w * stride] (lane-interleaved arena:
// lanes of a warp touching the same cell index hit consecutive words)
struct Arena {
    int64_t* base;
    int64_t stride;
    int64_t words;
};

struct Machine {
    int64_t slot[MAX_SLOTS];
    int64_t stk[MAX_STACK];
    int64_t vstart[MAX_VIEWS], vend[MAX_VIEWS], vrow[MAX_VIEWS];
    int32_t vstor[MAX_VIEWS];
    int64_t sbase[MAX_STOR], ssize[MAX_STOR];
    int32_t sfreed[MAX_STOR];
    int32_t lp_view[MAX_STOR];
    uint32_t lp_gen[MAX_STOR];
    int32_t shared_sid[MAX_SHARED];
    int64_t pval[MAX_KPARAMS];
    uint32_t labels[LABEL_WORDS];
    int64_t arena_peak;
};

struct Out {
    int status;  // Status
    int aux;     // halt code / needed input site / error code
};

SW_HD bool add_ovf(int64_t a, int64_t b, int64_t* r) {
    uint64_t u = (uint64_t)a + (uint64_t)b;
    *r = (int64_t)u;
    return ((a ^ *r) & (b ^ *r)) < 0;
}
SW_HD bool sub_ovf(int64_t a, int64_t b, int64_t* r) {
    uint64_t u = (uint64_t)a - (uint64_t)b;
    *r = (int64_t)u;
    return ((a ^ b) & (a ^ *r)) < 0;
}
SW_HD bool mul_ovf(int64_t a, int64_t b, int64_t* r) {
    __int128 p = (__int128)a * (__int128)b;
    *r = (int64_t)p;
    return p != (__int128)*r;
}

// Runs one execution.  inputs[0..arity) are the __input() values.
SW_HD Out run(const Prog& P, const int64_t* inputs, int arity, const Arena& A, Machine& m) {
    const int32_t* code = P.code;
    int64_t* stk = m.stk;
    int sp = 0, pc = 0;
    int nv = 0, ns = 0;
    int64_t bot = 0, top = A.words;
    uint32_t gen = 1;
    int64_t steps = 0;
    // builtins: tid xyz, bid xyz, bdim xyz, gdim xyz
    int64_t bi[12];
    for (int i = 0; i < 12; i++) bi[i] = 0;
    // launch state
    int kern = -1, ret_pc = 0, kentry = 0, knp = 0, kpoff = 0, kshared = 0;
    int host_nv = 0, launch_nv = 0, launch_ns = 0, thread_nv = 0, thread_ns = 0;
    int64_t launch_bot = 0;
    for (int s = 0; s < MAX_STOR; s++) m.lp_gen[s] = 0;
    for (int w = 0; w < LABEL_WORDS; w++) m.labels[w] = 0;
    m.arena_peak = 0;

    Out o{S_OK, 0};
#define SW_FAIL(st, code_) do { o.status = (st); o.aux = (code_); return o; } while (0)
#define SW_PUSH(v) do { if (sp >= MAX_STACK) SW_FAIL(S_ERROR, E_STACK); stk[sp++] = (v); } while (0)
#define CELL(w) A.base[(w) * A.stride]

    // shared storages use the ids reserved at block start (sid_out preset)
    auto new_storage = [&](int64_t size, bool shared, int64_t* sid_out) -> int {
        if (!shared && ns >= MAX_STOR) return E_STORAGES;
        if (size > top - bot) return E_ARENA;
        int64_t base;
        if (shared) {
            top -= size;
            base = top;
        } else {
            base = bot;
            bot += size;
        }
        int64_t used = bot + (A.words - top);
        if (used > m.arena_peak) m.arena_peak = used;
        for (int64_t w = 0; w < size; w++) CELL(base + w) = 0;
        int64_t id = shared ? *sid_out : ns++;
        m.sbase[id] = base;
        m.ssize[id] = size;
        m.sfreed[id] = 0;
        *sid_out = id;
        return 0;
    };
    auto new_view = [&](int sid, int64_t start, int64_t end, int64_t row, int64_t* vid) -> int {
        if (nv >= MAX_VIEWS) return E_VIEWS;
        m.vstor[nv] = sid;
        m.vstart[nv] = start;
        m.vend[nv] = end;
        m.vrow[nv] = row;
        *vid = nv++;
        return 0;
    };
    auto start_thread = [&]() {
        nv = thread_nv;
        ns = thread_ns;
        bot = launch_bot;
        for (int i = 0; i < knp; i++) m.slot[P.kparams[2 * (kpoff + i)]] = m.pval[i];
        gen++;
        pc = kentry;
    };
    auto start_block = [&]() {
        // block-shared storages: ids reserved per declaration, created lazily
        nv = launch_nv;
        top = A.words;
        for (int d = 0; d < kshared; d++) m.shared_sid[d] = -1;
        thread_nv = nv;
        thread_ns = launch_ns + kshared;
        bi[0] = bi[1] = bi[2] = 0;
    };

    for (;;) {
        if (++steps > P.step_limit) SW_FAIL(S_ERROR, E_STEPS);
        if (pc < 0 || pc >= P.n_code) SW_FAIL(S_ERROR, E_PROGRAM);
        const int32_t* ins = code + 4 * pc;
        const int op = ins[0], a = ins[1], b = ins[2], c = ins[3];
        pc++;
        switch (op) {
        case LIT: SW_PUSH(P.lits[a]); break;
        case LD: SW_PUSH(m.slot[a]); break;
        case INP:
            if (a >= arity) SW_FAIL(S_NEED, a);
            SW_PUSH(inputs[a]);
            break;
        case BLT: SW_PUSH(bi[a]); break;
        case BIN: {
            int64_t y = stk[--sp], x = stk[--sp], r = 0;
            bool ovf = false;
            switch (a) {
            case 0: ovf = add_ovf(x, y, &r); break;
            case 1: ovf = sub_ovf(x, y, &r); break;
            case 2: ovf = mul_ovf(x, y, &r); break;
            default:  // C truncation (solver.tdiv / tmod, oracle.py:214-229)
                if (y == 0) SW_FAIL(S_HALT, H_DIV0);
                if (x == INT64_MIN && y == -1) {
                    if (a == 3) ovf = true;
                    r = 0;
                } else {
                    r = a == 3 ? x / y : x % y;
                }
            }
            if (ovf) SW_FAIL(S_ERROR, E_OVERFLOW);
            stk[sp++] = r;
            break;
        }
        case CMP: {
            int64_t y = stk[--sp], x = stk[--sp];
            bool r = a == 0 ? x < y : a == 1 ? x <= y : a == 2 ? x > y : a == 3 ? x >= y : x == y;
            stk[sp++] = r;
            break;
        }
        case ST: m.slot[a] = stk[--sp]; break;
        case JZ:
            if (stk[--sp] == 0) pc = a;
            break;
        case JMP: pc = a; break;
        case ASRT:
            if (stk[--sp] == 0) SW_FAIL(S_HALT, H_ASSERT);
            break;
        case NNEG:
            for (int i = 1; i <= a; i++)
                if (stk[sp - i] < 0) SW_FAIL(S_HALT, c);
            break;
        case MALLOC: {  // oracle.py:336-346
            int64_t size = stk[--sp], sid, vid;
            if (size < 0) SW_FAIL(S_HALT, H_ALLOC);
            int e = new_storage(size, false, &sid);
            if (e) SW_FAIL(S_ERROR, e);
            e = new_view((int)sid, 0, size, -1, &vid);
            if (e) SW_FAIL(S_ERROR, e);
            m.slot[a] = vid;
            break;
        }
        case FREE: {  // oracle.py:347-362
            int s = m.vstor[m.slot[a]];
            if (m.sfreed[s]) m.labels[(b * 4) >> 5] |= (uint32_t)L_DFREE << ((b * 4) & 31);
            m.sfreed[s] = 1;
            break;
        }
        case RD: case WR: case ATOM: {  // oracle.py:162-204, 295-316, 400-420, 462-484
            int64_t value = 0;
            if (op != RD) value = stk[--sp];
            int ndims = op == ATOM ? 1 : c;
            int64_t off;
            int v = (int)m.slot[a];
            if (ndims == 2) {
                int64_t j = stk[--sp], i = stk[--sp], t;
                if (m.vrow[v] < 0) SW_FAIL(S_ERROR, E_ROWLEN);
                if (mul_ovf(i, m.vrow[v], &t) || add_ovf(t, j, &off)) SW_FAIL(S_ERROR, E_OVERFLOW);
            } else {
                off = stk[--sp];
            }
            int s = m.vstor[v];
            int64_t extent = m.vend[v] - m.vstart[v];
            uint32_t lab = m.sfreed[s] ? L_UAF : off < 0 ? L_UNDER : off >= extent ? L_UPPER : 0;
            if (lab) m.labels[(b * 4) >> 5] |= lab << ((b * 4) & 31);
            int64_t absol;
            if (add_ovf(m.vstart[v], off, &absol)) SW_FAIL(S_ERROR, E_OVERFLOW);
            bool in = absol >= 0 && absol < m.ssize[s] && !m.sfreed[s];
            if (op == RD) {
                SW_PUSH(in ? CELL(m.sbase[s] + absol) : 0);
            } else {
                if (value < 0) SW_FAIL(S_HALT, H_STORE);
                if (in) {
                    int64_t& cell = CELL(m.sbase[s] + absol);
                    if (op == WR) {
                        cell = value;
                    } else if (c == 0) {
                        int64_t r;
                        if (add_ovf(cell, value, &r)) SW_FAIL(S_ERROR, E_OVERFLOW);
                        cell = r;
                    } else if (c == 1) {
                        cell = value < cell ? value : cell;
                    } else {
                        cell = value > cell ? value : cell;
                    }
                }
            }
            break;
        }
        case XSHM: {  // oracle.py:427-438
            int64_t sid = m.shared_sid[b], vid;
            if (sid < 0) {
                sid = launch_ns + b;
                int e = new_storage(m.pval[MAX_KPARAMS - 1], true, &sid);
                if (e) SW_FAIL(S_ERROR, e);
                m.shared_sid[b] = (int32_t)sid;
            }
            int e = new_view((int)sid, 0, m.ssize[sid], -1, &vid);
            if (e) SW_FAIL(S_ERROR, e);
            m.slot[a] = vid;
            break;
        }
        case ADECL: {  // oracle.py:486-508
            int nd = c & 3;
            bool shared = (c >> 2) & 1;
            int64_t s1 = nd == 2 ? stk[--sp] : 0;
            int64_t s0 = stk[--sp];
            if (s0 < 0 || (nd == 2 && s1 < 0)) SW_FAIL(S_HALT, H_ALLOC);
            int64_t total = s0, row = -1;
            if (nd == 2) {
                if (mul_ovf(s0, s1, &total)) SW_FAIL(S_ERROR, E_OVERFLOW);
                row = s1;
            }
            int64_t sid, vid;
            if (shared) {
                sid = m.shared_sid[b];
                if (sid < 0) {
                    sid = launch_ns + b;
                    int e = new_storage(total, true, &sid);
                    if (e) SW_FAIL(S_ERROR, e);
                    m.shared_sid[b] = (int32_t)sid;
                }
            } else {
                int e = new_storage(total, false, &sid);
                if (e) SW_FAIL(S_ERROR, e);
            }
            int e = new_view((int)sid, 0, total, row, &vid);
            if (e) SW_FAIL(S_ERROR, e);
            m.slot[a] = vid;
            break;
        }
        case PART: {  // oracle.py:441-457
            int64_t off = stk[--sp], start, vid;
            int bv = (int)m.slot[b];
            int s = m.vstor[bv];
            if (add_ovf(m.vstart[bv], off, &start)) SW_FAIL(S_ERROR, E_OVERFLOW);
            int e = new_view(s, start, m.ssize[s], -1, &vid);
            if (e) SW_FAIL(S_ERROR, e);
            if (m.lp_gen[s] == gen) m.vend[m.lp_view[s]] = start;
            m.lp_gen[s] = gen;
            m.lp_view[s] = (int32_t)vid;
            m.slot[a] = vid;
            break;
        }
        case PARG: SW_PUSH(m.vstor[m.slot[a]]); break;
        case LAUNCH: {  // oracle.py:512-567
            const int32_t* K = P.kernels + 4 * a;
            kentry = K[0];
            knp = b;
            kpoff = K[2];
            kshared = K[3];
            if (knp > MAX_KPARAMS - 1 || kshared > MAX_SHARED) SW_FAIL(S_ERROR, E_PROGRAM);
            int64_t args[MAX_KPARAMS];
            for (int i = knp - 1; i >= 0; i--) args[i] = stk[--sp];
            int64_t shm = stk[--sp];
            int64_t dims[6];
            for (int i = 5; i >= 0; i--) dims[i] = stk[--sp];
            host_nv = nv;
            launch_ns = ns;
            launch_bot = bot;
            if (ns + kshared > MAX_STOR) SW_FAIL(S_ERROR, E_STORAGES);
            for (int i = 0; i < knp; i++) {
                if (P.kparams[2 * (kpoff + i) + 1]) {  // pointer: View(storage, 0, size)
                    int sid = (int)args[i];
                    int64_t vid;
                    int e = new_view(sid, 0, m.ssize[sid], -1, &vid);
                    if (e) SW_FAIL(S_ERROR, e);
                    m.pval[i] = vid;
                } else {
                    m.pval[i] = args[i];
                }
            }
            m.pval[MAX_KPARAMS - 1] = shm;
            launch_nv = nv;
            for (int i = 0; i < 3; i++) {
                bi[9 + i] = dims[i];
                bi[6 + i] = dims[3 + i];
            }
            ret_pc = pc;
            bool empty = false;
            for (int i = 0; i < 6; i++) empty |= dims[i] == 0;
            if (empty) {  // no block runs: nothing observable but the argument checks
                nv = host_nv;
                break;
            }
            kern = a;
            start_block();
            bi[3] = bi[4] = bi[5] = 0;
            start_thread();
            break;
        }
        case RET:
        case KEND: {
            if (kern < 0) SW_FAIL(S_ERROR, E_PROGRAM);
            if (++bi[0] < bi[6]) { start_thread(); break; }
            bi[0] = 0;
            if (++bi[1] < bi[7]) { start_thread(); break; }
            bi[1] = 0;
            if (++bi[2] < bi[8]) { start_thread(); break; }
            // block done
            int64_t keep[3] = {bi[3], bi[4], bi[5]};
            bool more = true;
            if (++keep[0] >= bi[9]) {
                keep[0] = 0;
                if (++keep[1] >= bi[10]) {
                    keep[1] = 0;
                    if (++keep[2] >= bi[11]) more = false;
                }
            }
            if (more) {
                start_block();
                bi[3] = keep[0];
                bi[4] = keep[1];
                bi[5] = keep[2];
                start_thread();
                break;
            }
            // launch done: release the launch's views/storages, back to host code
            nv = host_nv;
            ns = launch_ns;
            bot = launch_bot;
            top = A.words;
            kern = -1;
            gen++;
            pc = ret_pc;
            break;
        }
        case END: return o;
        default: SW_FAIL(S_ERROR, E_PROGRAM);
        }
    }
#undef SW_FAIL
#undef SW_PUSH
#undef CELL
}

}  // namespace sweep
