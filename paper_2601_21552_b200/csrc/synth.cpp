// synth.cpp -- seeded generator of analyzer-shaped OOB queries
// (include/scuba_oob_synth.h).  Emits exactly the constraint sequence the
// reference analyzer builds for an access (constraint_gen.py):
//   declare_geometry  :105-124  12 vars, 12 range constraints, 6 launch eqs
//   check             :297-302  solOffset [-M, M], solSize [0, M]
//   offset/size eqs   :303-306  (loop variables declared on first sight with
//                               their two bound constraints, :155-164)
//   add_context       :186-208  param bindings, host asserts, guards
// Variables are declared in first-appearance order, like _SetBuilder.var.
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/scuba_oob_synth.h"

namespace {

using i128 = __int128;

struct Rng {
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {  // splitmix64
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    int64_t uni(int64_t lo, int64_t hi) {
        if (hi < lo) hi = lo;
        return lo + (int64_t)(next() % (uint64_t)(hi - lo + 1));
    }
    bool chance(int pct) { return (int)(next() % 100) < pct; }
};

// ---- expression trees of the program (the analyzer's ETs) -------------------
enum EK { CONST, BUILTIN, UNK, LOOP, BIN };
struct Et {
    EK k;
    int64_t v;   // CONST value / BUILTIN axis / UNK id / LOOP id
    char op;     // BIN
    int l, r;    // BIN children; LOOP: lower, upper bound ETs
};

enum Axis { TidX, TidY, TidZ, BidX, BidY, BidZ, GDimX, GDimY, GDimZ, BDimX, BDimY, BDimZ };

struct Prog {
    std::vector<Et> e;
    int c(int64_t v) { e.push_back({CONST, v, 0, 0, 0}); return (int)e.size() - 1; }
    int b(int axis) { e.push_back({BUILTIN, axis, 0, 0, 0}); return (int)e.size() - 1; }
    int u(int id) { e.push_back({UNK, id, 0, 0, 0}); return (int)e.size() - 1; }
    int loop(int id, int lo, int hi) { e.push_back({LOOP, id, 0, lo, hi}); return (int)e.size() - 1; }
    int bin(char op, int l, int r) { e.push_back({BIN, 0, op, l, r}); return (int)e.size() - 1; }
    int add(int l, int r) { return bin('+', l, r); }
    int sub(int l, int r) { return bin('-', l, r); }
    int mul(int l, int r) { return bin('*', l, r); }
    int div(int l, int r) { return bin('/', l, r); }
};

struct Cmp {
    int rel;  // OOB_REL_*
    int l, r;
};

struct Access {
    int grid[6];                                 // GDimX..Z, BDimX..Z
    int offset = -1, size = -1;                  // -1: layout check
    int later = -1, earlier = -1;                // layout check operands
    std::vector<std::pair<int, int>> params;     // (param unknown id, arg ET)
    std::vector<Cmp> asserts, guards;
};

// ---- query builder (the analyzer's _SetBuilder) -------------------------------
struct QB {
    i128 M;
    const Prog& p;
    std::vector<int> var_code;
    std::vector<i128> vlo, vhi;
    std::vector<uint8_t> rel;
    std::vector<int32_t> lhs, rhs;
    std::vector<uint8_t> op;
    std::vector<int32_t> na, nb;
    std::vector<i128> lits;
    std::vector<int> loops_seen;
    QB(i128 m, const Prog& pr) : M(m), p(pr) {}

    int var(int code, i128 lo, i128 hi) {
        int idx = -1;
        for (size_t i = 0; i < var_code.size(); i++)
            if (var_code[i] == code) idx = (int)i;
        if (idx < 0) {
            idx = (int)var_code.size();
            var_code.push_back(code);
            vlo.push_back(lo);
            vhi.push_back(hi);
        }
        op.push_back(OOB_NODE_VAR);
        na.push_back(idx);
        nb.push_back(0);
        return (int)op.size() - 1;
    }
    int var(int code) { return var(code, 0, M); }
    int lit(i128 v) {
        lits.push_back(v);
        op.push_back(OOB_NODE_LIT);
        na.push_back((int)lits.size() - 1);
        nb.push_back(0);
        return (int)op.size() - 1;
    }
    int bin(char c, int l, int r) {
        uint8_t code = c == '+' ? OOB_NODE_ADD : c == '-' ? OOB_NODE_SUB : c == '*' ? OOB_NODE_MUL
                     : c == '/' ? OOB_NODE_DIV : OOB_NODE_MOD;
        op.push_back(code);
        na.push_back(l);
        nb.push_back(r);
        return (int)op.size() - 1;
    }
    void con(int r, int l, int rr) {
        rel.push_back((uint8_t)r);
        lhs.push_back(l);
        rhs.push_back(rr);
    }
    // translate (constraint_gen.py:142-173): left before right; loop vars are
    // declared on first sight and their bounds appended immediately.
    int tr(int id) {
        const Et& x = p.e[id];
        switch (x.k) {
        case CONST: return lit(x.v);
        case BUILTIN: return var((int)x.v);
        case UNK: return var(14 + (int)x.v);
        case LOOP: {
            int ref = var(14 + (int)x.v);
            bool seen = false;
            for (int s : loops_seen) seen = seen || s == x.v;
            if (!seen) {
                loops_seen.push_back((int)x.v);
                int lo = tr(x.l);
                int hi = tr(x.r);
                con(OOB_REL_GE, var(14 + (int)x.v), lo);
                con(OOB_REL_LT, var(14 + (int)x.v), hi);
            }
            return ref;
        }
        default: {
            int l = tr(x.l);
            int r = tr(x.r);
            return bin(x.op, l, r);
        }
        }
    }
    void cmp(const Cmp& c) {
        int l = tr(c.l);
        int r = tr(c.r);
        con(c.rel, l, r);
    }
};

// check: 0 upper, 1 lower, 2 layout
void build_query(const Access& a, const Prog& p, int check, i128 M, QB& q) {
    // declare_geometry (:105-124)
    for (int ax = 0; ax < 12; ax++) q.var(ax);
    q.op.clear(); q.na.clear(); q.nb.clear();  // declaration-only nodes are not needed
    static const int pairs[6][2] = {{TidX, BDimX}, {TidY, BDimY}, {TidZ, BDimZ},
                                    {BidX, GDimX}, {BidY, GDimY}, {BidZ, GDimZ}};
    for (auto& pr : pairs) {
        q.con(OOB_REL_GE, q.var(pr[0]), q.lit(0));
        q.con(OOB_REL_LT, q.var(pr[0]), q.var(pr[1]));
    }
    for (int g = 0; g < 6; g++) {
        int axv = q.var(GDimX + g);
        int et = q.tr(a.grid[g]);
        q.con(OOB_REL_EQ, axv, et);
    }
    if (check == 2) {
        int l = q.tr(a.later);
        int r = q.tr(a.earlier);
        q.con(OOB_REL_LT, l, r);
    } else {
        int off = q.var(12, -M, M);
        int size = q.var(13, 0, M);
        if (check == 0) q.con(OOB_REL_GE, off, size);
        else q.con(OOB_REL_LT, off, q.lit(0));
        int oe = q.tr(a.offset);
        q.con(OOB_REL_EQ, q.var(12, -M, M), oe);
        int se = q.tr(a.size);
        q.con(OOB_REL_EQ, q.var(13, 0, M), se);
    }
    // add_context (:186-208)
    for (auto& pa : a.params) {
        int pv = q.var(14 + pa.first);
        int av = q.tr(pa.second);
        q.con(OOB_REL_EQ, pv, av);
    }
    for (auto& c : a.asserts) q.cmp(c);
    for (auto& c : a.guards) q.cmp(c);
}

// ---- templates ---------------------------------------------------------------
struct Cfg {
    int config;
    i128 M;
    int kmin, kmax;   // input caps 2^k
    int bug_pct;
    int cap_log2;     // C5 override
};

int pick_blk(Rng& r) { return 8 << r.uni(0, 6); }  // 8..512

// T1 linear 1-D (saxpy / copy_guarded)
void t1(Prog& p, Access& a, Rng& r, const Cfg& c, bool bug) {
    int blk = pick_blk(r);
    int64_t cap = (int64_t)1 << r.uni(c.kmin, c.kmax);
    int kind = bug ? (int)r.uni(1, 4) : 0;
    int n = p.u(1);
    a.grid[0] = p.div(p.add(p.u(1), p.c(blk - 1)), p.c(blk));
    a.grid[1] = p.c(1); a.grid[2] = p.c(1);
    a.grid[3] = p.c(blk); a.grid[4] = p.c(1); a.grid[5] = p.c(1);
    int idx = p.add(p.b(TidX), p.mul(p.b(BidX), p.b(BDimX)));
    a.offset = kind == 3 ? p.add(idx, p.c(1)) : idx;
    a.size = kind == 4 ? p.sub(n, p.c(1)) : n;
    a.params.push_back({2, p.u(1)});
    a.asserts.push_back({OOB_REL_GE, p.u(1), p.c(1)});
    a.asserts.push_back({OOB_REL_LE, p.u(1), p.c(cap)});
    int gidx = p.add(p.b(TidX), p.mul(p.b(BidX), p.b(BDimX)));
    if (kind == 2) a.guards.push_back({OOB_REL_LE, gidx, p.u(2)});
    else if (kind != 1) a.guards.push_back({OOB_REL_LT, gidx, p.u(2)});
}

// T2 constant static extents (static_shared_oob / fluid_adv kernel side)
void t2(Prog& p, Access& a, Rng& r, const Cfg& c, bool bug) {
    int bx = 1 << r.uni(2, 5), by = 1 << r.uni(0, 4);
    int64_t cap = (int64_t)1 << r.uni(c.kmin, c.kmax);
    int kind = bug ? (int)r.uni(1, 2) : 0;
    a.grid[0] = p.u(1);
    a.grid[1] = p.c(1); a.grid[2] = p.c(1);
    a.grid[3] = p.c(bx); a.grid[4] = p.c(kind == 2 ? by + 1 : by); a.grid[5] = p.c(1);
    a.offset = p.add(p.mul(p.b(TidY), p.c(kind == 1 ? bx + 1 : bx)), p.b(TidX));
    a.size = p.c((int64_t)bx * by);
    a.asserts.push_back({OOB_REL_GE, p.u(1), p.c(1)});
    a.asserts.push_back({OOB_REL_LE, p.u(1), p.c(cap)});
}

// T3 product sizes (fluid_adv): size (c+1)^3 * N * K
void t3(Prog& p, Access& a, Rng& r, const Cfg& c, bool bug) {
    int capc = (int)r.uni(1, c.config == OOB_SYNTH_C4 ? 15 : 7);
    int64_t capn = (int64_t)1 << r.uni(c.kmin, c.kmax);
    int64_t K = bug ? (int64_t)r.uni(3, 255) : 256;
    a.grid[0] = p.u(2);
    a.grid[1] = p.c(1); a.grid[2] = p.c(1);
    a.grid[3] = p.c(16); a.grid[4] = p.c(16); a.grid[5] = p.c(1);
    a.offset = p.add(p.add(p.mul(p.b(BidX), p.c(256)), p.mul(p.b(TidY), p.c(16))), p.b(TidX));
    int cp1 = p.add(p.u(1), p.c(1));
    int cube = p.mul(p.mul(cp1, p.add(p.u(1), p.c(1))), p.add(p.u(1), p.c(1)));
    a.size = p.mul(p.mul(cube, p.u(2)), p.c(K));
    a.params.push_back({3, p.u(2)});
    a.asserts.push_back({OOB_REL_LE, p.u(1), p.c(capc)});
    a.asserts.push_back({OOB_REL_GE, p.u(2), p.c(1)});
    a.asserts.push_back({OOB_REL_LE, p.u(2), p.c(capn)});
}

// T4 loop-variable bounded (kalman): a[tid * n + i], i < n, size T * n
void t4(Prog& p, Access& a, Rng& r, const Cfg& c, bool bug) {
    int kmax = c.config == OOB_SYNTH_C4 ? 7 : c.kmax;
    int64_t capt = (int64_t)1 << r.uni(c.kmin, kmax);
    int64_t capn = (int64_t)1 << r.uni(c.kmin > 3 ? c.kmin - 2 : 2, kmax - 2);
    int kind = bug ? (int)r.uni(1, 2) : 0;
    a.grid[0] = p.c(1); a.grid[1] = p.c(1); a.grid[2] = p.c(1);
    a.grid[3] = p.u(1); a.grid[4] = p.c(1); a.grid[5] = p.c(1);
    int upper = kind == 1 ? p.add(p.u(3), p.c(1)) : p.u(3);
    int i = p.loop(4, p.c(0), upper);
    a.offset = p.add(p.mul(p.b(TidX), p.u(3)), i);
    a.size = kind == 2 ? p.sub(p.mul(p.u(1), p.u(2)), p.c(1)) : p.mul(p.u(1), p.u(2));
    a.params.push_back({3, p.u(2)});
    a.asserts.push_back({OOB_REL_GE, p.u(1), p.c(1)});
    a.asserts.push_back({OOB_REL_LE, p.u(1), p.c(capt)});
    a.asserts.push_back({OOB_REL_GE, p.u(2), p.c(1)});
    a.asserts.push_back({OOB_REL_LE, p.u(2), p.c(capn)});
}

// T5 dynamic-shared partitions (sosfilt_intra); check 2 = layout pre-check
void t5(Prog& p, Access& a, Rng& r, const Cfg& c, bool bug, bool layout) {
    int64_t caps = (int64_t)1 << r.uni(c.kmin > 3 ? c.kmin - 2 : 2, c.kmax - 3 > 2 ? c.kmax - 3 : 3);
    int64_t capw = (int64_t)1 << r.uni(c.kmin > 3 ? c.kmin - 2 : 2, c.kmax - 3 > 2 ? c.kmax - 3 : 3);
    a.grid[0] = p.c(1); a.grid[1] = p.c(1); a.grid[2] = p.c(1);
    a.grid[3] = p.u(1); a.grid[4] = p.c(1); a.grid[5] = p.c(1);
    if (layout) {
        // later partition s + s*w (+ bug: s*w - s) vs earlier s
        a.later = bug ? p.sub(p.mul(p.u(3), p.u(4)), p.u(3)) : p.add(p.u(3), p.mul(p.u(3), p.u(4)));
        a.earlier = p.u(3);
    } else {
        int i = p.loop(5, p.c(0), p.u(4));
        int base = p.add(p.mul(p.b(TidX), p.u(4)), i);
        a.offset = bug ? p.add(base, p.c(1)) : base;
        a.size = p.mul(p.u(1), p.u(2));
    }
    a.params.push_back({3, p.u(1)});
    a.params.push_back({4, p.u(2)});
    a.asserts.push_back({OOB_REL_GE, p.u(1), p.c(1)});
    a.asserts.push_back({OOB_REL_LE, p.u(1), p.c(caps)});
    a.asserts.push_back({OOB_REL_GE, p.u(2), p.c(1)});
    a.asserts.push_back({OOB_REL_LE, p.u(2), p.c(capw)});
}

// T6 data-dependent unknown (push_node)
void t6(Prog& p, Access& a, Rng& r, const Cfg& c, bool bug) {
    int64_t capv = (int64_t)1 << r.uni(c.kmin, c.kmax);
    int64_t capd = (int64_t)1 << r.uni(1, 3);
    int blk = pick_blk(r);
    bool neighbor = r.chance(50);
    a.grid[0] = p.div(p.add(p.u(1), p.c(blk - 1)), p.c(blk));
    a.grid[1] = p.c(1); a.grid[2] = p.c(1);
    a.grid[3] = p.c(blk); a.grid[4] = p.c(1); a.grid[5] = p.c(1);
    int idx = p.add(p.b(TidX), p.mul(p.b(BidX), p.b(BDimX)));
    if (neighbor) {
        a.offset = p.u(6);  // value loaded from memory: unconstrained in [0, M]
        a.size = p.u(1);
    } else {
        int j = p.loop(5, p.c(0), p.u(4));
        a.offset = p.add(p.mul(idx, p.u(4)), j);
        a.size = p.mul(p.u(1), p.u(2));
    }
    a.params.push_back({3, p.u(1)});
    a.params.push_back({4, p.u(2)});
    a.asserts.push_back({OOB_REL_GE, p.u(1), p.c(1)});
    a.asserts.push_back({OOB_REL_LE, p.u(1), p.c(capv)});
    a.asserts.push_back({OOB_REL_GE, p.u(2), p.c(1)});
    a.asserts.push_back({OOB_REL_LE, p.u(2), p.c(capd)});
    if (!bug) {
        a.guards.push_back({OOB_REL_LT, p.add(p.b(TidX), p.mul(p.b(BidX), p.b(BDimX))), p.u(3)});
        if (neighbor) a.guards.push_back({OOB_REL_LT, p.u(6), p.u(3)});
    }
}

// T7 2-D row * dim + j (lu_decomp); underflow when row may be 0
void t7(Prog& p, Access& a, Rng& r, const Cfg& c, bool bug) {
    int kmax = c.config == OOB_SYNTH_C4 ? 5 : c.kmax - 1;
    int64_t cap = (int64_t)1 << r.uni(c.kmin > 3 ? c.kmin - 1 : 2, kmax);
    int blk = 8 << r.uni(0, 2);
    a.grid[0] = p.div(p.add(p.u(1), p.c(blk - 1)), p.c(blk));
    a.grid[1] = p.c(1); a.grid[2] = p.c(1);
    a.grid[3] = p.c(blk); a.grid[4] = p.c(1); a.grid[5] = p.c(1);
    int j = p.add(p.b(TidX), p.mul(p.b(BidX), p.b(BDimX)));
    a.offset = p.add(p.mul(p.sub(p.u(4), p.c(1)), p.u(3)), j);
    a.size = p.mul(p.u(1), p.u(1));
    a.params.push_back({3, p.u(1)});
    a.params.push_back({4, p.u(2)});
    a.asserts.push_back({OOB_REL_LE, p.u(1), p.c(cap)});
    a.asserts.push_back({OOB_REL_LT, p.u(2), p.u(1)});
    if (!bug) a.asserts.push_back({OOB_REL_GE, p.u(2), p.c(1)});
    a.guards.push_back({OOB_REL_LT, p.add(p.b(TidX), p.mul(p.b(BidX), p.b(BDimX))), p.u(3)});
}

// T8 (C4) 3-D linearisation ((z * ny + y) * nx + x), sizes nx * ny * nz
void t8(Prog& p, Access& a, Rng& r, const Cfg& c, bool bug) {
    int64_t cap = (int64_t)1 << r.uni(1, 3);
    int bx = 8 << r.uni(0, 2);
    a.grid[0] = p.div(p.add(p.u(1), p.c(bx - 1)), p.c(bx));
    a.grid[1] = p.u(2); a.grid[2] = p.u(3);
    a.grid[3] = p.c(bx); a.grid[4] = p.c(1); a.grid[5] = p.c(1);
    int x = p.add(p.b(TidX), p.mul(p.b(BidX), p.b(BDimX)));
    a.offset = p.add(p.mul(p.add(p.mul(p.b(BidZ), p.u(5)), p.b(BidY)), p.u(4)), x);
    a.size = p.mul(p.mul(p.u(1), p.u(2)), p.u(3));
    a.params.push_back({4, p.u(1)});
    a.params.push_back({5, p.u(2)});
    for (int k = 1; k <= 3; k++) {
        a.asserts.push_back({OOB_REL_GE, p.u(k), p.c(1)});
        a.asserts.push_back({OOB_REL_LE, p.u(k), p.c(cap)});
    }
    if (!bug) a.guards.push_back({OOB_REL_LT, p.add(p.b(TidX), p.mul(p.b(BidX), p.b(BDimX))), p.u(4)});
}

Cfg cfg_of(int config, uint64_t key, int cap_log2) {
    Cfg c;
    c.config = config;
    c.cap_log2 = cap_log2;
    switch (config) {
    case OOB_SYNTH_C4:
        c.M = (key & 1) ? ((i128)1 << 59) : (((i128)1 << 31) - 1);
        c.kmin = 3; c.kmax = 10; c.bug_pct = 30;
        break;
    case OOB_SYNTH_C5:
        c.M = ((i128)1 << 31) - 1;
        c.kmin = c.kmax = cap_log2 > 0 ? cap_log2 : 20;
        c.bug_pct = 0;
        break;
    default:
        c.M = ((i128)1 << 31) - 1;
        c.kmin = 3; c.kmax = 7; c.bug_pct = 30;
        break;
    }
    return c;
}

uint64_t mix(uint64_t seed, uint64_t i) {
    Rng r(seed ^ (i * 0xD1B54A32D192ED03ull));
    r.next();
    return r.next();
}

}  // namespace

extern "C" int oob_synth_caps(int config, int64_t caps[4]) {
    (void)config;
    caps[0] = 32;
    caps[1] = 48;
    caps[2] = 320;
    caps[3] = 128;
    return 0;
}

extern "C" int oob_synth_generate(int config, uint64_t seed, int64_t first, int64_t n, int cap_log2,
                                  oob_synth_out* out) {
    int64_t caps[4];
    oob_synth_caps(config, caps);
    int64_t V = 0, C = 0, N = 0, L = 0;
    out->var_begin[0] = out->con_begin[0] = out->node_begin[0] = out->lit_begin[0] = 0;
    for (int64_t qi = 0; qi < n; qi++) {
        int64_t gq = first + qi;
        int64_t access = gq / 2;
        int check = (int)(gq % 2);
        Rng r(mix(seed, (uint64_t)access));
        Cfg c = cfg_of(config, r.next(), cap_log2);
        int ntempl = config == OOB_SYNTH_C4 ? 8 : 7;
        int t = (int)r.uni(1, ntempl);
        bool bug = r.chance(c.bug_pct);
        Prog p;
        Access a;
        bool layout = false;
        switch (t) {
        case 1: t1(p, a, r, c, bug); break;
        case 2: t2(p, a, r, c, bug); break;
        case 3: t3(p, a, r, c, bug); break;
        case 4: t4(p, a, r, c, bug); break;
        case 5: layout = r.chance(25); t5(p, a, r, c, bug, layout); break;
        case 6: t6(p, a, r, c, bug); break;
        case 7: t7(p, a, r, c, bug); break;
        default: t8(p, a, r, c, bug); break;
        }
        QB q(c.M, p);
        build_query(a, p, layout ? 2 : check, c.M, q);
        if ((int64_t)q.var_code.size() > caps[0] || (int64_t)q.rel.size() > caps[1] ||
            (int64_t)q.op.size() > caps[2] || (int64_t)q.lits.size() > caps[3])
            return 1;
        for (size_t v = 0; v < q.var_code.size(); v++) {
            out->var_lo[V].lo = (uint64_t)q.vlo[v];
            out->var_lo[V].hi = (int64_t)(q.vlo[v] >> 64);
            out->var_hi[V].lo = (uint64_t)q.vhi[v];
            out->var_hi[V].hi = (int64_t)(q.vhi[v] >> 64);
            out->name_code[V] = (uint16_t)q.var_code[v];
            V++;
        }
        for (size_t k = 0; k < q.rel.size(); k++, C++) {
            out->con_rel[C] = q.rel[k];
            out->con_lhs[C] = q.lhs[k];
            out->con_rhs[C] = q.rhs[k];
        }
        for (size_t k = 0; k < q.op.size(); k++, N++) {
            out->node_op[N] = q.op[k];
            out->node_a[N] = q.na[k];
            out->node_b[N] = q.nb[k];
        }
        for (size_t k = 0; k < q.lits.size(); k++, L++) {
            out->lits[L].lo = (uint64_t)q.lits[k];
            out->lits[L].hi = (int64_t)(q.lits[k] >> 64);
        }
        out->var_begin[qi + 1] = V;
        out->con_begin[qi + 1] = C;
        out->node_begin[qi + 1] = N;
        out->lit_begin[qi + 1] = L;
        out->tmpl[qi] = (uint8_t)(t * 4 + (layout ? 2 : check));
    }
    return 0;
}
