/*
 * oob_oracle.c -- CPU restatement of the reference solver, for TESTS ONLY.
 *
 * TEST INFRASTRUCTURE.  This file is the parity checker and the CPU baseline
 * ("port") of the B200 engine.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (paper_2601_21552_b200) never links, loads or calls it.
 *
 * It restates /root/reference/pkg/src/scuba_mini/solver.py function by
 * function, deliberately in the reference's own shape (recursive evaluation,
 * recursive narrowing, recursive DFS with a copied environment per child), so
 * that it stays an independent check of the GPU engine, whose structure is
 * different (postfix segments, explicit stacks, trail-based backtracking).
 *
 * Pinned against the real reference: the tests/golden JSONL files hold the Python
 * reference's verdict, first model, DFS node count and propagation pass count
 * for the corpus queries, the reference's own randomized test systems and
 * crafted edge cases (tools/golden.py); tests/test_oracle.py checks this file
 * reproduces all four for every record.
 *
 * Arithmetic: Python ints are unbounded; this restatement uses __int128 with
 * overflow checks on every operation.  A query whose arithmetic would overflow
 * gets OOB_ERROR (never a silently wrong answer).
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../include/scuba_oob.h"

typedef __int128 i128;

#define ORC_INF ((i128)1000000000000000000LL) /* _INF = 10**18, solver.py:23 */
#define ORC_PASS_CAP 10000                     /* _PASS_CAP, solver.py:24 */
#define LIT_ONE (-1)                           /* node id of the Lit(1) in side constraints */

typedef struct {
    i128 lo, hi;
} iv_t;

typedef struct {
    /* query view */
    int nv, ncon;
    const uint8_t* op;
    const int32_t* na;
    const int32_t* nb;
    const oob_i128* lit;
    uint8_t* rel;   /* ncon (user + side) */
    int32_t* lhs;
    int32_t* rhs;
    /* run state */
    int ovf;        /* sticky overflow flag */
    int timed_out;
    double deadline;
    int64_t node_budget;
    int64_t nodes, passes;
} qctx;

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static i128 from_w(oob_i128 w) { return (i128)(((unsigned __int128)(uint64_t)w.hi << 64) | w.lo); }
static oob_i128 to_w(i128 v) {
    oob_i128 w;
    w.lo = (uint64_t)v;
    w.hi = (int64_t)(v >> 64);
    return w;
}

/* ----- checked arithmetic --------------------------------------------------- */
static i128 cadd(qctx* c, i128 a, i128 b) { i128 r; if (__builtin_add_overflow(a, b, &r)) c->ovf = 1; return r; }
static i128 csub(qctx* c, i128 a, i128 b) { i128 r; if (__builtin_sub_overflow(a, b, &r)) c->ovf = 1; return r; }
static i128 cmul(qctx* c, i128 a, i128 b) { i128 r; if (__builtin_mul_overflow(a, b, &r)) c->ovf = 1; return r; }
static i128 imin(i128 a, i128 b) { return a < b ? a : b; }
static i128 imax(i128 a, i128 b) { return a > b ? a : b; }
static i128 iabs(i128 a) { return a < 0 ? -a : a; }

/* tdiv: solver.py:94-97 (truncation toward zero) */
static i128 tdiv(i128 a, i128 b) {
    i128 q = iabs(a) / iabs(b);
    return ((a < 0) != (b < 0)) ? -q : q;
}
/* tmod: solver.py:100-102 (a - b*tdiv(a,b); sign follows a) */
static i128 tmod(qctx* c, i128 a, i128 b) { return csub(c, a, cmul(c, b, tdiv(a, b))); }
/* Python floor division a // b */
static i128 fdiv(i128 a, i128 b) {
    i128 q = a / b, r = a % b;
    if (r != 0 && ((r < 0) != (b < 0))) q -= 1;
    return q;
}
/* _ceil_div: solver.py:105-106  -((-a) // b) */
static i128 ceil_div(i128 a, i128 b) { return -fdiv(-a, b); }

static i128 lit_value(const qctx* c, int32_t n) {
    return n == LIT_ONE ? (i128)1 : from_w(c->lit[c->na[n]]);
}
static int node_op(const qctx* c, int32_t n) { return n == LIT_ONE ? OOB_NODE_LIT : c->op[n]; }

/* ----- _eval_iv: solver.py:112-149 ------------------------------------------ */
static int eval_iv(qctx* c, int32_t e, const iv_t* env, iv_t* out) {
    int op = node_op(c, e);
    if (op == OOB_NODE_LIT) {                       /* :114-115 */
        out->lo = out->hi = lit_value(c, e);
        return 1;
    }
    if (op == OOB_NODE_VAR) {                       /* :116-118 */
        iv_t d = env[c->na[e]];
        if (d.lo > d.hi) return 0;
        *out = d;
        return 1;
    }
    iv_t l, r;                                      /* :119-122 */
    if (!eval_iv(c, c->na[e], env, &l)) return 0;
    if (!eval_iv(c, c->nb[e], env, &r)) return 0;
    i128 l0 = l.lo, l1 = l.hi, r0 = r.lo, r1 = r.hi;
    switch (op) {
    case OOB_NODE_ADD:                              /* :126-127 */
        out->lo = cadd(c, l0, r0);
        out->hi = cadd(c, l1, r1);
        return 1;
    case OOB_NODE_SUB:                              /* :128-129 */
        out->lo = csub(c, l0, r1);
        out->hi = csub(c, l1, r0);
        return 1;
    case OOB_NODE_MUL: {                            /* :130-132 */
        i128 k0 = cmul(c, l0, r0), k1 = cmul(c, l0, r1), k2 = cmul(c, l1, r0), k3 = cmul(c, l1, r1);
        out->lo = imin(imin(k0, k1), imin(k2, k3));
        out->hi = imax(imax(k0, k1), imax(k2, k3));
        return 1;
    }
    default: break;
    }
    i128 d0 = imax(r0, 1), d1 = r1;                 /* :136-138 */
    if (d0 > d1) return 0;
    if (op == OOB_NODE_DIV) {                       /* :139-141 */
        i128 k0 = tdiv(l0, d0), k1 = tdiv(l0, d1), k2 = tdiv(l1, d0), k3 = tdiv(l1, d1);
        out->lo = imin(imin(k0, k1), imin(k2, k3));
        out->hi = imax(imax(k0, k1), imax(k2, k3));
        return 1;
    }
    /* OOB_NODE_MOD  :142-148 */
    i128 m = d1 - 1;
    if (l0 >= 0) { out->lo = 0; out->hi = imin(l1, m); return 1; }
    if (l1 <= 0) { out->lo = imax(l0, -m); out->hi = 0; return 1; }
    out->lo = imax(l0, -m);
    out->hi = imin(l1, m);
    return 1;
}

/* ----- _Narrower.narrow: solver.py:159-226 ---------------------------------- */
static int narrow(qctx* c, int32_t e, i128 t0, i128 t1, iv_t* env, int* changed) {
    if (t0 > t1) return 0;                          /* :161-162 */
    int op = node_op(c, e);
    if (op == OOB_NODE_LIT) {                       /* :163-164 */
        i128 v = lit_value(c, e);
        return t0 <= v && v <= t1;
    }
    if (op == OOB_NODE_VAR) {                       /* :165-173 */
        iv_t* d = &env[c->na[e]];
        i128 nlo = imax(d->lo, t0), nhi = imin(d->hi, t1);
        if (nlo > nhi) return 0;
        if (nlo != d->lo || nhi != d->hi) {
            d->lo = nlo;
            d->hi = nhi;
            *changed = 1;
        }
        return 1;
    }
    iv_t l, r;                                      /* :174-177 */
    if (!eval_iv(c, c->na[e], env, &l)) return 0;
    if (!eval_iv(c, c->nb[e], env, &r)) return 0;
    i128 l0 = l.lo, l1 = l.hi, r0 = r.lo, r1 = r.hi;
    int32_t L = c->na[e], R = c->nb[e];
    switch (op) {
    case OOB_NODE_ADD:                              /* :181-185 (stale l for the right side) */
        return narrow(c, L, csub(c, t0, r1), csub(c, t1, r0), env, changed) &&
               narrow(c, R, csub(c, t0, l1), csub(c, t1, l0), env, changed);
    case OOB_NODE_SUB:                              /* :186-190 */
        return narrow(c, L, cadd(c, t0, r0), cadd(c, t1, r1), env, changed) &&
               narrow(c, R, csub(c, l0, t1), csub(c, l1, t0), env, changed);
    case OOB_NODE_MUL: {                            /* :191-216 */
        if (l0 < 0 || r0 < 0) return 1;
        if (t1 < 0) return 0;
        i128 t0n = imax(t0, 0);
        int32_t child[2] = {L, R};
        i128 olo[2] = {r0, l0}, ohi[2] = {r1, l1};
        for (int k = 0; k < 2; k++) {
            i128 lo_req = -ORC_INF, hi_req = ORC_INF;
            if (t0n > 0) {
                if (ohi[k] == 0) return 0;
                lo_req = ceil_div(t0n, ohi[k]);
            }
            if (olo[k] > 0) hi_req = fdiv(t1, olo[k]);
            if (!narrow(c, child[k], lo_req, hi_req, env, changed)) return 0;
        }
        return 1;
    }
    case OOB_NODE_DIV:                              /* :217-223 (literal divisor >= 1 only) */
        if (node_op(c, R) == OOB_NODE_LIT && lit_value(c, R) >= 1) {
            i128 cc = lit_value(c, R);
            i128 lo_req = t0 > 0 ? cmul(c, t0, cc) : csub(c, cmul(c, t0, cc), cc - 1);
            i128 hi_req = t1 >= 0 ? cadd(c, cmul(c, t1, cc), cc - 1) : cmul(c, t1, cc);
            return narrow(c, L, lo_req, hi_req, env, changed);
        }
        return 1;
    default:                                        /* % : forward-only, :224-225 */
        return 1;
    }
}

/* ----- _propagate_constraint: solver.py:229-261 ----------------------------- */
static int propagate_constraint(qctx* c, int k, iv_t* env, int* changed) {
    iv_t l, r;
    if (!eval_iv(c, c->lhs[k], env, &l)) return 0;
    if (!eval_iv(c, c->rhs[k], env, &r)) return 0;
    int32_t A = c->lhs[k], B = c->rhs[k];
    switch (c->rel[k]) {
    case OOB_REL_LT:
        return narrow(c, A, -ORC_INF, csub(c, r.hi, 1), env, changed) &&
               narrow(c, B, cadd(c, l.lo, 1), ORC_INF, env, changed);
    case OOB_REL_LE:
        return narrow(c, A, -ORC_INF, r.hi, env, changed) && narrow(c, B, l.lo, ORC_INF, env, changed);
    case OOB_REL_EQ: {
        i128 lo = imax(l.lo, r.lo), hi = imin(l.hi, r.hi);
        return narrow(c, A, lo, hi, env, changed) && narrow(c, B, lo, hi, env, changed);
    }
    case OOB_REL_GE:
        return narrow(c, A, r.lo, ORC_INF, env, changed) && narrow(c, B, -ORC_INF, l.hi, env, changed);
    default: /* OOB_REL_GT */
        return narrow(c, A, cadd(c, r.lo, 1), ORC_INF, env, changed) &&
               narrow(c, B, -ORC_INF, csub(c, l.hi, 1), env, changed);
    }
}

/* ----- propagate: solver.py:264-280 (env updated in place) ------------------ */
static int propagate(qctx* c, iv_t* env, int check_deadline) {
    for (int pass = 0; pass < ORC_PASS_CAP; pass++) {
        if (check_deadline && now_s() > c->deadline) { c->timed_out = 1; return 0; }
        c->passes++;
        int changed = 0;
        for (int k = 0; k < c->ncon; k++)
            if (!propagate_constraint(c, k, env, &changed)) return 0;
        if (!changed) break;
    }
    return 1;
}

/* ----- _eval_exact / check_model: solver.py:286-328 ------------------------- */
static int eval_exact(qctx* c, int32_t e, const i128* model, i128* out) {
    int op = node_op(c, e);
    if (op == OOB_NODE_LIT) { *out = lit_value(c, e); return 1; }
    if (op == OOB_NODE_VAR) { *out = model[c->na[e]]; return 1; }
    i128 a, b;
    if (!eval_exact(c, c->na[e], model, &a)) return 0;
    if (!eval_exact(c, c->nb[e], model, &b)) return 0;
    switch (op) {
    case OOB_NODE_ADD: *out = cadd(c, a, b); return 1;
    case OOB_NODE_SUB: *out = csub(c, a, b); return 1;
    case OOB_NODE_MUL: *out = cmul(c, a, b); return 1;
    default: break;
    }
    if (b == 0) return 0;                           /* :301-302 trap falsifies */
    *out = op == OOB_NODE_DIV ? tdiv(a, b) : tmod(c, a, b);
    return 1;
}

static int rel_holds(int rel, i128 a, i128 b) {
    switch (rel) {
    case OOB_REL_LT: return a < b;
    case OOB_REL_LE: return a <= b;
    case OOB_REL_EQ: return a == b;
    case OOB_REL_GE: return a >= b;
    default: return a > b;
    }
}

static int check_model(qctx* c, const i128* model) {
    for (int k = 0; k < c->ncon; k++) {
        i128 a, b;
        if (!eval_exact(c, c->lhs[k], model, &a)) return 0;
        if (!eval_exact(c, c->rhs[k], model, &b)) return 0;
        if (!rel_holds(c->rel[k], a, b)) return 0;
    }
    return 1;
}

/* ----- divisor side constraints: solver.py:334-357 -------------------------- */
static int same_term(const qctx* c, int32_t x, int32_t y) {
    if (x == y) return 1;
    int ox = node_op(c, x), oy = node_op(c, y);
    if (ox != oy) return 0;
    if (ox == OOB_NODE_LIT) return lit_value(c, x) == lit_value(c, y);
    if (ox == OOB_NODE_VAR) return c->na[x] == c->na[y];
    return same_term(c, c->na[x], c->na[y]) && same_term(c, c->nb[x], c->nb[y]);
}

static void collect_divisors(const qctx* c, int32_t e, int32_t* out, int* n) {
    int op = node_op(c, e);
    if (op < OOB_NODE_ADD) return;
    if (op == OOB_NODE_DIV || op == OOB_NODE_MOD) {
        int32_t R = c->nb[e];
        if (!(node_op(c, R) == OOB_NODE_LIT && lit_value(c, R) >= 1)) {
            int seen = 0;
            for (int i = 0; i < *n && !seen; i++) seen = same_term(c, out[i], R);
            if (!seen) out[(*n)++] = R;
        }
    }
    collect_divisors(c, c->na[e], out, n);
    collect_divisors(c, c->nb[e], out, n);
}

/* ----- _search: solver.py:385-416 ------------------------------------------- */
static int search(qctx* c, const iv_t* env_in, i128* model) {
    if (now_s() > c->deadline || (c->node_budget > 0 && c->nodes >= c->node_budget)) {
        c->timed_out = 1;                           /* :391-392 */
        return 0;
    }
    c->nodes++;
    iv_t* env = (iv_t*)alloca(sizeof(iv_t) * (c->nv ? c->nv : 1));
    memcpy(env, env_in, sizeof(iv_t) * c->nv);
    if (!propagate(c, env, 1) || c->ovf) return 0;  /* :393-395 */
    int pick = -1;                                  /* :397-404 smallest, ties by order */
    i128 pick_size = 0;
    for (int v = 0; v < c->nv; v++) {
        if (env[v].lo < env[v].hi) {
            i128 size = env[v].hi - env[v].lo + 1;
            if (pick < 0 || size < pick_size) { pick = v; pick_size = size; }
        }
    }
    if (pick < 0) {                                 /* :405-407 leaf */
        for (int v = 0; v < c->nv; v++) model[v] = env[v].lo;
        return check_model(c, model);
    }
    i128 lo = env[pick].lo, hi = env[pick].hi;      /* :408-415 lower half first */
    i128 mid = fdiv(lo + hi, 2);
    env[pick].lo = lo; env[pick].hi = mid;
    if (search(c, env, model)) return 1;
    if (c->timed_out || c->ovf) return 0;
    env[pick].lo = mid + 1; env[pick].hi = hi;
    return search(c, env, model);
}

/* ----- per-query setup ------------------------------------------------------ */
static int build_view(const oob_batch* b, int64_t q, int with_side, qctx* c) {
    memset(c, 0, sizeof(*c));
    int64_t vb = b->var_begin[q], cb = b->con_begin[q], nb = b->node_begin[q], lb = b->lit_begin[q];
    c->nv = (int)(b->var_begin[q + 1] - vb);
    int nuser = (int)(b->con_begin[q + 1] - cb);
    int nn = (int)(b->node_begin[q + 1] - nb);
    c->op = b->node_op + nb;
    c->na = b->node_a + nb;
    c->nb = b->node_b + nb;
    c->lit = b->lits + lb;
    int cap = nuser + (with_side ? nn : 0);
    c->rel = (uint8_t*)malloc(cap + 1);
    c->lhs = (int32_t*)malloc(sizeof(int32_t) * (cap + 1));
    c->rhs = (int32_t*)malloc(sizeof(int32_t) * (cap + 1));
    for (int k = 0; k < nuser; k++) {
        c->rel[k] = b->con_rel[cb + k];
        c->lhs[k] = b->con_lhs[cb + k];
        c->rhs[k] = b->con_rhs[cb + k];
    }
    c->ncon = nuser;
    if (with_side) {
        int32_t* divs = (int32_t*)malloc(sizeof(int32_t) * (nn + 1));
        int nd = 0;
        for (int k = 0; k < nuser; k++) {
            collect_divisors(c, c->lhs[k], divs, &nd);
            collect_divisors(c, c->rhs[k], divs, &nd);
        }
        for (int i = 0; i < nd; i++) {
            if (node_op(c, divs[i]) == OOB_NODE_LIT) continue;  /* :353-357 */
            c->rel[c->ncon] = OOB_REL_GE;
            c->lhs[c->ncon] = divs[i];
            c->rhs[c->ncon] = LIT_ONE;
            c->ncon++;
        }
        free(divs);
    }
    return 0;
}

static void free_view(qctx* c) {
    free(c->rel);
    free(c->lhs);
    free(c->rhs);
}

/* solve: solver.py:363-382 */
static void solve_one(const oob_batch* b, int64_t q, double timeout_s, int64_t node_budget, oob_result* out) {
    double start = now_s();
    qctx c;
    build_view(b, q, 1, &c);
    c.deadline = start + timeout_s;
    c.node_budget = node_budget;
    int64_t vb = b->var_begin[q];
    iv_t* env = (iv_t*)malloc(sizeof(iv_t) * (c.nv + 1));
    i128* model = (i128*)malloc(sizeof(i128) * (c.nv + 1));
    int bad = 0;
    for (int v = 0; v < c.nv; v++) {
        env[v].lo = from_w(b->var_lo[vb + v]);
        env[v].hi = from_w(b->var_hi[vb + v]);
        if (env[v].lo > env[v].hi) bad = 1;
    }
    int8_t verdict;
    if (bad) {
        verdict = OOB_UNSAT;                        /* :374-375 */
    } else if (timeout_s <= 0) {
        verdict = OOB_TIMEOUT;                      /* deadline already passed at :391 */
    } else {
        int found = search(&c, env, model);
        if (c.ovf) verdict = OOB_ERROR;
        else if (c.timed_out) verdict = OOB_TIMEOUT;
        else verdict = found ? OOB_SAT : OOB_UNSAT;
    }
    out->verdict[q] = verdict;
    if (verdict == OOB_SAT && out->model)
        for (int v = 0; v < c.nv; v++) out->model[vb + v] = to_w(model[v]);
    if (out->nodes) out->nodes[q] = c.nodes;
    if (out->passes) out->passes[q] = c.passes;
    if (out->elapsed_s) out->elapsed_s[q] = now_s() - start;
    free(env);
    free(model);
    free_view(&c);
}

/* ----- exported batch API (threads over queries) ---------------------------- */
typedef struct {
    const oob_batch* b;
    double timeout_s;
    int64_t node_budget;
    oob_result* out;
    atomic_llong next;
} job_t;

static void* worker(void* arg) {
    job_t* j = (job_t*)arg;
    for (;;) {
        long long q = atomic_fetch_add(&j->next, 1);
        if (q >= j->b->n_queries) break;
        solve_one(j->b, q, j->timeout_s, j->node_budget, j->out);
    }
    return NULL;
}

int oracle_solve_batch(const oob_batch* b, double timeout_s, int64_t node_budget, oob_result* out,
                       int n_threads) {
    job_t j;
    j.b = b;
    j.timeout_s = timeout_s;
    j.node_budget = node_budget;
    j.out = out;
    atomic_init(&j.next, 0);
    if (n_threads <= 1) {
        worker(&j);
        return 0;
    }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
    for (int i = 0; i < n_threads; i++) pthread_create(&th[i], NULL, worker, &j);
    for (int i = 0; i < n_threads; i++) pthread_join(th[i], NULL);
    free(th);
    return 0;
}

/* propagate(domains, constraints) as the public API: no side constraints, no deadline. */
int oracle_propagate_batch(const oob_batch* b, oob_i128* out_lo, oob_i128* out_hi, int8_t* status) {
    for (int64_t q = 0; q < b->n_queries; q++) {
        qctx c;
        build_view(b, q, 0, &c);
        int64_t vb = b->var_begin[q];
        iv_t* env = (iv_t*)malloc(sizeof(iv_t) * (c.nv + 1));
        for (int v = 0; v < c.nv; v++) {
            env[v].lo = from_w(b->var_lo[vb + v]);
            env[v].hi = from_w(b->var_hi[vb + v]);
        }
        int ok = propagate(&c, env, 0);
        status[q] = c.ovf ? -1 : (int8_t)ok;
        for (int v = 0; v < c.nv; v++) {
            out_lo[vb + v] = to_w(env[v].lo);
            out_hi[vb + v] = to_w(env[v].hi);
        }
        free(env);
        free_view(&c);
    }
    return 0;
}

int oracle_check_model_batch(const oob_batch* b, const oob_i128* model, int8_t* ok) {
    for (int64_t q = 0; q < b->n_queries; q++) {
        qctx c;
        build_view(b, q, 0, &c);
        int64_t vb = b->var_begin[q];
        i128* m = (i128*)malloc(sizeof(i128) * (c.nv + 1));
        for (int v = 0; v < c.nv; v++) m[v] = from_w(model[vb + v]);
        int r = check_model(&c, m);
        ok[q] = c.ovf ? -1 : (int8_t)r;
        free(m);
        free_view(&c);
    }
    return 0;
}

int oracle_side_constraint_count(const oob_batch* b, int64_t* counts) {
    for (int64_t q = 0; q < b->n_queries; q++) {
        qctx c;
        build_view(b, q, 1, &c);
        counts[q] = c.ncon - (int)(b->con_begin[q + 1] - b->con_begin[q]);
        free_view(&c);
    }
    return 0;
}
