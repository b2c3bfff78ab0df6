/*
 * scuba_oob.h -- C ABI of the B200 engine for the per-access OOB
 * satisfiability check of arXiv 2601.21552 ("scuba-mini" reference).
 *
 * The reference hot path is the pure-Python bounded-integer solver
 *   scuba_mini.solver.solve(variables, constraints, timeout_s)
 *     /root/reference/pkg/src/scuba_mini/solver.py:363-382
 * bound by name into the analyzer (analyzer.py:32) and called once per query
 * at analyzer.py:163 (partition-layout checks) and analyzer.py:211 (access
 * checks).  Its siblings propagate() (solver.py:264-280) and check_model()
 * (solver.py:319-328) are public API pinned by the reference tests.
 *
 * This header replaces those three functions with batched, caller-allocates
 * entry points.  A "batch" is n independent queries (one ConstraintSet each,
 * constraint_gen.py:65-73) in flat arrays; all offsets are per query so that
 * queries can be sliced or sharded without rewriting indices.
 *
 * Semantics preserved exactly:
 *   - variable order = list order (drives branching and model order);
 *   - divisor side constraints appended in reference order (solver.py:345);
 *   - any lo > hi  => UNSAT without search (solver.py:374);
 *   - timeout_s <= 0 => TIMEOUT for every query that reaches search;
 *   - the SAT model is the reference's first model (same DFS, same
 *     propagation schedule, same 10**18 clamp and 10 000-pass cap);
 *   - C truncating division; division/modulo by zero falsifies.
 *
 * Threading: every entry point is reentrant; the library keeps no pointer to
 * caller memory after return.  Device buffers are library-owned and pooled
 * per device (oob_release() frees them).
 */
#ifndef SCUBA_OOB_H
#define SCUBA_OOB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Two's-complement 128-bit integer, little-endian words. Python ints of the
 * reference are arbitrary precision; the engine is exact for every query whose
 * intermediate magnitudes fit in 126 bits (checked per query on the host;
 * queries beyond that get OOB_ERROR, never a silent wrong answer). */
typedef struct {
    uint64_t lo;
    int64_t hi;
} oob_i128;

/* Term node opcodes (solver.py:32-49: Lit, VarRef, BinE op in + - * / %). */
enum {
    OOB_NODE_LIT = 0,
    OOB_NODE_VAR = 1,
    OOB_NODE_ADD = 2,
    OOB_NODE_SUB = 3,
    OOB_NODE_MUL = 4,
    OOB_NODE_DIV = 5,
    OOB_NODE_MOD = 6
};

/* Relations, in the order of solver.py:26 RELS = ("<", "<=", "=", ">=", ">"). */
enum {
    OOB_REL_LT = 0,
    OOB_REL_LE = 1,
    OOB_REL_EQ = 2,
    OOB_REL_GE = 3,
    OOB_REL_GT = 4
};

/* Verdict codes (solver.py:69-84 Sat / Unsat / Timeout). */
enum {
    OOB_UNSAT = 0,
    OOB_SAT = 1,
    OOB_TIMEOUT = 2,
    OOB_ERROR = 3 /* query outside the exact regime / capacity; see last_error */
};

/* Return status of every entry point. */
enum {
    OOB_OK = 0,
    OOB_E_INVALID = 1, /* malformed batch (unknown op/rel, bad index) -> ValueError */
    OOB_E_CUDA = 2,    /* CUDA runtime error or no device                          */
    OOB_E_RANGE = 3,   /* some query exceeds the exact 126-bit regime              */
    OOB_E_NOMEM = 4
};

/*
 * Flat batch.  For query q:
 *   variables   [var_begin[q], var_begin[q+1])   domains var_lo/var_hi
 *   constraints [con_begin[q], con_begin[q+1])   rel + lhs/rhs root node
 *   nodes       [node_begin[q], node_begin[q+1]) op + operands
 *   literals    [lit_begin[q], lit_begin[q+1])
 * Node, variable and literal indices stored in con_lhs/con_rhs/node_a/node_b
 * are RELATIVE to the query's own ranges.  Nodes form a DAG in topological
 * order: a binary node's children have smaller indices than the node.
 *   LIT: node_a = literal index          VAR: node_a = variable index
 *   ADD..MOD: node_a = left child node,  node_b = right child node
 */
typedef struct {
    int64_t n_queries;
    const int64_t* var_begin;  /* n+1 */
    const oob_i128* var_lo;
    const oob_i128* var_hi;
    const int64_t* con_begin;  /* n+1 */
    const uint8_t* con_rel;
    const int32_t* con_lhs;
    const int32_t* con_rhs;
    const int64_t* node_begin; /* n+1 */
    const uint8_t* node_op;
    const int32_t* node_a;
    const int32_t* node_b;
    const int64_t* lit_begin;  /* n+1 */
    const oob_i128* lits;
} oob_batch;

typedef struct {
    double timeout_s;     /* per-query wall-clock budget (solver.py:366); <=0 => TIMEOUT */
    int64_t node_budget;  /* >0: TIMEOUT after this many DFS nodes (deterministic) */
    int32_t n_gpus;       /* devices to shard over; 0 = all visible               */
    int32_t device;       /* first device ordinal                                 */
    int32_t flags;        /* OOB_F_* below                                        */
    int32_t heavy_nodes;  /* DFS nodes after which a query moves to the warp-
                             cooperative frontier kernel; 0 = default (24;
                             fast mode: 96, SCUBA_OOB_FAST_HEAVY_NODES; 8 with
                             SCUBA_OOB_FAST_FRONTIER=1),
                             <0 = never (one lane per query throughout)      */
    int32_t jit_min;      /* structure classes with at least this many queries
                             in an int64 job run as run-time compiled kernels;
                             0 = default (SCUBA_OOB_JIT_MIN, else 1024)       */
} oob_options;

enum {
    OOB_F_NO_SORT = 1,   /* keep input order on device (testing the scheduler) */
    OOB_F_NO_DEMOTE = 2, /* decide wide-regime queries entirely in their proven
                            regime (no root-phase demotion; testing) */
    OOB_F_NO_JIT = 4,    /* interpret every structure class (no run-time
                            compiled class kernels; testing) */
    OOB_F_NO_X32 = 8,    /* keep int64-regime queries in int64 (no x32
                            demotion after the root phase; testing) */
    OOB_F_FAST = 16,     /* fast mode: heavy queries first meet a symbolic
                            Unsat prover (sound: a refuted query has no
                            integer solution in its root box, so the reference
                            can never return Sat on it); what it does not
                            refute is decided by the exact emulation (an
                            int64-regime query with a declared box of at most
                            SCUBA_OOB_ENUM_MAX = 4096 points is first
                            enumerated exhaustively: no check_model point =
                            Unsat).  Verdicts
                            and Sat models are the reference's; nodes/passes
                            of refuted queries are 0 (not the reference's
                            counters).  DESIGN.md section 4.9. */
    OOB_F_CHAIN = 32     /* with OOB_F_FAST: the int64 job's open entries first
                            run a warp-per-query search with warp-parallel
                            (Jacobi) propagation (chain.cuh); verdicts, Sat
                            models and node counts stay the reference's, pass
                            counts of the entries it decides are its rounds.
                            Opt-in: slower than the exact emulation on the
                            benchmark batches. */
};

/* Results (caller-allocated; optional arrays may be NULL). */
typedef struct {
    int8_t* verdict;     /* n: OOB_UNSAT / OOB_SAT / OOB_TIMEOUT / OOB_ERROR        */
    oob_i128* model;     /* var_begin[n] entries: SAT model at the query's var range;
                            every entry is written (zero for queries not SAT), so the
                            caller need not clear it */
    int64_t* nodes;      /* n, optional: DFS nodes visited (reference _search calls) */
    int64_t* passes;     /* n, optional: propagation passes (one _Narrower each)     */
    double* elapsed_s;   /* n, optional: device time spent on the query            */
} oob_result;

/* Batched solve(): replaces solver.py:363-416 (solve + _search). */
int oob_solve_batch(const oob_batch* batch, const oob_options* opt,
                    oob_result* out);

/* A stream of independent batches: results[i] are exactly oob_solve_batch's
 * for batches[i].  Consecutive batches are pipelined (the host compile and
 * upload of batch i+1 overlap the kernels of batch i; two sets of device
 * buffers alternate), so the throughput of a stream is bounded by the slower
 * of the host and device phases instead of their sum. */
int oob_solve_batches(const oob_batch* batches, int64_t n_batches, const oob_options* opt,
                      oob_result* results);

/* Batched propagate(domains, constraints): replaces solver.py:264-280.
 * Domains are var_lo/var_hi; constraints are used AS GIVEN (propagate() adds
 * no side constraints).  status[q] = 1 and out_lo/out_hi narrowed, or
 * status[q] = 0 for the reference's None (contradiction). */
int oob_propagate_batch(const oob_batch* batch, const oob_options* opt,
                        oob_i128* out_lo, oob_i128* out_hi, int8_t* status);

/* Batched check_model(constraints, model): replaces solver.py:319-328.
 * model has var_begin[n] entries; ok[q] = 1 iff every constraint holds. */
int oob_check_model_batch(const oob_batch* batch, const oob_options* opt,
                          const oob_i128* model, int8_t* ok);

/* Number of divisor side constraints solve() appends for query q
 * (solver.py:334-357); lets callers size buffers / audit the host compiler. */
int oob_side_constraint_count(const oob_batch* batch, int64_t* counts);
/* Host-only audit of the compiler: the exact-arithmetic regime each query is
 * decided in (0 immediate verdict, 1 int64, 2 int128, 3 256-bit, 4 out of
 * range -> OOB_ERROR).  No device is touched. */
int oob_query_regime(const oob_batch* batch, const oob_options* opt, int8_t* regime);
/* Fast-mode compiler audit (no device is touched): the Unsat certificates the
 * engine compiles for the batch's structure classes (csrc/cert.cuh layout:
 * per class [n] then n x [length][words]), each query's class entry in
 * words[] (cert_off[q], -1: none), and each query's literal slot values
 * (slots[slot_begin[q] .. slot_begin[q+1]), the order the certificates'
 * parameters index).  The device checks these certificates numerically. */
int oob_cert_compile(const oob_batch* batch, const oob_options* opt, uint64_t* words, int64_t words_cap,
                     int64_t* n_words, int64_t* cert_off, oob_i128* slots, int64_t slots_cap, int64_t* slot_begin);
/* Run-time specialisation audit: the CUDA source generated for query q's
 * structure class (written to src, NUL-terminated, truncated to src_cap) and
 * its NVRTC compile for sm_100a (*compile_ms); no device is touched. */
int oob_jit_compile(const oob_batch* batch, int64_t q, char* src, int64_t src_cap, double* compile_ms);

/*
 * Plans: compile and upload a batch once, then run the decision kernels on
 * device-resident records as often as needed (benchmarks, repeated checking).
 * The caller keeps `batch` alive until oob_plan_destroy().
 *   oob_plan_run      launches every device's kernels; *device_ms = the max
 *                     over devices of the CUDA-event time on the engine stream
 *   oob_plan_results  device->host copy + scatter (same contract as
 *                     oob_solve_batch's results)
 *   oob_plan_info     [0] queries on devices  [1] record bytes (descriptors +
 *                     class code + per-query data)  [2] result bytes
 *                     [3] structure classes  [4] device jobs  [5] kernel
 *                     launches per run  [6] queries in the int128 regime
 *                     [7] host compile time (us)  [8] bytes one solve call
 *                     copies host -> device (raw values or records,
 *                     descriptors, class code)
 */
typedef struct oob_plan oob_plan;
int oob_plan_create(const oob_batch* batch, const oob_options* opt, oob_plan** plan);
int oob_plan_run(oob_plan* plan, float* device_ms);
int oob_plan_results(oob_plan* plan, oob_result* out);
int oob_plan_info(const oob_plan* plan, int64_t info[9]);
void oob_plan_destroy(oob_plan* plan);

/* Diagnostics: host-side evaluation of the 256-bit regime arithmetic
 * (op 0 + 1 - 2 * 3 / 4 % 5 < 6 >>1; 4 little-endian words each). */
int oob_selftest_i256(int op, const int64_t* a, const int64_t* b, int64_t* out);

/* Last error message of the calling thread ("" if none). */
const char* oob_last_error(void);
/* Visible CUDA devices (0 when none). */
int oob_device_count(void);
/* Library build identification. */
const char* oob_version(void);
/* Free pooled device buffers on every device. */
void oob_release(void);

#ifdef __cplusplus
}
#endif

#endif /* SCUBA_OOB_H */
