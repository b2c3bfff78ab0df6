// format.h -- device-resident layout of a compiled query batch.
//
// The host compiler (host.cpp) turns the caller's flat oob_batch into:
//
//   code[]   u32 structure words, one block per STRUCTURE CLASS (queries whose
//            constraint/term shapes are identical share one block):
//              ncon constraint words   rel | lroot << 3 | rroot << 17
//              ncode node words        op | arg << 3
//            Nodes are laid out per constraint side as a contiguous postfix
//            segment (the DAG is expanded to a tree), so the subtree of node i
//            is [i - size(i) + 1, i], its right child is i - 1 and its left
//            child is i - 1 - size(i - 1).  arg = variable index (VAR), literal
//            slot (LIT, one slot per occurrence), or subtree size (binary op).
//   data[]   per query: nv (lo, hi) domain pairs then nlit literal slots, each
//            value W bytes (8 for the int64 regime, 16 for int128), 16-byte
//            aligned per query.
//   qdesc[]  per scheduled query (sorted by class, then by cost estimate):
//            where its code block and data block are and where results go.
#pragma once
#include "types.h"

#if defined(__CUDACC__)
#define OOB_HD __host__ __device__
#else
#define OOB_HD
#endif

namespace oob {

enum : uint32_t {
    NODE_LIT = 0,
    NODE_VAR = 1,
    NODE_ADD = 2,
    NODE_SUB = 3,
    NODE_MUL = 4,
    NODE_DIV = 5,
    NODE_MOD = 6
};
enum : uint32_t { REL_LT = 0, REL_LE = 1, REL_EQ = 2, REL_GE = 3, REL_GT = 4 };
enum : int { VERDICT_UNSAT = 0, VERDICT_SAT = 1, VERDICT_TIMEOUT = 2, VERDICT_ERROR = 3 };

constexpr int PASS_CAP = 10000;          // _PASS_CAP (solver.py:24)
constexpr uint32_t MAX_CODE = 16383;     // 14-bit node ids in constraint words
constexpr uint32_t MAX_TREE_DEPTH = 32;  // bounded pre-order narrowing stack

struct QDesc {
    uint32_t code_off;   // u32 index of the class's constraint words in code[]
    uint32_t nv_ncon;    // nv | ncon << 16
    uint32_t ncode_nlit; // ncode | nlit << 16
    uint32_t out_q;      // index of the query in the caller's batch
    uint64_t data_off;   // int64-word index of the query's data in data[]
    uint64_t out_v;      // caller var_begin[out_q] (model offset, in vars)
};
static_assert(sizeof(QDesc) == 32, "QDesc is two int4 words");

OOB_HD inline uint32_t con_word(uint32_t rel, uint32_t l, uint32_t r) {
    return rel | (l << 3) | (r << 17);
}
OOB_HD inline uint32_t node_word(uint32_t op, uint32_t arg) { return op | (arg << 3); }

// Per-launch geometry of the per-warp scratch slab (host-computed).
struct SlabGeom {
    uint32_t maxv, maxcode, maxlit, depth_cap, trail_cap, maxcsize;
    // shared-memory residency of the hot per-lane state (env, forward-interval
    // cache of the current constraint, literal slots): bytes per warp, 0 = the
    // global slab is used instead; offsets in units of T inside the warp's part
    uint32_t smem_per_warp;
    uint64_t o_s_env_lo, o_s_env_hi, o_s_val_lo, o_s_val_hi, o_s_lit, o_s_st0, o_s_st1;
    uint64_t o_s_stn_bytes;  // byte offset of the u32 stack-node slots in the warp's part
    uint32_t st_cap;         // narrowing stack entries (deepest term + 2)
    // word offsets (in units of T) of each array inside one warp's slab
    uint64_t o_env_lo, o_env_hi, o_val_lo, o_val_hi, o_lit, o_fr_mid, o_fr_hi, o_tr_lo, o_tr_hi, o_st0, o_st1;
    // u32-word offsets inside the u32 part of the slab
    uint64_t o_stamp, o_fr_pick, o_fr_mark, o_fr_clean, o_tr_var, o_stn;
    uint64_t slab_T_words, slab_u32_words;  // per-warp sizes
};

// One structure class: its code block (constraint words, node words, then 4
// membership words per variable) and its slice [q_begin, q_end) of the
// class-major schedule.
constexpr uint32_t NO_CLASS = 0xFFFFFFFFu;  // warp_class entry of a warp with nothing to do

struct ClassDesc {
    uint32_t code_off;
    uint32_t nv_ncon;
    uint32_t ncode_nlit;
    uint32_t q_begin;
    uint32_t q_end;
    uint32_t cert;     // fast mode: word offset of the class's Unsat certificates (cert.cuh), NO_CERT: none
    uint32_t pad[2];
};
constexpr uint32_t NO_CERT = 0xFFFFFFFFu;
static_assert(sizeof(ClassDesc) == 32, "ClassDesc is two int4 words");

// Regime demotion (SOLVE mode).  A query whose declared domains need the
// int128 / 256-bit regime first runs its ROOT node's propagation in that
// regime (oob_root_kernel); as soon as the bound proof restated at the
// narrowed domains fits a narrower regime, the query's state is written into
// a SHADOW entry of that regime's job, which resumes the search there.
// resume[] word per scheduled query:
//   0          fresh start from the declared domains
//   RES_SKIP   not live in this job (shadow not chosen / demoted / finished)
//   RES_ROOT | [RES_FIX] | passes   resume the root node after `passes`
//              propagation passes (RES_FIX: the last one changed nothing)
constexpr uint32_t RES_SKIP = 0xFFFFFFFFu;
constexpr uint32_t RES_ROOT = 0x80000000u;
constexpr uint32_t RES_FIX = 0x40000000u;
// the root state comes from the hand-off buffer (LaunchArgs::handoff): a query
// handed to the frontier while still at its root node resumes there
constexpr uint32_t RES_HANDOFF = 0x20000000u;
constexpr uint32_t RES_PASSES = 0x1FFFFFFFu;
constexpr uint32_t ROOT_MAX_PASSES = 64;      // wide root phases: pass budget before giving up on demotion
constexpr uint32_t ROOT_MAX_PASSES_X32 = 16;  // int64 root phase (x32 probe)

struct DemoteTarget {
    const QDesc* qdesc;     // target job's descriptors (data_off of the shadow)
    int64_t* data;          // target job's per-query data
    uint32_t* resume;       // target job's resume words
    uint64_t* t0;           // target job's per-query start times
    const uint32_t* slot;   // per entry of THIS job: its shadow's index in the target job
};

struct LaunchArgs {
    const QDesc* qdesc;       // per scheduled query
    const uint32_t* code;     // structure words (constraints + nodes), per class
    const int64_t* data;      // per query domains + literals (W/8 words per value)
    uint32_t n;               // scheduled queries
    uint32_t* next;           // work counter (aux kernel)
    const ClassDesc* classes; // per structure class
    uint32_t n_classes;
    uint32_t* class_next;     // per class work cursor (starts at q_begin)
    const uint32_t* warp_class;  // starting class of every warp
    void* slab_T;             // T-typed scratch, n_warps * slab_T_words
    uint32_t* slab_u32;       // u32 scratch, n_warps * slab_u32_words
    SlabGeom g;
    // heavy-query hand-off: the lockstep kernel gives up a query after
    // heavy_nodes DFS nodes and queues it for the frontier kernel
    uint32_t heavy_nodes;     // 0 = never hand off
    uint32_t heavy_passes;    // also hand off after this many propagation passes (0 = no)
    uint32_t handoff_gate;    // hand off only while a frontier warp of the launch waits (fast mode)
    uint32_t frontier_only;   // a tail launch: skip the lockstep phase, serve the heavy list
    uint32_t frontier_wait_us;  // bound on an idle frontier warp's wait for its launch's producers
    uint32_t* heavy_count;    // [0] listed [1] claimed [2] lockstep warps started [3] done [4] frontier
                              // warps waiting (8 words per launch)
    uint32_t* heavy_list;     // query index + 1 (0 = not yet published)
    uint64_t* heavy_t0;       // start time of each scheduled query (ns)
    uint32_t* heavy_next;     // frontier kernel work cursor
    // frontier scratch (frontier.cuh): fr_nregions regions shared by every
    // launch of the job; a warp holds one (bit set in fr_bitmap) only while it
    // expands a heavy query
    void* fr_region;
    uint64_t fr_region_bytes;
    uint32_t fr_ecap, fr_ucap, fr_logcap;
    uint32_t* fr_bitmap;
    uint32_t fr_nregions;
    // per-warp slabs of the SOLVE kernels: a pool of slab_nslots shared by the
    // job's launches, one held per running warp (null: slab index = warp id)
    uint32_t* slab_bitmap;
    uint32_t slab_nslots;
    // root state of queries handed off at their root node (data layout, at
    // QDesc::data_off; null: hand-offs restart from the declared domains)
    int64_t* handoff;
    // outputs (indexed by QDesc::out_q / out_v)
    int8_t* verdict;
    int64_t* model;           // int128 words, 2 per var
    int64_t* nodes;
    int64_t* passes;
    float* elapsed;
    int8_t* err;              // per query error reason (0 = none)
    // options
    uint64_t timeout_ns;      // 0 => unlimited
    int64_t node_budget;      // >0 => deterministic budget
    int mode;                 // MODE_SOLVE / MODE_PROPAGATE / MODE_CHECK
    uint32_t* resume;         // per scheduled query (null: all fresh)
    uint64_t* timeline;       // debug (SCUBA_OOB_TIMELINE): per entry start, hand-off, frontier start, end (ns)
    unsigned long long* stats;  // debug (SCUBA_OOB_TRACE=2): frontier / lockstep lane-efficiency counters
    DemoteTarget dem[3];      // root kernel: [0] int64 job, [1] int128 job, [2] x32 job (slot null: none)
    // fast mode (OOB_F_FAST): a heavy query first meets the symbolic Unsat
    // prover (symbolic.cuh) in the frontier phase; refuted = final Unsat
    uint32_t fast;
    unsigned long long* fast_stats;  // [0] heavy queries tried [1] refuted [2,3] cycles [4] certified (null: off)
    // fast mode certificate check (oob_cert_kernel): the job's full class
    // table (ClassDesc::cert) and the certificate words
    const ClassDesc* cert_classes;
    uint32_t cert_nclasses;
    uint32_t cert_kmax;       // most certificates of any class of the job
    const uint64_t* certs;
    // fast mode warp-per-query search of the int64 job's own entries
    // (chain.cuh, before the root kernel): entries [0, chain_n), per-warp DFS
    // frames, node and propagation-round budgets (beyond: the exact path)
    uint32_t chain_n;
    uint32_t chain_nodes;
    uint32_t chain_rounds;
    long long* chain_frames;
    // fast mode K3 (chain.cuh oob_enum_kernel): entries [0, enum_n) whose
    // declared box holds at most enum_max points are enumerated
    uint32_t enum_n;
    uint32_t enum_max;
    // frontier: speculative lanes stop after fr_abort x the leftmost lane's
    // passes (+16) once it has finished (frontier.cuh); 0 = never
    uint32_t fr_abort;
    uint32_t fr_abort_min;
};

enum { MODE_SOLVE = 0, MODE_PROPAGATE = 1, MODE_CHECK = 2 };
constexpr int8_t VERDICT_NONE = -1;  // entry not owned by this job (shadow / demoted)
enum { ERR_NONE = 0, ERR_DEPTH = 1, ERR_TRAIL = 2, ERR_STACK = 3 };

}  // namespace oob
