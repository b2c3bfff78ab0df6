// frontier.cuh -- warp-cooperative DFS for heavy queries (K1, second stage).
//
// The lockstep kernel hands a query off after `heavy_nodes` DFS nodes (or
// `heavy_passes` propagation passes: a long chain gets a warp of its own).  Here
// one warp owns one heavy query and its 32 lanes expand the 32 LEFTMOST
// pending nodes of the reference's DFS tree (solver.py:385-416) at once:
//
//   * pending nodes live on a unit stack in DFS order (top = leftmost); a unit
//     is (entry, half) where an entry holds a split node's narrowed domains,
//     its split variable and midpoint, its clean mask and its tree path;
//   * a round pops k <= 32 units, lane i expanding the i-th leftmost; every
//     lane runs the node's full propagate() pass-synchronously with the other
//     lanes (same class, so constraint code is warp-uniform);
//   * children are pushed back so the stack stays in DFS order;
//   * the first (lowest-lane) Sat leaf of a round is a candidate: everything
//     to its right -- the other lanes' children and the rest of the stack --
//     is discarded, so the search ends with the LEFTMOST Sat leaf, exactly
//     the model the sequential reference returns;
//   * every expanded node is logged with its path; when the answer is Sat the
//     reported node / pass counters are summed over the nodes that precede
//     the leaf in pre-order (what the sequential search would have visited),
//     so they too equal the reference's.
#pragma once
#include "engine.cuh"

namespace oob {

constexpr uint32_t UNIT_ROOT = 0xFFFFFFFFu;

template <typename T>
struct FrontierRegion {
    T* e_env;          // [ecap][2 * maxv]  (lo, hi) pairs of the parent's narrowed domains
    T* e_mid;          // [ecap]
    T* e_hi;           // [ecap]
    uint64_t* e_path;  // [ecap][2]  bit d = 1: the right half was taken at depth d
    uint64_t* log_path;  // [logcap][2]
    uint32_t* e_pick;  // [ecap]
    uint32_t* e_depth; // [ecap]
    uint32_t* e_clean; // [ecap][4]
    uint32_t* units;   // [ucap]
    uint32_t* freel;   // [ecap]
    uint32_t* log_meta;  // [logcap][2]  depth, passes

    __device__ void bind(unsigned char* base, uint32_t maxv, uint32_t ecap, uint32_t ucap, uint32_t logcap) {
        unsigned char* p = base;
        e_env = (T*)p; p += (size_t)ecap * 2 * maxv * sizeof(T);
        e_mid = (T*)p; p += (size_t)ecap * sizeof(T);
        e_hi = (T*)p; p += (size_t)ecap * sizeof(T);
        e_path = (uint64_t*)p; p += (size_t)ecap * 16;
        log_path = (uint64_t*)p; p += (size_t)logcap * 16;
        e_pick = (uint32_t*)p; p += (size_t)ecap * 4;
        e_depth = (uint32_t*)p; p += (size_t)ecap * 4;
        e_clean = (uint32_t*)p; p += (size_t)ecap * 16;
        units = (uint32_t*)p; p += (size_t)ucap * 4;
        freel = (uint32_t*)p; p += (size_t)ecap * 4;
        log_meta = (uint32_t*)p;
    }
};

// pre-order comparison of tree paths: does (pa, da) come no later than (pb, db)?
__device__ __forceinline__ bool path_le(uint64_t a0, uint64_t a1, uint32_t da, uint64_t b0, uint64_t b1,
                                        uint32_t db) {
    uint64_t x0 = a0 ^ b0, x1 = a1 ^ b1;
    uint32_t common = min(da, db);
    uint32_t first;  // first differing depth
    if (x0) first = __ffsll((long long)x0) - 1;
    else if (x1) first = 64 + __ffsll((long long)x1) - 1;
    else first = 128;
    if (first >= common) return da <= db;  // one is an ancestor of (or equal to) the other
    uint32_t abit = first < 64 ? (uint32_t)((a0 >> first) & 1) : (uint32_t)((a1 >> (first - 64)) & 1);
    return abit == 0;  // a went left where b went right
}

enum : int { FN_DEAD = 0, FN_SAT = 1, FN_SPLIT = 2, FN_NONE = 3 };

template <typename LaneT>
__device__ void frontier_query(LaneT& L, const LaunchArgs& a, FrontierRegion<typename LaneT::T>& R, uint32_t qi,
                               uint32_t lane) {
    using T = typename LaneT::T;
    const unsigned FULL = 0xffffffffu;
    const QDesc d = a.qdesc[qi];
    const uint32_t nv = L.nvars();
    const uint32_t ecap = a.fr_ecap, ucap = a.fr_ucap, logcap = a.fr_logcap;
    const uint64_t t0 = a.heavy_t0[qi];
    const uint64_t deadline = a.timeout_ns ? t0 + a.timeout_ns : 0;
    const uint32_t rs = a.resume ? a.resume[qi] : 0u;  // demoted: the root resumes (format.h)

    uint32_t nunits = 1, nfree = 0, ebump = 0, nlog = 0;
    if (lane == 0) R.units[0] = UNIT_ROOT;
    bool have_sat = false;
    uint64_t sat_p0 = 0, sat_p1 = 0;
    uint32_t sat_depth = 0;
    int64_t tot_nodes = 0, tot_passes = 0;
    int status = VERDICT_UNSAT;  // UNSAT / TIMEOUT / ERROR at the end
    int err = ERR_NONE;
    __syncwarp();

    while (nunits > 0) {
        if (a.node_budget > 0 && tot_nodes >= a.node_budget) {
            status = VERDICT_TIMEOUT;
            break;
        }
        // ---- take the k leftmost pending units ----
        uint32_t room_e = ecap - ebump + nfree, room_u = ucap - nunits;
        uint32_t k = min(min(32u, nunits), min(room_e, room_u));
        if (k == 0) {
            status = VERDICT_ERROR;
            err = ERR_DEPTH;
            break;
        }
        const bool has = lane < k;
        uint64_t p0 = 0, p1 = 0;
        uint32_t depth = 0, freed = 0xFFFFFFFFu, u = 0;
        bool resumed_root = false;
        if (has) {
            u = R.units[nunits - 1 - lane];
            L.depth = 0;  // no trail: every lane owns its node's domains
            L.clean0 = L.clean1 = 0;
            L.err = ERR_NONE;
            resumed_root = (u == UNIT_ROOT) && (rs & RES_ROOT);
            if (u != UNIT_ROOT) {
                uint32_t e = u >> 1, half = u & 1;
                const T* env = R.e_env + (size_t)e * 2 * nv;
                L.load_env(env);
                const uint32_t* c = R.e_clean + (size_t)e * 4;
                L.clean0 = ((uint64_t)c[1] << 32) | c[0];
                L.clean1 = ((uint64_t)c[3] << 32) | c[2];
                uint32_t pick = R.e_pick[e];
                uint32_t pd = R.e_depth[e];
                p0 = R.e_path[2 * e];
                p1 = R.e_path[2 * e + 1];
                if (half) {
                    if (pd < 64) p0 |= 1ull << pd;
                    else p1 |= 1ull << (pd - 64);
                    L.set_dom(pick, R.e_mid[e] + T(1), R.e_hi[e]);
                    freed = e;  // both units of e are consumed after this round
                } else {
                    L.set_dom(pick, L.get_lo(pick), R.e_mid[e]);
                }
                depth = pd + 1;
            }
        }
        __syncwarp();
        nunits -= k;
        // ---- expand: node start + pass-synchronous propagate() ----
        int outcome = FN_NONE;
        int64_t my_passes = resumed_root ? (int64_t)(rs & RES_PASSES) : 0;
        const int pin0 = (int)my_passes;
        bool prop = has && !(resumed_root && (rs & RES_FIX));
        if (__any_sync(FULL, has && deadline && global_ns() > deadline)) {
            status = VERDICT_TIMEOUT;
            break;
        }
        bool dead = false;
        // speculative lanes (right of the leftmost) stop once the leftmost
        // lane has finished and the round has run fr_abort times its passes
        // (+fr_abort_min): their units go back on the stack unexpanded, so a creeping
        // right sibling no longer holds up the leftmost path (a.fr_abort 0:
        // every lane runs to its fixpoint)
        bool aborted = false;
        int l0_end = -1;
        for (int pin = 0; __any_sync(FULL, prop); ++pin) {
            if (a.fr_abort) {
                if (l0_end < 0 && !__shfl_sync(FULL, prop ? 1 : 0, 0)) l0_end = pin;
                if (l0_end >= 0 && pin >= (int)a.fr_abort * l0_end + (int)a.fr_abort_min && prop) {
                    aborted = true;
                    prop = false;
                }
                if (!__any_sync(FULL, prop)) break;
            }
            if (prop) {
                if (pin + pin0 >= PASS_CAP) {
                    prop = false;
                } else {
                    ++my_passes;
                    L.changed = false;
                }
            }
            bool run = prop;
            if (L.pass_sync(run && !dead)) dead = true;
            if (run && (dead || !L.changed)) prop = false;
            if (__any_sync(FULL, run && deadline && global_ns() > deadline)) {
                status = VERDICT_TIMEOUT;
                break;
            }
        }
        if (status == VERDICT_TIMEOUT) break;
        // lanes from the first aborted one on are re-pushed unexpanded (a Sat
        // leaf right of an unexpanded unit need not be the leftmost one)
        const unsigned abm = __ballot_sync(FULL, aborted);
        const uint32_t cut = abm ? (uint32_t)(__ffs(abm) - 1) : 32u;
        const bool live = has && lane < cut;
        const bool repush = has && lane >= cut;
        // free the entries whose right unit was consumed
        {
            const bool fr = live && freed != 0xFFFFFFFFu;
            unsigned fm = __ballot_sync(FULL, fr);
            if (fr) R.freel[nfree + __popc(fm & ((1u << lane) - 1u))] = freed;
            nfree += __popc(fm);
        }
        uint32_t pick = 0;
        if (live) {
            if (L.err) {
                outcome = FN_DEAD;
                err = L.err;
            } else if (dead) {
                outcome = FN_DEAD;
            } else {
                int pk = L.pick_var();
                if (pk < 0) {
                    outcome = L.check_env() ? FN_SAT : FN_DEAD;
                } else {
                    outcome = FN_SPLIT;
                    pick = (uint32_t)pk;
                }
            }
        }
        if (__any_sync(FULL, live && L.err != ERR_NONE)) {
            status = VERDICT_ERROR;
            err = ERR_STACK;
            break;
        }
        // ---- log the expanded nodes (pre-order accounting) ----
        // paths hold 128 levels and the log `logcap` nodes: beyond that the
        // query ends with ERR_DEPTH and the host decides it again on the
        // sequential path with more scratch (counters stay exact)
        if (__any_sync(FULL, live && depth >= 128) || nlog + k > logcap) {
            status = VERDICT_ERROR;
            err = ERR_DEPTH;
            break;
        }
        {
            unsigned hm = __ballot_sync(FULL, live);  // a prefix of the lanes
            if (live) {
                uint32_t at = nlog + lane;
                R.log_path[2 * at] = p0;
                R.log_path[2 * at + 1] = p1;
                R.log_meta[2 * at] = depth;
                R.log_meta[2 * at + 1] = (uint32_t)my_passes;
            }
            nlog += __popc(hm);
            tot_nodes += __popc(hm);
            tot_passes += __reduce_add_sync(FULL, live ? (unsigned)my_passes : 0u);
        }
        // ---- Sat: the leftmost candidate wins; everything right of it goes ----
        unsigned sm = __ballot_sync(FULL, outcome == FN_SAT);
        uint32_t limit = 32;
        if (sm) {
            int j = __ffs(sm) - 1;
            limit = (uint32_t)j;
            if ((int)lane == j) {
                int64_t* m = a.model + 2 * d.out_v;
                L.store_model(m);
            }
            sat_p0 = __shfl_sync(FULL, p0, j);
            sat_p1 = __shfl_sync(FULL, p1, j);
            sat_depth = __shfl_sync(FULL, depth, j);
            have_sat = true;
            nunits = 0;  // the rest of the stack lies to the right of the leaf
        }
        // ---- push the children of splitting lanes left of the cut ----
        __syncwarp();  // freed entries written above are read below by other lanes
        const bool splits = outcome == FN_SPLIT && lane < limit;
        unsigned spm = __ballot_sync(FULL, splits);
        const unsigned rpm = sm ? 0u : __ballot_sync(FULL, repush);  // (a Sat cut drops them)
        uint32_t s = __popc(spm);
        const unsigned right = ~((2u << lane) - 1u);
        if (repush && !sm) R.units[nunits + 2 * __popc(spm & right) + __popc(rpm & right)] = u;
        if (splits) {
            uint32_t r = __popc(spm & ((1u << lane) - 1u));        // rank from the left
            uint32_t h = 2 * __popc(spm & right) + __popc(rpm & right);  // stack slots to my right
            uint32_t e = r < nfree ? R.freel[nfree - 1 - r] : ebump + (r - nfree);
            T* env = R.e_env + (size_t)e * 2 * nv;
            L.store_env(env);
            T lo = L.get_lo(pick), hi = L.get_hi(pick);
            R.e_mid[e] = (lo + hi) >> 1;  // floor midpoint (solver.py:409)
            R.e_hi[e] = hi;
            R.e_pick[e] = pick;
            R.e_depth[e] = depth;
            R.e_path[2 * e] = p0;
            R.e_path[2 * e + 1] = p1;
            uint32_t* c = R.e_clean + (size_t)e * 4;
            c[0] = (uint32_t)L.clean0;
            c[1] = (uint32_t)(L.clean0 >> 32);
            c[2] = (uint32_t)L.clean1;
            c[3] = (uint32_t)(L.clean1 >> 32);
            R.units[nunits + h] = (e << 1) | 1u;          // upper half, below
            R.units[nunits + h + 1] = (e << 1);           // lower half, on top
        }
        uint32_t from_free = min(s, nfree);
        nfree -= from_free;
        ebump += s - from_free;
        nunits += 2 * s + __popc(rpm);
        __syncwarp();
    }
    // ---- result ----
    int verdict = status;
    if (status == VERDICT_UNSAT && have_sat) verdict = VERDICT_SAT;
    int64_t out_nodes = tot_nodes, out_passes = tot_passes;
    if (verdict == VERDICT_SAT) {
        uint32_t cn = 0;
        uint64_t cp = 0;
        for (uint32_t i = lane; i < nlog; i += 32) {
            if (path_le(R.log_path[2 * i], R.log_path[2 * i + 1], R.log_meta[2 * i], sat_p0, sat_p1, sat_depth)) {
                ++cn;
                cp += R.log_meta[2 * i + 1];
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            cn += __shfl_xor_sync(FULL, cn, o);
            cp += __shfl_xor_sync(FULL, cp, o);
        }
        out_nodes = cn;
        out_passes = (int64_t)cp;
    }
    if (a.stats && lane == 0) {  // [6,7] Sat: expanded / reference passes, [8,9] Unsat
        const int o = verdict == VERDICT_SAT ? 6 : 8;
        atomicAdd(a.stats + o, (unsigned long long)tot_passes);
        atomicAdd(a.stats + o + 1, (unsigned long long)out_passes);
    }
    if (lane == 0) {
        a.verdict[qi] = (int8_t)verdict;
        a.err[qi] = (int8_t)err;
        a.nodes[qi] = out_nodes;
        a.passes[qi] = out_passes;
        a.elapsed[qi] = (float)((double)(global_ns() - t0) * 1e-9);
        if (a.timeline) a.timeline[4 * (size_t)qi + 3] = global_ns();
    }
    __syncwarp();
}

}  // namespace oob
