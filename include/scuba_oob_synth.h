/*
 * scuba_oob_synth.h -- seeded generator of analyzer-shaped OOB queries
 * (measurement harness of the engine; not part of the reference interface).
 *
 * Queries have exactly the shape the reference analyzer emits
 * (constraint_gen.py:105-124 geometry, :278-309 access checks, :186-208
 * context): 12 launch-geometry variables with their 12 range constraints and 6
 * launch equations, solOffset in [-M, M], solSize in [0, M], the check
 * (solOffset >= solSize, or solOffset < 0), the offset and size equations,
 * kernel-parameter bindings, host asserts and path guards -- instantiated from
 * templates modelled on the reference corpus access patterns:
 *   T1 linear tid + bid*bdim vs n with grid = (n + blk - 1) / blk   (saxpy)
 *   T2 constant static extents                                     (static_shared_oob)
 *   T3 product sizes                                               (fluid_adv)
 *   T4 loop-variable bounded                                       (kalman)
 *   T5 dynamic-shared partition differences                        (sosfilt_intra)
 *   T6 data-dependent unknown index                                (push_node)
 *   T7 2-D row * dim + j                                           (lu_decomp)
 * A fraction of instances carry a bug (dropped guard, off-by-one, short
 * allocation).  Query i of a (config, seed) stream depends only on (seed, i),
 * so any slice can be generated independently (sharding, pinning subsets).
 */
#ifndef SCUBA_OOB_SYNTH_H
#define SCUBA_OOB_SYNTH_H

#include <stdint.h>

#include "scuba_oob.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
    OOB_SYNTH_C3 = 3, /* M = 2^31-1, caps 2^3..2^7, 30% buggy                    */
    OOB_SYNTH_C4 = 4, /* M in {2^31-1, 2^59}, caps 2^3..2^10, deeper products     */
    OOB_SYNTH_C5 = 5  /* bug-free only (Unsat by construction); caps given below */
};

/* Per-query size caps of a config: [vars, constraints, nodes, literals]. */
int oob_synth_caps(int config, int64_t caps[4]);

/* Writable flat batch for the generator (arrays sized n * caps[...], offsets
 * n + 1).  name_code[v]: 0-11 geometry axes (ALL_AXES order), 12 solOffset,
 * 13 solSize, 14 + k program unknown k.  tmpl[q] = template * 4 + check
 * (check 0 upper, 1 lower, 2 partition-layout pre-check). */
typedef struct {
    int64_t* var_begin;
    oob_i128* var_lo;
    oob_i128* var_hi;
    int64_t* con_begin;
    uint8_t* con_rel;
    int32_t* con_lhs;
    int32_t* con_rhs;
    int64_t* node_begin;
    uint8_t* node_op;
    int32_t* node_a;
    int32_t* node_b;
    int64_t* lit_begin;
    oob_i128* lits;
    uint16_t* name_code;
    uint8_t* tmpl;
} oob_synth_out;

/* Generate queries [first, first + n) of stream (config, seed).  For C5,
 * `cap_log2` > 0 overrides the input cap (2^cap_log2; default 20). */
int oob_synth_generate(int config, uint64_t seed, int64_t first, int64_t n, int cap_log2,
                       oob_synth_out* out);

#ifdef __cplusplus
}
#endif

#endif /* SCUBA_OOB_SYNTH_H */
