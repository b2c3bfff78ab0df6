/*
 * scuba_oob_sweep.h -- C ABI of the device exhaustive oracle: brute-force
 * input sweeps and witness replay of MiniCUDA programs on one B200.
 *
 * Replaces, for the data-parallel part, the reference's program-level oracle
 *   brute_force_all(program, bound, stop_when_violated)
 *       /root/reference/pkg/src/scuba_mini/oracle.py:638-681
 *   brute_force_verdict(program, line, column, bound)   oracle.py:684-692
 *   replay_witness(program, input_values, default, line, column)
 *       oracle.py:695-720
 * which run the AST interpreter (oracle.py:260-580) once per input tuple.
 * The program arrives lowered to the flat bytecode of
 * paper_2601_21552_b200/sweep.py (compile_program); the arity-growth loop
 * (NeedMoreInput, oracle.py:675-680) stays with the caller, which gets the
 * first tuple that needed another input.
 *
 * Errors: int status (0 ok, see scuba_oob.h OOB_E_*) + oob_last_error().  A
 * tuple the device cannot execute exactly (a value beyond int64, arena or
 * table capacity after automatic arena growth, step limit) fails the whole
 * call -- never a silently different sweep.
 */
#ifndef SCUBA_OOB_SWEEP_H
#define SCUBA_OOB_SWEEP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t n_code;
    const int32_t* code;     /* n_code x 4: op, a, b, c (sweep.py OPS)           */
    int32_t n_lits;
    const int64_t* lits;
    int32_t n_kernels;
    const int32_t* kernels;  /* n_kernels x 4: entry pc, n_params, param off, n_shared */
    int32_t n_kparams;
    const int32_t* kparams;  /* n_kparams x 2: slot, kind (0 scalar, 1 pointer)  */
    int32_t n_sites;         /* access/free sites (line, column) of the program  */
    int32_t n_slots;
    int32_t n_input_sites;   /* count_input_sites (oracle.py:621-628)            */
} oob_sweep_program;

typedef struct {
    int32_t device;
    int64_t arena_words;     /* per-tuple cell arena; 0 = default, grows on demand */
    int64_t step_limit;      /* bytecode steps per tuple; 0 = 2^40               */
    int64_t max_threads;     /* resident device threads; 0 = fill the GPU         */
} oob_sweep_options;

typedef struct {
    int64_t executions;      /* (bound+1)^arity                                   */
    int64_t halted;          /* executions that halted (oracle.py:660-662)        */
    int64_t errors;          /* 0 on success                                      */
    int64_t need_tuple;      /* first tuple (product order) needing another input, -1 */
    int64_t need_site;       /* the input site it needed                          */
    int64_t error_tuple;
    int32_t error_code;
    int64_t arena_words_used;
    uint32_t* site_labels;      /* caller-allocated [n_sites]: label bits seen     */
    int64_t* site_first_tuple;  /* caller-allocated [n_sites][4]: first tuple index
                                   per label (upper, underflow, uaf, double-free), -1 */
    float device_ms;
} oob_sweep_result;

/* Sweep every tuple of [0, bound]^arity (itertools.product order: tuple t has
 * digit i = (t / (bound+1)^(arity-1-i)) % (bound+1)).  Violations of halted
 * executions are discarded. */
int oob_sweep_run(const oob_sweep_program* prog, int64_t bound, int32_t arity,
                  const oob_sweep_options* opt, oob_sweep_result* out);

/* Execute n explicit tuples of `arity` inputs each (row-major).  Per tuple:
 * status (0 ok, 1 halted, 2 needs input site aux, 3 error aux), aux (halt
 * reason code / site / error code) and labels[n][n_sites] (bits: 1 upper,
 * 2 underflow, 4 uaf, 8 double-free; zero when halted). */
int oob_sweep_replay(const oob_sweep_program* prog, int64_t n, int32_t arity,
                     const int64_t* tuples, const oob_sweep_options* opt,
                     int32_t* status, int32_t* aux, uint8_t* labels);

#ifdef __cplusplus
}
#endif
#endif
