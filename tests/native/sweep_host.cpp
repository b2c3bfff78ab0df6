// TEST INFRASTRUCTURE ONLY: a host build of the device sweep interpreter
// (paper_2601_21552_b200/csrc/sweep_vm.cuh) so the CPU suite can check the
// bytecode compiler and the interpreter's semantics against the reference's
// own brute_force_all / replay_witness (oracle.py:638-720) without a GPU.
// Same C ABI shapes as include/scuba_oob_sweep.h, sequential over tuples.
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/scuba_oob_sweep.h"
#include "../../paper_2601_21552_b200/csrc/sweep_vm.cuh"

static sweep::Prog prog_of(const oob_sweep_program* p) {
    return sweep::Prog{p->code, p->lits, p->kernels, p->kparams, p->n_code, p->n_sites,
                       p->n_slots, p->n_kernels, (int64_t)1 << 40};
}

static int64_t words_of(const oob_sweep_options* o) {
    return (o && o->arena_words > 0) ? o->arena_words : (int64_t)1 << 16;
}

extern "C" int sweep_host_run(const oob_sweep_program* pr, int64_t bound, int32_t arity,
                              const oob_sweep_options* opt, oob_sweep_result* out) {
    const int64_t arena_words = words_of(opt);
    sweep::Prog P = prog_of(pr);
    std::vector<int64_t> arena(arena_words);
    sweep::Arena A{arena.data(), 1, arena_words};
    auto* m = new sweep::Machine();
    int64_t total = 1;
    for (int i = 0; i < arity; i++) total *= bound + 1;
    out->executions = total;
    out->halted = out->errors = 0;
    out->need_tuple = out->need_site = out->error_tuple = -1;
    out->error_code = 0;
    out->arena_words_used = 0;
    for (int s = 0; s < pr->n_sites; s++) {
        out->site_labels[s] = 0;
        for (int l = 0; l < 4; l++) out->site_first_tuple[4 * s + l] = -1;
    }
    int64_t in[sweep::MAX_INPUTS];
    for (int64_t t = 0; t < total; t++) {
        int64_t r = t;
        for (int i = arity - 1; i >= 0; i--) {
            in[i] = r % (bound + 1);
            r /= bound + 1;
        }
        sweep::Out o = sweep::run(P, in, arity, A, *m);
        if (m->arena_peak > out->arena_words_used) out->arena_words_used = m->arena_peak;
        if (o.status == sweep::S_HALT) {
            out->halted++;
        } else if (o.status == sweep::S_ERROR) {
            if (out->errors++ == 0) {
                out->error_tuple = t;
                out->error_code = o.aux;
            }
        } else if (o.status == sweep::S_NEED) {
            if (out->need_tuple < 0) {
                out->need_tuple = t;
                out->need_site = o.aux;
            }
        } else {
            for (int s = 0; s < pr->n_sites; s++) {
                uint32_t bits = (m->labels[(s * 4) >> 5] >> ((s * 4) & 31)) & 15u;
                out->site_labels[s] |= bits;
                for (int l = 0; l < 4; l++)
                    if ((bits >> l & 1) && out->site_first_tuple[4 * s + l] < 0) out->site_first_tuple[4 * s + l] = t;
            }
        }
    }
    delete m;
    return 0;
}

extern "C" int sweep_host_replay(const oob_sweep_program* pr, int64_t n, int32_t arity,
                                 const int64_t* tuples, const oob_sweep_options* opt,
                                 int32_t* status, int32_t* aux, uint8_t* labels) {
    const int64_t arena_words = words_of(opt);
    sweep::Prog P = prog_of(pr);
    std::vector<int64_t> arena(arena_words);
    sweep::Arena A{arena.data(), 1, arena_words};
    auto* m = new sweep::Machine();
    for (int64_t t = 0; t < n; t++) {
        sweep::Out o = sweep::run(P, tuples + t * arity, arity, A, *m);
        status[t] = o.status;
        aux[t] = o.aux;
        for (int s = 0; s < pr->n_sites; s++)
            labels[t * pr->n_sites + s] =
                o.status == sweep::S_OK ? (m->labels[(s * 4) >> 5] >> ((s * 4) & 31)) & 15u : 0;
    }
    delete m;
    return 0;
}
