// TEST INFRASTRUCTURE ONLY: a host build of the fast mode's Unsat prover
// (paper_2601_21552_b200/csrc/symbolic.cuh), sequential over queries and
// target inequalities, so the CPU suite can check its soundness (never
// refutes a query the reference decides Sat) and its reach (which Unsat
// queries it refutes) on the golden records without a GPU.  The flat batch's
// term DAG is expanded into the device's postfix class code (format.h) here;
// divisor side constraints are not appended (fewer constraints: still sound).
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

#include "../../include/scuba_oob.h"
#include "../../paper_2601_21552_b200/csrc/symbolic.cuh"

namespace {

typedef __int128 i128;

i128 w128(const oob_i128& w) { return (i128)(((unsigned __int128)(uint64_t)w.hi << 64) | w.lo); }

struct Emit {
    const oob_batch* b;
    int64_t nb, lb;
    std::vector<uint32_t> code;
    std::vector<i128> lits;
    uint32_t node(int32_t i) {  // returns subtree size
        const int op = b->node_op[nb + i];
        if (op == OOB_NODE_LIT) {
            code.push_back(oob::node_word(OOB_NODE_LIT, (uint32_t)lits.size()));
            lits.push_back(w128(b->lits[lb + b->node_a[nb + i]]));
            return 1;
        }
        if (op == OOB_NODE_VAR) {
            code.push_back(oob::node_word(OOB_NODE_VAR, (uint32_t)b->node_a[nb + i]));
            return 1;
        }
        const uint32_t sa = node(b->node_a[nb + i]);
        const uint32_t sb = node(b->node_b[nb + i]);
        code.push_back(oob::node_word((uint32_t)op, 1 + sa + sb));
        return 1 + sa + sb;
    }
};

}  // namespace

// refuted[q] = 1: the prover derived a contradiction (Unsat); 0: unknown
extern "C" int sym_host_refute(const oob_batch* b, int8_t* refuted) {
    auto S = std::make_unique<oob::sym::Store>();
    auto W = std::make_unique<oob::sym::LaneWork>();
    for (int64_t q = 0; q < b->n_queries; ++q) {
        Emit e{b, b->node_begin[q], b->lit_begin[q], {}, {}};
        std::vector<uint32_t> cons;
        for (int64_t k = b->con_begin[q]; k < b->con_begin[q + 1]; ++k) {
            e.node(b->con_lhs[k]);
            const uint32_t lr = (uint32_t)e.code.size() - 1;
            e.node(b->con_rhs[k]);
            const uint32_t rr = (uint32_t)e.code.size() - 1;
            cons.push_back(oob::con_word(b->con_rel[k], lr, rr));
        }
        const int64_t vb = b->var_begin[q];
        const uint32_t nv = (uint32_t)(b->var_begin[q + 1] - vb);
        auto dom = [&](uint32_t i) -> i128 { return w128(i % 2 ? b->var_hi[vb + i / 2] : b->var_lo[vb + i / 2]); };
        auto lit = [&](uint32_t i) -> i128 { return e.lits[i]; };
        refuted[q] = oob::sym::refute_serial(*S, *W, cons.data(), e.code.data(), nv, (uint32_t)cons.size(), dom, lit);
    }
    return 0;
}

// Certificates (csrc/cert.cuh): one per structure class, compiled from up to
// `reps` representatives with the varying literal slots as parameters, then
// checked numerically for every query of the class (the device's job).
// refuted[q] = 1: refuted by its class certificate.  stats[0] classes,
// [1] classes with a certificate, [2] total certificate words.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include "../../paper_2601_21552_b200/csrc/cert.cuh"

extern "C" int sym_host_cert(const oob_batch* b, int32_t reps, int8_t* refuted, int64_t* stats) {
    struct Q {
        std::vector<uint32_t> cons, code;
        std::vector<i128> lits;
        uint32_t nv;
    };
    std::vector<Q> qs(b->n_queries);
    std::map<std::vector<uint32_t>, std::vector<int64_t>> classes;
    for (int64_t q = 0; q < b->n_queries; ++q) {
        Emit e{b, b->node_begin[q], b->lit_begin[q], {}, {}};
        for (int64_t k = b->con_begin[q]; k < b->con_begin[q + 1]; ++k) {
            e.node(b->con_lhs[k]);
            const uint32_t lr = (uint32_t)e.code.size() - 1;
            e.node(b->con_rhs[k]);
            const uint32_t rr = (uint32_t)e.code.size() - 1;
            qs[q].cons.push_back(oob::con_word(b->con_rel[k], lr, rr));
        }
        qs[q].code = e.code;
        qs[q].lits = e.lits;
        qs[q].nv = (uint32_t)(b->var_begin[q + 1] - b->var_begin[q]);
        std::vector<uint32_t> key = qs[q].cons;
        key.insert(key.end(), qs[q].code.begin(), qs[q].code.end());
        key.push_back(qs[q].nv);
        classes[key].push_back(q);
    }
    auto S = std::make_unique<oob::sym::Store>();
    auto W = std::make_unique<oob::sym::LaneWork>();
    auto M = std::make_unique<oob::sym::Moves>();
    auto B = std::make_unique<oob::cert::BoxV>();
    std::vector<uint64_t> blob(1 << 16);
    int64_t ncls = 0, ncert = 0, words = 0;
    for (auto& kv : classes) {
        const std::vector<int64_t>& mem = kv.second;
        ++ncls;
        const Q& r0 = qs[mem[0]];
        const uint32_t nlit = (uint32_t)r0.lits.size();
        std::vector<int16_t> pmap(nlit, -1), pslot;
        for (uint32_t i = 0; i < nlit; ++i)
            for (int64_t q : mem)
                if (qs[q].lits[i] != r0.lits[i]) {
                    pmap[i] = (int16_t)pslot.size();
                    pslot.push_back((int16_t)i);
                    break;
                }
        std::vector<std::vector<uint64_t>> certs;
        const int nr = std::max(1, std::min<int>(reps, (int)mem.size()));
        // the member with the widest domains first (as the engine does)
        int64_t widest = mem[0];
        auto width_bits = [&](int64_t q) {
            double w = 0;
            for (int64_t v = b->var_begin[q]; v < b->var_begin[q + 1]; ++v) {
                const i128 d = w128(b->var_hi[v]) - w128(b->var_lo[v]);
                w += d > 0 ? std::log2((double)d + 1.0) : 0.0;
            }
            return w;
        };
        for (int64_t q : mem)
            if (width_bits(q) > width_bits(widest)) widest = q;
        for (int ri = 0; ri <= nr; ++ri) {
            const int64_t rq = ri == 0 ? widest : mem[(size_t)(ri - 1) * mem.size() / nr];
            if (ri > 0 && rq == widest) continue;
            const Q& r = qs[rq];
            const int64_t vb = b->var_begin[rq];
            auto dom = [&](uint32_t i) -> i128 { return w128(i % 2 ? b->var_hi[vb + i / 2] : b->var_lo[vb + i / 2]); };
            auto lit = [&](uint32_t i) -> i128 { return r.lits[i]; };
            const size_t n = oob::cert::cert_build(*S, *W, *M, r.cons.data(), r.code.data(), r.nv,
                                                   (uint32_t)r.cons.size(), nlit, dom, lit, pmap.data(),
                                                   (int)pslot.size(), pslot.data(), blob.data(), blob.size());
            if (!n && getenv("SYM_DEBUG")) fprintf(stderr, "class of q%ld: no certificate from q%ld (line %d)\n", (long)mem[0], (long)rq, oob::cert::cert_fail_line());
            if (n) {
                std::vector<uint64_t> c(blob.begin(), blob.begin() + n);
                bool dup = false;
                for (auto& o : certs) dup = dup || o == c;
                if (!dup) certs.push_back(c);
            }
        }
        if (!certs.empty()) ++ncert;
        for (auto& c : certs) words += (int64_t)c.size();
        for (int64_t q : mem) {
            const int64_t vb = b->var_begin[q];
            auto dom = [&](uint32_t i) -> i128 { return w128(i % 2 ? b->var_hi[vb + i / 2] : b->var_lo[vb + i / 2]); };
            auto lit = [&](uint32_t i) -> i128 { return qs[q].lits[i]; };
            refuted[q] = 0;
            int why = 0;
            for (auto& c : certs)
                if (oob::cert::cert_check(c.data(), dom, lit, *B, &why) == oob::cert::C_REFUTED) {
                    refuted[q] = 1;
                    break;
                }
            if (!refuted[q] && getenv("SYM_DEBUG2")) fprintf(stderr, "q%ld class-of q%ld certs %zu why %d\n", (long)q, (long)mem[0], certs.size(), why);
        }
    }
    if (stats) {
        stats[0] = ncls;
        stats[1] = ncert;
        stats[2] = words;
    }
    return 0;
}
extern "C" int sym_host_cert_fail_line() { return oob::cert::cert_fail_line(); }

// Host check of the ENGINE's compiled certificates (oob_cert_compile): for
// every query, its class's certificates against its own domains and literal
// slots.  refuted[q] = 1 when one refutes; why[q] = the checker's stop reason.
extern "C" int sym_host_check_engine_certs(const oob_batch* b, const uint64_t* words, const int64_t* cert_off,
                                           const oob_i128* slots, const int64_t* slot_begin, int8_t* refuted,
                                           int8_t* why) {
    auto B = std::make_unique<oob::cert::BoxV>();
    for (int64_t q = 0; q < b->n_queries; ++q) {
        refuted[q] = 0;
        why[q] = 0;
        if (cert_off[q] < 0) continue;
        const int64_t vb = b->var_begin[q];
        auto dom = [&](uint32_t i) -> i128 { return w128(i % 2 ? b->var_hi[vb + i / 2] : b->var_lo[vb + i / 2]); };
        auto lit = [&](uint32_t i) -> i128 { return w128(slots[slot_begin[q] + i]); };
        const uint64_t* c = words + cert_off[q];
        const uint64_t n = *c++;
        for (uint64_t k = 0; k < n && !refuted[q]; ++k) {
            const uint64_t len = *c++;
            int w = 0;
            refuted[q] = oob::cert::cert_check(c, dom, lit, *B, &w) == oob::cert::C_REFUTED;
            why[q] = (int8_t)w;
            c += len;
        }
    }
    return 0;
}
