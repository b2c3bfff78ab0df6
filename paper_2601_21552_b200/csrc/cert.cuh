// cert.cuh -- Unsat certificates per structure class (fast mode).
//
// The symbolic prover (symbolic.cuh) is serial, branchy polynomial algebra: a
// poor fit for a GPU lane, and the same algebra would be redone for every
// query of a structure class -- queries that differ only in domain and literal
// VALUES.  So the algebra is compiled once per class on the host, with every
// literal slot whose value varies inside the class kept as a PARAMETER (a
// variable whose box is the point [value, value]), and the device only checks
// the resulting certificate numerically, one lane per query:
//
//   1. box: the query's declared domains, its parameter values, then every
//      atom's interval (division / modulo subterms, in creation order);
//   2. guards0 (>= 0 on that box): the conditions under which the atoms'
//      truncation constraints hold (dividend sign, literal divisor >= 1);
//   3. tighten: ROUNDS rounds of bound propagation over the compiled
//      constraints (entries g = k*v + s: k*v >= -max(s)); an empty box or a
//      constraint with a negative upper bound refutes;
//   4. guards1 (>= 0 on the tightened box): the multipliers of the
//      elimination steps of the proof found for the class's representative;
//   5. final: the proof's last polynomial P = k*P_t + sum m_i*G_i is >= 0 at
//      every solution when the guards hold; an upper bound < 0 refutes.
// Every step is sound for ANY values of the class's queries (the certificate
// is an identity between polynomials in the variables and parameters); a
// query whose guards fail is simply not refuted here.
//
// Blob layout (u64 words): see cert_check() -- header, parameter slots,
// folded constant slots (slot, value: checked per query), atoms, domain
// guards of eliminated variables, guards0, tighten entries, direct
// constraints, guards1, final.
// Polynomial: n, then n x (key, coef lo, coef hi).
#pragma once
#include "symbolic.cuh"

namespace oob {
namespace cert {

using sym::i128;
#if defined(__CUDA_ARCH__)
#define CERT_INL __forceinline__
#else
#define CERT_INL inline
#endif
constexpr uint64_t MAGIC = 0x4345525431ull;  // "CERT1"
constexpr int MAXB = 48;                     // box entries (variables + parameters + atoms)
constexpr uint64_t KCONST = 1ull << 32;      // tighten entry flag: the coefficient K is a constant

// ---- checker (one query; host build in tests, device in the cert kernel) ----
struct BoxV {  // [0, np) parameters, [np, np + nv) variables, then atoms
    // int64 storage (half the per-lane local memory of __int128): a query
    // with a bound beyond int64 is left to the search (never refuted here);
    // every product and sum is still exact __int128 (sym::smul / sadd)
    long long lo[MAXB], hi[MAXB];
    int np;
};
OOB_HD CERT_INL bool fits64(i128 x) { return x == (i128)(long long)x; }
// sym::fdiv / sym::tdiv with a 64-bit path: the 128-bit division is a long
// software loop on the device, and the checked values are mostly small
OOB_HD CERT_INL i128 fdiv64(i128 a, i128 b) {  // floor(a / b), b > 0
    if (b == 1) return a;
    const long long al = (long long)a, bl = (long long)b;
    if ((i128)al == a && (i128)bl == b) {
        long long q = al / bl;
        if ((al % bl != 0) && (al < 0)) --q;
        return q;
    }
    return sym::fdiv(a, b);
}
OOB_HD CERT_INL i128 tdiv64(i128 a, i128 b) {  // C truncation, b != 0
    if (b == 1) return a;
    const long long al = (long long)a, bl = (long long)b;
    if ((i128)al == a && (i128)bl == b && !(bl == -1 && al == (long long)(1ull << 63))) return al / bl;
    return sym::tdiv(a, b);
}

OOB_HD CERT_INL bool mono_iv_b(uint64_t k, const BoxV& B, i128& rl, i128& rh) {
    if (!(k << 8)) {  // a constant or a single variable (most terms)
        if (!k) {
            rl = rh = 1;
        } else {
            rl = B.lo[(k >> 56) - 1];
            rh = B.hi[(k >> 56) - 1];
        }
        return true;
    }
    rl = rh = 1;
    while (k >> 56) {
        const int v = (int)(k >> 56) - 1;
        int e = 0;
        while ((k >> 56) == (uint64_t)(v + 1)) {
            ++e;
            k <<= 8;
        }
        i128 pl, ph;
        if (!sym::ivpow(B.lo[v], B.hi[v], e, pl, ph) || !sym::ivmul(rl, rh, pl, ph, rl, rh)) return false;
    }
    return true;
}
// key without its parameter bytes; pv = the product of the parameters' values
OOB_HD CERT_INL uint64_t kstrip_b(uint64_t k, const BoxV& B, i128& pv, bool& ok) {
    uint64_t r = 0;
    int n = 0;
    pv = 1;
    while (k >> 56) {
        const uint64_t x = k >> 56;
        k <<= 8;
        if ((int)x <= B.np) {
            if (!sym::smul(pv, B.lo[x - 1], pv)) ok = false;
        } else {
            r |= x << (56 - 8 * n);
            ++n;
        }
    }
    return r;
}
// interval of the blob polynomial at p (advances p past it); parameter runs
// are collapsed first (sym::peval)
OOB_HD CERT_INL bool peval_blob(const uint64_t*& p, const BoxV& B, i128& lo, i128& hi) {
    const uint64_t n = *p++;
    const uint64_t* t = p;
    p += 3 * n;
    lo = hi = 0;
    auto coef = [&](uint64_t i) { return (i128)(((unsigned __int128)t[3 * i + 2] << 64) | t[3 * i + 1]); };
    if (B.np == 0) {  // no parameters: one term per monomial
        for (uint64_t i = 0; i < n; ++i) {
            const i128 c = coef(i);
            i128 a, b, x, y;
            if (!mono_iv_b(t[3 * i], B, a, b) || !sym::smul(c, a, x) || !sym::smul(c, b, y)) return false;
            if (c < 0) {
                i128 w = x;
                x = y;
                y = w;
            }
            if (!sym::sadd(lo, x, lo) || !sym::sadd(hi, y, hi)) return false;
        }
        return true;
    }
    for (uint64_t i = 0; i < n;) {
        bool ok = true;
        i128 pv, c = 0, u;
        const uint64_t rk = kstrip_b(t[3 * i], B, pv, ok);
        if (!ok || !sym::smul(coef(i), pv, u) || !sym::sadd(c, u, c)) return false;
        ++i;
        while (i < n) {
            const uint64_t rk2 = kstrip_b(t[3 * i], B, pv, ok);
            if (rk2 != rk) break;
            if (!ok || !sym::smul(coef(i), pv, u) || !sym::sadd(c, u, c)) return false;
            ++i;
        }
        if (c == 0) continue;
        i128 a, b, x, y;
        if (!mono_iv_b(rk, B, a, b) || !sym::smul(c, a, x) || !sym::smul(c, b, y)) return false;
        if (c < 0) {
            i128 w = x;
            x = y;
            y = w;
        }
        if (!sym::sadd(lo, x, lo) || !sym::sadd(hi, y, hi)) return false;
    }
    return true;
}
OOB_HD CERT_INL void skip_poly(const uint64_t*& p) { p += 1 + 3 * p[0]; }

enum : int { C_UNKNOWN = 0, C_REFUTED = 1 };

// dom(i): declared domain word i (lo/hi interleaved), lit(slot): literal slot
template <typename GetDom, typename GetLit>
OOB_HD CERT_INL int cert_check(const uint64_t* p, GetDom dom, GetLit lit, BoxV& B, int* why = nullptr) {
    int dummy;
    int& reason = why ? *why : dummy;  // 1 header 2 values 3 atoms 4 guards0 5 guards1 6 final
    if (p[0] != MAGIC) return C_UNKNOWN;
    const int nb = (int)(p[1] & 0xFFFF), nv = (int)((p[1] >> 16) & 0xFFFF), np = (int)((p[1] >> 32) & 0xFFFF),
              na = (int)(p[1] >> 48);
    reason = 1;
    if (nb > MAXB || nv + np + na != nb) return C_UNKNOWN;
    p += 2;
    reason = 2;
    B.np = np;
    for (int q = 0; q < np; ++q) {
        const i128 x = lit((uint32_t)p[q]);
        if (!fits64(x)) return C_UNKNOWN;
        B.lo[q] = B.hi[q] = (long long)x;
    }
    p += np;
    // literal slots the certificate folded as numbers must hold exactly those
    // numbers in this query (the certificate is an identity for its class's
    // structure with these constants)
    for (uint64_t k = *p++; k > 0; --k, p += 3) {
        const i128 want = (i128)(((unsigned __int128)p[2] << 64) | p[1]);
        if (lit((uint32_t)p[0]) != want) return C_UNKNOWN;
    }
    for (int v = 0; v < nv; ++v) {
        const i128 a = dom(2 * v), b = dom(2 * v + 1);
        if (!fits64(a) || !fits64(b)) return C_UNKNOWN;
        B.lo[np + v] = (long long)a;
        B.hi[np + v] = (long long)b;
    }
    reason = 3;
    // atoms, in creation order (each may use the earlier ones)
    for (int t = 0; t < na; ++t) {
        const uint64_t w = *p++;
        const int op = (int)(w & 0xFF), litdiv = (int)((w >> 8) & 0xFF);
        const int d = nv + np + t;
        i128 al, ah, bl, bh;
        if (!peval_blob(p, B, al, ah) || !peval_blob(p, B, bl, bh)) return C_UNKNOWN;
        i128 rlo, rhi;
        if (litdiv) {
            if (bl != bh || bl < 1) return C_UNKNOWN;  // guards0 also checks it
            rlo = tdiv64(al, bl);
            rhi = tdiv64(ah, bl);
        } else if (op == NODE_DIV) {
            if (al >= 0 && bl >= 1) {
                rlo = tdiv64(al, bh);
                rhi = tdiv64(ah, bl);
            } else {
                const i128 m = sym::imax(sym::iabs(al), sym::iabs(ah));
                rlo = -m;
                rhi = m;
            }
        } else {
            i128 m = sym::imax(sym::iabs(bl), sym::iabs(bh)) - 1;
            if (m < 0) m = 0;
            m = sym::imin(m, sym::imax(sym::iabs(al), sym::iabs(ah)));
            rlo = al < 0 ? -m : 0;
            rhi = ah > 0 ? m : 0;
        }
        if (!fits64(rlo) || !fits64(rhi)) return C_UNKNOWN;
        B.lo[d] = (long long)rlo;
        B.hi[d] = (long long)rhi;
    }
    // eliminated variables: their domain constraints were compiled with the
    // representative's bounds, valid for a query whose domain lies within them
    for (uint64_t g = *p++; g > 0; --g, p += 5) {
        const int v = (int)(p[0] & 0xFFFF), flags = (int)(p[0] >> 16);
        const i128 lo = (i128)(((unsigned __int128)p[2] << 64) | p[1]);
        const i128 hi = (i128)(((unsigned __int128)p[4] << 64) | p[3]);
        if ((flags & 1) && (i128)B.lo[v] < lo) return C_UNKNOWN;
        if ((flags & 2) && (i128)B.hi[v] > hi) return C_UNKNOWN;
    }
    // guards0 on the build box
    reason = 4;
    for (uint64_t g = *p++; g > 0; --g) {
        i128 lo, hi;
        if (!peval_blob(p, B, lo, hi) || lo < 0) return C_UNKNOWN;
    }
    // tighten (entry: v | KCONST flag, then the constant K or K's polynomial,
    // then s)
    const uint64_t ne = *p++;
    const uint64_t* ent = p;
    for (uint64_t e = 0; e < ne; ++e) {  // skip to the end of the entries
        const uint64_t w = *p++;
        if (w & KCONST) p += 1;
        else skip_poly(p);
        skip_poly(p);
    }
    for (int r = 0; r < sym::ROUNDS; ++r) {
        bool changed = false;
        const uint64_t* q = ent;
        for (uint64_t e = 0; e < ne; ++e) {
            const uint64_t w = *q++;
            const int v = (int)(w & 0xFFFFu);
            i128 k;
            if (w & KCONST) {
                k = (i128)(long long)*q++;
            } else {
                i128 klo, khi;
                const bool kok = peval_blob(q, B, klo, khi);
                k = (kok && klo == khi) ? klo : 0;
            }
            i128 slo, shi;
            if (!peval_blob(q, B, slo, shi) || k == 0) continue;
            if (k > 0) {
                const i128 nlo = -fdiv64(shi, k);
                if (nlo > B.lo[v]) {
                    if (nlo > B.hi[v]) return C_REFUTED;
                    B.lo[v] = (long long)nlo;
                    changed = true;
                }
            } else {
                const i128 nhi = fdiv64(shi, -k);
                if (nhi < B.hi[v]) {
                    if (nhi < B.lo[v]) return C_REFUTED;
                    B.hi[v] = (long long)nhi;
                    changed = true;
                }
            }
        }
        if (!changed) break;
    }
    // direct constraints (no unit-coefficient variable)
    for (uint64_t g = *p++; g > 0; --g) {
        i128 lo, hi;
        if (peval_blob(p, B, lo, hi) && hi < 0) return C_REFUTED;
    }
    // guards1 on the tightened box
    reason = 5;
    bool guards = true;
    for (uint64_t g = *p++; g > 0; --g) {
        i128 lo, hi;
        if (!peval_blob(p, B, lo, hi) || lo < 0) guards = false;
    }
    if (!guards) return C_UNKNOWN;
    reason = 6;
    if (*p++) {
        i128 lo, hi;
        if (peval_blob(p, B, lo, hi) && hi < 0) return C_REFUTED;
    }
    return C_UNKNOWN;
}

// ---- compiler (host functions) -----------------------------------------------
// the line of the last failed compile (diagnostics)
inline int& cert_fail_line() {
    static thread_local int line = 0;
    return line;
}
#define CERT_FAIL()                 \
    do {                            \
        cert_fail_line() = __LINE__; \
        return 0;                   \
    } while (0)
struct Blob {
    uint64_t* w;
    size_t n, cap;
    bool ok;
    void put(uint64_t x) {
        if (n < cap) w[n++] = x;
        else ok = false;
    }
    void poly(const sym::PV& p) {
        put((uint64_t)p.n);
        for (int i = 0; i < p.n; ++i) {
            put(p.k[i]);
            put((uint64_t)p.c[i]);
            put((uint64_t)((unsigned __int128)p.c[i] >> 64));
        }
    }
};

// Compile the certificate of one structure class from its representative
// query (domains dom, literal slots lit); pmap/pslot: the varying literal
// slots (parameters).  Returns the blob length in words (0: no certificate).
template <typename GetDom, typename GetLit>
inline size_t cert_build(sym::Store& S, sym::LaneWork& W, sym::Moves& M, const uint32_t* cons, const uint32_t* code,
                         uint32_t nv, uint32_t ncon, uint32_t nlit, GetDom dom, GetLit lit, const int16_t* pmap,
                         int np, const int16_t* pslot, uint64_t* out, size_t cap) {
    using namespace sym;
    if (!build(S, cons, code, nv, ncon, dom, lit, pmap, np, pslot)) CERT_FAIL();
    const int nb0 = S.nv;  // variables + parameters + atoms
    if (nb0 > MAXB) CERT_FAIL();
    // the build box (atom intervals depend on it); guards0 from the atoms
    Blob b{out, 0, cap, true};
    b.put(MAGIC);
    b.put((uint64_t)nb0 | (uint64_t)nv << 16 | (uint64_t)S.np << 32 | (uint64_t)S.natoms << 48);
    for (int q = 0; q < S.np; ++q) b.put((uint64_t)pslot[q]);
    // the folded (class-constant) literal slots and their values
    {
        uint64_t nconst = 0;
        for (uint32_t i = 0; i < nlit; ++i) nconst += pmap[i] < 0;
        b.put(nconst);
        for (uint32_t i = 0; i < nlit; ++i) {
            if (pmap[i] >= 0) continue;
            const i128 x = lit(i);
            b.put((uint64_t)i);
            b.put((uint64_t)x);
            b.put((uint64_t)((unsigned __int128)x >> 64));
        }
    }
    i128 gc[MAXA * 2][20];
    uint64_t gk[MAXA * 2][20];
    PV guards0[MAXA * 2];
    int ng0 = 0;
    for (int t = 0; t < S.natoms; ++t) {
        if (S.avar[t] != S.np + (int)nv + t) CERT_FAIL();  // atoms are numbered in creation order
        b.put((uint64_t)(uint8_t)S.aop[t] | (uint64_t)(uint8_t)S.alitdiv[t] << 8);
        PV a = atom_poly(S, 2 * t), d = atom_poly(S, 2 * t + 1);
        b.poly(a);
        b.poly(d);
        if (S.alitdiv[t]) {
            if (S.acase[t] == 0 || S.acase[t] == 1) {  // dividend sign
                PV g{gk[ng0], gc[ng0], 0, 20};
                PV z{nullptr, nullptr, 0, 0};
                if (!plin(a, S.acase[t] == 0 ? 1 : -1, z, 0, g)) CERT_FAIL();
                guards0[ng0++] = g;
            }
            if (d.k[0] != 0) {  // a parameter divisor: p - 1 >= 0
                PV g{gk[ng0], gc[ng0], 0, 20};
                if (!pcopy(d, g) || !pins(g, 0, -1)) CERT_FAIL();
                guards0[ng0++] = g;
            }
        }
    }
    PV w[4] = {work(W, 0), work(W, 1), work(W, 2), work(W, 3)};
    if (!eliminate(S, w) || S.nc > 64) CERT_FAIL();
    // domain-containment guards of the eliminated variables, then guards0
    b.put((uint64_t)S.nelim);
    for (int i = 0; i < S.nelim; ++i) {
        b.put((uint64_t)(uint16_t)S.elim_v[i] | (uint64_t)(uint8_t)S.elim_flags[i] << 16);
        b.put((uint64_t)S.elim_lo[i]);
        b.put((uint64_t)((unsigned __int128)S.elim_lo[i] >> 64));
        b.put((uint64_t)S.elim_hi[i]);
        b.put((uint64_t)((unsigned __int128)S.elim_hi[i] >> 64));
    }
    b.put((uint64_t)ng0);
    for (int i = 0; i < ng0; ++i) b.poly(guards0[i]);
    // tighten entries: every constraint, every variable with a (parametric)
    // constant coefficient: (v, K, s) for g = K*v + s
    size_t at_ne = b.n;
    b.put(0);
    uint64_t ne = 0;
    bool covered[MAXC];
    for (int j = 0; j < S.nc; ++j) {
        covered[j] = false;
        PV g = store_poly(S, j);
        for (int v = 0; v < S.nv; ++v) {
            PV K = w[1], s = w[0];
            if (!pcoef(g, v, 0, S.np, K, s)) continue;
            if (K.n == 1 && K.k[0] == 0 && K.c[0] == (i128)(long long)K.c[0]) {
                b.put((uint64_t)v | KCONST);
                b.put((uint64_t)(long long)K.c[0]);
            } else {
                b.put((uint64_t)v);
                b.poly(K);
            }
            b.poly(s);
            ++ne;
            covered[j] = true;
        }
    }
    if (b.ok) out[at_ne] = ne;
    int direct = 0;
    for (int j = 0; j < S.nc; ++j) direct += !covered[j];
    b.put((uint64_t)direct);
    for (int j = 0; j < S.nc; ++j)
        if (!covered[j]) b.poly(store_poly(S, j));
    // the representative's own proof
    const int r = tighten(S, w);
    if (r == R_REFUTED) {
        b.put(0);  // no guards1
        b.put(0);  // no final polynomial
        return b.ok ? b.n : 0;
    }
    for (int t = 0; t < S.nc; ++t) {
        if (!greedy_target(S, t, W, &M)) continue;
        int ng1 = M.n;
        for (int m = 0; m < M.n; ++m) ng1 += !(M.kn[m] == 1 && M.kk[m][0] == 0);
        b.put((uint64_t)ng1);
        for (int m = 0; m < M.n; ++m) {
            PV g{M.mk[m], M.mc[m], M.mn[m], MAXT};
            b.poly(g);  // multiplier >= 0
            if (!(M.kn[m] == 1 && M.kk[m][0] == 0)) {  // parametric factor K >= 1
                PV k{M.kk[m], M.kc[m], M.kn[m], MAXT};
                if (!pins(k, 0, -1)) CERT_FAIL();
                b.poly(k);
            }
        }
        b.put(1);
        PV fin{M.fk, M.fc, M.fn, MAXT};
        b.poly(fin);
        return b.ok ? b.n : 0;
    }
    CERT_FAIL();
}

}  // namespace cert
}  // namespace oob
