// wide.cuh -- 256-bit two's-complement integer for the widest exact regime.
//
// The reference computes with unbounded Python ints.  Some analyzer-shaped
// queries carry products of four or five declared domains (fluid_adv-like
// extents (c+1)^3 * N * K at M = 2^31-1 already need ~131 bits; at M = 2^59
// ~245 bits), so besides int64 and __int128 the engine instantiates its
// templates on this type.  The host proves every intermediate magnitude is
// below 2^253, so the truncating operations below are exact.
#pragma once
#include "types.h"

#if defined(__CUDACC__)
#define W_HD __host__ __device__ __forceinline__
#else
#define W_HD inline
#endif

namespace oob {

struct i256 {
    uint64_t w[4];  // little-endian limbs

    i256() = default;
    W_HD constexpr i256(long long v)
        : w{(uint64_t)v, v < 0 ? ~0ull : 0ull, v < 0 ? ~0ull : 0ull, v < 0 ? ~0ull : 0ull} {}
    W_HD constexpr i256(int v) : i256((long long)v) {}
    W_HD static i256 from128(__int128 v) {
        i256 r;
        r.w[0] = (uint64_t)v;
        r.w[1] = (uint64_t)(v >> 64);
        uint64_t s = v < 0 ? ~0ull : 0ull;
        r.w[2] = s;
        r.w[3] = s;
        return r;
    }
    W_HD __int128 low128() const { return (__int128)(((unsigned __int128)w[1] << 64) | w[0]); }
    W_HD bool neg() const { return (int64_t)w[3] < 0; }
    W_HD bool is_zero() const { return (w[0] | w[1] | w[2] | w[3]) == 0; }
};

W_HD i256 operator+(const i256& a, const i256& b) {
    i256 r;
    unsigned __int128 c = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        c += (unsigned __int128)a.w[i] + b.w[i];
        r.w[i] = (uint64_t)c;
        c >>= 64;
    }
    return r;
}
W_HD i256 operator~(const i256& a) {
    i256 r;
#pragma unroll
    for (int i = 0; i < 4; i++) r.w[i] = ~a.w[i];
    return r;
}
W_HD i256 operator-(const i256& a) { return ~a + i256(1); }
W_HD i256 operator-(const i256& a, const i256& b) {
    i256 r;
    uint64_t borrow = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        uint64_t x = a.w[i], y = b.w[i];
        uint64_t d = x - y - borrow;
        borrow = (x < y) || (x == y && borrow) ? 1 : 0;
        r.w[i] = d;
    }
    return r;
}
// true iff the value is a sign-extended int64 (the common case once domains
// have been narrowed): the hot operations below take a 64-bit fast path
W_HD bool fits64(const i256& a) {
    uint64_t s = (uint64_t)((int64_t)a.w[0] >> 63);
    return a.w[1] == s && a.w[2] == s && a.w[3] == s;
}
W_HD i256 from64(long long v) { return i256(v); }

W_HD i256 operator*(const i256& a, const i256& b) {  // low 256 bits (two's complement)
    if (fits64(a) && fits64(b)) return i256::from128((__int128)(long long)a.w[0] * (long long)b.w[0]);
    uint64_t r[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 4; i++) {
        unsigned __int128 carry = 0;
#pragma unroll
        for (int j = 0; j + i < 4; j++) {
            unsigned __int128 t = (unsigned __int128)a.w[i] * b.w[j] + r[i + j] + carry;
            r[i + j] = (uint64_t)t;
            carry = t >> 64;
        }
    }
    i256 o;
#pragma unroll
    for (int i = 0; i < 4; i++) o.w[i] = r[i];
    return o;
}
W_HD bool operator==(const i256& a, const i256& b) {
    return a.w[0] == b.w[0] && a.w[1] == b.w[1] && a.w[2] == b.w[2] && a.w[3] == b.w[3];
}
W_HD bool operator!=(const i256& a, const i256& b) { return !(a == b); }
W_HD bool operator<(const i256& a, const i256& b) {
    if (a.w[3] != b.w[3]) return (int64_t)a.w[3] < (int64_t)b.w[3];
    if (a.w[2] != b.w[2]) return a.w[2] < b.w[2];
    if (a.w[1] != b.w[1]) return a.w[1] < b.w[1];
    return a.w[0] < b.w[0];
}
W_HD bool operator>(const i256& a, const i256& b) { return b < a; }
W_HD bool operator<=(const i256& a, const i256& b) { return !(b < a); }
W_HD bool operator>=(const i256& a, const i256& b) { return !(a < b); }
W_HD i256 operator>>(const i256& a, int s) {  // arithmetic; s in [0, 63]
    if (s == 0) return a;
    i256 r;
    r.w[0] = (a.w[0] >> s) | (a.w[1] << (64 - s));
    r.w[1] = (a.w[1] >> s) | (a.w[2] << (64 - s));
    r.w[2] = (a.w[2] >> s) | (a.w[3] << (64 - s));
    r.w[3] = (uint64_t)((int64_t)a.w[3] >> s);
    return r;
}

// unsigned magnitude division n / d (d != 0)
W_HD void udivmod(const i256& n, const i256& d, i256& q, i256& r) {
    if ((d.w[1] | d.w[2] | d.w[3]) == 0) {  // 64-bit divisor: limb-wise long division
        uint64_t dv = d.w[0];
        unsigned __int128 rem = 0;
        for (int i = 3; i >= 0; i--) {
            unsigned __int128 cur = (rem << 64) | n.w[i];
            q.w[i] = (uint64_t)(cur / dv);
            rem = cur % dv;
        }
        r = i256(0);
        r.w[0] = (uint64_t)rem;
        return;
    }
    q = i256(0);
    r = i256(0);
    int top = 255;
    while (top >= 0 && !((n.w[top >> 6] >> (top & 63)) & 1)) top--;
    for (int i = top; i >= 0; i--) {
        // r = (r << 1) | bit
        r.w[3] = (r.w[3] << 1) | (r.w[2] >> 63);
        r.w[2] = (r.w[2] << 1) | (r.w[1] >> 63);
        r.w[1] = (r.w[1] << 1) | (r.w[0] >> 63);
        r.w[0] = (r.w[0] << 1) | ((n.w[i >> 6] >> (i & 63)) & 1);
        // unsigned compare r >= d
        bool ge = true;
        for (int k = 3; k >= 0; k--) {
            if (r.w[k] != d.w[k]) {
                ge = r.w[k] > d.w[k];
                break;
            }
        }
        if (ge) {
            r = r - d;
            q.w[i >> 6] |= 1ull << (i & 63);
        }
    }
}

// C semantics: quotient truncates toward zero, remainder takes the dividend's sign
W_HD i256 operator/(const i256& a, const i256& b) {
    if (fits64(a) && fits64(b)) {
        long long x = (long long)a.w[0], y = (long long)b.w[0];
        if (!(x == (-9223372036854775807LL - 1) && y == -1)) return i256(x / y);
    }
    bool na = a.neg(), nb = b.neg();
    i256 q, r;
    udivmod(na ? -a : a, nb ? -b : b, q, r);
    return (na != nb) ? -q : q;
}
W_HD i256 operator%(const i256& a, const i256& b) {
    if (fits64(a) && fits64(b)) {
        long long x = (long long)a.w[0], y = (long long)b.w[0];
        if (!(x == (-9223372036854775807LL - 1) && y == -1)) return i256(x % y);
    }
    bool na = a.neg(), nb = b.neg();
    i256 q, r;
    udivmod(na ? -a : a, nb ? -b : b, q, r);
    return na ? -r : r;
}

}  // namespace oob
