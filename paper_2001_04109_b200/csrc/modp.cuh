// Device-side Z/pZ arithmetic (p < 2^31) and the int8 limb representation.
//
// The reference stores residues as uint64 in [0, p) and reduces every
// product with a 64-bit '%' (include/fsyrk/fields.hpp:49-66).  On the GPU
// residues live as uint32 and products are reduced with Barrett (one
// 64-bit mul-hi, one correction); there is no hardware 64-bit divide.
#pragma once

#include <cstdint>

namespace fsyrk_b200 {

// Per-prime constants, computed on the host (see driver.cu: make_modp).
struct ModP {
    uint32_t p;
    uint32_t pad_;
    uint64_t mu;   // floor(2^64 / p)
    uint64_t off;  // multiple of p >= 2^62: lifts a signed |v| < 2^62 to unsigned
};

__host__ __device__ inline ModP make_modp(uint32_t p) {
    ModP m;
    m.p = p;
    m.pad_ = 0;
    m.mu = ~0ull / p;  // floor((2^64 - 1) / p) == floor(2^64 / p) for p not a power of 2
    m.off = (uint64_t)p * ((1ull << 62) / p + 1);
    return m;
}

// x mod p for any uint64 x.
__device__ __forceinline__ uint32_t mod_u64(uint64_t x, const ModP& m) {
    uint64_t q = __umul64hi(x, m.mu);
    uint64_t r = x - q * m.p;
    if (r >= m.p) r -= m.p;
    return (uint32_t)r;
}

// v mod p for signed |v| < 2^62.
__device__ __forceinline__ uint32_t mod_s64(int64_t v, const ModP& m) { return mod_u64((uint64_t)(v + (int64_t)m.off), m); }

// Branch-free forms (a, b < p < 2^31): the wrong candidate wraps around 2^32 and loses the
// unsigned min -- add, add, min instead of add, compare, add, select (the pre-addition kernels
// are integer-issue bound: profiles/r02/ncu_prep_tree_cfg2.md).
__device__ __forceinline__ uint32_t addm(uint32_t a, uint32_t b, uint32_t p) {
    const uint32_t s = a + b;
    return min(s, s - p);
}
__device__ __forceinline__ uint32_t subm(uint32_t a, uint32_t b, uint32_t p) {
    const uint32_t d = a - b;
    return min(d, d + p);
}
__device__ __forceinline__ uint32_t mulm(uint32_t a, uint32_t b, const ModP& m) {
    return mod_u64((uint64_t)a * b, m);
}

// Balanced int8 limbs.  A residue x is mapped to a representative r of its
// class inside the window [lo, lo + 256^L) with lo = -128 (256^L - 1)/255,
// then r = sum_l d_l 256^l with every d_l in [-128, 127].  The window holds
// 256^L >= p integers, so every residue has such an r (Appendix B of SURVEY).
template <int L>
struct Limbs {
    static constexpr int64_t span = 1ll << (8 * L);
    static constexpr int64_t lo = -128ll * ((span - 1) / 255);
    static constexpr int64_t hi = lo + span - 1;
};

template <int L>
__device__ __forceinline__ void split_limbs(uint32_t x, uint32_t p, int8_t (&d)[L]) {
    int64_t r = (int64_t)x;
    if (r > Limbs<L>::hi) r -= p;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        int64_t dl = ((r + 128) & 255) - 128;
        d[l] = (int8_t)dl;
        r = (r - dl) >> 8;
    }
}

// Same digits, packed: byte l of the result is d_l.  With the bias
// B = 128 (1 + 256 + ... + 256^(L-1)), r + B = sum (d_l + 128) 256^l has
// plain base-256 digits, and d_l = (byte l) - 128 = (byte l) ^ 0x80 as int8.
template <int L>
__device__ __forceinline__ uint32_t limb_word(uint32_t x, uint32_t p) {
    constexpr uint32_t bias = L == 1 ? 0x80u : L == 2 ? 0x8080u : L == 3 ? 0x808080u : 0x80808080u;
    const uint32_t hi = (uint32_t)Limbs<L>::hi;
    const uint32_t r = x > hi ? x - p : x;  // two's complement wrap is intended
    return (r + bias) ^ 0x80808080u;
}

// Gather byte l of four limb words into one 32-bit store (4 consecutive columns of plane l).
__device__ __forceinline__ uint32_t gather_byte(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, int l) {
    const uint32_t s = (uint32_t)l;
    const uint32_t lo = __byte_perm(w0, w1, s | ((s + 4) << 4));        // bytes: w0[l], w1[l]
    const uint32_t hi = __byte_perm(w2, w3, s | ((s + 4) << 4));        // bytes: w2[l], w3[l]
    return __byte_perm(lo, hi, 0x5410);
}

// Shoup multiplication by a constant w < p: wq = floor(w 2^32 / p), x < 2^32.
struct MulConst {
    uint32_t w, wq;
};
__host__ __device__ inline MulConst make_mulconst(uint32_t w, uint32_t p) {
    return MulConst{w, (uint32_t)(((uint64_t)w << 32) / p)};
}
__device__ __forceinline__ uint32_t mulc(uint32_t x, MulConst c, uint32_t p) {
    const uint32_t q = __umulhi(x, c.wq);
    const uint32_t r = x * c.w - q * p;  // exact mod 2^32, true value in [0, 2p)
    return min(r, r - p);
}

}  // namespace fsyrk_b200
