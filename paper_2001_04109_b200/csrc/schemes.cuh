// Digit schemes of the exact int8 tensor-core products.
//
// A residue x in [0, p) is stored as P int8 "planes" (one byte each).  An
// output tile accumulates NT tensor-core terms  acc[t.acc] += A_plane[t.a] *
// B_plane[t.b]^T  in int32 TMEM columns; the epilogue folds the NACC
// accumulators into C mod p.  Every term of a scheme has a fixed weight
// (a power of the digit base, possibly times a small constant), so
//     x * y = sum_acc  weight(acc) * acc   (mod p)
// holds exactly as long as no int32 accumulator overflows (kmax).
//
//  LIMB2/3/4 : balanced base-256 digits in [-128, 127] (any p < 2^16 / 2^24 / 2^31);
//              2L-1 accumulators, one per shift s = i + j, weights 256^s mod p.
//  M17       : p = 2^17 - 1.  Unsigned base-64 digits d0, d1, d2 (6 bits each).
//              Since 2^18 = 2 (mod p) and 2^24 = 2 * 2^6, the shifts 3 and 4
//              fold into accumulators 0 and 1 with doubled digits 2 d1, 2 d2
//              (<= 126): 3 accumulators instead of 5, which frees TMEM for a
//              160-column tile.  Fold: a0 + 2^6 a1 + 2^12 a2, Mersenne reduction.
//  M31       : p = 2^31 - 1.  Unsigned base-256 digits d0..d3 (d3 < 128).  Since
//              2^32 = 2, 2^40 = 2 * 2^8, 2^48 = 2 * 2^16 (mod p), every wrapped
//              term that touches d3 folds into accumulators 0..2 with the doubled
//              digit 2 d3 (<= 254, unsigned); only d2 e2 (weight 2) keeps its own
//              accumulator: 5 accumulators instead of 7 (96-column tiles instead
//              of 64).  Fold: a0 + 2^8 a1 + 2^16 a2 + 2^24 a3 + 2 a4.
#pragma once

#include <cstdint>

#include "modp.cuh"

namespace fsyrk_b200 {

enum SchemeId {
    SCHEME_LIMB2 = 0,
    SCHEME_LIMB3 = 1,
    SCHEME_LIMB4 = 2,
    SCHEME_M17 = 3,
    SCHEME_M31 = 4,
    SCHEME_M17N = 5  // M17 digits with 128-column tiles (fine multi-GPU partitions: blocks of 128)
};
// the digit arithmetic a scheme shares with another one (M17N is M17 with narrower tiles)
template <int S>
inline constexpr int digits_of = S == SCHEME_M17N ? SCHEME_M17 : S;

struct Term {
    int8_t a, b, acc;
};

// FSYRK_PAIR = 1: products run on CTA pairs (cta_group::2, 256-row tiles; each SM loads
// half of B), which halves the B operand bytes an SM pulls from L2 per MAC.  Measured
// slower than single CTAs on B200 even with the epilogue removed (cfg2 products 166 vs
// 155 us, cfg5 2.34 vs 2.17 ms; profiles/r01/variants.txt): the single-CTA main loop is
// not operand-feed bound, so the pair path stays available but off.
#ifndef FSYRK_PAIR
#define FSYRK_PAIR 0
#endif

template <int S>
struct Scheme;

// A wide-B term over overlapped accumulators: A digit plane a times the nb adjacent B digit
// planes b .. b + nb - 1 (one N = nb * BN MMA) into the adjacent accumulators acc .. acc + nb - 1.
// init: on the first 32-deep K step of a chunk the MMA overwrites instead of accumulating.
struct WideTerm {
    int8_t a, b, acc, nb, init;
};

#ifndef FSYRK_LIMB2_BN
#define FSYRK_LIMB2_BN 128
#endif
#ifndef FSYRK_LIMB2_BK
#define FSYRK_LIMB2_BK 128
#endif
#ifndef FSYRK_LIMB2_STAGES
#define FSYRK_LIMB2_STAGES (FSYRK_PAIR ? 4 : 3)
#endif
// LIMB2 wide-B (default): the two B digit planes sit next to each other in the stage, so one
// N = 2 BN MMA per A digit computes d_a [e0 | e1] into two adjacent accumulators: 2 MMAs of
// N = 256 instead of 4 of N = 128 per K step.  The tensor pipe time is the same, but every A
// operand byte read from shared memory now feeds 256 columns instead of 128 -- the operand
// reads per MMA cycle drop from 128 to 96 B (LIMB2 had the highest operand bandwidth of all
// schemes).  Four accumulators T00 | T01 | T10 | T11 (all 512 TMEM columns); the fold weights
// T01 and T10 alike (shift 1).
#ifndef FSYRK_LIMB2_WIDE
#define FSYRK_LIMB2_WIDE 1
#endif
// FSYRK_LIMB2_PAIR = 1: the wide-B layout on CTA pairs (cta_group::2, 256 x 128 tiles).  The
// N = 256 operand [e0 | e1] of a pair MMA is split by rows between the two CTAs, i.e. by
// PLANE: CTA r stages B digit plane r only (all BN rows) next to its own 128 rows of both A
// planes.  Per SM and 32-deep K step that is 12 KB of operands pulled from L2 instead of 16 KB
// (LIMB2 at full MMA rate asks for 64 B/clk/SM, above what L2 delivers to 148 SMs) and 64
// instead of 96 B/clk of shared-memory operand reads.
#ifndef FSYRK_LIMB2_PAIR
#define FSYRK_LIMB2_PAIR FSYRK_PAIR
#endif
#ifndef FSYRK_LIMB2_OVERLAP
#define FSYRK_LIMB2_OVERLAP 0
#endif
template <>
struct Scheme<SCHEME_LIMB2> {
    static constexpr bool UNSIGNED = false, PAIR = FSYRK_LIMB2_PAIR;
    static constexpr bool WIDE = FSYRK_LIMB2_WIDE;
    static constexpr bool SPLITB = WIDE && PAIR;  // B planes split across the CTA pair
    // FSYRK_LIMB2_OVERLAP: three accumulators, one per digit shift, the two wide MMAs overlapping
    // in the middle one (like LIMB3 / LIMB4 below): a quarter less TMEM to drain per tile
    static constexpr bool OVERLAP = FSYRK_LIMB2_OVERLAP && WIDE && !PAIR;
    static constexpr int PA = 2, PB = 2, NACC = WIDE && !OVERLAP ? 4 : 3, NT = WIDE ? 2 : 4, NB = WIDE ? 2 : 1,
                         BN = FSYRK_LIMB2_BN, BK = FSYRK_LIMB2_BK,
                         STAGES = SPLITB && FSYRK_LIMB2_BK == 128 ? 4 : FSYRK_LIMB2_STAGES;
    __host__ __device__ static constexpr Term term(int q) {
        constexpr Term T[4] = {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 2}};
        constexpr Term W[2] = {{0, 0, 0}, {1, 0, 2}};  // B planes 0..1 as one operand
        constexpr Term O[2] = {{0, 0, 0}, {1, 0, 1}};
        return OVERLAP ? O[q] : WIDE ? W[q] : T[q];
    }
    static constexpr int NT0 = 3;  // first K block of a chunk (OVERLAP)
    __host__ __device__ static constexpr WideTerm term0(int q) {
        constexpr WideTerm F[NT0] = {{1, 1, 2, 1, 1}, {0, 0, 0, 2, 1}, {1, 0, 1, 1, 0}};
        return F[q];
    }
    // digit shift (weight 256^shift) of accumulator s
    __host__ __device__ static constexpr int shift(int s) { return WIDE && !OVERLAP ? (s >> 1) + (s & 1) : s; }
};
// LIMB3 wide-B (FSYRK_LIMB3_WIDE): like LIMB4 below with 80-column tiles, 3 MMAs of N = 240 per
// 32-deep K step (360 cycles per 128 x 80 tile) instead of 9 of N = 96 (505 per 128 x 96).
#ifndef FSYRK_LIMB3_WIDE
#define FSYRK_LIMB3_WIDE 1
#endif
template <>
struct Scheme<SCHEME_LIMB3> {
    static constexpr bool UNSIGNED = false, PAIR = FSYRK_PAIR;
    static constexpr bool OVERLAP = FSYRK_LIMB3_WIDE && !FSYRK_PAIR;
    static constexpr int PA = 3, PB = 3, NACC = 5, NT = OVERLAP ? 3 : 9, NB = OVERLAP ? 3 : 1, BN = OVERLAP ? 80 : 96,
                         BK = 128, STAGES = FSYRK_PAIR ? 3 : 2;
    __host__ __device__ static constexpr Term term(int q) {
        constexpr Term T[9] = {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}, {0, 2, 2}, {1, 1, 2},
                               {2, 0, 2}, {1, 2, 3}, {2, 1, 3}, {2, 2, 4}};
        constexpr Term W[3] = {{0, 0, 0}, {1, 0, 1}, {2, 0, 2}};  // B planes 0..2 as one operand
        return OVERLAP ? W[q] : T[q];
    }
    // first K block of a chunk (OVERLAP): d2 [e1 | e2] initialises accumulators 3, 4; d0 [e0..e2]
    // initialises 0..2; d2 e0 and d1 [e0..e2] accumulate
    static constexpr int NT0 = 4;
    __host__ __device__ static constexpr WideTerm term0(int q) {
        constexpr WideTerm F[NT0] = {{2, 1, 3, 2, 1}, {0, 0, 0, 3, 1}, {2, 0, 2, 1, 0}, {1, 0, 1, 3, 0}};
        return F[q];
    }
};
// LIMB4 wide-B (default): accumulator s (digit shift s = i + j) sits at TMEM columns s * BN, so
// d_i [e0 | e1 | e2 | e3] lands on the adjacent accumulators i .. i + 3: 4 MMAs of N = 256 per
// 32-deep K step instead of 16 of N = 64.  An int8 MMA costs max(~54, N / 2) cycles
// (profiles/ubench/ubench_mma_rate.cu), so the 16 narrow ones ran at 60% of the tensor rate:
// 858 -> 512 cycles per K step.  Accumulators overlap between MMAs, so overwrite-vs-accumulate
// cannot be per accumulator: the first K block of a chunk issues d3 as d3 [e1 | e2 | e3]
// (initialising accumulators 4..6) and d3 e0 (accumulating into 3, after d0 [e0..e3] has
// initialised 0..3); MMAs into the same columns complete in issue order.
#ifndef FSYRK_LIMB4_WIDE
#define FSYRK_LIMB4_WIDE 1
#endif
template <>
struct Scheme<SCHEME_LIMB4> {
    static constexpr bool UNSIGNED = false, PAIR = FSYRK_PAIR;
    static constexpr bool OVERLAP = FSYRK_LIMB4_WIDE && !FSYRK_PAIR;
    static constexpr int PA = 4, PB = 4, NACC = 7, NT = OVERLAP ? 4 : 16, NB = OVERLAP ? 4 : 1, BN = 64, BK = 128,
                         STAGES = 2;
    __host__ __device__ static constexpr Term term(int q) {
        constexpr Term T[16] = {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}, {0, 2, 2}, {1, 1, 2}, {2, 0, 2},
                                {0, 3, 3}, {1, 2, 3}, {2, 1, 3}, {3, 0, 3}, {1, 3, 4}, {2, 2, 4},
                                {3, 1, 4}, {2, 3, 5}, {3, 2, 5}, {3, 3, 6}};
        constexpr Term W[4] = {{0, 0, 0}, {1, 0, 1}, {2, 0, 2}, {3, 0, 3}};  // B planes 0..3 as one operand
        return OVERLAP ? W[q] : T[q];
    }
    // first K block of a chunk (OVERLAP)
    static constexpr int NT0 = 5;
    __host__ __device__ static constexpr WideTerm term0(int q) {
        constexpr WideTerm F[NT0] = {{3, 1, 4, 3, 1}, {0, 0, 0, 4, 1}, {3, 0, 3, 1, 0}, {1, 0, 1, 4, 0}, {2, 0, 2, 4, 0}};
        return F[q];
    }
};
// planes (stored): {d0, d1, d2, 2 d1, 2 d2}.  Single CTA: A reads all 5, B the first 3.
// CTA pair: the doubled digits move to the B side (each SM holds only BN/2 rows of B,
// so the 5-plane operand is the narrow one): A reads {d0, d1, d2}, B all 5.
#ifndef FSYRK_M17_BN
#define FSYRK_M17_BN 160
#endif
#ifndef FSYRK_M17_BK
#define FSYRK_M17_BK 64
#endif
#ifndef FSYRK_M17_STAGES
#define FSYRK_M17_STAGES (FSYRK_PAIR ? 4 : 3)
#endif
template <>
struct Scheme<SCHEME_M17> {
    static constexpr bool UNSIGNED = true, PAIR = FSYRK_PAIR;
    static constexpr int PA = PAIR ? 3 : 5, PB = PAIR ? 5 : 3, NACC = 3, NT = 9, NB = 1, BN = FSYRK_M17_BN,
                         BK = FSYRK_M17_BK, STAGES = FSYRK_M17_STAGES;
    __host__ __device__ static constexpr Term term(int q) {
        // acc0: d0 e0 + 2^18 (d1 e2 + d2 e1);  acc1: d0 e1 + d1 e0 + 2^18 d2 e2 (weight 2^6);
        // acc2: d0 e2 + d1 e1 + d2 e0 (weight 2^12);  2^18 = 2 rides on a doubled digit
        constexpr Term TA[NT] = {{0, 0, 0}, {3, 2, 0}, {4, 1, 0}, {0, 1, 1}, {1, 0, 1},
                                 {4, 2, 1}, {0, 2, 2}, {1, 1, 2}, {2, 0, 2}};
        constexpr Term TB[NT] = {{0, 0, 0}, {1, 4, 0}, {2, 3, 0}, {0, 1, 1}, {1, 0, 1},
                                 {2, 4, 1}, {0, 2, 2}, {1, 1, 2}, {2, 0, 2}};
        return PAIR ? TB[q] : TA[q];
    }
};
template <>
struct Scheme<SCHEME_M17N> : Scheme<SCHEME_M17> {
    static constexpr int BN = 128;
};

// planes: A = B = {d0, d1, d2, d3, 2 d3}
// FSYRK_M31_ACC4 = 1: the weight-2 term d2 e2 is issued twice into accumulator 0 instead of
// getting its own accumulator: 17 MMAs into 4 accumulators, which fit 128-column tiles
// (4 x 128 = 512 TMEM columns) -- full MMA rate (N = 96 runs at 86%, ubench_mma_rate.cu).
// Accumulators are read as unsigned 32-bit (K <= 13210); 0: 16 MMAs, 5 accumulators, N = 96.
#ifndef FSYRK_M31_ACC4
#define FSYRK_M31_ACC4 1  // measured: cfg4 products 23.5 -> 20.2 ms (profiles/r01/variants.txt)
#endif
#ifndef FSYRK_M31_PAIR
#define FSYRK_M31_PAIR FSYRK_PAIR  // CTA pairs for M31 only (experiment, profiles/r01/variants.txt)
#endif
#ifndef FSYRK_M31_BK
#define FSYRK_M31_BK 64
#endif
#ifndef FSYRK_M31_STAGES
#define FSYRK_M31_STAGES (FSYRK_M31_ACC4 ? (FSYRK_M31_BK == 32 ? 5 : 2) : (FSYRK_PAIR ? 4 : 3))
#endif
template <>
struct Scheme<SCHEME_M31> {
    static constexpr bool ACC4 = FSYRK_M31_ACC4;
    static constexpr int PA = 5, PB = 5, NACC = ACC4 ? 4 : 5, NT = ACC4 ? 17 : 16, NB = 1, BN = ACC4 ? 128 : 96,
                         BK = FSYRK_M31_BK, STAGES = FSYRK_M31_STAGES;
    static constexpr bool UNSIGNED = true, PAIR = FSYRK_M31_PAIR;
    __host__ __device__ static constexpr Term term(int q) {
        constexpr Term T5[16] = {
        {0, 0, 0}, {1, 4, 0}, {4, 1, 0},             // s=0 and s=4 (2^32 = 2): d1 (2 e3) + (2 d3) e1
        {0, 1, 1}, {1, 0, 1}, {2, 4, 1}, {4, 2, 1},  // s=1 and s=5 (2^40 = 2 * 2^8)
        {0, 2, 2}, {1, 1, 2}, {2, 0, 2}, {4, 3, 2},  // s=2 and s=6 (2^48 = 2 * 2^16): (2 d3) e3
        {0, 3, 3}, {1, 2, 3}, {2, 1, 3}, {3, 0, 3},  // s=3
        {2, 2, 4}};                                  // d2 e2, weight 2^32 = 2
        constexpr Term T4[17] = {
        {0, 0, 0}, {1, 4, 0}, {4, 1, 0}, {2, 2, 0}, {2, 2, 0},  // s=0, s=4: ... + 2 d2 e2 as two MMAs
        {0, 1, 1}, {1, 0, 1}, {2, 4, 1}, {4, 2, 1},
        {0, 2, 2}, {1, 1, 2}, {2, 0, 2}, {4, 3, 2},
        {0, 3, 3}, {1, 2, 3}, {2, 1, 3}, {3, 0, 3}};
        return ACC4 ? T4[q] : T5[q];
    }
};

// --------------------------------------------------------------- encoding
// Byte l of the result is plane l of residue x (canonical, x < p).
template <int S>
__host__ __device__ inline uint64_t encode_planes(uint32_t x, uint32_t p) {
    if constexpr (digits_of<S> == SCHEME_M17) {
        const uint32_t d0 = x & 63u, d1 = (x >> 6) & 63u, d2 = x >> 12;
        return (uint64_t)d0 | (uint64_t)d1 << 8 | (uint64_t)d2 << 16 | (uint64_t)(2 * d1) << 24 |
               (uint64_t)(2 * d2) << 32;
    } else if constexpr (S == SCHEME_M31) {
        return (uint64_t)x | (uint64_t)(2 * (x >> 24)) << 32;
    } else {
        constexpr int L = S == SCHEME_LIMB2 ? 2 : S == SCHEME_LIMB3 ? 3 : 4;
        // balanced digits: r + B has plain base-256 digits (d_l + 128); xor 0x80 recentres them
        constexpr uint32_t bias = L == 2 ? 0x8080u : L == 3 ? 0x808080u : 0x80808080u;
        constexpr int64_t span = 1ll << (8 * L);
        constexpr int64_t lo = -128ll * ((span - 1) / 255);
        const uint32_t hi = (uint32_t)(lo + span - 1);
        const uint32_t r = x > hi ? x - p : x;
        return (uint64_t)((r + bias) ^ 0x80808080u);
    }
}

// planes stored for an operand read in both roles (leaf SYRK operands)
template <int S>
__host__ __device__ constexpr int planes_of() {
    return Scheme<S>::PA > Scheme<S>::PB ? Scheme<S>::PA : Scheme<S>::PB;
}

// ------------------------------------------------------------------ fold
// Epilogue: accumulators (as raw 32-bit TMEM words) -> residue.
// w: balanced weights (LIMB schemes only).
template <int S>
__device__ __forceinline__ uint32_t fold_acc(const uint32_t* a, const ModP& m, const int32_t* w) {
    if constexpr (digits_of<S> == SCHEME_M17) {
        // unsigned accumulators < 2^31: v < 2^44
        uint64_t v = (uint64_t)a[0] + ((uint64_t)a[1] << 6) + ((uint64_t)a[2] << 12);
        v = (v & 0x1FFFFull) + (v >> 17);  // < 2^28
        v = (v & 0x1FFFFull) + (v >> 17);  // < 2^17 + 2^11
        uint32_t r = (uint32_t)v;
        return r >= 0x1FFFFu ? r - 0x1FFFFu : r;
    } else if constexpr (S == SCHEME_M31) {
        uint64_t v = (uint64_t)a[0] + ((uint64_t)a[1] << 8) + ((uint64_t)a[2] << 16) + ((uint64_t)a[3] << 24);
        if constexpr (!Scheme<S>::ACC4) v += (uint64_t)a[Scheme<S>::NACC - 1] << 1;  // < 2^57
        v = (v & 0x7FFFFFFFull) + (v >> 31);  // < 2^31 + 2^25
        v = (v & 0x7FFFFFFFull) + (v >> 31);
        uint32_t r = (uint32_t)v;
        return r >= 0x7FFFFFFFu ? r - 0x7FFFFFFFu : r;
    } else {
        int64_t v = (int64_t)(int32_t)a[0];
#pragma unroll
        for (int s = 1; s < Scheme<S>::NACC; ++s) v += (int64_t)(int32_t)a[s] * (int64_t)w[s];
        return mod_s64(v, m);
    }
}

// Two-stage fold for the epilogue: partial() maps the accumulators to a compact value V
// congruent to the result (cheap; runs while the tile holds TMEM), final() reduces it to
// [0, p) after the accumulators are released.
template <int S>
struct SplitFold {
    static constexpr bool ok = false;
};
template <>
struct SplitFold<SCHEME_M17> {
    static constexpr bool ok = true;
    using V = uint32_t;
    // f(x) = (x mod 2^17) + (x >> 17) = x (mod 2^17 - 1); for x < 2^32: f(x) < 2^17 + 2^15
    __device__ __forceinline__ static uint32_t f(uint32_t x) { return (x & 0x1FFFFu) + (x >> 17); }
    // short_k (K <= 2048): per k, a0 <= 63*63 + 2*126*63 = 19845, a1 <= 15876, a2 <= 11907, so
    // a0 + 2^6 a1 + 2^12 f(a2) <= 40.6e6 + 2.08e9 + 2^29.0 < 2^32 -- five integer ops
    __device__ __forceinline__ static V partial(const uint32_t* a, bool short_k) {
        return short_k ? a[0] + (a[1] << 6) + (f(a[2]) << 12)
                       : f(a[0]) + (f(a[1]) << 6) + (f(a[2]) << 12);  // any a < 2^31: < 2^30
    }
    // accumulator s's share of partial() (the staggered epilogue adds them one by one)
    __device__ __forceinline__ static V term(int s, uint32_t a, bool short_k) {
        return s == 0 ? (short_k ? a : f(a)) : s == 1 ? (short_k ? a << 6 : f(a) << 6) : f(a) << 12;
    }
    __device__ __forceinline__ static uint32_t final(V v, const ModP&) {
        const uint32_t r = f(v);  // v < 2^32: r < 2^17 + 2^15 < 2p
        return r >= 0x1FFFFu ? r - 0x1FFFFu : r;
    }
};
template <>
struct SplitFold<SCHEME_M17N> : SplitFold<SCHEME_M17> {};
// LIMB2 (p <= 2^16): the exact integer  sum_x r_x r_y = a0 + 2^8 a1 + 2^16 a2  of the balanced
// representatives, |.| <= K 2^30 < 2^62 within the scheme's K bound; reduced mod p afterwards.
template <>
struct SplitFold<SCHEME_LIMB2> {
    static constexpr bool ok = true;
    using V = int64_t;
    __device__ __forceinline__ static V partial(const uint32_t* a, bool) {
        if constexpr (Scheme<SCHEME_LIMB2>::WIDE && !Scheme<SCHEME_LIMB2>::OVERLAP)  // T00 | T01 | T10 | T11
            return (int64_t)(int32_t)a[0] + ((int64_t)(int32_t)a[1] + (int64_t)(int32_t)a[2]) * 256 +
                   (int64_t)(int32_t)a[3] * 65536;
        return (int64_t)(int32_t)a[0] + (int64_t)(int32_t)a[1] * 256 + (int64_t)(int32_t)a[2] * 65536;
    }
    __device__ __forceinline__ static V term(int s, uint32_t a, bool) {
        return (int64_t)(int32_t)a << (8 * Scheme<SCHEME_LIMB2>::shift(s));
    }
    __device__ __forceinline__ static uint32_t final(V v, const ModP& m) { return mod_s64(v, m); }
};

}  // namespace fsyrk_b200
