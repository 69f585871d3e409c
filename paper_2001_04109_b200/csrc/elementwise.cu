// HBM-bound mod-p elementwise kernels of the recursion.
//
//  convert_in : uint64 reference-layout input -> uint32 residues with the
//               syrkd column transform folded in
//               (include/fsyrk/scaled_syrk.hpp:77-101).  Only used for syrkd;
//               otherwise the first pre-addition reads the caller's matrix.
//  prep       : the fused pre-additions of one level node, Table 3 steps
//               1, 2, 4, 6 (include/fsyrk/fast_syrk.hpp:100-115):
//                 S1 = (A21 - A11) Y, S2 = A22 - A21 Y, S3 = S1 - A22,
//                 S4 = S3 + A12,
//               with the Y multiplication (include/fsyrk/skew.hpp:124-167)
//               and the Pair-form zero padding (fast_syrk.hpp:34-57) fused in.
//               Reads each A element once (uint64 straight from the caller's
//               matrix at the top levels) and writes the GEMM / leaf operands
//               directly as int8 limb planes.
//  post       : the fused post-additions U1..U5 (fast_syrk.hpp:120-132):
//                 X11 = Low(P1 + P2), X21 = U1 + P4 + P3,
//                 X22 = Low(U1 + P4 + P4^T),  U1 = sym(P1 + P5),
//               over 32 x 32 tile pairs with shared-memory transposes; at the
//               root it also applies alpha / beta (the accumulating schedule's
//               scale_* and U5-with-beta, fast_syrk.hpp:202-239) and writes the
//               caller's uint64 C.
//  finalize / mirror / zero_upper: scale_lower_inplace-style accumulate for a
//               root leaf (matrix.hpp:248-263), mirror_lower_to_upper
//               (matrix.hpp:225-232), scrubbing of the scratch upper triangle.
//
// Vector variants move 4 consecutive columns per thread (16-byte loads,
// 4-byte packed limb stores); scalar variants cover unaligned shapes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "elementwise.cuh"
#include "pdl.cuh"
#include "per_device.h"

namespace fsyrk_b200 {

#ifndef FSYRK_PREP_MINB
#define FSYRK_PREP_MINB 3  // measured: cfg2 prep 104 -> 99 us, cfg5 289 -> 278 us (profiles/r01/variants.txt)
#endif
#ifndef FSYRK_CONVERT_ROWS
#define FSYRK_CONVERT_ROWS 1  // rows per iteration of the conversion (4: 0.161 vs 0.149 ms on cfg5)
#endif
// Fused subtree prep staging (cp.async of the caller's raw uint64 values, 44 KB per block and
// 5 blocks / SM).  FSYRK_TREE_OWN = 1: each thread copies exactly the 16 chunks its own level-0
// item reads and waits for those alone (no barrier before level 0); 0: chunks dealt out
// linearly, one barrier.  (A register-staged variant that narrowed to uint32 on the way in --
// 28 KB, 7 blocks / SM -- measured slower: profiles/r02/tree_narrow.txt.)
#ifndef FSYRK_TREE_OWN
#define FSYRK_TREE_OWN 1
#endif
#ifndef FSYRK_TREE_MINB
#define FSYRK_TREE_MINB 5  // fused subtree prep: blocks per SM the registers must allow
#endif
#ifndef FSYRK_POST_STAGED
#define FSYRK_POST_STAGED 1  // post_vec_pair: second-round loads staged by cp.async (one memory round trip per pair)
#endif
#ifndef FSYRK_POST_MINB
#define FSYRK_POST_MINB 6  // measured: cfg2 post 60 -> 55 us, cfg5 2.53 -> 2.13 ms
#endif

namespace {

__global__ void convert_in_kernel(const uint64_t* __restrict__ a, long long lda, int n, int kin, int kout,
                                  const ColMap* __restrict__ map, ModP m, uint32_t* __restrict__ out,
                                  long long ldo) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    (void)kin;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= kout) return;
    const ColMap cm = map ? map[c] : ColMap{{c, -1, -1, -1}, {1, 0, 0, 0}};
    // Shoup constants of this column's coefficients, once per thread: the per-element work is
    // then a 32-bit mul-hi and two multiplies per source (the 64-bit Barrett products made the
    // kernel instruction-bound at 22% of HBM bandwidth, ncu)
    MulConst mc[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) mc[t] = make_mulconst(cm.src[t] >= 0 ? cm.c[t] : 0, m.p);
    // R rows per iteration with every load issued first (memory-level parallelism)
    constexpr int R = FSYRK_CONVERT_ROWS;
    for (int i0 = blockIdx.y * R; i0 < n; i0 += gridDim.y * R) {
        uint64_t x[R][4];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const uint64_t* row = a + (long long)min(i0 + q, n - 1) * lda;
#pragma unroll
            for (int t = 0; t < 4; ++t) x[q][t] = cm.src[t] >= 0 ? row[cm.src[t]] : 0;
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
            if (i0 + q >= n) break;
            uint32_t v = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (cm.src[t] >= 0) {
                    const uint32_t r = x[q][t] < m.p ? (uint32_t)x[q][t] : mod_u64(x[q][t], m);  // canonical: no reduction
                    v = addm(v, mulc(r, mc[t], m.p), m.p);
                }
            out[(long long)(i0 + q) * ldo + c] = v;
        }
    }
}

// ------------------------------------------------------------ input access
struct Src {
    const uint32_t* p32;
    long long ld32;
    const uint64_t* p64;
    long long ld64;
    bool in64;
    // canonical residues are the contract (fields.hpp:32-36); reduce only when one is not
    static __device__ __forceinline__ uint32_t canon(uint64_t x, const ModP& m) {
        return x < m.p ? (uint32_t)x : mod_u64(x, m);
    }
    __device__ __forceinline__ uint32_t ld(int i, int c, const ModP& m) const {
        return in64 ? canon(__ldg(p64 + (long long)i * ld64 + c), m) : __ldg(p32 + (long long)i * ld32 + c);
    }
    // 4 consecutive columns starting at c (c % 4 == 0, rows 16-byte aligned)
    __device__ __forceinline__ uint4 ld4(int i, int c, const ModP& m) const {
        if (in64) {
            const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p64 + (long long)i * ld64 + c);
            const ulonglong2 x = __ldg(q), y = __ldg(q + 1);
            return make_uint4(canon(x.x, m), canon(x.y, m), canon(y.x, m), canon(y.y, m));
        }
        return __ldg(reinterpret_cast<const uint4*>(p32 + (long long)i * ld32 + c));
    }
};

__device__ __forceinline__ Src make_src(const InView& v, const uint64_t* a64, long long ld64) {
    const bool in64 = v.in64 != 0;
    Src s;
    s.in64 = in64;
    s.p32 = v.p32;
    s.ld32 = v.ld32;
    s.p64 = in64 ? a64 + (long long)v.r0 * ld64 + v.c0 : nullptr;
    s.ld64 = ld64;
    return s;
}

// The kernels below are templated on the digit scheme S (schemes.cuh): a residue
// becomes up to planes_of<S>() int8 planes, byte l of encode_planes<S>(x) going to
// plane l (GEMM operands keep only the planes their A / B role reads).
template <int S, int NPL = planes_of<S>()>
__device__ __forceinline__ void put_planes(int8_t* base, long long plane, long long off, uint32_t x, uint32_t p) {
    const uint64_t w = encode_planes<S>(x, p);
#pragma unroll
    for (int l = 0; l < NPL; ++l) base[l * plane + off] = (int8_t)(w >> (8 * l));
}

// Byte-sliced encoding of four residues: gather byte k of the four values into one word
// (3 PRMT), then form every digit plane with whole-word shifts and masks.  For the Mersenne
// schemes this is ~20 integer ops for all planes of four values instead of ~45 per-value ones
// (the pre-addition kernels are issue-bound on the encoding at the deeper levels).
__device__ __forceinline__ uint32_t bytes_k(const uint4& x, int k) { return gather_byte(x.x, x.y, x.z, x.w, k); }

template <int S>
__device__ __forceinline__ void planes4(uint4 x, uint32_t p, uint32_t (&w)[planes_of<S>()]) {
    if constexpr (digits_of<S> == SCHEME_M17) {  // x < 2^17: d0 = x[0:6), d1 = x[6:12), d2 = x[12:17)
        const uint32_t lo = bytes_k(x, 0), hi = bytes_k(x, 1), top = bytes_k(x, 2);
        w[0] = lo & 0x3F3F3F3Fu;
        w[1] = ((lo >> 6) & 0x03030303u) | ((hi << 2) & 0x3C3C3C3Cu);
        w[2] = ((hi >> 4) & 0x0F0F0F0Fu) | ((top << 4) & 0x10101010u);
        w[3] = w[1] << 1;  // 2 d1 <= 126: no carry into the next byte
        w[4] = w[2] << 1;  // 2 d2 <= 62
    } else if constexpr (S == SCHEME_M31) {  // x < 2^31: bytes d0..d3 (d3 < 128) and 2 d3
        w[0] = bytes_k(x, 0);
        w[1] = bytes_k(x, 1);
        w[2] = bytes_k(x, 2);
        w[3] = bytes_k(x, 3);
        w[4] = w[3] << 1;
    } else {
        const uint64_t e0 = encode_planes<S>(x.x, p), e1 = encode_planes<S>(x.y, p), e2 = encode_planes<S>(x.z, p),
                       e3 = encode_planes<S>(x.w, p);
#pragma unroll
        for (int l = 0; l < planes_of<S>(); ++l)
            w[l] = l < 4 ? gather_byte((uint32_t)e0, (uint32_t)e1, (uint32_t)e2, (uint32_t)e3, l)
                         : gather_byte((uint32_t)(e0 >> 32), (uint32_t)(e1 >> 32), (uint32_t)(e2 >> 32),
                                       (uint32_t)(e3 >> 32), l - 4);
    }
}

// four consecutive columns of one row, one 32-bit store per plane (the first NPL planes)
template <int S, int NPL = planes_of<S>()>
__device__ __forceinline__ void put_planes4(int8_t* base, long long plane, long long off, uint4 x, uint32_t p) {
    uint32_t w[planes_of<S>()];
    planes4<S>(x, p, w);
#pragma unroll
    for (int l = 0; l < NPL; ++l) *reinterpret_cast<uint32_t*>(base + l * plane + off) = w[l];
}

template <int L, bool VEC>
__global__ void split_planes_kernel(InView in, const uint64_t* a64, long long ld64, int rows, int k, ModP m,
                                    int8_t* __restrict__ planes, long long plane, long long rs) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    const Src src = make_src(in, a64, ld64);
    constexpr int V = VEC ? 4 : 1;
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) * V;
    if (c >= k) return;
    for (int i = blockIdx.y; i < rows; i += gridDim.y) {
        if constexpr (VEC) {
            put_planes4<L>(planes, plane, (long long)i * rs + c, src.ld4(i, c, m), m.p);
        } else {
            put_planes<L>(planes, plane, (long long)i * rs + c, src.ld(i, c, m), m.p);
        }
    }
}

// ------------------------------------------------------------------ prep
// (u, v) -> (a u - b v, b u + a v) on the column halves (skew.hpp:146-163)
__device__ __forceinline__ void pair_y(uint32_t u, uint32_t v, MulConst ca, MulConst cb, uint32_t p, uint32_t& ru,
                                       uint32_t& rv) {
    ru = subm(mulc(u, ca, p), mulc(v, cb, p), p);
    rv = addm(mulc(u, cb, p), mulc(v, ca, p), p);
}

// Scalar variant: one thread per (row i, column j) or, in Pair form, per column pair (j, j + half).
template <int L>
__global__ void prep_kernel(const __grid_constant__ PrepArgs args) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    const PrepNode nd = args.ninl ? args.inl[blockIdx.z] : args.nodes[blockIdx.z];
    const ModP m = args.m;
    const uint32_t p = m.p;
    const int h = args.h, kh = args.kh, half = args.half;
    const int ncw = args.pair ? half : args.kw;
    const int jp = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y * blockDim.y + threadIdx.y;
    if (jp >= ncw || i >= h) return;
    if (args.part_block && !((args.need_mask >> (i / args.part_block)) & 1ull)) return;  // not this rank's rows
    const Src src = make_src(nd.in, args.a64, args.ld64);

    const int nc = args.pair ? 2 : 1;
    int col[2] = {jp, jp + half};
    uint32_t a11[2], a12[2], a21[2], a22[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int c = col[t];
        const bool ok = t < nc && c < kh;
        a11[t] = ok ? src.ld(i, c, m) : 0;
        a12[t] = ok ? src.ld(i, kh + c, m) : 0;
        a21[t] = ok ? src.ld(i + h, c, m) : 0;
        a22[t] = ok ? src.ld(i + h, kh + c, m) : 0;
    }
    uint32_t s1[2], ay[2];
    if (args.pair) {
        pair_y(subm(a21[0], a11[0], p), subm(a21[1], a11[1], p), args.cya, args.cyb, p, s1[0], s1[1]);
        pair_y(a21[0], a21[1], args.cya, args.cyb, p, ay[0], ay[1]);
    } else {
        s1[0] = mulc(subm(a21[0], a11[0], p), args.cya, p);
        ay[0] = mulc(a21[0], args.cya, p);
        s1[1] = ay[1] = 0;
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        if (t >= nc) break;
        const int c = col[t];
        const uint32_t s2 = subm(a22[t], ay[t], p);
        const uint32_t s3 = subm(s1[t], a22[t], p);
        const uint32_t s4 = addm(s3, a12[t], p);
        const long long go = (long long)i * args.g_row + c;
        if (nd.s1) {
            put_planes<L, Scheme<L>::PA>(nd.s1, args.g_plane, go, s1[t], p);  // A-role: first PA planes
            put_planes<L, Scheme<L>::PA>(nd.a22, args.g_plane, go, a22[t], p);
            put_planes<L, Scheme<L>::PB>(nd.s2, args.g_plane, go, s2, p);  // B-role: first PB planes
            put_planes<L, Scheme<L>::PB>(nd.s4, args.g_plane, go, s4, p);
        } else {  // Winograd operands: residues
            uint32_t* r = nd.r_op + (long long)i * nd.ld_op + c;
            r[0] = s1[t];
            r[nd.op_stride] = s2;
            r[2 * nd.op_stride] = a22[t];
            r[3 * nd.op_stride] = s4;
        }
        if (c < kh) {
            if (nd.c_a11) put_planes<L>(nd.c_a11, args.c_plane, (long long)i * args.c_row + c, a11[t], p);
            if (nd.c_a12) put_planes<L>(nd.c_a12, args.c_plane, (long long)i * args.c_row + c, a12[t], p);
        }
        if (nd.c_s3) put_planes<L>(nd.c_s3, args.c3_plane, (long long)i * args.c3_row + c, s3, p);
        if (nd.r_s3) nd.r_s3[(long long)i * nd.ld_s3 + c] = s3;
    }
}

__device__ __forceinline__ uint4 sub4(uint4 a, uint4 b, uint32_t p) {
    return make_uint4(subm(a.x, b.x, p), subm(a.y, b.y, p), subm(a.z, b.z, p), subm(a.w, b.w, p));
}
__device__ __forceinline__ uint4 add4(uint4 a, uint4 b, uint32_t p) {
    return make_uint4(addm(a.x, b.x, p), addm(a.y, b.y, p), addm(a.z, b.z, p), addm(a.w, b.w, p));
}
__device__ __forceinline__ uint4 mulc4(uint4 a, MulConst c, uint32_t p) {
    return make_uint4(mulc(a.x, c, p), mulc(a.y, c, p), mulc(a.z, c, p), mulc(a.w, c, p));
}
__device__ __forceinline__ void pair_y4(uint4 u, uint4 v, MulConst ca, MulConst cb, uint32_t p, uint4& ru, uint4& rv) {
    pair_y(u.x, v.x, ca, cb, p, ru.x, rv.x);
    pair_y(u.y, v.y, ca, cb, p, ru.y, rv.y);
    pair_y(u.z, v.z, ca, cb, p, ru.z, rv.z);
    pair_y(u.w, v.w, ca, cb, p, ru.w, rv.w);
}

// Vector variant (kh % 4 == 0, half % 4 == 0, no padding): 4 columns (and, in
// Pair form, their 4 partners) per thread.
// 4 x NC quadrant vectors of row i: every load is issued before any is used (memory-level
// parallelism; no branch between loads), then the caller's uint64 values are narrowed with a
// single range check for the whole batch (canonical residues are the contract).
template <bool IN64, int NC>
__device__ __forceinline__ void load_quads(const Src& src, int i, int h, int kh, const int (&col)[2], const ModP& m,
                                           uint4 (&a11)[NC], uint4 (&a12)[NC], uint4 (&a21)[NC], uint4 (&a22)[NC]) {
    if constexpr (IN64) {
        ulonglong2 r[NC][4][2];
#pragma unroll
        for (int t = 0; t < NC; ++t) {
            const int cc[4][2] = {{i, col[t]}, {i, kh + col[t]}, {i + h, col[t]}, {i + h, kh + col[t]}};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const ulonglong2* ptr = reinterpret_cast<const ulonglong2*>(src.p64 + (long long)cc[q][0] * src.ld64 + cc[q][1]);
                r[t][q][0] = __ldg(ptr);
                r[t][q][1] = __ldg(ptr + 1);
            }
        }
        uint64_t big = 0;
#pragma unroll
        for (int t = 0; t < NC; ++t)
#pragma unroll
            for (int q = 0; q < 4; ++q) big |= (r[t][q][0].x | r[t][q][0].y | r[t][q][1].x | r[t][q][1].y) >> 31;
        bool slow = big != 0;
        if (!slow) {
            // all values < 2^31: narrow, then one compare per value decides the (rare) reduction
#pragma unroll
            for (int t = 0; t < NC; ++t)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint4 v = make_uint4((uint32_t)r[t][q][0].x, (uint32_t)r[t][q][0].y, (uint32_t)r[t][q][1].x,
                                               (uint32_t)r[t][q][1].y);
                    slow |= v.x >= m.p || v.y >= m.p || v.z >= m.p || v.w >= m.p;
                }
        }
#pragma unroll
        for (int t = 0; t < NC; ++t) {
            uint4 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint64_t x0 = r[t][q][0].x, x1 = r[t][q][0].y, x2 = r[t][q][1].x, x3 = r[t][q][1].y;
                v[q] = slow ? make_uint4(mod_u64(x0, m), mod_u64(x1, m), mod_u64(x2, m), mod_u64(x3, m))
                            : make_uint4((uint32_t)x0, (uint32_t)x1, (uint32_t)x2, (uint32_t)x3);
            }
            a11[t] = v[0];
            a12[t] = v[1];
            a21[t] = v[2];
            a22[t] = v[3];
        }
    } else {
#pragma unroll
        for (int t = 0; t < NC; ++t) {
            a11[t] = __ldg(reinterpret_cast<const uint4*>(src.p32 + (long long)i * src.ld32 + col[t]));
            a12[t] = __ldg(reinterpret_cast<const uint4*>(src.p32 + (long long)i * src.ld32 + kh + col[t]));
            a21[t] = __ldg(reinterpret_cast<const uint4*>(src.p32 + (long long)(i + h) * src.ld32 + col[t]));
            a22[t] = __ldg(reinterpret_cast<const uint4*>(src.p32 + (long long)(i + h) * src.ld32 + kh + col[t]));
        }
    }
}

template <int S, bool PAIR, bool IN64>
__device__ __forceinline__ void prep_vec_body(const PrepArgs& args, const PrepNode& nd, int i, int g) {
    const ModP m = args.m;
    const uint32_t p = m.p;
    const int h = args.h, kh = args.kh, half = args.half;
    const Src src = make_src(nd.in, args.a64, args.ld64);
    constexpr int NC = PAIR ? 2 : 1;
    const int col[2] = {4 * g, 4 * g + half};
    uint4 a11[NC], a12[NC], a21[NC], a22[NC];
    load_quads<IN64, NC>(src, i, h, kh, col, m, a11, a12, a21, a22);
    uint4 s1[NC], ay[NC];
    if constexpr (PAIR) {
        pair_y4(sub4(a21[0], a11[0], p), sub4(a21[1], a11[1], p), args.cya, args.cyb, p, s1[0], s1[1]);
        pair_y4(a21[0], a21[1], args.cya, args.cyb, p, ay[0], ay[1]);
    } else {
        s1[0] = mulc4(sub4(a21[0], a11[0], p), args.cya, p);
        ay[0] = mulc4(a21[0], args.cya, p);
    }
#pragma unroll
    for (int t = 0; t < NC; ++t) {
        const int c = col[t];
        const uint4 s2 = sub4(a22[t], ay[t], p);
        const uint4 s3 = sub4(s1[t], a22[t], p);
        const uint4 s4 = add4(s3, a12[t], p);
        const long long go = (long long)i * args.g_row + c;
        // GEMM operands keep the planes of their role; leaf operands (read as A and B) all
        constexpr int PA = Scheme<S>::PA, PB = Scheme<S>::PB;
        if (nd.s1) {
            put_planes4<S, PA>(nd.s1, args.g_plane, go, s1[t], p);
            put_planes4<S, PA>(nd.a22, args.g_plane, go, a22[t], p);
            put_planes4<S, PB>(nd.s2, args.g_plane, go, s2, p);
            put_planes4<S, PB>(nd.s4, args.g_plane, go, s4, p);
        } else {  // Winograd operands: residues (ld_op % 4 == 0, driver-checked via `aligned`)
            uint32_t* r = nd.r_op + (long long)i * nd.ld_op + c;
            *reinterpret_cast<uint4*>(r) = s1[t];
            *reinterpret_cast<uint4*>(r + nd.op_stride) = s2;
            *reinterpret_cast<uint4*>(r + 2 * nd.op_stride) = a22[t];
            *reinterpret_cast<uint4*>(r + 3 * nd.op_stride) = s4;
        }
        if (nd.c_a11) put_planes4<S>(nd.c_a11, args.c_plane, (long long)i * args.c_row + c, a11[t], p);
        if (nd.c_a12) put_planes4<S>(nd.c_a12, args.c_plane, (long long)i * args.c_row + c, a12[t], p);
        if (nd.c_s3) put_planes4<S>(nd.c_s3, args.c3_plane, (long long)i * args.c3_row + c, s3, p);
        if (nd.r_s3) *reinterpret_cast<uint4*>(nd.r_s3 + (long long)i * nd.ld_s3 + c) = s3;
    }
}

// Vector variant (kh % 4 == 0, half % 4 == 0, no padding): 4 columns (and, in
// Pair form, their 4 partners) per thread; one specialised body per input kind.
template <int S, bool PAIR>
__global__ void __launch_bounds__(256, FSYRK_PREP_MINB) prep_vec_kernel(const __grid_constant__ PrepArgs args) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    const int ncg = (PAIR ? args.half : args.kh) / 4;
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y * blockDim.y + threadIdx.y;
    if (g >= ncg || i >= args.h) return;
    if (args.part_block && !((args.need_mask >> (i / args.part_block)) & 1ull)) return;  // not this rank's rows
    const PrepNode local = args.ninl ? args.inl[blockIdx.z] : args.nodes[blockIdx.z];
    if (local.in.in64) prep_vec_body<S, PAIR, true>(args, local, i, g);
    else prep_vec_body<S, PAIR, false>(args, local, i, g);
}

// ------------------------------------------------------------ prep (fused subtree)
// All D levels of a complete uniform subtree in one pass over the caller's uint64 A
// (fast_syrk.hpp:100-115 at every node).  A CTA owns CP consecutive columns c0 .. c0 + CP of
// one row r of the leaf-sized fine block (in Pair form also their partners c + w/2: Y pairs
// columns half a quadrant apart at every level, so the partners of a CTA's columns are again
// its own columns) and stages their values in all 4^D fine blocks of A in shared memory.  Each
// level then forms S1..S4 of all its nodes from shared memory, writes the GEMM operands as
// digit planes (4 columns per thread, packed 4-byte stores) and hands A11, A12, S3 to the
// children in shared memory; the deepest level writes the leaf operands.  Compared with one
// launch per depth this drops the uint32 S3 residues of every non-leaf child (written once,
// read once) and the small latency-bound launches of the deep levels.
//
// Shared layout of level d (node t of 3^d, B = 2^(D-d) fine blocks per side, NC = 2 in Pair
// form): buf[((t * B + bi) * (B * NC) + v) * CP + cp], v = bj * NC + e the "virtual column"
// (fine block column bj, half e).  A quadrant is a half in each direction; the Pair partner of
// virtual column v (< V/2) of a V-wide quadrant is v + V/2.  Levels alternate between two
// buffers (level 0 and 2 in one, level 1 in the other).
// columns (column pairs) per CTA at most: 128 work items at level 0 for D = 3 (32) and D = 2 (128)
constexpr int kTreeCP = 32, kTreeCP2 = 128;
constexpr int kTreeThreads = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}

// One level d of the fused subtree: every node's S1..S4 from shared memory (level 0: the raw
// uint64 input), GEMM operand planes to HBM, children's inputs (or leaf operand planes) out.
// Everything but the column-group count is compile-time (powers of two: shifts and masks).
template <int S, bool PAIR, int D, int d>
__device__ __forceinline__ void tree_level(const PrepTreeArgs& a, const uint64_t* raw, const uint32_t* in,
                                           uint32_t* out, int r, int c0, int CP, int lgG) {
    constexpr int NC = PAIR ? 2 : 1, NU = PAIR ? 2 : 1;
    constexpr int PA = Scheme<S>::PA, PB = Scheme<S>::PB;
    constexpr int Bq = 1 << (D - d - 1), B = 2 * Bq;  // quadrant / node size in fine blocks
    constexpr int V = Bq * NC, W2 = 2 * V;            // virtual columns of a quadrant / of the node
    constexpr int U = PAIR ? V / 2 : V;               // work columns per quadrant row
    constexpr int NODES = d == 0 ? 1 : d == 1 ? 3 : 9;
    constexpr bool last = d == D - 1;
    const uint32_t p = a.m.p;
    const ModP m = a.m;
    const int half = a.w / 2, G = 1 << lgG;
    const long long gp = a.g_plane[d], gr = a.g_row[d];
    const int items = NODES * Bq * U << lgG;
    for (int it = threadIdx.x; it < items; it += kTreeThreads) {
        const int g = it & (G - 1);
        const int rest = it >> lgG;
        const int u = rest % U, qi = (rest / U) % Bq, t = rest / (U * Bq);
        const PrepTreeArgs::Ptrs& nd = a.tp[(d == 0 ? 0 : d == 1 ? 1 : 4) + t];
        uint4 a11[NU], a12[NU], a21[NU], a22[NU], s1[NU], ay[NU];
        auto at = [&](int bi, int v) -> uint4 {
            const int o = ((t * B + bi) * W2 + v) * CP + 4 * g;
            if constexpr (d > 0) {
                return *reinterpret_cast<const uint4*>(in + o);
            } else {
                // the caller's uint64 values: canonical residues are the contract (fields.hpp:32-36);
                // reduce only the ones that are not
                const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(raw + o);
                const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(raw + o + 2);
                // branch-free canonical test: every high word zero and every low word < p
                const uint32_t l0 = (uint32_t)x.x, l1 = (uint32_t)x.y, l2 = (uint32_t)y.x, l3 = (uint32_t)y.y;
                const uint32_t hi = (uint32_t)(x.x >> 32) | (uint32_t)(x.y >> 32) | (uint32_t)(y.x >> 32) |
                                    (uint32_t)(y.y >> 32);
                const bool ok = (hi == 0) & (l0 < p) & (l1 < p) & (l2 < p) & (l3 < p);
                if (!ok) return make_uint4(mod_u64(x.x, m), mod_u64(x.y, m), mod_u64(y.x, m), mod_u64(y.y, m));
                return make_uint4(l0, l1, l2, l3);
            }
        };
#pragma unroll
        for (int e = 0; e < NU; ++e) {
            const int ue = u + e * (V / 2);
            a11[e] = at(qi, ue);
            a12[e] = at(qi, V + ue);
            a21[e] = at(Bq + qi, ue);
            a22[e] = at(Bq + qi, V + ue);
        }
        if constexpr (PAIR) {
            pair_y4(sub4(a21[0], a11[0], p), sub4(a21[1], a11[1], p), a.cya, a.cyb, p, s1[0], s1[1]);
            pair_y4(a21[0], a21[1], a.cya, a.cyb, p, ay[0], ay[1]);
        } else {
            s1[0] = mulc4(sub4(a21[0], a11[0], p), a.cya, p);
            ay[0] = mulc4(a21[0], a.cya, p);
        }
        const long long row = (long long)qi * a.rows + r;
#pragma unroll
        for (int e = 0; e < NU; ++e) {
            const int uu = u + e * (V / 2);
            const uint4 s2 = sub4(a22[e], ay[e], p);
            const uint4 s3 = sub4(s1[e], a22[e], p);
            const uint4 s4 = add4(s3, a12[e], p);
            const int cin = c0 + 4 * g + (uu % NC) * half;  // column inside the fine block
            const long long go = row * gr + (long long)(uu / NC) * a.w + cin;
            put_planes4<S, PA>(nd.s1, gp, go, s1[e], p);  // A-role: first PA planes
            put_planes4<S, PA>(nd.a22, gp, go, a22[e], p);
            put_planes4<S, PB>(nd.s2, gp, go, s2, p);  // B-role: first PB planes
            put_planes4<S, PB>(nd.s4, gp, go, s4, p);
            if constexpr (last) {  // children are leaves: all planes
                const long long lo = (long long)r * a.c_row + cin;
                put_planes4<S>(nd.c_a11, a.c_plane, lo, a11[e], p);
                put_planes4<S>(nd.c_a12, a.c_plane, lo, a12[e], p);
                put_planes4<S>(nd.c_s3, a.c_plane, lo, s3, p);
            } else {  // child 3t + role (Bq x Bq blocks): virtual column uu of block row qi
                const int o = (qi * V + uu) * CP + 4 * g;
                const int cs = Bq * V * CP;  // one child's input
                *reinterpret_cast<uint4*>(out + (3 * t + 0) * cs + o) = a11[e];
                *reinterpret_cast<uint4*>(out + (3 * t + 1) * cs + o) = a12[e];
                *reinterpret_cast<uint4*>(out + (3 * t + 2) * cs + o) = s3;
            }
        }
    }
}

template <int S, bool PAIR, int D>
__global__ void __launch_bounds__(kTreeThreads, FSYRK_TREE_MINB) prep_tree_kernel(const __grid_constant__ PrepTreeArgs a) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    extern __shared__ __align__(16) uint32_t tsm[];
    constexpr int NC = PAIR ? 2 : 1, B = 1 << D;
    const int CP = a.cp, lgCP = 31 - __clz(CP);
    const int r = blockIdx.y, c0 = blockIdx.x * CP;
    const int half = a.w / 2;
    // buffer 0: the root's raw uint64 input, later level 2; buffer 1: level 1
    constexpr int kSegs = B * B * NC;
    uint64_t* raw = reinterpret_cast<uint64_t*>(tsm);
    uint32_t* buf1 = tsm + 2 * (kSegs << lgCP);
    const int lgG = lgCP - 2;
#if FSYRK_TREE_OWN
    {
        // Every raw value is read exactly once, by the level-0 work item that owns its four
        // columns: each thread copies its own item's 16 chunks (8 locations x 32 bytes) and waits
        // for those alone -- no block-wide barrier before level 0.
        constexpr int Bq = B / 2, V = Bq * NC, W2 = 2 * V, U = PAIR ? V / 2 : V, NU = PAIR ? 2 : 1;
        const int it = threadIdx.x;
        if (it < (Bq * U << lgG)) {
            const int g = it & ((1 << lgG) - 1), rest = it >> lgG;
            const int u = rest % U, qi = (rest / U) % Bq;
#pragma unroll
            for (int e = 0; e < NU; ++e) {
                const int ue = u + e * (V / 2);
                const int bis[2] = {qi, Bq + qi}, vs[2] = {ue, V + ue};
#pragma unroll
                for (int bb = 0; bb < 2; ++bb)
#pragma unroll
                    for (int vv = 0; vv < 2; ++vv) {
                        const int bi = bis[bb], v = vs[vv];
                        const int o = (bi * W2 + v) * CP + 4 * g;
                        const long long row = (long long)bi * a.rows + r;
                        const long long col = (long long)(v / NC) * a.w + c0 + 4 * g + (v % NC) * half;
                        const uint64_t* src = a.a64 + row * a.ld64 + col;
                        cp_async16(raw + o, src);
                        cp_async16(raw + o + 2, src + 2);
                    }
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
#else
    {
        // every 16-byte chunk of the CTA's 4^D x NC segments of CP columns in flight at once
        const int chunks = (kSegs << lgCP) / 2;
        for (int ch = threadIdx.x; ch < chunks; ch += kTreeThreads) {
            const int idx = 2 * ch, cp = idx & (CP - 1), seg = idx >> lgCP;
            const int v = seg % (B * NC), bi = seg / (B * NC);
            const long long row = (long long)bi * a.rows + r;
            const long long col = (long long)(v / NC) * a.w + c0 + cp + (v % NC) * half;
            cp_async16(raw + idx, a.a64 + row * a.ld64 + col);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
#endif
    tree_level<S, PAIR, D, 0>(a, raw, nullptr, D > 1 ? buf1 : nullptr, r, c0, CP, lgG);
    if constexpr (D > 1) {
        __syncthreads();
        tree_level<S, PAIR, D, (D > 1 ? 1 : 0)>(a, nullptr, buf1, tsm, r, c0, CP, lgG);
    }
    if constexpr (D > 2) {
        __syncthreads();
        tree_level<S, PAIR, D, (D > 2 ? 2 : 0)>(a, nullptr, tsm, nullptr, r, c0, CP, lgG);
    }
}

size_t prep_tree_smem(int D, bool pair, int cp) {
    const size_t nc = pair ? 2 : 1;
    // buffer 0: the root's uint64 input (4^D blocks; level 2's 9 x 4^(D-2) uint32 blocks fit in
    // it); buffer 1: level 1 = 3 * 4^(D-1) blocks of uint32
    return ((size_t)1 << (2 * D)) * nc * cp * 8 + 3 * ((size_t)1 << (2 * (D - 1))) * nc * cp * 4;
}

template <int S, bool PAIR, int D>
struct TreeAttrOnce : DeviceOnce {};
struct Post2AttrOnce : DeviceOnce {};

template <int S>
cudaError_t prep_tree_dispatch(const PrepTreeArgs& a, int nsm, cudaStream_t s) {
    (void)nsm;
    const bool pair = a.pair != 0;
    const int nc = pair ? 2 : 1;
    if (a.cp < 4 || a.cp > (a.depth == 3 ? kTreeCP : kTreeCP2) || (a.cp & (a.cp - 1)) || (a.w / nc) % a.cp ||
        (pair && a.w % 2) || a.depth < 2 || a.depth > 3)
        return cudaErrorInvalidValue;
    const size_t smem = prep_tree_smem(a.depth, pair, a.cp);
    dim3 grid(a.w / nc / a.cp, a.rows);
    auto kern = a.depth == 3 ? (pair ? prep_tree_kernel<S, true, 3> : prep_tree_kernel<S, false, 3>)
                             : (pair ? prep_tree_kernel<S, true, 2> : prep_tree_kernel<S, false, 2>);
    // thread-safe one-time setup per device (the attribute applies to the current device only)
    DeviceOnce& once = a.depth == 3 ? (pair ? static_cast<DeviceOnce&>(per_device<TreeAttrOnce<S, true, 3>>())
                                            : static_cast<DeviceOnce&>(per_device<TreeAttrOnce<S, false, 3>>()))
                                     : (pair ? static_cast<DeviceOnce&>(per_device<TreeAttrOnce<S, true, 2>>())
                                             : static_cast<DeviceOnce&>(per_device<TreeAttrOnce<S, false, 2>>()));
    std::call_once(once.flag, [&] {
        once.result = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max(prep_tree_smem(3, true, kTreeCP), prep_tree_smem(2, true, kTreeCP2)));
    });
    if (once.result != cudaSuccess) return once.result;
    return launch_pdl(kern, grid, dim3(kTreeThreads), smem, s, a);
}

// ------------------------------------------------------------------ post
constexpr int TS = 32;  // post / mirror tile

__device__ __forceinline__ void tri_decode(int t, int& I, int& J) {
    int r = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    I = r;
    J = t - r * (r + 1) / 2;
}

struct PostOut {
    uint32_t* x;
    long long ldx;
    uint64_t* c;
    long long ldc;
    bool out64, vec64;
    uint32_t alpha, beta;
    MulConst ca, cb;  // Shoup constants of alpha, beta (32-bit products instead of 64-bit Barrett)
    ModP m;
    // write element (i, j) of the node output (lower triangle for out64)
    __device__ __forceinline__ void put(long long i, long long j, uint32_t v) const {
        if (!out64) {
            x[i * ldx + j] = v;
            return;
        }
        c[i * ldc + j] = acc(v, beta != 0 ? c[i * ldc + j] : 0);
    }
    __device__ __forceinline__ uint32_t acc(uint32_t v, uint64_t cin) const {
        uint32_t r = alpha == 1 ? v : mulc(v, ca, m.p);
        if (beta != 0) {
            const uint32_t ci = cin < m.p ? (uint32_t)cin : mod_u64(cin, m);  // canonical C_in: no reduction
            r = addm(r, beta == 1 ? ci : mulc(ci, cb, m.p), m.p);
        }
        return r;
    }
    __device__ __forceinline__ void put4(long long i, long long j, uint4 v) const {
        if (!out64) {
            *reinterpret_cast<uint4*>(x + i * ldx + j) = v;
            return;
        }
        if (vec64) {  // ldc even, C 16-byte aligned: two 16-byte stores
            ulonglong2* q = reinterpret_cast<ulonglong2*>(c + i * ldc + j);
            ulonglong2 c0 = make_ulonglong2(0, 0), c1 = c0;
            if (beta != 0) {
                c0 = q[0];
                c1 = q[1];
            }
            q[0] = make_ulonglong2(acc(v.x, c0.x), acc(v.y, c0.y));
            q[1] = make_ulonglong2(acc(v.z, c1.x), acc(v.w, c1.y));
            return;
        }
        put(i, j, v.x);
        put(i, j + 1, v.y);
        put(i, j + 2, v.z);
        put(i, j + 3, v.w);
    }
};

__device__ __forceinline__ PostOut make_out(const PostArgs& a, const PostNode& nd) {
    PostOut o;
    o.x = nd.x;
    o.ldx = nd.ldx;
    o.c = a.c64;
    o.ldc = a.ldc;
    o.out64 = a.out64 != 0;
    o.vec64 = o.out64 && !(a.ldc % 2) && !(reinterpret_cast<uintptr_t>(a.c64) % 16);
    o.alpha = a.alpha;
    o.beta = a.beta;
    o.ca = a.calpha;
    o.cb = a.cbeta;
    o.m = a.m;
    return o;
}

// Block (32 x 8) per tile pair (I >= J) of one node.
__global__ void post_kernel(const __grid_constant__ PostArgs args) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    __shared__ uint32_t sU[TS][TS + 1];  // Low(P1 + P5), tile (I, J)
    __shared__ uint32_t sT[TS][TS + 1];  // P4 tile (J, I)
    const PostNode nd = post_node(args, args.ninl ? args.inl[blockIdx.z] : args.nodes[blockIdx.z]);
    const uint32_t p = args.m.p;
    const int h = args.h;
    const PostOut out = make_out(args, nd);
    int I, J;
    if (args.pairs) {
        I = args.pairs[blockIdx.x].x;
        J = args.pairs[blockIdx.x].y;
    } else {
        tri_decode(blockIdx.x, I, J);
    }
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int j = J * TS + tx;   // column inside tile (I, J)
    const int jt = I * TS + tx;  // column inside tile (J, I)
    for (int r = ty; r < TS; r += 8) {
        const int i = I * TS + r, it = J * TS + r;
        uint32_t u = 0, t4 = 0;
        if (i < h && j < h) u = addm(nd.p1[(long long)i * nd.ld1 + j], nd.p5[(long long)i * nd.ld5 + j], p);
        if (it < h && jt < h) t4 = nd.p4[(long long)it * nd.ld4 + jt];
        sU[r][tx] = u;
        sT[r][tx] = t4;
    }
    __syncthreads();
    for (int r = ty; r < TS; r += 8) {
        const int i = I * TS + r;
        if (i < h && j < h) {
            const uint32_t u1 = (I == J && tx > r) ? sU[tx][r] : sU[r][tx];
            const uint32_t p4 = nd.p4[(long long)i * nd.ld4 + j];
            const uint32_t p3 = nd.p3[(long long)i * nd.ld3 + j];
            const uint32_t u2 = addm(u1, p4, p);
            out.put(h + i, j, addm(u2, p3, p));
            if (!out.out64 || j <= i) {
                out.put(h + i, h + j, addm(u2, sT[tx][r], p));
                out.put(i, j, addm(nd.p1[(long long)i * nd.ld1 + j], nd.p2[(long long)i * nd.ld2 + j], p));
            }
        }
        if (I != J) {
            const int it = J * TS + r;
            if (it < h && jt < h)
                out.put(h + it, jt, addm(addm(sU[tx][r], sT[r][tx], p), nd.p3[(long long)it * nd.ld3 + jt], p));
        }
    }
}

// Vector variant (h, all ld % 4 == 0): block (8 x 32), thread = 4 columns of one row.
// One 32 x 32 tile pair (I >= J) of a node's post-addition, 8 x 32 threads.
// STAGED: the loads that do not feed the shared-memory transposes (P4, P3, P2 of tile (I, J) and
// P3 of tile (J, I)) start as cp.async copies into sP before anything else, each thread copying
// what it reads back itself, so the pair is one round trip to memory instead of two dependent
// ones (the root post was latency-bound at ~31% of DRAM throughput, profiles/r02/ncu_post_cfg2.md)
// without holding registers across the barrier.
template <bool STAGED>
__device__ __forceinline__ void post_vec_pair(const PostArgs& args, const PostNode& nd, int I, int J,
                                              uint32_t (&sU)[TS][TS + 1], uint32_t (&sT)[TS][TS + 1],
                                              uint4 (*sP)[TS][TS / 4]) {
    const uint32_t p = args.m.p;
    const int h = args.h;
    const PostOut out = make_out(args, nd);
    const int tx = threadIdx.x, r = threadIdx.y;
    const int c0 = 4 * tx;
    const int i = I * TS + r, j = J * TS + c0;        // tile (I, J)
    const int it = J * TS + r, jt = I * TS + c0;      // tile (J, I)
    const bool ok = i < h && j < h, okt = it < h && jt < h;
    if constexpr (STAGED) {
        if (ok) {
            cp_async16(&sP[0][r][tx], nd.p4 + (long long)i * nd.ld4 + j);
            cp_async16(&sP[1][r][tx], nd.p3 + (long long)i * nd.ld3 + j);
            cp_async16(&sP[2][r][tx], nd.p2 + (long long)i * nd.ld2 + j);
        }
        if (I != J && okt) cp_async16(&sP[3][r][tx], nd.p3 + (long long)it * nd.ld3 + jt);
    }
    uint4 p1 = {0, 0, 0, 0}, p5 = p1, p4t = p1;
    if (ok) {
        p1 = *reinterpret_cast<const uint4*>(nd.p1 + (long long)i * nd.ld1 + j);
        p5 = *reinterpret_cast<const uint4*>(nd.p5 + (long long)i * nd.ld5 + j);
    }
    if (okt) p4t = *reinterpret_cast<const uint4*>(nd.p4 + (long long)it * nd.ld4 + jt);
    const uint4 l15 = add4(p1, p5, p);
    sU[r][c0] = l15.x; sU[r][c0 + 1] = l15.y; sU[r][c0 + 2] = l15.z; sU[r][c0 + 3] = l15.w;
    sT[r][c0] = p4t.x; sT[r][c0 + 1] = p4t.y; sT[r][c0 + 2] = p4t.z; sT[r][c0 + 3] = p4t.w;
    if constexpr (STAGED) asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (ok) {
        const uint4 p4 = STAGED ? sP[0][r][tx] : *reinterpret_cast<const uint4*>(nd.p4 + (long long)i * nd.ld4 + j);
        const uint4 p3 = STAGED ? sP[1][r][tx] : *reinterpret_cast<const uint4*>(nd.p3 + (long long)i * nd.ld3 + j);
        const uint4 p2 = STAGED ? sP[2][r][tx] : *reinterpret_cast<const uint4*>(nd.p2 + (long long)i * nd.ld2 + j);
        uint32_t u1[4], t4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = c0 + e;
            u1[e] = (I == J && c > r) ? sU[c][r] : sU[r][c];
            t4[e] = sT[c][r];
        }
        const uint4 u2 = add4(make_uint4(u1[0], u1[1], u1[2], u1[3]), p4, p);
        const uint4 x21 = add4(u2, p3, p);
        const uint4 x22 = add4(u2, make_uint4(t4[0], t4[1], t4[2], t4[3]), p);
        const uint4 x11 = add4(p1, p2, p);
        out.put4(h + i, j, x21);
        if (!out.out64 || I != J) {
            out.put4(h + i, h + j, x22);
            out.put4(i, j, x11);
        } else {  // diagonal tile of the caller's C: lower entries only
            const uint32_t a22[4] = {x22.x, x22.y, x22.z, x22.w}, a11[4] = {x11.x, x11.y, x11.z, x11.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (c0 + e <= r) {
                    out.put(h + i, h + j + e, a22[e]);
                    out.put(i, j + e, a11[e]);
                }
        }
    }
    if (I != J && okt) {
        const uint4 p3t = STAGED ? sP[3][r][tx] : *reinterpret_cast<const uint4*>(nd.p3 + (long long)it * nd.ld3 + jt);
        uint32_t v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = addm(sU[c0 + e][r], sT[r][c0 + e], p);
        out.put4(h + it, jt, add4(make_uint4(v[0], v[1], v[2], v[3]), p3t, p));
    }
}

// INL: the node table is read from the launch parameters (PostArgs::inl) instead of HBM
template <bool INL>
__global__ void __launch_bounds__(256, FSYRK_POST_MINB) post_vec_kernel(const __grid_constant__ PostArgs args) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    __shared__ uint32_t sU[TS][TS + 1];
    __shared__ uint32_t sT[TS][TS + 1];
    __shared__ __align__(16) uint4 sP[FSYRK_POST_STAGED ? 4 : 1][TS][TS / 4];  // P4, P3, P2 (I, J), P3 (J, I)
    const PostNode nd = post_node(args, INL ? args.inl[blockIdx.z] : args.nodes[blockIdx.z]);
    int I, J;
    if (args.pairs) {
        I = args.pairs[blockIdx.x].x;
        J = args.pairs[blockIdx.x].y;
    } else {
        tri_decode(blockIdx.x, I, J);
    }
    post_vec_pair<FSYRK_POST_STAGED != 0>(args, nd, I, J, sU, sT, sP);
}

// ------------------------------------------------------------ post (two levels fused)
// A block owns one 32 x 32 tile pair (i, j) of the deepest nodes' quadrants for one parent t.
// Phase A: the three children (P1, P2, P5 of t) run their post-addition of pair (i, j) into
// shared memory: 4 output tiles each (slots 0: X11(i,j), 1: X21(i,j), 2: X21(j,i), 3: X22(i,j);
// slot 2 is slot 1 when i == j).  Slot s of a child's output is tile (I_s, J_s) of the child's
// X = the parent's quadrant, with (I_s, J_s) = (i,j), (T+i,j), (T+j,i), (T+i,T+j), T = h2 / 32:
// exactly the tile the parent's pair (I_s, J_s) reads from P1, P2, P5.  Phase B: the parent's
// pairs (I_s, J_s) from those tiles and its P3 / P4 in HBM.  The children's X never round-trip
// through HBM and one launch replaces two; every global load of a phase is issued before its
// barrier (3 blocks / SM by shared memory, so the registers allow it).
#ifndef FSYRK_POST2_UNROLL
#define FSYRK_POST2_UNROLL 1  // the seven steps fully unrolled; rolled (0) measured slower: cfg2 post 45.2 -> 48.2 us (profiles/r02/post2.txt)
#endif
#ifndef FSYRK_POST2_TILE
#define FSYRK_POST2_TILE 32  // measured: 16 -> cfg2 post 61 us, 32 -> 53 us (per-depth: 51 us, but one launch more)
#endif
constexpr int PT = FSYRK_POST2_TILE;  // post2 tile (PT x PT), PT / 4 x PT threads, 4 columns each
constexpr int kPostTile = PT * (PT + 1);

__device__ __forceinline__ uint4 ld4g(const uint32_t* base, long long ld, int i, int j, bool ok) {
    return ok ? *reinterpret_cast<const uint4*>(base + (long long)i * ld + j) : make_uint4(0, 0, 0, 0);
}
__device__ __forceinline__ void st4s(uint32_t* t, int r, int c, uint4 v) {
    t[r * (PT + 1) + c] = v.x;
    t[r * (PT + 1) + c + 1] = v.y;
    t[r * (PT + 1) + c + 2] = v.z;
    t[r * (PT + 1) + c + 3] = v.w;
}
__device__ __forceinline__ uint4 ld4s(const uint32_t* t, int r, int c) {
    return make_uint4(t[r * (PT + 1) + c], t[r * (PT + 1) + c + 1], t[r * (PT + 1) + c + 2], t[r * (PT + 1) + c + 3]);
}
// 4 consecutive columns c .. c + 3 of row r of the transpose of tile t
__device__ __forceinline__ uint4 ld4sT(const uint32_t* t, int r, int c) {
    return make_uint4(t[c * (PT + 1) + r], t[(c + 1) * (PT + 1) + r], t[(c + 2) * (PT + 1) + r], t[(c + 3) * (PT + 1) + r]);
}
// U1 tile (P1 + P5), symmetrised from its lower triangle on a diagonal pair
__device__ __forceinline__ uint4 u1_row(const uint32_t* u, int r, int c0, bool diag) {
    uint32_t v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int c = c0 + e;
        v[e] = (diag && c > r) ? u[c * (PT + 1) + r] : u[r * (PT + 1) + c];
    }
    return make_uint4(v[0], v[1], v[2], v[3]);
}

template <bool INL>
__global__ void __launch_bounds__(PT * PT / 4, 3) post2_kernel(const __grid_constant__ Post2Args args) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    extern __shared__ __align__(16) uint32_t psm[];
    uint32_t* sX = psm;                     // [3 children][4 slots] output tiles
    uint32_t* sU = psm + 12 * kPostTile;    // U1 tile of the current step (P1 + P5)
    uint32_t* sT = sU + kPostTile;          // P4 tile (J, I) of the current step, read transposed
    const uint32_t p = args.par.m.p;
    const int h2 = args.h2, T = h2 / PT;
    int i2, j2;
    tri_decode(blockIdx.x, i2, j2);
    const bool dg = i2 == j2;
    const int t = blockIdx.z;
    const int tx = threadIdx.x, r = threadIdx.y, c0 = 4 * tx;
    const PostNode pn = post_node(args.par, INL ? args.par.inl[t] : args.par.nodes[t]);
    const PostOut out = make_out(args.par, pn);
    const int h = args.par.h;
    // parent pair of child output slot s
    const int PI[4] = {i2, T + i2, T + j2, T + i2}, PJ[4] = {j2, j2, i2, T + j2};
    // Seven steps, one tile pair each: the three children's pair (i2, j2) (outputs to shared
    // memory), then the parent's pairs at the children's output slots (outputs to HBM).  The
    // next step's global loads are issued before the current step's barrier (software
    // pipelining: two temporary tiles instead of one per step, 3 blocks / SM).
    auto load = [&](int st, uint4 (&v)[7]) {
        if (st < 3) {
            const PostNode nd = INL ? args.chi[3 * t + st] : args.ch[3 * t + st];
            const int i = i2 * PT + r, j = j2 * PT + c0, it = j2 * PT + r, jt = i2 * PT + c0;
            v[0] = ld4g(nd.p1, nd.ld1, i, j, true);
            v[1] = ld4g(nd.p5, nd.ld5, i, j, true);
            v[2] = ld4g(nd.p4, nd.ld4, it, jt, true);
            v[3] = ld4g(nd.p4, nd.ld4, i, j, true);
            v[4] = ld4g(nd.p3, nd.ld3, i, j, true);
            v[5] = ld4g(nd.p2, nd.ld2, i, j, true);
            v[6] = ld4g(nd.p3, nd.ld3, it, jt, !dg);
        } else {
            const int s = st - 3, I = PI[s], J = PJ[s];
            const int i = I * PT + r, j = J * PT + c0, it = J * PT + r, jt = I * PT + c0;
            v[2] = ld4g(pn.p4, pn.ld4, it, jt, true);
            v[3] = ld4g(pn.p4, pn.ld4, i, j, true);
            v[4] = ld4g(pn.p3, pn.ld3, i, j, true);
            v[6] = ld4g(pn.p3, pn.ld3, it, jt, I != J);
        }
    };
    uint4 cur[7], nxt[7];
    load(0, cur);
#if FSYRK_POST2_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int st = 0; st < 7; ++st) {
        if (st == 5 && dg) continue;  // parent slot 2 is slot 1 on a diagonal pair
        const int s = st - 3;
        if (st < 3) {
            st4s(sU, r, c0, add4(cur[0], cur[1], p));
        } else {
            st4s(sU, r, c0, add4(ld4s(sX + (4 * 0 + s) * kPostTile, r, c0), ld4s(sX + (4 * 2 + s) * kPostTile, r, c0), p));
        }
        st4s(sT, r, c0, cur[2]);
        const int nst = st + 1 + ((st + 1 == 5 && dg) ? 1 : 0);
        if (nst < 7) load(nst, nxt);
        __syncthreads();
        if (st < 3) {  // child st: its four output slots into shared memory
            uint32_t* x = sX + 4 * st * kPostTile;
            const uint4 u2 = add4(u1_row(sU, r, c0, dg), cur[3], p);
            st4s(x + 0 * kPostTile, r, c0, add4(cur[0], cur[5], p));          // X11(i,j) = P1 + P2
            st4s(x + 1 * kPostTile, r, c0, add4(u2, cur[4], p));              // X21(i,j)
            st4s(x + 3 * kPostTile, r, c0, add4(u2, ld4sT(sT, r, c0), p));    // X22(i,j)
            if (!dg)                                                            // X21(j,i)
                st4s(x + 2 * kPostTile, r, c0, add4(add4(ld4sT(sU, r, c0), ld4s(sT, r, c0), p), cur[6], p));
        } else {  // the parent's pair at child slot s
            const int I = PI[s], J = PJ[s];
            const bool pdiag = I == J;
            const int i = I * PT + r, j = J * PT + c0;
            const uint4 u2 = add4(u1_row(sU, r, c0, pdiag), cur[3], p);
            const uint4 x21 = add4(u2, cur[4], p);
            const uint4 x22 = add4(u2, ld4sT(sT, r, c0), p);
            const uint4 x11 =
                add4(ld4s(sX + (4 * 0 + s) * kPostTile, r, c0), ld4s(sX + (4 * 1 + s) * kPostTile, r, c0), p);
            out.put4(h + i, j, x21);
            if (!out.out64 || !pdiag) {
                out.put4(h + i, h + j, x22);
                out.put4(i, j, x11);
            } else {  // diagonal tile of the caller's C: lower entries only
                const uint32_t a22[4] = {x22.x, x22.y, x22.z, x22.w}, a11[4] = {x11.x, x11.y, x11.z, x11.w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (c0 + e <= r) {
                        out.put(h + i, h + j + e, a22[e]);
                        out.put(i, j + e, a11[e]);
                    }
            }
            if (!pdiag) {
                const int it = J * PT + r, jt = I * PT + c0;
                out.put4(h + it, jt, add4(add4(ld4sT(sU, r, c0), ld4s(sT, r, c0), p), cur[6], p));
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 7; ++q) cur[q] = nxt[q];
    }
}

// Root post-addition overlapped with the product kernel (driver.cu, Plan::rounds).  Launched as
// the product kernel's programmatic dependent, so it starts while the products run, on the SMs
// they leave free.  Blocks take tile pairs in round order from a shared counter and, before a
// pair of round r, wait until every product tile of rounds <= r has been stored
// (round_done[r] >= target[r], counted by the product kernel's epilogue warps).  No
// griddepcontrol.wait: the products are still running.  A wait that never ends (a broken
// count) traps after ~4 s instead of hanging the device.
__global__ void __launch_bounds__(256, FSYRK_POST_MINB) post_rounds_kernel(const __grid_constant__ PostArgs args,
                                                                          const int* round_done,
                                                                          const int* target, int* next_pair) {
    __shared__ uint32_t sU[TS][TS + 1];
    __shared__ uint32_t sT[TS][TS + 1];
    __shared__ int s_idx;
    const PostNode nd = post_node(args, args.ninl ? args.inl[0] : args.nodes[0]);
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    int ready_round = -1;  // rounds <= ready_round are known complete
    for (;;) {
        if (tid == 0) s_idx = atomicAdd(next_pair, 1);
        __syncthreads();
        const int idx = s_idx;
        __syncthreads();
        if (idx >= args.npairs) break;
        const int2 pr = args.pairs[idx];
        const int r = pr.x >> 20, I = pr.x & ((1 << 20) - 1), J = pr.y;
        if (r > ready_round) {
            if (tid == 0) {
                const long long t0 = clock64();
                for (int q = ready_round + 1; q <= r; ++q) {
                    int v;
                    for (;;) {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(round_done + q) : "memory");
                        if (v >= target[q]) break;
                        __nanosleep(500);
                        if (clock64() - t0 > (8ll << 30)) __trap();
                    }
                }
            }
            __syncthreads();
            ready_round = r;
        }
        post_vec_pair<false>(args, nd, I, J, sU, sT, nullptr);
        __syncthreads();  // sU / sT are reused by the next pair
    }
}

__global__ void add_lower_kernel(const AddNode* __restrict__ nodes, int n, uint32_t p) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    const AddNode nd = nodes[blockIdx.z];
    const int i = blockIdx.y;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= i && j < n; j += gridDim.x * blockDim.x)
        nd.x[(long long)i * nd.ldx + j] = addm(nd.x1[(long long)i * nd.ld1 + j], nd.x2[(long long)i * nd.ld2 + j], p);
}

__global__ void finalize_kernel(const uint32_t* __restrict__ x, long long ldx, int n, uint64_t* __restrict__ c,
                                long long ldc, ModP m, uint32_t alpha, uint32_t beta) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    const int i = blockIdx.y;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= i && j < n; j += gridDim.x * blockDim.x) {
        uint32_t v = x ? x[(long long)i * ldx + j] : 0;
        if (alpha != 1) v = mulm(v, alpha, m);
        if (beta != 0) {
            uint32_t ci = mod_u64(c[(long long)i * ldc + j], m);
            v = addm(v, beta == 1 ? ci : mulm(ci, beta, m), m.p);
        }
        c[(long long)i * ldc + j] = v;
    }
}

// C[j][i] <- C[i][j] for i > j, 32 x 32 tiles through shared memory.
__global__ void mirror_kernel(uint64_t* __restrict__ c, long long ldc, int n) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    __shared__ uint64_t s[TS][TS + 1];
    int I, J;
    tri_decode(blockIdx.x, I, J);
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < TS; r += 8) {
        const int i = I * TS + r, j = J * TS + tx;
        s[r][tx] = (i < n && j < n) ? c[(long long)i * ldc + j] : 0;
    }
    __syncthreads();
    for (int r = ty; r < TS; r += 8) {
        const int i = J * TS + r, j = I * TS + tx;  // upper-triangle target
        if (i < n && j < n && j > i) c[(long long)i * ldc + j] = s[tx][r];
    }
}

// strict upper triangle of row i, up to the end of i's row block of `rb` rows (rb = 0: whole row)
__global__ void zero_upper_kernel(uint64_t* __restrict__ c, long long ldc, int n, int rb) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    const int i = blockIdx.y;
    const int end = rb > 0 ? min(n, (i / rb + 1) * rb) : n;
    for (int j = i + 1 + blockIdx.x * blockDim.x + threadIdx.x; j < end; j += gridDim.x * blockDim.x)
        c[(long long)i * ldc + j] = 0;
}

__global__ void u32_to_u64_kernel(const uint32_t* __restrict__ x, long long ldx, int rows, int cols,
                                  uint64_t* __restrict__ out, long long ldo) {
    pdl_wait();  // the previous kernel of the call has finished writing (pdl.cuh)
    pdl_trigger();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;  // 2-D grid: no 64-bit division per element
    if (j >= cols) return;
    for (int i = blockIdx.y; i < rows; i += gridDim.y) out[(long long)i * ldo + j] = x[(long long)i * ldx + j];
}

// Multi-GPU shares (driver.cu, mgpu): the root post-addition of a partitioned plan writes, for
// each owned 32 x 32 tile pair (I >= J) of the h x h quadrants, tile (I, J) of C11, C21 and
// C22 and tile (J, I) of C21 (elementwise.cu post_vec_pair).  A share is those tiles packed as
// uint32 residues, 4 x 1024 words per pair (slot t: 0 C11(I,J), 1 C21(I,J), 2 C22(I,J),
// 3 C21(J,I)); entries outside Low(C) or beyond h are skipped (pack writes 0 there).
__device__ __forceinline__ bool share_entry(int t, int I, int J, int r, int cl, int h, long long& gi,
                                            long long& gj) {
    if (t == 3 && I == J) return false;
    const int bi = t == 3 ? J : I, bj = t == 3 ? I : J;
    const int li = bi * 32 + r, lj = bj * 32 + cl;
    if (li >= h || lj >= h) return false;
    if ((t == 0 || t == 2) && I == J && cl > r) return false;  // diagonal tiles of C11 / C22: lower only
    gi = li + (t == 0 ? 0 : h);
    gj = lj + (t == 2 ? h : 0);
    return true;
}

__global__ void share_pack_kernel(const uint64_t* __restrict__ c, long long ldc, int h, const int2* __restrict__ pairs,
                                  uint32_t* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const int2 pr = pairs[blockIdx.x];
    const int t = blockIdx.y;
    uint32_t* o = out + ((long long)blockIdx.x * 4 + t) * 1024;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        long long gi, gj;
        const bool ok = share_entry(t, pr.x, pr.y, r, threadIdx.x, h, gi, gj);
        o[r * 32 + threadIdx.x] = ok ? (uint32_t)c[gi * ldc + gj] : 0u;
    }
}

__global__ void share_unpack_kernel(const uint32_t* __restrict__ in, int h, const int2* __restrict__ pairs,
                                    uint64_t* __restrict__ c, long long ldc) {
    pdl_wait();
    pdl_trigger();
    const int2 pr = pairs[blockIdx.x];
    const int t = blockIdx.y;
    const uint32_t* src = in + ((long long)blockIdx.x * 4 + t) * 1024;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        long long gi, gj;
        if (share_entry(t, pr.x, pr.y, r, threadIdx.x, h, gi, gj)) c[gi * ldc + gj] = src[r * 32 + threadIdx.x];
    }
}

// F_{p^2} helpers (herk / syrk over the quadratic extension, see driver.cu run_fp2)
// (a, b) pairs -> X = a parts, Y = b parts, both n x k row-major
__global__ void deinterleave_kernel(const uint64_t* __restrict__ a, long long ldp, int n, int k,
                                    uint64_t* __restrict__ x, uint64_t* __restrict__ y) {
    pdl_wait();
    pdl_trigger();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    for (int i = blockIdx.y; i < n; i += gridDim.y) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(a + 2 * ((long long)i * ldp + j));
        x[(long long)i * k + j] = v.x;
        y[(long long)i * k + j] = v.y;
    }
}

// C = R + x * I as (a, b) pairs: R = Low(re part) (uint64, ld ldr), I from G = Y X^T (conj:
// I = G - G^T, herk) or G = X Y^T (I = G + G^T, syrk); upper triangle = conj / plain mirror of
// the lower one when `mirror`, zeros otherwise.
__global__ void fp2_combine_kernel(const uint64_t* __restrict__ r, long long ldr, const uint32_t* __restrict__ g,
                                   long long ldg, int n, uint32_t p, int conj, int mirror, uint64_t* __restrict__ c,
                                   long long ldcp) {
    pdl_wait();
    pdl_trigger();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    for (int i = blockIdx.y; i < n; i += gridDim.y) {
        const int lo = i >= j ? i : j, hi = i >= j ? j : i;  // (lo, hi) = the lower-triangle position
        const uint32_t g_lh = g[(long long)lo * ldg + hi], g_hl = g[(long long)hi * ldg + lo];
        uint32_t re = (uint32_t)r[(long long)lo * ldr + hi];
        uint32_t im = conj ? subm(g_lh, g_hl, p) : addm(g_lh, g_hl, p);
        if (i < j) {  // upper triangle
            if (!mirror) re = im = 0;
            else if (conj) im = im ? p - im : 0;  // conj(C[j][i])
        }
        *reinterpret_cast<ulonglong2*>(c + 2 * ((long long)i * ldcp + j)) = make_ulonglong2(re, im);
    }
}

// ------------------------------------------------------------- Winograd
// Pre-additions of one Strassen-Winograd level (winograd.hpp:118-169) on uint32 residue
// blocks x11, x12, x21, x22 (rows x cols, stride ld); out = 4 contiguous blocks (stride ldo,
// block stride bs).  side 0 (A): S1 = x21 + x22, S2 = S1 - x11, S3 = x11 - x21, S4 = x12 - S2.
// side 1 (stored blocks of B, x11 = B'11, x12 = B'12, x21 = B'21, x22 = B'22):
//   T1 = x12 - x11, T2 = x22 - T1, T3 = x22 - x12, T4 = T2 - x21.
__global__ void wino_pre_kernel(const uint32_t* __restrict__ x11, const uint32_t* __restrict__ x12,
                                const uint32_t* __restrict__ x21, const uint32_t* __restrict__ x22, long long ld,
                                int rows, int cols, uint32_t p, int side, uint32_t* __restrict__ out, long long ldo,
                                long long bs) {
    pdl_wait();
    pdl_trigger();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    for (int i = blockIdx.y; i < rows; i += gridDim.y) {
        const long long o = (long long)i * ld + j;
        const uint32_t a = x11[o], b = x12[o], c = x21[o], d = x22[o];
        uint32_t r0, r1, r2, r3;
        if (side == 0) {
            r0 = addm(c, d, p);
            r1 = subm(r0, a, p);
            r2 = subm(a, c, p);
            r3 = subm(b, r1, p);
        } else {
            r0 = subm(b, a, p);
            r1 = subm(d, r0, p);
            r2 = subm(d, b, p);
            r3 = subm(r1, c, p);
        }
        const long long q = (long long)i * ldo + j;
        out[q] = r0;
        out[bs + q] = r1;
        out[2 * bs + q] = r2;
        out[3 * bs + q] = r3;
    }
}

// Post-additions: M1..M7 (rows x cols each, block stride bs, row stride ldm) -> the four
// quadrants of C (stride ldc): C11 = M1 + M2, U2 = M1 + M6, U3 = U2 + M7, U4 = U2 + M5,
// C12 = U4 + M3, C21 = U3 - M4, C22 = U3 + M5.
__global__ void wino_post_kernel(const uint32_t* __restrict__ mm, long long bs, long long ldm, int rows, int cols,
                                 uint32_t p, uint32_t* __restrict__ c, long long ldc) {
    pdl_wait();
    pdl_trigger();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    for (int i = blockIdx.y; i < rows; i += gridDim.y) {
        const long long o = (long long)i * ldm + j;
        const uint32_t m1 = mm[o], m2 = mm[bs + o], m3 = mm[2 * bs + o], m4 = mm[3 * bs + o], m5 = mm[4 * bs + o],
                       m6 = mm[5 * bs + o], m7 = mm[6 * bs + o];
        const uint32_t u2 = addm(m1, m6, p), u3 = addm(u2, m7, p), u4 = addm(u2, m5, p);
        uint32_t* r0 = c + (long long)i * ldc + j;
        uint32_t* r1 = c + (long long)(i + rows) * ldc + j;
        r0[0] = addm(m1, m2, p);
        r0[cols] = addm(u4, m3, p);
        r1[0] = subm(u3, m4, p);
        r1[cols] = addm(u3, m5, p);
    }
}

// rows covered by grid.y (each block loops over rows with stride gridDim.y): about 8 waves of 148 SMs
int rows_grid(int rows, int gx) {
    int gy = (148 * 32 + gx - 1) / gx;
    if (gy > rows) gy = rows;
    if (gy > 65535) gy = 65535;
    return gy < 1 ? 1 : gy;
}

int grid_for(long long total, int threads) {
    long long b = (total + threads - 1) / threads;
    if (b > 148 * 32) b = 148 * 32;
    return (int)(b < 1 ? 1 : b);
}

template <int L>
cudaError_t prep_dispatch(const PrepArgs& a, cudaStream_t s) {
    const bool vec = a.aligned && !(a.kh % 4) && !(a.half % 4) && a.kw == a.kh && !(a.g_row % 4) && !(a.c_row % 4) &&
                     !(a.c3_row % 4) &&
                     (a.in64 ? !(a.ld64 % 2) && !(reinterpret_cast<uintptr_t>(a.a64) % 16) : true);
    if (vec) {
        const int ncg = (a.pair ? a.half : a.kh) / 4;
        dim3 block(32, 8);
        dim3 grid((ncg + 31) / 32, (a.h + 7) / 8, a.nnodes);
        if (a.pair) return launch_pdl(prep_vec_kernel<L, true>, grid, block, 0, s, a);
        return launch_pdl(prep_vec_kernel<L, false>, grid, block, 0, s, a);
    } else {
        const int ncw = a.pair ? a.half : a.kw;
        dim3 block(32, 8);
        dim3 grid((ncw + 31) / 32, (a.h + 7) / 8, a.nnodes);
        return launch_pdl(prep_kernel<L>, grid, block, 0, s, a);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_convert_in(const uint64_t* a, long long lda, int n, int kin, int kout, const ColMap* map,
                              uint32_t p, uint32_t* out, long long ldo, cudaStream_t s) {
    if ((long long)n * kout == 0) return cudaSuccess;
    const dim3 grid((kout + 255) / 256, rows_grid((n + FSYRK_CONVERT_ROWS - 1) / FSYRK_CONVERT_ROWS, (kout + 255) / 256));
    return launch_pdl(convert_in_kernel, grid, dim3(256), 0, s, a, lda, n, kin, kout, map, make_modp(p), out, ldo);
}

cudaError_t launch_split_planes(int L, const InView& in, const uint64_t* a64, long long ld64, int rows, int k,
                                uint32_t p, int8_t* planes, long long plane_stride, long long row_stride,
                                cudaStream_t s) {
    if ((long long)rows * k == 0) return cudaSuccess;
    const bool in64 = in.in64 != 0;
    const bool vec = !(k % 4) && !(row_stride % 4) &&
                     (in64 ? !(ld64 % 2) && !(in.c0 % 2) && !(reinterpret_cast<uintptr_t>(a64) % 16)
                           : !(in.ld32 % 4) && !(reinterpret_cast<uintptr_t>(in.p32) % 16));
    const ModP m = make_modp(p);
    const int gx = ((vec ? k / 4 : k) + 255) / 256;
    const dim3 g(gx, rows_grid(rows, gx));
#define FSYRK_SPLIT(LL)                                                                                              \
    if (vec) split_planes_kernel<LL, true><<<g, 256, 0, s>>>(in, a64, ld64, rows, k, m, planes, plane_stride,       \
                                                              row_stride);                                         \
    else split_planes_kernel<LL, false><<<g, 256, 0, s>>>(in, a64, ld64, rows, k, m, planes, plane_stride,          \
                                                           row_stride);
    switch (L) {  // L: digit scheme id (schemes.cuh)
        case SCHEME_LIMB2: FSYRK_SPLIT(SCHEME_LIMB2) break;
        case SCHEME_LIMB3: FSYRK_SPLIT(SCHEME_LIMB3) break;
        case SCHEME_LIMB4: FSYRK_SPLIT(SCHEME_LIMB4) break;
        case SCHEME_M17: FSYRK_SPLIT(SCHEME_M17) break;
        case SCHEME_M17N: FSYRK_SPLIT(SCHEME_M17N) break;
        case SCHEME_M31: FSYRK_SPLIT(SCHEME_M31) break;
        default: return cudaErrorInvalidValue;
    }
#undef FSYRK_SPLIT
    return cudaGetLastError();
}

cudaError_t launch_prep(const PrepArgs& args, cudaStream_t s) {
    if (args.h == 0 || args.nnodes == 0 || args.kw == 0) return cudaSuccess;
    switch (args.L) {  // digit scheme id
        case SCHEME_LIMB2: return prep_dispatch<SCHEME_LIMB2>(args, s);
        case SCHEME_LIMB3: return prep_dispatch<SCHEME_LIMB3>(args, s);
        case SCHEME_LIMB4: return prep_dispatch<SCHEME_LIMB4>(args, s);
        case SCHEME_M17: return prep_dispatch<SCHEME_M17>(args, s);
        case SCHEME_M17N: return prep_dispatch<SCHEME_M17N>(args, s);
        case SCHEME_M31: return prep_dispatch<SCHEME_M31>(args, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_prep_tree(const PrepTreeArgs& a, int nsm, cudaStream_t s) {
    if (a.rows == 0 || a.w == 0) return cudaSuccess;
    switch (a.L) {
        case SCHEME_LIMB2: return prep_tree_dispatch<SCHEME_LIMB2>(a, nsm, s);
        case SCHEME_LIMB3: return prep_tree_dispatch<SCHEME_LIMB3>(a, nsm, s);
        case SCHEME_LIMB4: return prep_tree_dispatch<SCHEME_LIMB4>(a, nsm, s);
        case SCHEME_M17: return prep_tree_dispatch<SCHEME_M17>(a, nsm, s);
        case SCHEME_M17N: return prep_tree_dispatch<SCHEME_M17N>(a, nsm, s);
        case SCHEME_M31: return prep_tree_dispatch<SCHEME_M31>(a, nsm, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_post(const PostArgs& args, cudaStream_t s) {
    if (args.h == 0 || args.nnodes == 0) return cudaSuccess;
    const int T = (args.h + TS - 1) / TS;
    dim3 grid(args.pairs ? args.npairs : T * (T + 1) / 2, 1, args.nnodes);
    if (grid.x == 0) return cudaSuccess;
    // vector loads need h % 4 == 0 (every ld in the plan is h or a multiple of 4 then)
    if (args.h % 4 == 0)
        return args.ninl == args.nnodes ? launch_pdl(post_vec_kernel<true>, grid, dim3(8, 32), 0, s, args)
                                        : launch_pdl(post_vec_kernel<false>, grid, dim3(8, 32), 0, s, args);
    return launch_pdl(post_kernel, grid, dim3(32, 8), 0, s, args);
}

cudaError_t launch_post2(const Post2Args& a, cudaStream_t s) {
    if (a.h2 == 0 || a.par.nnodes == 0) return cudaSuccess;
    if (a.h2 % PT != 0 || a.par.h != 2 * a.h2) return cudaErrorInvalidValue;
    const int T = a.h2 / PT;
    const size_t smem = (size_t)14 * kPostTile * 4;  // 12 child output tiles + 2 step temporaries
    DeviceOnce& once = per_device<Post2AttrOnce>();
    std::call_once(once.flag, [&] {
        once.result = cudaFuncSetAttribute(post2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (once.result == cudaSuccess)
            once.result =
                cudaFuncSetAttribute(post2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (once.result != cudaSuccess) return once.result;
    const dim3 grid(T * (T + 1) / 2, 1, a.par.nnodes), block(PT / 4, PT);
    const bool inl = a.par.ninl == a.par.nnodes && a.nchi == 3 * a.par.nnodes;
    return inl ? launch_pdl(post2_kernel<true>, grid, block, smem, s, a)
               : launch_pdl(post2_kernel<false>, grid, block, smem, s, a);
}

cudaError_t launch_post_rounds(const PostArgs& args, const int* round_done, const int* target, int* next_pair,
                               int blocks, cudaStream_t s) {
    if (args.h == 0 || args.npairs == 0) return cudaSuccess;
    if (args.h % 4 != 0) return cudaErrorInvalidValue;
    return launch_pdl(post_rounds_kernel, dim3(blocks), dim3(8, 32), 0, s, args, round_done, target, next_pair);
}

cudaError_t launch_add_lower(const AddNode* nodes, int nnodes, int n, uint32_t p, cudaStream_t s) {
    if (n == 0 || nnodes == 0) return cudaSuccess;
    dim3 grid((n + 255) / 256, n, nnodes);
    return launch_pdl(add_lower_kernel, grid, dim3(256), 0, s, nodes, n, p);
}

cudaError_t launch_finalize(const uint32_t* x, long long ldx, int n, uint64_t* c, long long ldc, const ModP& m,
                            uint32_t alpha, uint32_t beta, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    dim3 grid((n + 255) / 256, n);
    return launch_pdl(finalize_kernel, grid, dim3(256), 0, s, x, ldx, n, c, ldc, m, alpha, beta);
}

cudaError_t launch_mirror(uint64_t* c, long long ldc, int n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int T = (n + TS - 1) / TS;
    return launch_pdl(mirror_kernel, dim3(T * (T + 1) / 2), dim3(32, 8), 0, s, c, ldc, n);
}

cudaError_t launch_zero_upper(uint64_t* c, long long ldc, int n, int rb, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int w = rb > 0 ? (rb < n ? rb : n) : n;
    return launch_pdl(zero_upper_kernel, dim3((w + 255) / 256, n), dim3(256), 0, s, c, ldc, n, rb);
}

cudaError_t launch_u32_to_u64(const uint32_t* x, long long ldx, int rows, int cols, uint64_t* out, long long ldo,
                              cudaStream_t s) {
    if ((long long)rows * cols == 0) return cudaSuccess;
    const int gx = (cols + 255) / 256;
    return launch_pdl(u32_to_u64_kernel, dim3(gx, rows_grid(rows, gx)), dim3(256), 0, s, x, ldx, rows, cols, out, ldo);
}

cudaError_t launch_share_pack(const uint64_t* c, long long ldc, int h, const int2* pairs, int npairs, uint32_t* out,
                              cudaStream_t s) {
    if (npairs == 0) return cudaSuccess;
    return launch_pdl(share_pack_kernel, dim3(npairs, 4), dim3(32, 8), 0, s, c, ldc, h, pairs, out);
}

cudaError_t launch_share_unpack(const uint32_t* in, int h, const int2* pairs, int npairs, uint64_t* c, long long ldc,
                                cudaStream_t s) {
    if (npairs == 0) return cudaSuccess;
    return launch_pdl(share_unpack_kernel, dim3(npairs, 4), dim3(32, 8), 0, s, in, h, pairs, c, ldc);
}

cudaError_t launch_wino_pre(const uint32_t* x11, const uint32_t* x12, const uint32_t* x21, const uint32_t* x22,
                            long long ld, int rows, int cols, uint32_t p, int side, uint32_t* out, long long ldo,
                            long long bs, cudaStream_t s) {
    if ((long long)rows * cols == 0) return cudaSuccess;
    const int gx = (cols + 255) / 256;
    return launch_pdl(wino_pre_kernel, dim3(gx, rows_grid(rows, gx)), dim3(256), 0, s, x11, x12, x21, x22, ld, rows,
                      cols, p, side, out, ldo, bs);
}

cudaError_t launch_wino_post(const uint32_t* m, long long bs, long long ldm, int rows, int cols, uint32_t p,
                             uint32_t* c, long long ldc, cudaStream_t s) {
    if ((long long)rows * cols == 0) return cudaSuccess;
    const int gx = (cols + 255) / 256;
    return launch_pdl(wino_post_kernel, dim3(gx, rows_grid(rows, gx)), dim3(256), 0, s, m, bs, ldm, rows, cols, p, c,
                      ldc);
}

cudaError_t launch_deinterleave(const uint64_t* a, long long ldp, int n, int k, uint64_t* x, uint64_t* y,
                                cudaStream_t s) {
    if ((long long)n * k == 0) return cudaSuccess;
    const int gx = (k + 255) / 256;
    return launch_pdl(deinterleave_kernel, dim3(gx, rows_grid(n, gx)), dim3(256), 0, s, a, ldp, n, k, x, y);
}

cudaError_t launch_fp2_combine(const uint64_t* r, long long ldr, const uint32_t* g, long long ldg, int n, uint32_t p,
                               int conj, int mirror, uint64_t* c, long long ldcp, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int gx = (n + 255) / 256;
    return launch_pdl(fp2_combine_kernel, dim3(gx, rows_grid(n, gx)), dim3(256), 0, s, r, ldr, g, ldg, n, p, conj,
                      mirror, c, ldcp);
}

}  // namespace fsyrk_b200
