// Exact mod-p products on the 5th-generation tensor cores.
//
// Replaces the reference's classical leaves -- syrk_classical and
// gemm_classical_nt with their unsigned __int128 dot products
// (include/fsyrk/matrix.hpp:144-160, 317-407) -- and, for the two general
// products of every recursion level, the Strassen-Winograd engine
// gemm_winograd_nt_into (include/fsyrk/winograd.hpp:195-202).
//
// Every residue is stored as P int8 digit planes (schemes.cuh); an output tile
// accumulates the scheme's NT int8 x int8 -> int32 products in TMEM with
// tcgen05.mma.kind::i8 and the epilogue folds its NACC accumulators mod p.
// Scheme choice (scheme_for):
//   p = 2^17 - 1 : M17  (9 MMAs, 3 accumulators, 128 x 160 tiles)
//   p = 2^31 - 1 : M31  (default ACC4: 17 MMAs -- d2 e2 issued twice -- into
//                        4 accumulators, 128 x 128 tiles; without ACC4:
//                        16 MMAs, 5 accumulators, 128 x 96)
//   p <= 2^16    : LIMB2 (wide-B: 2 MMAs of N = 256 into 4 accumulators, 128 x 128)
//   p <= 2^24    : LIMB3 (wide-B over overlapped accumulators: 3 MMAs of N = 240 into
//                        5 accumulators, 128 x 80)
//   otherwise    : LIMB4 (wide-B over overlapped accumulators: 4 MMAs of N = 256 into
//                        7 accumulators, 128 x 64)
// Above modmm_k_limit the kernel drains its int32 accumulators mod p every
// K chunk, so any inner dimension is exact.
// The tile N is as large as TMEM allows for the accumulators: the
// microbenchmark in profiles/ubench shows the int8 MMA rate falls with N
// (shared-memory operand bandwidth), so the accumulators are not double
// buffered; the persistent kernel prefetches the next tile while the epilogue
// drains instead.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "modp.cuh"
#include "schemes.cuh"
#include "sm100.cuh"
#include "tc_modmm.h"
#include "tc_modmm_kernel.cuh"

#ifndef FSYRK_M17N_RANKS
#define FSYRK_M17N_RANKS 0
#endif

namespace fsyrk_b200 {

using namespace tc;

namespace {

template <int S>
SchemeInfo info() {
    using Sc = Scheme<S>;
    // M31 with 4 accumulators issues d2 e2 twice (weight 2): 17 MMAs for 16 digit products
    // MMAs per 32-deep K step counted in BN-wide units (a wide-B MMA covers NB of them)
    const int nt = Sc::NT * Sc::NB;
    const int products = (S == SCHEME_M31 && Sc::NT == 17) ? 16 : nt;
    return SchemeInfo{S,      planes_of<S>(), Sc::PA,   Sc::PB,         Sc::NACC,       nt,
                      products, Sc::BN,       Sc::BK,   Cfg<S>::TILE_M, Cfg<S>::B_ROWS, Sc::UNSIGNED};
}

uint64_t powmod(uint64_t b, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    b %= p;
    while (e) {
        if (e & 1) r = (r * b) % p;
        b = (b * b) % p;
        e >>= 1;
    }
    return r;
}

}  // namespace

SchemeInfo scheme_for(uint64_t p, int nranks) {
    // FSYRK_M17N_RANKS (0 = never): partitioned plans over at least this many ranks use 128-column
    // M17 tiles so the partition blocks are 128 instead of 640 rows (measured: finer blocks
    // balance better but every rank then touches most blocks' pre-additions; off by default)
    if (p == 131071ull)
        return FSYRK_M17N_RANKS > 0 && nranks >= FSYRK_M17N_RANKS ? info<SCHEME_M17N>() : info<SCHEME_M17>();
    if (p == 2147483647ull) return info<SCHEME_M31>();
    if (p <= 65536ull) return info<SCHEME_LIMB2>();
    if (p <= 16777216ull) return info<SCHEME_LIMB3>();
    return info<SCHEME_LIMB4>();
}

size_t modmm_k_limit(const SchemeInfo& s, uint64_t p) {
    const uint64_t i32 = (1ull << 31) - 1;
    switch (s.id) {
        case SCHEME_M17:  // <= 3 terms of (2 d) e <= 126 * 63 per accumulator
        case SCHEME_M17N:
            return (size_t)(i32 / (3ull * 126 * 63));
        case SCHEME_M31:
            if (Scheme<SCHEME_M31>::ACC4)  // accumulator 0: 5 terms of <= 255 * 255, read as uint32
                return (size_t)(0xFFFFFFFFull / (5ull * 255 * 255));
            return (size_t)(i32 / (4ull * 255 * 254));  // <= 4 terms of <= 255 * 254 per accumulator
        default: {
            const int L = s.planes;
            const uint64_t k32 = i32 / ((uint64_t)L * 16384ull);  // |T_s| <= L K 2^14
            // int64 fold with balanced weights: L^2 K 2^14 (p / 2) <= 2^62
            const uint64_t k64 = (1ull << 62) / ((uint64_t)L * L * 16384ull * (p / 2 + 1));
            return (size_t)(k32 < k64 ? k32 : k64);
        }
    }
}

void modmm_set_k(GroupDesc& g, const SchemeInfo& s, uint64_t p, long long kpad) {
    g.k_blocks = (int)(kpad / s.bk);
    const long long cb = (long long)(modmm_k_limit(s, p) / (size_t)s.bk);
    g.chunk_blocks = (int)(cb < 1 ? 1 : cb < g.k_blocks ? cb : g.k_blocks > 0 ? g.k_blocks : 1);
}

void fill_fold_weights(const SchemeInfo& s, uint64_t p, int32_t* w) {
    for (int i = 0; i < 8; ++i) w[i] = 0;
    if (s.id == SCHEME_M17 || s.id == SCHEME_M17N || s.id == SCHEME_M31) return;  // constants inside fold_acc
    for (int i = 0; i < 8; ++i) {
        // accumulator i carries digit shift i, except in the wide-B LIMB2 layout T00|T01|T10|T11
        const int sh = s.id == SCHEME_LIMB2 ? Scheme<SCHEME_LIMB2>::shift(i) : i;
        uint64_t v = powmod(256, (uint64_t)sh, p);
        w[i] = v > p / 2 ? (int32_t)((int64_t)v - (int64_t)p) : (int32_t)v;
    }
}

cudaError_t modmm_launch(const SchemeInfo& s, const GroupedArgs& args, int grid, cudaStream_t stream) {
    switch (s.id) {
        case SCHEME_LIMB2: return launch_cfg<SCHEME_LIMB2>(args, grid, stream);
        case SCHEME_LIMB3: return launch_cfg<SCHEME_LIMB3>(args, grid, stream);
        case SCHEME_LIMB4: return launch_cfg<SCHEME_LIMB4>(args, grid, stream);
        case SCHEME_M17: return launch_cfg<SCHEME_M17>(args, grid, stream);
        case SCHEME_M17N: return launch_cfg<SCHEME_M17N>(args, grid, stream);
        case SCHEME_M31: return launch_cfg<SCHEME_M31>(args, grid, stream);
        default: return cudaErrorInvalidValue;
    }
}

#ifdef FSYRK_KTRACE
extern "C" int fsyrk_b200_debug_cta_span(unsigned long long* out, int n) {
    const int m = n < 1024 * 3 ? n : 1024 * 3;
    return (int)cudaMemcpyFromSymbol(out, g_cta_span, m * sizeof(unsigned long long));
}
extern "C" int fsyrk_b200_debug_ktrace(unsigned long long* out, int n) {
    const int m = n < kTraceTiles * 8 ? n : kTraceTiles * 8;
    return (int)cudaMemcpyFromSymbol(out, g_ktrace, m * sizeof(unsigned long long));
}
#endif

namespace {
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_tiled() {
    static const EncodeTiled fn = [] {  // thread-safe one-time lookup
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiled>(p);
        return EncodeTiled(nullptr);
    }();
    return fn;
}
}  // namespace

void modmm_set_output_map(GroupDesc& g, int batch) {
    g.tma_ok = 0;
    const long long bs = g.out_bs > 0 ? g.out_bs : (long long)g.M * g.ldo;
    if (g.ldo % 4 || bs % 4 || reinterpret_cast<uintptr_t>(g.out) % 16 || g.M <= 0 || g.N <= 0) return;
    EncodeTiled enc = encode_tiled();
    if (!enc) return;
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)(batch > 0 ? batch : 1)};
    cuuint64_t strides[2] = {(cuuint64_t)g.ldo * 4, (cuuint64_t)bs * 4};
    cuuint32_t box[3] = {16, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&g.tmO, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, g.out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        g.tma_ok = 1;
}

int modmm_epilogue_warps() { return kEpiWarpsDefault; }

int modmm_grid(const SchemeInfo& s, int nsm) {
    switch (s.id) {
        case SCHEME_LIMB2: return grid_for<SCHEME_LIMB2>(nsm);
        case SCHEME_LIMB3: return grid_for<SCHEME_LIMB3>(nsm);
        case SCHEME_LIMB4: return grid_for<SCHEME_LIMB4>(nsm);
        case SCHEME_M17: return grid_for<SCHEME_M17>(nsm);
        case SCHEME_M17N: return grid_for<SCHEME_M17N>(nsm);
        case SCHEME_M31: return grid_for<SCHEME_M31>(nsm);
        default: return nsm;
    }
}

}  // namespace fsyrk_b200
