// Exact mod-p products on the 5th-generation tensor cores.
//
// Replaces the reference's classical leaves -- syrk_classical and
// gemm_classical_nt with their unsigned __int128 dot products
// (include/fsyrk/matrix.hpp:144-160, 317-407) -- and, for the two general
// products of every recursion level, the Strassen-Winograd engine
// gemm_winograd_nt_into (include/fsyrk/winograd.hpp:195-202).
//
// Representation: every residue is split into L balanced int8 limbs
// (modp.cuh), stored as L planes [L][rows][K] per operand.  For an output
// tile the kernel accumulates the 2L-1 "shift" sums
//      T_s = sum_{i+j=s} A_i * B_j^T          (int32, exact)
// in TMEM with tcgen05.mma.kind::i8, reusing each staged limb tile for L
// products, and the epilogue folds them:  C = sum_s 256^s T_s  mod p.
// |T_s| <= L * K * 2^14 < 2^31 bounds K (checked on the host).
//
// Pipeline (one CTA = one 128 x BN output tile, 128 threads):
//   warp 0 lane 0 : TMA producer, STAGES-deep ring of {L A-limb, L B-limb} tiles
//   warp 1 lane 0 : tcgen05.mma issuer (L*L*BK/32 MMAs per stage)
//   warps 0..3    : epilogue, TMEM -> registers -> fold -> uint32 residues
// Batched over a uniform problem set (blockIdx.y); SYRK mode computes only
// the tiles that meet the lower triangle (host-side tile list).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "modp.cuh"
#include "sm100.cuh"
#include "tc_modmm.h"

namespace fsyrk_b200 {

namespace {

constexpr int BM = 128;
constexpr int BK = 128;  // int8 elements of K per stage = one 128-byte swizzle row

template <int L, int BN, int STAGES>
struct Cfg {
    static constexpr int NACC = 2 * L - 1;
    static constexpr int COLS_USED = NACC * BN;
    static constexpr int TMEM_COLS = COLS_USED <= 32 ? 32 : COLS_USED <= 64 ? 64 : COLS_USED <= 128 ? 128
                                     : COLS_USED <= 256 ? 256 : 512;
    static_assert(COLS_USED <= 512, "accumulators exceed TMEM");
    static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "invalid UMMA N for M=128");
    static constexpr int A_TILE = BM * BK;
    static constexpr int B_TILE = BN * BK;
    static_assert(B_TILE % 1024 == 0, "B tile must be a whole number of swizzle atoms");
    static constexpr int STAGE_BYTES = L * (A_TILE + B_TILE);
    static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;
};

template <int L>
__device__ __forceinline__ uint32_t fold(const int32_t (&t)[2 * L - 1], const ModP& m, uint32_t c32) {
    if constexpr (L <= 3) {
        int64_t v = 0;
#pragma unroll
        for (int s = 2 * L - 2; s >= 0; --s) v = (v << 8) + t[s];
        return mod_s64(v, m);
    } else {
        int64_t lo = 0, hi = 0;
#pragma unroll
        for (int s = 3; s >= 0; --s) lo = (lo << 8) + t[s];
#pragma unroll
        for (int s = 2 * L - 2; s >= 4; --s) hi = (hi << 8) + t[s];
        uint32_t rl = mod_s64(lo, m), rh = mod_s64(hi, m);
        return addm(rl, mulm(rh, c32, m), m.p);
    }
}

template <int L, int BN, int STAGES>
__global__ void __launch_bounds__(128, 1)
    modmm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const ModmmArgs args) {
    using C = Cfg<L, BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int batch = blockIdx.y;
    int tm, tn;
    if (args.tile_list) {
        int2 t = args.tile_list[blockIdx.x];
        tm = t.x;
        tn = t.y;
    } else {
        tm = blockIdx.x / args.tiles_n;
        tn = blockIdx.x % args.tiles_n;
    }

    if (warp == 0) {
        sm100::tmem_alloc(tmem_slot, C::TMEM_COLS);
    } else if (warp == 1 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], 1);
        }
        sm100::mbar_init(done, 1);
        sm100::fence_mbar_init();
    } else if (warp == 2 && lane == 0) {
        sm100::tma_prefetch(&tmA);
        sm100::tma_prefetch(&tmB);
    }
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int kblocks = args.k_blocks;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            const int bA = batch * args.a_batch_mult + args.a_batch_off;
            const int bB = batch * args.b_batch_mult + args.b_batch_off;
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                sm100::mbar_wait(&empty[s], ph ^ 1);
                sm100::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
                uint8_t* st = smem + s * C::STAGE_BYTES;
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    sm100::tma_load_4d(st + l * C::A_TILE, &tmA, &full[s], kb * BK, tm * BM, l, bA);
                    sm100::tma_load_4d(st + L * C::A_TILE + l * C::B_TILE, &tmB, &full[s], kb * BK, tn * BN, l, bB);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            constexpr uint32_t idesc = sm100::idesc_i8(BM, BN);
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                sm100::mbar_wait(&full[s], ph);
                sm100::tc_fence_after();
                const uint32_t st = sm100::smem_u32(smem + s * C::STAGE_BYTES);
#pragma unroll
                for (int i = 0; i < L; ++i) {
#pragma unroll
                    for (int j = 0; j < L; ++j) {
                        const int acc = i + j;
                        const int first_i = acc - (L - 1) > 0 ? acc - (L - 1) : 0;
                        const uint64_t ad = sm100::sdesc_sw128(st + i * C::A_TILE);
                        const uint64_t bd = sm100::sdesc_sw128(st + L * C::A_TILE + j * C::B_TILE);
#pragma unroll
                        for (int kk = 0; kk < BK / 32; ++kk) {
                            const uint32_t accum = (kb > 0 || kk > 0 || i != first_i) ? 1u : 0u;
                            // +32 bytes along K inside the swizzle row = +2 in the 16-byte address field
                            sm100::mma_i8(tmem + acc * BN, ad + 2 * kk, bd + 2 * kk, idesc, accum);
                        }
                    }
                }
                sm100::tc_commit(&empty[s]);
            }
            sm100::tc_commit(done);
        }
        __syncwarp();
    }

    // ---------------- epilogue: all four warps, warp w owns TMEM lanes 32w..32w+31
    sm100::mbar_wait(done, 0);
    sm100::tc_fence_after();
    const ModP m = args.modp;
    const int row = warp * 32 + lane;
    const long long grow = (long long)tm * BM + row;
    const bool row_ok = grow < args.M;
    uint32_t* out = args.out + (long long)batch * args.out_batch_stride + grow * args.ldo;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t raw[C::NACC][16];
#pragma unroll
        for (int s = 0; s < C::NACC; ++s) sm100::tmem_ld16(lane_base + s * BN + c0, raw[s]);
        sm100::tmem_wait_ld();
        const long long gc0 = (long long)tn * BN + c0;
        if (!row_ok || gc0 >= args.N) continue;
        uint32_t res[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            int32_t t[C::NACC];
#pragma unroll
            for (int s = 0; s < C::NACC; ++s) t[s] = (int32_t)raw[s][c];
            res[c] = fold<L>(t, m, args.c32);
        }
        const bool full_chunk = gc0 + 16 <= args.N && (!args.syrk || gc0 + 15 <= grow) && args.vec_ok;
        if (full_chunk) {
            uint4* o = reinterpret_cast<uint4*>(out + gc0);
#pragma unroll
            for (int q = 0; q < 4; ++q) o[q] = make_uint4(res[4 * q], res[4 * q + 1], res[4 * q + 2], res[4 * q + 3]);
        } else {
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const long long gc = gc0 + c;
                if (gc < args.N && (!args.syrk || gc <= grow)) out[gc] = res[c];
            }
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) sm100::tmem_dealloc(tmem, C::TMEM_COLS);
}

template <int L, int BN, int STAGES>
cudaError_t launch_cfg(const CUtensorMap& ta, const CUtensorMap& tb, const ModmmArgs& args, int ntiles, int batch,
                       cudaStream_t stream) {
    using C = Cfg<L, BN, STAGES>;
    auto kern = modmm_kernel<L, BN, STAGES>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    dim3 grid(ntiles, batch);
    kern<<<grid, 128, C::SMEM_BYTES, stream>>>(ta, tb, args);
    return cudaGetLastError();
}

}  // namespace

int modmm_block_n(int L) { return L == 2 ? 128 : L == 3 ? 96 : 64; }

size_t modmm_k_limit(int L) {
    // |T_s| <= L * K * 128 * 128 must stay below 2^31
    return (size_t)((1ull << 31) - 1) / ((size_t)L * 16384ull);
}

cudaError_t modmm_launch(int L, const CUtensorMap& ta, const CUtensorMap& tb, const ModmmArgs& args, int ntiles,
                         int batch, cudaStream_t stream) {
    switch (L) {
        case 2: return launch_cfg<2, 128, 3>(ta, tb, args, ntiles, batch, stream);
        case 3: return launch_cfg<3, 96, 2>(ta, tb, args, ntiles, batch, stream);
        case 4: return launch_cfg<4, 64, 2>(ta, tb, args, ntiles, batch, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fsyrk_b200
