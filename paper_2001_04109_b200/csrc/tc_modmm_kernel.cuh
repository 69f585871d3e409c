// tcgen05 int8 digit-plane mod-p product kernel (see tc_modmm.cu and schemes.cuh).
//
// Persistent and grouped: one launch runs every product of a recursion plan
// (the general products of all levels and the leaf SYRKs), described by up
// to kMaxGroups uniform problem groups and a host-built tile list in
// longest-K-first order.  Warp roles per CTA (one CTA per SM):
//   warp 0      : TMA producer (runs ahead across tiles)
//   warp 1      : tcgen05.mma issuer (the scheme's NT terms per 32-deep K step)
//   warps 2..   : epilogue; warp w drains TMEM lanes 32*(w%4).. for one part
//                 of the tile's columns and folds the accumulators mod p
// CTA-pair mode (Scheme::PAIR): the CTAs of a 2-CTA cluster share one 256 x BN
// output tile.  Each loads its 128 rows of A and half of B's BN rows into its
// own shared memory (completing bytes on the leader's barrier); the leader
// issues tcgen05.mma.cta_group::2 (M = 256), whose commits arrive in both CTAs;
// each CTA's epilogue drains its own TMEM rows and reports to the leader.  Per
// SM this halves the B operand bytes pulled from L2 per MAC.
// TMEM holds the NACC accumulators of one tile (<= 480 columns), twice when two
// sets fit (the next tile's MMAs then overlap this tile's epilogue); the producer
// prefetches the next tile's operands while the epilogue runs.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "modp.cuh"
#include "pdl.cuh"
#include "per_device.h"
#include "schemes.cuh"
#include "sm100.cuh"
#include "tc_modmm.h"

namespace fsyrk_b200 {
namespace tc {

#ifndef FSYRK_EPI_EXPERIMENT
#define FSYRK_EPI_EXPERIMENT 0
#endif
#ifndef FSYRK_TSTORE_ALL
#define FSYRK_TSTORE_ALL 0
#endif
#ifndef FSYRK_STG256
#define FSYRK_STG256 0  // 256-bit direct stores from the epilogue (experiment; with FSYRK_NO_TSTORE)
#endif
#ifndef FSYRK_LIMB2_TSTORE
#define FSYRK_LIMB2_TSTORE 0  // measured: products +3%, call within noise (profiles/r01/variants.txt)
#endif
#ifndef FSYRK_NO_TSTORE
#define FSYRK_NO_TSTORE 0
#endif
#ifndef FSYRK_STAGGER
#define FSYRK_STAGGER 1
#endif
#ifndef FSYRK_TMA_HINTS
#define FSYRK_TMA_HINTS 0  // L2 eviction hints on the operand loads of general products (experiment)
#endif
#ifndef FSYRK_EPI_WARPS
#define FSYRK_EPI_WARPS 8
#endif
constexpr int kEpiWarpsDefault = FSYRK_EPI_WARPS;
constexpr int BM = 128;  // accumulator rows per CTA (TMEM lanes)

#ifdef FSYRK_KTRACE
// timing experiment: per-tile clock64 stamps of CTA 0 (profiles/ktrace.py)
constexpr int kTraceTiles = 64;
__device__ unsigned long long g_ktrace[kTraceTiles][8];
#define KTRACE(it, slot)                                                                        \
    do {                                                                                        \
        if (blockIdx.x == 0 && (it) < kTraceTiles) g_ktrace[(it)][(slot)] = clock64();          \
    } while (0)
// per-CTA span (globaltimer ns): [0] past the prologue, [1] last epilogue warp done, [2] tiles
__device__ unsigned long long g_cta_span[1024][3];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#else
#define KTRACE(it, slot) \
    do {                 \
    } while (0)
#endif

// Scheme<S>::SPLITB if the scheme declares it
template <int S, class = void>
struct SplitB : std::false_type {};
template <int S>
struct SplitB<S, std::void_t<decltype(Scheme<S>::SPLITB)>> : std::bool_constant<Scheme<S>::SPLITB> {};
template <int S>
constexpr bool splitb_of() {
    return SplitB<S>::value;
}
// Scheme<S>::OVERLAP (wide-B MMAs over overlapped accumulators, schemes.cuh) if declared
template <int S, class = void>
struct Overlap : std::false_type {};
template <int S>
struct Overlap<S, std::void_t<decltype(Scheme<S>::OVERLAP)>> : std::bool_constant<Scheme<S>::OVERLAP> {};

template <int S>
struct Cfg {
    using Sc = Scheme<S>;
    static constexpr bool PAIR = Sc::PAIR;
    static constexpr int BN = Sc::BN, BK = Sc::BK, STAGES = Sc::STAGES, NACC = Sc::NACC;
    static constexpr int TILE_M = PAIR ? 2 * BM : BM;  // output rows per tile
    // CTA pairs split the B operand's rows: BN / 2 rows of every plane per CTA, or (wide-B: the
    // N = NB * BN operand is the planes side by side) all BN rows of one plane each
    static constexpr bool SPLITB = splitb_of<S>();
    static_assert(!SPLITB || (PAIR && Sc::NB == 2 && Sc::PB == 2), "plane split needs a pair and two B planes");
    static constexpr int B_ROWS = PAIR && !SPLITB ? BN / 2 : BN;  // B rows staged per CTA
    static constexpr int PB_STAGE = SPLITB ? 1 : Sc::PB;           // B planes staged per CTA
    static_assert(BK == 128 || BK == 64 || BK == 32, "BK must match a swizzle mode");
    static constexpr int COLS_USED = NACC * BN;
    // two accumulator sets when they fit: the MMAs of tile i+1 run while the epilogue drains tile i
    static constexpr int NBUF = 2 * COLS_USED <= 512 ? 2 : 1;
    static constexpr int COLS_ALL = NBUF * COLS_USED;
    static constexpr int TMEM_COLS = COLS_ALL <= 32 ? 32 : COLS_ALL <= 64 ? 64 : COLS_ALL <= 128 ? 128
                                     : COLS_ALL <= 256 ? 256 : 512;
    static_assert(COLS_USED <= 512, "accumulators exceed TMEM");
    static_assert(BN % (PAIR ? 32 : 16) == 0 && BN >= 16 && BN <= 256, "UMMA N (and 8-row groups per CTA half)");
    static constexpr int A_TILE = BM * BK;
    static constexpr int B_TILE = B_ROWS * BK;
    static_assert(B_TILE % 1024 == 0 && A_TILE % 1024 == 0, "tiles must be whole swizzle atoms");
    static constexpr int STAGE_BYTES = Sc::PA * A_TILE + PB_STAGE * B_TILE;
#ifdef FSYRK_M17_FAKE3  // timing experiment (wrong results, profiles/r02/operand_feed.txt): only the
    static constexpr int PA_LOAD = digits_of<S> == SCHEME_M17 ? 3 : Sc::PA;  // 3 digit planes of A are loaded
#else
    static constexpr int PA_LOAD = Sc::PA;
#endif
    static constexpr int LOAD_BYTES = PA_LOAD * A_TILE + PB_STAGE * B_TILE;
    static constexpr int BAR_BYTES = 384;  // mbarriers + TMEM slot + the tile-schedule ring
    static constexpr int EPI_WARPS = kEpiWarpsDefault;
    static constexpr int NCW = (BN / 16 + EPI_WARPS / 4 - 1) / (EPI_WARPS / 4);  // chunks per epilogue warp
    // TMA-store staging: one 32 x 16 u32 box (2 KB, 64-byte swizzle) per epilogue warp
    static constexpr int OUT_BYTES = EPI_WARPS * 2048;
    // shared memory: [STAGES operand stages][output staging][barriers]; the dynamic window is
    // 1024-aligned (__align__ on the extern array, checked at entry)
    // TMA stores: measured faster for the Mersenne schemes (cfg2 products 185 -> 178 us, cfg5
    // 3.18 -> 2.89 ms), neutral to slightly slower for LIMB2 (cfg3 251 -> 254 us)
    // TMA stores: M17 / M31 measured faster; LIMB2 optional (FSYRK_LIMB2_TSTORE)
    static constexpr bool TSTORE = !FSYRK_NO_TSTORE &&
                                   (digits_of<S> == SCHEME_M17 || S == SCHEME_M31 || (S == SCHEME_LIMB2 && FSYRK_LIMB2_TSTORE) ||
                                    FSYRK_TSTORE_ALL) &&
                                   STAGES * STAGE_BYTES + OUT_BYTES + BAR_BYTES <= 232448;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + (TSTORE ? OUT_BYTES : 0) + BAR_BYTES;
    static constexpr int BUF_COLS = 2 * COLS_USED <= 512 ? COLS_USED : 0;  // column offset of buffer 1
    // Staggered accumulator release (single TMEM buffer, separable partial fold): the epilogue
    // drains the tile accumulator by accumulator, adding each one's share of the partial fold,
    // and frees it at once; the next tile's first MMAs into that accumulator wait only for it.
    // Measured (profiles/r01/variants.txt): M17 products -1% (cfg2) / -2% (cfg5); LIMB2 +4% (off).
    static constexpr bool STAGGER =
        FSYRK_STAGGER && NBUF == 1 && !PAIR && SplitFold<S>::ok && digits_of<S> == SCHEME_M17;
    static_assert(SMEM_BYTES <= 232448, "shared memory");
};

// compile-time loop: fn(std::integral_constant<int, i>) for i in [0, N)
template <int N, int I = 0, class Fn>
__device__ __forceinline__ void static_for(Fn&& fn) {
    if constexpr (I < N) {
        fn(std::integral_constant<int, I>{});
        static_for<N, I + 1>(fn);
    }
}

// index of the first term (in issue order) that writes accumulator `acc`
template <int S>
__host__ __device__ constexpr int first_term(int acc) {
    for (int t = 0; t < Scheme<S>::NT; ++t)
        if (Scheme<S>::term(t).acc == acc) return t;
    return -1;
}

// O64: the variant whose epilogue can write alpha X + beta C_in into the caller's uint64 C
// (GroupDesc::out64, root-leaf plans).  A separate instantiation: the uint64 path's registers
// made the regular LIMB2 epilogue spill (160 bytes of stack, cfg3 products 0.203 -> 0.242 ms).
template <int S, int EPI = kEpiWarpsDefault, bool O64 = false>
__global__ void __launch_bounds__(64 + 32 * EPI, 1)
    modmm_kernel(const __grid_constant__ GroupedArgs args) {
    using C = Cfg<S>;
    using Sc = Scheme<S>;
    constexpr bool PAIR = C::PAIR;
    constexpr int BN = C::BN, BK = C::BK, STAGES = C::STAGES;
    constexpr int kParts = EPI / 4;  // column slices per lane quadrant
    static_assert(EPI == C::EPI_WARPS, "staging is sized for the default epilogue width");
    static_assert(EPI % 4 == 0 && BN % 16 == 0, "epilogue works in 16-column chunks");
    constexpr int SW = BK == 128 ? 2 : BK == 64 ? 4 : 6;  // descriptor layout: SWIZZLE_128B / 64B / 32B
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if (threadIdx.x == 0 && (sm100::smem_u32(smem) & 1023u)) __trap();  // swizzled tiles need 1024-B alignment
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES + (C::TSTORE ? C::OUT_BYTES : 0));
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;        // [NBUF]
    uint64_t* tmem_empty = tmem_full + C::NBUF;  // [NBUF] (the leader's counts both CTAs' epilogues)
    uint64_t* acc_empty = tmem_empty + C::NBUF;  // [NACC] staggered release: accumulator s drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + C::NACC);
    // dynamic schedule: the producer publishes the tile it claimed in a ring of kSched slots; the
    // MMA thread and every epilogue warp read it there
    constexpr int kSched = 4;
    uint64_t* sched_full = acc_empty + C::NACC + 1;  // [kSched], one arrival (the producer)
    uint64_t* sched_empty = sched_full + kSched;     // [kSched], 1 + EPI arrivals (the readers)
    int* sched = reinterpret_cast<int*>(sched_empty + kSched);
    static_assert((2 * STAGES + 2 * C::NBUF + C::NACC + 1 + 2 * kSched) * 8 + kSched * 4 <= C::BAR_BYTES, "barrier area");
    const bool dyn = !PAIR && args.dyn != nullptr;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? sm100::cluster_rank() : 0;
    const int unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // tile-scheduling unit
    const int nunits = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;

    if (warp == 0) {
        if constexpr (PAIR)
            sm100::tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
        else
            sm100::tmem_alloc(tmem_slot, C::TMEM_COLS);
    } else if (warp == 1 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < C::NBUF; ++b) {
            sm100::mbar_init(&tmem_full[b], 1);
            sm100::mbar_init(&tmem_empty[b], (PAIR ? 2 : 1) * EPI);
        }
        for (int s = 0; s < C::NACC; ++s) sm100::mbar_init(&acc_empty[s], EPI);
        for (int s = 0; s < kSched; ++s) {
            sm100::mbar_init(&sched_full[s], 1);
            sm100::mbar_init(&sched_empty[s], 1 + EPI);
        }
        sm100::fence_mbar_init();
    } else if (warp == 2 && lane == 0) {
        for (int g = 0; g < args.ngroups; ++g) {
            sm100::tma_prefetch(&args.g[g].tmA);
            sm100::tma_prefetch(&args.g[g].tmB);
            if (C::TSTORE && args.g[g].tma_ok) sm100::tma_prefetch(&args.g[g].tmO);
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) sm100::cluster_sync();  // peer barriers initialised before any remote arrive
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();  // setup above overlaps the previous kernel's tail; operands are ready from here
#ifdef FSYRK_KTRACE
    if (threadIdx.x == 0) g_cta_span[blockIdx.x][0] = gtimer();
#endif
    // round-aware post kernel: may launch once every CTA is resident and past the wait (it only
    // spins on round_done, so it can never hold resources this grid or its producers need)
    if (args.round_done) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    // this unit's tiles: a contiguous range of the balanced list, or the strided default
    int t_beg = unit, t_end = args.ntiles, t_step = nunits;
    if (args.tile_off) {
        t_beg = args.tile_off[unit];
        t_end = args.tile_off[unit + 1];
        t_step = 1;
    }
    // reader side of the schedule: the n-th tile of this CTA, or -1 after the last one
    // (whole_warp: called by all 32 lanes, one arrival per warp; else by a single thread)
    auto next_tile = [&](int n, bool whole_warp) -> int {
        if (!dyn) {
            const int t = t_beg + n * t_step;
            return t < t_end ? t : -1;
        }
        const int slot = n & (kSched - 1);
        sm100::mbar_wait(&sched_full[slot], (uint32_t)(n / kSched) & 1u);
        const int t = sched[slot];
        if (whole_warp) __syncwarp();  // every lane has read the slot before it is handed back
        if (!whole_warp || lane == 0) sm100::mbar_arrive(&sched_empty[slot]);
        return t;
    };
    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer (both CTAs of a pair)
            int stage = 0;
            uint32_t phase = 0;
#if FSYRK_TMA_HINTS
            const uint64_t pol_a = sm100::l2_policy_evict_last(), pol_b = sm100::l2_policy_evict_first();
#endif
            int t = dyn ? unit : t_beg;
            for (int n = 0;; ++n) {
                if (dyn) {  // publish the claimed tile (or the end marker)
                    const int slot = n & (kSched - 1);
                    sm100::mbar_wait(&sched_empty[slot], ((uint32_t)(n / kSched) & 1u) ^ 1u);
                    sched[slot] = t < args.ntiles ? t : -1;
                    sm100::mbar_arrive(&sched_full[slot]);
                    if (t >= args.ntiles) break;
                } else if (t >= t_end) {
                    break;
                }
                // claim the next tile now: the atomic's round trip overlaps this tile's loads
                const int t_next = dyn ? atomicAdd(args.dyn, 1) + nunits : t + t_step;
                const int4 tile = args.tiles[t];
                t = t_next;
                const GroupDesc& g = args.g[tile.x & ((1 << kTileGroupBits) - 1)];
                const int bA = tile.y * g.a_mult + g.a_off, bB = tile.y * g.b_mult + g.b_off;
                const int arow = tile.z * C::TILE_M + (int)rank * BM;
                const int brow = tile.w * BN + (C::SPLITB ? 0 : (int)rank * C::B_ROWS);
                for (int kb = 0; kb < g.k_blocks; ++kb) {
                    sm100::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* st = smem + stage * C::STAGE_BYTES;
                    if constexpr (PAIR) {
                        if (rank == 0) sm100::mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
#pragma unroll
                        for (int l = 0; l < Sc::PA; ++l)
                            sm100::tma_load_4d_pair(st + l * C::A_TILE, &g.tmA, &full[stage], kb * BK, arow, l, bA);
                        if constexpr (C::SPLITB) {  // this CTA's B digit plane
                            sm100::tma_load_4d_pair(st + Sc::PA * C::A_TILE, &g.tmB, &full[stage], kb * BK, brow,
                                                    (int)rank, bB);
                        } else {
#pragma unroll
                            for (int l = 0; l < Sc::PB; ++l)
                                sm100::tma_load_4d_pair(st + Sc::PA * C::A_TILE + l * C::B_TILE, &g.tmB, &full[stage],
                                                        kb * BK, brow, l, bB);
                        }
                    } else {
                        sm100::mbar_arrive_expect_tx(&full[stage], C::LOAD_BYTES);
#if FSYRK_TMA_HINTS
                        // general products: the A row panels of a 12-row tile group are read again by
                        // the next wave (column by column inside the group), the B column panels stream
                        const bool hint = !g.syrk;
#pragma unroll
                        for (int l = 0; l < C::PA_LOAD; ++l) {
                            if (hint)
                                sm100::tma_load_4d_hint(st + l * C::A_TILE, &g.tmA, &full[stage], kb * BK, arow, l, bA, pol_a);
                            else
                                sm100::tma_load_4d(st + l * C::A_TILE, &g.tmA, &full[stage], kb * BK, arow, l, bA);
                        }
#pragma unroll
                        for (int l = 0; l < Sc::PB; ++l) {
                            if (hint && FSYRK_TMA_HINTS == 1)
                                sm100::tma_load_4d_hint(st + Sc::PA * C::A_TILE + l * C::B_TILE, &g.tmB, &full[stage],
                                                        kb * BK, brow, l, bB, pol_b);
                            else
                                sm100::tma_load_4d(st + Sc::PA * C::A_TILE + l * C::B_TILE, &g.tmB, &full[stage],
                                                   kb * BK, brow, l, bB);
                        }
#else
#pragma unroll
                        for (int l = 0; l < C::PA_LOAD; ++l)
                            sm100::tma_load_4d(st + l * C::A_TILE, &g.tmA, &full[stage], kb * BK, arow, l, bA);
#pragma unroll
                        for (int l = 0; l < Sc::PB; ++l)
                            sm100::tma_load_4d(st + Sc::PA * C::A_TILE + l * C::B_TILE, &g.tmB, &full[stage],
                                               kb * BK, brow, l, bB);
#endif
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // ------------------------------------------------ MMA issuer (the leader of a pair)
            // N = NB * BN: a wide-B scheme multiplies one A digit by NB adjacent B digit planes
            constexpr uint32_t idesc = sm100::idesc_i8(C::TILE_M, BN * Sc::NB, !Sc::UNSIGNED);
            static_assert(BN * Sc::NB <= 256 && (Sc::NB == 1 || !PAIR || C::SPLITB), "UMMA N");
            int stage = 0;
            uint32_t phase = 0;
            uint32_t it = 0;
            for (int n = 0;; ++n) {
              const int t = next_tile(n, false);
              if (t < 0) break;
              const GroupDesc& g = args.g[args.tiles[t].x & ((1 << kTileGroupBits) - 1)];
              // K chunks: the accumulators are drained every chunk_blocks K-blocks (exactness
              // bound of the int32 accumulators); one chunk is one use of the TMEM buffer
              for (int kc = 0; kc < g.k_blocks; kc += g.chunk_blocks, ++it) {
                const int kend = min(g.k_blocks, kc + g.chunk_blocks);
                const int buf = C::NBUF == 2 ? (int)(it & 1) : 0;
                const uint32_t use = C::NBUF == 2 ? it >> 1 : it;  // uses of this buffer so far
                KTRACE(it, 0);
                if constexpr (!C::STAGGER) {
                    sm100::mbar_wait(&tmem_empty[buf], (use & 1) ^ 1);  // epilogue(s) drained this buffer
                    sm100::tc_fence_after();
                }
                KTRACE(it, 1);
                const uint32_t acc_base = tmem + buf * C::BUF_COLS;
                // issue term q of the scheme for K-block kb of the chunk from the stage at shared address st
                auto issue = [&](auto qc, uint32_t st, int kb) {
                    constexpr int q = decltype(qc)::value;
                    constexpr Term tm = Sc::term(q);
                    constexpr bool first = first_term<S>(tm.acc) == q;
                    constexpr int ta = tm.a >= C::PA_LOAD ? tm.a - 2 : tm.a;  // (FAKE3: the undoubled plane)
                    const uint64_t ad = sm100::sdesc_kmajor(st + ta * C::A_TILE, SW, 8 * BK);
                    const uint64_t bd = sm100::sdesc_kmajor(st + Sc::PA * C::A_TILE + tm.b * C::B_TILE, SW, 8 * BK);
#pragma unroll
                    for (int kk = 0; kk < BK / 32; ++kk) {
                        const uint32_t accum = (kb > kc || kk > 0 || !first) ? 1u : 0u;
                        // +32 bytes along K inside the swizzle row = +2 in the 16-byte address field
                        if constexpr (PAIR)
                            sm100::mma_i8_pair(acc_base + tm.acc * BN, ad + 2 * kk, bd + 2 * kk, idesc, accum);
                        else
                            sm100::mma_i8(acc_base + tm.acc * BN, ad + 2 * kk, bd + 2 * kk, idesc, accum);
                    }
                };
                // Overlapped wide-B schemes, first K block of a chunk: the scheme's term0 list, whose
                // init terms overwrite their accumulators on the first 32-deep step
                auto issue0 = [&](auto qc, uint32_t st) {
                    if constexpr (Overlap<S>::value) {
                        constexpr WideTerm tm = Sc::term0(decltype(qc)::value);
                        constexpr uint32_t idn = sm100::idesc_i8(C::TILE_M, BN * tm.nb, !Sc::UNSIGNED);
                        const uint64_t ad = sm100::sdesc_kmajor(st + tm.a * C::A_TILE, SW, 8 * BK);
                        const uint64_t bd = sm100::sdesc_kmajor(st + Sc::PA * C::A_TILE + tm.b * C::B_TILE, SW, 8 * BK);
#pragma unroll
                        for (int kk = 0; kk < BK / 32; ++kk)
                            sm100::mma_i8(acc_base + tm.acc * BN, ad + 2 * kk, bd + 2 * kk, idn,
                                          (kk > 0 || !tm.init) ? 1u : 0u);
                    }
                };
                auto advance = [&](int& s, uint32_t& ph) {
                    if (++s == STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                };
                int kb0 = kc;
                if constexpr (C::STAGGER) {
                    // The epilogue frees the accumulators one by one (0 first).  The terms of every
                    // accumulator but the last start as soon as theirs is free, for as many K-blocks
                    // as there are stages; the last accumulator's terms of those K-blocks follow once
                    // it is free (per accumulator the sums run in the same K order, so the int32
                    // results are the same).  The tensor pipe thus works while the epilogue drains.
                    constexpr int LAST = C::NACC - 1;
                    const int L = kend - kc < STAGES ? kend - kc : STAGES;
                    int s1 = stage;
                    uint32_t ph1 = phase;
                    for (int kb = kc; kb < kc + L; ++kb) {
                        sm100::mbar_wait(&full[s1], ph1);
                        sm100::tc_fence_after();
                        const uint32_t st = sm100::smem_u32(smem + s1 * C::STAGE_BYTES);
                        static_for<Sc::NT>([&](auto qc) {
                            constexpr Term tm = Sc::term(decltype(qc)::value);
                            if constexpr (tm.acc != LAST) {
                                if (kb == kc && first_term<S>(tm.acc) == decltype(qc)::value) {
                                    sm100::mbar_wait(&acc_empty[tm.acc], (use & 1) ^ 1);
                                    sm100::tc_fence_after();
                                }
                                issue(qc, st, kb);
                            }
                        });
                        advance(s1, ph1);
                    }
                    sm100::mbar_wait(&acc_empty[LAST], (use & 1) ^ 1);
                    sm100::tc_fence_after();
                    for (int kb = kc; kb < kc + L; ++kb) {
                        const uint32_t st = sm100::smem_u32(smem + stage * C::STAGE_BYTES);
                        static_for<Sc::NT>([&](auto qc) {
                            if constexpr (Sc::term(decltype(qc)::value).acc == LAST) issue(qc, st, kb);
                        });
                        sm100::tc_commit(&empty[stage]);
                        advance(stage, phase);
                    }
                    kb0 = kc + L;
                }
                for (int kb = kb0; kb < kend; ++kb) {
                    sm100::mbar_wait(&full[stage], phase);
                    sm100::tc_fence_after();
                    const uint32_t st = sm100::smem_u32(smem + stage * C::STAGE_BYTES);
                    if constexpr (Overlap<S>::value) {
                        static_assert(!Overlap<S>::value || (!PAIR && !C::STAGGER), "overlapped accumulators: single CTA");
                        if (kb == kc)
                            static_for<Sc::NT0>([&](auto qc) { issue0(qc, st); });
                        else
                            static_for<Sc::NT>([&](auto qc) { issue(qc, st, kb); });
                    } else {
                        static_for<Sc::NT>([&](auto qc) { issue(qc, st, kb); });
                    }
                    if constexpr (PAIR)
                        sm100::tc_commit_pair(&empty[stage]);
                    else
                        sm100::tc_commit(&empty[stage]);
                    advance(stage, phase);
                }
                if constexpr (PAIR)
                    sm100::tc_commit_pair(&tmem_full[buf]);
                else
                    sm100::tc_commit(&tmem_full[buf]);
                KTRACE(it, 2);
              }
            }
        }
    } else {
        // ---------------------------------------------------- epilogue
        const int quad = warp & 3;         // TMEM lane quadrant this warp may access
        const int part = (warp - 2) >> 2;  // column slice of the tile
        const ModP m = args.modp;
        // this warp's output staging: one 32 x 16 swizzled box per chunk (TMA-store path)
        uint8_t* stg = smem + STAGES * C::STAGE_BYTES + (warp - 2) * 2048;
        bool stores_pending = false;
        // round-aware post (args.round_done): the previous tile's outputs are reported once this
        // warp would idle anyway (before it waits for the next accumulators), not right after
        // its stores were issued
        int report_round = -1;
        auto report = [&]() {
            if (report_round < 0) return;
            if (stores_pending && lane == 0) {
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes complete, not just read
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            stores_pending = false;
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(args.round_done + report_round, 1);
            report_round = -1;
        };
        uint32_t it = 0;
        for (int n = 0;; ++n) {
          const int t = next_tile(n, true);
          if (t < 0) break;
          const int4 tile = args.tiles[t];
          const GroupDesc& g = args.g[tile.x & ((1 << kTileGroupBits) - 1)];
          const int nchunks = (g.k_blocks + g.chunk_blocks - 1) / g.chunk_blocks;
          for (int kc = 0; kc < nchunks; ++kc, ++it) {
            const int buf = C::NBUF == 2 ? (int)(it & 1) : 0;
            const uint32_t use = C::NBUF == 2 ? it >> 1 : it;
            const uint32_t lane_base = tmem + buf * C::BUF_COLS + ((uint32_t)(quad * 32) << 16);
            report();
            sm100::mbar_wait(&tmem_full[buf], use & 1);
            if (warp == 2 && lane == 0) KTRACE(it, 3);
            sm100::tc_fence_after();
            const int row0 = tile.z * C::TILE_M + (int)rank * BM + quad * 32;  // first row of this warp
            const long long grow = (long long)row0 + lane;
            const bool row_ok = grow < g.M;
            uint32_t* out = g.out + (long long)tile.y * g.out_bs + grow * g.ldo;
            const int nch = (BN / 16 - part + kParts - 1) / kParts;  // chunks c0 = 16 (part + j kParts)
            auto col_of = [&](int j) { return 16 * (part + j * kParts); };
            // direct stores (outputs a TMA box cannot describe): this lane's row, 16 columns
            // out64: C <- alpha X + beta C_in in the caller's uint64 C (scale_lower-style, the
            // reference's syrk_classical accumulate, matrix.hpp:372-407); canonical C_in is the
            // contract, others are reduced
            const bool o64 = O64 && g.out64;
            uint64_t* crow = o64 ? g.c64 + grow * g.ldc64 : nullptr;
            auto acc64 = [&](uint32_t x, uint64_t cin) -> uint64_t {
                uint32_t r = g.alpha == 1 ? x : mulc(x, g.calpha, m.p);
                if (g.beta != 0) {
                    const uint32_t ci = cin < m.p ? (uint32_t)cin : mod_u64(cin, m);
                    r = addm(r, g.beta == 1 ? ci : mulc(ci, g.cbeta, m.p), m.p);
                }
                return r;
            };
            auto store64 = [&](const uint32_t (&res)[16], int c0) {
                const long long gc0 = (long long)tile.w * BN + c0;
                if (!row_ok || gc0 >= g.N || (g.syrk && gc0 > grow)) return;
                const bool full_chunk = gc0 + 16 <= g.N && (!g.syrk || gc0 + 15 <= grow) &&
                                        (reinterpret_cast<uintptr_t>(crow + gc0) & 15) == 0;
                if (full_chunk) {
                    ulonglong2* q = reinterpret_cast<ulonglong2*>(crow + gc0);
                    ulonglong2 cin[8];
                    if (g.beta != 0) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) cin[e] = q[e];
                    }
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const uint64_t c0v = g.beta != 0 ? cin[e].x : 0, c1v = g.beta != 0 ? cin[e].y : 0;
                        q[e] = make_ulonglong2(acc64(res[2 * e], c0v), acc64(res[2 * e + 1], c1v));
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const long long gc = gc0 + c;
                        if (gc < g.N && (!g.syrk || gc <= grow))
                            crow[gc] = acc64(res[c], g.beta != 0 ? crow[gc] : 0);
                    }
                }
            };
            auto store_direct = [&](const uint32_t (&res)[16], int c0) {
                if constexpr (O64) {
                    if (o64) {
                        store64(res, c0);
                        return;
                    }
                }
                const long long gc0 = (long long)tile.w * BN + c0;
                if (!row_ok || gc0 >= g.N || (g.syrk && gc0 > grow)) return;
                const bool full_chunk = gc0 + 16 <= g.N && (!g.syrk || gc0 + 15 <= grow) && g.vec_ok;
                if (full_chunk) {
#if FSYRK_STG256
                    if ((reinterpret_cast<uintptr_t>(out + gc0) & 31) == 0) {  // two full 32-byte sectors
#pragma unroll
                        for (int q = 0; q < 2; ++q)
                            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(out + gc0 + 8 * q),
                                         "r"(res[8 * q]), "r"(res[8 * q + 1]), "r"(res[8 * q + 2]), "r"(res[8 * q + 3]),
                                         "r"(res[8 * q + 4]), "r"(res[8 * q + 5]), "r"(res[8 * q + 6]),
                                         "r"(res[8 * q + 7])
                                         : "memory");
                        return;
                    }
#endif
                    uint4* o = reinterpret_cast<uint4*>(out + gc0);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        o[q] = make_uint4(res[4 * q], res[4 * q + 1], res[4 * q + 2], res[4 * q + 3]);
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const long long gc = gc0 + c;
                        if (gc < g.N && (!g.syrk || gc <= grow)) out[gc] = res[c];
                    }
                }
            };
            // staged store of chunk j: row `lane` of the warp's 32 x 16 box (64-byte swizzle,
            // conflict-free), then one TMA store of the box.  The box is reused chunk after chunk:
            // the previous store must have read it first.
            auto stage_store = [&](const uint32_t (&res)[16], int j) {
                const int gc0 = tile.w * BN + col_of(j);
                if (row0 >= g.M || gc0 >= g.N || (g.syrk && gc0 > row0 + 31)) return;
                if (stores_pending) {
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                }
                uint8_t* box = stg + lane * 64;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int qs = q ^ ((lane >> 1) & 3);
                    *reinterpret_cast<uint4*>(box + qs * 16) =
                        make_uint4(res[4 * q], res[4 * q + 1], res[4 * q + 2], res[4 * q + 3]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    asm volatile(
                        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                            reinterpret_cast<uint64_t>(&g.tmO)),
                        "r"(gc0), "r"(row0), "r"(tile.y), "r"(sm100::smem_u32(stg))
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                stores_pending = true;
            };
            auto load = [&](uint32_t (&raw)[C::NACC][16], int c0) {
#pragma unroll
                for (int s = 0; s < C::NACC; ++s) sm100::tmem_ld16(lane_base + s * BN + c0, raw[s]);
            };
            auto ready = [&](uint32_t (&raw)[C::NACC][16]) {
                sm100::tmem_wait_ld();
#pragma unroll
                for (int s = 0; s < C::NACC; ++s) sm100::reg_fence16(raw[s]);
            };
            auto release = [&]() {  // this warp's TMEM reads are complete
                if (lane == 0 && warp == 2) KTRACE(it, 4);
                if (lane == 0 && warp == 9) KTRACE(it, 5);
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (PAIR)
                        sm100::mbar_arrive_cluster(&tmem_empty[buf], 0);  // the leader's MMA waits on both CTAs
                    else
                        sm100::mbar_arrive(&tmem_empty[buf]);
                }
            };
            auto fold = [&](const uint32_t (&raw)[C::NACC][16], uint32_t (&res)[16]) {
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    uint32_t a[C::NACC];
#pragma unroll
                    for (int s = 0; s < C::NACC; ++s) a[s] = raw[s][c];
                    res[c] = fold_acc<S>(a, m, args.w);
                }
            };
#if FSYRK_EPI_EXPERIMENT == 2  // timing experiment: no epilogue at all
            release();
            continue;
#endif
            const bool staged = C::TSTORE && g.tma_ok && !o64;
            uint32_t ra[C::NACC][16];
            if (nchunks > 1) {
                // K-chunked tile (K beyond the int32 exactness bound): every chunk's accumulators
                // are folded to residues and added mod p into the output rows (read-modify-write by
                // the lane that owns the row, so program order makes its own earlier writes
                // visible); the accumulators are released (either protocol) once drained
#pragma unroll
                for (int j = 0; j < C::NCW; ++j) {
                    if (j < nch) {
                        load(ra, col_of(j));
                        ready(ra);
                        uint32_t res[16];
                        fold(ra, res);
                        const long long gc0 = (long long)tile.w * BN + col_of(j);
                        if (row_ok) {
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                const long long gc = gc0 + c;
                                if (gc < g.N && (!g.syrk || gc <= grow)) {
                                    const uint32_t s2 = (kc == 0 ? 0u : out[gc]) + res[c];
                                    const uint32_t r2 = s2 >= m.p ? s2 - m.p : s2;
                                    if (o64 && kc + 1 == nchunks)
                                        crow[gc] = acc64(r2, g.beta != 0 ? crow[gc] : 0);
                                    else
                                        out[gc] = r2;
                                }
                            }
                        }
                    }
                }
                if constexpr (C::STAGGER) {
                    sm100::tc_fence_before();
                    __syncwarp();
                    if (lane == 0)
                        for (int s = 0; s < C::NACC; ++s) sm100::mbar_arrive(&acc_empty[s]);
                } else {
                    release();
                }
            } else if constexpr (C::STAGGER) {
                using V = typename SplitFold<S>::V;
                const bool short_k = g.k_blocks * BK <= 2048;
                V v[C::NCW][16];
#pragma unroll
                for (int s = 0; s < C::NACC; ++s) {
                    uint32_t raw[C::NCW][16];
#pragma unroll
                    for (int j = 0; j < C::NCW; ++j)
                        if (j < nch) sm100::tmem_ld16(lane_base + s * BN + col_of(j), raw[j]);
                    sm100::tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < C::NCW; ++j) sm100::reg_fence16(raw[j]);
                    sm100::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) sm100::mbar_arrive(&acc_empty[s]);  // accumulator s may be overwritten
#pragma unroll
                    for (int j = 0; j < C::NCW; ++j) {
                        if (j < nch) {
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                const V t = SplitFold<S>::term(s, raw[j][c], short_k);
                                v[j][c] = s == 0 ? t : v[j][c] + t;
                            }
                        }
                    }
                }
                if (lane == 0 && warp == 2) KTRACE(it, 4);
#pragma unroll
                for (int j = 0; j < C::NCW; ++j) {
                    if (j < nch) {
                        uint32_t res[16];
#pragma unroll
                        for (int c = 0; c < 16; ++c) res[c] = SplitFold<S>::final(v[j][c], m);
                        if (staged) stage_store(res, j);
                        else store_direct(res, col_of(j));
                    }
                }
            } else if constexpr (SplitFold<S>::ok) {
                // Only a cheap partial fold (one compact value per output) runs while the tile's
                // accumulators hold TMEM; the final reduction and the stores overlap the next
                // tile's MMAs.
                using V = typename SplitFold<S>::V;
                const bool short_k = g.k_blocks * BK <= 2048;
                V v[C::NCW][16];
#pragma unroll
                for (int j = 0; j < C::NCW; ++j) {
                    if (j < nch) {
                        load(ra, col_of(j));
                        ready(ra);
#pragma unroll
                        for (int c = 0; c < 16; ++c) {
                            uint32_t a[C::NACC];
#pragma unroll
                            for (int s = 0; s < C::NACC; ++s) a[s] = ra[s][c];
                            v[j][c] = SplitFold<S>::partial(a, short_k);
                        }
                    }
                }
                release();
#pragma unroll
                for (int j = 0; j < C::NCW; ++j) {
                    if (j < nch) {
                        uint32_t res[16];
#pragma unroll
                        for (int c = 0; c < 16; ++c) res[c] = SplitFold<S>::final(v[j][c], m);
                        if (staged) stage_store(res, j);
                        else store_direct(res, col_of(j));
                    }
                }
            } else {
                uint32_t v[C::NCW][16];  // this warp's folded outputs
#pragma unroll
                for (int j = 0; j < C::NCW; ++j) {
                    if (j < nch) {
                        load(ra, col_of(j));
                        ready(ra);
                        if (j + 1 == nch) release();
                        fold(ra, v[j]);
                        if (staged) stage_store(v[j], j);
                        else store_direct(v[j], col_of(j));
                    }
                }
            }
            if (args.round_done && kc + 1 == nchunks) report_round = tile.x >> kTileGroupBits;  // reported when the warp next idles
            if (lane == 0 && warp == 2) KTRACE(it, 6);
          }
        }
        report();
        if (stores_pending && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#ifdef FSYRK_KTRACE
        if (lane == 0) {
            atomicMax(&g_cta_span[blockIdx.x][1], gtimer());
            g_cta_span[blockIdx.x][2] = it;
        }
#endif
    }
    pdl_trigger_mm();  // this CTA's work is issued: the next kernel of the call may begin launching
    sm100::tc_fence_before();
    __syncthreads();
    if (dyn && threadIdx.x == 0) {
        // thread 0 made all of this CTA's claims; the last CTA to get here rearms the counters
        __threadfence();
        if (atomicAdd(args.dyn + 1, 1) == (int)gridDim.x - 1) {
            args.dyn[0] = 0;
            args.dyn[1] = 0;
            __threadfence();
        }
    }
    if constexpr (PAIR) sm100::cluster_sync();  // no CTA leaves while its peer may still signal it
    sm100::tc_fence_after();
    if (warp == 0) {
        if constexpr (PAIR)
            sm100::tmem_dealloc_pair(tmem, C::TMEM_COLS);
        else
            sm100::tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

template <int S, int EPI = kEpiWarpsDefault>
cudaLaunchConfig_t launch_config(int grid, cudaStream_t stream, cudaLaunchAttribute* attr) {
    using C = Cfg<S>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C::PAIR ? grid & ~1 : grid);
    cfg.blockDim = dim3(64 + 32 * EPI);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cfg.stream = stream;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C::PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cfg;
}

template <int S, int EPI, bool O64>
struct SmemAttrOnce : DeviceOnce {};

template <int S, int EPI, bool O64>
cudaError_t launch_variant(const GroupedArgs& args, int grid, cudaStream_t stream) {
    using C = Cfg<S>;
    auto kern = modmm_kernel<S, EPI, O64>;
    // thread-safe one-time setup per device (the attribute applies to the current device only)
    DeviceOnce& once = per_device<SmemAttrOnce<S, EPI, O64>>();
    std::call_once(once.flag, [&] {
        once.result = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    });
    if (once.result != cudaSuccess) return once.result;
    if (args.ntiles == 0) return cudaSuccess;
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = launch_config<S, EPI>(grid, stream, attr);
    return cudaLaunchKernelEx(&cfg, kern, args);
}

template <int S, int EPI = kEpiWarpsDefault>
cudaError_t launch_cfg(const GroupedArgs& args, int grid, cudaStream_t stream) {
    bool o64 = false;
    for (int g = 0; g < args.ngroups; ++g) o64 |= args.g[g].out64 != 0;
    return o64 ? launch_variant<S, EPI, true>(args, grid, stream) : launch_variant<S, EPI, false>(args, grid, stream);
}

// CTAs per launch: one per SM, or as many CTA pairs as can be co-resident.
template <int S, int EPI = kEpiWarpsDefault>
int grid_for(int nsm) {
    using C = Cfg<S>;
    if constexpr (!C::PAIR) {
        return nsm;
    } else {
        auto kern = modmm_kernel<S, EPI>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
        cudaLaunchAttribute attr[2];
        cudaLaunchConfig_t cfg = launch_config<S, EPI>(nsm, 0, attr);
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters <= 0) {
            cudaGetLastError();
            return nsm & ~1;
        }
        return 2 * clusters < nsm ? 2 * clusters : nsm & ~1;
    }
}

}  // namespace tc
}  // namespace fsyrk_b200
