// Host interface of the tensor-core mod-p product kernel (tc_modmm.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "modp.cuh"

namespace fsyrk_b200 {

constexpr int kMaxGroups = 6;

// One uniform batch of products C_b = A_b * B_b^T (mod p).  Operands are int8
// digit planes [slot][P][rows][kpad] reached through the two TMA descriptors;
// problem b reads A slot b * a_mult + a_off and B slot b * b_mult + b_off.
struct alignas(64) GroupDesc {
    CUtensorMap tmA;  // box BK (K) x 128 rows
    CUtensorMap tmB;  // box BK (K) x b_box rows
    CUtensorMap tmO;  // outputs [batch][M][N] u32, box 16 x 32 (64-byte swizzle) -- valid if tma_ok
    int M, N;         // output rows / cols
    int k_blocks;     // kpad / BK
    int chunk_blocks; // K-blocks per exact chunk: the accumulators are drained (folded mod p into
                      // a running residue) every chunk_blocks K-blocks, so any K stays exact
    int syrk;         // 1: only j <= i is written (lower triangle)
    int vec_ok;       // ldo % 4 == 0 (16-byte vector stores)
    int a_mult, a_off, b_mult, b_off;
    int tma_ok;       // outputs stored by TMA from shared memory (16-byte aligned rows)
    uint32_t* out;    // residues, problem b at out + b * out_bs
    long long out_bs;
    long long ldo;
    // out64 (one-problem groups): the epilogue writes C <- alpha X + beta C_in straight into the
    // caller's uint64 C (Low only for syrk) instead of uint32 residues -- a root-leaf plan's
    // finalisation fused into the products (out stays the K-chunk partial scratch)
    int out64;
    uint64_t* c64;
    long long ldc64;
    uint32_t alpha, beta;
    MulConst calpha, cbeta;
};

struct GroupedArgs {
    GroupDesc g[kMaxGroups];
    ModP modp;
    int32_t w[8];       // balanced fold weights (LIMB schemes)
    int ngroups;
    int ntiles;
    const int4* tiles;  // (group | round << 8, batch, tm, tn), longest K first
    // Balanced schedule (driver.cu, Plan::balance_tiles): scheduling unit u (CTA, or CTA pair)
    // runs tiles[tile_off[u] .. tile_off[u + 1]) in order; nullptr: unit u runs tiles u, u +
    // units, u + 2 units, ...
    const int* tile_off;
    // Dynamic schedule (single-CTA schemes): dyn[0] is the next unclaimed position of the tile
    // list (after the first `units` tiles, which are claimed by CTA index), dyn[1] counts finished
    // CTAs; the last one to finish resets both for the next launch.  nullptr: static schedule.
    int* dyn;
    // Root post overlap (driver.cu, Plan::rounds): every epilogue warp adds 1 to round_done[round
    // of the tile] once its stores of the tile are globally visible, and the launch lets its
    // programmatic dependent (the round-aware post kernel) start as soon as every CTA is past
    // its prologue.  nullptr: off.
    int* round_done;
};
constexpr int kTileGroupBits = 8;
// epilogue warps per CTA of the product kernel (each reports once per tile to round_done)
int modmm_epilogue_warps();

// Scheme selection and its parameters (schemes.cuh).
struct SchemeInfo {
    int id;
    int planes;   // planes stored for an operand read in both roles (leaf SYRK operands)
    int pa, pb;   // planes the A / B role reads (GEMM operands store only these)
    int nacc, nterms;  // accumulators; MMAs issued per 32-deep K step
    int products;      // distinct digit-plane products per modular MAC (the algorithmic count)
    int bn, bk;
    int bm;       // output rows per tile: 128, or 256 on a CTA pair
    int b_box;    // B rows one CTA stages per tile (bn, or bn / 2 on a CTA pair)
    bool is_unsigned;
};
// nranks >= 3: partitioned multi-GPU plans use narrower tiles where that makes the partition
// blocks (lcm of the tile sides) finer (p = 2^17 - 1: 128 instead of 640)
SchemeInfo scheme_for(uint64_t p, int nranks = 1);
// Largest inner dimension for which the scheme's int32 accumulators and fold stay exact: the
// product kernel drains its accumulators at least this often along K (chunk_blocks).
size_t modmm_k_limit(const SchemeInfo& s, uint64_t p);
// g.k_blocks / g.chunk_blocks for an operand K padded to kpad (a multiple of 128).
void modmm_set_k(GroupDesc& g, const SchemeInfo& s, uint64_t p, long long kpad);
void fill_fold_weights(const SchemeInfo& s, uint64_t p, int32_t* w);

cudaError_t modmm_launch(const SchemeInfo& s, const GroupedArgs& args, int grid, cudaStream_t stream);
// CTAs per persistent launch on a device with nsm SMs.
int modmm_grid(const SchemeInfo& s, int nsm);
// Output descriptor of a product group (sets g.tmO / g.tma_ok from g.out, M, N, ldo, out_bs).
void modmm_set_output_map(GroupDesc& g, int batch);

}  // namespace fsyrk_b200
