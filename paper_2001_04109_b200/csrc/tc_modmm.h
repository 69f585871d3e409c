// Host interface of the tensor-core mod-p product kernel (tc_modmm.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "modp.cuh"

namespace fsyrk_b200 {

struct ModmmArgs {
    ModP modp;
    uint32_t c32;             // 2^32 mod p (fold of the high shifts for L = 4)
    int M, N;                 // output rows / cols of every problem in the batch
    int k_blocks;             // ceil(K / 128)
    int tiles_n;              // column tiles (dense mode)
    int syrk;                 // 1: only j <= i is written (lower triangle)
    int vec_ok;               // ldo % 4 == 0 and out 16-byte aligned
    int a_batch_mult, a_batch_off;  // operand slot of problem b: b * mult + off
    int b_batch_mult, b_batch_off;
    const int2* tile_list;    // SYRK: (tm, tn) per CTA; dense: nullptr
    uint32_t* out;            // residues, problem b at out + b * out_batch_stride
    long long out_batch_stride;
    long long ldo;
};

int modmm_block_n(int L);
constexpr int modmm_block_m() { return 128; }
size_t modmm_k_limit(int L);

cudaError_t modmm_launch(int L, const CUtensorMap& ta, const CUtensorMap& tb, const ModmmArgs& args, int ntiles,
                         int batch, cudaStream_t stream);

}  // namespace fsyrk_b200
