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
// |T_s| <= L * K * 2^14 < 2^31 and the int64 fold bound limit K
// (modmm_k_limit, checked by the planner).
//
// Tile shape 128 x BN with BN as large as TMEM allows for the 2L-1
// accumulators (L=2: 128, L=3: 96, L=4: 64): the microbenchmark in
// profiles/ubench shows the int8 MMA rate falls with N (shared-memory
// operand bandwidth), so the accumulators are not double-buffered; instead
// the persistent kernel prefetches the next tile while the epilogue drains.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "modp.cuh"
#include "sm100.cuh"
#include "tc_modmm.h"
#include "tc_modmm_kernel.cuh"

namespace fsyrk_b200 {

using namespace tc;

int modmm_block_n(int L) { return L == 2 ? 128 : L == 3 ? 96 : 64; }
int modmm_block_k(int L) { (void)L; return 128; }

size_t modmm_k_limit(int L, uint64_t p) {
    // int32 shift sums: |T_s| <= L * K * 2^14 < 2^31
    const uint64_t k32 = ((1ull << 31) - 1) / ((uint64_t)L * 16384ull);
    // int64 fold with balanced weights: L^2 * K * 2^14 * (p / 2) <= 2^62
    const uint64_t k64 = (1ull << 62) / ((uint64_t)L * L * 16384ull * (p / 2 + 1));
    return (size_t)(k32 < k64 ? k32 : k64);
}

cudaError_t modmm_launch(int L, const GroupedArgs& args, int grid, cudaStream_t stream) {
    switch (L) {
        case 2: return launch_cfg<2, 128, 128, 3>(args, grid, stream);
        case 3: return launch_cfg<3, 96, 128, 2>(args, grid, stream);
        case 4: return launch_cfg<4, 64, 128, 2>(args, grid, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fsyrk_b200
