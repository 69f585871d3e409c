// Host interface of the HBM-bound elementwise mod-p kernels (elementwise.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "modp.cuh"

namespace fsyrk_b200 {

// Output column c of the converted operand is  c0 * A[:, src0] + c1 * A[:, src1]
// (src < 0: term absent).  Encodes the syrkd column transform
// (include/fsyrk/scaled_syrk.hpp:77-101); nullptr map = identity.
struct ColMap {
    int src0, src1;
    uint32_t c0, c1;
};

// One level node of the recursion for the fused pre-addition kernel.
struct PrepNode {
    const uint32_t* a;  // node input (n x k residues)
    long long lda;
    int8_t* s1;   // GEMM operand slots (limb-plane bases)
    int8_t* a22;
    int8_t* s2;
    int8_t* s4;
    int8_t* c_a11;  // leaf-operand slots of the children (nullable)
    int8_t* c_a12;
    int8_t* c_s3;
    uint32_t* r_s3;  // residue S3 for a non-leaf child (nullable)
    long long ld_s3;
};

struct PrepArgs {
    ModP m;
    int L;
    int h, kh, kw, half, pair;
    uint32_t ya, yb;
    long long g_plane, g_row;    // GEMM operand plane stride / row stride (bytes)
    long long c_plane, c_row;    // leaf operand planes for A11 / A12 (k = kh)
    long long c3_plane, c3_row;  // leaf operand planes for S3 (k = kw)
    const PrepNode* nodes;
    int nnodes;
};

struct PostNode {
    const uint32_t *p1, *p2, *p5, *p3, *p4;
    long long ld1, ld2, ld5, ld3, ld4;
    uint32_t* x;
    long long ldx;
};

struct PostArgs {
    uint32_t p;
    int h;
    const PostNode* nodes;
    int nnodes;
};

struct AddNode {
    const uint32_t *x1, *x2;
    long long ld1, ld2;
    uint32_t* x;
    long long ldx;
};

cudaError_t launch_convert_in(const uint64_t* a, long long lda, int n, int kin, int kout, const ColMap* map,
                              uint32_t p, uint32_t* out, long long ldo, cudaStream_t s);
cudaError_t launch_split_planes(int L, const uint32_t* a, long long lda, int rows, int k, uint32_t p, int8_t* planes,
                                long long plane_stride, long long row_stride, cudaStream_t s);
cudaError_t launch_prep(const PrepArgs& args, cudaStream_t s);
cudaError_t launch_post(const PostArgs& args, cudaStream_t s);
cudaError_t launch_add_lower(const AddNode* nodes, int nnodes, int n, uint32_t p, cudaStream_t s);
// C (uint64) <- alpha * X + beta * C on the lower triangle; then optional mirror.
cudaError_t launch_finalize(const uint32_t* x, long long ldx, int n, uint64_t* c, long long ldc, const ModP& m,
                            uint32_t alpha, uint32_t beta, int mirror, cudaStream_t s);
cudaError_t launch_zero_upper(uint64_t* c, long long ldc, int n, cudaStream_t s);
cudaError_t launch_u32_to_u64(const uint32_t* x, long long ldx, int rows, int cols, uint64_t* out, long long ldo,
                              cudaStream_t s);

}  // namespace fsyrk_b200
