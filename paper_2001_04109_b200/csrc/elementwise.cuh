// Host interface of the HBM-bound elementwise mod-p kernels (elementwise.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "modp.cuh"
#include "schemes.cuh"

namespace fsyrk_b200 {

// Output column c of the converted operand is  c0 * A[:, src0] + c1 * A[:, src1]
// (src < 0: term absent).  Encodes the syrkd column transform
// (include/fsyrk/scaled_syrk.hpp:77-101); nullptr map = identity.
// Column j of the transformed input = sum_t c[t] * A[:, src[t]] (src < 0: unused term).
// syrkd pairs two (scaled) columns (scaled_syrk.hpp:91-100); syrkbd first folds each 2x2
// antidiagonal block into (u + v, u - v) (:146-153), so a column mixes at most 4 of A's.
struct ColMap {
    int src[4];
    uint32_t c[4];
};

// Where a node reads its input: an internal uint32 residue buffer, or a
// window of the caller's uint64 matrix (base pointer supplied per call).
struct InView {
    const uint32_t* p32;  // used when in64 == 0
    long long ld32;
    int r0, c0;           // used when in64 == 1: window origin in the caller's matrix
    int in64;
};

// One level node of the recursion for the fused pre-addition kernel.
struct PrepNode {
    InView in;
    int8_t* s1;   // GEMM operand slots (limb-plane bases)
    int8_t* a22;
    int8_t* s2;
    int8_t* s4;
    int8_t* c_a11;  // leaf-operand slots of the children (nullable)
    int8_t* c_a12;
    int8_t* c_s3;
    uint32_t* r_s3;  // residue S3 for a non-leaf child (nullable)
    long long ld_s3;
    // Winograd general products (s1 == nullptr): S1, S2, A22, S4 as uint32 residues at
    // r_op + {0, 1, 2, 3} * op_stride, row stride ld_op (the Winograd engine's operands)
    uint32_t* r_op;
    long long ld_op, op_stride;
};

struct PrepArgs {
    ModP m;
    int L;
    int in64;                 // some node of the launch reads the caller's uint64 input
    const uint64_t* a64;      // caller's input (per call)
    long long ld64;
    int h, kh, kw, half, pair;
    uint32_t ya, yb;
    MulConst cya, cyb;
    long long g_plane, g_row;    // GEMM operand plane stride / row stride (bytes)
    long long c_plane, c_row;    // leaf operand planes for A11 / A12 (k = kh)
    long long c3_plane, c3_row;  // leaf operand planes for S3 (k = kw)
    const PrepNode* nodes;
    int nnodes;
    // ninl = nnodes when the node table also travels by value in inl[] (<= kInlineNodes nodes):
    // the kernels then read it from their parameter (constant) space instead of starting every
    // block with a dependent global load (measured on the fused subtree kernel: -8% of its time)
    int ninl;
    PrepNode inl[3];
    int aligned;  // every node's input rows allow 16-byte vector loads at 4-column steps (driver-checked)
    // multi-GPU partition: only rows i of blocks (i / part_block) set in need_mask are prepared
    // (the row blocks of this rank's block pairs); part_block = 0: all rows
    int part_block;
    unsigned long long need_mask;
};

// Fused pre-additions of a complete uniform subtree of D levels (D = 2, 3) read straight from
// the caller's uint64 A: every LEVEL node at depth d < D has the same (h, kh), no padding, and
// all nodes at depth D are leaves.  nodes[d] holds the depth-d PrepNode tables in tree order
// (node t's children P1, P2, P5 are 3t, 3t + 1, 3t + 2 at depth d + 1).
struct PrepTreeArgs {
    ModP m;
    int L;  // digit scheme
    int depth;
    const uint64_t* a64;  // caller's input (per call)
    long long ld64;
    int rows, w;  // fine block (the leaf operand): rows = n >> D, w = k >> D
    int cp;       // columns (Pair: column pairs) per CTA: a multiple of 4 dividing w / NC, <= 64
    int pair;
    MulConst cya, cyb;
    long long g_plane[4], g_row[4];  // GEMM operand plane / row stride per depth
    long long c_plane, c_row;        // leaf operand planes (depth D)
    const PrepNode* nodes[4];
    // The nodes' operand bases by value (node index: level 0 -> 0, level 1 -> 1 + t, level 2 ->
    // 4 + t): they reach the kernel in its parameter (constant) space, so an item's stores do
    // not wait on a dependent global load of the node table first.
    struct Ptrs {
        int8_t *s1, *a22, *s2, *s4, *c_a11, *c_a12, *c_s3;
    } tp[13];
};

struct PostNode {
    const uint32_t *p1, *p2, *p5, *p3, *p4;
    long long ld1, ld2, ld5, ld3, ld4;
    uint32_t* x;
    long long ldx;
};

struct PostArgs {
    ModP m;
    int h;
    const PostNode* nodes;
    int nnodes;
    int ninl;         // nodes also by value in inl[] (see PrepArgs::ninl); 0: read the device table
    PostNode inl[3];
    // out64: the root writes the caller's C directly: C <- alpha X + beta C on Low(C)
    int out64;
    uint64_t* c64;
    long long ldc;
    uint32_t alpha, beta;
    MulConst calpha, cbeta;  // make_mulconst(alpha / beta, p), set by the host with alpha, beta
    // multi-GPU partition: only these 32 x 32 tile pairs (I >= J); nullptr = all pairs
    const int2* pairs;
    int npairs;
    // low-memory schedule: the root's P4 / P3 live in the caller's scratch quadrant C12
    // (uint32 pairs per uint64 row, ld34 = 2 ldc); nullptr = the node table's buffers
    const uint32_t *p4o, *p3o;
    long long ld34o;
};

// the node of this block, with the per-call P3 / P4 override of the low-memory schedule
__host__ __device__ inline PostNode post_node(const PostArgs& a, const PostNode& n) {
    PostNode r = n;
    if (a.p4o) {
        r.p4 = a.p4o;
        r.p3 = a.p3o;
        r.ld3 = r.ld4 = a.ld34o;
    }
    return r;
}

// The two deepest post-addition levels fused (post2_kernel): the deepest level nodes (whose
// three products are leaves) and their parents in one launch.  par.nodes are the parents in
// tree order, ch the deepest nodes (parent t's children P1, P2, P5 at 3t, 3t + 1, 3t + 2);
// par.h is the parents' quadrant size, h2 = par.h / 2 the children's (a multiple of 32).
struct Post2Args {
    PostArgs par;
    const PostNode* ch;
    int h2;
    int nchi;          // children also by value in chi[] (<= 9); 0: read the device table
    PostNode chi[9];
};
constexpr int kInlineNodes = 3, kInlineChildren = 9;

struct AddNode {
    const uint32_t *x1, *x2;
    long long ld1, ld2;
    uint32_t* x;
    long long ldx;
};

// Root post-addition overlapped with the products: pairs (I | round << 20, J) in round order,
// taken through *next_pair (zeroed per call); waits for round_done[r] >= target[r].
cudaError_t launch_post_rounds(const PostArgs& args, const int* round_done, const int* target, int* next_pair,
                               int blocks, cudaStream_t s);
cudaError_t launch_convert_in(const uint64_t* a, long long lda, int n, int kin, int kout, const ColMap* map,
                              uint32_t p, uint32_t* out, long long ldo, cudaStream_t s);
// Residues (uint32 view, or the caller's uint64 window) -> limb planes.
cudaError_t launch_split_planes(int L, const InView& in, const uint64_t* a64, long long ld64, int rows, int k,
                                uint32_t p, int8_t* planes, long long plane_stride, long long row_stride,
                                cudaStream_t s);
cudaError_t launch_prep(const PrepArgs& args, cudaStream_t s);
cudaError_t launch_prep_tree(const PrepTreeArgs& args, int nsm, cudaStream_t s);
cudaError_t launch_post(const PostArgs& args, cudaStream_t s);
cudaError_t launch_post2(const Post2Args& args, cudaStream_t s);
cudaError_t launch_add_lower(const AddNode* nodes, int nnodes, int n, uint32_t p, cudaStream_t s);
// C (uint64) <- alpha * X + beta * C on the lower triangle (X == nullptr: X = 0).
cudaError_t launch_finalize(const uint32_t* x, long long ldx, int n, uint64_t* c, long long ldc, const ModP& m,
                            uint32_t alpha, uint32_t beta, cudaStream_t s);
cudaError_t launch_mirror(uint64_t* c, long long ldc, int n, cudaStream_t s);
// Strassen-Winograd level: pre-additions (side 0: A blocks -> S1..S4, side 1: stored B blocks ->
// T1..T4) and post-additions (M1..M7 -> the four quadrants of C)
cudaError_t launch_wino_pre(const uint32_t* x11, const uint32_t* x12, const uint32_t* x21, const uint32_t* x22,
                            long long ld, int rows, int cols, uint32_t p, int side, uint32_t* out, long long ldo,
                            long long bs, cudaStream_t s);
cudaError_t launch_wino_post(const uint32_t* m, long long bs, long long ldm, int rows, int cols, uint32_t p,
                             uint32_t* c, long long ldc, cudaStream_t s);
// F_{p^2}: split (a, b) pairs into X, Y; combine R (real part) and G into C pairs
cudaError_t launch_deinterleave(const uint64_t* a, long long ldp, int n, int k, uint64_t* x, uint64_t* y,
                                cudaStream_t s);
cudaError_t launch_fp2_combine(const uint64_t* r, long long ldr, const uint32_t* g, long long ldg, int n, uint32_t p,
                               int conj, int mirror, uint64_t* c, long long ldcp, cudaStream_t s);
cudaError_t launch_zero_upper(uint64_t* c, long long ldc, int n, int rb, cudaStream_t s);
// Multi-GPU shares: the 32 x 32 tiles of Low(C) a partitioned rank's root post writes for its
// tile pairs, packed as uint32 (4 x 1024 words per pair), and back into a uint64 C
cudaError_t launch_share_pack(const uint64_t* c, long long ldc, int h, const int2* pairs, int npairs, uint32_t* out,
                              cudaStream_t s);
cudaError_t launch_share_unpack(const uint32_t* in, int h, const int2* pairs, int npairs, uint64_t* c, long long ldc,
                                cudaStream_t s);
cudaError_t launch_u32_to_u64(const uint32_t* x, long long ldx, int rows, int cols, uint64_t* out, long long ldo,
                              cudaStream_t s);

}  // namespace fsyrk_b200
