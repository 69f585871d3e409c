// HBM-bound mod-p elementwise kernels of the recursion.
//
//  convert_in : uint64 reference-layout input -> uint32 residues, with the
//               optional syrkd column transform folded in
//               (include/fsyrk/scaled_syrk.hpp:77-101).
//  prep       : the fused pre-additions of one level node, Table 3 steps
//               1, 2, 4, 6 (include/fsyrk/fast_syrk.hpp:100-115):
//                 S1 = (A21 - A11) Y, S2 = A22 - A21 Y, S3 = S1 - A22,
//                 S4 = S3 + A12,
//               with the Y multiplication (include/fsyrk/skew.hpp:124-167)
//               and the zero padding of the Pair form (fast_syrk.hpp:34-57)
//               fused in.  Reads each A element once and writes the GEMM /
//               leaf operands directly as int8 limb planes.
//  post       : the fused post-additions U1..U5 (fast_syrk.hpp:120-132):
//                 X11 = Low(P1 + P2), X21 = U1 + P4 + P3,
//                 X22 = Low(U1 + P4 + P4^T),  U1 = sym(P1 + P5),
//               over 32 x 32 tile pairs with shared-memory transposes.
//  finalize   : C <- alpha X + beta C on Low(C) (scale_*/U5-with-beta of the
//               accumulating schedule, fast_syrk.hpp:202-239, matrix.hpp:248-263)
//               plus mirror_lower_to_upper (matrix.hpp:225-232).
#include <cuda_runtime.h>

#include <cstdint>

#include "elementwise.cuh"

namespace fsyrk_b200 {

namespace {

__global__ void convert_in_kernel(const uint64_t* __restrict__ a, long long lda, int n, int kin, int kout,
                                  const ColMap* __restrict__ map, ModP m, uint32_t* __restrict__ out,
                                  long long ldo) {
    const long long total = (long long)n * kout;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / kout), c = (int)(idx % kout);
        const uint64_t* row = a + (long long)i * lda;
        uint32_t v;
        if (map == nullptr) {
            v = mod_u64(row[c], m);
        } else {
            const ColMap cm = map[c];
            v = 0;
            if (cm.src0 >= 0) v = mulm(mod_u64(row[cm.src0], m), cm.c0, m);
            if (cm.src1 >= 0) v = addm(v, mulm(mod_u64(row[cm.src1], m), cm.c1, m), m.p);
        }
        out[(long long)i * ldo + c] = v;
    }
}

template <int L>
__device__ __forceinline__ void put_planes(int8_t* base, long long plane, long long off, uint32_t x, uint32_t p) {
    int8_t d[L];
    split_limbs<L>(x, p, d);
#pragma unroll
    for (int l = 0; l < L; ++l) base[l * plane + off] = d[l];
}

template <int L>
__global__ void split_planes_kernel(const uint32_t* __restrict__ a, long long lda, int rows, int k, uint32_t p,
                                    int8_t* __restrict__ planes, long long plane, long long rs) {
    const long long total = (long long)rows * k;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / k), c = (int)(idx % k);
        put_planes<L>(planes, plane, (long long)i * rs + c, a[(long long)i * lda + c], p);
    }
}

// One thread per (row i, column pair j) of the h x kw S-blocks.
template <int L>
__global__ void prep_kernel(const PrepArgs args) {
    const PrepNode nd = args.nodes[blockIdx.z];
    const ModP m = args.m;
    const uint32_t p = m.p;
    const int h = args.h, kh = args.kh, kw = args.kw, half = args.half;
    const int ncw = args.pair ? half : kw;
    const int jp = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y * blockDim.y + threadIdx.y;
    if (jp >= ncw || i >= h) return;

    const uint32_t* r1 = nd.a + (long long)i * nd.lda;            // row i of A11 | A12
    const uint32_t* r2 = nd.a + (long long)(i + h) * nd.lda;      // row i of A21 | A22
    const int nc = args.pair ? 2 : 1;
    int col[2] = {jp, jp + half};
    uint32_t a11[2], a12[2], a21[2], a22[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int c = col[t];
        const bool ok = t < nc && c < kh;
        a11[t] = ok ? r1[c] : 0;
        a12[t] = ok ? r1[kh + c] : 0;
        a21[t] = ok ? r2[c] : 0;
        a22[t] = ok ? r2[kh + c] : 0;
    }
    uint32_t s1[2], ay[2];
    if (args.pair) {
        const uint32_t d0 = subm(a21[0], a11[0], p), d1 = subm(a21[1], a11[1], p);
        // (u, v) -> (a u - b v, b u + a v) on the column halves (skew.hpp:146-163)
        s1[0] = subm(mulm(args.ya, d0, m), mulm(args.yb, d1, m), p);
        s1[1] = addm(mulm(args.yb, d0, m), mulm(args.ya, d1, m), p);
        ay[0] = subm(mulm(args.ya, a21[0], m), mulm(args.yb, a21[1], m), p);
        ay[1] = addm(mulm(args.yb, a21[0], m), mulm(args.ya, a21[1], m), p);
    } else {
        s1[0] = mulm(subm(a21[0], a11[0], p), args.ya, m);
        ay[0] = mulm(a21[0], args.ya, m);
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
        put_planes<L>(nd.s1, args.g_plane, go, s1[t], p);
        put_planes<L>(nd.a22, args.g_plane, go, a22[t], p);
        put_planes<L>(nd.s2, args.g_plane, go, s2, p);
        put_planes<L>(nd.s4, args.g_plane, go, s4, p);
        if (c < kh) {
            if (nd.c_a11) put_planes<L>(nd.c_a11, args.c_plane, (long long)i * args.c_row + c, a11[t], p);
            if (nd.c_a12) put_planes<L>(nd.c_a12, args.c_plane, (long long)i * args.c_row + c, a12[t], p);
        }
        if (nd.c_s3) put_planes<L>(nd.c_s3, args.c3_plane, (long long)i * args.c3_row + c, s3, p);
        if (nd.r_s3) nd.r_s3[(long long)i * nd.ld_s3 + c] = s3;
    }
}

constexpr int TS = 32;  // post / mirror tile

__device__ __forceinline__ void tri_decode(int t, int& I, int& J) {
    int r = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    I = r;
    J = t - r * (r + 1) / 2;
}

// Block (32 x 8) per tile pair (I >= J) of one node.
__global__ void post_kernel(const PostArgs args) {
    __shared__ uint32_t sU[TS][TS + 1];   // Low(P1 + P5), tile (I, J)
    __shared__ uint32_t sT[TS][TS + 1];   // P4 tile (J, I)
    const PostNode nd = args.nodes[blockIdx.z];
    const uint32_t p = args.p;
    const int h = args.h;
    int I, J;
    tri_decode(blockIdx.x, I, J);
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int j = J * TS + tx;       // column inside tile (I, J)
    const int jt = I * TS + tx;      // column inside tile (J, I)
    for (int r = ty; r < TS; r += 8) {
        const int i = I * TS + r, it = J * TS + r;
        uint32_t u = 0, t4 = 0;
        if (i < h && j < h) u = addm(nd.p1[(long long)i * nd.ld1 + j], nd.p5[(long long)i * nd.ld5 + j], p);
        if (it < h && jt < h) t4 = nd.p4[(long long)it * nd.ld4 + jt];
        sU[r][tx] = u;
        sT[r][tx] = t4;
    }
    __syncthreads();
    uint32_t* x11 = nd.x;
    uint32_t* x21 = nd.x + (long long)h * nd.ldx;
    uint32_t* x22 = x21 + h;
    for (int r = ty; r < TS; r += 8) {
        const int i = I * TS + r;
        if (i < h && j < h) {
            // U1(i, j) from the lower triangle (symmetric completion on the diagonal tile)
            const uint32_t u1 = (I == J && tx > r) ? sU[tx][r] : sU[r][tx];
            const uint32_t p4 = nd.p4[(long long)i * nd.ld4 + j];
            const uint32_t p3 = nd.p3[(long long)i * nd.ld3 + j];
            const uint32_t u2 = addm(u1, p4, p);
            x21[(long long)i * nd.ldx + j] = addm(u2, p3, p);
            x22[(long long)i * nd.ldx + j] = addm(u2, sT[tx][r], p);
            x11[(long long)i * nd.ldx + j] =
                addm(nd.p1[(long long)i * nd.ld1 + j], nd.p2[(long long)i * nd.ld2 + j], p);
        }
        if (I != J) {
            // tile (J, I) of X21: U1^T + P4(J, I) + P3(J, I)
            const int it = J * TS + r;
            if (it < h && jt < h) {
                const uint32_t v = addm(addm(sU[tx][r], sT[r][tx], p), nd.p3[(long long)it * nd.ld3 + jt], p);
                x21[(long long)it * nd.ldx + jt] = v;
            }
        }
    }
}

__global__ void add_lower_kernel(const AddNode* __restrict__ nodes, int n, uint32_t p) {
    const AddNode nd = nodes[blockIdx.z];
    const int i = blockIdx.y;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= i && j < n; j += gridDim.x * blockDim.x)
        nd.x[(long long)i * nd.ldx + j] = addm(nd.x1[(long long)i * nd.ld1 + j], nd.x2[(long long)i * nd.ld2 + j], p);
}

__global__ void finalize_kernel(const uint32_t* __restrict__ x, long long ldx, int n, uint64_t* __restrict__ c,
                                long long ldc, ModP m, uint32_t alpha, uint32_t beta) {
    const int i = blockIdx.y;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= i && j < n; j += gridDim.x * blockDim.x) {
        uint32_t v = x[(long long)i * ldx + j];
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

__global__ void zero_upper_kernel(uint64_t* __restrict__ c, long long ldc, int n) {
    const int i = blockIdx.y;
    for (int j = i + 1 + blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        c[(long long)i * ldc + j] = 0;
}

__global__ void u32_to_u64_kernel(const uint32_t* __restrict__ x, long long ldx, int rows, int cols,
                                  uint64_t* __restrict__ out, long long ldo) {
    const long long total = (long long)rows * cols;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / cols), j = (int)(idx % cols);
        out[(long long)i * ldo + j] = x[(long long)i * ldx + j];
    }
}

int grid_for(long long total, int threads) {
    long long b = (total + threads - 1) / threads;
    if (b > 148 * 32) b = 148 * 32;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t launch_convert_in(const uint64_t* a, long long lda, int n, int kin, int kout, const ColMap* map,
                              uint32_t p, uint32_t* out, long long ldo, cudaStream_t s) {
    (void)kin;
    const long long total = (long long)n * kout;
    if (total == 0) return cudaSuccess;
    convert_in_kernel<<<grid_for(total, 256), 256, 0, s>>>(a, lda, n, kin, kout, map, make_modp(p), out, ldo);
    return cudaGetLastError();
}

cudaError_t launch_split_planes(int L, const uint32_t* a, long long lda, int rows, int k, uint32_t p, int8_t* planes,
                                long long plane_stride, long long row_stride, cudaStream_t s) {
    const long long total = (long long)rows * k;
    if (total == 0) return cudaSuccess;
    const int g = grid_for(total, 256);
    switch (L) {
        case 2: split_planes_kernel<2><<<g, 256, 0, s>>>(a, lda, rows, k, p, planes, plane_stride, row_stride); break;
        case 3: split_planes_kernel<3><<<g, 256, 0, s>>>(a, lda, rows, k, p, planes, plane_stride, row_stride); break;
        case 4: split_planes_kernel<4><<<g, 256, 0, s>>>(a, lda, rows, k, p, planes, plane_stride, row_stride); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_prep(const PrepArgs& args, cudaStream_t s) {
    const int ncw = args.pair ? args.half : args.kw;
    if (ncw == 0 || args.h == 0 || args.nnodes == 0) return cudaSuccess;
    dim3 block(32, 8);
    dim3 grid((ncw + 31) / 32, (args.h + 7) / 8, args.nnodes);
    switch (args.L) {
        case 2: prep_kernel<2><<<grid, block, 0, s>>>(args); break;
        case 3: prep_kernel<3><<<grid, block, 0, s>>>(args); break;
        case 4: prep_kernel<4><<<grid, block, 0, s>>>(args); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_post(const PostArgs& args, cudaStream_t s) {
    if (args.h == 0 || args.nnodes == 0) return cudaSuccess;
    const int T = (args.h + TS - 1) / TS;
    dim3 grid(T * (T + 1) / 2, 1, args.nnodes);
    post_kernel<<<grid, dim3(32, 8), 0, s>>>(args);
    return cudaGetLastError();
}

cudaError_t launch_add_lower(const AddNode* nodes, int nnodes, int n, uint32_t p, cudaStream_t s) {
    if (n == 0 || nnodes == 0) return cudaSuccess;
    dim3 grid((n + 255) / 256, n, nnodes);
    add_lower_kernel<<<grid, 256, 0, s>>>(nodes, n, p);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const uint32_t* x, long long ldx, int n, uint64_t* c, long long ldc, const ModP& m,
                            uint32_t alpha, uint32_t beta, int mirror, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    dim3 grid((n + 255) / 256, n);
    finalize_kernel<<<grid, 256, 0, s>>>(x, ldx, n, c, ldc, m, alpha, beta);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !mirror) return e;
    const int T = (n + TS - 1) / TS;
    mirror_kernel<<<T * (T + 1) / 2, dim3(32, 8), 0, s>>>(c, ldc, n);
    return cudaGetLastError();
}

cudaError_t launch_zero_upper(uint64_t* c, long long ldc, int n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    zero_upper_kernel<<<dim3((n + 255) / 256, n), 256, 0, s>>>(c, ldc, n);
    return cudaGetLastError();
}

cudaError_t launch_u32_to_u64(const uint32_t* x, long long ldx, int rows, int cols, uint64_t* out, long long ldo,
                              cudaStream_t s) {
    const long long total = (long long)rows * cols;
    if (total == 0) return cudaSuccess;
    u32_to_u64_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, ldx, rows, cols, out, ldo);
    return cudaGetLastError();
}

}  // namespace fsyrk_b200
