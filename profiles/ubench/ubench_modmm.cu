// Microbenchmark of the persistent tcgen05 int8-limb product kernel (tiling study).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2001_04109_b200/csrc \
//        ubench_modmm.cu -o ubench_modmm
// Prints, per variant, ms and int8 TOP/s (2 * L^2 * M * N * K / t) on a dense batch of M x N x K products.
// r01 (non-persistent kernel) results are in profiles/r01/ubench_modmm_nonpersistent.txt.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tc_modmm_kernel.cuh"

using namespace fsyrk_b200;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn enc() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        fn = (EncodeFn)p;
    }
    return fn;
}
static CUtensorMap pmap(void* base, int kpad, int rows, int L, int batch, int box_rows, int bk) {
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)kpad, (cuuint64_t)rows, (cuuint64_t)L, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)kpad, (cuuint64_t)kpad * rows, (cuuint64_t)kpad * rows * L};
    cuuint32_t box[4] = {(cuuint32_t)bk, (cuuint32_t)box_rows, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       bk == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
    return m;
}

template <int L, int BN, int BK, int STAGES, int EPI = 8>
void run(const char* name, int M, int N, int K, int batch, int8_t* A, int8_t* B, uint32_t* out, int reps) {
    GroupedArgs a;
    memset(&a, 0, sizeof(a));
    a.modp = make_modp(131071);
    for (int s = 0; s < 8; ++s) a.w[s] = 1;
    a.ngroups = 1;
    GroupDesc& g = a.g[0];
    g.tmA = pmap(A, K, M, L, batch, 128, BK);
    g.tmB = pmap(B, K, N, L, batch, BN, BK);
    g.M = M; g.N = N; g.k_blocks = K / BK; g.syrk = 0; g.vec_ok = 1;
    g.a_mult = g.b_mult = 1;
    g.out = out; g.out_bs = (long long)M * N; g.ldo = N;
    std::vector<int4> tiles;
    for (int b = 0; b < batch; ++b)
        for (int tm = 0; tm < M / 128; ++tm)
            for (int tn = 0; tn * BN < N; ++tn) tiles.push_back(make_int4(0, b, tm, tn));
    int4* dt;
    CK(cudaMalloc(&dt, tiles.size() * sizeof(int4)));
    CK(cudaMemcpy(dt, tiles.data(), tiles.size() * sizeof(int4), cudaMemcpyHostToDevice));
    a.tiles = dt;
    a.ntiles = (int)tiles.size();
    int grid = a.ntiles < 148 ? a.ntiles : 148;
    for (int i = 0; i < 2; ++i) CK((tc::launch_cfg<L, BN, BK, STAGES, EPI>(a, grid, 0)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) CK((tc::launch_cfg<L, BN, BK, STAGES, EPI>(a, grid, 0)));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    double ops = 2.0 * L * L * (double)M * N * K * batch;
    printf("%-18s L=%d BN=%3d BK=%3d S=%d E=%2d  %2d x %4dx%4dx%5d  %.4f ms  %7.1f int8 TOP/s\n",
           name, L, BN, BK, STAGES, EPI, batch, M, N, K, ms, ops / ms / 1e9);
    cudaFree(dt);
}

int main() {
    size_t plane_max = (size_t)4 * 4096 * 8192;
    int8_t *A, *B; uint32_t* out;
    CK(cudaMalloc(&A, plane_max)); CK(cudaMalloc(&B, plane_max)); CK(cudaMalloc(&out, (size_t)4096 * 4096 * 4));
    std::vector<int8_t> h(plane_max);
    for (auto& x : h) x = (int8_t)(rand() & 255);
    CK(cudaMemcpy(A, h.data(), plane_max, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(B, h.data(), plane_max, cudaMemcpyHostToDevice));
    // pipeline depth / epilogue width study on the cfg2 recursion shapes and square products
    for (int K : {512, 2048}) {
        run<3, 96, 128, 2, 8>("L3 sq", 4096, 4096, K, 1, A, B, out, 20);
        run<3, 96, 64, 4, 8>("L3 sq", 4096, 4096, K, 1, A, B, out, 20);
        run<3, 96, 64, 5, 8>("L3 sq", 4096, 4096, K, 1, A, B, out, 20);
        run<3, 96, 128, 2, 12>("L3 sq", 4096, 4096, K, 1, A, B, out, 20);
        run<3, 96, 64, 4, 12>("L3 sq", 4096, 4096, K, 1, A, B, out, 20);
        run<3, 96, 64, 5, 12>("L3 sq", 4096, 4096, K, 1, A, B, out, 20);
    }
    run<3, 96, 128, 2, 8>("cfg2 depth0", 2048, 2048, 2048, 2, A, B, out, 20);
    run<3, 96, 64, 5, 12>("cfg2 depth0", 2048, 2048, 2048, 2, A, B, out, 20);
    run<3, 96, 128, 2, 8>("cfg2 depth2", 512, 512, 512, 18, A, B, out, 20);
    run<3, 96, 64, 4, 12>("cfg2 depth2", 512, 512, 512, 18, A, B, out, 20);
    run<3, 96, 64, 5, 12>("cfg2 depth2", 512, 512, 512, 18, A, B, out, 20);
    run<2, 128, 64, 6, 8>("L2 sq", 4096, 4096, 2048, 1, A, B, out, 20);
    run<2, 128, 128, 3, 8>("L2 sq", 4096, 4096, 2048, 1, A, B, out, 20);
    run<4, 64, 64, 4, 8>("L4 sq", 4096, 4096, 2048, 1, A, B, out, 20);
    run<4, 64, 128, 2, 8>("L4 sq", 4096, 4096, 2048, 1, A, B, out, 20);
    return 0;
}
