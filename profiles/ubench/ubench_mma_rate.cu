#include <string>
// Microbenchmark: raw tcgen05.mma.kind::i8 issue rate with operands resident in shared
// memory (no TMA, no epilogue) -- how the per-SM int8 MAC rate depends on the tile width N,
// the swizzle/K-block (BK), the number of accumulators the MMAs rotate over, and 1-CTA
// (M = 128) vs CTA-pair (cta_group::2, M = 256) issue.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I../../paper_2001_04109_b200/csrc ubench_mma_rate.cu -o ubench_mma_rate
// Prints one line per variant: cycles per MMA instruction and int8 MACs / clock / SM.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace fsyrk_b200;

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e = (x);                                                                      \
        if (e != cudaSuccess) {                                                                   \
            printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                          \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N, int BK, int NACC, bool PAIR, int TCOLS = 512, bool SIGNED = false>
__global__ void __launch_bounds__(128) mma_rate(int reps, unsigned long long* cycles) {
    constexpr int BROWS = PAIR ? N / 2 : N;  // B rows held by this CTA
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem;                   // 128 x BK
    uint8_t* B = smem + 128 * BK;        // BROWS x BK
    uint64_t* bar = reinterpret_cast<uint64_t*>(B + ((BROWS * BK + 1023) / 1024) * 1024);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    for (int i = threadIdx.x; i < (128 + BROWS) * BK / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = (uint32_t)(i * 2654435761u) & 0x3f3f3f3fu;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        if (PAIR)
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm100::smem_u32(slot)), "n"(TCOLS)
                         : "memory");
        else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm100::smem_u32(slot)), "n"(TCOLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    if (threadIdx.x == 32) {
        sm100::mbar_init(bar, 1);
        sm100::fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    sm100::tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();
    sm100::tc_fence_after();
    const uint32_t tmem = *slot;
    const bool leader = !PAIR || cluster_rank() == 0;
    if (threadIdx.x == 0 && leader) {
        const int layout = BK == 128 ? 2 : 4;
        const uint64_t ad = sm100::sdesc_kmajor(sm100::smem_u32(A), layout, 8 * BK);
        const uint64_t bd = sm100::sdesc_kmajor(sm100::smem_u32(B), layout, 8 * BK);
        const uint32_t idesc = sm100::idesc_i8(PAIR ? 256 : 128, N, SIGNED);
        long long t0 = clock64();
        int q = 0;
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int kk = 0; kk < BK / 32; ++kk) {
                const uint32_t d = tmem + (uint32_t)(q * N);
                q = q + 1 == NACC ? 0 : q + 1;
                if (PAIR)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(1)
                        : "memory");
                else
                    sm100::mma_i8(d, ad + 2 * kk, bd + 2 * kk, idesc, 1);
            }
        }
        if (PAIR)
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    sm100::smem_u32(bar)),
                "h"((uint16_t)3)
                : "memory");
        else
            sm100::tc_commit(bar);
        sm100::mbar_wait(bar, 0);
        long long t1 = clock64();
        cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    } else if (PAIR && threadIdx.x == 0) {
        sm100::mbar_wait(bar, 0);  // the leader's commit arrives here too
        cycles[blockIdx.x] = 0;
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();
    if (warp == 0) {
        if (PAIR) {
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
        }
    }
}

template <int N, int BK, int NACC, bool PAIR, int TCOLS = 512, bool SIGNED = false>
void run(int grid) {
    constexpr int BROWS = PAIR ? N / 2 : N;
    const int smem = 1024 + 128 * BK + ((BROWS * BK + 1023) / 1024) * 1024 + 64;
    auto k = mma_rate<N, BK, NACC, PAIR, TCOLS, SIGNED>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* d;
    CK(cudaMalloc(&d, grid * sizeof(unsigned long long)));
    const int reps = 4096 / (BK / 32);  // 4096 MMAs per CTA
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    for (int it = 0; it < 3; ++it) CK(cudaLaunchKernelEx(&cfg, k, reps, d));
    CK(cudaDeviceSynchronize());
    unsigned long long* h = (unsigned long long*)malloc(grid * sizeof(unsigned long long));
    CK(cudaMemcpy(h, d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    double sum = 0;
    int cnt = 0;
    for (int i = 0; i < grid; ++i)
        if (h[i]) {
            sum += (double)h[i];
            ++cnt;
        }
    const double cyc = sum / cnt / (reps * (BK / 32));
    const double macs_per_sm = (double)(PAIR ? 256 : 128) * N * 32 / (PAIR ? 2 : 1);
    printf("N=%3d BK=%3d NACC=%d %-5s %s grid=%3d tmem=%3d : %7.1f cyc/MMA  %7.0f MAC/clk per CTA  (smem B/MAC %.4f)\n", N,
           BK, NACC, PAIR ? "pair" : "1cta", SIGNED ? "s8" : "u8", grid, TCOLS, cyc, macs_per_sm / cyc,
           (128.0 + (PAIR ? N / 2.0 : N)) / (128.0 * N));
    free(h);
    CK(cudaFree(d));
}

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "signed") {  // s8 x s8 vs u8 x u8 at the tile shapes in use
        for (int grid : {1, 148}) {
            run<128, 128, 3, false, 512, false>(grid);
            run<128, 128, 3, false, 512, true>(grid);
            run<160, 64, 3, false, 512, false>(grid);
            run<160, 64, 3, false, 512, true>(grid);
            run<96, 128, 5, false, 512, true>(grid);
        }
        return 0;
    }
    // two CTAs per SM (grid 296, 256 TMEM columns each): does the tensor pipe overlap two issuers?
    run<80, 64, 3, false, 256>(296);
    run<80, 64, 3, false, 256>(148);
    run<64, 128, 3, false, 256>(296);
    run<128, 64, 1, false, 256>(296);
    for (int grid : {1, 148}) {
        run<64, 128, 1, false>(grid);
        run<80, 64, 3, false>(grid);
        run<96, 128, 1, false>(grid);
        run<128, 128, 1, false>(grid);
        run<128, 64, 3, false>(grid);
        run<160, 64, 1, false>(grid);
        run<160, 64, 3, false>(grid);
        run<160, 128, 3, false>(grid);
        run<256, 128, 1, false>(grid);
        run<80, 64, 3, true>(grid < 2 ? 2 : grid);
        run<128, 64, 3, true>(grid < 2 ? 2 : grid);
        run<160, 64, 3, true>(grid < 2 ? 2 : grid);
        run<256, 128, 1, true>(grid < 2 ? 2 : grid);
    }
    return 0;
}
