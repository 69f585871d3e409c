// Microbenchmark: the FP64 route north_star names as the alternative to int8 digit planes.
//
// Exact mod-p products in FP64 need K_c * (p - 1)^2 < 2^53 per K chunk (delayed reduction,
// SURVEY App. B): one FP64 FMA per modular MAC.  sm_100a has no tcgen05 FP64 kind, so the FP64
// tensor path is the warp-level DMMA (mma.sync.aligned.m16n8k4 .f64).  This measures its peak
// issue rate with operands in registers (no memory traffic at all, i.e. an upper bound for any
// FP64 kernel), and the plain FP64 FMA pipe for comparison, and prints the exact modular MAC
// rate each route could reach next to the int8 schemes' ceilings.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_dmma.cu -o ubench_dmma
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);       \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

// NACC independent m16n8k4 accumulators per warp (hides the DMMA latency)
template <int NACC>
__global__ void dmma_rate(int reps, double* sink) {
    double a = 1.0 + threadIdx.x * 1e-3, b = 2.0 - threadIdx.x * 1e-3;
    double c[NACC][4];  // m16n8k4 f64 fragments: A 2, B 1, C / D 4 doubles per thread
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < NACC; ++i)
            asm volatile(
                "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
                : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                : "d"(a), "d"(b), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) sink[threadIdx.x] = s;
}

template <int NACC>
__global__ void ffma64_rate(int reps, double* sink) {
    double a = 1.0 + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-9;
    double c[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = i;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i];
    if (s == 12345.678) sink[threadIdx.x] = s;
}

template <class K>
float time_kernel(K kern, int blocks, int threads, int reps, double* sink) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    kern<<<blocks, threads>>>(reps / 10, sink);  // warm-up
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(reps, sink);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms;
}

int main() {
    int dev = 0, nsm = 0, clk_khz = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    double* sink;
    CK(cudaMalloc(&sink, 1024 * sizeof(double)));
    const int reps = 20000;
    printf("SMs %d, max clock %.0f MHz\n", nsm, clk_khz / 1e3);
    double best = 0;
    for (int warps : {4, 8, 16}) {
        const int threads = 32 * warps, blocks = nsm;
        const float ms = time_kernel(dmma_rate<8>, blocks, threads, reps, sink);
        // m16n8k4: 16 * 8 * 4 = 512 FMAs = 1024 flops per warp instruction
        const double flops = (double)blocks * warps * reps * 8 * 1024.0;
        const double tf = flops / (ms * 1e-3) / 1e12;
        best = tf > best ? tf : best;
        printf("DMMA m16n8k4 f64: %2d warps/SM x 8 accumulators: %.3f ms, %.2f TFLOP/s\n", warps, ms, tf);
    }
    for (int warps : {8, 32}) {
        const int threads = 32 * warps, blocks = nsm;
        const float ms = time_kernel(ffma64_rate<8>, blocks, threads, reps, sink);
        const double flops = (double)blocks * threads * reps * 8 * 2.0;
        printf("DFMA (CUDA cores):  %2d warps/SM x 8 chains:        %.3f ms, %.2f TFLOP/s\n", warps, ms,
               flops / (ms * 1e-3) / 1e12);
    }
    // exact modular MACs per second: FP64 = 1 FMA per MAC; int8 schemes = NT int8 MACs per MAC
    const double fp64_macs = best * 1e12 / 2;
    printf("\nexact mod-p MAC rate ceilings (products only)\n");
    printf("  FP64 DMMA (1 FMA / MAC, K chunk < 2^53 / (p-1)^2):  %.1f T MAC/s\n", fp64_macs / 1e12);
    const double i8_nominal = 16384.0 * nsm * (clk_khz * 1e3) / 2;  // int8 MAC/s (16384 ops / clk / SM)
    const struct { const char* name; int nt; } sch[] = {{"LIMB2 (p <= 2^16)", 4}, {"M17 (2^17 - 1)", 9},
                                                         {"LIMB3 (p <= 2^24)", 9}, {"LIMB4", 16}, {"M31 (2^31 - 1)", 17}};
    for (auto& s : sch)
        printf("  int8 tcgen05 %-18s (%2d MMAs / MAC):     %.1f T MAC/s nominal (%.1fx FP64)\n", s.name, s.nt,
               i8_nominal / s.nt / 1e12, i8_nominal / s.nt / fp64_macs);
    return 0;
}
