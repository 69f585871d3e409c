// Host <-> device transfer microbenchmark for the e2e path: PCIe bandwidth from pinned
// memory (H2D, D2H, both directions at once) and the host-thread cost of narrowing the
// caller's uint64 residues to uint32 / packing them to b bits (and back), by thread count.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -O3,-march=native,-pthread
#include <cuda_runtime.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class F>
static double par(int T, size_t n, F f) {
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            size_t lo = n * t / T, hi = n * (t + 1) / T;
            f(lo, hi);
        });
    for (auto& x : th) x.join();
    return now() - t0;
}

static void pack17(const uint64_t* s, uint32_t* d, size_t lo, size_t hi) {
    // lo, hi multiples of 32: 32 values -> 17 words
    for (size_t g = lo; g < hi; g += 32) {
        uint32_t* o = d + g / 32 * 17;
        uint64_t acc = 0;
        int nb = 0, w = 0;
        for (int i = 0; i < 32; ++i) {
            acc |= (s[g + i] & 0x1ffff) << nb;
            nb += 17;
            if (nb >= 32) {
                o[w++] = (uint32_t)acc;
                acc >>= 32;
                nb -= 32;
            }
        }
    }
}

int main() {
    const size_t N = 64ull << 20;  // 64 Mi elements = 512 MB uint64
    uint64_t* h64;
    uint32_t* h32;
    cudaHostAlloc(&h64, N * 8, 0);
    cudaHostAlloc(&h32, N * 4, 0);
    std::vector<uint64_t> pageable(N);
    std::mt19937_64 r(1);
    for (size_t i = 0; i < N; ++i) pageable[i] = h64[i] = r() % 131071;
    void *d1, *d2;
    cudaMalloc(&d1, N * 8);
    cudaMalloc(&d2, N * 8);
    cudaStream_t s1, s2;
    cudaStreamCreate(&s1);
    cudaStreamCreate(&s2);
    const size_t B = 256ull << 20;
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        cudaMemcpyAsync(d1, h64, B, cudaMemcpyHostToDevice, s1);
        cudaStreamSynchronize(s1);
        double t1 = now();
        cudaMemcpyAsync(h64, d1, B, cudaMemcpyDeviceToHost, s1);
        cudaStreamSynchronize(s1);
        double t2 = now();
        cudaMemcpyAsync(d1, h64, B, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync((char*)h64 + B, d2, B, cudaMemcpyDeviceToHost, s2);
        cudaStreamSynchronize(s1);
        cudaStreamSynchronize(s2);
        double t3 = now();
        cudaMemcpy(d1, pageable.data(), B, cudaMemcpyHostToDevice);
        double t4 = now();
        printf("pcie 256MB: h2d %.1f GB/s  d2h %.1f GB/s  duplex %.1f GB/s total  pageable h2d %.1f GB/s\n",
               B / (t1 - t0) / 1e9, B / (t2 - t1) / 1e9, 2 * B / (t3 - t2) / 1e9, B / (t4 - t3) / 1e9);
    }
    unsigned hc = std::thread::hardware_concurrency();
    printf("hardware_concurrency %u\n", hc);
    for (int T : {1, 2, 4, 8, 16, 32, 64}) {
        if ((unsigned)T > hc) break;
        double tn = 1e9, tp = 1e9, tw = 1e9, tc = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            tn = std::min(tn, par(T, N, [&](size_t lo, size_t hi) {
                              const uint64_t* s = pageable.data();
                              for (size_t i = lo; i < hi; ++i) h32[i] = (uint32_t)s[i];
                          }));
            tp = std::min(tp, par(T, N / 32, [&](size_t lo, size_t hi) {
                              pack17(pageable.data(), h32, lo * 32, hi * 32);
                          }));
            tw = std::min(tw, par(T, N, [&](size_t lo, size_t hi) {
                              uint64_t* d = pageable.data();
                              for (size_t i = lo; i < hi; ++i) d[i] = h32[i];
                          }));
            tc = std::min(tc, par(T, N, [&](size_t lo, size_t hi) {
                              std::memcpy(h64 + lo, pageable.data() + lo, (hi - lo) * 8);
                          }));
        }
        printf("T=%2d  narrow u64->u32 %.1f GB/s(src)  pack17 %.1f GB/s(src)  widen u32->u64 %.1f GB/s(dst)  "
               "memcpy %.1f GB/s\n",
               T, N * 8 / tn / 1e9, N * 8 / tp / 1e9, N * 8 / tw / 1e9, N * 8 / tc / 1e9);
    }
    return 0;
}
