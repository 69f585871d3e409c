// Per-device library state.
//
// Streams, events, device buffers and kernel attributes belong to the device that was current
// when they were made.  A process may drive several GPUs (the single-process multi-GPU entry
// point, or a caller switching devices between calls), so every such piece of state is kept
// once per device and looked up through the current device.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>

namespace fsyrk_b200 {

inline int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) {
        cudaGetLastError();
        d = 0;
    }
    return d;
}

// The T of the current device, created on first use (never destroyed before process exit).
template <class T>
T& per_device() {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<T>> by_dev;
    const int d = current_device();
    std::lock_guard<std::mutex> lk(mu);
    std::unique_ptr<T>& p = by_dev[d];
    if (!p) p.reset(new T);
    return *p;
}

// One-time per-device initialisation: fn() runs once per device, its result is kept.
struct DeviceOnce {
    std::once_flag flag;
    cudaError_t result = cudaSuccess;
};

}  // namespace fsyrk_b200
