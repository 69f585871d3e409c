// Programmatic dependent launch: every kernel of a call is launched with programmatic
// stream serialization, starts with griddepcontrol.wait (nothing it reads or writes is
// touched before the previous kernel's results are visible) and lets the next kernel's
// launch begin early (griddepcontrol.launch_dependents), so launch latency and block
// scheduling overlap the previous kernel's tail instead of idling between kernels.
// FSYRK_B200_NO_PDL=1 turns the launch attribute off (plain stream order).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace fsyrk_b200 {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifndef FSYRK_PDL_TRIGGER
#define FSYRK_PDL_TRIGGER 1  // early trigger in the elementwise kernels
#endif
#ifndef FSYRK_PDL_TRIGGER_MM
#define FSYRK_PDL_TRIGGER_MM 0  // early trigger in the product kernel: measured +0.3 ms on cfg5 (off)
#endif
__device__ __forceinline__ void pdl_trigger() {
#if FSYRK_PDL_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger_mm() {
#if FSYRK_PDL_TRIGGER_MM
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

inline bool pdl_enabled() {
    static const bool on = std::getenv("FSYRK_B200_NO_PDL") == nullptr;
    return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace fsyrk_b200
