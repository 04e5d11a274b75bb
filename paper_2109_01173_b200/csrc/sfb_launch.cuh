// Kernel launches with programmatic dependent launch (PDL).
//
// Every kernel of the library starts with SFB_PDL_PROLOGUE(): it first lets
// the next kernel in the stream be scheduled (griddepcontrol.launch_dependents)
// and then waits until the previous kernel has completed and its writes are
// visible (griddepcontrol.wait).  Launched with the programmatic-serialization
// attribute, the launch latency of kernel N+1 overlaps the tail of kernel N —
// the MO-PCG iteration is a chain of 5-13 dependent kernels, so this removes
// most of the per-node gap inside the CUDA graph.  The dependent grid is only
// released once every CTA of the primary has started, so waiting CTAs can
// never starve the primary.  On by default (SYLFEM_B200_PDL=0 disables the
// launch attribute; the prologue is then a no-op).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_set>
#include <utility>

#include "sfb_common.cuh"

#define SFB_PDL_PROLOGUE()                                                  \
    do {                                                                    \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");     \
        asm volatile("griddepcontrol.wait;" ::: "memory");                  \
    } while (0)

namespace sfb {

inline bool pdl_enabled() {
    // on by default (measured: banded MO-PCG iteration -0.8 %, GEMM iteration
    // -0.3 %); SYLFEM_B200_PDL=0 turns it off (thread-safe one-time init)
    static const bool on = [] {
        const char* e = std::getenv("SYLFEM_B200_PDL");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    return on;
}

// One shared-memory carveout for every kernel of the library: consecutive
// kernels with different L1/shared splits force the SM to drain and
// reconfigure between launches; pinning the maximum shared carveout
// everywhere keeps dependent kernels back to back.  SYLFEM_B200_CARVEOUT=0
// leaves the driver default.
inline bool carveout_pinned() {
    static const bool on = [] {
        const char* e = std::getenv("SYLFEM_B200_CARVEOUT");  // opt-in: measured neutral
        return e && std::strcmp(e, "1") == 0;
    }();
    return on;
}

inline bool first_launch(const void* fn) {
    static std::mutex mu;
    static std::unordered_set<const void*> seen;
    std::lock_guard<std::mutex> lock(mu);
    return seen.insert(fn).second;
}

// Dynamic shared memory above 48 KB must be opted into per kernel and per
// device; the (kernel, device, bytes) triples already set are remembered
// (thread-safe, so several devices or threads in one process are fine).
template <typename... KArgs>
inline int ensure_dynamic_smem(void (*kernel)(KArgs...), size_t bytes) {
    if (bytes <= 48 * 1024) return SFB_OK;
    static std::mutex mu;
    static std::unordered_set<std::string> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const std::string key = std::to_string(reinterpret_cast<uintptr_t>(kernel)) + "/" + std::to_string(dev) + "/" +
                            std::to_string(bytes);
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return SFB_OK;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) {
        set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
        return SFB_ERR_CUDA;
    }
    done.insert(key);
    return SFB_OK;
}

template <typename... KArgs>
inline void pin_carveout(void (*kernel)(KArgs...)) {
    if (first_launch(reinterpret_cast<const void*>(kernel))) {
        // a hint only: its own failure is ignored without touching errors
        // pending from earlier asynchronous work
        if (carveout_pinned())
            (void)cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       (int)cudaSharedmemCarveoutMaxShared);
    }
}

template <typename... KArgs, typename... Args>
inline int launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                         Args&&... args) {
    pin_carveout(kernel);
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
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
    if (e != cudaSuccess) {
        set_error(std::string("kernel launch: ") + cudaGetErrorString(e));
        return SFB_ERR_CUDA;
    }
    return SFB_OK;
}

}  // namespace sfb
