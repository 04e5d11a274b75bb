// Shared device/host helpers of the sm_100a MO-FEM library.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/sylfem_b200.h"

#include <nvtx3/nvToolsExt.h>

namespace sfb {

// NVTX range over an entry point (SURVEY §5 tracing): named ranges in nsys /
// ncu timelines; header-only NVTX costs nothing without an attached tool.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define SFB_NVTX(name) ::sfb::NvtxRange sfb_nvtx_range_(name)

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);

#define SFB_CUDA_TRY(expr)                                                       \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) {                                                 \
            ::sfb::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
            return SFB_ERR_CUDA;                                                 \
        }                                                                        \
    } while (0)

#define SFB_CHECK_LAUNCH()                                                       \
    do {                                                                         \
        cudaError_t _e = cudaGetLastError();                                     \
        if (_e != cudaSuccess) {                                                 \
            ::sfb::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
            return SFB_ERR_CUDA;                                                 \
        }                                                                        \
    } while (0)

#define SFB_TRY(expr)                      \
    do {                                   \
        int _s = (expr);                   \
        if (_s != SFB_OK) return _s;       \
    } while (0)

inline int arg_error(const std::string& msg) {
    set_error(msg);
    return SFB_ERR_ARG;
}

constexpr int kNumSMs = 148;

// device allocation of n doubles (at least one), SFB_ERR_NOMEM on failure
inline int dalloc(double** p, size_t n) {
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(double));
    if (e != cudaSuccess) {
        set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
        return SFB_ERR_NOMEM;
    }
    return SFB_OK;
}

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// ------------------------------------------------- device scalar state ----
// State of one MO-PCG solve, resident on the device (solvers.py:391-453).
struct PcgState {
    int status;        // SFB_PCG_*
    int iter;          // completed iterations s
    int max_iter;
    int rule;          // SFB_RULE_*
    double value;      // stop threshold
    double res0;
    double rz;         // <Z,R> of the current direction
    double rz_next;    // <Z,R> produced by the last preconditioner apply
    double alpha;
    double qq;         // |Q|^2 of the current direction
    double bad_value;
    int bad_iter;
    int n_iterates;    // record_iterates capacity
    int recorded;      // last recorded iterate index (-1: none)
    unsigned counter[8];
};

// Generic reduction slots used outside MO-PCG.
struct RedSlots {
    double v[8];
    unsigned counter[4];
};

// -------------------------------------------------- block reductions ------
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0) {
        #pragma unroll
        for (int i = 0; i < NT / 32; ++i) r += sh[i];
    }
    return r;  // valid in thread 0
}

// Deterministic "last block finishes the reduction" pattern: every block
// publishes its partial(s) then increments a counter; the block that sees
// count == nblocks-1 sums all partials in fixed index order.
__device__ __forceinline__ bool arrive_last(unsigned* counter, unsigned nblocks) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned prev = atomicAdd(counter, 1u);
        s_last = (prev == nblocks - 1);
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

// Sum nparts partials (stride `stride` doubles apart) in a fixed order with
// the whole block; result valid in thread 0.
template <int NT>
__device__ __forceinline__ double sum_partials(const double* p, int nparts, int stride, double* sh) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nparts; i += NT) v += __ldcg(p + (size_t)i * stride);
    return block_sum<NT>(v, sh);
}

}  // namespace sfb
