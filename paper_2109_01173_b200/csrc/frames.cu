// Trajectory frames as 16-bit PGM on the device: the
// min-max normalisation and quantisation of harness.write_pgm
// (harness.py:475-491) for snapshot-sized grids (an 8192^2 frame is 512 MB
// of fp64; only the 128 MB of big-endian uint16 pixels leave the GPU).
// Same arithmetic as the reference: scaled = rint((a - lo) / span * 65535)
// (round half to even, like np.round), frames that are constant up to
// roundoff (span <= max(1e-12 max(|hi|, |lo|), 1e-14)) map to zeros.
#include <cuda_runtime.h>

#include <cmath>

#include "sfb_common.cuh"
#include "sfb_launch.cuh"

namespace sfb {
namespace {

constexpr int FT = 256;

__device__ __forceinline__ double block_min(double v, double* sh) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = v;
    if (threadIdx.x == 0)
        for (int i = 0; i < FT / 32; ++i) r = fmin(r, sh[i]);
    return r;
}

__global__ void __launch_bounds__(FT) frame_minmax_kernel(const double* A, int lda, int rows, int cols,
                                                           double* partials, unsigned* counter, double* lohi) {
    SFB_PDL_PROLOGUE();
    double lo = INFINITY, hi = -INFINITY;
    const long long n = (long long)rows * cols;
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        const double a = A[(i / cols) * lda + i % cols];
        lo = fmin(lo, a);
        hi = fmax(hi, a);
    }
    __shared__ double sh[FT / 32];
    lo = block_min(lo, sh);
    hi = -block_min(-hi, sh);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = lo;
        partials[2 * blockIdx.x + 1] = hi;
    }
    if (arrive_last(counter, gridDim.x)) {
        double l2 = INFINITY, h2 = -INFINITY;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += FT) {
            l2 = fmin(l2, __ldcg(partials + 2 * b));
            h2 = fmax(h2, __ldcg(partials + 2 * b + 1));
        }
        l2 = block_min(l2, sh);
        h2 = -block_min(-h2, sh);
        if (threadIdx.x == 0) {
            *counter = 0;
            lohi[0] = l2;
            lohi[1] = h2;
        }
    }
}

__global__ void __launch_bounds__(FT) frame_quantize_kernel(const double* A, int lda, int rows, int cols,
                                                             const double* lohi, unsigned short* out) {
    SFB_PDL_PROLOGUE();
    const double lo = lohi[0], hi = lohi[1];
    const double span = hi - lo;
    const bool flat = !(span > fmax(1e-12 * fmax(fabs(hi), fabs(lo)), 1e-14));
    const long long n = (long long)rows * cols;
    for (long long i = (long long)blockIdx.x * FT + threadIdx.x; i < n; i += (long long)gridDim.x * FT) {
        unsigned short v = 0;
        if (!flat) {
            const double a = A[(i / cols) * lda + i % cols];
            v = (unsigned short)rint(__dmul_rn(__ddiv_rn(__dsub_rn(a, lo), span), 65535.0));
        }
        out[i] = (unsigned short)((v >> 8) | (v << 8));  // big-endian (">u2")
    }
}

}  // namespace
}  // namespace sfb

extern "C" int sfb_frame_pgm16(const double* A, int lda, int rows, int cols, unsigned short* out, double* lohi_host,
                               void* stream) {
    using namespace sfb;
    if (!A || !out || rows <= 0 || cols <= 0 || lda < cols) return arg_error("frame: bad array");
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = 4 * kNumSMs;
    double* ws = nullptr;
    SFB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ws), (2 * grid + 2) * 8 + 64, s));
    unsigned* counter = reinterpret_cast<unsigned*>(ws + 2 * grid + 2);
    double* lohi = ws + 2 * grid;
    int rc = SFB_OK;
    if (cudaMemsetAsync(counter, 0, 64, s) != cudaSuccess) rc = SFB_ERR_CUDA;
    if (rc == SFB_OK)
        rc = launch_kernel(frame_minmax_kernel, dim3(grid), dim3(FT), 0, s, A, lda, rows, cols, ws, counter, lohi);
    if (rc == SFB_OK)
        rc = launch_kernel(frame_quantize_kernel, dim3(grid), dim3(FT), 0, s, A, lda, rows, cols,
                           (const double*)lohi, out);
    if (rc == SFB_OK && lohi_host) {
        if (cudaMemcpyAsync(lohi_host, lohi, 16, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            rc = SFB_ERR_CUDA;
    }
    cudaFreeAsync(ws, s);
    if (rc == SFB_ERR_CUDA) set_error("frame: CUDA failure");
    return rc;
}
