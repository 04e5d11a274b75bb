// Sparse matrix-vector product for the Kronecker (vector) cross-check path
// (SURVEY §8 f4): y = K x with K in CSR, the assembled vec-form matrix of
// operators.py:141-155 (to_kronecker) as used by vector_pcg
// (solvers.py:456-517, `w = K @ q`).
//
// Rows have ~T (2b+1)^2 nonzeros (25-125); eight lanes share a row (strided
// over its nonzeros, then a shuffle tree), four rows per warp.  The sum order
// is fixed, so repeated products are bit-identical.
#include <algorithm>

#include "sfb_common.cuh"
#include "sfb_kernels.cuh"
#include "sfb_launch.cuh"

namespace sfb {

namespace {

constexpr int LANES = 8;   // lanes per row
constexpr int CT = 256;    // threads per CTA

__global__ void __launch_bounds__(CT) csr_spmv_kernel(int n, const long long* __restrict__ indptr,
                                                      const int* __restrict__ indices,
                                                      const double* __restrict__ data,
                                                      const double* __restrict__ x, double* __restrict__ y) {
    SFB_PDL_PROLOGUE();
    const int sub = threadIdx.x % LANES;
    // the loop bound is uniform per warp (rows r0 .. r0+3 of this warp), so
    // every lane reaches the shuffles
    const long long warps = (long long)gridDim.x * (CT / 32);
    const long long wid = (long long)blockIdx.x * (CT / 32) + threadIdx.x / 32;
    for (long long r0 = wid * (32 / LANES); r0 < n; r0 += warps * (32 / LANES)) {
        const long long row = r0 + (threadIdx.x % 32) / LANES;
        double v = 0.0;
        if (row < n) {
            const long long b = indptr[row], e = indptr[row + 1];
            for (long long k = b + sub; k < e; k += LANES) v = fma(data[k], x[indices[k]], v);
        }
        #pragma unroll
        for (int o = LANES / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (sub == 0 && row < n) y[row] = v;
    }
}

}  // namespace

int launch_csr_spmv(int n, const long long* indptr, const int* indices, const double* data, const double* x,
                    double* y, cudaStream_t s) {
    if (n <= 0) return SFB_OK;
    const long long rows_per_cta = CT / LANES;
    const int grid = (int)std::min<long long>((n + rows_per_cta - 1) / rows_per_cta, 32LL * kNumSMs);
    SFB_TRY(launch_kernel(csr_spmv_kernel, dim3(grid), dim3(CT), 0, s, n, indptr, indices, data, x, y));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

}  // namespace sfb
