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

// Sparse LU solve z = P^-1 r of a generic sparse preconditioner, factored
// once on the host as Pr P Pc = L U (SuperLU, like the reference's
// spla.splu(P).solve, solvers.py:473).  One CTA: y = Pr r, forward
// substitution with L level by level, backward substitution with U level by
// level (rows of one level are independent; a CTA barrier separates
// levels), z = Pc x.  Each row sums its entries in CSR order, so the solve
// is deterministic.  Meant for the cross-check sizes vector_pcg runs at.
constexpr int LU_T = 1024;

__device__ __forceinline__ void tri_level_sweep(const long long* __restrict__ ptr, const int* __restrict__ ind,
                                                const double* __restrict__ val, const int* __restrict__ lev_ptr,
                                                const int* __restrict__ lev_rows, int nlev, double* y) {
    for (int l = 0; l < nlev; ++l) {
        for (int k = lev_ptr[l] + threadIdx.x; k < lev_ptr[l + 1]; k += LU_T) {
            const int i = lev_rows[k];
            double s = y[i], d = 1.0;
            for (long long p = ptr[i]; p < ptr[i + 1]; ++p) {
                const int j = ind[p];
                if (j == i) d = val[p];
                else s = fma(-val[p], y[j], s);
            }
            y[i] = s / d;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(LU_T) lu_solve_kernel(int n, const long long* Lp, const int* Li, const double* Lv,
                                                       const int* Llp, const int* Llr, int nlL, const long long* Up,
                                                       const int* Ui, const double* Uv, const int* Ulp,
                                                       const int* Ulr, int nlU, const int* perm_r,
                                                       const int* perm_c, const double* r, double* z, double* y) {
    for (int i = threadIdx.x; i < n; i += LU_T) y[perm_r[i]] = r[i];  // Pr r
    __syncthreads();
    tri_level_sweep(Lp, Li, Lv, Llp, Llr, nlL, y);
    tri_level_sweep(Up, Ui, Uv, Ulp, Ulr, nlU, y);
    for (int i = threadIdx.x; i < n; i += LU_T) z[i] = y[perm_c[i]];  // Pc x: (Pc x)[i] = x[perm_c[i]]
}

}  // namespace

int launch_lu_solve(int n, const long long* Lp, const int* Li, const double* Lv, const int* Llp, const int* Llr,
                    int nlL, const long long* Up, const int* Ui, const double* Uv, const int* Ulp, const int* Ulr,
                    int nlU, const int* perm_r, const int* perm_c, const double* r, double* z, double* y,
                    cudaStream_t s) {
    lu_solve_kernel<<<1, LU_T, 0, s>>>(n, Lp, Li, Lv, Llp, Llr, nlL, Up, Ui, Uv, Ulp, Ulr, nlU, perm_r, perm_c, r,
                                       z, y);
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

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
