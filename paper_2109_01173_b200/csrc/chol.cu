// Banded SPD preconditioner solves:  Z = P_L^-1 X P_R^-1.
//
// Same operator as the reference's LU solves (solvers.py:134-143): both
// factors are banded SPD (half-bandwidth <= k), so a banded
// Cholesky P = C C^T factorised once on the host turns every application into
// forward/backward substitutions costing O(q^2 k) instead of the dense
// O(q^3).  Band storage: band[i][d] = C[i][i - b + d] for d < b, and
// band[i][b] = 1 / C[i][i] (reciprocal diagonal, so the sweep multiplies).
//
//  * left factor  : independent systems per column j; one thread per column
//                   marches down the rows (warp accesses are row-contiguous).
//  * right factor : independent systems per row i; a warp owns 32 rows and
//                   streams 32-column tiles through padded shared memory so
//                   global accesses stay coalesced while each lane sweeps
//                   its own row.
#include "sfb_common.cuh"
#include "sfb_kernels.cuh"

namespace sfb {

namespace {

template <int B>
__global__ void __launch_bounds__(128) chol_cols_kernel(const double* __restrict__ band, int n,
                                                        const double* __restrict__ Xin, int ldi,
                                                        double* __restrict__ X, int ld, int ncols,
                                                        const PcgState* st) {
    if (st != nullptr && st->status != SFB_PCG_RUNNING) return;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ncols) return;
    double w[B > 0 ? B : 1];
    #pragma unroll
    for (int d = 0; d < B; ++d) w[d] = 0.0;
    // forward: C y = x
    #pragma unroll 4
    for (int i = 0; i < n; ++i) {
        const double* c = band + (size_t)i * (B + 1);
        double v = Xin[(size_t)i * ldi + j];
        #pragma unroll
        for (int d = 0; d < B; ++d) v = fma(-c[d], w[d], v);  // w[d] = y[i-B+d]
        v *= c[B];
        #pragma unroll
        for (int d = 0; d + 1 < B; ++d) w[d] = w[d + 1];
        if (B > 0) w[B - 1] = v;
        X[(size_t)i * ld + j] = v;
    }
    // backward: C^T z = y
    #pragma unroll
    for (int d = 0; d < B; ++d) w[d] = 0.0;  // w[e-1] = z[i+e]
    #pragma unroll 4
    for (int i = n - 1; i >= 0; --i) {
        double v = X[(size_t)i * ld + j];
        #pragma unroll
        for (int e = B; e >= 1; --e) {
            if (i + e < n) v = fma(-band[(size_t)(i + e) * (B + 1) + B - e], w[e - 1], v);
        }
        v *= band[(size_t)i * (B + 1) + B];
        #pragma unroll
        for (int e = B - 1; e >= 1; --e) w[e] = w[e - 1];
        if (B > 0) w[0] = v;
        X[(size_t)i * ld + j] = v;
    }
}

constexpr int RT = 32;  // rows per warp / tile width

template <int B>
__global__ void __launch_bounds__(32) chol_rows_kernel(const double* __restrict__ band, int n,
                                                       double* __restrict__ X, int ld, int nrows,
                                                       ZrDot zr) {
    if (zr.pcg != nullptr && zr.pcg->status != SFB_PCG_RUNNING) return;
    __shared__ double tile[RT][RT + 1];
    double dot = 0.0;
    const int lane = threadIdx.x;
    const int i0 = blockIdx.x * RT;
    const int my_row = i0 + lane;
    double w[B > 0 ? B : 1];
    #pragma unroll
    for (int d = 0; d < B; ++d) w[d] = 0.0;
    const int nchunks = (n + RT - 1) / RT;
    // ---- forward along the row ----
    for (int ch = 0; ch < nchunks; ++ch) {
        const int j0 = ch * RT, jc = j0 + lane;
        #pragma unroll 8
        for (int r = 0; r < RT; ++r) {
            const int gi = i0 + r;
            tile[r][lane] = (gi < nrows && jc < n) ? X[(size_t)gi * ld + jc] : 0.0;
        }
        __syncwarp();
        const int jmax = min(RT, n - j0);
        for (int jj = 0; jj < jmax; ++jj) {
            const int j = j0 + jj;
            const double* c = band + (size_t)j * (B + 1);
            double v = tile[lane][jj];
            #pragma unroll
            for (int d = 0; d < B; ++d) v = fma(-c[d], w[d], v);
            v *= c[B];
            #pragma unroll
            for (int d = 0; d + 1 < B; ++d) w[d] = w[d + 1];
            if (B > 0) w[B - 1] = v;
            tile[lane][jj] = v;
        }
        __syncwarp();
        #pragma unroll 8
        for (int r = 0; r < RT; ++r) {
            const int gi = i0 + r;
            if (gi < nrows && jc < n) X[(size_t)gi * ld + jc] = tile[r][lane];
        }
        __syncwarp();
    }
    // ---- backward along the row ----
    #pragma unroll
    for (int d = 0; d < B; ++d) w[d] = 0.0;
    for (int ch = nchunks - 1; ch >= 0; --ch) {
        const int j0 = ch * RT, jc = j0 + lane;
        #pragma unroll 8
        for (int r = 0; r < RT; ++r) {
            const int gi = i0 + r;
            tile[r][lane] = (gi < nrows && jc < n) ? X[(size_t)gi * ld + jc] : 0.0;
        }
        __syncwarp();
        const int jmax = min(RT, n - j0);
        for (int jj = jmax - 1; jj >= 0; --jj) {
            const int j = j0 + jj;
            double v = tile[lane][jj];
            #pragma unroll
            for (int e = B; e >= 1; --e) {
                if (j + e < n) v = fma(-band[(size_t)(j + e) * (B + 1) + B - e], w[e - 1], v);
            }
            v *= band[(size_t)j * (B + 1) + B];
            #pragma unroll
            for (int e = B - 1; e >= 1; --e) w[e] = w[e - 1];
            if (B > 0) w[0] = v;
            tile[lane][jj] = v;
        }
        __syncwarp();
        #pragma unroll 8
        for (int r = 0; r < RT; ++r) {
            const int gi = i0 + r;
            if (gi < nrows && jc < n) {
                const double z = tile[r][lane];
                X[(size_t)gi * ld + jc] = z;
                if (zr.R != nullptr) dot = fma(z, zr.R[(size_t)gi * zr.ldr + jc], dot);
            }
        }
        __syncwarp();
    }
    (void)my_row;
    if (zr.R != nullptr) {  // <Z,R> for beta (solvers.py:448), deterministic
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (lane == 0) zr.partials[blockIdx.x] = dot;
        if (arrive_last(zr.counter, gridDim.x)) {
            double v = 0.0;
            for (unsigned i = lane; i < gridDim.x; i += 32) v += __ldcg(zr.partials + i);
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) {
                *zr.counter = 0;
                if (zr.pcg != nullptr) zr.pcg->rz_next = v;
                if (zr.dot_out != nullptr) *zr.dot_out = v;
            }
        }
    }
}

}  // namespace

int launch_band_chol_cols(const double* lband, int bw, int n, const double* Xin, int ldi, double* X, int ld,
                          int ncols, const PcgState* st, cudaStream_t s) {
    const dim3 grid((ncols + 127) / 128);
    switch (bw) {
        case 0: chol_cols_kernel<0><<<grid, 128, 0, s>>>(lband, n, Xin, ldi, X, ld, ncols, st); break;
        case 1: chol_cols_kernel<1><<<grid, 128, 0, s>>>(lband, n, Xin, ldi, X, ld, ncols, st); break;
        case 2: chol_cols_kernel<2><<<grid, 128, 0, s>>>(lband, n, Xin, ldi, X, ld, ncols, st); break;
        case 3: chol_cols_kernel<3><<<grid, 128, 0, s>>>(lband, n, Xin, ldi, X, ld, ncols, st); break;
        case 4: chol_cols_kernel<4><<<grid, 128, 0, s>>>(lband, n, Xin, ldi, X, ld, ncols, st); break;
        default: set_error("banded Cholesky: half-bandwidth > 4"); return SFB_ERR_UNSUPPORTED;
    }
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_band_chol_rows(const double* rband, int bw, int n, double* X, int ld, int nrows, const ZrDot& zr,
                          cudaStream_t s) {
    const dim3 grid((nrows + RT - 1) / RT);
    switch (bw) {
        case 0: chol_rows_kernel<0><<<grid, 32, 0, s>>>(rband, n, X, ld, nrows, zr); break;
        case 1: chol_rows_kernel<1><<<grid, 32, 0, s>>>(rband, n, X, ld, nrows, zr); break;
        case 2: chol_rows_kernel<2><<<grid, 32, 0, s>>>(rband, n, X, ld, nrows, zr); break;
        case 3: chol_rows_kernel<3><<<grid, 32, 0, s>>>(rband, n, X, ld, nrows, zr); break;
        case 4: chol_rows_kernel<4><<<grid, 32, 0, s>>>(rband, n, X, ld, nrows, zr); break;
        default: set_error("banded Cholesky: half-bandwidth > 4"); return SFB_ERR_UNSUPPORTED;
    }
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int band_chol_rows_blocks(int nrows) { return (nrows + RT - 1) / RT; }

}  // namespace sfb
