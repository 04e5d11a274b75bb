// Generalized SPD eigendecomposition on the device — the setup of the
// spectral caches (SURVEY §8 b "spectral_setup"; solvers.py:256-281 calls
// scipy.linalg.eigh(A, B), LAPACK dsygvd, on the host).  Off the iteration
// loop: B = L L^T (cuSOLVER potrf), the standard problem L^-1 A L^-T
// (cuSOLVER syevd), V = L^-T Y (cuBLAS trsm), then the reference's sign rule
// (solvers.py:203-208: each eigenvector's largest-magnitude component
// positive, first index on ties like np.argmax).  Eigenvalues ascending, V
// B-orthonormal, like dsygvd.
//
// cuSOLVER / cuBLAS are resolved at run time (dlopen by soname), so the
// library reuses the copies the host process already loaded (e.g. PyTorch's)
// instead of pinning a second version into the process.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <mutex>
#include <string>

#include "sfb_common.cuh"
#include "sfb_kernels.cuh"

namespace sfb {
namespace {

struct DnApi {
    decltype(&cusolverDnCreate) create = nullptr;
    decltype(&cusolverDnDestroy) destroy = nullptr;
    decltype(&cusolverDnSetStream) set_stream = nullptr;
    decltype(&cusolverDnDpotrf_bufferSize) potrf_ws = nullptr;
    decltype(&cusolverDnDpotrf) potrf = nullptr;
    decltype(&cusolverDnDsyevd_bufferSize) syevd_ws = nullptr;
    decltype(&cusolverDnDsyevd) syevd = nullptr;
    decltype(&cublasCreate_v2) bcreate = nullptr;
    decltype(&cublasDestroy_v2) bdestroy = nullptr;
    decltype(&cublasSetStream_v2) bset_stream = nullptr;
    decltype(&cublasDtrsm_v2) trsm = nullptr;
    bool ok = false;
    std::string why;
};

void* open_lib(const char* soname, const char* fallback) {
    void* h = dlopen(soname, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen(fallback, RTLD_NOW | RTLD_GLOBAL);
    return h;
}

const DnApi& api() {
    static DnApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* blas = open_lib("libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so.12");
        void* dn = open_lib("libcusolver.so.11", "/usr/local/cuda/lib64/libcusolver.so.11");
        if (!blas || !dn) {
            a.why = "cuSOLVER / cuBLAS shared libraries not found";
            return;
        }
#define SFB_SYM(lib, field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(lib, name))
        SFB_SYM(dn, create, "cusolverDnCreate");
        SFB_SYM(dn, destroy, "cusolverDnDestroy");
        SFB_SYM(dn, set_stream, "cusolverDnSetStream");
        SFB_SYM(dn, potrf_ws, "cusolverDnDpotrf_bufferSize");
        SFB_SYM(dn, potrf, "cusolverDnDpotrf");
        SFB_SYM(dn, syevd_ws, "cusolverDnDsyevd_bufferSize");
        SFB_SYM(dn, syevd, "cusolverDnDsyevd");
        SFB_SYM(blas, bcreate, "cublasCreate_v2");
        SFB_SYM(blas, bdestroy, "cublasDestroy_v2");
        SFB_SYM(blas, bset_stream, "cublasSetStream_v2");
        SFB_SYM(blas, trsm, "cublasDtrsm_v2");
#undef SFB_SYM
        a.ok = a.create && a.destroy && a.set_stream && a.potrf_ws && a.potrf && a.syevd_ws && a.syevd && a.bcreate &&
               a.bdestroy && a.bset_stream && a.trsm;
        if (!a.ok) a.why = "cuSOLVER / cuBLAS entry points missing";
    });
    return a;
}

// X = 0.5 (X + X^T) in place, q x q contiguous
__global__ void symmetrize_kernel(double* X, int q) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (j < q && j > i) {
        const double v = 0.5 * (X[(size_t)i * q + j] + X[(size_t)j * q + i]);
        X[(size_t)i * q + j] = v;
        X[(size_t)j * q + i] = v;
    }
}

// column-major V (ld q): each column's largest-magnitude entry made positive
// (first index on ties, like np.argmax; a zero column keeps its sign)
__global__ void sign_fix_kernel(double* V, int q) {
    const int j = blockIdx.x;
    double* col = V + (size_t)j * q;
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < q; i += blockDim.x) {
        const double a = fabs(col[i]);
        if (a > best) {  // strictly greater: keeps the first index within the thread
            best = a;
            bi = i;
        }
    }
    __shared__ double sb[256];
    __shared__ int si[256];
    sb[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            const double b2 = sb[threadIdx.x + o];
            const int i2 = si[threadIdx.x + o];
            if (b2 > sb[threadIdx.x] || (b2 == sb[threadIdx.x] && i2 < si[threadIdx.x])) {
                sb[threadIdx.x] = b2;
                si[threadIdx.x] = i2;
            }
        }
        __syncthreads();
    }
    const int idx = si[0];
    const double s = (idx < q && col[idx] < 0.0) ? -1.0 : 1.0;
    if (s < 0.0)
        for (int i = threadIdx.x; i < q; i += blockDim.x) col[i] = -col[i];
}

struct DevScratch {
    void* p = nullptr;
    ~DevScratch() { cudaFree(p); }
};

}  // namespace
}  // namespace sfb

extern "C" int sfb_geigh(int q, const double* A, int lda, const double* B, int ldb, double* lam_host, double* V,
                         int ldv, void* stream) {
    SFB_NVTX("sfb_geigh");
    using namespace sfb;
    if (q <= 0 || !A || !B || !lam_host || !V || lda < q || ldb < q || ldv < q) return arg_error("geigh: bad arguments");
    const DnApi& L = api();
    if (!L.ok) {
        set_error(L.why);
        return SFB_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const size_t qq = (size_t)q * q;
    DevScratch mem;
    SFB_CUDA_TRY(cudaMalloc(&mem.p, (2 * qq + q) * 8 + 64));
    double* a = static_cast<double*>(mem.p);
    double* b = a + qq;
    double* w = b + qq;
    int* info = reinterpret_cast<int*>(w + q);
    // symmetric inputs: the row-major arrays are their own column-major images
    SFB_CUDA_TRY(cudaMemcpy2DAsync(a, (size_t)q * 8, A, (size_t)lda * 8, (size_t)q * 8, q, cudaMemcpyDefault, s));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(b, (size_t)q * 8, B, (size_t)ldb * 8, (size_t)q * 8, q, cudaMemcpyDefault, s));
    const dim3 sg((q + 127) / 128, q);
    symmetrize_kernel<<<sg, 128, 0, s>>>(b, q);
    SFB_CHECK_LAUNCH();
    cusolverDnHandle_t dn = nullptr;
    cublasHandle_t bl = nullptr;
    if (L.create(&dn) != CUSOLVER_STATUS_SUCCESS || L.bcreate(&bl) != CUBLAS_STATUS_SUCCESS) {
        if (dn) L.destroy(dn);
        set_error("geigh: creating cuSOLVER / cuBLAS handles failed");
        return SFB_ERR_CUDA;
    }
    int rc = SFB_OK;
    DevScratch work;
    auto lib_fail = [&](const char* what) {
        set_error(std::string("geigh: ") + what + " failed");
        rc = SFB_ERR_CUDA;
    };
    do {
        if (L.set_stream(dn, s) != CUSOLVER_STATUS_SUCCESS || L.bset_stream(bl, s) != CUBLAS_STATUS_SUCCESS) {
            lib_fail("stream binding");
            break;
        }
        int lw1 = 0, lw2 = 0;
        if (L.potrf_ws(dn, CUBLAS_FILL_MODE_LOWER, q, b, q, &lw1) != CUSOLVER_STATUS_SUCCESS ||
            L.syevd_ws(dn, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, q, a, q, w, &lw2) !=
                CUSOLVER_STATUS_SUCCESS) {
            lib_fail("workspace query");
            break;
        }
        const int lw = lw1 > lw2 ? lw1 : lw2;
        if (cudaMalloc(&work.p, (size_t)lw * 8 + 8) != cudaSuccess) {
            set_error("geigh: workspace allocation failed");
            rc = SFB_ERR_NOMEM;
            break;
        }
        double* ws = static_cast<double*>(work.p);
        // B = L L^T
        if (L.potrf(dn, CUBLAS_FILL_MODE_LOWER, q, b, q, ws, lw, info) != CUSOLVER_STATUS_SUCCESS) {
            lib_fail("potrf");
            break;
        }
        int hinfo = 0;
        if (cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            lib_fail("potrf status");
            break;
        }
        if (hinfo != 0) {  // the caller retries with the other term order (solvers.py:267-281)
            set_error("geigh: the second matrix of the pencil is not positive definite");
            rc = SFB_ERR_ARG;
            break;
        }
        const double one = 1.0;
        // M = L^-1 A L^-T
        if (L.trsm(bl, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, q, q, &one, b, q,
                   a, q) != CUBLAS_STATUS_SUCCESS ||
            L.trsm(bl, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, q, q, &one, b,
                   q, a, q) != CUBLAS_STATUS_SUCCESS) {
            lib_fail("trsm");
            break;
        }
        symmetrize_kernel<<<sg, 128, 0, s>>>(a, q);
        if (cudaGetLastError() != cudaSuccess) {
            lib_fail("symmetrize");
            break;
        }
        if (L.syevd(dn, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, q, a, q, w, ws, lw, info) !=
            CUSOLVER_STATUS_SUCCESS) {
            lib_fail("syevd");
            break;
        }
        // V = L^-T Y
        if (L.trsm(bl, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, q, q, &one, b, q,
                   a, q) != CUBLAS_STATUS_SUCCESS) {
            lib_fail("trsm");
            break;
        }
        sign_fix_kernel<<<q, 256, 0, s>>>(a, q);
        if (cudaGetLastError() != cudaSuccess) {
            lib_fail("sign fix");
            break;
        }
        // column-major eigenvectors -> row-major V[i][j] = component i of eigenvector j
        rc = launch_transpose(a, q, V, ldv, q, q, s);
        if (rc != SFB_OK) break;
        if (cudaMemcpyAsync(lam_host, w, (size_t)q * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            lib_fail("result copy");
            break;
        }
        if (hinfo != 0) {
            set_error("geigh: syevd did not converge");
            rc = SFB_ERR_CUDA;
        }
    } while (false);
    L.bdestroy(bl);
    L.destroy(dn);
    return rc;
}
