// FP64 tensor-core GEMM for sm_100a: C = A * Bt^T with fused epilogues.
//
// Replaces the dense numpy GEMM chains of the reference:
//   solvers.py:292      U = P1 @ (K * (P1.T @ rhs @ P2)) @ P2.T   (reduced solve)
//   solvers.py:134-143  Z = P_L^-1 R P_R^-1                         (preconditioner)
//   operators.py:130    out += G @ U @ H  (only for factors too wide for the
//                                          banded kernel)
//
// sm_100a has no FP64 tcgen05 kind, so the FP64 tensor path is the warp-level
// DMMA.8x8x4 (mma.sync m8n8k4 f64).  Tiles are staged by TMA
// (cp.async.bulk.tensor, SWIZZLE_128B) into a 4-stage shared-memory ring
// guarded by mbarriers; one thread issues the copies three k-tiles ahead and
// all eight warps (two per SM sub-partition, 255-register budget) issue DMMA.
// Both operands are K-contiguous ("NT"), which lets every fragment load be a
// conflict-free LDS.128: thread t of a quad owns the
// physical k = 4t+s for mma step s, so A[row][4t..4t+3] and Bt[col][4t..4t+3]
// are two 16-byte chunks per 128-byte row.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "sfb_common.cuh"
#include "sfb_kernels.cuh"

namespace sfb {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4;
constexpr int NWARPS = 8;                   // 2 x 4 warp grid, 64 x 32 per warp
constexpr int NTHREADS = NWARPS * 32;       // 2 warps per SM sub-partition (<= 255 regs each)
constexpr int TILE_BYTES = BM * BK * 8;     // 16 KB per operand per stage
constexpr int SMEM_BYTES = 2 * STAGES * TILE_BYTES + STAGES * 8 + 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(NTHREADS, 1)
    dgemm_nt_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    int M, int N, int K, GemmEpi ep) {
    if (ep.pcg != nullptr && ep.pcg->status != SFB_PCG_RUNNING) return;  // uniform gate

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * TILE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * STAGES * TILE_BYTES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int KT = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        // prologue: fill STAGES-1 slots
        for (int kt = 0; kt < STAGES - 1 && kt < KT; ++kt) {
            mbar_expect_tx(&full[kt], 2 * TILE_BYTES);
            tma_load_2d(sA + kt * TILE_BYTES, &tmA, &full[kt], kt * BK, m0);
            tma_load_2d(sB + kt * TILE_BYTES, &tmB, &full[kt], kt * BK, n0);
        }
    }
    __syncthreads();

    double acc[8][4][2];
    #pragma unroll
    for (int i = 0; i < 8; ++i)
        #pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int wm = warp >> 2, wn = warp & 3;  // consumer warp grid 2 x 4 (64 x 32 each)
    const int g = lane >> 2, t = lane & 3;

    // One thread issues TMA for k-tile kt+STAGES-1 into the slot consumed at
    // kt-1; the block barrier at the top of each step guarantees every warp
    // has finished reading that slot (WAR), the mbarrier signals the bytes.
    for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        __syncthreads();
        if (threadIdx.x == 0) {
            const int kn = kt + STAGES - 1;
            if (kn < KT) {
                const int sn = kn % STAGES;
                mbar_expect_tx(&full[sn], 2 * TILE_BYTES);
                tma_load_2d(sA + sn * TILE_BYTES, &tmA, &full[sn], kn * BK, m0);
                tma_load_2d(sB + sn * TILE_BYTES, &tmB, &full[sn], kn * BK, n0);
            }
        }
        mbar_wait(&full[s], (kt / STAGES) & 1);
        const uint8_t* a_base = sA + s * TILE_BYTES + (wm * 64 + g) * 128;
        const uint8_t* b_base = sB + s * TILE_BYTES + (wn * 32 + g) * 128;
        #pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int chunk = ((2 * t + half) ^ g) << 4;  // SWIZZLE_128B: chunk ^= row & 7 (= g)
            double2 a[8], b[4];
            #pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const double2*>(a_base + i * 8 * 128 + chunk);
            #pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const double2*>(b_base + j * 8 * 128 + chunk);
            #pragma unroll
            for (int i = 0; i < 8; ++i)
                #pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
            #pragma unroll
            for (int i = 0; i < 8; ++i)
                #pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
        }
    }

    // ---------------- epilogue (registers -> global) ----------------
    double dot = 0.0;
    {
        #pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int m = m0 + wm * 64 + i * 8 + g;
            if (m >= M) continue;
            #pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = n0 + wn * 32 + j * 8 + 2 * t;
                double v0 = acc[i][j][0], v1 = acc[i][j][1];
                const bool ok0 = n < N, ok1 = n + 1 < N;
                switch (ep.mode) {
                    case EPI_STORE_T:
                        if (ok0) ep.C[(size_t)n * ep.ldc + m] = v0;
                        if (ok1) ep.C[(size_t)(n + 1) * ep.ldc + m] = v1;
                        break;
                    case EPI_ACCUM:
                        if (ok0) ep.C[(size_t)m * ep.ldc + n] += v0;
                        if (ok1) ep.C[(size_t)m * ep.ldc + n + 1] += v1;
                        break;
                    default: {
                        if (ep.mode == EPI_HADAMARD_SUM) {
                            if (ok0) v0 *= 1.0 / (ep.sr[m] + ep.sc[n]);
                            if (ok1) v1 *= 1.0 / (ep.sr[m] + ep.sc[n + 1]);
                        } else if (ep.mode == EPI_HADAMARD_PROD) {
                            if (ok0) v0 *= ep.sr[m] * ep.sc[n];
                            if (ok1) v1 *= ep.sr[m] * ep.sc[n + 1];
                        }
                        double* c = ep.C + (size_t)m * ep.ldc + n;
                        if (ok1) {
                            *reinterpret_cast<double2*>(c) = make_double2(v0, v1);
                        } else if (ok0) {
                            c[0] = v0;
                        }
                        if (ep.mode == EPI_STORE_DOT) {
                            const double* d = ep.D + (size_t)m * ep.ldd + n;
                            if (ok0) dot = fma(v0, d[0], dot);
                            if (ok1) dot = fma(v1, d[1], dot);
                        }
                    }
                }
            }
        }
    }
    if (ep.mode == EPI_STORE_DOT) {
        __shared__ double sh[NTHREADS / 32];
        const double part = block_sum<NTHREADS>(dot, sh);
        const unsigned nblk = gridDim.x * gridDim.y;
        if (threadIdx.x == 0) ep.partials[blockIdx.y * gridDim.x + blockIdx.x] = part;
        if (arrive_last(ep.counter, nblk)) {
            const double tot = sum_partials<NTHREADS>(ep.partials, nblk, 1, sh);
            if (threadIdx.x == 0) {
                *ep.counter = 0;
                if (ep.pcg != nullptr) ep.pcg->rz_next = tot;
                if (ep.dot_out != nullptr) *ep.dot_out = tot;
            }
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (fn == nullptr) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

int make_map(CUtensorMap* map, const double* ptr, int rows, int cols, int ld) {
    auto fn = encode_fn();
    if (fn == nullptr) {
        set_error("cuTensorMapEncodeTiled entry point unavailable");
        return SFB_ERR_CUDA;
    }
    if ((ld % 2) != 0 || (reinterpret_cast<uintptr_t>(ptr) % 16) != 0)
        return arg_error("DMMA GEMM operands need 16-byte aligned rows (even leading dimension)");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
    cuuint32_t box[2] = {BK, BM};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box,
                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
        return SFB_ERR_CUDA;
    }
    return SFB_OK;
}

}  // namespace

int gemm_smem_bytes() { return SMEM_BYTES; }

// C[M x N] = A[M x K] * Bt[N x K]^T, both row-major K-contiguous.
int launch_dgemm_nt(const double* A, int lda, const double* Bt, int ldb, int M, int N, int K,
                    const GemmEpi& ep, cudaStream_t stream) {
    static bool attr_set = false;
    if (!attr_set) {
        SFB_CUDA_TRY(cudaFuncSetAttribute(dgemm_nt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          SMEM_BYTES));
        attr_set = true;
    }
    if (M <= 0 || N <= 0 || K <= 0) return arg_error("empty GEMM");
    CUtensorMap ma, mb;
    SFB_TRY(make_map(&ma, A, M, K, lda));
    SFB_TRY(make_map(&mb, Bt, N, K, ldb));
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
    dgemm_nt_kernel<<<grid, NTHREADS, SMEM_BYTES, stream>>>(ma, mb, M, N, K, ep);
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int gemm_grid_blocks(int M, int N) { return ((N + BN - 1) / BN) * ((M + BM - 1) / BM); }

}  // namespace sfb
