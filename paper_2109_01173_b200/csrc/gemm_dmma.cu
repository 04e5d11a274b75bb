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
// (cp.async.bulk.tensor, SWIZZLE_128B, 16-wide k boxes) into a shared-memory
// ring guarded by full/empty mbarriers — 128 x 128 tiles: 3 stages of 32 k
// (two boxes per operand, 64 KB), two k-tiles ahead; 64 x 64 tiles: 5 stages
// of 16 k, three ahead — one thread issues the copies once the slot's empty
// barrier completes (every warp released it), and the warps (four per SM
// sub-partition for 128 x 128, 32 x 32 warp tiles, 128 registers) issue DMMA.
// Both operands are K-contiguous ("NT"), which lets every fragment load be a
// conflict-free LDS.128: thread t of a quad owns the
// physical k = 4t+s for mma step s, so A[row][4t..4t+3] and Bt[col][4t..4t+3]
// are two 16-byte chunks per 128-byte row.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "sfb_common.cuh"
#include "sfb_kernels.cuh"
#include "sfb_launch.cuh"
#include "sfb_tma.cuh"

#include <cstdlib>
#include <string>

namespace sfb {

int num_sms();

namespace {

#ifndef GEMM_EMPTY
#define GEMM_EMPTY 1  // per-stage empty barriers (1) or a CTA barrier per k-tile (0)
#endif
constexpr int KBOX = 16;  // doubles per 128-byte swizzled TMA box row (one box per operand and 16 k)
#ifndef GEMM_GROUP_M
#define GEMM_GROUP_M 0  // tile raster: bands of GROUP_M tile rows (0: row-major)
#endif
#ifndef GEMM_HYBRID
#define GEMM_HYBRID 1  // full waves data parallel + stream-K tail (0: stream-K over all tiles)
#endif
#ifndef GEMM_SMALL_MINWORK
#define GEMM_SMALL_MINWORK 4  // k-tiles per CTA at least, 64x64 tiles
#endif
#ifndef GEMM_WIDE_STORE
#define GEMM_WIDE_STORE 1  // plain-store epilogue of whole tiles in 128-byte row segments
#endif
#ifndef GEMM_WM
#define GEMM_WM 32  // rows per warp, 128 x 128 tiles: 32 (128 regs; measured +4 % at q = 2047 over 64 rows / 255 regs)
#endif


// CTA tile BM x BN: 128 x 128 with 16 warps (one CTA per SM) for large
// GEMMs; 64 x 64 when the 128-tiles would not fill the machine (fewer than
// 64 of them: q < 1024), so the stream-K pieces stay short and the fix-up
// traffic small — with 16 warps of 16 x 16 at <= 40 128-tiles (q <= 768,
// the cfg1 reduced solve), where one warp per SM sub-partition cannot hide
// the DMMA dependency latency, else 4 warps of 32 x 32 (two CTAs per SM).
template <int BM_, int BN_, int BK_, int STAGES_, int WM_ = 32, int WN_ = 32>
struct Tile {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_;
    static constexpr int WM = WM_, WN = WN_;          // warp tile WM x WN
    static constexpr int MI = WM / 8, NJ = WN / 8;    // MI x NJ DMMA 8x8 blocks per warp
    static_assert(BK % KBOX == 0, "k-tile must be a multiple of the TMA box width");
    // k-tiles in flight ahead of the one being consumed: all but one slot with
    // few deep stages (the refill then waits for the slowest warp's previous
    // k-tile: measured +0.1-0.3 % for 3 x 64 KB), else one slot of slack so
    // warps drift by a k-tile without stalling the issuing thread
    static constexpr int LOOKAHEAD = (GEMM_EMPTY && STAGES > 3) ? STAGES - 2 : STAGES - 1;
    static constexpr int WARPS_N = BN / WN;
    static constexpr int NWARPS = (BM / WM) * WARPS_N;
    static constexpr int NTHREADS = NWARPS * 32;
    static constexpr int CTAS_PER_SM = NWARPS >= 16 ? 1 : 2;
    static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
    static constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + 2 * STAGES * 8 + 1024;
};
#ifndef GEMM_BIG_BK
#define GEMM_BIG_BK 32  // measured: 36.3 vs 35.4 TF/s at q = 8192 (3 x 64 KB stages vs 5 x 32 KB)
#endif
#ifndef GEMM_BIG_STAGES
#define GEMM_BIG_STAGES (GEMM_BIG_BK == 32 ? 3 : 5)
#endif
using BigTile = Tile<128, 128, GEMM_BIG_BK, GEMM_BIG_STAGES, GEMM_WM, 32>;
using SmallTile = Tile<64, 64, 16, 5, 32, 32>;  // 4 warps, 2 CTAs/SM
using TinyTile = Tile<64, 64, 16, 5, 16, 16>;   // 16 warps of 16 x 16: latency-bound sizes

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 lds128(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

// Hybrid schedule: `waves` full waves of whole tiles in data-parallel order
// (CTA c takes tiles c, c + G, c + 2G, ...: the CTAs of a wave walk k in
// lockstep over neighbouring tiles and share their A / B k-slices in L2),
// then the remaining tiles' (tile, k-tile) iterations split stream-K over
// all G CTAs (CTA c owns tail iterations [c U / G, (c+1) U / G)), which
// balances the last partial wave.
struct Sched {
    int tiles_n;         // tiles along N
    int KT;              // k-tiles per output tile
    long long U;         // stream-K (tail) iterations
    int G;               // CTAs
    int tiles_total;     // output tiles (one <C,D> partial each)
    int tiles_per;       // output tiles per problem (batched launch: tile / tiles_per = problem)
    long long c_stride;  // doubles between the problems' outputs (batched launch)
    int waves;           // data-parallel full waves (tiles 0 .. waves * G - 1)
    __device__ long long start(int c) const { return (long long)c * U / G; }
    // tile -> output origin: tiles run down GROUP_M-row bands column by column,
    // so the CTAs in flight share A and B panels in L2 (plain row-major with 0)
    __device__ void origin(int tile, int bm, int bn, int& m0, int& n0) const {
#if GEMM_GROUP_M > 0
        const int tiles_m = tiles_per / tiles_n;
        const int band = tile / (GEMM_GROUP_M * tiles_n), first = band * GEMM_GROUP_M;
        const int gm = min(tiles_m - first, GEMM_GROUP_M), in = tile - band * GEMM_GROUP_M * tiles_n;
        m0 = (first + in % gm) * bm;
        n0 = (in / gm) * bn;
#else
        m0 = (tile / tiles_n) * bm;
        n0 = (tile % tiles_n) * bn;
#endif
    }
    __device__ int owner(long long i) const {  // CTA whose tail range holds tail iteration i
        int c = (int)((i * G) / U);
        while (c + 1 < G && start(c + 1) <= i) ++c;
        while (c > 0 && start(c) > i) --c;
        return c;
    }
};

// Parking slot of a split tile's piece: a CTA holds at most one continuation
// piece (k0 != 0, the first work of its range) and at most one split first
// piece (k0 == 0, the last work of its range).
template <class T>
__device__ __forceinline__ size_t ws_slot(int cta, int k0) {
    return ((size_t)2 * cta + (k0 == 0 ? 1 : 0)) * (T::BM * T::BN);
}

// Epilogue of one finished tile (registers -> global).
template <class T>
__device__ __forceinline__ double tile_epilogue(double (&acc)[T::MI][T::NJ][2], const GemmEpi& ep, int M, int N, int m0,
                                                int n0, int wm, int wn, int g, int t, size_t coff = 0) {
    constexpr int MI = T::MI, NJ = T::NJ;
    double dot = 0.0;
#if GEMM_WIDE_STORE
    // Plain store of a whole tile: lanes of neighbouring quads (g, g ^ 1) swap one of
    // their two 8 x 8 blocks, so every store instruction writes four rows of 128
    // contiguous bytes (two blocks side by side) instead of eight rows of 64.
    if (ep.mode == EPI_STORE && (NJ % 2) == 0 && m0 + T::BM <= M && n0 + T::BN <= N && (ep.ldc % 2) == 0 &&
        ((reinterpret_cast<uintptr_t>(ep.C) + coff * 8) & 15) == 0) {
        const int odd = g & 1;
        #pragma unroll
        for (int i = 0; i < MI; ++i) {
            const int me = m0 + wm * T::WM + i * 8 + (g & ~1);  // the pair's even row
            #pragma unroll
            for (int jp = 0; jp < NJ / 2; ++jp) {
                const double a0 = acc[i][2 * jp][0], a1 = acc[i][2 * jp][1];          // row g, columns of block 2jp
                const double b0 = acc[i][2 * jp + 1][0], b1 = acc[i][2 * jp + 1][1];  // row g, columns of block 2jp + 1
                // even g sends its right block (it stores the left one of both rows), odd g its left block
                const double s0 = odd ? a0 : b0, s1 = odd ? a1 : b1;
                const double r0 = __shfl_xor_sync(0xffffffffu, s0, 4), r1 = __shfl_xor_sync(0xffffffffu, s1, 4);
                const int n = n0 + wn * T::WN + (2 * jp + odd) * 8 + 2 * t;
                double* c = ep.C + coff + (size_t)me * ep.ldc + n;
                // even g: row me <- own left block, row me + 1 <- the neighbour's left block;
                // odd g:  row me <- the neighbour's right block, row me + 1 <- own right block
                *reinterpret_cast<double2*>(c) = odd ? make_double2(r0, r1) : make_double2(a0, a1);
                *reinterpret_cast<double2*>(c + ep.ldc) = odd ? make_double2(b0, b1) : make_double2(r0, r1);
            }
        }
        return 0.0;
    }
#endif
    #pragma unroll
    for (int i = 0; i < MI; ++i) {
        const int m = m0 + wm * T::WM + i * 8 + g;
        if (m >= M) continue;
        #pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int n = n0 + wn * T::WN + j * 8 + 2 * t;
            double v0 = acc[i][j][0], v1 = acc[i][j][1];
            const bool ok0 = n < N, ok1 = n + 1 < N;
            switch (ep.mode) {
                case EPI_SCATTER: {
                    int d = 0;
                    while (d + 1 < ep.nseg && m >= ep.seg[d + 1]) ++d;
                    double* c = ep.dst[d] + (size_t)(m - ep.seg[d]) * ep.ldd_seg[d] + ep.col_off + n;
                    if (ok1 && (reinterpret_cast<uintptr_t>(c) & 15) == 0) {
                        *reinterpret_cast<double2*>(c) = make_double2(v0, v1);
                    } else {
                        if (ok0) c[0] = v0;
                        if (ok1) c[1] = v1;
                    }
                    break;
                }
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
                    double* c = ep.C + coff + (size_t)m * ep.ldc + n;
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
    return dot;
}

// Persistent stream-K schedule: CTA c owns the linear (tile, k-tile)
// iterations [c U / G, (c+1) U / G).  A tile split across CTAs is finished by
// whichever of its pieces arrives last: the others park their partial tile in
// `ws` and take a ticket in `flags[tile]`; the last arriver (usually the k = 0
// piece, the last work of its CTA, which then parks nothing) sums the pieces
// in k order and runs the epilogue.  No CTA waits on another, so the kernel is
// deadlock-free however many kernels share the GPU.  <C,D> partials are per
// tile, so every sum is independent of who finished.  With ws == nullptr
// every CTA owns whole tiles (grid = tile count).
// BATCH: a strided batch of independent problems of one shape in one
// persistent launch (plain store epilogue; the leaf products of the Strassen
// schedule): the operands are stacks of matrices behind rank-3 tensor maps,
// tile / tiles_per is the problem (the maps' third coordinate, and the
// output's offset), so the whole batch shares one wave schedule and one
// stream-K tail.
struct GemmMaps {
    CUtensorMap a, b;
};

template <class T, bool BATCH>
__global__ void __launch_bounds__(T::NTHREADS, T::CTAS_PER_SM)
    dgemm_nt_kernel(const __grid_constant__ GemmMaps maps, int M, int N, int K, GemmEpi ep, Sched sc) {
    constexpr int BM = T::BM, BN = T::BN, NWARPS = T::NWARPS, NTHREADS = T::NTHREADS;
    constexpr int BK = T::BK, STAGES = T::STAGES, LOOKAHEAD = T::LOOKAHEAD;
    constexpr int A_BYTES = T::A_BYTES, B_BYTES = T::B_BYTES;
    SFB_PDL_PROLOGUE();
    if (ep.pcg != nullptr && ep.pcg->status != SFB_PCG_RUNNING) return;  // uniform gate

    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t sA = base, sB = base + STAGES * A_BYTES, full = sB + STAGES * B_BYTES;
    const uint32_t empty = full + 8 * STAGES;  // one arrive per warp when it is done reading a slot

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp / T::WARPS_N, wn = warp % T::WARPS_N;  // (BM/WM) x (BN/WN) warps, WM x WN each
    constexpr int MI = T::MI, NJ = T::NJ, WM = T::WM, WN = T::WN;
    const int g = lane >> 2, t = lane & 3;
    const int KT = sc.KT;
    const long long beg = sc.start(blockIdx.x), fin = sc.start(blockIdx.x + 1);  // tail range
    const int n_dp = sc.waves * KT;               // data-parallel iterations of this CTA
    const int n_it = n_dp + (int)(fin - beg);
    const int tail0 = sc.waves * sc.G;            // first tail tile
    // local iteration -> (tile, k-tile)
    auto locate = [&](int it, int& tile, int& kt) {
        if (it < n_dp) {
            tile = (int)blockIdx.x + (it / KT) * sc.G;
            kt = it % KT;
        } else {
            const long long li = beg + (it - n_dp);
            tile = tail0 + (int)(li / KT);
            kt = (int)(li - (long long)(tile - tail0) * KT);
        }
    };

    auto issue = [&](int it) {  // TMA for local iteration `it` into its ring slot
        int tile, kt;
        locate(it, tile, kt);
        int m0, n0;
        const int prob = BATCH ? tile / sc.tiles_per : 0;
        sc.origin(BATCH ? tile - prob * sc.tiles_per : tile, BM, BN, m0, n0);
        const int sl = it % STAGES;
        mbar_expect_tx_u32(full + 8 * sl, A_BYTES + B_BYTES);
        #pragma unroll
        for (int kb = 0; kb < BK / KBOX; ++kb) {
            const uint32_t da = sA + sl * A_BYTES + kb * BM * KBOX * 8, db = sB + sl * B_BYTES + kb * BN * KBOX * 8;
            if constexpr (BATCH) {
                tma_load3_u32(da, &maps.a, full + 8 * sl, kt * BK + kb * KBOX, m0, prob);
                tma_load3_u32(db, &maps.b, full + 8 * sl, kt * BK + kb * KBOX, n0, prob);
            } else {
                tma_load_u32(da, &maps.a, full + 8 * sl, kt * BK + kb * KBOX, m0);
                tma_load_u32(db, &maps.b, full + 8 * sl, kt * BK + kb * KBOX, n0);
            }
        }
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init_u32(full + 8 * s, 1);
            mbar_init_u32(empty + 8 * s, NWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.b)) : "memory");
        for (int it = 0; it < LOOKAHEAD && it < n_it; ++it) issue(it);
    }
    __syncthreads();

    __shared__ int s_fin;
    __shared__ double sh_dot[NTHREADS / 32];
    double acc[MI][NJ][2];
    int it = 0;
    while (it < n_it) {
        int tile, k0;
        locate(it, tile, k0);
        const int seg_end = (int)min((long long)n_it, (long long)it + (KT - k0));
        const int kl = k0 + (seg_end - it) - 1;  // last k-tile of this piece
        #pragma unroll
        for (int i = 0; i < MI; ++i)
            #pragma unroll
            for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

        for (; it < seg_end; ++it) {
            const int s = it % STAGES;
#if GEMM_EMPTY
            if (threadIdx.x == 0 && it + LOOKAHEAD < n_it) {
                const int nx = it + LOOKAHEAD;  // its slot was last read in local iteration nx - STAGES
                if (nx >= STAGES) mbar_wait_u32(empty + 8 * (nx % STAGES), ((nx / STAGES) - 1) & 1);
                issue(nx);
            }
#else
            __syncthreads();  // every warp is done with the slot refilled below (WAR)
            if (threadIdx.x == 0 && it + LOOKAHEAD < n_it) issue(it + LOOKAHEAD);
#endif
            mbar_wait_u32(full + 8 * s, (it / STAGES) & 1);
            #pragma unroll
            for (int hh = 0; hh < 2 * (BK / KBOX); ++hh) {
                const int half = hh & 1, kb = hh >> 1;  // box kb of the stage, 8-double half of its row
                const uint32_t a_base = sA + s * A_BYTES + kb * BM * KBOX * 8 + (wm * WM + g) * 128;
                const uint32_t b_base = sB + s * B_BYTES + kb * BN * KBOX * 8 + (wn * WN + g) * 128;
                const uint32_t ch = ((2 * t + half) ^ g) << 4;  // SWIZZLE_128B: chunk ^= row & 7 (= g)
                double2 a[MI], b[NJ];
                #pragma unroll
                for (int i = 0; i < MI; ++i) a[i] = lds128(a_base + i * 1024 + ch);
                #pragma unroll
                for (int j = 0; j < NJ; ++j) b[j] = lds128(b_base + j * 1024 + ch);
                #pragma unroll
                for (int i = 0; i < MI; ++i)
                    #pragma unroll
                    for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
                #pragma unroll
                for (int i = 0; i < MI; ++i)
                    #pragma unroll
                    for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
            }
#if GEMM_EMPTY
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * s) : "memory");
#endif
        }

        int m0, n0;
        const int prob = BATCH ? tile / sc.tiles_per : 0;
        sc.origin(BATCH ? tile - prob * sc.tiles_per : tile, BM, BN, m0, n0);
        bool finish = true;
        if (k0 != 0 || kl != KT - 1) {
            // split tile: the last piece to arrive finishes it (no CTA ever
            // waits on another, so any residency order makes progress)
            // (only tail tiles are split)
            const long long t0 = (long long)(tile - tail0) * KT;
            const int c_first = sc.owner(t0), c_last = sc.owner(t0 + KT - 1);
            const int me = (int)blockIdx.x;
            const unsigned others = (unsigned)(c_last - c_first);
            auto park = [&]() {
                double* w = ep.sk_ws + ws_slot<T>(me, k0);
                #pragma unroll
                for (int i = 0; i < MI; ++i)
                    #pragma unroll
                    for (int j = 0; j < NJ; ++j)
                        __stcg(reinterpret_cast<double2*>(w + (size_t)((i * NJ + j) * 2) * NTHREADS) + threadIdx.x,
                               make_double2(acc[i][j][0], acc[i][j][1]));
            };
            auto fold = [&](int c, int piece_k0, bool assign) {  // acc (=|+=) parked piece of CTA c
                const double* w = ep.sk_ws + ws_slot<T>(c, piece_k0);
                #pragma unroll
                for (int i = 0; i < MI; ++i)
                    #pragma unroll
                    for (int j = 0; j < NJ; ++j) {
                        const double2 v = __ldcg(
                            reinterpret_cast<const double2*>(w + (size_t)((i * NJ + j) * 2) * NTHREADS) + threadIdx.x);
                        acc[i][j][0] = assign ? v.x : acc[i][j][0] + v.x;
                        acc[i][j][1] = assign ? v.y : acc[i][j][1] + v.y;
                    }
            };
            finish = false;
            if (k0 == 0) {
                // the k = 0 piece is the last work of its CTA and usually the last
                // to arrive: when every other piece is already counted (parked),
                // finish without parking it
                if (threadIdx.x == 0) {
                    unsigned seen;
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(ep.sk_flags + tile) : "memory");
                    s_fin = (seen == others) ? 1 : 0;
                }
                __syncthreads();
                finish = s_fin != 0;
            }
            bool parked = false;
            if (!finish) {
                park();
                parked = true;
                __threadfence();
                __syncthreads();
                if (threadIdx.x == 0) s_fin = (atomicAdd(ep.sk_flags + tile, 1u) == others) ? 1 : 0;
                __syncthreads();
                finish = s_fin != 0;
            }
            if (finish) {
                if (threadIdx.x == 0) ep.sk_flags[tile] = 0;  // ready for the next launch
                __threadfence();
                // sum the pieces in k order whoever finishes (bit-reproducible):
                // the k = 0 piece first, then the continuations in CTA order
                if (me != c_first) {
                    if (!parked) park();  // our continuation is re-read in its place (same thread, L2)
                    fold(c_first, 0, true);
                }
                for (int c = c_first + 1; c <= c_last; ++c) fold(c, 1, false);
            }
            __syncthreads();  // s_fin is rewritten by the next split piece
        }
        if (finish) {
            const double d = tile_epilogue<T>(acc, ep, M, N, m0, n0, wm, wn, g, t,
                                              BATCH ? (size_t)prob * (size_t)sc.c_stride : 0);
            if (ep.mode == EPI_STORE_DOT) {  // one partial per tile: the sum order does not depend on who finished
                const double part = block_sum<NTHREADS>(d, sh_dot);
                if (threadIdx.x == 0) ep.partials[tile] = part;
            }
        }
    }

    if (ep.mode == EPI_STORE_DOT) {
        const unsigned nblk = gridDim.x;
        if (arrive_last(ep.counter, nblk)) {
            const double tot = sum_partials<NTHREADS>(ep.partials, sc.tiles_total, 1, sh_dot);
            if (threadIdx.x == 0) {
                *ep.counter = 0;
                if (ep.pcg != nullptr) ep.pcg->rz_next = tot;
                if (ep.dot_out != nullptr) *ep.dot_out = tot;
            }
        }
    }
}

int make_map(CUtensorMap* map, const double* ptr, int rows, int cols, int ld, int box_rows) {
    if (!tma_aligned(ptr, ld)) return arg_error("DMMA GEMM operands need 16-byte aligned rows (even leading dimension)");
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint32_t box[2] = {KBOX, (cuuint32_t)box_rows};
    return tma_make_map(map, ptr, 2, dims, ld, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

inline int tiles_of(int M, int N, int bm, int bn) { return ((N + bn - 1) / bn) * ((M + bm - 1) / bm); }

// SYLFEM_B200_GEMM_TILE=128|64|16 forces one tile shape (measurement switch: 16 =
// 64 x 64 tiles with 16 x 16 warp tiles);
// default: 64 x 64 tiles when the 128 x 128 tiles would not fill the SMs.
int tile_mode() {
    static const int m = [] {
        const char* e = std::getenv("SYLFEM_B200_GEMM_TILE");
        return e == nullptr ? 0 : std::atoi(e);
    }();
    return m;
}

// SYLFEM_B200_BATCH_SCHED=streamk: the strided batch as pure stream-K (tile
// boundaries, hence epilogue store bursts, spread over time across the CTAs)
// instead of data-parallel waves + a stream-K tail
bool batch_stream_k() {
    static const bool v = [] {
        const char* e = std::getenv("SYLFEM_B200_BATCH_SCHED");
        return e != nullptr && std::string(e) == "streamk";
    }();
    return v;
}

int make_map3(CUtensorMap* map, const double* ptr, int rows, int cols, int ld, int box_rows, int nb) {
    if (!tma_aligned(ptr, ld)) return arg_error("DMMA GEMM operands need 16-byte aligned rows (even leading dimension)");
    const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)nb};
    const cuuint32_t box[3] = {KBOX, (cuuint32_t)box_rows, 1};
    return tma_make_map(map, ptr, 3, dims, ld, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// nb > 0: strided batch (A: nb stacked M x lda matrices, Bt: nb stacked N x ldb, C_b = ep.C + b * c_stride)
template <class T, bool BATCH>
int launch_tile_batch(const double* A, int lda, const double* Bt, int ldb, int nb, int M, int N, int K,
                      long long c_stride, const GemmEpi& ep, cudaStream_t stream) {
    SFB_TRY(ensure_dynamic_smem(dgemm_nt_kernel<T, BATCH>, T::SMEM_BYTES));
    GemmMaps maps;
    if (BATCH) {
        SFB_TRY(make_map3(&maps.a, A, M, K, lda, T::BM, nb));
        SFB_TRY(make_map3(&maps.b, Bt, N, K, ldb, T::BN, nb));
    } else {
        SFB_TRY(make_map(&maps.a, A, M, K, lda, T::BM));
        SFB_TRY(make_map(&maps.b, Bt, N, K, ldb, T::BN));
    }
    const int NB = BATCH ? nb : 1;
    Sched sc;
    sc.tiles_n = (N + T::BN - 1) / T::BN;
    sc.KT = (K + T::BK - 1) / T::BK;
    sc.tiles_per = tiles_of(M, N, T::BM, T::BN);
    sc.c_stride = c_stride;
    const int tiles = NB * sc.tiles_per;
    sc.tiles_total = tiles;
    sc.waves = 0;
    const bool have_ws = ep.sk_ws != nullptr && ep.sk_flags != nullptr;
    // grid: at most CTAS_PER_SM CTAs per SM.  Without a workspace, or when the
    // tiles fill whole waves, one CTA per tile (data parallel).  Otherwise the
    // full waves of whole tiles run data parallel and the rest stream-K (at
    // least a few k-tiles per CTA), so the last partial wave is balanced.
    const int slots = num_sms() * T::CTAS_PER_SM;
    if (!have_ws || tiles % slots == 0) {
        sc.G = tiles;
        sc.waves = 1;  // CTA c: tile c, whole
        sc.U = 0;
    } else if (tiles > slots && GEMM_HYBRID && !(BATCH && batch_stream_k())) {
        sc.G = slots;
        sc.waves = tiles / slots - 1;  // keep one wave + the remainder in the stream-K tail
        sc.U = (long long)(tiles - sc.waves * slots) * sc.KT;
    } else {
        const long long min_work = T::BM >= 128 ? 8 : GEMM_SMALL_MINWORK;
        sc.U = (long long)tiles * sc.KT;
        sc.G = (int)std::max(1LL, std::min<long long>(slots, sc.U / min_work));
    }
    return launch_kernel(dgemm_nt_kernel<T, BATCH>, dim3(sc.G), dim3(T::NTHREADS), T::SMEM_BYTES, stream, maps, M, N,
                         K, ep, sc);
}

template <class T>
int launch_tile(const double* A, int lda, const double* Bt, int ldb, int M, int N, int K, const GemmEpi& ep,
                cudaStream_t stream) {
    return launch_tile_batch<T, false>(A, lda, Bt, ldb, 1, M, N, K, 0, ep, stream);
}

}  // namespace

int num_sms() {
    static const int n = [] {  // thread-safe one-time query (every device of the box is a B200)
        int dev = 0, m = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&m, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || m <= 0) m = kNumSMs;
        return m;
    }();
    return n;
}

// C[M x N] = A[M x K] * Bt[N x K]^T, both row-major K-contiguous.
int launch_dgemm_nt(const double* A, int lda, const double* Bt, int ldb, int M, int N, int K,
                    const GemmEpi& ep, cudaStream_t stream) {
    if (M <= 0 || N <= 0 || K <= 0) return arg_error("empty GEMM");
    const int mode = tile_mode();
    // measured (128 x 128 tiles with 32-deep stages): 64-tiles win below 64
    // 128-tiles (q = 256: 22 vs 38 us; q = 512: 27 vs 55 us; q = 768: 47 vs 55 us)
    // and lose from 64 (q = 1024: 84.3 vs 81.6 us); below ~40 of them the DMMA pipe
    // is latency bound with one warp per SM sub-partition and 16 warps of 16 x 16
    // win (q = 256: 18.4 vs 21.6 us, q = 768: 45.7 vs 47.0 us)
    const int t128 = tiles_of(M, N, 128, 128);
    if (mode == 16 || (mode == 0 && t128 <= 40)) return launch_tile<TinyTile>(A, lda, Bt, ldb, M, N, K, ep, stream);
    const bool small = mode == 64 || (mode != 128 && t128 < 64);
    return small ? launch_tile<SmallTile>(A, lda, Bt, ldb, M, N, K, ep, stream)
                 : launch_tile<BigTile>(A, lda, Bt, ldb, M, N, K, ep, stream);
}

// nb independent products C_b[M x N] = A_b Bt_b^T of one shape in one launch
// (128 x 128 tiles, plain store): A_b = A + b * M * lda, Bt_b = Bt + b * N * ldb
// (stacked matrices behind rank-3 tensor maps), C_b = ep.C + b * c_stride.
int gemm_batch_max(int M, int N) { return gemm_max_tiles() / tiles_of(M, N, 128, 128); }

int launch_dgemm_nt_batch(const double* A, int lda, const double* Bt, int ldb, int nb, int M, int N, int K,
                          long long c_stride, const GemmEpi& ep, cudaStream_t stream) {
    if (M <= 0 || N <= 0 || K <= 0 || nb <= 0) return arg_error("empty GEMM");
    if (ep.mode != EPI_STORE) return arg_error("batched GEMM: plain store epilogue only");
    if (nb > gemm_batch_max(M, N)) return arg_error("batched GEMM: too many tiles for one launch");
    return launch_tile_batch<BigTile, true>(A, lda, Bt, ldb, nb, M, N, K, c_stride, ep, stream);
}

// Upper bound of the output tiles of any tile shape (one <C,D> partial each).
int gemm_grid_blocks(int M, int N) { return tiles_of(M, N, SmallTile::BM, SmallTile::BN); }

int gemm_smem_bytes() { return BigTile::SMEM_BYTES; }

// Stream-K parking: two slots per CTA of the largest grid of either shape.
size_t gemm_workspace_doubles() {
    return std::max((size_t)2 * num_sms() * BigTile::CTAS_PER_SM * BigTile::BM * BigTile::BN,
                    (size_t)2 * num_sms() * SmallTile::CTAS_PER_SM * SmallTile::BM * SmallTile::BN);
}
int gemm_max_tiles() { return 65536; }

}  // namespace sfb
