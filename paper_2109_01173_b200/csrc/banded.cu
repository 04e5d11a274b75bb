// Banded multiterm sandwich  W = sum_t G_t X H_t  (one fused pass over X).
//
// Replaces the 2T dense GEMMs of SylvesterOperator.apply (operators.py:124-131)
// and the rectangular rhs builders (operators.py:206-207, 228-232, 266-268,
// 281-282).  All FEM factors are banded with half-bandwidth <= k (SURVEY
// App. B), so each output element needs a (W x W) window of X.
//
// One CTA owns a TX-column strip of RY output rows (RY sized so the grid is
// one wave of 2-3 CTAs per SM).  A producer warp streams the (RY+W-1) x
// (TX+W-1) input halo down the strip in chunks of CH rows through a 3-stage
// TMA ring (full/empty mbarriers; out-of-bounds rows/columns arrive
// zero-filled), together with the left-factor coefficients of those rows,
// read as a box of the row-skewed copy gskew[j][t*W+d] = G_t[j-d][d] made at
// creation.  Four consumer warps (one thread per output column, right-factor
// band in registers) sweep the rows of each landed chunk: Y_t(r) =
// sum_e X[r][c+e] h_t[e] is formed once per row and scattered into a ring of
// W partial outputs with the left-factor coefficients (shared-memory
// broadcasts).  The MO-PCG direction update Q = Z + beta Q is applied inline
// as the halo values are read (the new Q column is stored by its owner), and
// the previous iteration's U += alpha Q rides along (U's rows come through
// the same TMA ring; Q_prev is already there), so the update pass that
// follows only handles R; the
// IMEX heat source and the DIB kinetics are applied to the landed chunk in
// shared memory first (named barrier among the consumers).  Epilogues: plain
// store, or the MO-PCG store + <W,Q>, |Q|^2 partials with a last-block alpha
// step (solvers.py:424-431).
//
// Cost per output element: 2*T*W FMAs (the FP64 pipe bounds the plain
// 5-term apply; the MO-PCG pass also moves four grids through HBM).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sfb_common.cuh"
#include "sfb_kernels.cuh"
#include "sfb_launch.cuh"
#include "sfb_tma.cuh"

namespace sfb {

namespace {

constexpr int TX = 128;                   // output columns per CTA (one consumer thread each)
constexpr int NTH = TX + 32;              // + one producer warp
#ifndef BAND_NS
#define BAND_NS 3
#endif
#ifndef BAND_ACC2
#define BAND_ACC2 0  // 1: split accumulators (measured: plain apply -2 %, MO-PCG pass +2 %)
#endif
#ifndef BAND_MUNROLL
#define BAND_MUNROLL 2
#endif
#ifndef BAND_MINB
#define BAND_MINB 2
#endif

constexpr int NS = BAND_NS;
constexpr int kMUnroll = BAND_MUNROLL;  // unroll of the chunk's W-row groups                       // TMA ring stages
// CTAs per SM (2 x 5 warps: 168 registers per thread keep the 5-term band
// in registers; measured faster than 3 CTAs at 128 registers)
#ifndef BAND_MINB_WIDE
#define BAND_MINB_WIDE 2
#endif
#ifndef BAND_PCG_XF_MINW
#define BAND_PCG_XF_MINW 7  // MO-PCG direction update as a shared-memory pass from this band width on
#endif
template <int W>
constexpr int band_minb() { return W >= 7 ? BAND_MINB_WIDE : BAND_MINB; }
constexpr int RY_MIN = 32;

// Ring shape: NS stages of chunk_rows<W>() rows, or with FINE (MO-PCG pass of
// narrow operators on short strips) 4 stages of W rows: the first rows land
// sooner and the last chunk is shorter, which measured 44.0 -> 41.6 us at
// q = 2047 (114 rows per CTA) and 144 -> 149 us at q = 4095 (455 rows).
constexpr int FINE_NS = 4;
constexpr int FINE_MAX_ROWS = 160;  // rows per CTA up to which the fine ring is used
template <int W, bool FINE>
__host__ __device__ constexpr int chunk_rows() {
    return FINE ? W : W * (W >= 8 ? 1 : (8 + W - 1) / W);  // a multiple of W (static ring slots)
}

__host__ __device__ constexpr int pad128(int doubles) { return (doubles + 15) / 16 * 16; }

template <int T, int W, bool FINE = false>
struct BandCfg {
    static constexpr int NS = FINE ? FINE_NS : ::sfb::NS;
    static constexpr int CH = chunk_rows<W, FINE>();
    static constexpr int HC = TX + W - 1;    // halo columns
    static constexpr int HCB = HC + 2;       // box columns: boxes start at an even column (16-byte rows)
    static constexpr int TWP = (T * W + 1) / 2 * 2;  // a row's T*W left coefficients, padded to pairs
    static constexpr int XS = CH * HCB;      // doubles of one input box
    static constexpr int GS = CH * TWP;      // doubles of the chunk's left coefficients
    static constexpr int XSP = pad128(XS);   // 128-byte aligned regions
    static constexpr int GSP = pad128(GS);
    static constexpr int STAGE = 2 * XSP + GSP;
    static constexpr int USP = pad128(CH * TX);  // MO-PCG: the strip's rows of U (deferred U += alpha Q)
    static constexpr int SMEM = NS * STAGE * 8 + 128;
    static constexpr int SMEM_PCG = NS * (STAGE + USP) * 8 + 128;
};
template <int T, int W, int MODE, bool FINE>
__host__ __device__ constexpr int band_stage() {
    return BandCfg<T, W, FINE>::STAGE + (MODE == LD_PCG ? BandCfg<T, W, FINE>::USP : 0);
}
template <int T, int W, int MODE, bool FINE>
__host__ __device__ constexpr int band_smem() {
    return MODE == LD_PCG ? BandCfg<T, W, FINE>::SMEM_PCG : BandCfg<T, W, FINE>::SMEM;
}

struct BandMaps {
    CUtensorMap a;       // input A (X / Z / U / eta), box {HCB, CH}
    CUtensorMap b[2];    // input B (Q0, Q1 / F / theta)
    CUtensorMap g;       // gskew, box {TWP, CH}
    CUtensorMap u;       // MO-PCG: U, box {TX, CH}
};

// rows per CTA and row blocks for an output of `rows` x `cols`
// (one wave of `minb` CTAs per SM)
__host__ inline void band_geometry(int rows, int cols, int minb, int* ry, int* nrb) {
    const int nstrips = (cols + TX - 1) / TX;
    const int want = std::max(1, minb * kNumSMs / nstrips);
    const int r = std::max(RY_MIN, (rows + want - 1) / want);
    *ry = r;
    *nrb = (rows + r - 1) / r;
}

// MODE = the loader (LD_*); the MO-PCG loader always comes with the MO-PCG epilogue.
template <int T, int W, int MODE, bool FINE>
__global__ void __launch_bounds__(TX + 32, band_minb<W>()) band_kernel(BandArgs a, const __grid_constant__ BandMaps maps, int ry) {
    SFB_PDL_PROLOGUE();
    if (a.gate != nullptr && a.gate->status != SFB_PCG_RUNNING) return;  // uniform gate
    using C = BandCfg<T, W, FINE>;
    constexpr int CH = C::CH, HCB = C::HCB, TWP = C::TWP, NS = C::NS;
    constexpr int NPAIR = HCB / 2;           // HCB is even (W odd)
    constexpr int NPP = (NPAIR + 63) / 64;   // column pairs per thread in the transform
    constexpr int NRR = (CH + 1) / 2;        // rows per thread and chunk in the transform
    extern __shared__ double sm_raw[];       // NS x {A[CH][HCB], B[CH][HCB], G[CH][TWP]}
    // 128-byte aligned ring (pointer arithmetic on the shared array keeps LDS/STS addressing)
    double* sm = sm_raw + (((128u - (smem_u32(sm_raw) & 127u)) & 127u) >> 3);
    __shared__ __align__(8) uint64_t full[NS], empty[NS];

    constexpr int mode = MODE;
    constexpr bool pcg_ep = mode == LD_PCG;
    PcgState* st = a.pcg;
    int s = 0;
    double beta = 0.0, alpha_prev = 0.0;
    if constexpr (mode == LD_PCG) {
        if (st->status != SFB_PCG_RUNNING) return;  // uniform gate
        s = st->iter;
        if (s > 0) {
            beta = st->rz_next / st->rz;             // solvers.py:448-452
            alpha_prev = st->alpha;                  // the previous iteration's U += alpha Q, deferred here
        }
    }
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * ry;
    const int rows_here = min(ry, a.out_rows - y0);
    const int hry = rows_here + W - 1;             // halo rows streamed by this CTA
    const int nch = (hry + CH - 1) / CH;
    const int t = threadIdx.x, c = t, gc = x0 + c;
    const int goff = a.goff, hoff = a.hoff;

    // ---- sources ----
    int acs = 0, ars = 0;
    bool hasB = false;
    const CUtensorMap* mb = &maps.b[0];
    double* Qcur = nullptr;
    if constexpr (mode == LD_PCG) {
        Qcur = (s & 1) ? a.Q1 : a.Q0;
        hasB = s > 0;
        mb = &maps.b[(s & 1) ? 0 : 1];  // previous direction
    } else if constexpr (mode == LD_HEAT) {  // interior state U at offset (rs, cs): zero outside
        ars = a.rs;
        acs = a.cs;
        hasB = a.X2 != nullptr;
    } else if constexpr (mode == LD_DIB) {
        hasB = true;
    }
    // A's box starts at full-grid column x0 + hoff - shA (U column minus acs), B's at x0 + hoff - shB;
    // both even, so every box row is 16-byte aligned in global memory
    const int shA = (hoff - acs) & 1, shB = hoff & 1;
    constexpr int STG = band_stage<T, W, MODE, FINE>();  // doubles per ring stage
    // MO-PCG from the second iteration on: U's rows ride in the ring too
    const bool withU = mode == LD_PCG && hasB;
    const uint32_t tx_bytes = (uint32_t)((hasB ? 2 : 1) * C::XS + C::GS + (withU ? CH * TX : 0)) * 8;
    const bool producer = t >= TX;  // warp 4 feeds the ring; warps 0-3 consume it

    if (t == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init_u32(smem_u32(&full[i]), 1);
            mbar_init_u32(smem_u32(&empty[i]), TX / 32);  // one arrive per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    double pdot = 0.0, pqq = 0.0;  // MO-PCG: <W,Q>, |Q|^2; residual epilogue: |B - W|^2, |B|^2
    const bool resid = mode == LD_PLAIN && a.ep_mode == EP_RESID;
    bool flag = false;
    double vmax = 0.0;
    if (producer) {
        if (t == TX) {
            for (int k = 0; k < nch; ++k) {
                const int sl = k % NS;
                if (k >= NS) mbar_wait_u32(smem_u32(&empty[sl]), ((k / NS) - 1) & 1);
                double* A = sm + sl * STG;
                const uint32_t bar = smem_u32(&full[sl]);
                const int r0 = k * CH;
                mbar_expect_tx_u32(bar, tx_bytes);
                tma_load_u32(smem_u32(A), &maps.a, bar, x0 + hoff - acs - shA, y0 + goff + r0 - ars);
                if (hasB) tma_load_u32(smem_u32(A + C::XSP), mb, bar, x0 + hoff - shB, y0 + goff + r0);
                tma_load_u32(smem_u32(A + 2 * C::XSP), &maps.g, bar, 0, y0 + r0);
                if (withU) tma_load_u32(smem_u32(A + 2 * C::XSP + C::GSP), &maps.u, bar, x0, y0 + goff + r0);
            }
        }
    } else {
        // ---- HEAT / DIB: per-thread transform geometry, smem column pairs pc, pc + 64 of rows rh, rh + 2, ...
        // (A's column space: smem column m holds full-grid column x0 + hoff - shA + m) ----
        const int pc = t & 63, rh = t >> 6;
        unsigned mdom[NPP];
        #pragma unroll
        for (int j = 0; j < NPP; ++j) {
            const int pp = pc + 64 * j;
            const int gx = x0 + hoff - shA + 2 * pp;
            auto pm = [](int col, int n) {
                return ((unsigned)col < (unsigned)n ? 1u : 0u) | ((unsigned)(col + 1) < (unsigned)n ? 2u : 0u);
            };
            // in the grid and in this CTA's halo (the box's extra columns stay out of the checks)
            mdom[j] = pp < NPAIR ? (pm(gx, a.in_cols) & pm(2 * pp - shA, C::HC)) : 0u;
        }
        // wide bands (W >= 7): the MO-PCG direction update Q = Z + beta Q_prev
        // is applied once per halo element in shared memory instead of inline
        // in each of the W taps that read it (W x fewer updates and Q_prev
        // reads; measured slower for W = 5)
        constexpr bool pcg_xf = mode == LD_PCG && W >= BAND_PCG_XF_MINW;
        constexpr bool smem_pass = mode == LD_HEAT || mode == LD_DIB || pcg_xf;
        // visit this thread's pairs of a landed chunk: f(gr, j, double2* a_pair, const double* b_elems),
        // b_elems = B at the same full-grid columns (16-byte aligned unless shA != shB: heat only)
        auto for_pairs = [&](double* A, int r0, auto&& f) {
            const double* B = A + C::XSP + (shB - shA);
            #pragma unroll
            for (int i = 0; i < NRR; ++i) {
                const int rr = rh + 2 * i;
                if (rr < CH) {
                    const int gr = y0 + goff + r0 + rr;
                    #pragma unroll
                    for (int j = 0; j < NPP; ++j) {
                        if (j == 0 || pc + 64 * j < NPAIR) {
                            const int o = rr * HCB + 2 * (pc + 64 * j);
                            f(gr, j, reinterpret_cast<double2*>(A + o), B + o);
                        }
                    }
                }
            }
        };
        auto check = [&](double v) {
            if (!isfinite(v)) flag = true;
            else vmax = fmax(vmax, fabs(v));
        };

        // ---- right-factor band of this thread's column, in registers ----
        double h[T][W];
        #pragma unroll
        for (int tt = 0; tt < T; ++tt)
            #pragma unroll
            for (int e = 0; e < W; ++e)
                h[tt][e] = (tt < a.nterms && gc < a.out_cols) ? a.hband[((size_t)tt * a.out_cols + gc) * W + e] : 0.0;

        // two partial accumulators per ring slot (even / odd terms): twice the
        // independent FMA chains in the scatter
        double acc[W], acc2[W], cen[W];
        #pragma unroll
        for (int d = 0; d < W; ++d) acc[d] = acc2[d] = cen[d] = 0.0;
        const bool col_ok = gc < a.out_cols;
        double* const Wout = a.W;
        const int ldw = a.ldw;
        const bool upd = hasB;  // PCG: Q = Z + beta Qprev from the second iteration on

        for (int k = 0; k < nch; ++k) {
            const int sl = k % NS;
            double* A = sm + sl * STG;
            const double* Us = A + 2 * C::XSP + C::GSP;  // MO-PCG: U at halo row rr, column c
            const double* Bs = A + C::XSP;
            const double* G = A + 2 * C::XSP;
            const int r0 = k * CH;
            mbar_wait_u32(smem_u32(&full[sl]), (k / NS) & 1);
            // ---- input transform, in place; consumers sync on named barrier 1 ----
            if constexpr (mode == LD_HEAT) {
                const double cc = a.c;
                const bool chk = a.check != nullptr;
                const int in_rows = a.in_rows;
                for_pairs(A, r0, [&](int gr, int j, double2* ap, const double* bp) {
                    double2 v = *ap;
                    if (hasB) {
                        v.x = v.x + cc * bp[0];
                        v.y = v.y + cc * bp[1];
                        *ap = v;
                    }
                    if (chk && (unsigned)gr < (unsigned)in_rows) {
                        if (mdom[j] & 1u) check(v.x);
                        if (mdom[j] & 2u) check(v.y);
                    }
                });
            } else if constexpr (mode == LD_DIB) {  // models.py:74-82 and timestepping.py:201-207
                const double* p = a.kp;  // alpha, gamma_k, A1, A2, B, C, D, k2, k3
                const double cc = a.c;
                const bool sp0 = a.species == 0, chk = a.check != nullptr;
                const int in_rows = a.in_rows;
                for_pairs(A, r0, [&](int gr, int j, double2* ap, const double* bp) {
                    const double2 e2 = *ap, t2 = *reinterpret_cast<const double2*>(bp);
                    const unsigned m = (unsigned)gr < (unsigned)in_rows ? mdom[j] : 0u;
                    double v[2];
                    const double ev[2] = {e2.x, e2.y}, tv[2] = {t2.x, t2.y};
                    #pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const double eta = ev[q], th = tv[q];
                        double r;
                        if (sp0) {
                            const double f = p[2] * (1.0 - th) * eta - p[3] * (eta * eta * eta) - p[4] * (th - p[0]);
                            r = eta + cc * f;
                        } else {
                            const double g = p[5] * (1.0 + p[7] * eta) * (1.0 - th) * (1.0 - p[1] * (1.0 - th)) -
                                             p[6] * th * (1.0 + p[1] * th) * (1.0 + p[8] * eta);
                            r = th + cc * g;
                        }
                        v[q] = (m >> q) & 1u ? r : 0.0;  // outside the grid the halo is zero
                        if (chk && ((m >> q) & 1u)) check(v[q]);
                    }
                    *ap = make_double2(v[0], v[1]);
                });
            }
            if constexpr (pcg_xf) {
                if (upd) {
                    for_pairs(A, r0, [&](int, int, double2* ap, const double* bp) {
                        const double2 z = *ap, qp = *reinterpret_cast<const double2*>(bp);
                        *ap = make_double2(__dadd_rn(__dmul_rn(beta, qp.x), z.x), __dadd_rn(__dmul_rn(beta, qp.y), z.y));
                    });
                }
            }
            if constexpr (smem_pass)
                asm volatile("bar.sync 1, %0;" ::"n"(TX) : "memory");  // transformed chunk visible

            // ---- sweep the chunk's halo rows (rows past the halo feed only unstored outputs) ----
            #pragma unroll kMUnroll
            for (int m = 0; m < CH / W; ++m) {
                #pragma unroll
                for (int u = 0; u < W; ++u) {
                    const int rr = m * W + u;  // r0 + rr == u (mod W)
                    // Y_t(row) = sum_e X[row][c+e] h_t[e]: one input value live at a
                    // time, T independent chains
                    double y[T];
                    #pragma unroll
                    for (int tt = 0; tt < T; ++tt) y[tt] = 0.0;
                    #pragma unroll
                    for (int e = 0; e < W; ++e) {
                        const double z = A[rr * HCB + shA + c + e];
                        double q = z;
                        if constexpr (mode == LD_PCG && !pcg_xf)  // Q*=beta; Q+=Z (solvers.py:448-452), inline
                            q = upd ? __dadd_rn(__dmul_rn(beta, Bs[rr * HCB + shA + c + e]), z) : z;
                        if (e == (W - 1) / 2) cen[u] = q;
                        #pragma unroll
                        for (int tt = 0; tt < T; ++tt) y[tt] = fma(q, h[tt][e], y[tt]);
                    }
                    if constexpr (mode == LD_PCG) {
                        // this thread's column of the new direction, interior rows only; the
                        // previous iteration's U += alpha Q (solvers.py:432) rides along: Q_prev
                        // is already in shared memory, so it costs only U's read and write
                        const int gr = y0 + goff + r0 + rr;
                        if (gr >= y0 && gr < y0 + rows_here && col_ok) {
                            Qcur[(size_t)gr * a.ldq + gc] = cen[u];
                            if (upd)  // U's rows arrive with the halo (TMA), U += alpha_prev Q_prev
                                a.U[(size_t)gr * a.ldq + gc] =
                                    __dadd_rn(Us[rr * TX + c], __dmul_rn(alpha_prev, Bs[rr * HCB + shA + c + (W - 1) / 2]));
                        }
                    }
                    // scatter: the row's T*W left coefficients are contiguous (pairs may
                    // straddle two terms), G[rr][tt*W + d] multiplies Y_tt into output row r - d
                    const double2* gp = reinterpret_cast<const double2*>(G + rr * TWP);
                    #pragma unroll
                    for (int f2 = 0; f2 < TWP / 2; ++f2) {
                        const double2 g = gp[f2];
                        #pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const int f = 2 * f2 + q;
                            if (f < T * W) {
                                const int tt = f / W, d = f - tt * W;
                                const int sl = (u - d + 2 * W) % W;
#if BAND_ACC2
                                if (tt & 1) acc2[sl] = fma(q == 0 ? g.x : g.y, y[tt], acc2[sl]);
                                else
#endif
                                    acc[sl] = fma(q == 0 ? g.x : g.y, y[tt], acc[sl]);
                            }
                        }
                    }
                    const int i = r0 + rr - (W - 1);
                    const int slot = (u + 1) % W;
                    // branch-free epilogue: predicated store, masked dot terms
                    const bool store = (unsigned)i < (unsigned)rows_here && col_ok;
#if BAND_ACC2
                    const double w = acc[slot] + acc2[slot];
                    acc2[slot] = 0.0;
#else
                    const double w = acc[slot];
#endif
                    if (resid) {  // the residual of a reduced solve: no W store
                        const double bv = store ? a.B[(size_t)(y0 + i) * a.ldb + gc] : 0.0;
                        const double rv = store ? bv - w : 0.0;
                        pdot = fma(rv, rv, pdot);
                        pqq = fma(bv, bv, pqq);
                    } else if (store) {
                        Wout[(size_t)(y0 + i) * ldw + gc] = w;
                    }
                    if constexpr (pcg_ep) {
                        // Q at (y0 + i, gc): centre of halo row i - goff = r - (W-1)/2
                        const double q = store ? cen[(u - (W - 1) / 2 + W) % W] : 0.0;
                        pdot = fma(w, q, pdot);
                        pqq = fma(q, q, pqq);
                    }
                    acc[slot] = 0.0;
                }
            }
            // release the stage to the producer (generic writes ordered before the TMA refill)
            if constexpr (smem_pass) fence_proxy_async_smem();
            __syncwarp();
            if ((t & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[sl])) : "memory");
        }
    }
    if (a.check != nullptr) {
        if (flag) atomicOr(a.check + 1, 1ull);
        if (vmax > 0.0) atomicMax(a.check, (unsigned long long)__double_as_longlong(vmax));
    }

    if (mode == LD_PLAIN && a.ep_mode == EP_RESID) {  // uniform: sum in fixed order, last block finishes
        __shared__ double shr[NTH / 32];
        const unsigned nblk = gridDim.x * gridDim.y;
        const unsigned bid = blockIdx.y * gridDim.x + blockIdx.x;
        const double p0 = block_sum<NTH>(pdot, shr);
        const double p1 = block_sum<NTH>(pqq, shr);
        if (threadIdx.x == 0) {
            a.partials[bid] = p0;
            a.partials[nblk + bid] = p1;
        }
        if (arrive_last(&a.res->counter[0], nblk)) {
            const double rr = sum_partials<NTH>(a.partials, nblk, 1, shr);
            const double bb = sum_partials<NTH>(a.partials + nblk, nblk, 1, shr);
            if (threadIdx.x == 0) {
                a.res->counter[0] = 0;
                a.res->v[0] = sqrt(rr);
                a.res->v[3] = sqrt(bb);
            }
        }
    }
    if constexpr (pcg_ep) {
        __shared__ double sh[NTH / 32];
        const unsigned nblk = gridDim.x * gridDim.y;
        const unsigned bid = blockIdx.y * gridDim.x + blockIdx.x;
        const double p0 = block_sum<NTH>(pdot, sh);
        const double p1 = block_sum<NTH>(pqq, sh);
        if (threadIdx.x == 0) {
            a.partials[bid] = p0;
            a.partials[nblk + bid] = p1;
        }
        if (arrive_last(&st->counter[0], nblk)) {
            const double qw = sum_partials<NTH>(a.partials, nblk, 1, sh);
            const double qq = sum_partials<NTH>(a.partials + nblk, nblk, 1, sh);
            if (threadIdx.x == 0) {
                st->counter[0] = 0;
                st->rz = st->rz_next;
                st->qq = qq;
                if (qw <= 0.0) {  // solvers.py:426-430
                    st->status = SFB_PCG_INDEFINITE;
                    st->bad_value = qw;
                    st->bad_iter = s;
                } else {
                    st->alpha = st->rz / qw;  // solvers.py:431
                }
            }
        }
    }
}

template <int T, int W, int MODE, bool FINE>
int launch_twmf(const BandArgs& a, int ry, int nrb, cudaStream_t stream) {
    using C = BandCfg<T, W, FINE>;
    constexpr int smem = band_smem<T, W, MODE, FINE>();
    SFB_TRY(ensure_dynamic_smem(band_kernel<T, W, MODE, FINE>, smem));
    // tensor maps of the inputs (zero fill outside each source's extents)
    BandMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const cuuint32_t xbox[2] = {(cuuint32_t)C::HCB, (cuuint32_t)C::CH};
    auto xmap = [&](CUtensorMap* m, const double* p, int ld, int rows, int cols) {
        const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        return tma_make_map(m, p, 2, dims, ld, xbox, CU_TENSOR_MAP_SWIZZLE_NONE);
    };
    if (a.ld_mode == LD_HEAT) {
        SFB_TRY(xmap(&maps.a, a.X, a.ldx, a.in_rows - 2 * a.rs, a.in_cols - 2 * a.cs));
        if (a.X2 != nullptr) SFB_TRY(xmap(&maps.b[0], a.X2, a.ldx2, a.in_rows, a.in_cols));
    } else {
        SFB_TRY(xmap(&maps.a, a.X, a.ldx, a.in_rows, a.in_cols));
        if (a.ld_mode == LD_PCG) {
            SFB_TRY(xmap(&maps.b[0], a.Q0, a.ldq, a.in_rows, a.in_cols));
            SFB_TRY(xmap(&maps.b[1], a.Q1, a.ldq, a.in_rows, a.in_cols));
        } else if (a.ld_mode == LD_DIB) {
            SFB_TRY(xmap(&maps.b[0], a.X2, a.ldx2, a.in_rows, a.in_cols));
        }
    }
    {
        if (a.gskew_terms != T) return arg_error("banded kernel: skewed coefficients built for another term count");
        const cuuint64_t dims[2] = {(cuuint64_t)C::TWP, (cuuint64_t)a.gskew_rows};
        const cuuint32_t gbox[2] = {(cuuint32_t)C::TWP, (cuuint32_t)C::CH};
        SFB_TRY(tma_make_map(&maps.g, a.gskew, 2, dims, C::TWP, gbox, CU_TENSOR_MAP_SWIZZLE_NONE));
    }
    if (a.ld_mode == LD_PCG) {
        if (a.U == nullptr) return arg_error("banded kernel: the MO-PCG pass needs U");
        const cuuint64_t dims[2] = {(cuuint64_t)a.out_cols, (cuuint64_t)a.out_rows};
        const cuuint32_t ubox[2] = {(cuuint32_t)TX, (cuuint32_t)C::CH};
        SFB_TRY(tma_make_map(&maps.u, a.U, 2, dims, a.ldq, ubox, CU_TENSOR_MAP_SWIZZLE_NONE));
    }
    dim3 grid((a.out_cols + TX - 1) / TX, nrb);
    SFB_TRY(launch_kernel(band_kernel<T, W, MODE, FINE>, grid, dim3(NTH), smem, stream, a, maps, ry));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

template <int T, int W, int MODE>
int launch_twm(const BandArgs& a, cudaStream_t stream) {
    int ry, nrb;
    band_geometry(a.out_rows, a.out_cols, band_minb<W>(), &ry, &nrb);
    if constexpr (MODE == LD_PCG && W <= 5) {
        // 2 CTAs/SM must still fit: 4 stages of W rows (+ U) is < 110 KB for W <= 5
        static_assert(band_smem<T, W, MODE, true>() <= 110 * 1024, "fine ring too large for 2 CTAs/SM");
        if (ry <= FINE_MAX_ROWS) return launch_twmf<T, W, MODE, true>(a, ry, nrb, stream);
    }
    return launch_twmf<T, W, MODE, false>(a, ry, nrb, stream);
}

template <int T, int W>
int launch_tw(const BandArgs& a, cudaStream_t stream) {
    switch (a.ld_mode) {
        case LD_PLAIN: return launch_twm<T, W, LD_PLAIN>(a, stream);
        case LD_PCG: return launch_twm<T, W, LD_PCG>(a, stream);
    }
    if constexpr (T == 1) {  // the rhs maps are single-term
        if (a.ld_mode == LD_HEAT) return launch_twm<T, W, LD_HEAT>(a, stream);
        if (a.ld_mode == LD_DIB) return launch_twm<T, W, LD_DIB>(a, stream);
    }
    set_error("banded kernel: unsupported loader for this term count");
    return SFB_ERR_UNSUPPORTED;
}

template <int T>
int launch_t(const BandArgs& a, cudaStream_t stream) {
    switch (a.width) {
        case 1: return launch_tw<T, 1>(a, stream);
        case 3: return launch_tw<T, 3>(a, stream);
        case 5: return launch_tw<T, 5>(a, stream);
        case 7: return launch_tw<T, 7>(a, stream);
        case 9: return launch_tw<T, 9>(a, stream);
    }
    set_error("banded kernel: unsupported band width " + std::to_string(a.width));
    return SFB_ERR_UNSUPPORTED;
}

}  // namespace

bool band_supported(int nterms, int width) {
    return nterms >= 1 && nterms <= 5 && width >= 1 && width <= 9 && (width % 2) == 1;
}

int band_grid_blocks(int out_rows, int out_cols) {  // upper bound over band widths
    int ry, nrb;
    band_geometry(out_rows, out_cols, std::max(BAND_MINB, 2), &ry, &nrb);
    return ((out_cols + TX - 1) / TX) * nrb;
}

int launch_band(const BandArgs& a, cudaStream_t stream) {
    if (!band_supported(a.nterms, a.width)) {
        set_error("banded kernel: unsupported term count / width");
        return SFB_ERR_UNSUPPORTED;
    }
    if (a.out_rows <= 0 || a.out_cols <= 0) return SFB_OK;
    if ((a.ep_mode == EP_PCG) != (a.ld_mode == LD_PCG)) return arg_error("banded kernel: MO-PCG loader without its epilogue");
    if (a.ep_mode == EP_RESID && (a.ld_mode != LD_PLAIN || !a.B || !a.res || !a.partials))
        return arg_error("banded kernel: the residual epilogue needs the plain loader, B, partials and a result slot");
    if (a.ep_mode == EP_PCG && (a.goff != -(a.width - 1) / 2 || a.hoff != -(a.width - 1) / 2)) {
        set_error("banded kernel: the MO-PCG epilogue needs a centred square operator");
        return SFB_ERR_UNSUPPORTED;
    }
    if (a.gskew == nullptr || a.gskew_rows != a.out_rows + a.width - 1)
        return arg_error("banded kernel: missing skewed left-factor coefficients");
    BandArgs b = a;
    if (a.nterms == 1) return launch_t<1>(b, stream);
    if (a.nterms == 2) return launch_t<2>(b, stream);
    return launch_t<5>(b, stream);
}

// gskew[j][t * w + d] = gband[t][j - d][d] for 0 <= j - d < rows (zero
// elsewhere), j in [0, rows + w - 1), t < band_skew_terms(nterms) (the
// kernel's term slots), rows padded to an even number of doubles.
int band_skew_terms(int nterms) { return nterms <= 1 ? 1 : (nterms == 2 ? 2 : 5); }

std::vector<double> band_skew(const double* gband, int nterms, int rows, int w) {
    const int R = rows + w - 1, T = band_skew_terms(nterms), TWP = (T * w + 1) / 2 * 2;
    std::vector<double> out((size_t)R * TWP, 0.0);
    for (int t = 0; t < nterms; ++t)
        for (int j = 0; j < R; ++j)
            for (int d = 0; d < w; ++d) {
                const int i = j - d;
                if (i >= 0 && i < rows) out[(size_t)j * TWP + t * w + d] = gband[((size_t)t * rows + i) * w + d];
            }
    return out;
}

}  // namespace sfb
