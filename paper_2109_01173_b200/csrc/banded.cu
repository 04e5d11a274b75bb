// Banded multiterm sandwich  W = sum_t G_t X H_t  (one fused pass over X).
//
// Replaces the 2T dense GEMMs of SylvesterOperator.apply (operators.py:124-131)
// and the rectangular rhs builders (operators.py:206-207, 228-232, 266-268,
// 281-282).  All FEM factors are banded with half-bandwidth <= k (SURVEY
// App. B), so each output element needs a (W x W) window of X.
//
// One CTA owns a TY x TX output tile.  It stages the (TY+W-1) x (TX+W-1)
// halo of X in shared memory (applying an input transform on the way in:
// the MO-PCG direction update Q = Z + beta Q, the IMEX heat source, or the
// DIB kinetics), keeps the right-factor band of its column in registers and
// sweeps down the halo rows: Y_t(r) = sum_e X[r][c+e] h_t[e] is formed once
// per row and scattered into a ring of W partial outputs with the left-factor
// coefficients (shared-memory broadcasts).  Epilogues: plain store, or the
// MO-PCG store + <W,Q>, |Q|^2 partials with a last-block alpha step
// (solvers.py:424-431).
#include "sfb_common.cuh"
#include "sfb_kernels.cuh"
#include "sfb_launch.cuh"

namespace sfb {

namespace {

constexpr int TX = 128;
constexpr int TY = 32;

template <int W>
__host__ __device__ constexpr int wpad() {
    return W + 1;  // even: the coefficients of one halo row load as 16-byte pairs
}

template <int T, int W>
constexpr int band_smem() {
    return ((TY + W - 1) * (TX + W - 1) + T * (TY + W - 1) * wpad<W>()) * 8;
}

template <int T, int W>
__global__ void __launch_bounds__(TX) band_kernel(BandArgs a) {
    SFB_PDL_PROLOGUE();
    constexpr int HR = TY + W - 1, HC = TX + W - 1;
    extern __shared__ double sm[];
    double* Qs = sm;             // [HR][HC]
    double* Gs = sm + HR * HC;   // [T][HR][W+1]

    PcgState* st = a.pcg;
    int s = 0;
    double beta = 0.0;
    if (a.ld_mode == LD_PCG) {
        if (st->status != SFB_PCG_RUNNING) return;  // uniform gate
        s = st->iter;
        if (s > 0) beta = st->rz_next / st->rz;      // solvers.py:448-452
    }
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int c = threadIdx.x, gc = x0 + c;
    double* Qcur = (s & 1) ? a.Q1 : a.Q0;
    const double* Qprev = (s & 1) ? a.Q0 : a.Q1;

    // ---- stage the input halo (with its transform) ----
    const int urows = a.in_rows - 2 * a.rs, ucols = a.in_cols - 2 * a.cs;
    bool flag = false;
    double vmax = 0.0;
    #pragma unroll 4
    for (int idx = threadIdx.x; idx < HR * HC; idx += TX) {
        const int r = idx / HC, cc = idx - r * HC;  // HC is a compile-time constant
        const int gr = y0 + a.goff + r, gx = x0 + a.hoff + cc;
        double v = 0.0;
        if (gr >= 0 && gr < a.in_rows && gx >= 0 && gx < a.in_cols) {
            switch (a.ld_mode) {
                case LD_PCG: {
                    v = a.X[(size_t)gr * a.ldx + gx];
                    if (s > 0) v = __dadd_rn(__dmul_rn(beta, Qprev[(size_t)gr * a.ldq + gx]), v);  // Q*=beta; Q+=Z
                    if (gr >= y0 && gr < y0 + TY && gx >= x0 && gx < x0 + TX)
                        Qcur[(size_t)gr * a.ldq + gx] = v;
                    break;
                }
                case LD_HEAT: {
                    const int ur = gr - a.rs, uc = gx - a.cs;
                    const double u =
                        (ur >= 0 && ur < urows && uc >= 0 && uc < ucols) ? a.X[(size_t)ur * a.ldx + uc] : 0.0;
                    v = a.X2 ? u + a.c * a.X2[(size_t)gr * a.ldx2 + gx] : u;
                    break;
                }
                case LD_DIB: {
                    // models.py:74-82 and timestepping.py:201-207
                    const double* p = a.kp;  // alpha, gamma_k, A1, A2, B, C, D, k2, k3
                    const double eta = a.X[(size_t)gr * a.ldx + gx];
                    const double th = a.X2[(size_t)gr * a.ldx + gx];
                    if (a.species == 0) {
                        const double f = p[2] * (1.0 - th) * eta - p[3] * (eta * eta * eta) - p[4] * (th - p[0]);
                        v = eta + a.c * f;
                    } else {
                        const double g = p[5] * (1.0 + p[7] * eta) * (1.0 - th) * (1.0 - p[1] * (1.0 - th)) -
                                         p[6] * th * (1.0 + p[1] * th) * (1.0 + p[8] * eta);
                        v = th + a.c * g;
                    }
                    break;
                }
                default:
                    v = a.X[(size_t)gr * a.ldx + gx];
            }
            if (a.check != nullptr) {
                if (!isfinite(v)) flag = true;
                else vmax = fmax(vmax, fabs(v));
            }
        }
        Qs[r * HC + cc] = v;
    }
    if (a.check != nullptr) {
        if (flag) atomicOr(a.check + 1, 1ull);
        if (vmax > 0.0) atomicMax(a.check, (unsigned long long)__double_as_longlong(vmax));
    }
    // ---- left-factor coefficients of this row tile (zero outside [0,TY)) ----
    // halo-row-major: Gs[t][r][d] multiplies Y_t(r) into output row i = r - d
    constexpr int WP = wpad<W>();
    for (int idx = threadIdx.x; idx < T * HR * WP; idx += TX) {
        const int t = idx / (HR * WP), rem = idx - t * HR * WP, r = rem / WP, d = rem - r * WP;
        const int i = r - d, gi = y0 + i;
        double v = 0.0;
        if (d < W && t < a.nterms && i >= 0 && i < TY && gi < a.out_rows)
            v = a.gband[((size_t)t * a.out_rows + gi) * W + d];
        Gs[idx] = v;
    }
    // ---- right-factor band of this thread's column, in registers ----
    double h[T][W];
    #pragma unroll
    for (int t = 0; t < T; ++t)
        #pragma unroll
        for (int e = 0; e < W; ++e)
            h[t][e] = (t < a.nterms && gc < a.out_cols) ? a.hband[((size_t)t * a.out_cols + gc) * W + e] : 0.0;
    __syncthreads();

    // ---- sweep: ring of W partial output rows ----
    double acc[W];
    #pragma unroll
    for (int d = 0; d < W; ++d) acc[d] = 0.0;
    double pdot = 0.0, pqq = 0.0;
    const bool col_ok = gc < a.out_cols;
    for (int r0 = 0; r0 < HR; r0 += W) {
        #pragma unroll
        for (int u = 0; u < W; ++u) {
            const int r = r0 + u;
            if (r < HR) {
                double qv[W];
                #pragma unroll
                for (int e = 0; e < W; ++e) qv[e] = Qs[r * HC + c + e];
                #pragma unroll
                for (int t = 0; t < T; ++t) {
                    double y = 0.0;
                    #pragma unroll
                    for (int e = 0; e < W; ++e) y = fma(qv[e], h[t][e], y);
                    const double2* gp = reinterpret_cast<const double2*>(Gs + (t * HR + r) * WP);
                    #pragma unroll
                    for (int dd = 0; dd < WP / 2; ++dd) {
                        const double2 g = gp[dd];
                        const int s0 = (u - 2 * dd + 2 * W) % W;
                        acc[s0] = fma(g.x, y, acc[s0]);
                        if (2 * dd + 1 < W) {
                            const int s1 = (u - 2 * dd - 1 + 2 * W) % W;
                            acc[s1] = fma(g.y, y, acc[s1]);
                        }
                    }
                }
                const int i = r - (W - 1);
                const int slot = (u + 1) % W;
                if (i >= 0) {
                    const int gi = y0 + i;
                    if (col_ok && gi < a.out_rows) {
                        const double w = acc[slot];
                        a.W[(size_t)gi * a.ldw + gc] = w;
                        if (a.ep_mode == EP_PCG) {
                            const double q = Qs[(i - a.goff) * HC + c - a.hoff];
                            pdot = fma(w, q, pdot);
                            pqq = fma(q, q, pqq);
                        }
                    }
                    acc[slot] = 0.0;
                }
            }
        }
    }

    if (a.ep_mode == EP_PCG) {
        __shared__ double sh[TX / 32];
        const unsigned nblk = gridDim.x * gridDim.y;
        const unsigned bid = blockIdx.y * gridDim.x + blockIdx.x;
        const double p0 = block_sum<TX>(pdot, sh);
        const double p1 = block_sum<TX>(pqq, sh);
        if (threadIdx.x == 0) {
            a.partials[bid] = p0;
            a.partials[nblk + bid] = p1;
        }
        if (arrive_last(&st->counter[0], nblk)) {
            const double qw = sum_partials<TX>(a.partials, nblk, 1, sh);
            const double qq = sum_partials<TX>(a.partials + nblk, nblk, 1, sh);
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

template <int T, int W>
int launch_tw(const BandArgs& a, cudaStream_t stream) {
    constexpr int smem = band_smem<T, W>();
    static bool attr = false;
    if (!attr) {
        SFB_CUDA_TRY(cudaFuncSetAttribute(band_kernel<T, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    dim3 grid((a.out_cols + TX - 1) / TX, (a.out_rows + TY - 1) / TY);
    SFB_TRY(launch_kernel(band_kernel<T, W>, dim3(grid), dim3(TX), smem, stream, a));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
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

int band_grid_blocks(int out_rows, int out_cols) {
    return ((out_cols + TX - 1) / TX) * ((out_rows + TY - 1) / TY);
}

int launch_band(const BandArgs& a, cudaStream_t stream) {
    if (!band_supported(a.nterms, a.width)) {
        set_error("banded kernel: unsupported term count / width");
        return SFB_ERR_UNSUPPORTED;
    }
    if (a.out_rows <= 0 || a.out_cols <= 0) return SFB_OK;
    if (a.nterms == 1) return launch_t<1>(a, stream);
    if (a.nterms == 2) return launch_t<2>(a, stream);
    return launch_t<5>(a, stream);
}

}  // namespace sfb
