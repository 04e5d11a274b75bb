// Banded SPD preconditioner solves by a SPIKE partition.
//
// Z = P_L^-1 R P_R^-1 with P_L, P_R symmetric positive definite and banded
// (half-bandwidth b <= 4; the preconditioner factors of solvers.py:103-143,
// handed over as their banded Cholesky factors).  Each line (a column of R
// for P_L, a row for P_R) is an independent length-n system P y = x.  The
// line is cut into segments of S = 64 (one 64 x 64 tile per CTA); with
// D = blockdiag(P_p) and the b x b couplings E_p between neighbouring
// segments,
//
//     y_p = g_p - V_p t_{p+1} - W_p u_{p-1},   g_p = P_p^-1 x_p,
//     V_p = P_p^-1 [0; E_p],  W_p = P_p^-1 [E_{p-1}^T; 0]      (S x b spikes)
//
// where t_p / u_p are the first / last b values of y_p.  Those interface
// values solve a block-tridiagonal system with 2b x 2b blocks that is the
// same for every line, so its block-LU is precomputed and each line does one
// forward and one backward chain of P steps.  Per factor this is one tile
// pass (local solve), one per-line chain kernel and one tile pass (spike
// correction); the left factor's correction is fused with the right factor's
// local solve, so Z costs 3 tile passes + 2 chains (the triangular-solve
// formulation it replaces needed 6 + 4).
//
// The local solve P_p g = x runs in shared memory with the segment's own
// Cholesky factor (precomputed per segment): every thread sweeps one 16-long
// sub-segment of one line (256 threads = 64 lines x 4 sub-segments), a
// 4-step chain joins the sub-segments and a correction with the 16-long
// responses completes the forward solve; the backward solve repeats this
// from the other end.  Results equal the sequential banded solves up to
// rounding (the MO-PCG parity tests run in this mode).
#include <algorithm>
#include <cmath>
#include <vector>

#include "sfb_common.cuh"
#include "sfb_kernels.cuh"
#include "sfb_launch.cuh"
#include "sfb_tma.cuh"

namespace sfb {

namespace {

constexpr int S = 64;          // segment length == tile edge
constexpr int SS = 16;         // sub-segment length (one thread's sweep)
constexpr int NSUB = S / SS;   // sub-segments per segment
constexpr int NT = S * NSUB;   // threads per tile CTA
#ifndef CHAIN_L
#define CHAIN_L 8              // lines per interface-chain CTA (2B threads each; 8: 87 vs 93 us per apply at 16)
#endif

enum { DIR_COL = 0, DIR_ROW = 1 };
enum { PH_LOCAL = 0, PH_FUSED = 1 };  // plain local solve, or the previous factor's correction first

// tile[k][c] (padded): k = position along the sweep, c = line.  DIR_COL:
// lines are columns (P acts from the left), DIR_ROW: lines are rows (P acts
// from the right); the tile is stored transposed for DIR_ROW so both sweep
// along the first index.  All NT threads move the tile, coalesced along the
// contiguous global index.
template <int DIR, int NTH = NT>
__device__ __forceinline__ void tile_load(double (*tile)[S + 1], const double* X, int ld, int sweep0, int line0,
                                          int nsweep, int nlines) {
    constexpr int NSUB = NTH / S;  // row groups
    const int t = threadIdx.x, lo = t % S, hi = t / S;
    const int rb = DIR == DIR_COL ? sweep0 : line0, cb = DIR == DIR_COL ? line0 : sweep0;
    const int nr = DIR == DIR_COL ? nsweep : nlines, nc = DIR == DIR_COL ? nlines : nsweep;
    const double* p = X + (size_t)(rb + hi) * ld + cb + lo;
    const size_t step = (size_t)NSUB * ld;
    double v[S / NSUB];
    if (rb + S <= nr && cb + S <= nc) {  // interior tile (uniform)
        #pragma unroll
        for (int u = 0; u < S / NSUB; ++u) v[u] = p[u * step];
    } else {
        const bool cok = cb + lo < nc;
        #pragma unroll
        for (int u = 0; u < S / NSUB; ++u) v[u] = (cok && rb + hi + u * NSUB < nr) ? p[u * step] : 0.0;
    }
    #pragma unroll
    for (int u = 0; u < S / NSUB; ++u) {
        const int kk = hi + u * NSUB;
        if (DIR == DIR_COL) tile[kk][lo] = v[u];
        else tile[lo][kk] = v[u];
    }
}

// Store the tile; with R != nullptr also return this thread's part of
// <tile, R> over the same (valid) elements.
template <int DIR, int NTH = NT>
__device__ __forceinline__ double tile_store(double (*tile)[S + 1], double* X, int ld, int sweep0, int line0,
                                             int nsweep, int nlines, const double* R = nullptr, int ldr = 0) {
    constexpr int NSUB = NTH / S;  // row groups
    const int t = threadIdx.x, lo = t % S, hi = t / S;
    const int rb = DIR == DIR_COL ? sweep0 : line0, cb = DIR == DIR_COL ? line0 : sweep0;
    const int nr = DIR == DIR_COL ? nsweep : nlines, nc = DIR == DIR_COL ? nlines : nsweep;
    double* p = X + (size_t)(rb + hi) * ld + cb + lo;
    const double* q = R != nullptr ? R + (size_t)(rb + hi) * ldr + cb + lo : nullptr;
    const size_t step = (size_t)NSUB * ld, stepr = (size_t)NSUB * ldr;
    double dot = 0.0;
    if (rb + S <= nr && cb + S <= nc) {  // interior tile (uniform)
        if (q != nullptr) {
            double r[S / NSUB];
            #pragma unroll
            for (int u = 0; u < S / NSUB; ++u) r[u] = q[u * stepr];
            #pragma unroll
            for (int u = 0; u < S / NSUB; ++u) {
                const int kk = hi + u * NSUB;
                const double v = DIR == DIR_COL ? tile[kk][lo] : tile[lo][kk];
                p[u * step] = v;
                dot = fma(v, r[u], dot);
            }
        } else {
            #pragma unroll
            for (int u = 0; u < S / NSUB; ++u) {
                const int kk = hi + u * NSUB;
                p[u * step] = DIR == DIR_COL ? tile[kk][lo] : tile[lo][kk];
            }
        }
    } else if (cb + lo < nc) {
        #pragma unroll
        for (int u = 0; u < S / NSUB; ++u) {
            const int kk = hi + u * NSUB;
            if (rb + kk < nr) {
                const double v = DIR == DIR_COL ? tile[kk][lo] : tile[lo][kk];
                p[u * step] = v;
                if (q != nullptr) dot = fma(v, q[u * stepr], dot);
            }
        }
    }
    return dot;
}

struct SpikeArgs {
    // the factor solved in this pass
    const double* band;  // [n + B][B + 1] segment-local Cholesky rows: L[i][i-B+d] (d < B), 1/L_ii at d = B
    const double* Hf16;  // [P16][SS][B] sub-segment responses (forward, backward)
    const double* Hb16;
    const double* Tf16;  // [P16][B][B] sub-segment transfers
    const double* Tb16;
    const double* V;     // [P][S][B] spikes
    const double* W;
    double* sv;          // [P][2B][nlines] interface values / solution
    int n, nlines;
    // PH_FUSED: the previous (left) factor's correction, applied first
    const double* pV;
    const double* pW;
    const double* psv;
    int pn;              // order of the previous factor (= this pass's nlines)
    const double* Xin;
    int ldi;
    double* X;
    int ld;
    // <Z,R> (spike_fix_kernel of the right factor)
    const double* R;
    int ldr;
    double* partials;
    unsigned* counter;
    PcgState* pcg;
    double* dot_out;
    const PcgState* gate;
};

// Two-level triangular solve of the tile's lines in place (zero state at the
// segment boundary).  FWD: L y = x with L's rows in bandS; otherwise L^T.
// Every thread sweeps its 16-row sub-segment with a zero incoming state and
// parks the sub-segment's outgoing boundary values (last / first B of the
// local solution) in sst; after one barrier each thread chains the boundary
// values of the sub-segments before it (at most 3 steps of B x B work)
// itself and corrects its own rows: two barriers per direction, no idle
// phase.
template <int B, bool FWD>
__device__ __forceinline__ void tile_solve(double (*tile)[S + 1], double (*sst)[B > 0 ? B : 1][S],
                                           const double* bandS, const double* H16s, const double* T16s, int len,
                                           int c, int k, bool live) {
    constexpr int BB = B > 0 ? B : 1;
    const int a0 = min(k * SS, len), a1 = min(k * SS + SS, len);  // this thread's rows
    if (live && a0 < a1) {
        double w[BB];
        #pragma unroll
        for (int d = 0; d < BB; ++d) w[d] = 0.0;
        if (FWD) {
            for (int kk = a0; kk < a1; ++kk) {
                const double* cb = bandS + kk * (B + 1);
                double v = tile[kk][c];
                #pragma unroll
                for (int d = 0; d < B; ++d) v = fma(-cb[d], w[d], v);
                v *= cb[B];
                #pragma unroll
                for (int d = 0; d + 1 < B; ++d) w[d] = w[d + 1];
                if (B > 0) w[B - 1] = v;
                tile[kk][c] = v;
            }
        } else {
            for (int kk = a1 - 1; kk >= a0; --kk) {  // w[e-1] = z[kk+e]
                double v = tile[kk][c];
                #pragma unroll
                for (int e = B; e >= 1; --e) v = fma(-bandS[(kk + e) * (B + 1) + B - e], w[e - 1], v);
                v *= bandS[kk * (B + 1) + B];
                #pragma unroll
                for (int e = B - 1; e >= 1; --e) w[e] = w[e - 1];
                if (B > 0) w[0] = v;
                tile[kk][c] = v;
            }
        }
        // outgoing boundary values of this sub-segment's local solution, in
        // the order the transfer matrices expect (zero-padded when shorter than B)
        #pragma unroll
        for (int d = 0; d < B; ++d) {
            const int r = FWD ? a1 - B + d : a0 + d;
            const bool inside = FWD ? r >= a0 : r < a1;
            sst[k][d][c] = inside ? tile[r][c] : 0.0;
        }
    }
    __syncthreads();
    if (B == 0) return;
    const int kfirst = FWD ? 0 : (len - 1) / SS;  // first sub-segment in sweep order
    if (live && a0 < a1 && k != kfirst) {
        double s[BB];
        #pragma unroll
        for (int d = 0; d < BB; ++d) s[d] = 0.0;
        #pragma unroll
        for (int step = 0; step < NSUB - 1; ++step) {
            const int kk = FWD ? step : kfirst - step;  // sub-segments before mine, in sweep order
            if (FWD ? kk < k : kk > k) {
                const double* T = T16s + kk * BB * BB;
                double nx[BB];
                #pragma unroll
                for (int d = 0; d < B; ++d) {
                    double v = sst[kk][d][c];
                    #pragma unroll
                    for (int e = 0; e < B; ++e) v = fma(T[d * B + e], s[e], v);
                    nx[d] = v;
                }
                #pragma unroll
                for (int d = 0; d < B; ++d) s[d] = nx[d];
            }
        }
        const double* H = H16s + k * SS * BB;
        for (int kk = a0; kk < a1; ++kk) {
            double v = tile[kk][c];
            #pragma unroll
            for (int d = 0; d < B; ++d) v = fma(H[(kk - a0) * B + d], s[d], v);
            tile[kk][c] = v;
        }
    }
    __syncthreads();
}

template <int B, int DIR, int PH>
__global__ void __launch_bounds__(NT) spike_tile_kernel(SpikeArgs a) {
    SFB_PDL_PROLOGUE();
    if (a.gate != nullptr && a.gate->status != SFB_PCG_RUNNING) return;
    constexpr int BB = B > 0 ? B : 1;
    __shared__ double tile[S][S + 1];
    __shared__ double sst[NSUB][BB][S];     // incoming states of the sub-segments, per line
    __shared__ double bandS[(S + 4) * 5];   // rows start .. start+S+B-1 of the segment factor
    __shared__ double H16s[NSUB * SS * BB];
    __shared__ double T16s[NSUB * BB * BB];
    // PH_FUSED: the previous factor's spikes, used before the local solve
    // needs sst, aliased onto it (2 S B <= NSUB B S)
    double (*VWs)[S * BB] = reinterpret_cast<double (*)[S * BB]>(&sst[0][0][0]);
    const int p = blockIdx.x;             // segment along the sweep
    const int line0 = blockIdx.y * S;     // first line of this tile
    const int start = p * S;
    const int len = min(S, a.n - start);
    const int t = threadIdx.x, c = t % S, k = t / S;  // line, sub-segment
    const int gl = line0 + c;
    const bool live = gl < a.nlines;

    for (int i = t; i < (S + B) * (B + 1); i += NT) {
        const int row = start + i / (B + 1);
        bandS[i] = row < a.n + B ? a.band[(size_t)start * (B + 1) + i] : 0.0;
    }
    if (PH == PH_FUSED && B > 0) {
        // the previous factor acts along this tile's lines: its segment is blockIdx.y
        const int pp = blockIdx.y;
        for (int i = t; i < S * B; i += NT) {
            VWs[0][i] = a.pV[(size_t)pp * S * B + i];
            VWs[1][i] = a.pW[(size_t)pp * S * B + i];
        }
    }
    tile_load<DIR>(tile, a.Xin, a.ldi, start, line0, a.n, a.nlines);
    __syncthreads();

    if (PH == PH_FUSED && B > 0) {
        // previous factor's spike correction, in the transposed view: its lines
        // are this tile's sweep positions (k index), its rows this tile's lines
        const int pp = blockIdx.y, pP = (a.pn + S - 1) / S;
        const int pc = t % S;  // previous factor's line = this tile's column position
        const int gpc = start + pc;
        if (gpc < a.n) {
            double tn[BB], up[BB];
            #pragma unroll
            for (int d = 0; d < B; ++d) {
                tn[d] = pp + 1 < pP ? a.psv[((size_t)(pp + 1) * 2 * B + d) * a.n + gpc] : 0.0;
                up[d] = pp > 0 ? a.psv[((size_t)(pp - 1) * 2 * B + B + d) * a.n + gpc] : 0.0;
            }
            #pragma unroll 4
            for (int r = t / S; r < S; r += NSUB) {  // r: previous factor's position (this tile's line)
                double v = tile[pc][r];
                #pragma unroll
                for (int d = 0; d < B; ++d) {
                    v = fma(-VWs[0][r * B + d], tn[d], v);
                    v = fma(-VWs[1][r * B + d], up[d], v);
                }
                tile[pc][r] = v;
            }
        }
        __syncthreads();
    }

    // local solve P_p g = x: forward with L_p, backward with L_p^T
    const int n16 = (a.n + SS - 1) / SS;
    for (int i = t; i < NSUB * SS * BB; i += NT)
        H16s[i] = p * NSUB + i / (SS * BB) < n16 ? a.Hf16[(size_t)p * NSUB * SS * BB + i] : 0.0;
    for (int i = t; i < NSUB * BB * BB; i += NT)
        T16s[i] = p * NSUB + i / (BB * BB) < n16 ? a.Tf16[(size_t)p * NSUB * BB * BB + i] : 0.0;
    __syncthreads();
    tile_solve<B, true>(tile, sst, bandS, H16s, T16s, len, c, k, live);
    for (int i = t; i < NSUB * SS * BB; i += NT)
        H16s[i] = p * NSUB + i / (SS * BB) < n16 ? a.Hb16[(size_t)p * NSUB * SS * BB + i] : 0.0;
    for (int i = t; i < NSUB * BB * BB; i += NT)
        T16s[i] = p * NSUB + i / (BB * BB) < n16 ? a.Tb16[(size_t)p * NSUB * BB * BB + i] : 0.0;
    __syncthreads();
    tile_solve<B, false>(tile, sst, bandS, H16s, T16s, len, c, k, live);
    if (B > 0 && live && k == 0) {
        // interface values of g: first B and last B rows of the segment
        #pragma unroll
        for (int d = 0; d < B; ++d) {
            a.sv[((size_t)p * 2 * B + d) * a.nlines + gl] = d < len ? tile[d][c] : 0.0;
            const int r = len - B + d;
            a.sv[((size_t)p * 2 * B + B + d) * a.nlines + gl] = r >= 0 ? tile[r][c] : 0.0;
        }
    }
    tile_store<DIR>(tile, a.X, a.ld, start, line0, a.n, a.nlines);
}

// Interface system of one factor, one thread per line: block-LU forward
// chain d_p = K_p gamma_p - KA_p u(d_{p-1}), backward z_p = d_p - Ch_p t(z_{p+1})
// (K, KA, Ch precomputed; read through L1, the same for every line).  The CTA
// first stages its lines' gamma values in shared memory with all loads in
// flight, runs both chains there in place (every operand off the chain is a
// shared-memory or L1 load that can be issued early) and writes the
// interface solution z_p = (t_p, u_p) back in one coalesced pass.
// Spike correction y = g - V_p t_{p+1} - W_p u_{p-1} of one 64 x 64 tile,
// register to register: each thread keeps the tile elements of one global
// column (the load/store mapping of tile_load/tile_store, coalesced) and
// the interface values of the tile's 64 lines come from shared memory.
// <Z,R> optional (one partial per CTA, last CTA sums them in order).
template <int B, int DIR>
__global__ void __launch_bounds__(NT) spike_fix_kernel(SpikeArgs a) {
    SFB_PDL_PROLOGUE();
    if (a.gate != nullptr && a.gate->status != SFB_PCG_RUNNING) return;
    constexpr int BB = B > 0 ? B : 1;
    __shared__ double tu[2][BB][S];     // t_{p+1}, u_{p-1} of the tile's lines
    __shared__ double VW[2][S][BB];     // this segment's spikes
    const int p = blockIdx.x, line0 = blockIdx.y * S, start = p * S;
    const int P = (a.n + S - 1) / S;
    const int t = threadIdx.x, lo = t % S, hi = t / S;
    for (int i = t; i < 2 * B * S; i += NT) {
        const int which = i / (B * S), d = (i / S) % B, l = i % S, gl = line0 + l;
        double v = 0.0;
        if (gl < a.nlines) {
            if (which == 0 && p + 1 < P) v = a.sv[((size_t)(p + 1) * 2 * B + d) * a.nlines + gl];
            if (which == 1 && p > 0) v = a.sv[((size_t)(p - 1) * 2 * B + B + d) * a.nlines + gl];
        }
        tu[which][d][l] = v;
    }
    for (int i = t; i < S * B; i += NT) {
        VW[0][i / B][i % B] = a.V[(size_t)p * S * B + i];
        VW[1][i / B][i % B] = a.W[(size_t)p * S * B + i];
    }
    __syncthreads();
    // global rows rb + hi + NSUB u, column cb + lo (as tile_load/tile_store)
    const int rb = DIR == DIR_COL ? start : line0, cb = DIR == DIR_COL ? line0 : start;
    const int nr = DIR == DIR_COL ? a.n : a.nlines, nc = DIR == DIR_COL ? a.nlines : a.n;
    const bool cok = cb + lo < nc;
    const double* gp = a.Xin + (size_t)(rb + hi) * a.ldi + cb + lo;
    double* yp = a.X + (size_t)(rb + hi) * a.ld + cb + lo;
    const double* rp = a.R != nullptr ? a.R + (size_t)(rb + hi) * a.ldr + cb + lo : nullptr;
    const size_t si = (size_t)NSUB * a.ldi, so = (size_t)NSUB * a.ld, sr = (size_t)NSUB * a.ldr;
    double g[S / NSUB], r[S / NSUB];
    #pragma unroll
    for (int u = 0; u < S / NSUB; ++u) {
        const bool ok = cok && rb + hi + u * NSUB < nr;
        g[u] = ok ? gp[u * si] : 0.0;
        r[u] = (ok && rp != nullptr) ? rp[u * sr] : 0.0;
    }
    double dot = 0.0;
    #pragma unroll
    for (int u = 0; u < S / NSUB; ++u) {
        const int kk = hi + u * NSUB;             // tile row
        const int pos = DIR == DIR_COL ? kk : lo;  // position along the sweep
        const int ln = DIR == DIR_COL ? lo : kk;   // line within the tile
        double v = g[u];
        #pragma unroll
        for (int d = 0; d < B; ++d) {
            v = fma(-VW[0][pos][d], tu[0][d][ln], v);
            v = fma(-VW[1][pos][d], tu[1][d][ln], v);
        }
        if (cok && rb + kk < nr) {
            yp[u * so] = v;
            dot = fma(v, r[u], dot);
        }
    }
    if (a.R != nullptr) {
        __shared__ double sh[NT / 32];
        const double part = block_sum<NT>(dot, sh);
        const unsigned nblk = gridDim.x * gridDim.y;
        if (threadIdx.x == 0) a.partials[blockIdx.y * gridDim.x + blockIdx.x] = part;
        if (arrive_last(a.counter, nblk)) {
            const double tot = sum_partials<NT>(a.partials, nblk, 1, sh);
            if (threadIdx.x == 0) {
                *a.counter = 0;
                if (a.pcg != nullptr) a.pcg->rz_next = tot;
                if (a.dot_out != nullptr) *a.dot_out = tot;
            }
        }
    }
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}

// One line's interface chain is spread over 2B threads (one per interface
// value, consecutive lanes): each thread forms one row of the 2B x 2B block
// step and the b values the next step needs travel by shuffle, so the
// sequential critical path per step is two FMAs and a shuffle instead of a
// whole block product, and the 2047-line chain occupies 4x the warps.
// The two sweeps of one line's interface chain (the kernel below); inlined
// once with the staged shared-memory coefficients and once with the global
// ones, so every shared access compiles to LDS (a pointer that may point to
// either space compiles to generic loads).  The step-to-step dependence is
// only through the b interface values (prev / nx): K_p gamma_p is formed one
// step ahead.
template <int B>
__device__ __forceinline__ void chain_lines(const double* __restrict__ cf, double* gs, double* sv, int nlines, int P,
                                            int line0, int l, int i, bool live, int gbase) {
    constexpr int B2 = 2 * B;
    constexpr int L = CHAIN_L;
    constexpr int PER = B2 * B2 + 2 * B2 * B;
    const unsigned gmask = 0xffffffffu;
    const bool line_ok = line0 + l < nlines;
    auto kdot = [&](int p) {
        const double* K = cf + (size_t)p * PER + i * B2;
        double a0 = 0.0, a1 = 0.0;
        #pragma unroll
        for (int j = 0; j < B2; j += 2) {
            a0 = fma(K[j], line_ok ? gs[(p * B2 + j) * L + l] : 0.0, a0);
            a1 = fma(K[j + 1], line_ok ? gs[(p * B2 + j + 1) * L + l] : 0.0, a1);
        }
        return a0 + a1;
    };
    double prev[B];  // u part of d_{p-1}
    #pragma unroll
    for (int d = 0; d < B; ++d) prev[d] = 0.0;
    double kg = kdot(0);
    for (int p = 0; p < P; ++p) {
        const double kg_p = kg;
        if (p + 1 < P) kg = kdot(p + 1);
        const double* KA = cf + (size_t)p * PER + B2 * B2 + i * B;
        double v = kg_p;
        #pragma unroll
        for (int j = 0; j < B; ++j) v = fma(-KA[j], prev[j], v);
        __syncwarp();  // the line's other rows have read step p's values
        if (live) gs[(p * B2 + i) * L + l] = v;
        #pragma unroll
        for (int d = 0; d < B; ++d) prev[d] = __shfl_sync(gmask, v, gbase + B + d);
    }
    __syncwarp();
    double nx[B];  // t part of z_{p+1}
    #pragma unroll
    for (int d = 0; d < B; ++d) nx[d] = 0.0;
    for (int p = P - 1; p >= 0; --p) {
        const double* Ch = cf + (size_t)p * PER + B2 * B2 + B2 * B + i * B;
        double v = live ? gs[(p * B2 + i) * L + l] : 0.0;
        #pragma unroll
        for (int j = 0; j < B; ++j) v = fma(-Ch[j], nx[j], v);
        if (live) sv[((size_t)p * B2 + i) * nlines + line0 + l] = v;
        #pragma unroll
        for (int d = 0; d < B; ++d) nx[d] = __shfl_sync(gmask, v, gbase + d);
    }
}

__host__ __device__ constexpr int chain_group(int b) { return b == 1 ? 2 : (b == 2 ? 4 : 8); }  // 2B -> power of 2

template <int B>
__global__ void __launch_bounds__(CHAIN_L * chain_group(B)) spike_chain_kernel(int nlines, int P, const double* __restrict__ coef,
                                                                      double* sv, int coef_in_smem,
                                                                      const PcgState* gate) {
    SFB_PDL_PROLOGUE();
    if (gate != nullptr && gate->status != SFB_PCG_RUNNING) return;
    constexpr int B2 = 2 * B;
    constexpr int L = CHAIN_L;                 // lines per CTA
    constexpr int PER = B2 * B2 + 2 * B2 * B;  // K (2B x 2B), KA (2B x B), Ch (2B x B)
    extern __shared__ double gs[];             // [P][2B][L], then the coefficients when they fit
    constexpr int GP = chain_group(B);         // lanes per line (2B rounded up to a power of two)
    const int t = threadIdx.x, l = t / GP, i0 = t % GP, line0 = blockIdx.x * L;
    const bool live = line0 + l < nlines && i0 < B2;
    const int i = i0 < B2 ? i0 : 0;            // padding lanes mirror row 0 and store nothing
    const unsigned gmask = 0xffffffffu;        // whole warps (GP divides 32): every lane shuffles
    const int gbase = (t & 31) - i0;           // lane of this line's row 0
    // stage with every load in flight: the coefficients (the same block for
    // every CTA, P * PER doubles) as one bulk copy, the lines' values by cp.async
    double* cs = gs + (size_t)P * B2 * L;
    __shared__ __align__(8) uint64_t cbar;
    if (coef_in_smem && t == 0) {
        mbar_init_u32(smem_u32(&cbar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t bytes = (uint32_t)P * PER * 8;
        mbar_expect_tx_u32(smem_u32(&cbar), bytes);
        bulk_load_u32(smem_u32(cs), coef, bytes, smem_u32(&cbar));
    }
    {  // consecutive threads take consecutive lines of one row (coalesced segments)
        const int nl = min(L, nlines - line0);
        for (int k = t; k < P * B2 * L; k += L * GP) {
            const int row = k / L, ll = k - row * L;
            if (ll < nl) cp_async8(gs + row * L + ll, sv + (size_t)row * nlines + line0 + ll);
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();  // (also publishes the barrier init)
    if (coef_in_smem) {
        mbar_wait_u32(smem_u32(&cbar), 0);
        chain_lines<B>(cs, gs, sv, nlines, P, line0, l, i, live, gbase);  // shared-space coefficient reads
    } else {
        chain_lines<B>(coef, gs, sv, nlines, P, line0, l, i, live, gbase);
    }
}

template <int B>
int chain(const SpikeFactor& f, int nlines, double* sv, const PcgState* gate, cudaStream_t s) {
    if constexpr (B == 0) {
        return SFB_OK;  // diagonal factor: no interfaces
    } else {
        const int P = (f.n + S - 1) / S;
        constexpr size_t cap = 200 * 1024;
        constexpr int L = CHAIN_L;
        size_t sm = (size_t)P * 2 * B * L * 8;
        if (sm > cap) {
            set_error("banded preconditioner: order too large for the interface chain");
            return SFB_ERR_UNSUPPORTED;
        }
        const size_t csm = (size_t)P * (8 * B * B) * 8;
        const int cin = sm + csm <= cap ? 1 : 0;  // staged coefficients (measured: L1 reads 20 % slower)
        if (cin) sm += csm;
        SFB_TRY(ensure_dynamic_smem(spike_chain_kernel<B>, sm));
        return launch_kernel(spike_chain_kernel<B>, dim3((nlines + L - 1) / L), dim3(L * chain_group(B)), sm, s, nlines, P,
                             f.coef, sv, cin, gate);
    }
}

SpikeArgs args_for(const SpikeFactor& f, int nlines, double* sv, const PcgState* gate) {
    SpikeArgs a{};
    a.band = f.band;
    a.Hf16 = f.Hf16;
    a.Hb16 = f.Hb16;
    a.Tf16 = f.Tf16;
    a.Tb16 = f.Tb16;
    a.V = f.V;
    a.W = f.W;
    a.sv = sv;
    a.n = f.n;
    a.nlines = nlines;
    a.gate = gate;
    return a;
}

template <int BL, int BR>
int run_pair(const SpikeFactor& L, const SpikeFactor& Rf, const double* Rin, int ldr, double* Z, int ldz,
             const SegDot* dot, double* svL, double* svR, const PcgState* gate, cudaStream_t s) {
    const int qy = L.n, qx = Rf.n;
    const dim3 gL((qy + S - 1) / S, (qx + S - 1) / S), gR((qx + S - 1) / S, (qy + S - 1) / S);
    // left factor: local solve along columns, interface chain
    SpikeArgs a = args_for(L, qx, svL, gate);
    a.Xin = Rin;
    a.ldi = ldr;
    a.X = Z;
    a.ld = ldz;
    SFB_TRY(launch_kernel(spike_tile_kernel<BL, DIR_COL, PH_LOCAL>, gL, dim3(NT), 0, s, a));
    SFB_TRY(chain<BL>(L, qx, svL, gate, s));
    // right factor: (left correction +) local solve along rows, chain, correction (+ <Z,R>)
    SpikeArgs b = args_for(Rf, qy, svR, gate);
    b.Xin = Z;
    b.ldi = ldz;
    b.X = Z;
    b.ld = ldz;
    if (BL == BR) {
        b.pV = L.V;
        b.pW = L.W;
        b.psv = svL;
        b.pn = qy;
        SFB_TRY(launch_kernel(spike_tile_kernel<BR, DIR_ROW, PH_FUSED>, gR, dim3(NT), 0, s, b));
    } else {
        SpikeArgs c = a;
        c.Xin = Z;
        c.ldi = ldz;
        SFB_TRY(launch_kernel(spike_fix_kernel<BL, DIR_COL>, gL, dim3(NT), 0, s, c));
        SFB_TRY(launch_kernel(spike_tile_kernel<BR, DIR_ROW, PH_LOCAL>, gR, dim3(NT), 0, s, b));
    }
    SFB_TRY(chain<BR>(Rf, qy, svR, gate, s));
    if (dot != nullptr) {
        b.R = dot->R;
        b.ldr = dot->ldr;
        b.partials = dot->partials;
        b.counter = dot->counter;
        b.pcg = dot->pcg;
        b.dot_out = dot->dot_out;
    }
    return launch_kernel(spike_fix_kernel<BR, DIR_ROW>, gR, dim3(NT), 0, s, b);
}

template <int BL>
int run_bl(const SpikeFactor& L, const SpikeFactor& R, const double* Rin, int ldr, double* Z, int ldz,
           const SegDot* dot, double* svL, double* svR, const PcgState* gate, cudaStream_t s) {
    switch (R.b) {
        case 0: return run_pair<BL, 0>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
        case 1: return run_pair<BL, 1>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
        case 2: return run_pair<BL, 2>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
        case 3: return run_pair<BL, 3>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
        case 4: return run_pair<BL, 4>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
    }
    return arg_error("banded preconditioner: half-bandwidth 0..4");
}

// ---------------------------------------------------------------- host ----
// dense helpers for the 2b x 2b interface algebra
using Mat = std::vector<double>;
Mat mat_mul(const Mat& A, const Mat& B, int n, int m, int k) {  // (n x m)(m x k)
    Mat C((size_t)n * k, 0.0);
    for (int i = 0; i < n; ++i)
        for (int l = 0; l < m; ++l)
            for (int j = 0; j < k; ++j) C[(size_t)i * k + j] += A[(size_t)i * m + l] * B[(size_t)l * k + j];
    return C;
}
bool mat_inv(Mat A, int n, Mat& inv) {  // Gauss-Jordan, partial pivoting
    inv.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) inv[(size_t)i * n + i] = 1.0;
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (std::fabs(A[(size_t)r * n + c]) > std::fabs(A[(size_t)piv * n + c])) piv = r;
        if (A[(size_t)piv * n + c] == 0.0) return false;
        for (int j = 0; j < n; ++j) {
            std::swap(A[(size_t)c * n + j], A[(size_t)piv * n + j]);
            std::swap(inv[(size_t)c * n + j], inv[(size_t)piv * n + j]);
        }
        const double d = 1.0 / A[(size_t)c * n + c];
        for (int j = 0; j < n; ++j) {
            A[(size_t)c * n + j] *= d;
            inv[(size_t)c * n + j] *= d;
        }
        for (int r = 0; r < n; ++r) {
            if (r == c) continue;
            const double m = A[(size_t)r * n + c];
            if (m == 0.0) continue;
            for (int j = 0; j < n; ++j) {
                A[(size_t)r * n + j] -= m * A[(size_t)c * n + j];
                inv[(size_t)r * n + j] -= m * inv[(size_t)c * n + j];
            }
        }
    }
    return true;
}

}  // namespace

int spike_length() { return S; }

int launch_spike_pre(const SpikeFactor& L, const SpikeFactor& R, const double* Rin, int ldr, double* Z, int ldz,
                     const SegDot* dot, double* svL, double* svR, const PcgState* gate, cudaStream_t s) {
    switch (L.b) {
        case 0: return run_bl<0>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
        case 1: return run_bl<1>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
        case 2: return run_bl<2>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
        case 3: return run_bl<3>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
        case 4: return run_bl<4>(L, R, Rin, ldr, Z, ldz, dot, svL, svR, gate, s);
    }
    return arg_error("banded preconditioner: half-bandwidth 0..4");
}

size_t spike_interface_doubles(int n, int b, int nlines) {
    return (size_t)((n + S - 1) / S) * 2 * std::max(b, 1) * nlines;
}

// Host precompute from the global banded Cholesky factor C (band[i][d] =
// C[i][i-b+d] for d < b, band[i][b] = 1/C_ii, the layout of
// solvers.py::_cholesky_band): P = C C^T, per-segment Cholesky factors,
// spikes, the interface block-LU and the 16-long sub-segment responses.
int build_spike_factor(int n, int b, const double* cband, SpikeFactor& f) {
    const int bb = std::max(b, 1), P = (n + S - 1) / S;
    auto Cg = [&](int i, int j) -> double {  // C[i][j], lower banded
        if (j > i || i - j > b || j < 0) return 0.0;
        if (i == j) return 1.0 / cband[(size_t)i * (b + 1) + b];
        return cband[(size_t)i * (b + 1) + (j - i + b)];
    };
    auto Pm = [&](int i, int j) -> double {  // (C C^T)[i][j]
        if (i < 0 || j < 0 || i >= n || j >= n || std::abs(i - j) > b) return 0.0;
        double v = 0.0;
        for (int k = std::max(std::max(i, j) - b, 0); k <= std::min(i, j); ++k) v += Cg(i, k) * Cg(j, k);
        return v;
    };
    // segment-local Cholesky factors in the device band layout
    std::vector<double> band((size_t)(n + b) * (b + 1), 0.0);
    std::vector<double> Lf((size_t)n * (b + 1), 0.0);  // L[i][i-d] at d (d = 0 diagonal)
    for (int p = 0; p < P; ++p) {
        const int s0 = p * S, s1 = std::min(n, s0 + S);
        for (int i = s0; i < s1; ++i) {
            for (int d = std::min(b, i - s0); d >= 0; --d) {  // L[i][j], j = i - d
                const int j = i - d;
                double v = Pm(i, j);
                for (int k = std::max(std::max(i, j) - b, s0); k < j; ++k) v -= Lf[(size_t)i * (b + 1) + (i - k)] *
                                                                            Lf[(size_t)j * (b + 1) + (j - k)];
                if (d == 0) {
                    if (!(v > 0.0)) {
                        set_error("banded preconditioner: a segment block is not positive definite");
                        return SFB_ERR_ARG;
                    }
                    Lf[(size_t)i * (b + 1)] = std::sqrt(v);
                } else {
                    Lf[(size_t)i * (b + 1) + d] = v / Lf[(size_t)j * (b + 1)];
                }
            }
            for (int d = 1; d <= b; ++d) band[(size_t)i * (b + 1) + (b - d)] = i - d >= s0 ? Lf[(size_t)i * (b + 1) + d] : 0.0;
            band[(size_t)i * (b + 1) + b] = 1.0 / Lf[(size_t)i * (b + 1)];
        }
    }
    auto seg_solve = [&](int p, std::vector<double>& x) {  // P_p x = rhs, x has the segment's length
        const int s0 = p * S, len = (int)x.size();
        for (int k = 0; k < len; ++k) {  // L y = x
            const int i = s0 + k;
            double v = x[k];
            for (int d = 1; d <= std::min(b, k); ++d) v -= Lf[(size_t)i * (b + 1) + d] * x[k - d];
            x[k] = v / Lf[(size_t)i * (b + 1)];
        }
        for (int k = len - 1; k >= 0; --k) {  // L^T z = y
            const int i = s0 + k;
            double v = x[k];
            for (int d = 1; d <= b && k + d < len; ++d) v -= Lf[(size_t)(i + d) * (b + 1) + d] * x[k + d];
            x[k] = v / Lf[(size_t)i * (b + 1)];
        }
    };
    // spikes V_p = P_p^-1 [0; E_p], W_p = P_p^-1 [E_{p-1}^T; 0]
    std::vector<double> V((size_t)P * S * bb, 0.0), W((size_t)P * S * bb, 0.0);
    for (int p = 0; p < P; ++p) {
        const int s0 = p * S, len = std::min(S, n - s0), s1 = s0 + len;
        for (int j = 0; j < b; ++j) {
            std::vector<double> x(len, 0.0);
            if (s1 < n) {
                for (int r = std::max(0, len - b); r < len; ++r) x[r] = Pm(s0 + r, s1 + j);
                seg_solve(p, x);
                for (int r = 0; r < len; ++r) V[((size_t)p * S + r) * bb + j] = x[r];
            }
            std::fill(x.begin(), x.end(), 0.0);
            if (p > 0) {
                for (int r = 0; r < std::min(b, len); ++r) x[r] = Pm(s0 + r, s0 - b + j);
                seg_solve(p, x);
                for (int r = 0; r < len; ++r) W[((size_t)p * S + r) * bb + j] = x[r];
            }
        }
    }
    // interface block-LU: z_p + Abar_p z_{p-1} + Cbar_p z_{p+1} = gamma_p
    const int B2 = 2 * b, PER = B2 * B2 + 2 * B2 * b;
    std::vector<double> coef((size_t)P * std::max(PER, 1), 0.0);
    if (b > 0) {
        Mat Chat((size_t)B2 * B2, 0.0);  // previous \hat C (2b x 2b)
        for (int p = 0; p < P; ++p) {
            const int len = std::min(S, n - p * S);
            auto spike_rows = [&](const std::vector<double>& Sp, Mat& M) {  // (t rows; u rows) x b
                M.assign((size_t)B2 * b, 0.0);
                for (int d = 0; d < b; ++d)
                    for (int j = 0; j < b; ++j) {
                        M[(size_t)d * b + j] = d < len ? Sp[((size_t)p * S + d) * bb + j] : 0.0;
                        const int r = len - b + d;
                        M[(size_t)(b + d) * b + j] = r >= 0 ? Sp[((size_t)p * S + r) * bb + j] : 0.0;
                    }
            };
            Mat A, Cm;
            spike_rows(W, A);   // acts on u_{p-1}
            spike_rows(V, Cm);  // acts on t_{p+1}
            Mat Abar((size_t)B2 * B2, 0.0), Cbar((size_t)B2 * B2, 0.0);
            for (int i = 0; i < B2; ++i)
                for (int j = 0; j < b; ++j) {
                    Abar[(size_t)i * B2 + b + j] = A[(size_t)i * b + j];
                    Cbar[(size_t)i * B2 + j] = Cm[(size_t)i * b + j];
                }
            Mat M((size_t)B2 * B2, 0.0);
            for (int i = 0; i < B2; ++i) M[(size_t)i * B2 + i] = 1.0;
            if (p > 0) {
                const Mat AC = mat_mul(Abar, Chat, B2, B2, B2);
                for (size_t i = 0; i < M.size(); ++i) M[i] -= AC[i];
            }
            Mat K;
            if (!mat_inv(M, B2, K)) {
                set_error("banded preconditioner: singular interface system");
                return SFB_ERR_ARG;
            }
            const Mat KA = mat_mul(K, Abar, B2, B2, B2);
            Chat = mat_mul(K, Cbar, B2, B2, B2);
            double* cp = coef.data() + (size_t)p * PER;
            for (int i = 0; i < B2 * B2; ++i) cp[i] = K[i];
            for (int i = 0; i < B2; ++i)
                for (int j = 0; j < b; ++j) {
                    cp[B2 * B2 + i * b + j] = KA[(size_t)i * B2 + b + j];  // u columns
                    cp[B2 * B2 + B2 * b + i * b + j] = Chat[(size_t)i * B2 + j];  // t columns
                }
        }
    }
    // 16-long sub-segment responses of the segment-local factor (zero state at
    // every sub-segment start; couplings across a 64-segment start are zero)
    const int P16 = (n + SS - 1) / SS;
    std::vector<double> Hf16((size_t)P16 * SS * bb, 0.0), Hb16((size_t)P16 * SS * bb, 0.0);
    std::vector<double> Tf16((size_t)P16 * bb * bb, 0.0), Tb16((size_t)P16 * bb * bb, 0.0);
    auto Lb = [&](int i, int d) { return band[(size_t)i * (b + 1) + d]; };  // device layout
    std::vector<double> w(bb);
    for (int q = 0; q < P16; ++q) {
        const int start = q * SS, len = std::min(SS, n - start), end = start + len;
        for (int d = 0; d < b; ++d) {
            std::fill(w.begin(), w.end(), 0.0);
            w[d] = 1.0;
            for (int k = 0; k < len; ++k) {
                const int i = start + k;
                double v = 0.0;
                for (int e = 0; e < b; ++e) v -= Lb(i, e) * w[e];
                v *= Lb(i, b);
                for (int e = 0; e + 1 < b; ++e) w[e] = w[e + 1];
                w[b - 1] = v;
                Hf16[((size_t)q * SS + k) * bb + d] = v;
            }
            for (int o = 0; o < b; ++o) {
                const int r = end - b + o;
                Tf16[((size_t)q * bb + o) * bb + d] = r >= start ? Hf16[((size_t)q * SS + (r - start)) * bb + d]
                                                                 : (r - (start - b) == d ? 1.0 : 0.0);
            }
            std::fill(w.begin(), w.end(), 0.0);
            w[d] = 1.0;
            for (int k = len - 1; k >= 0; --k) {
                const int i = start + k;
                double v = 0.0;
                for (int e = b; e >= 1; --e) v -= (i + e < n + b ? Lb(i + e, b - e) : 0.0) * w[e - 1];
                v *= Lb(i, b);
                for (int e = b - 1; e >= 1; --e) w[e] = w[e - 1];
                w[0] = v;
                Hb16[((size_t)q * SS + k) * bb + d] = v;
            }
            for (int o = 0; o < b; ++o) {
                const int r = start + o;
                Tb16[((size_t)q * bb + o) * bb + d] = r < end ? Hb16[((size_t)q * SS + (r - start)) * bb + d]
                                                             : (r - end == d ? 1.0 : 0.0);
            }
        }
    }
    f.n = n;
    f.b = b;
    auto up = [](double** dst, const std::vector<double>& v) {
        if (dalloc(dst, v.size()) != SFB_OK) return SFB_ERR_NOMEM;
        if (cudaMemcpy(*dst, v.data(), v.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
            set_error("uploading banded preconditioner failed");
            return SFB_ERR_CUDA;
        }
        return SFB_OK;
    };
    SFB_TRY(up(&f.band, band));
    SFB_TRY(up(&f.Hf16, Hf16));
    SFB_TRY(up(&f.Hb16, Hb16));
    SFB_TRY(up(&f.Tf16, Tf16));
    SFB_TRY(up(&f.Tb16, Tb16));
    SFB_TRY(up(&f.V, V));
    SFB_TRY(up(&f.W, W));
    SFB_TRY(up(&f.coef, coef));
    return SFB_OK;
}

void free_spike_factor(SpikeFactor& f) {
    double* ptrs[] = {f.band, f.Hf16, f.Hb16, f.Tf16, f.Tb16, f.V, f.W, f.coef};
    for (double* p : ptrs) cudaFree(p);
    f = SpikeFactor{};
}

}  // namespace sfb
