// Banded SPD preconditioner by segmented triangular solves.
//
// Z = P_L^-1 R P_R^-1 with P = C C^T (banded Cholesky, half-bandwidth b <= 4,
// factorised once on the host).  A plain forward/backward substitution is a
// q-long sequential chain per line (latency bound: ~1 ms at q = 2047).  Here
// the chain is cut at two levels:
//
//  * segments of S = 64 (one 64 x 64 tile per CTA): each segment is solved
//    with a zero incoming state, a b-dimensional scan over segment
//    boundaries (one thread per line, P steps of b^2 flops) propagates the
//    true states, and a fix-up adds H_p s_p, where H_p (64 x b) are the
//    segment's responses to unit incoming states (precomputed once);
//  * inside a tile, every thread sweeps one 16-long sub-segment of one line
//    (256 threads = 64 lines x 4 sub-segments), a 4-step scan chains the
//    sub-segments and a fix-up with the 16-long responses completes the
//    tile-local solve.  The sequential depth per tile drops from 64 to ~20.
//
// The same linear algebra summed in a different order: results agree with the
// sequential solve to rounding (the MO-PCG parity tests run in this mode).
//
// Tiles are S x S in a padded shared-memory tile, so global traffic is
// coalesced for both directions:
//   DIR_COL  lines = columns, sweep along rows    (left factor  P_L^-1 R)
//   DIR_ROW  lines = rows,    sweep along columns (right factor R P_R^-1)
// Per factor: fwd-local -> scan -> fix + bwd-local -> scan -> fix (5 launches,
// 3 tile passes + 2 small scans).  The final fix of the right factor also
// produces <Z,R> for MO-PCG's beta.
#include "sfb_common.cuh"
#include "sfb_kernels.cuh"
#include "sfb_launch.cuh"

namespace sfb {

namespace {

constexpr int S = 64;          // segment length == tile edge
constexpr int SS = 16;         // sub-segment length (one thread's sweep)
constexpr int NSUB = S / SS;   // sub-segments per segment
constexpr int NT = S * NSUB;   // threads per tile CTA

enum { DIR_COL = 0, DIR_ROW = 1 };
enum { PH_FWD = 0, PH_FIX_BWD = 1, PH_FIX = 2 };

// tile[a][c]: a = position along the sweep, c = line within the tile.  All
// NT threads move the tile, coalesced along the contiguous global index; the
// loads of one thread are issued back to back.
template <int DIR>
__device__ __forceinline__ void tile_load(double (*tile)[S + 1], const double* X, int ld, int sweep0, int line0,
                                          int nsweep, int nlines) {
    // global rows rb + hi + 4u, columns cb + lo (lo = lane-contiguous)
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

template <int DIR>
__device__ __forceinline__ void tile_store(double (*tile)[S + 1], double* X, int ld, int sweep0, int line0,
                                           int nsweep, int nlines) {
    const int t = threadIdx.x, lo = t % S, hi = t / S;
    const int rb = DIR == DIR_COL ? sweep0 : line0, cb = DIR == DIR_COL ? line0 : sweep0;
    const int nr = DIR == DIR_COL ? nsweep : nlines, nc = DIR == DIR_COL ? nlines : nsweep;
    double* p = X + (size_t)(rb + hi) * ld + cb + lo;
    const size_t step = (size_t)NSUB * ld;
    const bool full = rb + S <= nr && cb + S <= nc;
    const bool cok = cb + lo < nc;
    #pragma unroll
    for (int u = 0; u < S / NSUB; ++u) {
        const int kk = hi + u * NSUB;
        const double v = DIR == DIR_COL ? tile[kk][lo] : tile[lo][kk];
        if (full || (cok && rb + kk < nr)) p[u * step] = v;
    }
}

struct SegArgs {
    const double* band;  // [n + B][B + 1]: C[i][i-B+d] (d < B), 1/C[i][i] at d = B; B zero rows appended
    const double* Hf;    // [P][S][B] forward responses (64-level)
    const double* Hb;    // [P][S][B] backward responses
    const double* Hf16;  // [P16][SS][B] forward responses (16-level)
    const double* Hb16;
    const double* Tf16;  // [P16][B][B]
    const double* Tb16;
    const double* sf;    // [P][B][nlines] forward incoming states
    const double* sb;    // [P][B][nlines] backward incoming states
    const double* Xin;   // input of the forward-local phase
    int ldi;
    double* X;           // working / output buffer
    int ld;
    int n;               // length of the sweep (order of the factor)
    int nlines;
    // fused <Z,R> (final phase of the right factor)
    const double* R;
    int ldr;
    double* partials;
    unsigned* counter;
    PcgState* pcg;
    double* dot_out;
};

// `band` points at the shared-memory copy of rows start .. start + S + B - 1
template <int B>
__device__ __forceinline__ void fwd_sweep(double (*tile)[S + 1], const double* band, int a0, int a1, int c) {
    double w[B > 0 ? B : 1];
    #pragma unroll
    for (int d = 0; d < B; ++d) w[d] = 0.0;
    for (int k = a0; k < a1; ++k) {
        const double* cb = band + k * (B + 1);
        double v = tile[k][c];
        #pragma unroll
        for (int d = 0; d < B; ++d) v = fma(-cb[d], w[d], v);
        v *= cb[B];
        #pragma unroll
        for (int d = 0; d + 1 < B; ++d) w[d] = w[d + 1];
        if (B > 0) w[B - 1] = v;
        tile[k][c] = v;
    }
}

template <int B>
__device__ __forceinline__ void bwd_sweep(double (*tile)[S + 1], const double* band, int a0, int a1, int c) {
    double w[B > 0 ? B : 1];  // w[e-1] = z[i+e]
    #pragma unroll
    for (int d = 0; d < B; ++d) w[d] = 0.0;
    for (int k = a1 - 1; k >= a0; --k) {
        double v = tile[k][c];
        #pragma unroll
        for (int e = B; e >= 1; --e) v = fma(-band[(k + e) * (B + 1) + B - e], w[e - 1], v);
        v *= band[k * (B + 1) + B];
        #pragma unroll
        for (int e = B - 1; e >= 1; --e) w[e] = w[e - 1];
        if (B > 0) w[0] = v;
        tile[k][c] = v;
    }
}

template <int B, int DIR, int PH>
__global__ void __launch_bounds__(NT) seg_tile_kernel(SegArgs a) {
    SFB_PDL_PROLOGUE();
    if (a.pcg != nullptr && a.pcg->status != SFB_PCG_RUNNING) return;
    constexpr int BB = B > 0 ? B : 1;
    __shared__ double tile[S][S + 1];
    __shared__ double sst[NSUB][BB][S];  // incoming states of the sub-segments, per line
    const int p = blockIdx.x;             // segment along the sweep
    const int line0 = blockIdx.y * S;     // first line of this tile
    const int start = p * S;
    const int len = min(S, a.n - start);
    const int t = threadIdx.x, c = t % S, k = t / S;  // line, sub-segment
    const int gl = line0 + c;
    const bool live = gl < a.nlines;
    const int a0 = min(k * SS, len), a1 = min(k * SS + SS, len);  // my rows [a0, a1)
    const int p16 = p * NSUB + k;
    // coefficients of this segment, staged once (every sweep step reads them)
    __shared__ double bandS[(S + 4) * 5];          // rows start .. start+S+B-1 of the band
    __shared__ double Hs[S * BB];                 // 64-level responses of segment p
    __shared__ double H16s[NSUB * SS * BB];       // 16-level responses of its sub-segments
    __shared__ double T16s[NSUB * BB * BB];       // 16-level transfers
    for (int i = t; i < (S + B) * (B + 1); i += NT) {
        const int row = start + i / (B + 1);
        bandS[i] = row < a.n + B ? a.band[(size_t)start * (B + 1) + i] : 0.0;
    }
    if (B > 0) {
        const double* Hg = PH == PH_FIX ? a.Hb : a.Hf;
        const double* H16g = PH == PH_FWD ? a.Hf16 : a.Hb16;
        const double* T16g = PH == PH_FWD ? a.Tf16 : a.Tb16;
        const int n16 = (a.n + SS - 1) / SS;
        for (int i = t; i < S * BB; i += NT) Hs[i] = Hg[(size_t)p * S * BB + i];
        for (int i = t; i < NSUB * SS * BB; i += NT)
            H16s[i] = p * NSUB + i / (SS * BB) < n16 ? H16g[(size_t)p * NSUB * SS * BB + i] : 0.0;
        for (int i = t; i < NSUB * BB * BB; i += NT)
            T16s[i] = p * NSUB + i / (BB * BB) < n16 ? T16g[(size_t)p * NSUB * BB * BB + i] : 0.0;
    }
    tile_load<DIR>(tile, PH == PH_FWD ? a.Xin : a.X, PH == PH_FWD ? a.ldi : a.ld, start, line0, a.n, a.nlines);
    __syncthreads();

    if (PH == PH_FIX_BWD && live && B > 0) {
        // tile-level fix with the true incoming state of this segment
        const double* H = Hs;
        double s[BB];
        #pragma unroll
        for (int d = 0; d < B; ++d) s[d] = a.sf[((size_t)p * B + d) * a.nlines + gl];
        for (int kk = a0; kk < a1; ++kk) {
            double v = tile[kk][c];
            #pragma unroll
            for (int d = 0; d < B; ++d) v = fma(H[kk * B + d], s[d], v);
            tile[kk][c] = v;
        }
    }
    if (PH == PH_FWD || PH == PH_FIX_BWD) {
        // sub-segment local solves (zero state at the sub-segment boundary)
        if (live) {
            if (PH == PH_FWD) fwd_sweep<B>(tile, bandS, a0, a1, c);
            else bwd_sweep<B>(tile, bandS, a0, a1, c);
        }
        if (B > 0) {
            __syncthreads();
            if (k == 0 && live) {
                // 4-step chain over the sub-segments of this line
                double s[BB];
                #pragma unroll
                for (int d = 0; d < B; ++d) s[d] = 0.0;
                #pragma unroll
                for (int step = 0; step < NSUB; ++step) {
                    const int kk = PH == PH_FWD ? step : NSUB - 1 - step;
                    const int s0 = kk * SS, s1 = min(s0 + SS, len);
                    if (s0 >= len) continue;  // empty sub-segment at the end of the line
                    #pragma unroll
                    for (int d = 0; d < B; ++d) sst[kk][d][c] = s[d];
                    const double* T = T16s + kk * BB * BB;
                    double nx[BB];
                    #pragma unroll
                    for (int d = 0; d < B; ++d) {
                        const int r = PH == PH_FWD ? s1 - B + d : s0 + d;
                        const bool inside = PH == PH_FWD ? r >= s0 : r < s1;
                        double v = inside ? tile[r][c] : 0.0;
                        #pragma unroll
                        for (int e = 0; e < B; ++e) v = fma(T[d * B + e], s[e], v);
                        nx[d] = v;
                    }
                    #pragma unroll
                    for (int d = 0; d < B; ++d) s[d] = nx[d];
                }
            }
            __syncthreads();
            if (live && a0 < a1) {
                const double* H = H16s + k * SS * BB;
                double s[BB];
                #pragma unroll
                for (int d = 0; d < B; ++d) s[d] = sst[k][d][c];
                for (int kk = a0; kk < a1; ++kk) {
                    double v = tile[kk][c];
                    #pragma unroll
                    for (int d = 0; d < B; ++d) v = fma(H[(kk - a0) * B + d], s[d], v);
                    tile[kk][c] = v;
                }
            }
        }
    } else if (live && B > 0) {  // PH_FIX: tile-level backward fix-up
        const double* H = Hs;
        double s[BB];
        #pragma unroll
        for (int d = 0; d < B; ++d) s[d] = a.sb[((size_t)p * B + d) * a.nlines + gl];
        for (int kk = a0; kk < a1; ++kk) {
            double v = tile[kk][c];
            #pragma unroll
            for (int d = 0; d < B; ++d) v = fma(H[kk * B + d], s[d], v);
            tile[kk][c] = v;
        }
    }
    __syncthreads();
    if (PH != PH_FIX && B > 0 && k == 0 && live) {
        // boundary values of the tile-local solution for the segment scan:
        // forward -> last B rows, backward -> first B rows
        double* sv = const_cast<double*>(PH == PH_FWD ? a.sf : a.sb);
        #pragma unroll
        for (int d = 0; d < B; ++d) {
            const int r = PH == PH_FWD ? len - B + d : d;
            const bool inside = PH == PH_FWD ? r >= 0 : r < len;
            sv[((size_t)p * B + d) * a.nlines + gl] = inside ? tile[r][c] : 0.0;
        }
    }
    tile_store<DIR>(tile, a.X, a.ld, start, line0, a.n, a.nlines);
    if (PH == PH_FIX && a.R != nullptr) {
        // <Z,R> over this tile (deterministic: fixed thread/tile order)
        double dot = 0.0;
        const int lo = t % S, hi = t / S;
        #pragma unroll 4
        for (int kk = hi; kk < S; kk += NSUB) {
            if (DIR == DIR_COL) {
                const int i = start + kk, j = line0 + lo;
                if (kk < len && j < a.nlines) dot = fma(tile[kk][lo], a.R[(size_t)i * a.ldr + j], dot);
            } else {
                const int i = line0 + kk, j = start + lo;
                if (i < a.nlines && lo < len) dot = fma(tile[lo][kk], a.R[(size_t)i * a.ldr + j], dot);
            }
        }
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

// Boundary scans over the 64-segments: one thread per line, P sequential
// steps of a b x b update.  The tile kernels left the boundary values of the
// tile-local solutions in `sv` ([P][B][nlines], coalesced); the scan reads a
// chunk of them, then overwrites them in place with the true incoming states.
template <int B, bool FWD>
__global__ void __launch_bounds__(64) seg_scan_kernel(int nlines, int P, const double* T, double* sv,
                                                      const PcgState* pcg) {
    SFB_PDL_PROLOGUE();
    if (pcg != nullptr && pcg->status != SFB_PCG_RUNNING) return;
    // the P transfer matrices, staged once: every step of the chain reads one
    extern __shared__ double Ts[];
    for (int i = threadIdx.x; i < P * B * B; i += blockDim.x) Ts[i] = T[i];
    __syncthreads();
    const int gl = blockIdx.x * blockDim.x + threadIdx.x;
    if (gl >= nlines) return;
    constexpr int BB = B > 0 ? B : 1;
    constexpr int CH = 32 / BB;  // boundary values in flight per thread
    double s[BB];
    #pragma unroll
    for (int d = 0; d < B; ++d) s[d] = 0.0;
    for (int s0 = 0; s0 < P; s0 += CH) {
        double tail[CH][BB];
        #pragma unroll
        for (int u = 0; u < CH; ++u) {
            const int step = s0 + u;
            const int p = FWD ? step : P - 1 - step;
            #pragma unroll
            for (int d = 0; d < B; ++d) tail[u][d] = step < P ? sv[((size_t)p * B + d) * nlines + gl] : 0.0;
        }
        #pragma unroll
        for (int u = 0; u < CH; ++u) {
            const int step = s0 + u;
            if (step >= P) break;
            const int p = FWD ? step : P - 1 - step;
            #pragma unroll
            for (int d = 0; d < B; ++d) sv[((size_t)p * B + d) * nlines + gl] = s[d];
            double nx[BB];
            const double* Tp = Ts + p * B * B;
            #pragma unroll
            for (int d = 0; d < B; ++d) {
                double v = tail[u][d];
                #pragma unroll
                for (int e = 0; e < B; ++e) v = fma(Tp[d * B + e], s[e], v);
                nx[d] = v;
            }
            #pragma unroll
            for (int d = 0; d < B; ++d) s[d] = nx[d];
        }
    }
}

template <int B, int DIR>
int run_factor(const SegFactor& f, const double* Xin, int ldi, double* X, int ld, int nlines, const SegDot* dot,
               double* sv_f, double* sv_b, const PcgState* pcg_gate, cudaStream_t s) {
    SegArgs a{};
    a.band = f.band;
    a.Hf = f.Hf;
    a.Hb = f.Hb;
    a.Hf16 = f.Hf16;
    a.Hb16 = f.Hb16;
    a.Tf16 = f.Tf16;
    a.Tb16 = f.Tb16;
    a.sf = sv_f;
    a.sb = sv_b;
    a.Xin = Xin;
    a.ldi = ldi;
    a.X = X;
    a.ld = ld;
    a.n = f.n;
    a.nlines = nlines;
    a.pcg = const_cast<PcgState*>(pcg_gate);
    const int P = (f.n + S - 1) / S;
    const dim3 grid(P, (nlines + S - 1) / S);
    const dim3 sgrid((nlines + 63) / 64);
    SFB_TRY(launch_kernel(seg_tile_kernel<B, DIR, PH_FWD>, grid, dim3(NT), 0, s, a));
    const size_t tsm = (size_t)P * B * B * 8;
    if (tsm > 48 * 1024) {
        set_error("banded preconditioner: order too large for the segment scan");
        return SFB_ERR_UNSUPPORTED;
    }
    if (B > 0) SFB_TRY(launch_kernel(seg_scan_kernel<B, true>, sgrid, dim3(64), tsm, s, nlines, P, f.Tf, sv_f, pcg_gate));
    SFB_TRY(launch_kernel(seg_tile_kernel<B, DIR, PH_FIX_BWD>, grid, dim3(NT), 0, s, a));
    if (B > 0) SFB_TRY(launch_kernel(seg_scan_kernel<B, false>, sgrid, dim3(64), tsm, s, nlines, P, f.Tb, sv_b, pcg_gate));
    if (dot != nullptr) {
        a.R = dot->R;
        a.ldr = dot->ldr;
        a.partials = dot->partials;
        a.counter = dot->counter;
        a.pcg = dot->pcg;
        a.dot_out = dot->dot_out;
    }
    return launch_kernel(seg_tile_kernel<B, DIR, PH_FIX>, grid, dim3(NT), 0, s, a);
}

template <int B>
int run_b(const SegFactor& f, int dir, const double* Xin, int ldi, double* X, int ld, int nlines, const SegDot* dot,
          double* sv_f, double* sv_b, const PcgState* pcg_gate, cudaStream_t s) {
    if (dir == DIR_COL) return run_factor<B, DIR_COL>(f, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
    return run_factor<B, DIR_ROW>(f, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
}

}  // namespace

int seg_length() { return S; }
int seg_sub_length() { return SS; }

int launch_seg_factor(const SegFactor& f, int along_rows, const double* Xin, int ldi, double* X, int ld,
                      int nlines, const SegDot* dot, double* sv_f, double* sv_b, const PcgState* pcg_gate,
                      cudaStream_t s) {
    const int dir = along_rows ? DIR_ROW : DIR_COL;
    switch (f.b) {
        case 0: return run_b<0>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
        case 1: return run_b<1>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
        case 2: return run_b<2>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
        case 3: return run_b<3>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
        case 4: return run_b<4>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
    }
    set_error("segmented Cholesky: half-bandwidth > 4");
    return SFB_ERR_UNSUPPORTED;
}

}  // namespace sfb
