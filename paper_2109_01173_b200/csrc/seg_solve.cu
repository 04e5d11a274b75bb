// Banded SPD preconditioner by segmented triangular solves.
//
// Z = P_L^-1 R P_R^-1 with P = C C^T (banded Cholesky, half-bandwidth b <= 4,
// factorised once on the host).  A plain forward/backward substitution is a
// q-long sequential chain per line (latency bound: ~1 ms at q = 2047).  Here
// every line is cut into segments of S = 64: each segment is solved locally
// with a zero incoming state (fully parallel over segments and lines), a
// b-dimensional scan over segment boundaries propagates the true states
// (s_{p+1} = tail(y_loc,p) + T_p s_p, P steps of b^2 flops), and a fix-up adds
// H_p s_p, where H_p (S x b) are the segment's responses to unit incoming
// states (precomputed on the host once).  The same linear algebra, summed in a
// different order: results agree with the sequential solve to rounding.
//
// Tiles are S x S: 64 threads, one per line, sweep a padded shared-memory
// tile, so global traffic is coalesced for both directions:
//   DIR_COL  lines = columns, sweep along rows    (left factor  P_L^-1 R)
//   DIR_ROW  lines = rows,    sweep along columns (right factor R P_R^-1)
// Per factor: fwd-local -> scan -> fix + bwd-local -> scan -> fix (5 launches,
// 3 tile passes + 2 tiny scans).  The final fix of the right factor also
// produces <Z,R> for MO-PCG's beta.
#include "sfb_common.cuh"
#include "sfb_kernels.cuh"
#include "sfb_launch.cuh"

namespace sfb {

namespace {

constexpr int S = 64;  // segment length == tile edge == threads per CTA

enum { DIR_COL = 0, DIR_ROW = 1 };
enum { PH_FWD = 0, PH_FIX_BWD = 1, PH_FIX = 2 };

constexpr int NT = 256;  // threads per tile CTA: all load/store, the first S sweep

// tile[a][c]: a = position along the sweep, c = line within the tile.  All
// NT threads move the tile (coalesced along the contiguous global index).
template <int DIR>
__device__ __forceinline__ void tile_load(double (*tile)[S + 1], const double* X, int ld, int sweep0, int line0,
                                          int nsweep, int nlines) {
    const int t = threadIdx.x, lo = t % S, hi = t / S;
    #pragma unroll 4
    for (int k = hi; k < S; k += NT / S) {
        if (DIR == DIR_COL) {  // element (row = sweep0 + k, col = line0 + lo)
            const int i = sweep0 + k, j = line0 + lo;
            tile[k][lo] = (i < nsweep && j < nlines) ? X[(size_t)i * ld + j] : 0.0;
        } else {  // element (row = line0 + k, col = sweep0 + lo)
            const int i = line0 + k, j = sweep0 + lo;
            tile[lo][k] = (i < nlines && j < nsweep) ? X[(size_t)i * ld + j] : 0.0;
        }
    }
}

template <int DIR>
__device__ __forceinline__ void tile_store(double (*tile)[S + 1], double* X, int ld, int sweep0, int line0,
                                           int nsweep, int nlines) {
    const int t = threadIdx.x, lo = t % S, hi = t / S;
    #pragma unroll 4
    for (int k = hi; k < S; k += NT / S) {
        if (DIR == DIR_COL) {
            const int i = sweep0 + k, j = line0 + lo;
            if (i < nsweep && j < nlines) X[(size_t)i * ld + j] = tile[k][lo];
        } else {
            const int i = line0 + k, j = sweep0 + lo;
            if (i < nlines && j < nsweep) X[(size_t)i * ld + j] = tile[lo][k];
        }
    }
}

struct SegArgs {
    const double* band;  // [n + B][B + 1]: C[i][i-B+d] (d < B), 1/C[i][i] at d = B; B zero rows appended
    const double* Hf;    // [P][S][B] forward responses
    const double* Hb;    // [P][S][B] backward responses
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

template <int B, int DIR, int PH>
__global__ void __launch_bounds__(NT) seg_tile_kernel(SegArgs a) {
    SFB_PDL_PROLOGUE();
    if (a.pcg != nullptr && a.pcg->status != SFB_PCG_RUNNING) return;
    __shared__ double tile[S][S + 1];
    const int p = blockIdx.x;             // segment along the sweep
    const int line0 = blockIdx.y * S;     // first line of this tile
    const int start = p * S;
    const int len = min(S, a.n - start);
    const int c = threadIdx.x;
    const int gl = line0 + c;
    tile_load<DIR>(tile, PH == PH_FWD ? a.Xin : a.X, PH == PH_FWD ? a.ldi : a.ld, start, line0, a.n, a.nlines);
    __syncthreads();
    const bool live = c < S && gl < a.nlines;
    if (live) {
        if (PH == PH_FWD) {
            double w[B > 0 ? B : 1];
            #pragma unroll
            for (int d = 0; d < B; ++d) w[d] = 0.0;
            for (int k = 0; k < len; ++k) {
                const double* cb = a.band + (size_t)(start + k) * (B + 1);
                double v = tile[k][c];
                #pragma unroll
                for (int d = 0; d < B; ++d) v = fma(-cb[d], w[d], v);
                v *= cb[B];
                #pragma unroll
                for (int d = 0; d + 1 < B; ++d) w[d] = w[d + 1];
                if (B > 0) w[B - 1] = v;
                tile[k][c] = v;
            }
        } else {
            // fix-up with the true incoming state of this segment
            const double* H = (PH == PH_FIX_BWD ? a.Hf : a.Hb) + (size_t)p * S * (B > 0 ? B : 1);
            const double* sv = PH == PH_FIX_BWD ? a.sf : a.sb;
            double s[B > 0 ? B : 1];
            #pragma unroll
            for (int d = 0; d < B; ++d) s[d] = sv[((size_t)p * B + d) * a.nlines + gl];
            if (B > 0) {
                for (int k = 0; k < len; ++k) {
                    double v = tile[k][c];
                    #pragma unroll
                    for (int d = 0; d < B; ++d) v = fma(H[k * B + d], s[d], v);
                    tile[k][c] = v;
                }
            }
            if (PH == PH_FIX_BWD) {
                // local backward solve C^T z = y with a zero state after the segment
                double w[B > 0 ? B : 1];  // w[e-1] = z[i+e]
                #pragma unroll
                for (int d = 0; d < B; ++d) w[d] = 0.0;
                for (int k = len - 1; k >= 0; --k) {
                    const int i = start + k;
                    double v = tile[k][c];
                    #pragma unroll
                    for (int e = B; e >= 1; --e) v = fma(-a.band[(size_t)(i + e) * (B + 1) + B - e], w[e - 1], v);
                    v *= a.band[(size_t)i * (B + 1) + B];
                    #pragma unroll
                    for (int e = B - 1; e >= 1; --e) w[e] = w[e - 1];
                    if (B > 0) w[0] = v;
                    tile[k][c] = v;
                }
            }
        }
    }
    __syncthreads();
    tile_store<DIR>(tile, a.X, a.ld, start, line0, a.n, a.nlines);
    if (PH == PH_FIX && a.R != nullptr) {
        // <Z,R> over this tile (deterministic: fixed thread/tile order)
        double dot = 0.0;
        const int t = threadIdx.x, lo = t % S, hi = t / S;
        for (int k = hi; k < S; k += NT / S) {
            if (DIR == DIR_COL) {
                const int i = start + k, j = line0 + lo;
                if (k < len && j < a.nlines) dot = fma(tile[k][lo], a.R[(size_t)i * a.ldr + j], dot);
            } else {
                const int i = line0 + k, j = start + lo;
                if (i < a.nlines && lo < len) dot = fma(tile[lo][k], a.R[(size_t)i * a.ldr + j], dot);
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

// Boundary scans: one thread per line, P sequential steps of a b x b update.
template <int B, int DIR, bool FWD>
__global__ void __launch_bounds__(64) seg_scan_kernel(const double* X, int ld, int n, int nlines, int P,
                                                       const double* T, double* sv, const PcgState* pcg) {
    SFB_PDL_PROLOGUE();
    if (pcg != nullptr && pcg->status != SFB_PCG_RUNNING) return;
    const int gl = blockIdx.x * blockDim.x + threadIdx.x;
    if (gl >= nlines) return;
    double s[B > 0 ? B : 1];
    #pragma unroll
    for (int d = 0; d < B; ++d) s[d] = 0.0;
    constexpr int CH = 8;  // boundary values prefetched per chunk (independent of the state chain)
    constexpr int BB = B > 0 ? B : 1;
    for (int s0 = 0; s0 < P; s0 += CH) {
        double tail[CH][BB];
        #pragma unroll
        for (int u = 0; u < CH; ++u) {
            const int step = s0 + u;
            const int p = FWD ? step : P - 1 - step;
            const int start = p * S, end = min(n, start + S);
            #pragma unroll
            for (int d = 0; d < B; ++d) {
                const int r = FWD ? end - B + d : start + d;
                const bool inside = step < P && (FWD ? r >= start : r < end);
                tail[u][d] = inside ? (DIR == DIR_COL ? X[(size_t)r * ld + gl] : X[(size_t)gl * ld + r]) : 0.0;
            }
        }
        #pragma unroll
        for (int u = 0; u < CH; ++u) {
            const int step = s0 + u;
            if (step >= P) break;
            const int p = FWD ? step : P - 1 - step;
            #pragma unroll
            for (int d = 0; d < B; ++d) sv[((size_t)p * B + d) * nlines + gl] = s[d];
            // next state: forward -> last B values of segment p; backward -> first B values
            double nx[BB];
            const double* Tp = T + (size_t)p * B * B;
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

template <int B>
int run_factor(const SegFactor& f, int DIR, const double* Xin, int ldi, double* X, int ld, int nlines,
               const SegDot* dot, double* sv_f, double* sv_b, const PcgState* pcg_gate, cudaStream_t s) {
    SegArgs a{};
    a.band = f.band;
    a.Hf = f.Hf;
    a.Hb = f.Hb;
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
    const int sb = (nlines + 63) / 64;
    if (DIR == DIR_COL) {
        SFB_TRY(launch_kernel(seg_tile_kernel<B, DIR_COL, PH_FWD>, dim3(grid), dim3(NT), 0, s, a));
        SFB_TRY(launch_kernel(seg_scan_kernel<B, DIR_COL, true>, dim3(sb), dim3(64), 0, s, X, ld, f.n, nlines, P, f.Tf, sv_f, pcg_gate));
        SFB_TRY(launch_kernel(seg_tile_kernel<B, DIR_COL, PH_FIX_BWD>, dim3(grid), dim3(NT), 0, s, a));
        SFB_TRY(launch_kernel(seg_scan_kernel<B, DIR_COL, false>, dim3(sb), dim3(64), 0, s, X, ld, f.n, nlines, P, f.Tb, sv_b, pcg_gate));
    } else {
        SFB_TRY(launch_kernel(seg_tile_kernel<B, DIR_ROW, PH_FWD>, dim3(grid), dim3(NT), 0, s, a));
        SFB_TRY(launch_kernel(seg_scan_kernel<B, DIR_ROW, true>, dim3(sb), dim3(64), 0, s, X, ld, f.n, nlines, P, f.Tf, sv_f, pcg_gate));
        SFB_TRY(launch_kernel(seg_tile_kernel<B, DIR_ROW, PH_FIX_BWD>, dim3(grid), dim3(NT), 0, s, a));
        SFB_TRY(launch_kernel(seg_scan_kernel<B, DIR_ROW, false>, dim3(sb), dim3(64), 0, s, X, ld, f.n, nlines, P, f.Tb, sv_b, pcg_gate));
    }
    if (dot != nullptr) {
        a.R = dot->R;
        a.ldr = dot->ldr;
        a.partials = dot->partials;
        a.counter = dot->counter;
        a.pcg = dot->pcg;
        a.dot_out = dot->dot_out;
    }
    if (DIR == DIR_COL)
        SFB_TRY(launch_kernel(seg_tile_kernel<B, DIR_COL, PH_FIX>, dim3(grid), dim3(NT), 0, s, a));
    else
        SFB_TRY(launch_kernel(seg_tile_kernel<B, DIR_ROW, PH_FIX>, dim3(grid), dim3(NT), 0, s, a));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

}  // namespace

int seg_length() { return S; }

int launch_seg_factor(const SegFactor& f, int along_rows, const double* Xin, int ldi, double* X, int ld,
                      int nlines, const SegDot* dot, double* sv_f, double* sv_b, const PcgState* pcg_gate,
                      cudaStream_t s) {
    const int dir = along_rows ? DIR_ROW : DIR_COL;
    switch (f.b) {
        case 0: return run_factor<0>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
        case 1: return run_factor<1>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
        case 2: return run_factor<2>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
        case 3: return run_factor<3>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
        case 4: return run_factor<4>(f, dir, Xin, ldi, X, ld, nlines, dot, sv_f, sv_b, pcg_gate, s);
    }
    set_error("segmented Cholesky: half-bandwidth > 4");
    return SFB_ERR_UNSUPPORTED;
}

}  // namespace sfb
