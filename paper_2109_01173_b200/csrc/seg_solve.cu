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

namespace sfb {

namespace {

constexpr int S = 64;  // segment length == tile edge == threads per CTA

enum { DIR_COL = 0, DIR_ROW = 1 };
enum { PH_FWD = 0, PH_FIX_BWD = 1, PH_FIX = 2 };

// tile[a][c]: a = position along the sweep, c = line within the tile
template <int DIR>
__device__ __forceinline__ void tile_load(double (*tile)[S + 1], const double* X, int ld, int sweep0, int line0,
                                          int nsweep, int nlines) {
    const int t = threadIdx.x;
    if (DIR == DIR_COL) {  // element (row = sweep0 + a, col = line0 + t)
        for (int a = 0; a < S; ++a) {
            const int i = sweep0 + a, j = line0 + t;
            tile[a][t] = (i < nsweep && j < nlines) ? X[(size_t)i * ld + j] : 0.0;
        }
    } else {  // element (row = line0 + c, col = sweep0 + t)
        for (int c = 0; c < S; ++c) {
            const int i = line0 + c, j = sweep0 + t;
            tile[t][c] = (i < nlines && j < nsweep) ? X[(size_t)i * ld + j] : 0.0;
        }
    }
}

template <int DIR>
__device__ __forceinline__ void tile_store(double (*tile)[S + 1], double* X, int ld, int sweep0, int line0,
                                           int nsweep, int nlines) {
    const int t = threadIdx.x;
    if (DIR == DIR_COL) {
        for (int a = 0; a < S; ++a) {
            const int i = sweep0 + a, j = line0 + t;
            if (i < nsweep && j < nlines) X[(size_t)i * ld + j] = tile[a][t];
        }
    } else {
        for (int c = 0; c < S; ++c) {
            const int i = line0 + c, j = sweep0 + t;
            if (i < nlines && j < nsweep) X[(size_t)i * ld + j] = tile[t][c];
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
__global__ void __launch_bounds__(S) seg_tile_kernel(SegArgs a) {
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
    const bool live = gl < a.nlines;
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
        if (DIR == DIR_COL) {
            for (int k = 0; k < len; ++k)
                if (live) dot = fma(tile[k][c], a.R[(size_t)(start + k) * a.ldr + gl], dot);
        } else {
            for (int cc = 0; cc < S; ++cc) {
                const int i = line0 + cc, j = start + c;
                if (i < a.nlines && c < len) dot = fma(tile[c][cc], a.R[(size_t)i * a.ldr + j], dot);
            }
        }
        __shared__ double sh[S / 32];
        const double part = block_sum<S>(dot, sh);
        const unsigned nblk = gridDim.x * gridDim.y;
        if (threadIdx.x == 0) a.partials[blockIdx.y * gridDim.x + blockIdx.x] = part;
        if (arrive_last(a.counter, nblk)) {
            const double tot = sum_partials<S>(a.partials, nblk, 1, sh);
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
__global__ void __launch_bounds__(128) seg_scan_kernel(const double* X, int ld, int n, int nlines, int P,
                                                       const double* T, double* sv, const PcgState* pcg) {
    if (pcg != nullptr && pcg->status != SFB_PCG_RUNNING) return;
    const int gl = blockIdx.x * blockDim.x + threadIdx.x;
    if (gl >= nlines) return;
    double s[B > 0 ? B : 1];
    #pragma unroll
    for (int d = 0; d < B; ++d) s[d] = 0.0;
    for (int step = 0; step < P; ++step) {
        const int p = FWD ? step : P - 1 - step;
        const int start = p * S, end = min(n, start + S);
        #pragma unroll
        for (int d = 0; d < B; ++d) sv[((size_t)p * B + d) * nlines + gl] = s[d];
        // next state: forward -> last B values up to `end`; backward -> first B values from `start`
        double nx[B > 0 ? B : 1];
        const double* Tp = T + (size_t)p * B * B;
        #pragma unroll
        for (int d = 0; d < B; ++d) {
            const int r = FWD ? end - B + d : start + d;
            const bool inside = FWD ? r >= start : r < end;
            double v = 0.0;
            if (inside) v = DIR == DIR_COL ? X[(size_t)r * ld + gl] : X[(size_t)gl * ld + r];
            #pragma unroll
            for (int e = 0; e < B; ++e) v = fma(Tp[d * B + e], s[e], v);
            nx[d] = v;
        }
        #pragma unroll
        for (int d = 0; d < B; ++d) s[d] = nx[d];
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
    const int sb = (nlines + 127) / 128;
    if (DIR == DIR_COL) {
        seg_tile_kernel<B, DIR_COL, PH_FWD><<<grid, S, 0, s>>>(a);
        seg_scan_kernel<B, DIR_COL, true><<<sb, 128, 0, s>>>(X, ld, f.n, nlines, P, f.Tf, sv_f, pcg_gate);
        seg_tile_kernel<B, DIR_COL, PH_FIX_BWD><<<grid, S, 0, s>>>(a);
        seg_scan_kernel<B, DIR_COL, false><<<sb, 128, 0, s>>>(X, ld, f.n, nlines, P, f.Tb, sv_b, pcg_gate);
    } else {
        seg_tile_kernel<B, DIR_ROW, PH_FWD><<<grid, S, 0, s>>>(a);
        seg_scan_kernel<B, DIR_ROW, true><<<sb, 128, 0, s>>>(X, ld, f.n, nlines, P, f.Tf, sv_f, pcg_gate);
        seg_tile_kernel<B, DIR_ROW, PH_FIX_BWD><<<grid, S, 0, s>>>(a);
        seg_scan_kernel<B, DIR_ROW, false><<<sb, 128, 0, s>>>(X, ld, f.n, nlines, P, f.Tb, sv_b, pcg_gate);
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
        seg_tile_kernel<B, DIR_COL, PH_FIX><<<grid, S, 0, s>>>(a);
    else
        seg_tile_kernel<B, DIR_ROW, PH_FIX><<<grid, S, 0, s>>>(a);
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
