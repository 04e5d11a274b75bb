// Memory-bound MO-PCG passes, fused with their reductions.
//
//   pcg_update  : U += alpha Q; R -= alpha W; |R|^2; last block -> stop test
//                 (solvers.py:432-446)
//   pcg_init_*  : R = rhs (- op(u0)); |R_0| (solvers.py:391-397, 415-416)
//   copy_dot    : identity preconditioner Z = R with <Z,R> (solvers.py:124-126)
//   direction / dots : the dense-operator fallback of the fused banded path
//   norms       : |A - B|, max|A|, #non-finite (timestepping.py:89-91, 155, 210)
//
// Grid: 2 CTAs per SM x 256 threads, rows distributed round-robin over CTAs,
// columns over threads (coalesced).  Every reduction is deterministic: one
// partial per CTA, summed in fixed order by the last CTA to finish.
#include "sfb_common.cuh"
#include "sfb_kernels.cuh"
#include "sfb_launch.cuh"

namespace sfb {

namespace {

constexpr int VT = 256;
constexpr int VB = 8 * kNumSMs;  // full occupancy: enough bytes in flight for HBM

#define ROW_LOOP(rows, cols)                                         \
    for (int r = blockIdx.x; r < (rows); r += gridDim.x)            \
        for (int cc = threadIdx.x; cc < (cols); cc += VT)

__device__ __forceinline__ void pcg_finish_update(PcgState* st, double rr, double* hist, double* incs) {
    // solvers.py:434-446 (runs in one thread of the last CTA)
    const int s = st->iter;
    const double res = sqrt(rr);
    if (!isfinite(res)) {
        st->status = SFB_PCG_NONFINITE;
        st->bad_iter = s;
        return;
    }
    hist[s + 1] = res;
    const double inc = fabs(st->alpha) * sqrt(st->qq);
    incs[s] = inc;
    st->iter = s + 1;
    if (st->rule == SFB_RULE_RESIDUAL && res <= st->value * st->res0) {
        st->status = SFB_PCG_TOLERANCE;
    } else if (st->rule == SFB_RULE_INCREMENT && inc <= st->value) {
        st->status = SFB_PCG_INCREMENT;
    } else if (s + 1 >= st->max_iter) {
        st->status = SFB_PCG_MAX_ITER;
    }
}

__global__ void __launch_bounds__(VT) pcg_update_kernel(double* __restrict__ U, double* __restrict__ R,
                                                        const double* __restrict__ W, const double* Q0,
                                                        const double* Q1, int ld, int rows, int cols,
                                                        double* partials, PcgState* st, double* hist,
                                                        double* incs) {
    SFB_PDL_PROLOGUE();
    if (st->status != SFB_PCG_RUNNING) return;
    const int s = st->iter;
    const double alpha = st->alpha;
    const double* Q = (s & 1) ? Q1 : Q0;
    double rr = 0.0;
    // The solver's buffers are rows x ld with zero padding columns that every
    // kernel leaves at zero, so the update runs over the flat padded array in
    // 16-byte vectors (the padding contributes exactly 0 to |R|^2).
    const size_t n2 = (size_t)rows * ld / 2;
    double2* U2 = reinterpret_cast<double2*>(U);
    double2* R2 = reinterpret_cast<double2*>(R);
    const double2* Q2 = reinterpret_cast<const double2*>(Q);
    const double2* W2 = reinterpret_cast<const double2*>(W);
    (void)cols;
    #pragma unroll 2
    for (size_t i = (size_t)blockIdx.x * VT + threadIdx.x; i < n2; i += (size_t)gridDim.x * VT) {
        const double2 q = __ldg(Q2 + i), wv = __ldg(W2 + i);
        double2 u = U2[i], rv = R2[i];
        u.x = __dadd_rn(u.x, __dmul_rn(alpha, q.x));  // U += alpha Q
        u.y = __dadd_rn(u.y, __dmul_rn(alpha, q.y));
        rv.x = __dsub_rn(rv.x, __dmul_rn(alpha, wv.x));  // R -= alpha W
        rv.y = __dsub_rn(rv.y, __dmul_rn(alpha, wv.y));
        U2[i] = u;
        R2[i] = rv;
        rr = fma(rv.x, rv.x, rr);
        rr = fma(rv.y, rv.y, rr);
    }
    __shared__ double sh[VT / 32];
    const double p = block_sum<VT>(rr, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = p;
    if (arrive_last(&st->counter[1], gridDim.x)) {
        const double tot = sum_partials<VT>(partials, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            st->counter[1] = 0;
            pcg_finish_update(st, tot, hist, incs);
        }
    }
}

// R -= alpha W, |R|^2 and the stop test: the update pass of the banded
// iteration, whose U += alpha Q is deferred into the next banded operator
// pass (it re-reads Q there anyway) and, after the last iteration, into
// pcg_ufinal_kernel.  Same arithmetic as pcg_update_kernel.
__global__ void __launch_bounds__(VT) pcg_rupdate_kernel(double* __restrict__ R, const double* __restrict__ W,
                                                         int ld, int rows, double* partials, PcgState* st,
                                                         double* hist, double* incs,
                                                         cudaGraphConditionalHandle handle, int use_handle) {
    SFB_PDL_PROLOGUE();
    if (st->status != SFB_PCG_RUNNING) {  // e.g. INDEFINITE from this iteration's operator pass
        if (use_handle && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(handle, 0u);
        return;
    }
    const double alpha = st->alpha;
    double rr = 0.0;
    const size_t n2 = (size_t)rows * ld / 2;
    double2* R2 = reinterpret_cast<double2*>(R);
    const double2* W2 = reinterpret_cast<const double2*>(W);
    #pragma unroll 4
    for (size_t i = (size_t)blockIdx.x * VT + threadIdx.x; i < n2; i += (size_t)gridDim.x * VT) {
        const double2 wv = __ldg(W2 + i);
        double2 rv = R2[i];
        rv.x = __dsub_rn(rv.x, __dmul_rn(alpha, wv.x));  // R -= alpha W
        rv.y = __dsub_rn(rv.y, __dmul_rn(alpha, wv.y));
        R2[i] = rv;
        rr = fma(rv.x, rv.x, rr);
        rr = fma(rv.y, rv.y, rr);
    }
    __shared__ double sh[VT / 32];
    const double p = block_sum<VT>(rr, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = p;
    if (arrive_last(&st->counter[1], gridDim.x)) {
        const double tot = sum_partials<VT>(partials, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            st->counter[1] = 0;
            pcg_finish_update(st, tot, hist, incs);
            // the loop control of the iteration graph (loop_ctl_kernel's rule),
            // here so the banded iteration needs no extra kernel: the rest of
            // the body (the preconditioner) does not change the status
            const unsigned runs = ++st->counter[6];
            const bool keep = st->status == SFB_PCG_RUNNING && st->iter < st->max_iter &&
                              runs <= (unsigned)st->max_iter + 2u;
            if (use_handle) cudaGraphSetConditional(handle, keep ? 1u : 0u);
        }
    }
}

// The last completed iteration's deferred U += alpha Q (after the loop).  No
// pending update after INDEFINITE (that operator pass already applied it) or
// NONFINITE (the solve raises).
__global__ void __launch_bounds__(VT) pcg_ufinal_kernel(double* __restrict__ U, const double* Q0, const double* Q1,
                                                        int ld, int rows, const PcgState* st) {
    SFB_PDL_PROLOGUE();
    const int n = st->iter;
    if (n < 1 || st->status == SFB_PCG_INDEFINITE || st->status == SFB_PCG_NONFINITE) return;
    const double alpha = st->alpha;
    const double* Q = ((n - 1) & 1) ? Q1 : Q0;
    const size_t n2 = (size_t)rows * ld / 2;
    double2* U2 = reinterpret_cast<double2*>(U);
    const double2* Q2 = reinterpret_cast<const double2*>(Q);
    for (size_t i = (size_t)blockIdx.x * VT + threadIdx.x; i < n2; i += (size_t)gridDim.x * VT) {
        const double2 q = __ldg(Q2 + i);
        double2 u = U2[i];
        u.x = __dadd_rn(u.x, __dmul_rn(alpha, q.x));  // U += alpha Q
        u.y = __dadd_rn(u.y, __dmul_rn(alpha, q.y));
        U2[i] = u;
    }
}

__device__ __forceinline__ void pcg_finish_init(PcgState* st, double rr, double* hist) {
    const double res0 = sqrt(rr);
    st->res0 = res0;
    hist[0] = res0;
    if (res0 == 0.0) st->status = SFB_PCG_TOLERANCE;  // solvers.py:415-416
}

__global__ void __launch_bounds__(VT) pcg_init_plain_kernel(const double* rhs, int ldr, double* R, double* U,
                                                            int ld, int rows, int cols, double* partials,
                                                            PcgState* st, double* hist) {
    SFB_PDL_PROLOGUE();
    double rr = 0.0;
    ROW_LOOP(rows, cols) {
        const double v = rhs[(size_t)r * ldr + cc];
        R[(size_t)r * ld + cc] = v;
        U[(size_t)r * ld + cc] = 0.0;
        rr = fma(v, v, rr);
    }
    __shared__ double sh[VT / 32];
    const double p = block_sum<VT>(rr, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = p;
    if (arrive_last(&st->counter[2], gridDim.x)) {
        const double tot = sum_partials<VT>(partials, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            st->counter[2] = 0;
            pcg_finish_init(st, tot, hist);
        }
    }
}

__global__ void __launch_bounds__(VT) pcg_init_warm_kernel(const double* rhs, int ldr, const double* W, double* R,
                                                           int ld, int rows, int cols, double* partials,
                                                           PcgState* st, double* hist) {
    SFB_PDL_PROLOGUE();
    double rr = 0.0;
    ROW_LOOP(rows, cols) {
        const double v = __dsub_rn(rhs[(size_t)r * ldr + cc], W[(size_t)r * ld + cc]);  // R = rhs - op(U)
        R[(size_t)r * ld + cc] = v;
        rr = fma(v, v, rr);
    }
    __shared__ double sh[VT / 32];
    const double p = block_sum<VT>(rr, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = p;
    if (arrive_last(&st->counter[2], gridDim.x)) {
        const double tot = sum_partials<VT>(partials, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            st->counter[2] = 0;
            pcg_finish_init(st, tot, hist);
        }
    }
}

__global__ void __launch_bounds__(VT) pcg_direction_kernel(const double* Z, double* Q0, double* Q1, int ld,
                                                           int rows, int cols, PcgState* st) {
    SFB_PDL_PROLOGUE();
    if (st->status != SFB_PCG_RUNNING) return;
    const int s = st->iter;
    const double beta = s > 0 ? st->rz_next / st->rz : 0.0;
    double* Qc = (s & 1) ? Q1 : Q0;
    const double* Qp = (s & 1) ? Q0 : Q1;
    ROW_LOOP(rows, cols) {
        const size_t o = (size_t)r * ld + cc;
        Qc[o] = s > 0 ? __dadd_rn(__dmul_rn(beta, Qp[o]), Z[o]) : Z[o];
    }
}

__global__ void __launch_bounds__(VT) pcg_dots_kernel(const double* W, const double* Q0, const double* Q1, int ld,
                                                      int rows, int cols, double* partials, PcgState* st) {
    SFB_PDL_PROLOGUE();
    if (st->status != SFB_PCG_RUNNING) return;
    const int s = st->iter;
    const double* Q = (s & 1) ? Q1 : Q0;
    double wq = 0.0, qq = 0.0;
    ROW_LOOP(rows, cols) {
        const size_t o = (size_t)r * ld + cc;
        const double q = Q[o];
        wq = fma(W[o], q, wq);
        qq = fma(q, q, qq);
    }
    __shared__ double sh[VT / 32];
    const double p0 = block_sum<VT>(wq, sh);
    const double p1 = block_sum<VT>(qq, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = p0;
        partials[gridDim.x + blockIdx.x] = p1;
    }
    if (arrive_last(&st->counter[0], gridDim.x)) {
        const double qw = sum_partials<VT>(partials, gridDim.x, 1, sh);
        const double q2 = sum_partials<VT>(partials + gridDim.x, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            st->counter[0] = 0;
            st->rz = st->rz_next;
            st->qq = q2;
            if (qw <= 0.0) {
                st->status = SFB_PCG_INDEFINITE;
                st->bad_value = qw;
                st->bad_iter = s;
            } else {
                st->alpha = st->rz / qw;
            }
        }
    }
}

__global__ void __launch_bounds__(VT) pcg_record_kernel(const double* U, int ld, int rows, int cols,
                                                        double* iterates, PcgState* st, const double* Q0,
                                                        const double* Q1) {
    SFB_PDL_PROLOGUE();
    // record_iterates (solvers.py:441-442): copy U_s once per completed iteration;
    // with Q0 != nullptr (banded iteration) U still lacks the deferred
    // alpha_{s-1} Q_{s-1}, which is added here with the same arithmetic
    const int it = st->iter;
    if (it >= st->n_iterates || st->recorded >= it) return;
    if (st->status == SFB_PCG_INDEFINITE || st->status == SFB_PCG_NONFINITE) return;
    double* dst = iterates + (size_t)it * rows * cols;
    if (Q0 != nullptr && it >= 1) {
        const double alpha = st->alpha;
        const double* Q = ((it - 1) & 1) ? Q1 : Q0;
        ROW_LOOP(rows, cols) dst[(size_t)r * cols + cc] =
            __dadd_rn(U[(size_t)r * ld + cc], __dmul_rn(alpha, Q[(size_t)r * ld + cc]));
    } else {
        ROW_LOOP(rows, cols) dst[(size_t)r * cols + cc] = U[(size_t)r * ld + cc];
    }
    if (arrive_last(&st->counter[5], gridDim.x)) {
        if (threadIdx.x == 0) {
            st->counter[5] = 0;
            st->recorded = it;
        }
    }
}

__global__ void __launch_bounds__(VT) copy_dot_kernel(const double* __restrict__ R, double* __restrict__ Z, int ld,
                                                      int rows, int cols, double* partials, PcgState* st,
                                                      double* dot_out, unsigned* counter) {
    SFB_PDL_PROLOGUE();
    if (st != nullptr && st->status != SFB_PCG_RUNNING) return;
    double zr = 0.0;
    const bool vec = (ld & 1) == 0 && ((reinterpret_cast<uintptr_t>(R) | reinterpret_cast<uintptr_t>(Z)) & 15) == 0;
    if (vec) {
        // 16-byte pairs per row; several loads in flight per thread
        const int np = cols / 2;
        for (int r = blockIdx.x; r < rows; r += gridDim.x) {
            const double2* R2 = reinterpret_cast<const double2*>(R + (size_t)r * ld);
            double2* Z2 = reinterpret_cast<double2*>(Z + (size_t)r * ld);
            #pragma unroll 4
            for (int q = threadIdx.x; q < np; q += VT) {
                const double2 v = R2[q];
                Z2[q] = v;
                zr = fma(v.x, v.x, zr);
                zr = fma(v.y, v.y, zr);
            }
            if ((cols & 1) && threadIdx.x == 0) {
                const double v = R[(size_t)r * ld + cols - 1];
                Z[(size_t)r * ld + cols - 1] = v;
                zr = fma(v, v, zr);
            }
        }
    } else {
        ROW_LOOP(rows, cols) {
            const size_t o = (size_t)r * ld + cc;
            const double v = R[o];
            Z[o] = v;
            zr = fma(v, v, zr);
        }
    }
    __shared__ double sh[VT / 32];
    const double p = block_sum<VT>(zr, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = p;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = sum_partials<VT>(partials, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            *counter = 0;
            if (st != nullptr) st->rz_next = tot;
            if (dot_out != nullptr) *dot_out = tot;
        }
    }
}

__global__ void loop_ctl_kernel(PcgState* st, cudaGraphConditionalHandle handle, int use_handle) {
    SFB_PDL_PROLOGUE();
    // continue while running and below max_iter; the body counter is a hard
    // backstop so a logic error can never spin the device forever.
    const unsigned runs = ++st->counter[6];
    const bool keep = st->status == SFB_PCG_RUNNING && st->iter < st->max_iter &&
                      runs <= (unsigned)st->max_iter + 2u;
    if (use_handle) cudaGraphSetConditional(handle, keep ? 1u : 0u);
}

__global__ void __launch_bounds__(VT) norms_kernel(const double* A, int lda, const double* B, int ldb, int rows,
                                                   int cols, double* partials, RedSlots* out) {
    SFB_PDL_PROLOGUE();
    // v = { |A - B|, max|A| (finite entries), #non-finite(A), |A| }
    double d2 = 0.0, a2 = 0.0, mx = 0.0, bad = 0.0;
    ROW_LOOP(rows, cols) {
        const double a = A[(size_t)r * lda + cc];
        const double d = B ? a - B[(size_t)r * ldb + cc] : a;
        d2 = fma(d, d, d2);
        a2 = fma(a, a, a2);
        if (isfinite(a)) mx = fmax(mx, fabs(a));
        else bad += 1.0;
    }
    __shared__ double sh[VT / 32];
    __shared__ double smx[VT / 32];
    const double p0 = block_sum<VT>(d2, sh);
    const double p2 = block_sum<VT>(bad, sh);
    const double p3 = block_sum<VT>(a2, sh);
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
    __syncthreads();
    const unsigned nb = gridDim.x;
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int i = 0; i < VT / 32; ++i) m = fmax(m, smx[i]);
        partials[blockIdx.x] = p0;
        partials[nb + blockIdx.x] = m;
        partials[2 * nb + blockIdx.x] = p2;
        partials[3 * nb + blockIdx.x] = p3;
    }
    if (arrive_last(&out->counter[0], nb)) {
        const double t0 = sum_partials<VT>(partials, nb, 1, sh);
        const double t2 = sum_partials<VT>(partials + 2 * nb, nb, 1, sh);
        const double t3 = sum_partials<VT>(partials + 3 * nb, nb, 1, sh);
        double m = 0.0;  // max over the block maxima, by the whole block (a serial
        for (unsigned i = threadIdx.x; i < nb; i += VT) m = fmax(m, __ldcg(partials + nb + i));  // loop cost ~50 us)
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        __syncthreads();
        if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int i = 0; i < VT / 32; ++i) m = fmax(m, smx[i]);
            out->counter[0] = 0;
            out->v[0] = sqrt(t0);
            out->v[1] = m;
            out->v[2] = t2;
            out->v[3] = sqrt(t3);
        }
    }
}

// ---- host-synchronous building blocks of the sharded (multi-GPU) MO-PCG ----
__global__ void __launch_bounds__(VT) sh_update_kernel(double* U, double* R, const double* Q, const double* W, int ld,
                                                       int rows, int cols, double alpha, double* partials,
                                                       RedSlots* out) {
    SFB_PDL_PROLOGUE();
    double rr = 0.0;
    ROW_LOOP(rows, cols) {
        const size_t o = (size_t)r * ld + cc;
        U[o] = __dadd_rn(U[o], __dmul_rn(alpha, Q[o]));
        const double rv = __dsub_rn(R[o], __dmul_rn(alpha, W[o]));
        R[o] = rv;
        rr = fma(rv, rv, rr);
    }
    __shared__ double sh[VT / 32];
    const double p = block_sum<VT>(rr, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = p;
    if (arrive_last(&out->counter[0], gridDim.x)) {
        const double t = sum_partials<VT>(partials, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            out->counter[0] = 0;
            out->v[0] = t;
        }
    }
}

__global__ void __launch_bounds__(VT) sh_xpby_kernel(double* Q, int ldq, const double* Z, int ldz, int rows, int cols,
                                                     double beta, int first) {
    SFB_PDL_PROLOGUE();
    ROW_LOOP(rows, cols) {
        const double z = Z[(size_t)r * ldz + cc];
        double* q = Q + (size_t)r * ldq + cc;
        *q = first ? z : __dadd_rn(__dmul_rn(beta, *q), z);
    }
}

__global__ void __launch_bounds__(VT) sh_dots_kernel(const double* A, const double* B, const double* C,
                                                     const double* D, int ld, int rows, int cols, double* partials,
                                                     RedSlots* out) {
    SFB_PDL_PROLOGUE();
    double ab = 0.0, cd = 0.0;
    ROW_LOOP(rows, cols) {
        const size_t o = (size_t)r * ld + cc;
        ab = fma(A[o], B[o], ab);
        if (C) cd = fma(C[o], D[o], cd);
    }
    __shared__ double sh[VT / 32];
    const double p0 = block_sum<VT>(ab, sh);
    const double p1 = block_sum<VT>(cd, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = p0;
        partials[gridDim.x + blockIdx.x] = p1;
    }
    if (arrive_last(&out->counter[0], gridDim.x)) {
        const double t0 = sum_partials<VT>(partials, gridDim.x, 1, sh);
        const double t1 = sum_partials<VT>(partials + gridDim.x, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            out->counter[0] = 0;
            out->v[0] = t0;
            out->v[1] = t1;
        }
    }
}

// ---- device-resident sharded MO-PCG (no host round trip per iteration) ----
// The scalars of the column-sharded iteration live on the device: a PcgState
// (status, alpha, rz, ...) plus a slot array whose local sums are all-reduced
// in place by the communicator (NCCL on the stream).  Every kernel that
// changes the iterate is gated on the status, so a host that only looks at
// the status every few iterations sees exactly the reference trajectory.
//   slots[0] <W,Q>  slots[1] |Q|^2  slots[2] |R|^2  slots[3] <Z,R>  slots[4] beta
__global__ void __launch_bounds__(VT) shard_dots_kernel(const double* A, int lda, const double* B, int ldb,
                                                        const double* C, int ldc, const double* D, int ldd,
                                                        int rows, int cols, double* partials, unsigned* counter,
                                                        double* out0, double* out1) {
    SFB_PDL_PROLOGUE();
    double ab = 0.0, cd = 0.0;
    ROW_LOOP(rows, cols) {
        ab = fma(A[(size_t)r * lda + cc], B[(size_t)r * ldb + cc], ab);
        if (C) cd = fma(C[(size_t)r * ldc + cc], D[(size_t)r * ldd + cc], cd);
    }
    __shared__ double sh[VT / 32];
    const double p0 = block_sum<VT>(ab, sh);
    const double p1 = block_sum<VT>(cd, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = p0;
        partials[gridDim.x + blockIdx.x] = p1;
    }
    if (arrive_last(counter, gridDim.x)) {
        const double t0 = sum_partials<VT>(partials, gridDim.x, 1, sh);
        const double t1 = sum_partials<VT>(partials + gridDim.x, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            *counter = 0;
            *out0 = t0;
            if (out1) *out1 = t1;
        }
    }
}

// alpha = rz / <W,Q> (global), U += alpha Q, R -= alpha W, local |R|^2 -> slots[2]
__global__ void __launch_bounds__(VT) shard_update_kernel(double* U, int ldu, double* R, int ldr, const double* Q,
                                                          int ldq, const double* W, int ldw, int rows, int cols,
                                                          PcgState* st, double* slots, double* partials) {
    SFB_PDL_PROLOGUE();
    if (st->status != SFB_PCG_RUNNING) return;  // uniform gate
    const double wq = slots[0];
    const bool ok = wq > 0.0;
    const double alpha = st->rz / wq;
    double rr = 0.0;
    if (ok) {
        ROW_LOOP(rows, cols) {
            double* u = U + (size_t)r * ldu + cc;
            double* rp = R + (size_t)r * ldr + cc;
            *u = __dadd_rn(*u, __dmul_rn(alpha, Q[(size_t)r * ldq + cc]));
            const double rv = __dsub_rn(*rp, __dmul_rn(alpha, W[(size_t)r * ldw + cc]));
            *rp = rv;
            rr = fma(rv, rv, rr);
        }
    }
    __shared__ double sh[VT / 32];
    const double p = block_sum<VT>(rr, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = p;
    if (arrive_last(&st->counter[5], gridDim.x)) {
        const double t = sum_partials<VT>(partials, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            st->counter[5] = 0;
            if (!ok) {  // solvers.py:426-429
                st->status = SFB_PCG_INDEFINITE;
                st->bad_value = wq;
                st->bad_iter = st->iter;
            } else {
                st->alpha = alpha;
                st->qq = slots[1];
                slots[2] = t;
            }
        }
    }
}

// after the all-reduce of {|R_0|^2, <Z_0,R_0>}: res0, history[0], rz
__global__ void shard_start_kernel(PcgState* st, double* slots, double* hist) {
    const double res0 = sqrt(slots[2]);
    st->res0 = res0;
    st->rz = slots[3];
    hist[0] = res0;
    st->status = res0 == 0.0 ? SFB_PCG_TOLERANCE : (st->max_iter <= 0 ? SFB_PCG_MAX_ITER : SFB_PCG_RUNNING);
}

// after the all-reduce of {|R|^2, <Z,R>}: history, increment, stop test, beta
__global__ void shard_control_kernel(PcgState* st, double* slots, double* hist, double* incs) {
    if (st->status != SFB_PCG_RUNNING) return;
    pcg_finish_update(st, slots[2], hist, incs);
    const double rz_new = slots[3];
    slots[4] = rz_new / st->rz;
    st->rz = rz_new;
}

// Q = Z + beta Q (first: Q = Z), gated
__global__ void __launch_bounds__(VT) shard_xpby_kernel(double* Q, int ldq, const double* Z, int ldz, int rows,
                                                        int cols, const PcgState* st, const double* slots,
                                                        int first) {
    SFB_PDL_PROLOGUE();
    if (st->status != SFB_PCG_RUNNING) return;
    const double beta = slots[4];
    ROW_LOOP(rows, cols) {
        const double z = Z[(size_t)r * ldz + cc];
        double* q = Q + (size_t)r * ldq + cc;
        *q = first ? z : __dadd_rn(__dmul_rn(beta, *q), z);
    }
}

}  // namespace

int launch_shard_dots(const double* A, int lda, const double* B, int ldb, const double* C, int ldc, const double* D,
                      int ldd, int rows, int cols, double* partials, unsigned* counter, double* out0, double* out1,
                      cudaStream_t s) {
    SFB_TRY(launch_kernel(shard_dots_kernel, dim3(std::max(1, std::min(VB, rows))), dim3(VT), 0, s, A, lda, B, ldb,
                          C, ldc, D, ldd, rows, cols, partials, counter, out0, out1));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_shard_update(double* U, int ldu, double* R, int ldr, const double* Q, int ldq, const double* W, int ldw,
                        int rows, int cols, PcgState* st, double* slots, double* partials, cudaStream_t s) {
    SFB_TRY(launch_kernel(shard_update_kernel, dim3(std::max(1, std::min(VB, rows))), dim3(VT), 0, s, U, ldu, R, ldr,
                          Q, ldq, W, ldw, rows, cols, st, slots, partials));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_shard_start(PcgState* st, double* slots, double* hist, cudaStream_t s) {
    shard_start_kernel<<<1, 1, 0, s>>>(st, slots, hist);
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_shard_control(PcgState* st, double* slots, double* hist, double* incs, cudaStream_t s) {
    shard_control_kernel<<<1, 1, 0, s>>>(st, slots, hist, incs);
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_shard_xpby(double* Q, int ldq, const double* Z, int ldz, int rows, int cols, const PcgState* st,
                      const double* slots, int first, cudaStream_t s) {
    SFB_TRY(launch_kernel(shard_xpby_kernel, dim3(std::max(1, std::min(VB, rows))), dim3(VT), 0, s, Q, ldq, Z, ldz,
                          rows, cols, st, slots, first));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

// dst = src^T (rows x cols -> cols x rows) through 32 x 33 shared tiles.
__global__ void transpose_kernel(const double* __restrict__ src, int lds, double* __restrict__ dst, int ldd,
                                 int rows, int cols) {
    __shared__ double tl[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int r = r0 + k, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tl[k][threadIdx.x] = src[(size_t)r * lds + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int c = c0 + k, r = r0 + threadIdx.x;
        if (c < cols && r < rows) dst[(size_t)c * ldd + r] = tl[threadIdx.x][k];
    }
}

// ---- Strassen schedule around the DMMA GEMM, L levels flattened -----------
// C = A Bt^T with 2 x 2 blocks per level, B = Bt^T (B11 = Bt11^T, B12 = Bt21^T,
// B21 = Bt12^T, B22 = Bt22^T):
//   M0 = (A11 + A22)(B11 + B22)   M1 = (A21 + A22) B11     M2 = A11 (B12 - B22)
//   M3 = A22 (B21 - B11)          M4 = (A11 + A12) B22     M5 = (A21 - A11)(B11 + B12)
//   M6 = (A12 - A22)(B21 + B22)
//   C11 = M0 + M3 - M4 + M6   C12 = M2 + M4   C21 = M1 + M3   C22 = M0 - M1 + M2 + M5
// L levels are one bilinear algorithm with 7^L leaf products of 2^-L-size
// blocks: leaf l = (i_1 * 7 + i_2) * 7 + ... takes product i_1 at the top
// level, i_2 below it, and so on.  strassen_operands_kernel forms all 7^L leaf
// operands of one matrix in one pass (each thread holds the 4^L blocks' values
// at one position and walks the levels depth-first in registers: read 4^L,
// write 7^L blocks); strassen_assemble_kernel forms C from the 7^L leaf
// products the same way (read 7^L, write 4^L blocks), with the optional <C,D>
// of the MO-PCG preconditioner step (solvers.py:448) as a deterministic
// last-block reduction.  Blocks are indexed by their quadrant digits
// (q_1 ... q_L), q = 2 * (lower half) + (right half), most significant first.
constexpr int ST = 128;  // threads per CTA of the Strassen passes (one position per thread and step)

__host__ __device__ constexpr int pow_int(int b, int e) { return e == 0 ? 1 : b * pow_int(b, e - 1); }

// product i of a level: first quadrant (coefficient +1), second quadrant or -1, its sign
template <int SIDE>
struct StrassenIn {
    // SIDE 0 (A):  A11+A22, A21+A22, A11, A22, A11+A12, A21-A11, A12-A22
    // SIDE 1 (Bt): Bt11+Bt22, Bt11, Bt21-Bt22, Bt12-Bt11, Bt22, Bt11+Bt21, Bt12+Bt22
    __device__ static constexpr int qa(int i) {
        constexpr int a0[7] = {0, 2, 0, 3, 0, 2, 1}, a1[7] = {0, 0, 2, 1, 3, 0, 1};
        return SIDE == 0 ? a0[i] : a1[i];
    }
    __device__ static constexpr int qb(int i) {
        constexpr int b0[7] = {3, 3, -1, -1, 1, 0, 3}, b1[7] = {3, -1, 3, 0, -1, 2, 3};
        return SIDE == 0 ? b0[i] : b1[i];
    }
    __device__ static constexpr bool minus(int i) {
        constexpr bool m0[7] = {false, false, false, false, false, true, true},
                       m1[7] = {false, false, true, true, false, false, false};
        return SIDE == 0 ? m0[i] : m1[i];
    }
};

template <int L, int SIDE>
struct StrassenDown {
    template <class Store>
    __device__ __forceinline__ static void run(const double (&x)[pow_int(4, L)], int prefix, Store&& st) {
        constexpr int NS = pow_int(4, L - 1);
        #pragma unroll
        for (int i = 0; i < 7; ++i) {
            double y[NS];
            const int qa = StrassenIn<SIDE>::qa(i), qb = StrassenIn<SIDE>::qb(i);
            #pragma unroll
            for (int m = 0; m < NS; ++m) {
                if (qb < 0) y[m] = x[qa * NS + m];
                else y[m] = StrassenIn<SIDE>::minus(i) ? x[qa * NS + m] - x[qb * NS + m] : x[qa * NS + m] + x[qb * NS + m];
            }
            if constexpr (L == 1) st(prefix * 7 + i, y[0]);
            else StrassenDown<L - 1, SIDE>::run(y, prefix * 7 + i, st);
        }
    }
};

template <int L>
struct StrassenUp {
    // out[4^L] = the C blocks of the node whose leaves start at prefix * 7^L
    template <class Load>
    __device__ __forceinline__ static void run(double (&out)[pow_int(4, L)], int prefix, Load&& ld) {
        constexpr int NS = pow_int(4, L - 1);
        // product i adds into quadrant ca (+) and cb (minus when mb; -1: none); the first writer of a quadrant assigns
        constexpr int ca[7] = {0, 2, 1, 0, 1, 3, 0};     // +C11 +C21 +C12 +C11 +C12 +C22 +C11
        constexpr int cb[7] = {3, 3, 3, 2, 0, -1, -1};   // +C22 -C22 +C22 +C21 -C11
        constexpr bool mb[7] = {false, true, false, false, true, false, false};
        #pragma unroll
        for (int i = 0; i < 7; ++i) {
            double y[NS];
            if constexpr (L == 1) y[0] = ld(prefix * 7 + i);
            else StrassenUp<L - 1>::run(y, prefix * 7 + i, ld);
            #pragma unroll
            for (int m = 0; m < NS; ++m) {
                // i = 0 assigns C11, C22; i = 1 assigns C21; i = 2 assigns C12
                if (i == 0) {
                    out[0 * NS + m] = y[m];
                    out[3 * NS + m] = y[m];
                } else {
                    if (i == 1 || i == 2) out[ca[i] * NS + m] = y[m];
                    else out[ca[i] * NS + m] += y[m];
                    if (cb[i] >= 0) out[cb[i] * NS + m] = mb[i] ? out[cb[i] * NS + m] - y[m] : out[cb[i] * NS + m] + y[m];
                }
            }
        }
    }
};

// block (q_1 ... q_L) -> its row / column block index
template <int L>
__host__ __device__ constexpr int quad_row(int idx) {
    int r = 0;
    for (int l = 0; l < L; ++l) r |= ((idx >> (2 * l + 1)) & 1) << l;
    return r;
}
template <int L>
__host__ __device__ constexpr int quad_col(int idx) {
    int c = 0;
    for (int l = 0; l < L; ++l) c |= ((idx >> (2 * l)) & 1) << l;
    return c;
}

// X: rows x cols (ldx), read as (rh 2^L) x (ch 2^L) with zeros past its
// extents (odd shapes are padded virtually); leaf operand l at S + l * sstride
// (rh x ch, lds)
template <int L, int SIDE>
__global__ void __launch_bounds__(ST) strassen_operands_kernel(const double* __restrict__ X, int ldx, int rows,
                                                               int cols, int rh, int ch, double* __restrict__ S,
                                                               int lds, size_t sstride, const PcgState* gate) {
    SFB_PDL_PROLOGUE();
    if (gate != nullptr && gate->status != SFB_PCG_RUNNING) return;
    constexpr int NQ = pow_int(4, L);
    // work items: (row, ST-column chunk), round-robin over the CTAs (an even share
    // for every CTA of the VB-block grid whatever the row count)
    const int nchunk = (ch + ST - 1) / ST;
    for (int item = blockIdx.x; item < rh * nchunk; item += gridDim.x) {
        const int r = item / nchunk, c = (item - r * nchunk) * ST + threadIdx.x;
        if (c < ch) {
            double x[NQ];
            #pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int row = quad_row<L>(q) * rh + r, col = quad_col<L>(q) * ch + c;
                x[q] = (row < rows && col < cols) ? X[(size_t)row * ldx + col] : 0.0;
            }
            const size_t o = (size_t)r * lds + c;
            StrassenDown<L, SIDE>::run(x, 0, [&](int leaf, double v) { S[leaf * sstride + o] = v; });
        }
    }
}

// leaf product l at Mp + l * mstride (rh x ch, ldm); C: rows x cols (ldc), the
// leading part of the assembled (rh 2^L) x (ch 2^L)
template <int L, bool SCATTER>
__global__ void __launch_bounds__(ST) strassen_assemble_kernel(const double* __restrict__ Mp, int ldm, size_t mstride,
                                                               int rh, int ch, double* __restrict__ C, int ldc,
                                                               int rows, int cols, const double* __restrict__ D,
                                                               int ldd, double* partials, PcgState* st, double* dot_out,
                                                               unsigned* counter, int hmode, const double* __restrict__ sr,
                                                               const double* __restrict__ sc,
                                                               const __grid_constant__ ScatterArgs sa) {
    SFB_PDL_PROLOGUE();
    if (st != nullptr && st->status != SFB_PCG_RUNNING) return;
    constexpr int NQ = pow_int(4, L);
    double dot = 0.0;
    const int nchunk = (ch + ST - 1) / ST;
    for (int item = blockIdx.x; item < rh * nchunk; item += gridDim.x) {
        const int r = item / nchunk, c = (item - r * nchunk) * ST + threadIdx.x;
        if (c < ch) {
            const size_t o = (size_t)r * ldm + c;
            double out[NQ];
            StrassenUp<L>::run(out, 0, [&](int leaf) { return __ldg(Mp + leaf * mstride + o); });
            #pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int row = quad_row<L>(q) * rh + r, col = quad_col<L>(q) * ch + c;
                if (row < rows && col < cols) {
                    double v = out[q];
                    // the spectral sandwich's Hadamard scaling, as in the GEMM epilogues (solvers.py:245-253)
                    if (hmode == EPI_HADAMARD_SUM) v *= 1.0 / (sr[row] + sc[col]);
                    else if (hmode == EPI_HADAMARD_PROD) v *= sr[row] * sc[col];
                    if constexpr (SCATTER) {
                        int d = 0;
                        while (d + 1 < sa.nseg && row >= sa.seg[d + 1]) ++d;
                        sa.dst[d][(size_t)(row - sa.seg[d]) * sa.ldd[d] + sa.col_off + col] = v;
                    } else {
                        C[(size_t)row * ldc + col] = v;
                    }
                    if (D != nullptr) dot = fma(v, D[(size_t)row * ldd + col], dot);
                }
            }
        }
    }
    if (D == nullptr) return;  // uniform
    __shared__ double sh[ST / 32];
    const double p = block_sum<ST>(dot, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = p;
    if (arrive_last(counter, gridDim.x)) {
        const double tot = sum_partials<ST>(partials, gridDim.x, 1, sh);
        if (threadIdx.x == 0) {
            *counter = 0;
            if (st != nullptr) st->rz_next = tot;
            if (dot_out != nullptr) *dot_out = tot;
        }
    }
}

int vector_grid_blocks() { return VB; }

int launch_strassen_operands(int levels, int side, const double* X, int ldx, int rows, int cols, int rh, int ch,
                             double* S, int lds, size_t sstride, const PcgState* gate, cudaStream_t s) {
    const dim3 grid(std::max(1, std::min(VB, rh * ((ch + ST - 1) / ST)))), block(ST);
#define SFB_OPERANDS(L, SIDE)                                                                                      \
    if (levels == L && side == SIDE) {                                                                             \
        SFB_TRY(launch_kernel(strassen_operands_kernel<L, SIDE>, grid, block, 0, s, X, ldx, rows, cols, rh, ch, S, \
                              lds, sstride, gate));                                                                \
        SFB_CHECK_LAUNCH();                                                                                        \
        return SFB_OK;                                                                                             \
    }
    SFB_OPERANDS(1, 0)
    SFB_OPERANDS(1, 1)
    SFB_OPERANDS(2, 0)
    SFB_OPERANDS(2, 1)
    SFB_OPERANDS(3, 0)
    SFB_OPERANDS(3, 1)
#undef SFB_OPERANDS
    return arg_error("Strassen operands: 1 to 3 levels, side 0 or 1");
}

int launch_strassen_assemble(int levels, const double* Mp, int ldm, size_t mstride, int rh, int ch, double* C, int ldc,
                             int rows, int cols, const double* D, int ldd, double* partials, PcgState* st,
                             double* dot_out, unsigned* counter, cudaStream_t s, int hmode, const double* sr,
                             const double* sc, const ScatterArgs* scatter) {
    const dim3 grid(std::max(1, std::min(VB, rh * ((ch + ST - 1) / ST)))), block(ST);
    const ScatterArgs none;
#define SFB_ASSEMBLE(L)                                                                                          \
    if (levels == L) {                                                                                           \
        if (scatter != nullptr) {                                                                                \
            SFB_TRY(launch_kernel(strassen_assemble_kernel<L, true>, grid, block, 0, s, Mp, ldm, mstride, rh, ch, C, \
                                  ldc, rows, cols, D, ldd, partials, st, dot_out, counter, hmode, sr, sc, *scatter)); \
        } else {                                                                                                 \
            SFB_TRY(launch_kernel(strassen_assemble_kernel<L, false>, grid, block, 0, s, Mp, ldm, mstride, rh, ch, C, \
                                  ldc, rows, cols, D, ldd, partials, st, dot_out, counter, hmode, sr, sc, none)); \
        }                                                                                                        \
        SFB_CHECK_LAUNCH();                                                                                      \
        return SFB_OK;                                                                                           \
    }
    SFB_ASSEMBLE(1)
    SFB_ASSEMBLE(2)
    SFB_ASSEMBLE(3)
#undef SFB_ASSEMBLE
    return arg_error("Strassen assembly: 1 to 3 levels");
}

int launch_pcg_init_plain(const double* rhs, int ldr, double* R, double* U, int ld, int rows, int cols,
                          double* partials, PcgState* st, double* hist, cudaStream_t s) {
    SFB_TRY(launch_kernel(pcg_init_plain_kernel, dim3(VB), dim3(VT), 0, s, rhs, ldr, R, U, ld, rows, cols, partials, st, hist));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_pcg_init_warm(const double* rhs, int ldr, const double* W, double* R, int ld, int rows, int cols,
                         double* partials, PcgState* st, double* hist, cudaStream_t s) {
    SFB_TRY(launch_kernel(pcg_init_warm_kernel, dim3(VB), dim3(VT), 0, s, rhs, ldr, W, R, ld, rows, cols, partials, st, hist));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_pcg_direction(const double* Z, double* Q0, double* Q1, int ld, int rows, int cols, PcgState* st,
                         cudaStream_t s) {
    SFB_TRY(launch_kernel(pcg_direction_kernel, dim3(VB), dim3(VT), 0, s, Z, Q0, Q1, ld, rows, cols, st));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_pcg_dots(const double* W, const double* Q0, const double* Q1, int ld, int rows, int cols,
                    double* partials, PcgState* st, cudaStream_t s) {
    SFB_TRY(launch_kernel(pcg_dots_kernel, dim3(VB), dim3(VT), 0, s, W, Q0, Q1, ld, rows, cols, partials, st));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_pcg_update(double* U, double* R, const double* W, const double* Q0, const double* Q1, int ld,
                      int rows, int cols, double* partials, PcgState* st, double* hist, double* incs,
                      cudaStream_t s) {
    SFB_TRY(launch_kernel(pcg_update_kernel, dim3(VB), dim3(VT), 0, s, U, R, W, Q0, Q1, ld, rows, cols, partials, st, hist, incs));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_pcg_rupdate(double* R, const double* W, int ld, int rows, double* partials, PcgState* st, double* hist,
                       double* incs, cudaStream_t s, unsigned long long handle, int use_handle) {
    SFB_TRY(launch_kernel(pcg_rupdate_kernel, dim3(VB), dim3(VT), 0, s, R, W, ld, rows, partials, st, hist, incs,
                          (cudaGraphConditionalHandle)handle, use_handle));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_pcg_ufinal(double* U, const double* Q0, const double* Q1, int ld, int rows, PcgState* st, cudaStream_t s) {
    SFB_TRY(launch_kernel(pcg_ufinal_kernel, dim3(VB), dim3(VT), 0, s, U, Q0, Q1, ld, rows, (const PcgState*)st));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_pcg_record(const double* U, int ld, int rows, int cols, double* iterates, PcgState* st,
                      cudaStream_t s, const double* Q0, const double* Q1) {
    SFB_TRY(launch_kernel(pcg_record_kernel, dim3(VB), dim3(VT), 0, s, U, ld, rows, cols, iterates, st, Q0, Q1));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_copy_dot(const double* R, double* Z, int ld, int rows, int cols, double* partials, PcgState* st,
                    RedSlots* red, cudaStream_t s) {
    unsigned* counter = st ? &st->counter[3] : &red->counter[1];
    double* dot_out = red ? &red->v[3] : nullptr;
    SFB_TRY(launch_kernel(copy_dot_kernel, dim3(VB), dim3(VT), 0, s, R, Z, ld, rows, cols, partials, st, dot_out, counter));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_loop_ctl(PcgState* st, unsigned long long handle, int use_handle, cudaStream_t s) {
    SFB_TRY(launch_kernel(loop_ctl_kernel, dim3(1), dim3(1), 0, s, st, (cudaGraphConditionalHandle)handle, use_handle));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_norms(const double* A, int lda, const double* B, int ldb, int rows, int cols, double* partials,
                 RedSlots* out, cudaStream_t s) {
    // one block per row (ROW_LOOP): no more blocks than rows
    SFB_TRY(launch_kernel(norms_kernel, dim3(std::max(1, std::min(VB, rows))), dim3(VT), 0, s, A, lda, B, ldb, rows,
                          cols, partials, out));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_sh_update(double* U, double* R, const double* Q, const double* W, int ld, int rows, int cols,
                     double alpha, double* partials, RedSlots* out, cudaStream_t s) {
    SFB_TRY(launch_kernel(sh_update_kernel, dim3(VB), dim3(VT), 0, s, U, R, Q, W, ld, rows, cols, alpha, partials, out));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_sh_xpby(double* Q, int ldq, const double* Z, int ldz, int rows, int cols, double beta, int first,
                   cudaStream_t s) {
    SFB_TRY(launch_kernel(sh_xpby_kernel, dim3(VB), dim3(VT), 0, s, Q, ldq, Z, ldz, rows, cols, beta, first));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_sh_dots(const double* A, const double* B, const double* C, const double* D, int ld, int rows, int cols,
                   double* partials, RedSlots* out, cudaStream_t s) {
    SFB_TRY(launch_kernel(sh_dots_kernel, dim3(VB), dim3(VT), 0, s, A, B, C, D, ld, rows, cols, partials, out));
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

int launch_transpose(const double* src, int lds, double* dst, int ldd, int rows, int cols, cudaStream_t s) {
    const dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
    transpose_kernel<<<grid, block, 0, s>>>(src, lds, dst, ldd, rows, cols);
    SFB_CHECK_LAUNCH();
    return SFB_OK;
}

}  // namespace sfb
