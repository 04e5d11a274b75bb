// Objects behind the C ABI (include/sylfem_b200.h): device-resident operators,
// rhs maps, preconditioners and the MO-PCG driver.
//
// MO-PCG (solvers.py:365-453) runs entirely on the device: scalars (alpha,
// beta, |R|, stop test) live in a PcgState and are produced by the last CTA
// of the kernel that finishes each reduction, so no iteration needs a host
// round trip.  One iteration is captured once into the body of a CUDA-graph
// WHILE node whose condition is set by a one-thread control kernel; a whole
// solve is then a single graph launch and one final synchronisation.
#include <cuda.h>

#include <atomic>
#include <cstdlib>
#include <functional>
#include <cstring>
#include <mutex>
#include <vector>

#include "sfb_common.cuh"
#include "sfb_kernels.cuh"
#include "sfb_tma.cuh"

namespace sfb {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

namespace {

template <class T>
int talloc(T** p, size_t bytes) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
    if (e != cudaSuccess) {
        set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
        return SFB_ERR_NOMEM;
    }
    return SFB_OK;
}

// Upload a host matrix (rows x cols, contiguous) into a device buffer with
// leading dimension ld (zero padded).
// src may be host or device memory (unified addressing decides the copy)
int upload_padded(double* dst, int ld, const double* src, int rows, int cols) {
    SFB_CUDA_TRY(cudaMemset(dst, 0, (size_t)rows * ld * sizeof(double)));
    SFB_CUDA_TRY(cudaMemcpy2D(dst, (size_t)ld * sizeof(double), src, (size_t)cols * sizeof(double),
                              (size_t)cols * sizeof(double), rows, cudaMemcpyDefault));
    return SFB_OK;
}

struct ScopedFree {
    std::vector<void*> ptrs;
    cudaStream_t s;
    explicit ScopedFree(cudaStream_t st) : s(st) {}
    ~ScopedFree() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
    }
    template <class T>
    int get(T** p, size_t bytes) {
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), bytes ? bytes : 8, s);
        if (e != cudaSuccess) {
            set_error(std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
            return SFB_ERR_NOMEM;
        }
        ptrs.push_back(*p);
        return SFB_OK;
    }
};

inline int pad_ld(int cols) { return round_up(cols < 1 ? 1 : cols, 32); }

// The banded kernel reads its inputs by TMA (16-byte aligned rows).  Inputs
// that are not (odd leading dimension, offset views) are first copied into
// padded stream-ordered scratch.
int stage_aligned(ScopedFree& tmp, const double*& p, int& ld, int rows, int cols, cudaStream_t s) {
    if (p == nullptr || rows <= 0 || cols <= 0 || tma_aligned(p, ld)) return SFB_OK;
    const int pl = pad_ld(cols);
    double* q;
    SFB_TRY(tmp.get(&q, (size_t)rows * pl * 8));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(q, (size_t)pl * 8, p, (size_t)ld * 8, (size_t)cols * 8, rows,
                                   cudaMemcpyDeviceToDevice, s));
    p = q;
    ld = pl;
    return SFB_OK;
}

int launch_band_staged(BandArgs a, cudaStream_t s) {
    ScopedFree tmp(s);
    if (a.ld_mode == LD_HEAT) {
        SFB_TRY(stage_aligned(tmp, a.X, a.ldx, a.in_rows - 2 * a.rs, a.in_cols - 2 * a.cs, s));
        SFB_TRY(stage_aligned(tmp, a.X2, a.ldx2, a.in_rows, a.in_cols, s));
    } else if (a.ld_mode == LD_DIB) {
        SFB_TRY(stage_aligned(tmp, a.X, a.ldx, a.in_rows, a.in_cols, s));
        SFB_TRY(stage_aligned(tmp, a.X2, a.ldx2, a.in_rows, a.in_cols, s));
    } else if (a.ld_mode == LD_PLAIN) {
        SFB_TRY(stage_aligned(tmp, a.X, a.ldx, a.in_rows, a.in_cols, s));
    }
    return launch_band(a, s);
}

}  // namespace

// Stream-K workspace of the DMMA GEMM (partial tiles + per-tile counters).
struct GemmWs {
    double* ws = nullptr;
    unsigned* flags = nullptr;
    double* seg_f = nullptr;  // segmented-solve boundary states (banded preconditioner)
    double* seg_b = nullptr;
    double* strassen = nullptr;  // strassen_scratch_doubles(): operand sums and the seven products
};

// Temporary stream-K workspace from the stream-ordered pool.
template <class Pool>
int temp_ws(Pool& tmp, GemmWs& w, cudaStream_t s) {
    SFB_TRY(tmp.get(&w.ws, gemm_workspace_doubles() * sizeof(double)));
    SFB_TRY(tmp.get(&w.flags, (size_t)gemm_max_tiles() * sizeof(unsigned)));
    SFB_CUDA_TRY(cudaMemsetAsync(w.flags, 0, (size_t)gemm_max_tiles() * sizeof(unsigned), s));
    return SFB_OK;
}

inline GemmEpi with_ws(GemmEpi e, const GemmWs* w) {
    if (w != nullptr) {
        e.sk_ws = w->ws;
        e.sk_flags = w->flags;
    }
    return e;
}

}  // namespace sfb

using namespace sfb;

// =========================================================== operators ====
struct sfb_op {
    int qy = 0, qx = 0, nterms = 0;
    int in_cols = 0;  // == qx except for halo-extended column blocks (sharded)
    bool dense = false;
    int width = 1, goff = 0, hoff = 0;
    double* gband = nullptr;
    double* gskew = nullptr;  // band_skew(gband): TMA-boxable left coefficients
    double* hband = nullptr;
    // dense fallback: G_t (qy x qy) and H_t^T (qx x qx), padded rows
    double* G = nullptr;
    double* Ht = nullptr;
    int ldG = 0, ldH = 0;
};

struct sfb_map {
    int out_rows = 0, out_cols = 0, in_rows = 0, in_cols = 0;
    int width = 1, goff = 0, hoff = 0;
    double* gband = nullptr;
    double* gskew = nullptr;
    double* hband = nullptr;
};

namespace sfb {
namespace {
struct StrassenPlan;  // block sums of a constant left operand (defined with the Strassen driver below)
}
}  // namespace sfb

struct sfb_pre {
    int kind = SFB_PRE_IDENTITY;
    int qy = 0, qx = 0;
    // INVERSE: A1 = P_L^-1, B1 = (P_R^-1)^T.  SPECTRAL: A1 = V_L, A1t = V_L^T,
    // B1 = V_R, B1t = V_R^T, sl/sr = lambda (sum) or 1/lambda (prod).
    double *A1 = nullptr, *A1t = nullptr, *B1 = nullptr, *B1t = nullptr;
    int ldA = 0, ldB = 0;
    double *sl = nullptr, *sr = nullptr;
    // INVERSE, large shapes divisible by 4: the five Strassen block sums of
    // A1 and B1 (the constant left operands of the two products), formed once
    sfb::StrassenPlan *planA = nullptr, *planB = nullptr;    // of A1, B1
    sfb::StrassenPlan *planAt = nullptr, *planBt = nullptr;  // of A1t, B1t (spectral sandwich)
    int strassen_levels = 0;
    bool strassen = false;
    // BANDED: factors prepared for the SPIKE solves (spike.cu)
    SpikeFactor fl, fr;
    size_t seg_doubles = 0;  // scratch per interface buffer
};

namespace sfb {
namespace {

inline int seg_tiles(int qy, int qx) {
    const int S = spike_length();
    return ((qx + S - 1) / S) * ((qy + S - 1) / S);
}

// Banded-kernel arguments describing an operator's factors (every use).
BandArgs op_band_args(const sfb_op* op) {
    BandArgs a;
    a.out_rows = a.in_rows = op->qy;
    a.out_cols = op->qx;
    a.in_cols = op->in_cols;
    a.nterms = op->nterms;
    a.width = op->width;
    a.goff = op->goff;
    a.hoff = op->hoff;
    a.gband = op->gband;
    a.gskew = op->gskew;
    a.gskew_rows = op->qy + op->width - 1;
    a.gskew_terms = band_skew_terms(op->nterms);
    a.hband = op->hband;
    return a;
}

// W = op(U) on device buffers (U must have an even ld and 16B alignment for
// the dense path).  T1 is qx x qy scratch (ld ldt) for the dense path.
int op_apply_impl(const sfb_op* op, const double* U, int ldu, double* W, int ldw, double* T1, int ldt,
                  const GemmWs* gw, cudaStream_t s) {
    if (!op->dense) {
        BandArgs a = op_band_args(op);
        a.ld_mode = LD_PLAIN;
        a.X = U;
        a.ldx = ldu;
        a.ep_mode = EP_STORE;
        a.W = W;
        a.ldw = ldw;
        return launch_band_staged(a, s);
    }
    for (int t = 0; t < op->nterms; ++t) {
        GemmEpi e1;
        e1.mode = EPI_STORE_T;  // T1 = (U H_t)^T
        e1.C = T1;
        e1.ldc = ldt;
        SFB_TRY(launch_dgemm_nt(U, ldu, op->Ht + (size_t)t * op->qx * op->ldH, op->ldH, op->qy, op->qx, op->qx,
                                with_ws(e1, gw), s));
        GemmEpi e2;
        e2.mode = t == 0 ? EPI_STORE : EPI_ACCUM;  // W (+)= G_t (U H_t)
        e2.C = W;
        e2.ldc = ldw;
        SFB_TRY(launch_dgemm_nt(op->G + (size_t)t * op->qy * op->ldG, op->ldG, T1, ldt, op->qy, op->qx, op->qy,
                                with_ws(e2, gw), s));
    }
    return SFB_OK;
}

// ---- Strassen around the DMMA GEMM ---------------------------------------
// The inverse-form preconditioner (solvers.py:103-143 as two dense products)
// multiplies by the same two matrices every iteration, so the leaf operands
// of the constant left factors are formed once (StrassenPlan, built in
// sfb_pre_create).  Per product: one pass forms the variable operand's 7^L
// leaf operands, one strided-batch DMMA launch does the 7^L leaf products,
// one pass assembles the result (and <Z,R>).  Three levels do 343/512 of the
// flops.  Used for shapes of at least strassen_min_q() (any parity: the
// passes pad odd shapes virtually) with leaves of at least a quarter of the
// threshold (SYLFEM_B200_STRASSEN_MINQ, default 2000, 0 = never;
// SYLFEM_B200_STRASSEN_LEVELS, default 3).  Measured per preconditioner
// application against one DMMA GEMM per product: q = 8192 (343 leaves of
// 1024^3) 45.5 vs 62.2 ms; q = 4095 (343 of 512^3) 6.58 vs 8.03 ms; q = 2047
// (49 of 512^3) 1.03 vs 1.10 ms; q = 1024: no gain (0.21 ms either way).
std::atomic<int>& strassen_min_q_slot() {
    static std::atomic<int> v([] {
        const char* e = std::getenv("SYLFEM_B200_STRASSEN_MINQ");
        return e ? std::atoi(e) : 2000;
    }());
    return v;
}
int strassen_min_q() { return strassen_min_q_slot().load(std::memory_order_relaxed); }
std::atomic<int>& strassen_max_levels_slot() {
    static std::atomic<int> v([] {
        const char* e = std::getenv("SYLFEM_B200_STRASSEN_LEVELS");
        return e ? std::max(0, std::min(3, std::atoi(e))) : 3;
    }());
    return v;
}

// leaf dimension of q with L levels: q padded (virtually, with zeros) to a
// multiple of 2^(L+1), so every leaf has an even dimension (16-byte rows)
int strassen_leaf(int q, int L) { return (round_up(q, 2 << L)) >> L; }

int strassen_levels_of(int q) {
    const int m = strassen_min_q();
    if (m <= 0 || q < m) return 0;
    const int leaf = std::max(m / 4, 16);
    for (int L = strassen_max_levels_slot().load(std::memory_order_relaxed); L > 0; --L)
        if (strassen_leaf(q, L) >= leaf) return L;
    return 0;
}
int strassen_levels(int qy, int qx) { return std::min(strassen_levels_of(qy), strassen_levels_of(qx)); }

// The constant left operand of a product (M x K): its 7^levels leaf operands
// (mh x ldk each, stacked), formed once.
struct StrassenPlan {
    int levels = 0, M = 0, K = 0, mh = 0, kh = 0, ldk = 0, leaves = 0;
    double* leaf = nullptr;
};

void free_strassen_plan(StrassenPlan* p) {
    if (!p) return;
    cudaFree(p->leaf);
    delete p;
}

int build_strassen_plan(const double* A, int lda, int M, int K, int levels, StrassenPlan** out) {
    auto* p = new StrassenPlan;
    p->levels = levels;
    p->M = M;
    p->K = K;
    p->leaves = 1;
    for (int l = 0; l < levels; ++l) p->leaves *= 7;
    p->mh = strassen_leaf(M, levels);
    p->kh = strassen_leaf(K, levels);
    p->ldk = pad_ld(p->kh);
    const size_t sa = (size_t)p->mh * p->ldk;
    int rc = dalloc(&p->leaf, sa * p->leaves);
    if (rc == SFB_OK && cudaMemset(p->leaf, 0, sa * p->leaves * 8) != cudaSuccess) rc = SFB_ERR_CUDA;
    if (rc == SFB_OK)
        rc = launch_strassen_operands(levels, 0, A, lda, M, K, p->mh, p->kh, p->leaf, p->ldk, sa, nullptr, nullptr);
    if (rc != SFB_OK) {
        free_strassen_plan(p);
        return rc;
    }
    *out = p;
    return SFB_OK;
}

// scratch of a product: the variable operand's leaf operands and the leaf products
size_t strassen_scratch_doubles(int qy, int qx, int levels) {
    const int h = strassen_leaf(std::max(qy, qx), levels);
    size_t leaves = 1;
    for (int l = 0; l < levels; ++l) leaves *= 7;
    return 2 * leaves * (size_t)h * pad_ld(h);
}

// C[M x N] = A[M x K] Bt[N x K]^T with A's leaf operands in `pl`: one pass
// for Bt's leaf operands, the leaf products as one strided-batch DMMA launch
// (split only when they exceed the stream-K ticket array), one assembly pass.
int strassen_apply(const StrassenPlan* pl, const double* Bt, int ldb, int N, double* scratch, double* C, int ldc,
                   const double* D, int ldd, double* partials, PcgState* pcg, double* dot_out, unsigned* counter,
                   const GemmWs* gw, cudaStream_t s, int hmode = EPI_STORE, const double* sr = nullptr,
                   const double* sc = nullptr, const ScatterArgs* scatter = nullptr) {
    const int L = pl->levels, mh = pl->mh, nh = strassen_leaf(N, L), kh = pl->kh;
    const int ldk = pl->ldk, ldn = pad_ld(nh);
    const size_t sa = (size_t)mh * ldk, sb = (size_t)nh * ldk, sm = (size_t)mh * ldn;
    double* Bl = scratch;
    double* Mp = scratch + (size_t)pl->leaves * sb;
    SFB_TRY(launch_strassen_operands(L, 1, Bt, ldb, N, pl->K, nh, kh, Bl, ldk, sb, pcg, s));
    GemmEpi e;
    e.mode = EPI_STORE;
    e.ldc = ldn;
    e.pcg = pcg;
    const int per = std::max(1, gemm_batch_max(mh, nh));
    for (int l0 = 0; l0 < pl->leaves; l0 += per) {
        const int nb = std::min(per, pl->leaves - l0);
        e.C = Mp + (size_t)l0 * sm;
        SFB_TRY(launch_dgemm_nt_batch(pl->leaf + (size_t)l0 * sa, ldk, Bl + (size_t)l0 * sb, ldk, nb, mh, nh, kh,
                                      (long long)sm, with_ws(e, gw), s));
    }
    return launch_strassen_assemble(L, Mp, ldn, sm, mh, nh, C, ldc, pl->M, N, D, ldd, partials, pcg, dot_out, counter,
                                    s, hmode, sr, sc, scatter);
}

// Z = P^-1 R (or the reduced-solve sandwich).  R/Z device buffers with even
// ld; T1 (qx x qy, ldt1) and T2 (qy x qx, ldt2) scratch.  When `pcg` is set,
// kernels are gated on its status and <Z,R> lands in pcg->rz_next; otherwise
// it lands in red->v[3] when red is set.
int pre_apply_impl(const sfb_pre* p, const double* R, int ldr, double* Z, int ldz, double* T1, int ldt1,
                   double* T2, int ldt2, double* partials, PcgState* pcg, RedSlots* red, const GemmWs* gw,
                   cudaStream_t s) {
    const int qy = p->qy, qx = p->qx;
    unsigned* counter = pcg ? &pcg->counter[4] : (red ? &red->counter[2] : nullptr);
    GemmEpi last;
    last.mode = (pcg || red) ? EPI_STORE_DOT : EPI_STORE;
    last.C = Z;
    last.ldc = ldz;
    last.D = R;
    last.ldd = ldr;
    last.partials = partials;
    last.counter = counter;
    last.pcg = pcg;
    last.dot_out = red ? &red->v[3] : nullptr;
    switch (p->kind) {
        case SFB_PRE_IDENTITY:
            if (ldr != ldz) return arg_error("identity preconditioner needs matching leading dimensions");
            return launch_copy_dot(R, Z, ldz, qy, qx, partials, pcg, red, s);
        case SFB_PRE_INVERSE: {
            if (p->strassen && gw != nullptr && gw->strassen != nullptr) {
                // T1 = P_R^-T R^T, then Z = P_L^-1 T1^T with <Z,R> in the assembly pass
                SFB_TRY(strassen_apply(p->planB, R, ldr, qy, gw->strassen, T1, ldt1, nullptr, 0, nullptr, pcg, nullptr,
                                       nullptr, gw, s));
                const bool dot = pcg || red;
                return strassen_apply(p->planA, T1, ldt1, qx, gw->strassen, Z, ldz, dot ? R : nullptr, ldr, partials,
                                      pcg, red ? &red->v[3] : nullptr, counter, gw, s);
            }
            GemmEpi e1;  // T1 = (R P_R^-1)^T
            e1.mode = EPI_STORE_T;
            e1.C = T1;
            e1.ldc = ldt1;
            e1.pcg = pcg;
            SFB_TRY(launch_dgemm_nt(R, ldr, p->B1, p->ldB, qy, qx, qx, with_ws(e1, gw), s));
            // Z = P_L^-1 (R P_R^-1)
            return launch_dgemm_nt(p->A1, p->ldA, T1, ldt1, qy, qx, qy, with_ws(last, gw), s);
        }
        case SFB_PRE_SPECTRAL_PROD:
        case SFB_PRE_SPECTRAL_SUM: {
            if (p->strassen && gw != nullptr && gw->strassen != nullptr) {
                // the same four products with the constant factor on the left of each:
                // T1 = V_R^T R^T; T2 = (V_L^T T1^T) o K; T1 = V_R T2^T; Z = V_L T1^T (+ <Z,R>)
                const int hm = p->kind == SFB_PRE_SPECTRAL_SUM ? EPI_HADAMARD_SUM : EPI_HADAMARD_PROD;
                SFB_TRY(strassen_apply(p->planBt, R, ldr, qy, gw->strassen, T1, ldt1, nullptr, 0, nullptr, pcg, nullptr,
                                       nullptr, gw, s));
                SFB_TRY(strassen_apply(p->planAt, T1, ldt1, qx, gw->strassen, T2, ldt2, nullptr, 0, nullptr, pcg,
                                       nullptr, nullptr, gw, s, hm, p->sl, p->sr));
                SFB_TRY(strassen_apply(p->planB, T2, ldt2, qy, gw->strassen, T1, ldt1, nullptr, 0, nullptr, pcg, nullptr,
                                       nullptr, gw, s));
                const bool dot = pcg || red;
                return strassen_apply(p->planA, T1, ldt1, qx, gw->strassen, Z, ldz, dot ? R : nullptr, ldr, partials,
                                      pcg, red ? &red->v[3] : nullptr, counter, gw, s);
            }
            GemmEpi e1;  // T1 = (R V_R)^T
            e1.mode = EPI_STORE_T;
            e1.C = T1;
            e1.ldc = ldt1;
            e1.pcg = pcg;
            SFB_TRY(launch_dgemm_nt(R, ldr, p->B1t, p->ldB, qy, qx, qx, with_ws(e1, gw), s));
            GemmEpi e2;  // T2 = (V_L^T R V_R) o K
            e2.mode = p->kind == SFB_PRE_SPECTRAL_SUM ? EPI_HADAMARD_SUM : EPI_HADAMARD_PROD;
            e2.C = T2;
            e2.ldc = ldt2;
            e2.sr = p->sl;
            e2.sc = p->sr;
            e2.pcg = pcg;
            SFB_TRY(launch_dgemm_nt(p->A1t, p->ldA, T1, ldt1, qy, qx, qy, with_ws(e2, gw), s));
            GemmEpi e3;  // T1 = (T2 V_R^T)^T
            e3.mode = EPI_STORE_T;
            e3.C = T1;
            e3.ldc = ldt1;
            e3.pcg = pcg;
            SFB_TRY(launch_dgemm_nt(T2, ldt2, p->B1, p->ldB, qy, qx, qx, with_ws(e3, gw), s));
            // Z = V_L (T2 V_R^T)
            return launch_dgemm_nt(p->A1, p->ldA, T1, ldt1, qy, qx, qy, with_ws(last, gw), s);
        }
        case SFB_PRE_BANDED: {
            // Z = P_L^-1 R P_R^-1 by SPIKE solves (left along columns, right
            // along rows) with <Z,R> fused into the last tile pass.
            if (gw == nullptr || gw->seg_f == nullptr) return arg_error("banded preconditioner needs scratch");
            SegDot dot;
            dot.R = R;
            dot.ldr = ldr;
            dot.partials = partials;
            dot.counter = counter;
            dot.pcg = pcg;
            dot.dot_out = red ? &red->v[3] : nullptr;
            return launch_spike_pre(p->fl, p->fr, R, ldr, Z, ldz, (pcg || red) ? &dot : nullptr, gw->seg_f,
                                    gw->seg_b, pcg, s);
        }
    }
    return arg_error("unknown preconditioner kind");
}

}  // namespace
}  // namespace sfb

// =============================================================== PCG =====
struct sfb_pcg {
    const sfb_op* op = nullptr;
    const sfb_pre* pre = nullptr;
    int qy = 0, qx = 0, ld = 0, ldt1 = 0, ldt2 = 0;
    double *U = nullptr, *R = nullptr, *Z = nullptr, *Q0 = nullptr, *Q1 = nullptr, *W = nullptr, *B = nullptr;
    double *T1 = nullptr, *T2 = nullptr;
    double* partials = nullptr;
    GemmWs gw;
    PcgState* st = nullptr;
    double* hist = nullptr;
    double* incs = nullptr;
    int cap = 0;  // capacity of hist/incs (iterations)
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool conditional = false;
    int chunk = 0;
    double* graph_iterates = nullptr;
    std::mutex mu;
};

namespace sfb {
namespace {

// Enqueue one MO-PCG iteration; *ctl_done tells whether the iteration already
// set the WHILE condition (banded iteration: the R update's last CTA does it)
int pcg_enqueue_iteration(sfb_pcg* s, double* iterates, unsigned long long handle = 0, int use_handle = 0,
                          bool* ctl_done = nullptr) {
    if (ctl_done) *ctl_done = false;
    cudaStream_t st = s->stream;
    const sfb_op* op = s->op;
    if (!op->dense) {
        BandArgs a = op_band_args(op);
        a.ld_mode = LD_PCG;
        a.X = s->Z;
        a.ldx = s->ld;
        a.Q0 = s->Q0;
        a.Q1 = s->Q1;
        a.ldq = s->ld;
        a.ep_mode = EP_PCG;
        a.W = s->W;
        a.ldw = s->ld;
        a.partials = s->partials;
        a.pcg = s->st;
        a.U = s->U;  // receives the previous iteration's deferred U += alpha Q
        SFB_TRY(launch_band(a, st));
        SFB_TRY(launch_pcg_rupdate(s->R, s->W, s->ld, s->qy, s->partials, s->st, s->hist, s->incs, st, handle,
                                   use_handle));
        if (ctl_done) *ctl_done = true;
        if (iterates != nullptr)
            SFB_TRY(launch_pcg_record(s->U, s->ld, s->qy, s->qx, iterates, s->st, st, s->Q0, s->Q1));
    } else {
        // dense operator: single direction buffer updated in place
        SFB_TRY(launch_pcg_direction(s->Z, s->Q0, s->Q0, s->ld, s->qy, s->qx, s->st, st));
        for (int t = 0; t < op->nterms; ++t) {
            GemmEpi e1;
            e1.mode = EPI_STORE_T;
            e1.C = s->T1;
            e1.ldc = s->ldt1;
            e1.pcg = s->st;
            SFB_TRY(launch_dgemm_nt(s->Q0, s->ld, op->Ht + (size_t)t * op->qx * op->ldH, op->ldH, s->qy, s->qx,
                                    s->qx, with_ws(e1, &s->gw), st));
            GemmEpi e2;
            e2.mode = t == 0 ? EPI_STORE : EPI_ACCUM;
            e2.C = s->W;
            e2.ldc = s->ld;
            e2.pcg = s->st;
            SFB_TRY(launch_dgemm_nt(op->G + (size_t)t * op->qy * op->ldG, op->ldG, s->T1, s->ldt1, s->qy, s->qx,
                                    s->qy, with_ws(e2, &s->gw), st));
        }
        SFB_TRY(launch_pcg_dots(s->W, s->Q0, s->Q0, s->ld, s->qy, s->qx, s->partials, s->st, st));
        SFB_TRY(launch_pcg_update(s->U, s->R, s->W, s->Q0, s->Q0, s->ld, s->qy, s->qx, s->partials, s->st,
                                  s->hist, s->incs, st));
        if (iterates != nullptr) SFB_TRY(launch_pcg_record(s->U, s->ld, s->qy, s->qx, iterates, s->st, st));
    }
    return pre_apply_impl(s->pre, s->R, s->ld, s->Z, s->ld, s->T1, s->ldt1, s->T2, s->ldt2, s->partials, s->st,
                          nullptr, &s->gw, st);
}

void drop_graph(sfb_pcg* s) {
    if (s->exec) cudaGraphExecDestroy(s->exec);
    s->exec = nullptr;
}

// Build the iteration graph: a WHILE conditional node whose body is one
// MO-PCG iteration + the loop-control kernel.  Falls back to a plain graph of
// `chunk` iterations (host-driven) if conditional nodes are unavailable.
int build_graph(sfb_pcg* s, double* iterates) {
    drop_graph(s);
    cudaGraph_t g = nullptr;
    SFB_CUDA_TRY(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    // SYLFEM_B200_GRAPH=chunked forces the host-driven fallback (ncu cannot
    // profile kernel nodes of graphs that contain conditional nodes).
    const char* mode = std::getenv("SYLFEM_B200_GRAPH");
    const bool want_cond = !(mode && std::strcmp(mode, "chunked") == 0);
    bool ok = want_cond && cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
    if (ok) {
        alignas(cudaGraphNodeParams) unsigned char raw[sizeof(cudaGraphNodeParams)];
        std::memset(raw, 0, sizeof(raw));
        cudaGraphNodeParams& p = *reinterpret_cast<cudaGraphNodeParams*>(raw);
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        ok = cudaGraphAddNode(&node, g, nullptr, 0, &p) == cudaSuccess;
        if (ok) {
            cudaGraph_t body = p.conditional.phGraph_out[0];
            ok = cudaStreamBeginCaptureToGraph(s->stream, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                bool ctl = false;
                int rc = pcg_enqueue_iteration(s, iterates, (unsigned long long)h, 1, &ctl);
                if (rc == SFB_OK && !ctl) rc = launch_loop_ctl(s->st, (unsigned long long)h, 1, s->stream);
                cudaGraph_t captured = nullptr;
                cudaError_t e = cudaStreamEndCapture(s->stream, &captured);
                if (rc != SFB_OK) {
                    cudaGraphDestroy(g);
                    return rc;
                }
                ok = e == cudaSuccess;
            }
        }
        if (ok) ok = cudaGraphInstantiate(&s->exec, g, 0) == cudaSuccess;
    }
    cudaGraphDestroy(g);
    cudaGetLastError();  // clear any error from an unsupported conditional path
    if (ok) {
        s->conditional = true;
        s->graph_iterates = iterates;
        return SFB_OK;
    }
    // fallback: plain graph of `chunk` iterations
    s->conditional = false;
    s->chunk = 16;
    drop_graph(s);
    SFB_CUDA_TRY(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    int rc = SFB_OK;
    for (int i = 0; i < s->chunk && rc == SFB_OK; ++i) {
        bool ctl = false;
        rc = pcg_enqueue_iteration(s, iterates, 0, 0, &ctl);
        if (rc == SFB_OK && !ctl) rc = launch_loop_ctl(s->st, 0, 0, s->stream);
    }
    cudaGraph_t cg = nullptr;
    cudaError_t e = cudaStreamEndCapture(s->stream, &cg);
    if (rc != SFB_OK) {
        if (cg) cudaGraphDestroy(cg);
        return rc;
    }
    SFB_CUDA_TRY(e);
    cudaError_t ei = cudaGraphInstantiate(&s->exec, cg, 0);
    cudaGraphDestroy(cg);
    SFB_CUDA_TRY(ei);
    s->graph_iterates = iterates;
    return SFB_OK;
}

}  // namespace
}  // namespace sfb

// ================================================================ ABI =====
namespace sfb {
namespace {
template <class Fn>
int reduce_call(double* out, int n, cudaStream_t s, Fn fn) {
    ScopedFree tmp(s);
    double* parts;
    RedSlots* red;
    SFB_TRY(tmp.get(&parts, (size_t)2 * vector_grid_blocks() * 8));
    SFB_TRY(tmp.get(&red, sizeof(RedSlots)));
    SFB_CUDA_TRY(cudaMemsetAsync(red, 0, sizeof(RedSlots), s));
    SFB_TRY(fn(parts, red));
    RedSlots h;
    SFB_CUDA_TRY(cudaMemcpyAsync(&h, red, sizeof(h), cudaMemcpyDeviceToHost, s));
    SFB_CUDA_TRY(cudaStreamSynchronize(s));
    for (int i = 0; i < n; ++i) out[i] = h.v[i];
    return SFB_OK;
}
}  // namespace
}  // namespace sfb

extern "C" {

int sfb_version(void) { return 1; }

const char* sfb_last_error(void) { return g_last_error.c_str(); }

int sfb_set_strassen_min_q(int min_q) {
    const int prev = strassen_min_q();
    strassen_min_q_slot().store(min_q < 0 ? 0 : min_q, std::memory_order_relaxed);
    return prev;
}

int sfb_pre_uses_strassen(const sfb_pre* p) { return p != nullptr && p->strassen ? p->strassen_levels : 0; }

int sfb_set_strassen_levels(int levels) {
    const int prev = strassen_max_levels_slot().load(std::memory_order_relaxed);
    strassen_max_levels_slot().store(std::max(0, std::min(3, levels)), std::memory_order_relaxed);
    return prev;
}

int sfb_init(int device, int* sm_count) {
    SFB_CUDA_TRY(cudaSetDevice(device));
    int n = 0;
    SFB_CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    if (sm_count) *sm_count = n;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return SFB_OK;
}

// ------------------------------------------------------------ operator ---
int sfb_op_create(int qy, int qx, int nterms, int gw, int goff, const double* gband, int hw, int hoff,
                  const double* hband, sfb_op** out) {
    if (qy <= 0 || qx <= 0 || nterms <= 0) return arg_error("operator needs positive shape and terms");
    if (gw != hw) return arg_error("left and right band widths must be padded to a common width");
    if (!band_supported(nterms, gw)) {
        set_error("banded operator: unsupported width/terms");
        return SFB_ERR_UNSUPPORTED;
    }
    auto* op = new sfb_op;
    op->qy = qy;
    op->qx = qx;
    op->in_cols = qx;
    op->nterms = nterms;
    op->width = gw;
    op->goff = goff;
    op->hoff = hoff;
    const std::vector<double> skew = band_skew(gband, nterms, qy, gw);
    int rc = dalloc(&op->gband, (size_t)nterms * qy * gw);
    if (rc == SFB_OK) rc = dalloc(&op->gskew, skew.size());
    if (rc == SFB_OK && cudaMemcpy(op->gskew, skew.data(), skew.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = SFB_ERR_CUDA;
    if (rc == SFB_OK) rc = dalloc(&op->hband, (size_t)nterms * qx * hw);
    if (rc == SFB_OK && cudaMemcpy(op->gband, gband, (size_t)nterms * qy * gw * 8, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = SFB_ERR_CUDA;
    if (rc == SFB_OK && cudaMemcpy(op->hband, hband, (size_t)nterms * qx * hw * 8, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = SFB_ERR_CUDA;
    if (rc != SFB_OK) {
        if (rc == SFB_ERR_CUDA) set_error("uploading operator bands failed");
        sfb_op_destroy(op);
        return rc;
    }
    *out = op;
    return SFB_OK;
}

int sfb_op_create_block(int qy, int out_cols, int in_cols, int nterms, int w, int goff, const double* gband,
                        int hoff, const double* hband, sfb_op** out) {
    if (in_cols < out_cols) return arg_error("halo-extended block needs in_cols >= out_cols");
    SFB_TRY(sfb_op_create(qy, out_cols, nterms, w, goff, gband, w, hoff, hband, out));
    (*out)->in_cols = in_cols;
    return SFB_OK;
}

int sfb_op_create_dense(int qy, int qx, int nterms, const double* G, const double* H, sfb_op** out) {
    if (qy <= 0 || qx <= 0 || nterms <= 0) return arg_error("operator needs positive shape and terms");
    auto* op = new sfb_op;
    op->dense = true;
    op->qy = qy;
    op->qx = qx;
    op->in_cols = qx;
    op->nterms = nterms;
    op->ldG = pad_ld(qy);
    op->ldH = pad_ld(qx);
    int rc = dalloc(&op->G, (size_t)nterms * qy * op->ldG);
    if (rc == SFB_OK) rc = dalloc(&op->Ht, (size_t)nterms * qx * op->ldH);
    std::vector<double> tr((size_t)qx * qx);
    for (int t = 0; t < nterms && rc == SFB_OK; ++t) {
        rc = upload_padded(op->G + (size_t)t * qy * op->ldG, op->ldG, G + (size_t)t * qy * qy, qy, qy);
        const double* Ht = H + (size_t)t * qx * qx;
        for (int i = 0; i < qx; ++i)
            for (int j = 0; j < qx; ++j) tr[(size_t)j * qx + i] = Ht[(size_t)i * qx + j];
        if (rc == SFB_OK) rc = upload_padded(op->Ht + (size_t)t * qx * op->ldH, op->ldH, tr.data(), qx, qx);
    }
    if (rc != SFB_OK) {
        sfb_op_destroy(op);
        return rc;
    }
    *out = op;
    return SFB_OK;
}

int sfb_op_apply(const sfb_op* op, const double* U, int ldu, double* W, int ldw, void* stream) {
    SFB_NVTX("sfb_op_apply");
    if (!op) return arg_error("null operator");
    cudaStream_t s = (cudaStream_t)stream;
    if (!op->dense) return op_apply_impl(op, U, ldu, W, ldw, nullptr, 0, nullptr, s);
    ScopedFree tmp(s);
    const int ld = pad_ld(op->qx), ldt = pad_ld(op->qy);
    double *Ub, *Wb, *T1;
    SFB_TRY(tmp.get(&Ub, (size_t)op->qy * ld * 8));
    SFB_TRY(tmp.get(&Wb, (size_t)op->qy * ld * 8));
    SFB_TRY(tmp.get(&T1, (size_t)op->qx * ldt * 8));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(Ub, (size_t)ld * 8, U, (size_t)ldu * 8, (size_t)op->qx * 8, op->qy,
                                   cudaMemcpyDeviceToDevice, s));
    GemmWs gw;
    SFB_TRY(temp_ws(tmp, gw, s));
    SFB_TRY(op_apply_impl(op, Ub, ld, Wb, ld, T1, ldt, &gw, s));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(W, (size_t)ldw * 8, Wb, (size_t)ld * 8, (size_t)op->qx * 8, op->qy,
                                   cudaMemcpyDeviceToDevice, s));
    return SFB_OK;
}

int sfb_op_residual(const sfb_op* op, const double* U, int ldu, const double* rhs, int ldr, double* out2,
                    void* stream) {
    if (!op) return arg_error("null operator");
    cudaStream_t s = (cudaStream_t)stream;
    ScopedFree tmp(s);
    const int ld = pad_ld(op->qx);
    double *Wb, *parts;
    RedSlots* red;
    SFB_TRY(tmp.get(&Wb, (size_t)op->qy * ld * 8));
    SFB_TRY(tmp.get(&parts, (size_t)4 * vector_grid_blocks() * 8));
    SFB_TRY(tmp.get(&red, 2 * sizeof(RedSlots)));
    SFB_CUDA_TRY(cudaMemsetAsync(red, 0, 2 * sizeof(RedSlots), s));
    SFB_TRY(sfb_op_apply(op, U, ldu, Wb, ld, stream));
    SFB_TRY(launch_norms(Wb, ld, rhs, ldr, op->qy, op->qx, parts, red, s));
    SFB_TRY(launch_norms(rhs, ldr, nullptr, 0, op->qy, op->qx, parts, red + 1, s));
    RedSlots h[2];
    SFB_CUDA_TRY(cudaMemcpyAsync(h, red, sizeof(h), cudaMemcpyDeviceToHost, s));
    SFB_CUDA_TRY(cudaStreamSynchronize(s));
    out2[0] = h[0].v[0];
    out2[1] = h[1].v[0];
    return SFB_OK;
}

int sfb_op_destroy(sfb_op* op) {
    if (!op) return SFB_OK;
    cudaFree(op->gband);
    cudaFree(op->gskew);
    cudaFree(op->hband);
    cudaFree(op->G);
    cudaFree(op->Ht);
    delete op;
    return SFB_OK;
}

// ----------------------------------------------------------------- maps ---
int sfb_map_create(int out_rows, int out_cols, int in_rows, int in_cols, int gw, int goff, const double* gband,
                   int hw, int hoff, const double* hband, sfb_map** out) {
    if (out_rows <= 0 || out_cols <= 0 || in_rows <= 0 || in_cols <= 0) return arg_error("empty map");
    if (gw != hw) return arg_error("left and right band widths must be padded to a common width");
    if (!band_supported(1, gw)) {
        set_error("rhs map: unsupported band width");
        return SFB_ERR_UNSUPPORTED;
    }
    auto* m = new sfb_map;
    m->out_rows = out_rows;
    m->out_cols = out_cols;
    m->in_rows = in_rows;
    m->in_cols = in_cols;
    m->width = gw;
    m->goff = goff;
    m->hoff = hoff;
    const std::vector<double> skew = band_skew(gband, 1, out_rows, gw);
    int rc = dalloc(&m->gband, (size_t)out_rows * gw);
    if (rc == SFB_OK) rc = dalloc(&m->gskew, skew.size());
    if (rc == SFB_OK) rc = dalloc(&m->hband, (size_t)out_cols * hw);
    if (rc == SFB_OK && (cudaMemcpy(m->gband, gband, (size_t)out_rows * gw * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
                         cudaMemcpy(m->gskew, skew.data(), skew.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
                         cudaMemcpy(m->hband, hband, (size_t)out_cols * hw * 8, cudaMemcpyHostToDevice) != cudaSuccess)) {
        set_error("uploading map bands failed");
        rc = SFB_ERR_CUDA;
    }
    if (rc != SFB_OK) {
        sfb_map_destroy(m);
        return rc;
    }
    *out = m;
    return SFB_OK;
}

namespace {
BandArgs map_args(const sfb_map* m, double* out, int ldo) {
    BandArgs a;
    a.out_rows = m->out_rows;
    a.out_cols = m->out_cols;
    a.in_rows = m->in_rows;
    a.in_cols = m->in_cols;
    a.nterms = 1;
    a.width = m->width;
    a.goff = m->goff;
    a.hoff = m->hoff;
    a.gband = m->gband;
    a.gskew = m->gskew;
    a.gskew_rows = m->out_rows + m->width - 1;
    a.gskew_terms = band_skew_terms(1);
    a.hband = m->hband;
    a.ep_mode = EP_STORE;
    a.W = out;
    a.ldw = ldo;
    return a;
}

int run_checked(BandArgs& a, double* check2, cudaStream_t s) {
    if (check2 == nullptr) return launch_band_staged(a, s);
    ScopedFree tmp(s);
    unsigned long long* chk;
    SFB_TRY(tmp.get(&chk, 2 * sizeof(unsigned long long)));
    SFB_CUDA_TRY(cudaMemsetAsync(chk, 0, 2 * sizeof(unsigned long long), s));
    a.check = chk;
    SFB_TRY(launch_band_staged(a, s));
    unsigned long long h[2];
    SFB_CUDA_TRY(cudaMemcpyAsync(h, chk, sizeof(h), cudaMemcpyDeviceToHost, s));
    SFB_CUDA_TRY(cudaStreamSynchronize(s));
    double mx;
    std::memcpy(&mx, &h[0], 8);
    check2[0] = mx;
    check2[1] = (double)h[1];
    return SFB_OK;
}
}  // namespace

int sfb_map_apply(const sfb_map* m, const double* F, int ldf, double* out, int ldo, void* stream) {
    if (!m) return arg_error("null map");
    BandArgs a = map_args(m, out, ldo);
    a.ld_mode = LD_PLAIN;
    a.X = F;
    a.ldx = ldf;
    return launch_band_staged(a, (cudaStream_t)stream);
}

int sfb_map_apply_heat(const sfb_map* m, const double* U, int ldu, int row_shift, int col_shift, double c,
                       const double* F, int ldf, double* out, int ldo, double* check2, void* stream) {
    SFB_NVTX("sfb_map_apply_heat");
    if (!m) return arg_error("null map");
    BandArgs a = map_args(m, out, ldo);
    a.ld_mode = LD_HEAT;
    a.X = U;
    a.ldx = ldu;
    a.X2 = F;
    a.ldx2 = ldf;
    a.c = c;
    a.rs = row_shift;
    a.cs = col_shift;
    return run_checked(a, check2, (cudaStream_t)stream);
}

int sfb_map_apply_dib(const sfb_map* m, const double* U, const double* V, int ld, int species, double tau_rho,
                      const double* params, double* out, int ldo, double* check2, void* stream) {
    SFB_NVTX("sfb_map_apply_dib");
    if (!m) return arg_error("null map");
    // zero-flux: the input grid is the output grid, or a column block of it
    // extended by a halo (in_cols > out_cols, the sharded IMEX driver)
    if (m->in_rows != m->out_rows || m->in_cols < m->out_cols)
        return arg_error("DIB rhs expects a zero-flux (square) map");
    BandArgs a = map_args(m, out, ldo);
    a.ld_mode = LD_DIB;
    a.X = U;
    a.X2 = V;
    a.ldx = ld;
    a.ldx2 = ld;
    a.species = species;
    a.c = tau_rho;
    for (int i = 0; i < 9; ++i) a.kp[i] = params[i];
    return run_checked(a, check2, (cudaStream_t)stream);
}

int sfb_map_destroy(sfb_map* m) {
    if (!m) return SFB_OK;
    cudaFree(m->gband);
    cudaFree(m->gskew);
    cudaFree(m->hband);
    delete m;
    return SFB_OK;
}

// ------------------------------------------------------- preconditioner ---
int sfb_pre_create(int qy, int qx, int kind, const double* L, const double* R, const double* lamL,
                   const double* lamR, sfb_pre** out) {
    if (qy <= 0 || qx <= 0) return arg_error("preconditioner needs a positive shape");
    auto* p = new sfb_pre;
    p->kind = kind;
    p->qy = qy;
    p->qx = qx;
    p->ldA = pad_ld(qy);
    p->ldB = pad_ld(qx);
    int rc = SFB_OK;
    auto fail = [&](int code) {
        sfb_pre_destroy(p);
        return code;
    };
    if (kind == SFB_PRE_IDENTITY) {
        *out = p;
        return SFB_OK;
    }
    if (kind == SFB_PRE_INVERSE) {
        if (!L || !R) return fail(arg_error("inverse preconditioner needs both factors"));
        rc = dalloc(&p->A1, (size_t)qy * p->ldA);
        if (rc == SFB_OK) rc = dalloc(&p->B1, (size_t)qx * p->ldB);
        if (rc == SFB_OK) rc = upload_padded(p->A1, p->ldA, L, qy, qy);
        if (rc == SFB_OK) rc = upload_padded(p->B1, p->ldB, R, qx, qx);
        const int levels = strassen_levels(qy, qx);
        if (rc == SFB_OK && levels > 0) {
            rc = build_strassen_plan(p->A1, p->ldA, qy, qy, levels, &p->planA);
            if (rc == SFB_OK) rc = build_strassen_plan(p->B1, p->ldB, qx, qx, levels, &p->planB);
            if (rc == SFB_OK && cudaDeviceSynchronize() != cudaSuccess) rc = SFB_ERR_CUDA;
            p->strassen = rc == SFB_OK;
            p->strassen_levels = levels;
        }
        if (rc != SFB_OK) return fail(rc);
        *out = p;
        return SFB_OK;
    }
    if (kind == SFB_PRE_SPECTRAL_PROD || kind == SFB_PRE_SPECTRAL_SUM) {
        if (!L || !R || !lamL || !lamR) return fail(arg_error("spectral sandwich needs V_L, V_R and eigenvalues"));
        rc = dalloc(&p->A1, (size_t)qy * p->ldA);
        if (rc == SFB_OK) rc = dalloc(&p->A1t, (size_t)qy * p->ldA);
        if (rc == SFB_OK) rc = dalloc(&p->B1, (size_t)qx * p->ldB);
        if (rc == SFB_OK) rc = dalloc(&p->B1t, (size_t)qx * p->ldB);
        if (rc == SFB_OK) rc = dalloc(&p->sl, qy);
        if (rc == SFB_OK) rc = dalloc(&p->sr, qx);
        // V (host or device memory) is copied once; the transposes are made on the device
        if (rc == SFB_OK) rc = upload_padded(p->A1, p->ldA, L, qy, qy);
        if (rc == SFB_OK) rc = cudaMemset(p->A1t, 0, (size_t)qy * p->ldA * 8) == cudaSuccess ? SFB_OK : SFB_ERR_CUDA;
        if (rc == SFB_OK) rc = launch_transpose(p->A1, p->ldA, p->A1t, p->ldA, qy, qy, nullptr);
        if (rc == SFB_OK) rc = upload_padded(p->B1, p->ldB, R, qx, qx);
        if (rc == SFB_OK) rc = cudaMemset(p->B1t, 0, (size_t)qx * p->ldB * 8) == cudaSuccess ? SFB_OK : SFB_ERR_CUDA;
        if (rc == SFB_OK) rc = launch_transpose(p->B1, p->ldB, p->B1t, p->ldB, qx, qx, nullptr);
        if (rc == SFB_OK && cudaDeviceSynchronize() != cudaSuccess) rc = SFB_ERR_CUDA;
        const int levels = strassen_levels(qy, qx);
        if (rc == SFB_OK && levels > 0) {
            rc = build_strassen_plan(p->A1, p->ldA, qy, qy, levels, &p->planA);
            if (rc == SFB_OK) rc = build_strassen_plan(p->A1t, p->ldA, qy, qy, levels, &p->planAt);
            if (rc == SFB_OK) rc = build_strassen_plan(p->B1, p->ldB, qx, qx, levels, &p->planB);
            if (rc == SFB_OK) rc = build_strassen_plan(p->B1t, p->ldB, qx, qx, levels, &p->planBt);
            if (rc == SFB_OK && cudaDeviceSynchronize() != cudaSuccess) rc = SFB_ERR_CUDA;
            p->strassen = rc == SFB_OK;
            p->strassen_levels = levels;
        }
        std::vector<double> vl(lamL, lamL + qy), vr(lamR, lamR + qx);
        if (kind == SFB_PRE_SPECTRAL_PROD) {
            for (auto& v : vl) v = 1.0 / v;
            for (auto& v : vr) v = 1.0 / v;
        }
        if (rc == SFB_OK && (cudaMemcpy(p->sl, vl.data(), qy * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
                             cudaMemcpy(p->sr, vr.data(), qx * 8, cudaMemcpyHostToDevice) != cudaSuccess)) {
            set_error("uploading eigenvalues failed");
            rc = SFB_ERR_CUDA;
        }
        if (rc != SFB_OK) return fail(rc);
        *out = p;
        return SFB_OK;
    }
    return fail(arg_error("unknown preconditioner kind"));
}

int sfb_pre_create_banded(int qy, int qx, int bwL, const double* lband, int bwR, const double* rband,
                          sfb_pre** out) {
    if (qy <= 0 || qx <= 0 || bwL < 0 || bwR < 0 || bwL > 4 || bwR > 4)
        return arg_error("bad banded preconditioner shape (half-bandwidth 0..4)");
    auto* p = new sfb_pre;
    p->kind = SFB_PRE_BANDED;
    p->qy = qy;
    p->qx = qx;
    int rc = build_spike_factor(qy, bwL, lband, p->fl);
    if (rc == SFB_OK) rc = build_spike_factor(qx, bwR, rband, p->fr);
    if (rc != SFB_OK) {
        sfb_pre_destroy(p);
        return rc;
    }
    p->seg_doubles = std::max(spike_interface_doubles(qy, bwL, qx), spike_interface_doubles(qx, bwR, qy));
    *out = p;
    return SFB_OK;
}

int sfb_pre_apply(const sfb_pre* p, const double* R, int ldr, double* Z, int ldz, void* stream) {
    SFB_NVTX("sfb_pre_apply");
    if (!p) return arg_error("null preconditioner");
    cudaStream_t s = (cudaStream_t)stream;
    ScopedFree tmp(s);
    const int ld = pad_ld(p->qx), ldt1 = pad_ld(p->qy);
    double *Rb, *Zb, *T1 = nullptr, *T2 = nullptr;
    SFB_TRY(tmp.get(&Rb, (size_t)p->qy * ld * 8));
    SFB_TRY(tmp.get(&Zb, (size_t)p->qy * ld * 8));
    if (p->kind != SFB_PRE_IDENTITY && p->kind != SFB_PRE_BANDED) {
        SFB_TRY(tmp.get(&T1, (size_t)p->qx * ldt1 * 8));
        SFB_TRY(tmp.get(&T2, (size_t)p->qy * ld * 8));
    }
    double* parts = nullptr;
    RedSlots* red = nullptr;
    SFB_TRY(tmp.get(&parts, (size_t)std::max(std::max(vector_grid_blocks(), gemm_grid_blocks(p->qy, p->qx)),
                                             seg_tiles(p->qy, p->qx)) * 8));
    SFB_TRY(tmp.get(&red, sizeof(RedSlots)));
    SFB_CUDA_TRY(cudaMemsetAsync(red, 0, sizeof(RedSlots), s));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(Rb, (size_t)ld * 8, R, (size_t)ldr * 8, (size_t)p->qx * 8, p->qy,
                                   cudaMemcpyDeviceToDevice, s));
    GemmWs gw;
    if (T1 != nullptr) SFB_TRY(temp_ws(tmp, gw, s));
    if (p->kind == SFB_PRE_BANDED) {
        SFB_TRY(tmp.get(&gw.seg_f, p->seg_doubles * 8));
        SFB_TRY(tmp.get(&gw.seg_b, p->seg_doubles * 8));
    }
    if (p->strassen) {
        // (padding columns of the scratch blocks are never read)
        SFB_TRY(tmp.get(&gw.strassen, strassen_scratch_doubles(p->qy, p->qx, p->strassen_levels) * 8));
    }
    SFB_TRY(pre_apply_impl(p, Rb, ld, Zb, ld, T1, ldt1, T2, ld, parts, nullptr, red, &gw, s));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(Z, (size_t)ldz * 8, Zb, (size_t)ld * 8, (size_t)p->qx * 8, p->qy,
                                   cudaMemcpyDeviceToDevice, s));
    return SFB_OK;
}

// ------------------------------------------------------- reduced solve ---
// solve_reduced (solvers.py:284-300) as one object: persistent padded
// buffers and GEMM workspace, and the whole solve — the spectral sandwich
// U = P1 [(P1^T B P2) / (lam1_i + lam2_j)] P2^T, the operator apply for the
// residual and its two norms — captured once into a CUDA graph.  A call is
// two copies, one graph launch and one sync (the per-call allocations and
// launches dominated small solves: cfg1, q = 256).
struct sfb_reduced {
    const sfb_pre* pre = nullptr;
    const sfb_op* op = nullptr;
    int qy = 0, qx = 0, ld = 0, ldt1 = 0;
    double *B = nullptr, *U = nullptr, *W = nullptr, *T1 = nullptr, *T2 = nullptr, *parts = nullptr;
    RedSlots* red = nullptr;
    double* host = nullptr;  // page-locked result scalars
    GemmWs gw;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::mutex mu;
};

int sfb_reduced_destroy(sfb_reduced* r) {
    if (!r) return SFB_OK;
    if (r->exec) cudaGraphExecDestroy(r->exec);
    for (void* p : {(void*)r->B, (void*)r->U, (void*)r->W, (void*)r->T1, (void*)r->T2, (void*)r->parts,
                    (void*)r->red, (void*)r->gw.ws, (void*)r->gw.flags, (void*)r->gw.strassen})
        cudaFree(p);
    if (r->host) cudaFreeHost(r->host);
    if (r->stream) cudaStreamDestroy(r->stream);
    if (r->ev_in) cudaEventDestroy(r->ev_in);
    if (r->ev_out) cudaEventDestroy(r->ev_out);
    delete r;
    return SFB_OK;
}

int sfb_reduced_create(const sfb_pre* pre, const sfb_op* op, sfb_reduced** out) {
    if (!pre || !op || !out) return arg_error("reduced solve: null argument");
    if (pre->kind != SFB_PRE_SPECTRAL_SUM) return arg_error("reduced solve needs a spectral-sum sandwich");
    if (pre->qy != op->qy || pre->qx != op->qx) return arg_error("reduced solve: operator and cache shapes differ");
    auto* r = new sfb_reduced;
    r->pre = pre;
    r->op = op;
    r->qy = op->qy;
    r->qx = op->qx;
    r->ld = pad_ld(r->qx);
    r->ldt1 = pad_ld(r->qy);
    const size_t g = (size_t)r->qy * r->ld;
    const size_t nparts = (size_t)std::max(std::max(vector_grid_blocks(), gemm_grid_blocks(r->qy, r->qx)),
                                           band_grid_blocks(r->qy, r->qx));
    int rc = dalloc(&r->B, g);
    if (rc == SFB_OK) rc = dalloc(&r->U, g);
    if (rc == SFB_OK) rc = dalloc(&r->W, g);
    if (rc == SFB_OK) rc = dalloc(&r->T1, (size_t)r->qx * r->ldt1);
    if (rc == SFB_OK) rc = dalloc(&r->T2, g);
    if (rc == SFB_OK) rc = dalloc(&r->parts, 4 * nparts);  // launch_norms: 4 partials per block
    if (rc == SFB_OK) rc = dalloc(&r->gw.ws, gemm_workspace_doubles());
    if (rc == SFB_OK && pre->strassen)
        rc = dalloc(&r->gw.strassen, strassen_scratch_doubles(r->qy, r->qx, pre->strassen_levels));
    if (rc == SFB_OK && (cudaMalloc(reinterpret_cast<void**>(&r->red), 3 * sizeof(RedSlots)) != cudaSuccess ||
                         cudaMalloc(reinterpret_cast<void**>(&r->gw.flags), gemm_max_tiles() * sizeof(unsigned)) !=
                             cudaSuccess ||
                         cudaMallocHost(reinterpret_cast<void**>(&r->host), 4 * sizeof(double)) != cudaSuccess))
        rc = SFB_ERR_NOMEM;
    // padding columns stay zero; the stream-K tile counters start (and return to) zero
    if (rc == SFB_OK) {
        for (double* p : {r->B, r->U, r->W, r->T2}) cudaMemset(p, 0, g * 8);
        cudaMemset(r->T1, 0, (size_t)r->qx * r->ldt1 * 8);
        cudaMemset(r->gw.flags, 0, gemm_max_tiles() * sizeof(unsigned));
        if (cudaDeviceSynchronize() != cudaSuccess) rc = SFB_ERR_CUDA;
    }
    if (rc == SFB_OK && (cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking) != cudaSuccess ||
                         cudaEventCreateWithFlags(&r->ev_in, cudaEventDisableTiming) != cudaSuccess ||
                         cudaEventCreateWithFlags(&r->ev_out, cudaEventDisableTiming) != cudaSuccess))
        rc = SFB_ERR_CUDA;
    if (rc == SFB_OK) {
        cudaStream_t st = r->stream;
        cudaGraph_t graph = nullptr;
        if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            rc = SFB_ERR_CUDA;
        } else {
            int c = cudaMemsetAsync(r->red, 0, 3 * sizeof(RedSlots), st) == cudaSuccess ? SFB_OK : SFB_ERR_CUDA;
            if (c == SFB_OK)
                // plain store epilogue: the reduced solve needs no <U,B>
                c = pre_apply_impl(pre, r->B, r->ld, r->U, r->ld, r->T1, r->ldt1, r->T2, r->ld, r->parts, nullptr,
                                   nullptr, &r->gw, st);
            if (c == SFB_OK && !op->dense) {
                // banded operator: the residual |B - L(U)|, |B| in the operator pass itself
                BandArgs a = op_band_args(op);
                a.ld_mode = LD_PLAIN;
                a.X = r->U;
                a.ldx = r->ld;
                a.ep_mode = EP_RESID;
                a.B = r->B;
                a.ldb = r->ld;
                a.res = r->red;
                a.partials = r->parts;
                c = launch_band(a, st);
            } else if (c == SFB_OK) {
                c = op_apply_impl(op, r->U, r->ld, r->W, r->ld, r->T1, r->ldt1, &r->gw, st);
                // one pass: red[0] = { |B - W|, max|B|, #non-finite, |B| }
                if (c == SFB_OK) c = launch_norms(r->B, r->ld, r->W, r->ld, r->qy, r->qx, r->parts, r->red, st);
            }
            const cudaError_t e = cudaStreamEndCapture(st, &graph);
            rc = c != SFB_OK ? c : (e == cudaSuccess ? SFB_OK : SFB_ERR_CUDA);
            if (rc == SFB_OK && cudaGraphInstantiate(&r->exec, graph, 0) != cudaSuccess) rc = SFB_ERR_CUDA;
            if (graph) cudaGraphDestroy(graph);
        }
    }
    if (rc != SFB_OK) {
        if (rc == SFB_ERR_CUDA) set_error("reduced solve: building the solve graph failed");
        sfb_reduced_destroy(r);
        return rc;
    }
    *out = r;
    return SFB_OK;
}

int sfb_reduced_solve(sfb_reduced* r, const double* B, int ldb, double* U, int ldu, double* res2_host,
                                 void* stream) {
    SFB_NVTX("sfb_reduced_solve");
    if (!r || !B || !U) return arg_error("reduced solve: null argument");
    std::lock_guard<std::mutex> lock(r->mu);
    cudaStream_t cs = (cudaStream_t)stream, st = r->stream;
    SFB_CUDA_TRY(cudaEventRecord(r->ev_in, cs));
    SFB_CUDA_TRY(cudaStreamWaitEvent(st, r->ev_in, 0));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(r->B, (size_t)r->ld * 8, B, (size_t)ldb * 8, (size_t)r->qx * 8, r->qy,
                                   cudaMemcpyDeviceToDevice, st));
    SFB_CUDA_TRY(cudaGraphLaunch(r->exec, st));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(U, (size_t)ldu * 8, r->U, (size_t)r->ld * 8, (size_t)r->qx * 8, r->qy,
                                   cudaMemcpyDeviceToDevice, st));
    if (res2_host) {
        SFB_CUDA_TRY(cudaMemcpyAsync(r->host, &r->red[0].v[0], 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
        SFB_CUDA_TRY(cudaStreamSynchronize(st));
        res2_host[0] = r->host[0];  // |B - U|-residual numerator
        res2_host[1] = r->host[3];  // |B|
        return SFB_OK;              // everything is complete: the caller's stream needs no edge
    }
    SFB_CUDA_TRY(cudaEventRecord(r->ev_out, st));
    SFB_CUDA_TRY(cudaStreamWaitEvent(cs, r->ev_out, 0));
    return SFB_OK;
}

int sfb_pre_transform(const sfb_pre* p, const double* X, int ldx, double* Y, int ldy, void* stream) {
    if (!p) return arg_error("null preconditioner");
    if (p->kind != SFB_PRE_SPECTRAL_PROD && p->kind != SFB_PRE_SPECTRAL_SUM)
        return arg_error("spectral transform needs a spectral sandwich");
    cudaStream_t s = (cudaStream_t)stream;
    ScopedFree tmp(s);
    const int ld = pad_ld(p->qx), ldt1 = pad_ld(p->qy);
    double *Xb, *Yb, *T1;
    SFB_TRY(tmp.get(&Xb, (size_t)p->qy * ld * 8));
    SFB_TRY(tmp.get(&Yb, (size_t)p->qy * ld * 8));
    SFB_TRY(tmp.get(&T1, (size_t)p->qx * ldt1 * 8));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(Xb, (size_t)ld * 8, X, (size_t)ldx * 8, (size_t)p->qx * 8, p->qy,
                                   cudaMemcpyDeviceToDevice, s));
    GemmEpi e1;  // T1 = (X V_R)^T
    e1.mode = EPI_STORE_T;
    e1.C = T1;
    e1.ldc = ldt1;
    GemmWs gw;
    SFB_TRY(temp_ws(tmp, gw, s));
    SFB_TRY(launch_dgemm_nt(Xb, ld, p->B1t, p->ldB, p->qy, p->qx, p->qx, with_ws(e1, &gw), s));
    GemmEpi e2;  // Y = V_L^T X V_R
    e2.mode = EPI_STORE;
    e2.C = Yb;
    e2.ldc = ld;
    SFB_TRY(launch_dgemm_nt(p->A1t, p->ldA, T1, ldt1, p->qy, p->qx, p->qy, with_ws(e2, &gw), s));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(Y, (size_t)ldy * 8, Yb, (size_t)ld * 8, (size_t)p->qx * 8, p->qy,
                                   cudaMemcpyDeviceToDevice, s));
    return SFB_OK;
}

int sfb_pre_destroy(sfb_pre* p) {
    if (!p) return SFB_OK;
    cudaFree(p->A1);
    cudaFree(p->A1t);
    cudaFree(p->B1);
    cudaFree(p->B1t);
    cudaFree(p->sl);
    cudaFree(p->sr);
    free_strassen_plan(p->planA);
    free_strassen_plan(p->planB);
    free_strassen_plan(p->planAt);
    free_strassen_plan(p->planBt);
    free_spike_factor(p->fl);
    free_spike_factor(p->fr);
    delete p;
    return SFB_OK;
}

// ------------------------------------------------------------------ PCG ---
int sfb_pcg_create(const sfb_op* op, const sfb_pre* pre, sfb_pcg** out) {
    if (!op || !pre) return arg_error("mo_pcg needs an operator and a preconditioner");
    if (op->qy != pre->qy || op->qx != pre->qx) return arg_error("preconditioner shape does not match operator");
    // SFB_PRE_SPECTRAL_SUM is accepted: the exact inverse of a two-term SPD
    // operator is a valid (opt-in) MO-PCG preconditioner.
    auto* s = new sfb_pcg;
    s->op = op;
    s->pre = pre;
    s->qy = op->qy;
    s->qx = op->qx;
    s->ld = pad_ld(op->qx);
    s->ldt1 = pad_ld(op->qy);
    s->ldt2 = s->ld;
    const size_t n = (size_t)s->qy * s->ld;
    int rc = SFB_OK;
    double** bufs[] = {&s->U, &s->R, &s->Z, &s->Q0, &s->Q1, &s->W, &s->B, &s->T2};
    for (double** b : bufs)
        if (rc == SFB_OK) rc = dalloc(b, n);
    if (rc == SFB_OK) rc = dalloc(&s->T1, (size_t)s->qx * s->ldt1);
    const int nparts = 2 * std::max(std::max(vector_grid_blocks(), band_grid_blocks(s->qy, s->qx)),
                                    std::max(gemm_grid_blocks(s->qy, s->qx), seg_tiles(s->qy, s->qx)));
    if (rc == SFB_OK) rc = dalloc(&s->partials, nparts);
    if (rc == SFB_OK) rc = talloc(&s->st, sizeof(PcgState));
    if (rc == SFB_OK) rc = dalloc(&s->gw.ws, gemm_workspace_doubles());
    if (rc == SFB_OK) rc = talloc(&s->gw.flags, (size_t)gemm_max_tiles() * sizeof(unsigned));
    if (rc == SFB_OK && cudaMemset(s->gw.flags, 0, (size_t)gemm_max_tiles() * sizeof(unsigned)) != cudaSuccess)
        rc = SFB_ERR_CUDA;
    if (rc == SFB_OK && pre->kind == SFB_PRE_BANDED) {
        rc = dalloc(&s->gw.seg_f, pre->seg_doubles);
        if (rc == SFB_OK) rc = dalloc(&s->gw.seg_b, pre->seg_doubles);
    }
    if (rc == SFB_OK && pre->strassen) {
        const size_t ns = strassen_scratch_doubles(s->qy, s->qx, pre->strassen_levels);
        rc = dalloc(&s->gw.strassen, ns);
        if (rc == SFB_OK) cudaMemset(s->gw.strassen, 0, ns * 8);
    }
    if (rc == SFB_OK) {
        for (double** b : bufs) cudaMemset(*b, 0, n * 8);
        cudaMemset(s->T1, 0, (size_t)s->qx * s->ldt1 * 8);
        if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_out, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreate(&s->ev_t0) != cudaSuccess || cudaEventCreate(&s->ev_t1) != cudaSuccess) {
            set_error("creating the MO-PCG stream/events failed");
            rc = SFB_ERR_CUDA;
        }
    }
    if (rc != SFB_OK) {
        sfb_pcg_destroy(s);
        return rc;
    }
    *out = s;
    return SFB_OK;
}

int sfb_pcg_solve(sfb_pcg* s, const double* rhs, int ldr, const double* u0, int ldu0, double* U, int ldu, int rule,
                  double value, int max_iter, double* history, double* increments, double* iterates,
                  int n_iterates, sfb_pcg_result* res, void* stream) {
    SFB_NVTX("sfb_pcg_solve");
    if (!s) return arg_error("null solver");
    if (max_iter < 0) return arg_error("max_iter must be nonnegative");
    std::lock_guard<std::mutex> lock(s->mu);
    cudaStream_t cs = (cudaStream_t)stream, st = s->stream;
    const int qy = s->qy, qx = s->qx, ld = s->ld;
    // capacity for history / increments
    if (max_iter + 1 > s->cap) {
        drop_graph(s);
        cudaFree(s->hist);
        cudaFree(s->incs);
        s->hist = s->incs = nullptr;
        s->cap = std::max(max_iter + 1, 64);
        SFB_TRY(dalloc(&s->hist, s->cap));
        SFB_TRY(dalloc(&s->incs, s->cap));
    }
    if (n_iterates <= 0) iterates = nullptr;
    if (s->exec == nullptr || s->graph_iterates != iterates) SFB_TRY(build_graph(s, iterates));

    SFB_CUDA_TRY(cudaEventRecord(s->ev_in, cs));
    SFB_CUDA_TRY(cudaStreamWaitEvent(st, s->ev_in, 0));
    PcgState h;
    std::memset(&h, 0, sizeof(h));
    h.status = SFB_PCG_RUNNING;
    h.max_iter = max_iter;
    h.rule = rule;
    h.value = value;
    h.n_iterates = iterates ? n_iterates : 0;
    h.recorded = -1;
    if (max_iter == 0) h.status = SFB_PCG_MAX_ITER;
    SFB_CUDA_TRY(cudaMemcpyAsync(s->st, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    SFB_CUDA_TRY(cudaMemcpy2DAsync(s->B, (size_t)ld * 8, rhs, (size_t)ldr * 8, (size_t)qx * 8, qy,
                                   cudaMemcpyDeviceToDevice, st));
    // initial residual (solvers.py:391-397)
    if (u0 != nullptr) {
        SFB_CUDA_TRY(cudaMemcpy2DAsync(s->U, (size_t)ld * 8, u0, (size_t)ldu0 * 8, (size_t)qx * 8, qy,
                                       cudaMemcpyDeviceToDevice, st));
        SFB_TRY(op_apply_impl(s->op, s->U, ld, s->W, ld, s->T1, s->ldt1, &s->gw, st));
        SFB_TRY(launch_pcg_init_warm(s->B, ld, s->W, s->R, ld, qy, qx, s->partials, s->st, s->hist, st));
    } else {
        SFB_TRY(launch_pcg_init_plain(s->B, ld, s->R, s->U, ld, qy, qx, s->partials, s->st, s->hist, st));
    }
    if (iterates) SFB_TRY(launch_pcg_record(s->U, ld, qy, qx, iterates, s->st, st));
    if (max_iter == 0) {
        // nothing to iterate; max_iter status was preset (res0 still computed)
    }
    // Z = P^-1 R_0, rz (solvers.py:418-420)
    SFB_TRY(pre_apply_impl(s->pre, s->R, ld, s->Z, ld, s->T1, s->ldt1, s->T2, s->ldt2, s->partials, s->st, nullptr,
                           &s->gw, st));
    SFB_CUDA_TRY(cudaEventRecord(s->ev_t0, st));
    int chunks = 0;
    if (s->conditional) {
        SFB_CUDA_TRY(cudaGraphLaunch(s->exec, st));
        chunks = 1;
    } else {
        for (;;) {
            SFB_CUDA_TRY(cudaGraphLaunch(s->exec, st));
            ++chunks;
            PcgState cur;
            SFB_CUDA_TRY(cudaMemcpyAsync(&cur, s->st, sizeof(cur), cudaMemcpyDeviceToHost, st));
            SFB_CUDA_TRY(cudaStreamSynchronize(st));
            if (cur.status != SFB_PCG_RUNNING || cur.iter >= max_iter) break;
        }
    }
    // the banded iteration defers U += alpha Q into the next operator pass:
    // apply the last completed iteration's
    if (!s->op->dense) SFB_TRY(launch_pcg_ufinal(s->U, s->Q0, s->Q1, ld, qy, s->st, st));
    SFB_CUDA_TRY(cudaEventRecord(s->ev_t1, st));
    // outputs
    SFB_CUDA_TRY(cudaMemcpy2DAsync(U, (size_t)ldu * 8, s->U, (size_t)ld * 8, (size_t)qx * 8, qy,
                                   cudaMemcpyDeviceToDevice, st));
    PcgState fin;
    SFB_CUDA_TRY(cudaMemcpyAsync(&fin, s->st, sizeof(fin), cudaMemcpyDeviceToHost, st));
    SFB_CUDA_TRY(cudaStreamSynchronize(st));
    const int n = fin.iter;
    if (history) SFB_CUDA_TRY(cudaMemcpy(history, s->hist, (size_t)(n + 1) * 8, cudaMemcpyDeviceToHost));
    if (increments && n > 0) SFB_CUDA_TRY(cudaMemcpy(increments, s->incs, (size_t)n * 8, cudaMemcpyDeviceToHost));
    SFB_CUDA_TRY(cudaEventRecord(s->ev_out, st));
    SFB_CUDA_TRY(cudaStreamWaitEvent(cs, s->ev_out, 0));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s->ev_t0, s->ev_t1);
    if (res) {
        res->iterations = n;
        res->stop_reason = fin.status == SFB_PCG_RUNNING ? SFB_PCG_MAX_ITER : fin.status;
        res->bad_iter = fin.bad_iter;
        res->chunks = chunks;
        res->res0 = fin.res0;
        res->bad_value = fin.bad_value;
        res->device_ms = ms;
    }
    return SFB_OK;
}

// Device time of each pass of one MO-PCG iteration, launched `reps` times
// back to back on the solver's stream over its own buffers (after a solve):
// ms[0] banded operator pass (direction update + W = L(Q) + <W,Q>, |Q|^2 +
// the deferred U += alpha Q), ms[1] vector update pass (R, |R|), ms[2]
// preconditioner.  A scratch
// state keeps the gates open; the solver's buffers are clobbered (the next
// solve re-initialises them).
int sfb_pcg_shape(const sfb_pcg* s, int* qy, int* qx) {
    if (!s || !qy || !qx) return arg_error("null solver or output");
    *qy = s->qy;
    *qx = s->qx;
    return SFB_OK;
}

int sfb_pcg_pass_times(sfb_pcg* s, int reps, double* ms) {
    if (!s || !ms || reps <= 0) return arg_error("pass timing needs a solver, reps > 0 and 3 outputs");
    if (s->op->dense) {
        set_error("pass timing covers the banded operator");
        return SFB_ERR_UNSUPPORTED;
    }
    std::lock_guard<std::mutex> lock(s->mu);
    cudaStream_t st = s->stream;
    ScopedFree tmp(st);
    PcgState* ps;
    double *hist, *incs;
    const int cap = 2 * reps + 8;
    SFB_TRY(tmp.get(&ps, sizeof(PcgState)));
    SFB_TRY(tmp.get(&hist, (size_t)cap * 8));
    SFB_TRY(tmp.get(&incs, (size_t)cap * 8));
    PcgState h;
    std::memset(&h, 0, sizeof(h));
    h.status = SFB_PCG_RUNNING;
    h.iter = 1;
    h.max_iter = 1 << 30;
    h.rule = SFB_RULE_RESIDUAL;
    h.value = 0.0;
    h.res0 = 1.0;
    h.rz = h.rz_next = 1.0;
    h.recorded = -1;
    SFB_CUDA_TRY(cudaMemcpyAsync(ps, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    const sfb_op* op = s->op;
    BandArgs a = op_band_args(op);
    a.ld_mode = LD_PCG;
    a.X = s->Z;
    a.ldx = s->ld;
    a.Q0 = s->Q0;
    a.Q1 = s->Q1;
    a.ldq = s->ld;
    a.ep_mode = EP_PCG;
    a.W = s->W;
    a.ldw = s->ld;
    a.partials = s->partials;
    a.pcg = ps;
    a.U = s->U;
    auto band = [&]() { return launch_band(a, st); };
    auto update = [&]() {  // the banded iteration's update pass: R only (U rides in the operator pass)
        return launch_pcg_rupdate(s->R, s->W, s->ld, s->qy, s->partials, ps, hist, incs, st);
    };
    auto pre = [&]() {
        return pre_apply_impl(s->pre, s->R, s->ld, s->Z, s->ld, s->T1, s->ldt1, s->T2, s->ldt2, s->partials, ps,
                              nullptr, &s->gw, st);
    };
    std::function<int()> passes[3] = {band, update, pre};
    for (int k = 0; k < 3; ++k) {
        // reset the iteration counter so the update's history slots stay in range
        SFB_CUDA_TRY(cudaMemcpyAsync(ps, &h, sizeof(h), cudaMemcpyHostToDevice, st));
        SFB_TRY(passes[k]());  // warm
        SFB_CUDA_TRY(cudaEventRecord(s->ev_t0, st));
        for (int r = 0; r < reps; ++r) SFB_TRY(passes[k]());
        SFB_CUDA_TRY(cudaEventRecord(s->ev_t1, st));
        SFB_CUDA_TRY(cudaEventSynchronize(s->ev_t1));
        float el = 0.f;
        SFB_CUDA_TRY(cudaEventElapsedTime(&el, s->ev_t0, s->ev_t1));
        ms[k] = (double)el / reps;
    }
    PcgState after;
    SFB_CUDA_TRY(cudaMemcpyAsync(&after, ps, sizeof(after), cudaMemcpyDeviceToHost, st));
    SFB_CUDA_TRY(cudaStreamSynchronize(st));
    if (after.status != SFB_PCG_RUNNING) {
        set_error("pass timing: a gate closed during the run (status " + std::to_string(after.status) + ")");
        return SFB_ERR_CUDA;
    }
    return SFB_OK;
}

int sfb_pcg_destroy(sfb_pcg* s) {
    if (!s) return SFB_OK;
    drop_graph(s);
    double* bufs[] = {s->U, s->R, s->Z, s->Q0, s->Q1, s->W, s->B, s->T1, s->T2, s->partials, s->hist, s->incs};
    for (double* b : bufs) cudaFree(b);
    cudaFree(s->st);
    cudaFree(s->gw.ws);
    cudaFree(s->gw.flags);
    cudaFree(s->gw.seg_f);
    cudaFree(s->gw.seg_b);
    cudaFree(s->gw.strassen);
    if (s->stream) cudaStreamDestroy(s->stream);
    cudaEvent_t evs[] = {s->ev_in, s->ev_out, s->ev_t0, s->ev_t1};
    for (auto e : evs)
        if (e) cudaEventDestroy(e);
    delete s;
    return SFB_OK;
}

// ----------------------------------------------------------------- GEMM ---
int sfb_dgemm_nt(const double* A, int lda, const double* Bt, int ldb, int M, int N, int K, double* C, int ldc,
                 void* stream) {
    SFB_NVTX("sfb_dgemm_nt");
    GemmEpi e;
    e.mode = EPI_STORE;
    e.C = C;
    e.ldc = ldc;
    cudaStream_t s = (cudaStream_t)stream;
    ScopedFree tmp(s);
    GemmWs gw;
    SFB_TRY(temp_ws(tmp, gw, s));
    return launch_dgemm_nt(A, lda, Bt, ldb, M, N, K, with_ws(e, &gw), s);
}

int sfb_dgemm_nt_batch(int nb, const double* A, int lda, const double* Bt, int ldb, int M, int N, int K, double* C,
                       int ldc, long long c_stride, void* stream) {
    SFB_NVTX("sfb_dgemm_nt_batch");
    if (!A || !Bt || !C) return arg_error("batched GEMM: null argument");
    GemmEpi e;
    e.mode = EPI_STORE;
    e.C = C;
    e.ldc = ldc;
    cudaStream_t s = (cudaStream_t)stream;
    ScopedFree tmp(s);
    GemmWs gw;
    SFB_TRY(temp_ws(tmp, gw, s));
    return launch_dgemm_nt_batch(A, lda, Bt, ldb, nb, M, N, K, c_stride, with_ws(e, &gw), s);
}

int sfb_dgemm_nt_scatter(const double* A, int lda, const double* Bt, int ldb, int M, int N, int K, int nseg,
                         const int* seg_host, double* const* dst_host, const int* ldd_host, int col_off,
                         void* stream) {
    if (nseg <= 0 || nseg > kMaxScatter) return arg_error("scatter GEMM: 1..8 destinations");
    if (!seg_host || !dst_host || !ldd_host) return arg_error("scatter GEMM: null destination table");
    GemmEpi e;
    e.mode = EPI_SCATTER;
    e.nseg = nseg;
    for (int d = 0; d <= nseg; ++d) e.seg[d] = seg_host[d];
    if (e.seg[0] != 0 || e.seg[nseg] != M) return arg_error("scatter GEMM: segments must cover the M rows");
    for (int d = 0; d < nseg; ++d) {
        if (e.seg[d + 1] < e.seg[d]) return arg_error("scatter GEMM: segments must be increasing");
        if (!dst_host[d] && e.seg[d + 1] > e.seg[d]) return arg_error("scatter GEMM: null destination");
        e.dst[d] = dst_host[d];
        e.ldd_seg[d] = ldd_host[d];
    }
    e.col_off = col_off;
    cudaStream_t s = (cudaStream_t)stream;
    ScopedFree tmp(s);
    GemmWs gw;
    SFB_TRY(temp_ws(tmp, gw, s));
    return launch_dgemm_nt(A, lda, Bt, ldb, M, N, K, with_ws(e, &gw), s);
}

int sfb_copy2d(double* dst, int ldd, const double* src, int lds, int rows, int cols, void* stream) {
    if (rows <= 0 || cols <= 0) return SFB_OK;
    SFB_CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)ldd * 8, src, (size_t)lds * 8, (size_t)cols * 8, rows,
                                   cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return SFB_OK;
}

// CUDA IPC of device buffers (the sharded preconditioner's receive buffers):
// the handle names the whole allocation, so the pointer's offset inside it
// travels with the handle.
int sfb_ipc_get_handle(const void* ptr, unsigned char* handle64, unsigned long long* offset) {
    if (!ptr || !handle64 || !offset) return arg_error("ipc handle: null argument");
    using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static const RangeFn range = [] {  // thread-safe one-time lookup
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess) p = nullptr;
        return reinterpret_cast<RangeFn>(p);
    }();
    if (range == nullptr) {
        set_error("cuMemGetAddressRange entry point unavailable");
        return SFB_ERR_CUDA;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) {
        set_error("cuMemGetAddressRange failed");
        return SFB_ERR_CUDA;
    }
    cudaIpcMemHandle_t h;
    SFB_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(handle64, &h, sizeof(h));
    *offset = (unsigned long long)((CUdeviceptr)ptr - base);
    return SFB_OK;
}

int sfb_ipc_open(const unsigned char* handle64, unsigned long long offset, void** base, void** ptr) {
    if (!handle64 || !base || !ptr) return arg_error("ipc open: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    SFB_CUDA_TRY(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
    *ptr = static_cast<char*>(*base) + offset;
    return SFB_OK;
}

int sfb_ipc_close(void* base) {
    if (!base) return SFB_OK;
    SFB_CUDA_TRY(cudaIpcCloseMemHandle(base));
    return SFB_OK;
}

// ------------------------------------------------ sharded MO-PCG blocks ---

int sfb_vec_update(double* U, double* R, const double* Q, const double* W, int ld, int rows, int cols, double alpha,
                   double* rr_host, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    return reduce_call(rr_host, 1, s, [&](double* parts, RedSlots* red) {
        return launch_sh_update(U, R, Q, W, ld, rows, cols, alpha, parts, red, s);
    });
}

int sfb_vec_xpby(double* Q, int ldq, const double* Z, int ldz, int rows, int cols, double beta, int first,
                 void* stream) {
    return launch_sh_xpby(Q, ldq, Z, ldz, rows, cols, beta, first, (cudaStream_t)stream);
}

int sfb_vec_dots(const double* A, const double* B, const double* C, const double* D, int ld, int rows, int cols,
                 double* out2_host, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    return reduce_call(out2_host, 2, s, [&](double* parts, RedSlots* red) {
        return launch_sh_dots(A, B, C, D, ld, rows, cols, parts, red, s);
    });
}

// ---------------------------------- device-resident sharded MO-PCG state --
// One object per sharded solve: the PcgState, the all-reduce slots and the
// history live on the device; the host reads them once per chunk of
// iterations (sfb_shard_result), never inside the iteration.
struct sfb_shard {
    PcgState* st = nullptr;
    double* slots = nullptr;  // [8]: <W,Q>, |Q|^2, |R|^2, <Z,R>, beta (local sums, all-reduced in place)
    double* hist = nullptr;   // [max_iter + 1]
    double* incs = nullptr;   // [max(max_iter, 1)]
    double* partials = nullptr;
    unsigned* counter = nullptr;
    int max_iter = 0;
    GemmWs gw;                // stream-K workspace of the gated GEMMs; SPIKE interface scratch (grown once)
    size_t seg_doubles = 0;
};

int sfb_shard_destroy(sfb_shard* h) {
    if (!h) return SFB_OK;
    for (void* p : {(void*)h->st, (void*)h->slots, (void*)h->hist, (void*)h->incs, (void*)h->partials,
                    (void*)h->counter, (void*)h->gw.ws, (void*)h->gw.flags, (void*)h->gw.seg_f, (void*)h->gw.seg_b})
        cudaFree(p);
    delete h;
    return SFB_OK;
}

int sfb_shard_create(int max_iter, int rule, double value, sfb_shard** out) {
    if (!out || max_iter < 0) return arg_error("shard state: bad argument");
    if (rule != SFB_RULE_RESIDUAL && rule != SFB_RULE_INCREMENT && rule != SFB_RULE_BUDGET)
        return arg_error("shard state: unknown stopping rule");
    auto* h = new sfb_shard;
    h->max_iter = max_iter;
    int rc = talloc(&h->st, sizeof(PcgState));
    if (rc == SFB_OK) rc = talloc(&h->slots, 8 * sizeof(double));
    if (rc == SFB_OK) rc = talloc(&h->hist, (size_t)(max_iter + 1) * sizeof(double));
    if (rc == SFB_OK) rc = talloc(&h->incs, (size_t)std::max(max_iter, 1) * sizeof(double));
    if (rc == SFB_OK) rc = talloc(&h->partials, (size_t)2 * vector_grid_blocks() * sizeof(double));
    if (rc == SFB_OK) rc = talloc(&h->counter, 4 * sizeof(unsigned));
    if (rc == SFB_OK) rc = talloc(&h->gw.ws, gemm_workspace_doubles() * sizeof(double));
    if (rc == SFB_OK) rc = talloc(&h->gw.flags, (size_t)gemm_max_tiles() * sizeof(unsigned));
    if (rc == SFB_OK && cudaMemset(h->gw.flags, 0, (size_t)gemm_max_tiles() * sizeof(unsigned)) != cudaSuccess)
        rc = SFB_ERR_CUDA;
    if (rc == SFB_OK) {
        PcgState st{};
        st.status = SFB_PCG_RUNNING;
        st.max_iter = max_iter;
        st.rule = rule;
        st.value = value;
        st.recorded = -1;
        if (cudaMemcpy(h->st, &st, sizeof(st), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemset(h->slots, 0, 8 * sizeof(double)) != cudaSuccess ||
            cudaMemset(h->counter, 0, 4 * sizeof(unsigned)) != cudaSuccess) {
            set_error("shard state: initialisation failed");
            rc = SFB_ERR_CUDA;
        }
    }
    if (rc != SFB_OK) {
        sfb_shard_destroy(h);
        return rc;
    }
    *out = h;
    return SFB_OK;
}

double* sfb_shard_slots(sfb_shard* h) { return h ? h->slots : nullptr; }

int sfb_shard_dots(sfb_shard* h, const double* A, int lda, const double* B, int ldb, const double* C, int ldc,
                   const double* D, int ldd, int rows, int cols, int slot, void* stream) {
    if (!h || !A || !B || slot < 0 || slot + (C ? 1 : 0) > 7) return arg_error("shard dots: bad argument");
    return launch_shard_dots(A, lda, B, ldb, C, ldc, D, ldd, rows, cols, h->partials, h->counter, h->slots + slot,
                             C ? h->slots + slot + 1 : nullptr, (cudaStream_t)stream);
}

int sfb_shard_start(sfb_shard* h, void* stream) {
    if (!h) return arg_error("shard start: null state");
    return launch_shard_start(h->st, h->slots, h->hist, (cudaStream_t)stream);
}

int sfb_shard_update(sfb_shard* h, double* U, int ldu, double* R, int ldr, const double* Q, int ldq, const double* W,
                     int ldw, int rows, int cols, void* stream) {
    if (!h || !U || !R || !Q || !W) return arg_error("shard update: null argument");
    return launch_shard_update(U, ldu, R, ldr, Q, ldq, W, ldw, rows, cols, h->st, h->slots, h->partials,
                               (cudaStream_t)stream);
}

int sfb_shard_control(sfb_shard* h, void* stream) {
    if (!h) return arg_error("shard control: null state");
    return launch_shard_control(h->st, h->slots, h->hist, h->incs, (cudaStream_t)stream);
}

int sfb_shard_xpby(sfb_shard* h, double* Q, int ldq, const double* Z, int ldz, int rows, int cols, int first,
                   void* stream) {
    if (!h || !Q || !Z) return arg_error("shard xpby: null argument");
    return launch_shard_xpby(Q, ldq, Z, ldz, rows, cols, h->st, h->slots, first, (cudaStream_t)stream);
}

// The heavy kernels of a sharded iteration, gated on the shard state: once
// the solve has stopped, the iterations issued ahead by the host cost only
// their (cheap) communication, not their GEMMs / SPIKE passes / band pass.
int sfb_shard_apply(sfb_shard* h, const sfb_op* op, const double* X, int ldx, double* W, int ldw, void* stream) {
    if (!h || !op || !X || !W) return arg_error("shard apply: null argument");
    if (op->dense) return arg_error("shard apply: banded operators only");
    BandArgs a = op_band_args(op);
    a.ld_mode = LD_PLAIN;
    a.X = X;
    a.ldx = ldx;
    a.ep_mode = EP_STORE;
    a.W = W;
    a.ldw = ldw;
    a.gate = h->st;
    return launch_band_staged(a, (cudaStream_t)stream);
}

int sfb_shard_gemm(sfb_shard* h, const double* A, int lda, const double* Bt, int ldb, int M, int N, int K, double* C,
                   int ldc, void* stream) {
    if (!h || !A || !Bt || !C) return arg_error("shard GEMM: null argument");
    GemmEpi e;
    e.C = C;
    e.ldc = ldc;
    e.pcg = h->st;  // STORE epilogue: the PcgState only gates
    return launch_dgemm_nt(A, lda, Bt, ldb, M, N, K, with_ws(e, &h->gw), (cudaStream_t)stream);
}

int sfb_shard_gemm_scatter(sfb_shard* h, const double* A, int lda, const double* Bt, int ldb, int M, int N, int K,
                           int nseg, const int* seg, double* const* dst, const int* ldd, int col_off, void* stream) {
    if (!h || !A || !Bt || !seg || !dst || !ldd || nseg < 1 || nseg > kMaxScatter)
        return arg_error("shard scatter GEMM: bad argument");
    GemmEpi e;
    e.mode = EPI_SCATTER;
    e.nseg = nseg;
    for (int i = 0; i <= nseg; ++i) e.seg[i] = seg[i];
    if (e.seg[0] != 0 || e.seg[nseg] != M) return arg_error("shard scatter GEMM: segments must cover the M rows");
    for (int i = 0; i < nseg; ++i) {
        if (e.seg[i + 1] < e.seg[i]) return arg_error("shard scatter GEMM: segments must be increasing");
        if (!dst[i] && e.seg[i + 1] > e.seg[i]) return arg_error("shard scatter GEMM: null destination");
        e.dst[i] = dst[i];
        e.ldd_seg[i] = ldd[i];
    }
    e.col_off = col_off;
    e.pcg = h->st;
    return launch_dgemm_nt(A, lda, Bt, ldb, M, N, K, with_ws(e, &h->gw), (cudaStream_t)stream);
}

// ---- a constant left operand of repeated products (sharded preconditioner) ----
// The column-sharded inverse-form preconditioner multiplies by the full P_L^-1 and
// P_R^-T every iteration (C = A Bt^T with Bt a rank's rows / columns): the operand is
// prepared once -- its Strassen leaf operands and the scratch for right operands of up
// to max_n rows -- and the products run as in the single-GPU schedule (operands pass,
// one strided-batch leaf launch, assembly pass; the assembly can scatter its rows to
// peer GPUs' buffers like the GEMM's EPI_SCATTER epilogue).  Below the Strassen
// threshold it is the plain DMMA GEMM.
struct sfb_const {
    const double* A = nullptr;
    int lda = 0, M = 0, K = 0, max_n = 0;
    sfb::StrassenPlan* plan = nullptr;
    double* scratch = nullptr;
};

int sfb_const_destroy(sfb_const* c) {
    if (!c) return SFB_OK;
    free_strassen_plan(c->plan);
    cudaFree(c->scratch);
    delete c;
    return SFB_OK;
}

int sfb_const_create(const double* A, int lda, int M, int K, int max_n, sfb_const** out) {
    if (!A || !out || M <= 0 || K <= 0 || max_n <= 0) return arg_error("constant operand: bad argument");
    auto* c = new sfb_const;
    c->A = A;
    c->lda = lda;
    c->M = M;
    c->K = K;
    c->max_n = max_n;
    int levels = std::min(strassen_levels_of(M), strassen_levels_of(K));
    while (levels > 0 && strassen_leaf(max_n, levels) < 16) --levels;  // thin shards: fewer levels
    if (levels > 0) {
        int rc = build_strassen_plan(A, lda, M, K, levels, &c->plan);
        if (rc == SFB_OK) {
            const int mh = strassen_leaf(M, levels), nh = strassen_leaf(max_n, levels);
            const size_t n = (size_t)c->plan->leaves * ((size_t)nh * c->plan->ldk + (size_t)mh * pad_ld(nh));
            rc = dalloc(&c->scratch, n);
        }
        if (rc == SFB_OK && cudaDeviceSynchronize() != cudaSuccess) rc = SFB_ERR_CUDA;
        if (rc != SFB_OK) {
            sfb_const_destroy(c);
            return rc;
        }
    }
    *out = c;
    return SFB_OK;
}

int sfb_const_levels(const sfb_const* c) { return c != nullptr && c->plan != nullptr ? c->plan->levels : 0; }

int sfb_shard_gemm_const(sfb_shard* h, const sfb_const* c, const double* Bt, int ldb, int N, double* C, int ldc,
                         void* stream) {
    if (!h || !c || !Bt || !C) return arg_error("shard GEMM: null argument");
    if (c->plan == nullptr || N > c->max_n)
        return sfb_shard_gemm(h, c->A, c->lda, Bt, ldb, c->M, N, c->K, C, ldc, stream);
    return strassen_apply(c->plan, Bt, ldb, N, c->scratch, C, ldc, nullptr, 0, nullptr, h->st, nullptr, nullptr, &h->gw,
                          (cudaStream_t)stream);
}

int sfb_shard_gemm_scatter_const(sfb_shard* h, const sfb_const* c, const double* Bt, int ldb, int N, int nseg,
                                 const int* seg, double* const* dst, const int* ldd, int col_off, void* stream) {
    if (!h || !c || !Bt) return arg_error("shard scatter GEMM: null argument");
    if (c->plan == nullptr || N > c->max_n)
        return sfb_shard_gemm_scatter(h, c->A, c->lda, Bt, ldb, c->M, N, c->K, nseg, seg, dst, ldd, col_off, stream);
    if (!seg || !dst || !ldd || nseg < 1 || nseg > kMaxScatter) return arg_error("shard scatter GEMM: bad argument");
    ScatterArgs sa;
    sa.nseg = nseg;
    for (int i = 0; i <= nseg; ++i) sa.seg[i] = seg[i];
    if (sa.seg[0] != 0 || sa.seg[nseg] != c->M) return arg_error("shard scatter GEMM: segments must cover the M rows");
    for (int i = 0; i < nseg; ++i) {
        if (sa.seg[i + 1] < sa.seg[i]) return arg_error("shard scatter GEMM: segments must be increasing");
        if (!dst[i] && sa.seg[i + 1] > sa.seg[i]) return arg_error("shard scatter GEMM: null destination");
        sa.dst[i] = dst[i];
        sa.ldd[i] = ldd[i];
    }
    sa.col_off = col_off;
    return strassen_apply(c->plan, Bt, ldb, N, c->scratch, nullptr, 0, nullptr, 0, nullptr, h->st, nullptr, nullptr,
                          &h->gw, (cudaStream_t)stream, EPI_STORE, nullptr, nullptr, &sa);
}

int sfb_shard_pre_apply(sfb_shard* h, const sfb_pre* p, const double* R, int ldr, double* Z, int ldz, void* stream) {
    if (!h || !p || !R || !Z) return arg_error("shard preconditioner: null argument");
    if (p->kind != SFB_PRE_BANDED) return arg_error("shard preconditioner: banded (SPIKE) form only");
    if (!tma_aligned(R, ldr) || !tma_aligned(Z, ldz)) return arg_error("shard preconditioner: 16-byte aligned rows");
    if (h->seg_doubles < p->seg_doubles) {  // grown once, before any graph capture (first chunk runs eagerly)
        cudaFree(h->gw.seg_f);
        cudaFree(h->gw.seg_b);
        h->gw.seg_f = h->gw.seg_b = nullptr;
        h->seg_doubles = 0;
        SFB_TRY(talloc(&h->gw.seg_f, p->seg_doubles * sizeof(double)));
        SFB_TRY(talloc(&h->gw.seg_b, p->seg_doubles * sizeof(double)));
        h->seg_doubles = p->seg_doubles;
    }
    return launch_spike_pre(p->fl, p->fr, R, ldr, Z, ldz, nullptr, h->gw.seg_f, h->gw.seg_b, h->st,
                            (cudaStream_t)stream);
}

int sfb_shard_result(sfb_shard* h, sfb_pcg_result* res, double* hist_host, double* incs_host, void* stream) {
    if (!h || !res) return arg_error("shard result: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    PcgState st;
    SFB_CUDA_TRY(cudaMemcpyAsync(&st, h->st, sizeof(st), cudaMemcpyDeviceToHost, s));
    SFB_CUDA_TRY(cudaStreamSynchronize(s));
    res->iterations = st.iter;
    res->stop_reason = st.status;
    res->bad_iter = st.bad_iter;
    res->bad_value = st.bad_value;
    res->res0 = st.res0;
    res->chunks = 0;
    res->device_ms = 0.0;
    if (hist_host) SFB_CUDA_TRY(cudaMemcpy(hist_host, h->hist, (size_t)(st.iter + 1) * 8, cudaMemcpyDeviceToHost));
    if (incs_host && st.iter > 0)
        SFB_CUDA_TRY(cudaMemcpy(incs_host, h->incs, (size_t)st.iter * 8, cudaMemcpyDeviceToHost));
    return SFB_OK;
}

// ------------------------------------------------------------ reductions --
int sfb_diff_norm(const double* A, int lda, const double* B, int ldb, int rows, int cols, double* out4,
                  void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    ScopedFree tmp(s);
    double* parts;
    RedSlots* red;
    SFB_TRY(tmp.get(&parts, (size_t)4 * vector_grid_blocks() * 8));
    SFB_TRY(tmp.get(&red, sizeof(RedSlots)));
    SFB_CUDA_TRY(cudaMemsetAsync(red, 0, sizeof(RedSlots), s));
    SFB_TRY(launch_norms(A, lda, B, ldb, rows, cols, parts, red, s));
    RedSlots h;
    SFB_CUDA_TRY(cudaMemcpyAsync(&h, red, sizeof(h), cudaMemcpyDeviceToHost, s));
    SFB_CUDA_TRY(cudaStreamSynchronize(s));
    for (int i = 0; i < 4; ++i) out4[i] = h.v[i];
    return SFB_OK;
}

}  // extern "C"

// --------------------------------------------------------------- sparse ---
// ---------------------- sparse LU of a generic vector_pcg preconditioner --
struct sfb_lu {
    int n = 0, nlev_l = 0, nlev_u = 0;
    long long *Lp = nullptr, *Up = nullptr;
    int *Li = nullptr, *Ui = nullptr, *Llp = nullptr, *Llr = nullptr, *Ulp = nullptr, *Ulr = nullptr;
    int *perm_r = nullptr, *perm_c = nullptr;
    double *Lv = nullptr, *Uv = nullptr, *y = nullptr;
};

int sfb_lu_destroy(sfb_lu* h) {
    if (!h) return SFB_OK;
    for (void* p : {(void*)h->Lp, (void*)h->Up, (void*)h->Li, (void*)h->Ui, (void*)h->Llp, (void*)h->Llr,
                    (void*)h->Ulp, (void*)h->Ulr, (void*)h->perm_r, (void*)h->perm_c, (void*)h->Lv, (void*)h->Uv,
                    (void*)h->y})
        cudaFree(p);
    delete h;
    return SFB_OK;
}

namespace {
// dependency levels of a triangular CSR factor (lower: rows in increasing
// order, upper: decreasing); rows grouped by level
int tri_levels(int n, const long long* ptr, const int* ind, bool lower, std::vector<int>& lev_ptr,
               std::vector<int>& lev_rows) {
    std::vector<int> lev(n, 0);
    int nlev = 0;
    for (int k = 0; k < n; ++k) {
        const int i = lower ? k : n - 1 - k;
        int l = 0;
        for (long long p = ptr[i]; p < ptr[i + 1]; ++p) {
            const int j = ind[p];
            if (j < 0 || j >= n || (lower ? j > i : j < i)) return -1;
            if (j != i) l = std::max(l, lev[j] + 1);
        }
        lev[i] = l;
        nlev = std::max(nlev, l + 1);
    }
    lev_ptr.assign(nlev + 1, 0);
    for (int i = 0; i < n; ++i) ++lev_ptr[lev[i] + 1];
    for (int l = 0; l < nlev; ++l) lev_ptr[l + 1] += lev_ptr[l];
    lev_rows.assign(n, 0);
    std::vector<int> fill(lev_ptr.begin(), lev_ptr.end() - 1);
    for (int i = 0; i < n; ++i) lev_rows[fill[lev[i]]++] = i;
    return nlev;
}
}  // namespace

int sfb_lu_create(int n, long long nnz_l, const long long* Lp, const int* Li, const double* Lv, long long nnz_u,
                  const long long* Up, const int* Ui, const double* Uv, const int* perm_r, const int* perm_c,
                  sfb_lu** out) {
    if (n <= 0 || !Lp || !Up || !perm_r || !perm_c || !out) return arg_error("sparse LU: bad argument");
    std::vector<int> llp, llr, ulp, ulr;
    const int nl = tri_levels(n, Lp, Li, true, llp, llr), nu = tri_levels(n, Up, Ui, false, ulp, ulr);
    if (nl < 0 || nu < 0) return arg_error("sparse LU: factors are not triangular CSR");
    auto* h = new sfb_lu;
    h->n = n;
    h->nlev_l = nl;
    h->nlev_u = nu;
    int rc = SFB_OK;
    auto up = [&](auto** dst, const void* src, size_t bytes) {
        if (rc != SFB_OK) return;
        if (cudaMalloc(reinterpret_cast<void**>(dst), bytes ? bytes : 8) != cudaSuccess ||
            (src && bytes && cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)) {
            set_error("uploading the sparse LU factors failed");
            rc = SFB_ERR_NOMEM;
        }
    };
    up(&h->Lp, Lp, (size_t)(n + 1) * 8);
    up(&h->Li, Li, (size_t)nnz_l * 4);
    up(&h->Lv, Lv, (size_t)nnz_l * 8);
    up(&h->Up, Up, (size_t)(n + 1) * 8);
    up(&h->Ui, Ui, (size_t)nnz_u * 4);
    up(&h->Uv, Uv, (size_t)nnz_u * 8);
    up(&h->Llp, llp.data(), llp.size() * 4);
    up(&h->Llr, llr.data(), llr.size() * 4);
    up(&h->Ulp, ulp.data(), ulp.size() * 4);
    up(&h->Ulr, ulr.data(), ulr.size() * 4);
    up(&h->perm_r, perm_r, (size_t)n * 4);
    up(&h->perm_c, perm_c, (size_t)n * 4);
    up(&h->y, nullptr, (size_t)n * 8);
    if (rc != SFB_OK) {
        sfb_lu_destroy(h);
        return rc;
    }
    *out = h;
    return SFB_OK;
}

int sfb_lu_solve(sfb_lu* h, const double* r, double* z, void* stream) {
    if (!h || !r || !z) return arg_error("sparse LU solve: null argument");
    return launch_lu_solve(h->n, h->Lp, h->Li, h->Lv, h->Llp, h->Llr, h->nlev_l, h->Up, h->Ui, h->Uv, h->Ulp, h->Ulr,
                           h->nlev_u, h->perm_r, h->perm_c, r, z, h->y, (cudaStream_t)stream);
}

struct sfb_csr {
    int n = 0;
    long long nnz = 0;
    long long* indptr = nullptr;
    int* indices = nullptr;
    double* data = nullptr;
};

int sfb_csr_create(int n, long long nnz, const long long* indptr, const int* indices, const double* data,
                   sfb_csr** out) {
    if (n <= 0 || nnz < 0 || !indptr || (nnz > 0 && (!indices || !data)) || !out)
        return arg_error("CSR matrix needs n > 0 and its three arrays");
    auto* K = new sfb_csr;
    K->n = n;
    K->nnz = nnz;
    int rc = SFB_OK;
    auto up = [&](void** dst, const void* src, size_t bytes) {
        if (rc != SFB_OK) return;
        if (cudaMalloc(dst, bytes ? bytes : 8) != cudaSuccess ||
            (bytes && cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)) {
            set_error("uploading the CSR matrix failed");
            rc = SFB_ERR_NOMEM;
        }
    };
    up(reinterpret_cast<void**>(&K->indptr), indptr, (size_t)(n + 1) * sizeof(long long));
    up(reinterpret_cast<void**>(&K->indices), indices, (size_t)nnz * sizeof(int));
    up(reinterpret_cast<void**>(&K->data), data, (size_t)nnz * sizeof(double));
    if (rc != SFB_OK) {
        sfb_csr_destroy(K);
        return rc;
    }
    *out = K;
    return SFB_OK;
}

int sfb_csr_spmv(const sfb_csr* K, const double* x, double* y, void* stream) {
    if (!K || !x || !y) return arg_error("null CSR operand");
    return launch_csr_spmv(K->n, K->indptr, K->indices, K->data, x, y, (cudaStream_t)stream);
}

int sfb_csr_destroy(sfb_csr* K) {
    if (!K) return SFB_OK;
    cudaFree(K->indptr);
    cudaFree(K->indices);
    cudaFree(K->data);
    delete K;
    return SFB_OK;
}
