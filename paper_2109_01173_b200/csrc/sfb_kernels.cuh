// Kernel-level interfaces shared between the translation units.
#pragma once

#include <vector>

#include "sfb_common.cuh"

namespace sfb {

// ------------------------------------------------------------- GEMM -------
enum GemmEpiMode {
    EPI_STORE = 0,          // C[m][n] = acc
    EPI_STORE_T = 1,        // C[n][m] = acc
    EPI_HADAMARD_SUM = 2,   // C[m][n] = acc / (sr[m] + sc[n])      (solvers.py:245-253)
    EPI_HADAMARD_PROD = 3,  // C[m][n] = acc * sr[m] * sc[n]        (sr, sc = 1/lambda)
    EPI_STORE_DOT = 4,      // C[m][n] = acc; dot += acc * D[m][n]  (<Z,R>, solvers.py:448)
    EPI_ACCUM = 5,          // C[m][n] += acc
    EPI_SCATTER = 6         // row m of C goes to destination d (seg[d] <= m < seg[d+1]):
                            // dst[d][(m - seg[d]) * ldd[d] + col_off + n] = acc  (the
                            // transpose all-to-all of the sharded preconditioner fused
                            // into the GEMM: dst[d] are peer GPUs' buffers over NVLink)
};
constexpr int kMaxScatter = 8;

struct GemmEpi {
    int mode = EPI_STORE;
    double* C = nullptr;
    int ldc = 0;
    const double* sr = nullptr;
    const double* sc = nullptr;
    const double* D = nullptr;
    int ldd = 0;
    double* partials = nullptr;   // one per output tile (EPI_STORE_DOT)
    unsigned* counter = nullptr;  // last-block counter (EPI_STORE_DOT)
    PcgState* pcg = nullptr;      // status gate; receives rz_next
    double* dot_out = nullptr;    // receives the dot total when non-null
    double* sk_ws = nullptr;      // stream-K partial tiles (gemm_workspace_doubles())
    unsigned* sk_flags = nullptr; // stream-K per-tile counters (gemm_max_tiles(), zeroed once)
    // EPI_SCATTER destinations
    int nseg = 0;
    int seg[kMaxScatter + 1] = {};
    double* dst[kMaxScatter] = {};
    int ldd_seg[kMaxScatter] = {};
    int col_off = 0;
};

int launch_dgemm_nt(const double* A, int lda, const double* Bt, int ldb, int M, int N, int K,
                    const GemmEpi& ep, cudaStream_t stream);
// strided batch of nb products of one shape in one persistent launch (plain store)
int launch_dgemm_nt_batch(const double* A, int lda, const double* Bt, int ldb, int nb, int M, int N, int K,
                          long long c_stride, const GemmEpi& ep, cudaStream_t stream);
int gemm_batch_max(int M, int N);  // most problems of this shape per launch
int gemm_grid_blocks(int M, int N);
int gemm_smem_bytes();
size_t gemm_workspace_doubles();
int gemm_max_tiles();

// ----------------------------------------------------------- banded -------
enum BandLoad { LD_PLAIN = 0, LD_PCG = 1, LD_HEAT = 2, LD_DIB = 3 };
enum BandEpi { EP_STORE = 0, EP_PCG = 1, EP_RESID = 2 };  // EP_RESID: |B - L(X)|, |B| (no store)

struct BandArgs {
    int out_rows = 0, out_cols = 0, in_rows = 0, in_cols = 0;
    int nterms = 0, width = 1, goff = 0, hoff = 0;
    const double* gband = nullptr;  // [nterms][out_rows][width]
    const double* gskew = nullptr;  // [gskew_rows][terms * width, padded even] (band_skew)
    int gskew_rows = 0;             // out_rows + width - 1
    int gskew_terms = 0;            // band_skew_terms(nterms)
    const double* hband = nullptr;  // [nterms][out_cols][width]
    // loader
    int ld_mode = LD_PLAIN;
    const double* X = nullptr;  // plain input / Z (PCG) / U (heat, DIB)
    int ldx = 0;
    const double* X2 = nullptr;  // V (DIB) / F (heat)
    int ldx2 = 0;
    double* Q0 = nullptr;  // PCG direction double buffer
    double* Q1 = nullptr;
    int ldq = 0;
    double* U = nullptr;   // PCG: the iterate, receives the deferred U += alpha_{s-1} Q_{s-1} (ld = ldq)
    double c = 0.0;        // heat source scale / DIB tau*rho
    int rs = 0, cs = 0;    // heat: full-grid offset of the interior state
    int species = 0;
    double kp[9] = {0};    // DIB parameters
    unsigned long long* check = nullptr;  // [max|W| bits, non-finite flag]
    // epilogue
    int ep_mode = EP_STORE;
    double* W = nullptr;
    int ldw = 0;
    double* partials = nullptr;  // [2][nblocks]
    PcgState* pcg = nullptr;
    const PcgState* gate = nullptr;  // any loader: no-op unless gate->status == running (sharded MO-PCG)
    // EP_RESID (plain loader): res->v[0] = |B - W|_F, res->v[3] = |B|_F, W not stored
    const double* B = nullptr;
    int ldb = 0;
    RedSlots* res = nullptr;
};

// Every input of `a` needs 16-byte aligned rows (even leading dimension).
int launch_band(const BandArgs& a, cudaStream_t stream);
std::vector<double> band_skew(const double* gband, int nterms, int rows, int w);
int band_skew_terms(int nterms);
bool band_supported(int nterms, int width);
int band_grid_blocks(int out_rows, int out_cols);

// ----------------------------------------------------------- vector -------
int launch_pcg_init_plain(const double* rhs, int ldr, double* R, double* U, int ld, int rows, int cols,
                          double* partials, PcgState* st, double* hist, cudaStream_t s);
int launch_pcg_init_warm(const double* rhs, int ldr, const double* W, double* R, int ld, int rows,
                         int cols, double* partials, PcgState* st, double* hist, cudaStream_t s);
int launch_pcg_direction(const double* Z, double* Q0, double* Q1, int ld, int rows, int cols,
                         PcgState* st, cudaStream_t s);
int launch_pcg_dots(const double* W, const double* Q0, const double* Q1, int ld, int rows, int cols,
                    double* partials, PcgState* st, cudaStream_t s);
// use_handle: also the loop control of the conditional iteration graph
int launch_pcg_rupdate(double* R, const double* W, int ld, int rows, double* partials, PcgState* st, double* hist,
                       double* incs, cudaStream_t s, unsigned long long handle = 0, int use_handle = 0);
int launch_pcg_ufinal(double* U, const double* Q0, const double* Q1, int ld, int rows, PcgState* st,
                      cudaStream_t s);
int launch_pcg_update(double* U, double* R, const double* W, const double* Q0, const double* Q1, int ld,
                      int rows, int cols, double* partials, PcgState* st, double* hist, double* incs,
                      cudaStream_t s);
// Q0/Q1 non-null: add the deferred alpha Q of the banded iteration to the record
int launch_pcg_record(const double* U, int ld, int rows, int cols, double* iterates, PcgState* st,
                      cudaStream_t s, const double* Q0 = nullptr, const double* Q1 = nullptr);
int launch_copy_dot(const double* R, double* Z, int ld, int rows, int cols, double* partials,
                    PcgState* st, RedSlots* red, cudaStream_t s);
int launch_loop_ctl(PcgState* st, unsigned long long handle, int use_handle, cudaStream_t s);
int launch_norms(const double* A, int lda, const double* B, int ldb, int rows, int cols, double* partials,
                 RedSlots* out, cudaStream_t s);
int vector_grid_blocks();
// Row-scatter destinations of an assembled product (the sharded preconditioner's
// transpose fused into its product, as EPI_SCATTER of the GEMM): row m of C with
// seg[d] <= m < seg[d+1] goes to dst[d][(m - seg[d]) * ldd[d] + col_off + n]
struct ScatterArgs {
    int nseg = 0;
    int seg[kMaxScatter + 1] = {};
    double* dst[kMaxScatter] = {};
    int ldd[kMaxScatter] = {};
    int col_off = 0;
};

// Strassen schedule, `levels` levels flattened (vector.cu): all 7^levels leaf
// operands (rh x ch each, at S + l * sstride) of X (rows x cols, read as
// (rh 2^levels) x (ch 2^levels) with zeros past its extents; side 0: left
// operand A, side 1: right operand Bt), and the assembly of C (rows x cols)
// from the leaf products at Mp + l * mstride, with <C,D> when D is set
int launch_strassen_operands(int levels, int side, const double* X, int ldx, int rows, int cols, int rh, int ch,
                             double* S, int lds, size_t sstride, const PcgState* gate, cudaStream_t s);
int launch_strassen_assemble(int levels, const double* Mp, int ldm, size_t mstride, int rh, int ch, double* C, int ldc,
                             int rows, int cols, const double* D, int ldd, double* partials, PcgState* st,
                             double* dot_out, unsigned* counter, cudaStream_t s, int hmode = EPI_STORE,
                             const double* sr = nullptr, const double* sc = nullptr,  // hmode: EPI_HADAMARD_* scaling
                             const ScatterArgs* scatter = nullptr);  // set: rows go to the destinations, C unused
int launch_transpose(const double* src, int lds, double* dst, int ldd, int rows, int cols, cudaStream_t s);
int launch_sh_update(double* U, double* R, const double* Q, const double* W, int ld, int rows, int cols,
                     double alpha, double* partials, RedSlots* out, cudaStream_t s);
int launch_sh_xpby(double* Q, int ldq, const double* Z, int ldz, int rows, int cols, double beta, int first,
                   cudaStream_t s);
int launch_shard_dots(const double* A, int lda, const double* B, int ldb, const double* C, int ldc, const double* D,
                      int ldd, int rows, int cols, double* partials, unsigned* counter, double* out0, double* out1,
                      cudaStream_t s);
int launch_shard_update(double* U, int ldu, double* R, int ldr, const double* Q, int ldq, const double* W, int ldw,
                        int rows, int cols, PcgState* st, double* slots, double* partials, cudaStream_t s);
int launch_shard_start(PcgState* st, double* slots, double* hist, cudaStream_t s);
int launch_shard_control(PcgState* st, double* slots, double* hist, double* incs, cudaStream_t s);
int launch_shard_xpby(double* Q, int ldq, const double* Z, int ldz, int rows, int cols, const PcgState* st,
                      const double* slots, int first, cudaStream_t s);
int launch_sh_dots(const double* A, const double* B, const double* C, const double* D, int ld, int rows, int cols,
                   double* partials, RedSlots* out, cudaStream_t s);

// ------------------------------------------ banded preconditioner solves ----
// One SPD banded preconditioner factor prepared for the SPIKE solves (spike.cu).
struct SpikeFactor {
    int n = 0, b = 0;
    double* band = nullptr;  // [n + b][b + 1] segment-local Cholesky rows (1/L_ii at d = b)
    double* Hf16 = nullptr;  // [P16][16][b] sub-segment responses, forward / backward
    double* Hb16 = nullptr;
    double* Tf16 = nullptr;  // [P16][b][b] sub-segment transfers
    double* Tb16 = nullptr;
    double* V = nullptr;     // [P][64][b] spikes
    double* W = nullptr;
    double* coef = nullptr;  // [P][(2b)^2 + 2 (2b) b] interface block-LU
};
struct SegDot {
    const double* R = nullptr;
    int ldr = 0;
    double* partials = nullptr;  // one per tile
    unsigned* counter = nullptr;
    PcgState* pcg = nullptr;
    double* dot_out = nullptr;
};
int spike_length();
size_t spike_interface_doubles(int n, int b, int nlines);
int build_spike_factor(int n, int b, const double* cholesky_band_host, SpikeFactor& f);
void free_spike_factor(SpikeFactor& f);
// Z = P_L^-1 R P_R^-1 (Z may alias nothing but itself; R is read once).
// svL / svR: interface scratch of spike_interface_doubles(qy, bL, qx) and
// spike_interface_doubles(qx, bR, qy) doubles.  `dot` (nullable) receives <Z,R>.
int launch_spike_pre(const SpikeFactor& L, const SpikeFactor& R, const double* Rin, int ldr, double* Z, int ldz,
                     const SegDot* dot, double* svL, double* svR, const PcgState* gate, cudaStream_t s);

// ------------------------------------------------------------ sparse -----
int launch_lu_solve(int n, const long long* Lp, const int* Li, const double* Lv, const int* Llp, const int* Llr,
                    int nlL, const long long* Up, const int* Ui, const double* Uv, const int* Ulp, const int* Ulr,
                    int nlU, const int* perm_r, const int* perm_c, const double* r, double* z, double* y,
                    cudaStream_t s);
int launch_csr_spmv(int n, const long long* indptr, const int* indices, const double* data, const double* x,
                    double* y, cudaStream_t s);

}  // namespace sfb
