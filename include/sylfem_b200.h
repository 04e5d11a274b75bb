/*
 * sylfem_b200.h — C ABI of the B200-native MO-FEM solve path.
 *
 * The reference (`sylfem`, a pure-Python package) has no FFI: its plugin
 * boundary is the Python API.  These entry points are what a ctypes/cffi
 * binding of that API binds; each cites the reference
 * function it replaces (paths relative to /root/reference/pkg/src/sylfem/).
 *
 * Conventions
 *  - Grid matrices are q_y x q_x, row-major (rows follow y, columns follow x,
 *    operators.py:1-9) with an explicit leading dimension `ld*`.
 *  - Pointers named *_dev are device pointers; *_host are host pointers.
 *  - `stream` is a cudaStream_t (may be NULL = legacy default stream).  Calls
 *    order themselves after prior work on `stream`, and work they leave
 *    pending is ordered before later work on `stream`.
 *  - Every function returns SFB_OK (0) or a negative status; the message is
 *    available from sfb_last_error() (thread-local).  The Python shim maps
 *    statuses to the reference exception classes and messages.
 *  - Band storage: a left factor G (q_y x q_y) is stored as gband[i][d] =
 *    G[i][i + goff + d], d = 0..gw-1; a right factor H (acting as U H) is
 *    stored by columns: hband[j][e] = H[j + hoff + e][j], e = 0..hw-1.
 *    Multi-term operators store all terms back to back ([nterms][rows][w]).
 */
#ifndef SYLFEM_B200_H
#define SYLFEM_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to sylfem exceptions by the Python shim) ---- */
enum {
    SFB_OK = 0,
    SFB_ERR_ARG = -1,          /* bad argument / shape      -> OperatorError  */
    SFB_ERR_CUDA = -2,         /* CUDA runtime failure      -> SolverError    */
    SFB_ERR_NOMEM = -3,        /* device allocation failed  -> SolverError    */
    SFB_ERR_UNSUPPORTED = -4   /* band width / term count beyond the kernels  */
};

/* MO-PCG stop reasons (solvers.py:415-453) */
enum {
    SFB_PCG_RUNNING = 0,
    SFB_PCG_TOLERANCE = 1,     /* "tolerance"                                 */
    SFB_PCG_INCREMENT = 2,     /* "increment"                                 */
    SFB_PCG_INDEFINITE = 3,    /* <L(Q),Q> <= 0   -> OperatorError            */
    SFB_PCG_NONFINITE = 4,     /* residual not finite -> SolverError          */
    SFB_PCG_MAX_ITER = 5       /* "max_iter" (report, not an error)           */
};

/* stopping rule kinds (solvers.py:53-83).  SFB_RULE_BUDGET has no reference
 * counterpart: no tolerance test, every solve runs exactly max_iter
 * iterations and ends with SFB_PCG_MAX_ITER, which the IMEX loops then treat
 * as a completed step rather than "did not converge" (fixed-work
 * benchmarking, SURVEY §8 d). */
enum { SFB_RULE_RESIDUAL = 0, SFB_RULE_INCREMENT = 1, SFB_RULE_BUDGET = 2 };

/* preconditioner / spectral sandwich kinds (solvers.py:103-150, 211-300) */
enum {
    SFB_PRE_IDENTITY = 0,      /* Z = R (copy)                                */
    SFB_PRE_INVERSE = 1,       /* Z = Linv R RinvT^T    (2 DMMA GEMMs)        */
    SFB_PRE_SPECTRAL_PROD = 2, /* Z = VL [(VL^T R VR) / (lamL_i lamR_j)] VR^T */
    SFB_PRE_SPECTRAL_SUM = 3,  /* Z = VL [(VL^T R VR) / (lamL_i + lamR_j)] VR^T (reduced solve) */
    SFB_PRE_BANDED = 4         /* Z = PL^-1 R PR^-1 by banded Cholesky sweeps */
};

/* IMEX run outcomes (timestepping.py:62-69, 86-112) */
enum {
    SFB_IMEX_OK = 0,
    SFB_IMEX_BLOWUP = 1,        /* non-finite or > 1e100 state   -> BlowUpError(step, species, state) */
    SFB_IMEX_NOT_CONVERGED = 2, /* inner MO-PCG hit max_iter     -> SolverError "did not converge"   */
    SFB_IMEX_INDEFINITE = 3,    /* inner MO-PCG: <L(Q),Q> <= 0   -> OperatorError                    */
    SFB_IMEX_NONFINITE = 4      /* inner MO-PCG residual non-finite -> SolverError                   */
};

typedef struct sfb_op sfb_op;
typedef struct sfb_map sfb_map;
typedef struct sfb_pre sfb_pre;
typedef struct sfb_pcg sfb_pcg;
typedef struct sfb_csr sfb_csr;
typedef struct sfb_reduced sfb_reduced;

typedef struct {
    int iterations;       /* completed iterations                        */
    int stop_reason;      /* SFB_PCG_*                                   */
    int bad_iter;         /* iteration of INDEFINITE / NONFINITE         */
    int chunks;           /* graph launches used                         */
    double res0;          /* |R_0|                                       */
    double bad_value;     /* <L(Q),Q> at INDEFINITE                      */
    double device_ms;     /* device time of the iteration loop           */
} sfb_pcg_result;

typedef struct {
    int steps_done;       /* completed time steps                        */
    int fail_step;        /* step of the failure (-1: none)              */
    int fail_kind;        /* SFB_IMEX_*                                  */
    int fail_species;     /* 0 = u (eta), 1 = v (theta); -1: none        */
    int steady_step;      /* first steady step of the run (-1: none)     */
    int pcg_bad_iter;     /* inner MO-PCG iteration of an INDEFINITE / NONFINITE failure */
    double pcg_bad_value; /* <L(Q),Q> of an INDEFINITE failure           */
} sfb_imex_result;

/* ---- library ---------------------------------------------------------- */
int sfb_version(void);
const char* sfb_last_error(void);
/* Select the device and warm the driver entry points; reports SM count. */
int sfb_init(int device, int* sm_count);

/* ---- operator: SylvesterOperator (operators.py:97-138) ----------------- */
/* Banded term list W = sum_t G_t U H_t.  Bands are uploaded once. */
int sfb_op_create(int qy, int qx, int nterms,
                  int gw, int goff, const double* gband_host,
                  int hw, int hoff, const double* hband_host, sfb_op** out);
/* Halo-extended column block of a banded operator (column-sharded MO-PCG,
 * SURVEY §8 e): out_cols local output columns computed from in_cols input
 * columns (the local block plus the neighbours' halo). */
int sfb_op_create_block(int qy, int out_cols, int in_cols, int nterms, int w, int goff,
                        const double* gband_host, int hoff, const double* hband_host,
                        sfb_op** out);
/* Dense term list (factors too wide for the banded kernels). */
int sfb_op_create_dense(int qy, int qx, int nterms, const double* G_host,
                        const double* H_host, sfb_op** out);
/* W = op(U)  (SylvesterOperator.apply, operators.py:124-131). */
int sfb_op_apply(const sfb_op* op, const double* U_dev, int ldu,
                 double* W_dev, int ldw, void* stream);
/* out2_host = { |op(U) - rhs|_F, |rhs|_F }  (solvers.py:293-294). */
int sfb_op_residual(const sfb_op* op, const double* U_dev, int ldu,
                    const double* rhs_dev, int ldr, double* out2_host, void* stream);
int sfb_op_destroy(sfb_op* op);

/* ---- rectangular banded map: the rhs builders (operators.py:206-207,
 *      228-232, 266-268, 281-282) --------------------------------------- */
int sfb_map_create(int out_rows, int out_cols, int in_rows, int in_cols,
                   int gw, int goff, const double* gband_host,
                   int hw, int hoff, const double* hband_host, sfb_map** out);
/* out = G F H^T over the full node grid F. */
int sfb_map_apply(const sfb_map* m, const double* F_dev, int ldf,
                  double* out_dev, int ldo, void* stream);
/* IMEX heat rhs (timestepping.py:150-153): W = expand(U) + c F, checked for
 * blow-up, then out = G W H^T.  U is the interior state placed at full-grid
 * offset (row_shift, col_shift); F may be NULL.  check2_host (nullable) =
 * { max|W|, number of non-finite entries }. */
int sfb_map_apply_heat(const sfb_map* m, const double* U_dev, int ldu,
                       int row_shift, int col_shift, double c,
                       const double* F_dev, int ldf, double* out_dev, int ldo,
                       double* check2_host, void* stream);
/* IMEX DIB rhs (timestepping.py:201-207, models.py:74-82): species 0 uses
 * W = U + tau_rho f(U,V), species 1 W = V + tau_rho g(U,V); then
 * out = G W H^T.  params = {alpha, gamma_k, A1, A2, B, C, D, k2, k3}.
 * The map may read a halo-extended column block (in_cols > out_cols, same
 * rows): the column-sharded IMEX driver's local rhs. */
int sfb_map_apply_dib(const sfb_map* m, const double* U_dev, const double* V_dev,
                      int ld, int species, double tau_rho, const double* params_host,
                      double* out_dev, int ldo, double* check2_host, void* stream);
int sfb_map_destroy(sfb_map* m);

/* ---- preconditioner / spectral sandwich (solvers.py:103-150, 284-300) -- */
/* kind SFB_PRE_INVERSE: L = P_L^-1 (q_y x q_y), R = (P_R^-1)^T (q_x x q_x).
 * kind SFB_PRE_SPECTRAL_*: L = V_L, R = V_R, lamL/lamR eigenvalues.
 * kind SFB_PRE_BANDED: L/R = banded Cholesky factors, see sfb_pre_create_banded.
 * L/R are row-major and copied once; they may live in host or device memory
 * (a device-resident eigendecomposition is not staged through the host).
 * lamL/lamR are host arrays. */
int sfb_pre_create(int qy, int qx, int kind, const double* L,
                   const double* R, const double* lamL_host,
                   const double* lamR_host, sfb_pre** out);
/* The inverse-form products Z = P_L^-1 (R P_R^-1) of shapes with q_y, q_x >=
 * min_q run as up to three levels of Strassen around the DMMA GEMM (odd
 * shapes are padded with zeros inside the passes): one pass forms the 7^L leaf operands of
 * the variable factor (those of the constant factors are formed at creation),
 * one strided-batch DMMA launch does the 7^L leaf products, one pass
 * assembles Z (and <Z,R>).  Same value as the two dense solves of
 * Preconditioner.apply_inverse (solvers.py:134-143), other summation order.
 * Applies to preconditioners created afterwards; 0 = never (default:
 * SYLFEM_B200_STRASSEN_MINQ or 2000).  Returns the previous threshold. */
int sfb_set_strassen_min_q(int min_q);
/* Most Strassen levels taken (0..3, default SYLFEM_B200_STRASSEN_LEVELS or 3);
 * the leaves must be at least min_q / 4 (not below 16).
 * Returns the previous value. */
int sfb_set_strassen_levels(int levels);
/* Strassen levels this preconditioner's products use (0: classic GEMMs). */
int sfb_pre_uses_strassen(const sfb_pre* p);
/* Banded SPD factors: lower Cholesky factors in band storage
 * lband[i][d] = C_L[i][i - bw + d] (d = 0..bw), same for the right factor. */
int sfb_pre_create_banded(int qy, int qx, int bwL, const double* lband_host,
                          int bwR, const double* rband_host, sfb_pre** out);
/* Z = P^-1 R  (Preconditioner.apply_inverse, solvers.py:134-143), or the
 * reduced-solve sandwich (solvers.py:292) for SFB_PRE_SPECTRAL_SUM. */
int sfb_pre_apply(const sfb_pre* p, const double* R_dev, int ldr,
                  double* Z_dev, int ldz, void* stream);
/* Y = V_L^T X V_R for the spectral kinds (the forward spectral transform;
 * used by the closed-form residual, solvers.py:345-348). */
/* The reduced solve of a two-term operator (solvers.py:284-300) as one
 * object: the spectral-sum sandwich of `pre` (SFB_PRE_SPECTRAL_SUM) and the
 * residual |L(U) - B| through `op`, captured once into a CUDA graph with
 * persistent buffers.  solve: U = sandwich(B); res2_host (may be NULL) <-
 * { |L(U) - B|_F, |B|_F } (solvers.py:293-294).  Thread-safe per object. */
int sfb_reduced_create(const sfb_pre* pre, const sfb_op* op, sfb_reduced** out);
int sfb_reduced_solve(sfb_reduced* r, const double* B_dev, int ldb, double* U_dev, int ldu,
                      double* res2_host, void* stream);
int sfb_reduced_destroy(sfb_reduced* r);
int sfb_pre_transform(const sfb_pre* p, const double* X_dev, int ldx, double* Y_dev, int ldy, void* stream);
int sfb_pre_destroy(sfb_pre* p);

/* ---- MO-PCG (solvers.py:365-453) --------------------------------------- */
int sfb_pcg_create(const sfb_op* op, const sfb_pre* pre, sfb_pcg** out);
/* Runs the full device-resident loop.  u0_dev may be NULL (U0 = 0).
 * history_host holds max_iter+1 doubles (|R_s|), increments_host max_iter
 * (|alpha| |Q|).  iterates_dev (nullable) receives up to n_iterates
 * contiguous q_y x q_x copies of U_0, U_1, ... (record_iterates). */
int sfb_pcg_solve(sfb_pcg* s, const double* rhs_dev, int ldr,
                  const double* u0_dev, int ldu0, double* U_dev, int ldu,
                  int rule, double value, int max_iter,
                  double* history_host, double* increments_host,
                  double* iterates_dev, int n_iterates,
                  sfb_pcg_result* res, void* stream);
/* Device time (ms per launch, averaged over `reps` back-to-back launches)
 * of the passes of one MO-PCG iteration on the solver's buffers, for the
 * roofline report: ms[0] banded operator pass (direction update, W = L(Q),
 * <W,Q>, |Q|^2 and the previous iteration's deferred U += alpha Q),
 * ms[1] vector update pass (R -= alpha W, |R|, stop test),
 * ms[2] preconditioner.  Call after a solve; clobbers the solver buffers.
 * Measurement only: no reference counterpart. */
int sfb_pcg_pass_times(sfb_pcg* s, int reps, double* ms);
int sfb_pcg_destroy(sfb_pcg* s);
/* grid shape (q_y, q_x) the solver was created for */
int sfb_pcg_shape(const sfb_pcg* s, int* qy, int* qx);

/* ---- IMEX-Euler step loops (timestepping.py:126-159, 162-220) --------- */
/* Heat: per step k, W = expand(U) + c_host[k] F (F may be NULL: no source;
 * row/col shifts place the interior state in the full node grid as in
 * sfb_map_apply_heat), rhs = G W H^T, blow-up check of W, MO-PCG on
 * `solver` warm started from U (rule/value/max_iter per step), increment
 * |U_new - U| and finiteness of U_new; then U = U_new.  c_host[k] = tau *
 * s(k tau) for a separable source s(t) F.  U_dev (ldu) holds u0 on entry and
 * the final state on exit — or, when res->fail_kind != SFB_IMEX_OK, the
 * state at the start of the failing step.  iterations_host / increments_host
 * receive n_steps entries (the completed ones are valid). */
int sfb_imex_heat_run(sfb_pcg* solver, const sfb_map* rhs_map, int row_shift, int col_shift,
                      const double* F_dev, int ldf, const double* c_host, int n_steps,
                      int rule, double value, int max_iter, double* U_dev, int ldu,
                      int* iterations_host, double* increments_host, sfb_imex_result* res,
                      void* stream);
/* Two-species reaction-diffusion (DIB kinetics, params as in
 * sfb_map_apply_dib): per step both rhs from the state at the start of the
 * step, species u solved on solver_u then species v on solver_v (checks in
 * the reference's order), increments and the steady test |dU|,|dV| <=
 * steady_eps |U_new|.  U_dev, V_dev (ld) in: state0, out: final state (or
 * the state at the start of the failing step).  iterations_host and
 * increments_host are n_steps x 2 (row-major: u, v). */
int sfb_imex_rds_run(sfb_pcg* solver_u, sfb_pcg* solver_v, const sfb_map* rhs_map,
                     const double* params_host, double tau_rho, int n_steps,
                     int rule, double value, int max_iter, double steady_eps,
                     double* U_dev, double* V_dev, int ld,
                     int* iterations_host, double* increments_host, sfb_imex_result* res,
                     void* stream);

/* ---- FP64 tensor-core GEMM (the kernel behind every spectral / inverse
 *      application): C = A Bt^T, A (M x K) and Bt (N x K) row-major with even
 *      leading dimensions and 16-byte aligned rows (TMA requirement). ------ */
int sfb_dgemm_nt(const double* A_dev, int lda, const double* Bt_dev, int ldb,
                 int M, int N, int K, double* C_dev, int ldc, void* stream);

/* A strided batch of nb independent products of one shape in one persistent
 * launch (128 x 128 tiles, one wave schedule and stream-K tail for the whole
 * batch; rank-3 tensor maps): C_b = A_b Bt_b^T with A_b = A_dev + b * M * lda,
 * Bt_b = Bt_dev + b * N * ldb, C_b = C_dev + b * c_stride -- the leaf products
 * of the Strassen schedule of the inverse-form preconditioner
 * (solvers.py:134-143).  nb * ceil(M/128) * ceil(N/128) <= 65536. */
int sfb_dgemm_nt_batch(int nb, const double* A_dev, int lda, const double* Bt_dev, int ldb,
                       int M, int N, int K, double* C_dev, int ldc, long long c_stride,
                       void* stream);

/* ---- host-synchronous blocks of the column-sharded MO-PCG (one rank's
 *      columns; the collectives run between these calls) --------------- */
/* U += alpha Q; R -= alpha W; *rr_host = local sum R^2 (solvers.py:432-434). */
/* C = A Bt^T with row m of C sent to destination d, seg[d] <= m < seg[d+1]
 * (seg_host: nseg + 1 increasing row offsets from 0 to M, nseg <= 8):
 * dst[d][(m - seg[d]) * ldd[d] + col_off + n] = C[m][n].  The destinations
 * may be peer GPUs' buffers (CUDA IPC, NVLink stores): the column-sharded
 * preconditioner's second transpose all-to-all fused into its GEMM. */
int sfb_dgemm_nt_scatter(const double* A_dev, int lda, const double* Bt_dev, int ldb,
                         int M, int N, int K, int nseg, const int* seg_host,
                         double* const* dst_dev_host, const int* ldd_host, int col_off,
                         void* stream);
/* dst (ldd) <- src (lds), rows x cols doubles; either side may be a peer GPU's
 * buffer (the first transpose of the sharded preconditioner as P2P copies). */
int sfb_copy2d(double* dst_dev, int ldd, const double* src_dev, int lds, int rows, int cols,
               void* stream);
/* CUDA IPC of a device buffer: a 64-byte handle of its allocation plus the
 * buffer's offset inside it; open returns the mapped allocation base (for
 * close) and the buffer pointer. */
int sfb_ipc_get_handle(const void* ptr_dev, unsigned char* handle64_host,
                       unsigned long long* offset_host);
int sfb_ipc_open(const unsigned char* handle64_host, unsigned long long offset,
                 void** base_dev, void** ptr_dev);
int sfb_ipc_close(void* base_dev);

int sfb_vec_update(double* U_dev, double* R_dev, const double* Q_dev, const double* W_dev,
                   int ld, int rows, int cols, double alpha, double* rr_host, void* stream);
/* Q = Z + beta Q (first != 0: Q = Z) (solvers.py:419, 451-452). */
int sfb_vec_xpby(double* Q_dev, int ldq, const double* Z_dev, int ldz, int rows, int cols,
                 double beta, int first, void* stream);
/* out2_host = { <A,B>, <C,D> } (C, D may be NULL) over the local block. */
int sfb_vec_dots(const double* A_dev, const double* B_dev, const double* C_dev,
                 const double* D_dev, int ld, int rows, int cols, double* out2_host,
                 void* stream);

/* ---- device-resident sharded MO-PCG (distributed.py; reference solvers.py:
 * 389-452 split over column shards).  The scalars live on the device: the
 * communicator all-reduces the slot array in place (NCCL on the stream) and
 * the host reads the state once per chunk of iterations with
 * sfb_shard_result.  slots: [0] <W,Q>, [1] |Q|^2, [2] |R|^2, [3] <Z,R>,
 * [4] beta.  Kernels that change the iterate are gated on the status, so
 * iterations issued after the stop are no-ops. */
typedef struct sfb_shard sfb_shard;
int sfb_shard_create(int max_iter, int rule, double value, sfb_shard** out);
int sfb_shard_destroy(sfb_shard* h);
double* sfb_shard_slots(sfb_shard* h);
/* slots[slot] = <A,B>, slots[slot+1] = <C,D> (C, D may be NULL) over the local block */
int sfb_shard_dots(sfb_shard* h, const double* A_dev, int lda, const double* B_dev, int ldb,
                   const double* C_dev, int ldc, const double* D_dev, int ldd, int rows, int cols,
                   int slot, void* stream);
/* after the all-reduce of slots[2..3] = {|R_0|^2, <Z_0,R_0>}: res0, history[0], rz */
int sfb_shard_start(sfb_shard* h, void* stream);
/* alpha = rz / slots[0] (INDEFINITE when <= 0), U += alpha Q, R -= alpha W, slots[2] = local |R|^2 */
int sfb_shard_update(sfb_shard* h, double* U_dev, int ldu, double* R_dev, int ldr, const double* Q_dev,
                     int ldq, const double* W_dev, int ldw, int rows, int cols, void* stream);
/* after the all-reduce of slots[2..3]: history, increment, stop test, beta = slots[4] */
int sfb_shard_control(sfb_shard* h, void* stream);
/* Q = Z + beta Q (first: Q = Z), gated on the status */
int sfb_shard_xpby(sfb_shard* h, double* Q_dev, int ldq, const double* Z_dev, int ldz, int rows,
                   int cols, int first, void* stream);
/* the heavy kernels of a sharded iteration, gated on the shard state (no-ops once the
 * solve has stopped): the banded block operator W = L(X), a DMMA GEMM C = A Bt^T (store),
 * the scatter GEMM of the peer transposes, the SPIKE preconditioner on a shard */
int sfb_shard_apply(sfb_shard* h, const sfb_op* op, const double* X_dev, int ldx, double* W_dev,
                    int ldw, void* stream);
int sfb_shard_gemm(sfb_shard* h, const double* A_dev, int lda, const double* Bt_dev, int ldb, int M,
                   int N, int K, double* C_dev, int ldc, void* stream);
int sfb_shard_gemm_scatter(sfb_shard* h, const double* A_dev, int lda, const double* Bt_dev, int ldb,
                           int M, int N, int K, int nseg, const int* seg_host,
                           double* const* dst_host, const int* ldd_host, int col_off, void* stream);
/* A constant left operand A (M x K) of repeated products C = A Bt^T, Bt of up
 * to max_n rows -- the full P_L^-1 / P_R^-T of the column-sharded inverse-form
 * preconditioner (solvers.py:134-143 on shards): prepared once (Strassen leaf
 * operands and scratch when M, K reach the threshold of sfb_set_strassen_min_q;
 * sfb_const_levels reports the levels, 0 = plain DMMA GEMM); the products are
 * gated on the shard state like sfb_shard_gemm / sfb_shard_gemm_scatter.  A
 * must outlive the handle. */
typedef struct sfb_const sfb_const;
int sfb_const_create(const double* A_dev, int lda, int M, int K, int max_n, sfb_const** out);
int sfb_const_levels(const sfb_const* c);
int sfb_const_destroy(sfb_const* c);
int sfb_shard_gemm_const(sfb_shard* h, const sfb_const* c, const double* Bt_dev, int ldb, int N,
                         double* C_dev, int ldc, void* stream);
int sfb_shard_gemm_scatter_const(sfb_shard* h, const sfb_const* c, const double* Bt_dev, int ldb, int N,
                                 int nseg, const int* seg_host, double* const* dst_dev_host,
                                 const int* ldd_host, int col_off, void* stream);
int sfb_shard_pre_apply(sfb_shard* h, const sfb_pre* p, const double* R_dev, int ldr, double* Z_dev,
                        int ldz, void* stream);
/* status, iterations, bad value / iteration; history (iterations + 1) and increments (iterations) */
int sfb_shard_result(sfb_shard* h, sfb_pcg_result* res, double* hist_host, double* incs_host,
                     void* stream);

/* ---- reductions for the IMEX drivers (timestepping.py:89-91, 155, 210-215) */
/* out4_host = { |A - B|_F (B may be NULL), max|A|, #non-finite(A), |A|_F }. */
int sfb_diff_norm(const double* A_dev, int lda, const double* B_dev, int ldb,
                  int rows, int cols, double* out4_host, void* stream);

/* ---- spectral setup (solvers.py:256-281 build_spectral_cache) --------- */
/* Generalized SPD eigendecomposition A v = lam B v (scipy.linalg.eigh(A, B)
 * of the reference, LAPACK dsygvd) on the device: cuSOLVER potrf + syevd,
 * cuBLAS trsm; eigenvalues ascending into lam_host (q), B-orthonormal
 * eigenvectors as the columns of V_dev (q x q row-major, ldv), each
 * column's largest-magnitude entry positive (solvers.py:203-208).  A and B
 * (symmetric) may be host or device memory.  SFB_ERR_ARG when B is not
 * positive definite (the caller then tries the other term order). */
int sfb_geigh(int q, const double* A, int lda, const double* B, int ldb,
              double* lam_host, double* V_dev, int ldv, void* stream);

/* ---- trajectory frames (harness.py:475-491 write_pgm) --- */
/* out_dev (rows x cols, contiguous) <- the 16-bit big-endian PGM pixels of
 * A: min-max normalised per frame, rint((a - lo) / span * 65535), zeros for
 * a frame constant up to roundoff; lohi_host (may be NULL) <- {min, max}. */
int sfb_frame_pgm16(const double* A_dev, int lda, int rows, int cols,
                    unsigned short* out_dev, double* lohi_host, void* stream);

/* ---- sparse vec-form matrices for the Kronecker cross-check path
 *      (operators.py:141-155 to_kronecker; vector_pcg, solvers.py:456-517) */
/* ---- vector_pcg with a generic sparse preconditioner (solvers.py:473:
 * spla.splu(P).solve): P factored once on the host as Pr P Pc = L U
 * (CSR, 0-based; L unit or not, U upper), solved on the device level by
 * level in one CTA.  z = P^-1 r for device vectors of length n. */
typedef struct sfb_lu sfb_lu;
int sfb_lu_create(int n, long long nnz_l, const long long* Lp, const int* Li, const double* Lv,
                  long long nnz_u, const long long* Up, const int* Ui, const double* Uv,
                  const int* perm_r, const int* perm_c, sfb_lu** out);
int sfb_lu_solve(sfb_lu* h, const double* r_dev, double* z_dev, void* stream);
int sfb_lu_destroy(sfb_lu* h);

/* K (n x n) in CSR from host arrays: indptr n+1 (int64), indices nnz (int32,
 * column indices), data nnz (fp64); copied once. */
int sfb_csr_create(int n, long long nnz, const long long* indptr_host, const int* indices_host,
                   const double* data_host, sfb_csr** out);
/* y = K x (`w = K @ q`, solvers.py:486); deterministic sum order. */
int sfb_csr_spmv(const sfb_csr* K, const double* x_dev, double* y_dev, void* stream);
int sfb_csr_destroy(sfb_csr* K);

#ifdef __cplusplus
}
#endif
#endif /* SYLFEM_B200_H */
