// IMEX-Euler step loops as native entry points (SURVEY §8 b, "imex_heat_run"
// and "imex_rds_run"): the whole time loop of imex_euler_heat
// (timestepping.py:126-159) and imex_euler_rds (timestepping.py:162-220) runs
// here, layered on the library's own entry points — the fused rhs map (with
// the explicit source / DIB kinetics and the blow-up check), the device
// MO-PCG (one graph launch per solve, warm started from the previous state)
// and the increment / finiteness norms.  States stay on the device between
// steps; the only host traffic per step is the handful of scalars the
// reference's control flow needs (blow-up flags, iteration counts, norms).
//
// Failure semantics follow the reference's order of checks (rhs of u, solve
// of u, rhs of v, solve of v): the run stops at the first failure, reports
// (step, kind, species) in sfb_imex_result, and leaves the state buffers at
// the last finite state (the state at the start of the failing step), which
// is what BlowUpError carries (timestepping.py:62-69, 86-91).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "sfb_common.cuh"

namespace {

constexpr double kBlowupLimit = 1e100;  // timestepping.py BLOWUP_LIMIT

// Step scratch (rhs and the next states) from the stream-ordered pool: a
// run of one step (the benchmark's per-step calls) costs no cudaMalloc /
// cudaFree synchronisation, and the pool keeps the blocks for the next run.
struct DevBuf {
    double* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

int alloc_grid(DevBuf& b, int rows, int ld, cudaStream_t s) {
    b.s = s;
    if (cudaMallocAsync(reinterpret_cast<void**>(&b.p), (size_t)rows * ld * 8, s) != cudaSuccess) {
        b.p = nullptr;
        sfb::set_error("imex run: device allocation failed");
        return SFB_ERR_NOMEM;
    }
    if (cudaMemsetAsync(b.p, 0, (size_t)rows * ld * 8, s) != cudaSuccess) return SFB_ERR_CUDA;
    return SFB_OK;
}

inline bool bad_check(const double* chk) { return chk[1] > 0.0 || chk[0] > kBlowupLimit; }

void init_result(sfb_imex_result* r) {
    std::memset(r, 0, sizeof(*r));
    r->fail_step = -1;
    r->fail_kind = SFB_IMEX_OK;
    r->fail_species = -1;
    r->steady_step = -1;
}

// one implicit solve; maps the MO-PCG outcome onto the IMEX failure kinds
// (max_iter -> "inner PCG did not converge", timestepping.py:106-112)
int solve_step(sfb_pcg* s, const double* rhs, const double* warm, double* out, int ld, int rule, double value,
               int max_iter, int* iters, int* kind, sfb_imex_result* r, cudaStream_t st) {
    sfb_pcg_result pr;
    SFB_TRY(sfb_pcg_solve(s, rhs, ld, warm, ld, out, ld, rule, value, max_iter, nullptr, nullptr, nullptr, 0, &pr,
                          st));
    *iters = pr.iterations;
    *kind = SFB_IMEX_OK;
    if (pr.stop_reason == SFB_PCG_MAX_ITER && rule != SFB_RULE_BUDGET) *kind = SFB_IMEX_NOT_CONVERGED;
    else if (pr.stop_reason == SFB_PCG_INDEFINITE) *kind = SFB_IMEX_INDEFINITE;
    else if (pr.stop_reason == SFB_PCG_NONFINITE) *kind = SFB_IMEX_NONFINITE;
    if (*kind != SFB_IMEX_OK) {
        r->pcg_bad_iter = pr.bad_iter;
        r->pcg_bad_value = pr.bad_value;
    }
    return SFB_OK;
}

}  // namespace

extern "C" {

int sfb_imex_heat_run(sfb_pcg* solver, const sfb_map* rhs_map, int row_shift, int col_shift, const double* F,
                      int ldf, const double* c_host, int n_steps, int rule, double value, int max_iter, double* U,
                      int ldu, int* iterations_host, double* increments_host, sfb_imex_result* res, void* stream) {
    SFB_NVTX("sfb_imex_heat_run");
    if (!solver || !rhs_map || !U || !res) return sfb::arg_error("imex heat run: null argument");
    if (n_steps < 0 || max_iter < 0) return sfb::arg_error("imex heat run: negative step or iteration count");
    init_result(res);
    cudaStream_t st = (cudaStream_t)stream;
    int qy = 0, qx = 0;
    SFB_TRY(sfb_pcg_shape(solver, &qy, &qx));
    DevBuf rhs, Un;
    SFB_TRY(alloc_grid(rhs, qy, ldu, st));
    SFB_TRY(alloc_grid(Un, qy, ldu, st));
    for (int k = 0; k < n_steps; ++k) {
        // W = expand(U) + c_k F, rhs = G W H^T, blow-up check of W (timestepping.py:148-153)
        double chk[2] = {0.0, 0.0};
        SFB_TRY(sfb_map_apply_heat(rhs_map, U, ldu, row_shift, col_shift, c_host ? c_host[k] : 0.0, F, ldf, rhs.p,
                                   ldu, chk, st));
        if (bad_check(chk)) {
            res->fail_step = k;
            res->fail_kind = SFB_IMEX_BLOWUP;
            res->fail_species = 0;
            return SFB_OK;
        }
        int it = 0, kind = SFB_IMEX_OK;
        SFB_TRY(solve_step(solver, rhs.p, U, Un.p, ldu, rule, value, max_iter, &it, &kind, res, st));
        if (kind != SFB_IMEX_OK) {
            res->fail_step = k;
            res->fail_kind = kind;
            res->fail_species = 0;
            return SFB_OK;
        }
        double nrm[4];
        SFB_TRY(sfb_diff_norm(Un.p, ldu, U, ldu, qy, qx, nrm, st));
        if (nrm[2] > 0.0 || nrm[1] > kBlowupLimit) {
            res->fail_step = k;
            res->fail_kind = SFB_IMEX_BLOWUP;
            res->fail_species = 0;
            return SFB_OK;
        }
        if (increments_host) increments_host[k] = nrm[0];
        if (iterations_host) iterations_host[k] = it;
        SFB_CUDA_TRY(cudaMemcpy2DAsync(U, (size_t)ldu * 8, Un.p, (size_t)ldu * 8, (size_t)qx * 8, qy,
                                       cudaMemcpyDeviceToDevice, st));
        res->steps_done = k + 1;
    }
    SFB_CUDA_TRY(cudaStreamSynchronize(st));
    return SFB_OK;
}

int sfb_imex_rds_run(sfb_pcg* solver_u, sfb_pcg* solver_v, const sfb_map* rhs_map, const double* params_host,
                     double tau_rho, int n_steps, int rule, double value, int max_iter, double steady_eps,
                     double* U, double* V, int ld, int* iterations_host, double* increments_host,
                     sfb_imex_result* res, void* stream) {
    SFB_NVTX("sfb_imex_rds_run");
    if (!solver_u || !solver_v || !rhs_map || !params_host || !U || !V || !res)
        return sfb::arg_error("imex rds run: null argument");
    if (n_steps < 0 || max_iter < 0) return sfb::arg_error("imex rds run: negative step or iteration count");
    init_result(res);
    cudaStream_t st = (cudaStream_t)stream;
    int qy = 0, qx = 0, qy2 = 0, qx2 = 0;
    SFB_TRY(sfb_pcg_shape(solver_u, &qy, &qx));
    SFB_TRY(sfb_pcg_shape(solver_v, &qy2, &qx2));
    if (qy != qy2 || qx != qx2) return sfb::arg_error("imex rds run: the two species' solvers differ in shape");
    DevBuf rhs, Un, Vn;
    SFB_TRY(alloc_grid(rhs, qy, ld, st));
    SFB_TRY(alloc_grid(Un, qy, ld, st));
    SFB_TRY(alloc_grid(Vn, qy, ld, st));
    sfb_pcg* solvers[2] = {solver_u, solver_v};
    double* cur[2] = {U, V};
    double* nxt[2] = {Un.p, Vn.p};
    for (int k = 0; k < n_steps; ++k) {
        double nrm[2][4];
        for (int sp = 0; sp < 2; ++sp) {
            // W = S + tau rho kin_sp(U, V) from the state at the start of the step
            // (timestepping.py:200-209), then the species' implicit solve
            double chk[2] = {0.0, 0.0};
            SFB_TRY(sfb_map_apply_dib(rhs_map, U, V, ld, sp, tau_rho, params_host, rhs.p, ld, chk, st));
            if (bad_check(chk)) {
                res->fail_step = k;
                res->fail_kind = SFB_IMEX_BLOWUP;
                res->fail_species = sp;
                return SFB_OK;
            }
            int it = 0, kind = SFB_IMEX_OK;
            SFB_TRY(solve_step(solvers[sp], rhs.p, cur[sp], nxt[sp], ld, rule, value, max_iter, &it, &kind, res, st));
            if (kind != SFB_IMEX_OK) {
                res->fail_step = k;
                res->fail_kind = kind;
                res->fail_species = sp;
                return SFB_OK;
            }
            SFB_TRY(sfb_diff_norm(nxt[sp], ld, cur[sp], ld, qy, qx, nrm[sp], st));
            if (nrm[sp][2] > 0.0 || nrm[sp][1] > kBlowupLimit) {
                res->fail_step = k;
                res->fail_kind = SFB_IMEX_BLOWUP;
                res->fail_species = sp;
                return SFB_OK;
            }
            if (iterations_host) iterations_host[2 * k + sp] = it;
        }
        if (increments_host) {
            increments_host[2 * k] = nrm[0][0];
            increments_host[2 * k + 1] = nrm[1][0];
        }
        for (int sp = 0; sp < 2; ++sp)
            SFB_CUDA_TRY(cudaMemcpy2DAsync(cur[sp], (size_t)ld * 8, nxt[sp], (size_t)ld * 8, (size_t)qx * 8, qy,
                                           cudaMemcpyDeviceToDevice, st));
        // steady state: both increments <= eps |U_new| (timestepping.py:213-216)
        const double thr = steady_eps * std::fmax(nrm[0][3], 1e-300);
        if (res->steady_step < 0 && nrm[0][0] <= thr && nrm[1][0] <= thr) res->steady_step = k;
        res->steps_done = k + 1;
    }
    SFB_CUDA_TRY(cudaStreamSynchronize(st));
    return SFB_OK;
}

}  // extern "C"
