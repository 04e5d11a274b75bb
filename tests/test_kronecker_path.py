"""the Kronecker (vector) cross-check path.

CPU: to_kronecker / as_kronecker assembly against the oracle's dense terms
and factors (solvers.py:145-150, operators.py:141-155), the guard.
GPU: vector_pcg (device CSR SpMV + fused vector passes) iterate by iterate
against mo_pcg and the oracle, solve_direct against a dense direct solve."""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as orc
import paper_2109_01173_b200 as pb
from _cases import sine_source
from conftest import relerr
from test_host_logic import WAVE

D = pb.BCKind.DIRICHLET


def _dense_kron(terms):
    return sum(np.kron(H.T, G) for G, H in terms)


@pytest.mark.parametrize("k,N,lumped", [(1, 12, False), (2, 12, False), (4, 8, False), (1, 12, True)])
def test_to_kronecker_matches_oracle_terms(k, N, lumped):
    x, y = pb.build_direction_sets(WAVE, k, N, D, lumped=lumped)
    op, _ = pb.elliptic_operator(x, y, 1.0, lumped=lumped)
    ox, oy = orc.direction_sets(orc.wave_domain(), k, N, orc.DIRICHLET, lumped=lumped)
    terms, _ = orc.elliptic_terms(ox, oy, 1.0, lumped=lumped)
    K = pb.to_kronecker(op)
    assert sp.issparse(K)
    assert np.abs(K.toarray() - _dense_kron(terms)).max() <= 1e-12 * np.abs(_dense_kron(terms)).max()
    U = np.random.default_rng(k).standard_normal(op.shape)
    assert np.allclose(K @ pb.vec(U), pb.vec(orc.apply_terms(terms, U)), atol=1e-12)


def test_as_kronecker_and_guard():
    x, y = pb.build_direction_sets(WAVE, 2, 12, D)
    pre = pb.make_preconditioner("elliptic_xnormal", x, y)
    P = pre.as_kronecker((y.q, x.q))
    ox, oy = orc.direction_sets(orc.wave_domain(), 2, 12, orc.DIRICHLET)
    L, R, _, _ = orc.precond_factors("elliptic_xnormal", ox, oy)
    assert np.allclose(P.toarray(), np.kron(R.T, L), atol=1e-13)
    assert P.sfb_pre is pre and P.sfb_shape == (y.q, x.q)
    xb, yb = pb.build_direction_sets(pb.SQUARE, 1, 460, D)
    op, _ = pb.elliptic_operator(xb, yb, 1.0)
    with pytest.raises(pb.OperatorError, match="guarded"):
        pb.to_kronecker(op)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["inverse", "banded"])
def test_vector_pcg_matches_mo_pcg_iterate_by_iterate(mode):
    N = 16
    x, y = pb.build_direction_sets(WAVE, 2, N, D)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    rhs = rhs_of(sine_source(N, N, 3))
    pre = pb.make_preconditioner("elliptic_xnormal", x, y, mode=mode)
    stop = pb.relative_residual(1e-10)
    rm = pb.mo_pcg(op, rhs, precond=pre, stop=stop, record_iterates=True)
    rv = pb.vector_pcg(pb.to_kronecker(op), pb.vec(rhs), P=pre.as_kronecker(op.shape), stop=stop,
                       record_iterates=True)
    assert rv.method == "vector-pcg" and abs(rv.iterations - rm.iterations) <= 1
    for s in range(min(8, rm.iterations)):
        assert relerr(pb.unvec(rv.diagnostics["iterates"][s + 1], op.shape),
                      rm.diagnostics["iterates"][s + 1]) <= 1e-10
    assert relerr(pb.unvec(rv.solution, op.shape), rm.solution) <= 1e-8
    # the oracle's vector-free recurrences agree as well
    ox, oy = orc.direction_sets(orc.wave_domain(), 2, N, orc.DIRICHLET)
    terms, _ = orc.elliptic_terms(ox, oy, 1.0)
    oref = orc.mo_pcg(terms, rhs, orc.LUPrecond(*orc.precond_factors("elliptic_xnormal", ox, oy)).inverse,
                      ("residual", 1e-10))
    assert abs(rv.iterations - oref["iterations"]) <= 1


@pytest.mark.gpu
def test_vector_pcg_identity_warm_start_increment_rule_and_errors():
    x, y = pb.build_direction_sets(WAVE, 1, 12, D)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    K = pb.to_kronecker(op)
    b = pb.vec(rhs_of(sine_source(12, 12, 3)))
    x0 = 1e-3 * np.random.default_rng(2).standard_normal(b.size)
    r = pb.vector_pcg(K, b, stop=pb.relative_residual(1e-12), x0=x0, max_iter=5000)
    exact = np.linalg.solve(K.toarray(), b)
    assert r.stop_reason == "tolerance" and relerr(r.solution, exact) <= 1e-9
    r2 = pb.vector_pcg(K, b, stop=pb.increment_threshold(1e-10), max_iter=5000)
    assert r2.stop_reason == "increment"
    assert pb.vector_pcg(K, np.zeros_like(b)).iterations == 0
    # a plain sparse P (not from as_kronecker) is factored like the reference's splu
    r3 = pb.vector_pcg(K, b, P=sp.identity(b.size, format="csr"), stop=pb.relative_residual(1e-12), max_iter=5000)
    assert r3.iterations == pb.vector_pcg(K, b, stop=pb.relative_residual(1e-12), max_iter=5000).iterations
    with pytest.raises(pb.OperatorError, match="does not match"):
        pb.vector_pcg(K, b, P=sp.identity(b.size + 1, format="csr"))
    with pytest.raises(pb.OperatorError, match="not positive definite"):
        pb.vector_pcg(-K, b, max_iter=10)


@pytest.mark.gpu
@pytest.mark.parametrize("k,N", [(1, 14), (2, 12)])
def test_solve_direct_matches_dense_solve(k, N):
    x, y = pb.build_direction_sets(WAVE, k, N, D)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    rhs = rhs_of(sine_source(N, N, 3))
    rep = pb.solve_direct(op, rhs)
    K = pb.to_kronecker(op).toarray()
    exact = pb.unvec(np.linalg.solve(K, pb.vec(rhs)), op.shape)
    assert rep.method == "direct" and rep.stop_reason == "direct" and rep.iterations == 0
    assert rep.residual_history[0] <= 1e-12
    assert relerr(rep.solution, exact) <= 1e-10
    assert rep.diagnostics["n"] == op.shape[0] * op.shape[1]


@pytest.mark.gpu
def test_solve_direct_non_spd_and_singular_operators():
    """Operators not flagged SPD take the reference's route (SuperLU factors
    of the Kronecker matrix, solved on the device); reference
    tests/test_solvers.py:295-330: identity returns the rhs, a singular
    operator raises SolverError."""
    rng = np.random.default_rng(9)
    q = 9
    G = np.eye(q) * 4 + np.diag(np.ones(q - 1), 1) * 1.5 - np.diag(np.ones(q - 1), -1) * 0.5  # non-symmetric
    H = np.eye(q) * 3 + np.diag(np.ones(q - 1), -1)
    op = pb.SylvesterOperator([(G, H), (np.eye(q), np.diag(np.arange(1.0, q + 1)))])
    rhs = rng.standard_normal((q, q))
    rep = pb.solve_direct(op, rhs)
    K = pb.to_kronecker(op).toarray()
    assert relerr(rep.solution, pb.unvec(np.linalg.solve(K, pb.vec(rhs)), op.shape)) <= 1e-12
    assert rep.residual_history[0] <= 1e-12
    ident = pb.SylvesterOperator([(np.eye(5), np.eye(5))])
    r5 = rng.standard_normal((5, 5))
    assert np.allclose(pb.solve_direct(ident, r5).solution, r5, atol=1e-13)
    x, y = pb.build_direction_sets(pb.SQUARE, 1, 8, pb.BCKind.NEUMANN)
    A, M = np.asarray(x.mats.A), np.asarray(x.mats.M)
    sing = pb.SylvesterOperator([(A, M), (M, A)], symmetric=True, positive_definite=False)
    with pytest.raises(pb.SolverError):
        pb.solve_direct(sing, np.ones(sing.shape))


@pytest.mark.gpu
def test_vector_imex_drivers_match_reference_trajectories(golden):
    # heat, cfg4-type (5-term step operator: MO-PCG to round-off per step)
    x, y = pb.build_direction_sets(WAVE, 4, 8, D)
    F = sine_source(8, 8, 4)
    tr = pb.vector_imex_heat(WAVE, x, y, 1.0, pb.SeparableSource(F, lambda t: np.exp(-t)), golden["heat/u0"],
                             pb.TimeGrid(1e-3, 5e-3))
    assert np.all(tr.iterations == 0)
    assert relerr(tr.final[0], golden["heat/t12/U"]) <= 1e-10
    # DIB, cfg5-type (two-term step operators: spectral direct solves)
    p = pb.dib_presets("spots_worms").replace(rho=400.0)
    xl, yl = pb.build_direction_sets(pb.SQUARE, 1, 15, pb.BCKind.NEUMANN, lumped=True)
    tau = 5e-3 / p.rho
    tv = pb.vector_imex_rds(pb.SQUARE, xl, yl, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho,
                            (golden["dib/eta0"], golden["dib/theta0"]), pb.TimeGrid(tau, 6 * tau), lumped=True)
    assert relerr(tv.final[0], golden["dib/t12/U"]) <= 1e-10
    assert relerr(tv.final[1], golden["dib/t12/V"]) <= 1e-10


@pytest.mark.gpu
def test_vector_pcg_generic_sparse_preconditioner_vs_reference_algorithm():
    """A P that is not Kronecker-structured (here: an incomplete-Cholesky-like
    sparse SPD matrix, the Kronecker matrix's own tridiagonal-block part):
    factored once like the reference (spla.splu(P), solvers.py:473) and solved
    on the device (sfb_lu_solve).  Iterates against the reference recurrence
    with the host LU solve on the same inputs."""
    import scipy.sparse.linalg as spla
    N = 12
    x, y = pb.build_direction_sets(WAVE, 2, N, D)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    K = sp.csr_matrix(pb.to_kronecker(op))
    # a generic SPD preconditioner: K without its far off-diagonal couplings
    C = K.tocoo()
    keep = np.abs(C.row - C.col) <= 2
    P = sp.csr_matrix((C.data[keep], (C.row[keep], C.col[keep])), shape=K.shape)
    P = 0.5 * (P + P.T) + sp.diags(np.abs(P).sum(axis=1).A.ravel())  # diagonally dominant SPD
    b = pb.vec(rhs_of(sine_source(N, N, 3)))
    stop = pb.relative_residual(1e-10)
    rep = pb.vector_pcg(K, b, P=P, stop=stop, record_iterates=True)
    # the reference recurrence (solvers.py:456-517) with SuperLU on the host (checker)
    solve = spla.splu(sp.csc_matrix(P)).solve
    xr = np.zeros_like(b)
    r = b.copy()
    z = solve(r)
    q = z.copy()
    rz = r @ z
    its = [xr.copy()]
    res0 = np.linalg.norm(r)
    n_it = 0
    for s in range(1000):
        w = K @ q
        a = rz / (q @ w)
        xr += a * q
        r -= a * w
        its.append(xr.copy())
        n_it = s + 1
        if np.linalg.norm(r) <= 1e-10 * res0:
            break
        z = solve(r)
        rzn = r @ z
        q = z + (rzn / rz) * q
        rz = rzn
    assert rep.stop_reason == "tolerance"
    assert abs(rep.iterations - n_it) <= 1
    for a_, b_ in list(zip(rep.diagnostics["iterates"], its))[1:10]:
        assert relerr(a_, b_) <= 1e-10
    assert relerr(rep.solution, its[-1]) <= 1e-9
    # the device LU solve itself
    from paper_2109_01173_b200.solvers import _DeviceLU
    import torch
    lu = _DeviceLU(P, P.shape[0])
    rr = np.random.default_rng(2).standard_normal(P.shape[0])
    zd = torch.empty((1, P.shape[0]), dtype=torch.float64, device="cuda")
    lu.solve(torch.from_numpy(rr.reshape(1, -1)).cuda(), zd)
    assert relerr(zd.cpu().numpy().ravel(), solve(rr)) <= 1e-13
