"""The inverse-form preconditioner's dense products as one to three levels of
Strassen around the DMMA GEMM (large shapes divisible by 4; BASELINE cfg5,
q = 8192, runs three), and the strided-batch GEMM of their leaf products.

The reference applies P_L^-1 U P_R^-1 by two dense solves
(solvers.py:134-143).  Strassen changes the summation order of the two
products, not their value: the checks are the product against the classic
schedule (normwise, at the level of the GEMM's own rounding), MO-PCG iterates
against the oracle at the north-star tolerance (1e-10), and the <Z,R> of the
assembly pass through the iteration counts of a converged solve.  The
threshold is lowered for these desk sizes and restored afterwards; the
full-size cfg5 test (test_gpu_fullsize.py) runs the default threshold.
"""

import numpy as np
import pytest

import oracle as orc
import paper_2109_01173_b200 as pb
from conftest import relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[1, 2, 3], ids=["one-level", "two-levels", "three-levels"])
def strassen_from_256(request):
    prev, prev_levels = pb.set_strassen_min_q(256), pb.set_strassen_levels(request.param)
    yield request.param
    pb.set_strassen_min_q(prev)
    pb.set_strassen_levels(prev_levels)


def _lumped_sets(Nx, Ny):
    return pb.build_direction_sets(pb.SQUARE, 1, (Nx, Ny), pb.BCKind.NEUMANN, lumped=True)


@pytest.mark.parametrize("Nx,Ny", [(511, 511), (767, 511), (255, 383), (512, 510), (300, 277)])
def test_strassen_product_matches_classic_schedule(Nx, Ny, strassen_from_256):
    x, y = _lumped_sets(Nx, Ny)
    d, tau = 20.0, 1.25e-5
    kw = {"d_u": d, "tau": tau, "lumped": True}
    pre_s = pb.make_preconditioner("parabolic_lumped", x, y, mode="inverse", **kw)
    # leaves of at least 64 (a quarter of the threshold): q < 498 takes at most two levels
    # (odd shapes are padded to a multiple of 2^(L+1))
    assert pre_s.uses_strassen() == (strassen_from_256 if min(x.q, y.q) >= 498 else min(strassen_from_256, 2))
    prev = pb.set_strassen_min_q(0)
    try:
        pre_c = pb.make_preconditioner("parabolic_lumped", x, y, mode="inverse", **kw)
        assert not pre_c.uses_strassen()
    finally:
        pb.set_strassen_min_q(prev)
    rng = np.random.default_rng(11)
    R = rng.standard_normal((y.q, x.q))
    Zs, Zc = pre_s.apply_inverse(R), pre_c.apply_inverse(R)
    assert relerr(Zs, Zc) <= 1e-13
    # and against the oracle's LU solves
    ox, oy = orc.direction_sets(orc.unit_square(), 1, (Nx, Ny), orc.NEUMANN, lumped=True)
    opre = orc.LUPrecond(*orc.precond_factors("parabolic_lumped", ox, oy, d_u=d, tau=tau, lumped=True))
    assert relerr(Zs, opre.inverse(R)) <= 1e-11


def test_strassen_below_the_threshold_keeps_the_classic_schedule(strassen_from_256):
    x, y = _lumped_sets(511, 200)  # q_y = 201 < 256
    pre = pb.make_preconditioner("parabolic_lumped", x, y, mode="inverse", d_u=1.0, tau=1e-4, lumped=True)
    assert pre.uses_strassen() == 0


def test_strassen_odd_shape_five_term_mo_pcg_vs_oracle(strassen_from_256):
    """cfg3-type system (P2, wave domain, Dirichlet: q = N - 1 is odd, five terms,
    the elliptic_xnormal preconditioner): the passes pad the odd shape with zeros."""
    N = 320  # q = N - 1 = 319
    wave = pb.DomainSpec(pb.DomainKind.XNORMAL, pb.ProfileFn(
        lambda s: 1.0 + 0.3 * np.sin(2 * np.pi * np.asarray(s, float)),
        lambda s: 0.6 * np.pi * np.cos(2 * np.pi * np.asarray(s, float)), name="wave"))
    x, y = pb.build_direction_sets(wave, 2, N, pb.BCKind.DIRICHLET)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    a, b, c = orc.seeded_modes(3)
    s = np.arange(N + 1) / N
    F = sum(c[m] * np.sin(b[m] * np.pi * s)[:, None] * np.sin(a[m] * np.pi * s)[None, :] for m in range(8))
    rhs = rhs_of(F)
    pre = pb.make_preconditioner("elliptic_xnormal", x, y, mode="inverse")
    assert op.shape == (319, 319) and pre.uses_strassen() == min(strassen_from_256, 2)
    ox, oy = orc.direction_sets(orc.wave_domain(), 2, N, orc.DIRICHLET)
    terms, orhs = orc.elliptic_terms(ox, oy, 1.0)
    opre = orc.LUPrecond(*orc.precond_factors("elliptic_xnormal", ox, oy))
    K = 10
    ref = orc.mo_pcg(terms, orhs(F), opre.inverse, ("residual", 1e-300), max_iter=K)
    rep = pb.mo_pcg(op, rhs, precond=pre, stop=pb.fixed_budget(), max_iter=K)
    assert rep.iterations == K
    assert relerr(rep.solution, ref["solution"]) <= 1e-10
    h = np.asarray(ref["history"])
    assert np.max(np.abs(rep.residual_history - h) / h) <= 1e-10


@pytest.mark.parametrize("d,tau", [(1.0, 5e-4), (20.0, 1.25e-5)])
def test_strassen_mo_pcg_iterates_vs_oracle(d, tau, strassen_from_256):
    """cfg5-type step system (lumped P1, Neumann, square) at q = 512: K-th
    iterates and residual histories against the oracle, then a converged solve."""
    N = 511
    x, y = _lumped_sets(N, N)
    op, rhs_of = pb.parabolic_operator(x, y, d, tau, lumped=True)
    ox, oy = orc.direction_sets(orc.unit_square(), 1, N, orc.NEUMANN, lumped=True)
    terms, orhs = orc.parabolic_terms(ox, oy, d, tau, True)
    opre = orc.LUPrecond(*orc.precond_factors("parabolic_lumped", ox, oy, d_u=d, tau=tau, lumped=True))
    rng = np.random.default_rng(5)
    S = 1e-3 * rng.uniform(-1.0, 1.0, (N + 1, N + 1))
    rhs = orhs(S)
    assert relerr(rhs_of(S), rhs) <= 1e-13
    pre = pb.make_preconditioner("parabolic_lumped", x, y, mode="inverse", d_u=d, tau=tau, lumped=True)
    assert pre.uses_strassen() == strassen_from_256
    K = 6
    ref = orc.mo_pcg(terms, rhs, opre.inverse, ("residual", 1e-300), u0=S, max_iter=K)
    rep = pb.mo_pcg(op, rhs, precond=pre, stop=pb.fixed_budget(), u0=S, max_iter=K)
    assert rep.iterations == K
    assert relerr(rep.solution, ref["solution"]) <= 1e-10
    h = np.asarray(ref["history"])
    assert np.max(np.abs(rep.residual_history - h) / h) <= 1e-10
    full = orc.mo_pcg(terms, rhs, opre.inverse, ("residual", 1e-10), max_iter=500)
    rep = pb.mo_pcg(op, rhs, precond=pre, stop=pb.relative_residual(1e-10), max_iter=500)
    assert rep.stop_reason == "tolerance"
    assert abs(rep.iterations - full["iterations"]) <= 1
    assert relerr(rep.solution, full["solution"]) <= 1e-9


@pytest.mark.parametrize("nb", [1, 7, 49])
@pytest.mark.parametrize("M,N,K", [(256, 256, 256), (384, 256, 512), (130, 258, 100)])
def test_batched_gemm_matches_fp64_matmul(M, N, K, nb):
    """sfb_dgemm_nt_batch: nb stacked products in one persistent launch (rank-3
    tensor maps; padded leading dimensions as the Strassen leaves have)."""
    import torch

    from paper_2109_01173_b200 import _native as nat

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    lda, ldb, ldc = K + 2, K + 4, N + (N % 2) + 2
    A = torch.randn(nb, M, lda, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(nb, N, ldb, dtype=torch.float64, device="cuda", generator=g)
    out = torch.zeros(nb, M, ldc, dtype=torch.float64, device="cuda")
    nat.check(nat.lib().sfb_dgemm_nt_batch(nb, A.data_ptr(), lda, B.data_ptr(), ldb, M, N, K, out.data_ptr(), ldc,
                                           M * ldc, nat.stream()), "batched GEMM")
    torch.cuda.synchronize()
    for b in range(nb):
        ref = A[b, :, :K] @ B[b, :, :K].T
        assert float((out[b, :, :N] - ref).norm() / ref.norm()) <= 1e-14
    assert float(out[:, :, N:].abs().max()) == 0.0  # nothing stored past the N columns


# ---- the spectral sandwich (four products, Hadamard scaling in the second assembly pass) ----
def test_strassen_spectral_preconditioner_form_matches_classic(strassen_from_256):
    x, y = _lumped_sets(383, 511)  # q = (512, 384)
    kw = {"d_u": 20.0, "tau": 1.25e-5, "lumped": True}
    pre_s = pb.make_preconditioner("parabolic_lumped", x, y, mode="spectral", **kw)
    assert pre_s.uses_strassen() == min(strassen_from_256, 2)
    prev = pb.set_strassen_min_q(0)
    try:
        pre_c = pb.make_preconditioner("parabolic_lumped", x, y, mode="spectral", **kw)
        assert pre_c.uses_strassen() == 0
    finally:
        pb.set_strassen_min_q(prev)
    R = np.random.default_rng(3).standard_normal((y.q, x.q))
    Zs, Zc = pre_s.apply_inverse(R), pre_c.apply_inverse(R)
    assert relerr(Zs, Zc) <= 1e-12
    ox, oy = orc.direction_sets(orc.unit_square(), 1, (383, 511), orc.NEUMANN, lumped=True)
    opre = orc.LUPrecond(*orc.precond_factors("parabolic_lumped", ox, oy, **kw))
    assert relerr(Zs, opre.inverse(R)) <= 1e-10


def test_strassen_reduced_solve_vs_oracle(strassen_from_256):
    """cfg1-type reduced solve (square, P1, Dirichlet) at q = 511 (odd: padded inside the passes)."""
    N = 512
    x, y = pb.build_direction_sets(pb.SQUARE, 1, N, pb.BCKind.DIRICHLET)
    op, rhs_of = pb.elliptic_operator(x, y, 1.0)
    a, b, c = orc.seeded_modes(1)
    s = np.arange(N + 1) / N
    F = sum(c[m] * np.sin(b[m] * np.pi * s)[:, None] * np.sin(a[m] * np.pi * s)[None, :] for m in range(8))
    rhs = rhs_of(F)
    cache = pb.build_spectral_cache(op)
    assert cache.uses_strassen() == strassen_from_256
    rep = pb.solve_reduced(op, rhs, cache=cache)
    ox, oy = orc.direction_sets(orc.unit_square(), 1, N, orc.DIRICHLET)
    terms, orhs = orc.elliptic_terms(ox, oy, 1.0)
    U, res, _ = orc.reduced_solve(terms, orhs(F))
    assert relerr(rep.solution, U) <= 1e-10
    assert rep.residual_history[-1] <= 1e-10


def test_strassen_reduced_solve_swapped_pencil_vs_oracle(strassen_from_256):
    """cfg2-type reduced solve (Neumann P3 on [0,2]x[0,1], the swapped pencil) at q = 304."""
    from paper_2109_01173_b200 import workloads as wl

    w = wl.cfg2(N=303)
    assert w.op.shape == (304, 304)
    cache = pb.build_spectral_cache(w.op)
    assert cache.uses_strassen() == min(strassen_from_256, 2)
    rep = pb.solve_reduced(w.op, w.rhs, cache=cache)
    ox, oy = orc.direction_sets(orc.rect_domain(), 3, w.N, orc.NEUMANN)
    terms, orhs = orc.elliptic_terms(ox, oy, 0.5)
    rhs = orhs(wl.cosine_source_rect(w.N, 2))
    assert relerr(w.rhs, rhs) <= 1e-13
    U, res, c = orc.reduced_solve(terms, rhs)
    assert bool(c["swapped"]) and rep.diagnostics["pencil_swapped"] is True
    assert relerr(rep.solution, U) <= 1e-10
