"""Host-side logic of the product package against the oracle — CPU only.

Band assembly, term lists, rhs-builder bands, preconditioner factors and
guards are setup code that runs on the host; they are checked here against
the oracle's dense restatement of the reference (no kernels launched)."""

import numpy as np
import pytest

import oracle as orc
import paper_2109_01173_b200 as pb
from paper_2109_01173_b200 import solvers as psol
from paper_2109_01173_b200.banded import Band
from _cases import OBC, ODOMS, OP_CASES

PDOM = {"square": pb.SQUARE, "cap": pb.CAP_DOMAIN, "jar": pb.JAR_DOMAIN}
WAVE = pb.DomainSpec(pb.DomainKind.XNORMAL, pb.ProfileFn(
    lambda s: 1.0 + 0.3 * np.sin(2 * np.pi * np.asarray(s, float)),
    lambda s: 0.6 * np.pi * np.cos(2 * np.pi * np.asarray(s, float)), name="wave"))
RECT = pb.DomainSpec(pb.DomainKind.XNORMAL, pb.ProfileFn(
    lambda s: 2.0 * np.ones_like(np.asarray(s, float)),
    lambda s: np.zeros_like(np.asarray(s, float)), name="rect2"))
PDOM.update(wave=WAVE, rect=RECT)
PBC = {"d": pb.BCKind.DIRICHLET, "n": pb.BCKind.NEUMANN}


def desk():
    out = []
    for k in (1, 2, 3, 4):
        for n in (8, 16, 24):
            if n % k:
                continue
            for name in ("square", "cap", "jar", "wave"):
                for bc in ("d", "n"):
                    out.append((k, n, name, bc))
    return out


@pytest.mark.parametrize("case", desk(), ids=str)
def test_band_assembly_matches_oracle(case):
    k, n, name, bc = case
    x, y = pb.build_direction_sets(PDOM[name], k, n, PBC[bc], lumped=(k == 1))
    ox, oy = orc.direction_sets(ODOMS[name](), k, n, OBC[bc], lumped=(k == 1))
    for s, o in ((x, ox), (y, oy)):
        for nm, m in s.mats.named().items():
            ref = o["mats"][nm]
            assert isinstance(m, Band)
            assert np.max(np.abs(np.asarray(m) - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))), nm
            assert m.half_bandwidth() <= k + (1 if nm.endswith("_full") else 0)
        if k == 1:
            for nm, m in s.lumped.named().items():
                assert np.max(np.abs(np.asarray(m) - o["lumped"][nm])) <= 1e-13


@pytest.mark.parametrize("i", range(len(OP_CASES)))
def test_term_lists_and_rhs_bands(i):
    kind, k, n, dn, bc, p, lumped = OP_CASES[i]
    x, y = pb.build_direction_sets(PDOM[dn], k, n, PBC[bc], lumped=lumped)
    ox, oy = orc.direction_sets(ODOMS[dn](), k, n, OBC[bc], lumped=lumped)
    if kind == "ell":
        op, rhs = pb.elliptic_operator(x, y, p, lumped=lumped)
        ot, orhs = orc.elliptic_terms(ox, oy, p, lumped)
    else:
        op, rhs = pb.parabolic_operator(x, y, 1.0, p, lumped=lumped)
        ot, orhs = orc.parabolic_terms(ox, oy, 1.0, p, lumped)
    assert len(op) == len(ot)
    for (G, H), (oG, oH) in zip(op.terms, ot):
        assert np.max(np.abs(np.asarray(G) - oG)) <= 1e-13 * max(1, np.max(np.abs(oG)))
        assert np.max(np.abs(np.asarray(H) - oH)) <= 1e-13 * max(1, np.max(np.abs(oH)))
    # uploaded band layout reproduces every factor
    w, off, g, h = op.band_layout()
    for t, (G, H) in enumerate(op.terms):
        Gd = np.zeros(op.shape[0] * 2 * [1][0:1] and (op.shape[0], op.shape[0]))
        for d in range(w):
            for r in range(op.shape[0]):
                c = r + off + d
                if 0 <= c < op.shape[0]:
                    Gd[r, c] = g[t, r, d]
        assert np.array_equal(Gd, np.asarray(G))
    # rhs builder bands reproduce the dense rhs map on a random full grid
    F = np.random.default_rng(i).standard_normal(rhs.in_shape)
    wd, goff, gb, hoff, hb = rhs.layout()
    out = np.zeros(rhs.out_shape)
    Fp = np.pad(F, 16)
    for a in range(out.shape[0]):
        for b in range(out.shape[1]):
            blk = Fp[16 + a + goff:16 + a + goff + wd, 16 + b + hoff:16 + b + hoff + wd]
            out[a, b] = gb[a] @ blk @ hb[b]
    assert np.allclose(out, orhs(F), rtol=1e-13, atol=1e-14)


def test_unit_profile_collapses_to_two_terms():
    x, y = pb.build_direction_sets(pb.SQUARE, 2, 8, pb.BCKind.DIRICHLET)
    op, _ = pb.elliptic_operator(x, y, 1.0)
    assert len(op) == 2 and pb.is_unit_degenerate(y)


def test_pruning_and_shape_errors():
    with pytest.raises(pb.OperatorError, match="no nonzero terms"):
        pb.SylvesterOperator([(np.zeros((3, 3)), np.eye(3))])
    with pytest.raises(pb.OperatorError, match="inconsistent"):
        pb.SylvesterOperator([(np.eye(3), np.eye(3)), (np.eye(2), np.eye(3))])
    op = pb.SylvesterOperator([(np.eye(3), np.zeros((3, 3))), (2 * np.eye(3), np.eye(3))])
    assert len(op) == 1
    with pytest.raises(pb.OperatorError, match="does not match"):
        op.apply(np.zeros((2, 3)))


def test_operator_constructor_guards():
    x, y = pb.build_direction_sets(pb.SQUARE, 1, 8, pb.BCKind.NEUMANN)
    with pytest.raises(pb.OperatorError, match="gamma > 0"):
        pb.elliptic_operator(x, y, 0.0)
    with pytest.raises(pb.OperatorError, match="nonnegative"):
        pb.elliptic_operator(x, y, -1.0)
    with pytest.raises(pb.OperatorError):
        pb.parabolic_operator(x, y, 0.0, 0.1)


def test_basis_rules():
    assert pb.build_basis(1, 2, pb.BCKind.DIRICHLET).q == 1
    assert pb.build_basis(2, 24, pb.BCKind.DIRICHLET).n_elements == 12
    with pytest.raises(pb.AssemblyError):
        pb.build_basis(3, 8, pb.BCKind.DIRICHLET)
    with pytest.raises(pb.AssemblyError):
        pb.build_basis(5, 10, pb.BCKind.DIRICHLET)
    b = pb.build_basis(3, 12, pb.BCKind.NEUMANN)
    assert np.allclose(b.evaluate(b.nodes), np.eye(b.q), atol=1e-12)
    A, M = pb.assemble_standard(pb.build_basis(1, 2, pb.BCKind.DIRICHLET))
    assert np.allclose(A, [[4.0]]) and np.allclose(M, [[1 / 3]])


def test_preconditioner_factors_and_guard():
    x, y = pb.build_direction_sets(pb.CAP_DOMAIN, 2, 8, pb.BCKind.DIRICHLET)
    ox, oy = orc.direction_sets(orc.cap_domain(), 2, 8, orc.DIRICHLET)
    p = pb.make_preconditioner("elliptic_xnormal", x, y)
    L, R, ln, rn = orc.precond_factors("elliptic_xnormal", ox, oy)
    assert (p.left_name, p.right_name) == (ln, rn)
    assert np.allclose(p.left, L, atol=1e-14) and np.allclose(p.right, R, atol=1e-14)
    x, y = pb.build_direction_sets(pb.CAP_DOMAIN, 1, 8, pb.BCKind.NEUMANN)
    with pytest.raises(pb.SolverError, match="B1"):
        pb.make_preconditioner("elliptic_xnormal", x, y)
    with pytest.raises(pb.SolverError):
        pb.make_preconditioner("magic", x, y)
    assert pb.make_preconditioner("identity", None, None).is_identity


@pytest.mark.parametrize("k", [1, 2, 4])
def test_banded_cholesky_layout(k):
    x, y = pb.build_direction_sets(WAVE, k, 8 * k, pb.BCKind.DIRICHLET)
    P = y.mats.M3 + 1e-3 * y.mats.B1
    q = P.shape[0]
    b, band = psol._cholesky_band(P, q)
    assert b == k
    C = np.zeros((q, q))
    for i in range(q):
        for d in range(b):
            j = i - b + d
            if j >= 0:
                C[i, j] = band[i, d]
        C[i, i] = 1.0 / band[i, b]
    assert np.allclose(C @ C.T, np.asarray(P), rtol=1e-13, atol=1e-15)


def test_stopping_rules_and_timegrid():
    assert "R_0" in pb.relative_residual(1e-8).describe()
    assert pb.reference_increment(2.0).value == pytest.approx(0.1)
    assert pb.timestep_residual(0.01).value == 0.01
    assert pb.TimeGrid(tau=0.3, t_final=1.0).n_steps == 4
    assert pb.TimeGrid(tau=1.25e-5, t_final=0.75).n_steps == 60000
    with pytest.raises(pb.ConfigError):
        pb.TimeGrid(tau=0.0, t_final=1.0)


def test_models_match_oracle(golden):
    p = pb.dib_presets("spots_worms").replace(rho=400.0)
    f, g = pb.dib_kinetics(golden["kin/eta"], golden["kin/theta"], p)
    assert np.allclose(f, golden["kin/f"], rtol=1e-15) and np.allclose(g, golden["kin/g"], rtol=1e-15)
    e, t = pb.initial_fields((6, 5), pb.InitialData(amplitude=1e-3, seed=7))
    assert np.array_equal(e, golden["init/eta"]) and np.array_equal(t, golden["init/theta"])
    kin = pb.dib_kinetics_pair(p)
    assert np.allclose(kin[0](golden["kin/eta"], golden["kin/theta"]), golden["kin/f"])


def test_spectral_cache_host_route(golden):
    # the eigen setup is host LAPACK, identical to the reference's route
    x, y = pb.build_direction_sets(RECT, 3, 12, pb.BCKind.NEUMANN)
    op, _ = pb.elliptic_operator(x, y, 0.5)
    cache = pb.build_spectral_cache(op)
    assert cache.swapped
    ox, oy = orc.direction_sets(orc.rect_domain(), 3, 12, orc.NEUMANN)
    oc = orc.spectral_cache(orc.elliptic_terms(ox, oy, 0.5)[0])
    assert np.allclose(cache.lam1, oc["lam1"], rtol=1e-10, atol=1e-12)
    # columns whose largest entries tie in magnitude may flip sign under 1-ulp
    # assembly differences; the sandwich P (K o P^T B P) P^T is sign invariant
    sgn = np.sign(np.sum(cache.P1 * oc["P1"], axis=0))
    assert np.allclose(cache.P1 * sgn, oc["P1"], atol=1e-10)
    Z = np.diag([1.0, 2.0])
    bad = pb.SylvesterOperator([(Z, np.eye(2)), (np.eye(2), np.diag([-1.0, 3.0]))])
    with pytest.raises(pb.SolverError, match="singular"):
        pb.build_spectral_cache(bad).check_pencils()


def test_rcond_guard_uses_the_exact_condition_near_the_threshold():
    """solvers.py:90-100 guards with the exact 1-norm condition number; the
    banded LAPACK estimate is only trusted far from the 1e-14 threshold."""
    import scipy.sparse as sp

    from paper_2109_01173_b200.banded import Band
    from paper_2109_01173_b200.solvers import RCOND_GUARD, _rcond, _rcond_guard
    n = 40
    for eps in (1e-17, 3e-15, 1e-13, 1e-6):
        d = np.ones(n)
        d[7] = eps
        A = sp.diags([d], [0]).tocsr()
        exact = 1.0 / np.linalg.cond(A.toarray(), 1)
        assert _rcond(Band(A)) == pytest.approx(exact, rel=1e-12)
        if exact < RCOND_GUARD:
            with pytest.raises(pb.SolverError, match="singular"):
                _rcond_guard(Band(A), "P_L")
        else:
            _rcond_guard(Band(A), "P_L")


def test_spectral_form_rejects_non_symmetric_factors():
    """The spectral form of the preconditioner is the reference's LU solve
    only for symmetric factors: a non-symmetric one raises instead of being
    silently symmetrised."""
    from paper_2109_01173_b200.solvers import Preconditioner
    F = np.eye(6) * 4 + np.diag(np.ones(5), 1)
    with pytest.raises(pb.SolverError, match="symmetric"):
        Preconditioner._eigh(F, 6)
    lam, V = Preconditioner._eigh(F + F.T, 6)
    assert np.allclose(V @ np.diag(lam) @ V.T, F + F.T)


# reference pkg/tests/test_solvers.py TestClosedForm, host-side pieces
@pytest.mark.parametrize("n", [2, 4, 8, 16])
@pytest.mark.parametrize("gamma", [0.0, 1.0])
def test_dirichlet_eigenvalues_match_assembled_pencil(n, gamma):
    """TestClosedForm.test_smallest_eigenvalue / test_eigenvalues_match_assembled_pencil."""
    basis = pb.build_basis(1, n, pb.BCKind.DIRICHLET)
    A, M = pb.assemble_standard(basis)
    A, M = np.asarray(A), np.asarray(M)
    lam = np.sort(np.linalg.eigvals(np.linalg.solve(M, A) + 0.5 * gamma * np.eye(n - 1)).real)
    ref = np.sort(pb.dirichlet_p1_eigenvalues(n, gamma))
    assert np.max(np.abs(lam - ref)) < 1e-10 * max(1.0, np.max(ref))
    if n == 2 and gamma == 0.0:
        assert np.allclose(ref, [12.0])


def test_sine_basis_eigenvectors_and_involution():
    """TestClosedForm.test_sine_basis_matches_numerical_eigenvectors / test_sine_basis_involution."""
    A, _ = pb.assemble_standard(pb.build_basis(1, 4, pb.BCKind.DIRICHLET))
    A = np.asarray(A)
    _, vecs = np.linalg.eigh(A)
    X = pb.dirichlet_sine_basis(4)
    for j in range(3):
        a = vecs[:, j] / np.linalg.norm(vecs[:, j])
        b = X[:, j] / np.linalg.norm(X[:, j])
        assert min(np.linalg.norm(a - b), np.linalg.norm(a + b)) < 1e-12
    for n in (4, 8, 16):
        X = pb.dirichlet_sine_basis(n)
        assert np.allclose(X @ X, n / 2 * np.eye(n - 1), atol=1e-12)
