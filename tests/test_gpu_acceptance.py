"""The reference's acceptance desk matrix through the CUDA path.

Reference tests/test_acceptance.py:109-154 (criterion 5) runs 60 small
(k, N, domain, bc) configurations (tests/conftest.py:12-22) and checks that
operator apply, the spectral reduction, the closed form and MO-PCG agree with
the sparse direct solve.  Here every one of those solves runs on the device
(through the C ABI) and is compared with the reference's OWN outputs on the
same seeded inputs (tests/golden, written by make_golden.py from the
unmodified reference): apply and rhs <= 1e-12, direct / reduced / closed-form
/ MO-PCG solutions <= 1e-10 relative Frobenius.  MO-PCG iteration counts must
stay within the reference's own rounding envelope: the oracle re-run under
deliberate changes of rounding (oracle.iteration_envelope: re-associated
GEMMs, reversed term order, 1-ulp rhs perturbations, the preconditioner as LU
/ Cholesky / explicit-inverse solves) spans [lo, hi]; the device count must
lie within that width (+1) of the reference's count.  Neumann cases run MO-PCG with the identity
preconditioner, as the reference does.

Also reference tests/test_solvers.py:249-269: short preconditioned parabolic
runs on the cap (lumped and consistent mass) must coincide iterate by iterate
with the vec-form PCG.
"""

import numpy as np
import pytest

import oracle as orc
import paper_2109_01173_b200 as pb
from _cases import DESK_CASES, desk_oracle
from conftest import relerr

pytestmark = pytest.mark.gpu

BCS = {"d": pb.BCKind.DIRICHLET, "n": pb.BCKind.NEUMANN}


@pytest.mark.parametrize("i", range(len(DESK_CASES)), ids=lambda i: "{}-{}-{}-{}".format(*DESK_CASES[i]))
def test_desk_matrix_vs_reference(golden, i):
    k, n, name, bc = DESK_CASES[i]
    tag = f"desk/{i}"
    x, y = pb.build_direction_sets(pb.domain_from_name(name), k, n, BCS[bc], lumped=k == 1)
    gamma = 0.0 if bc == "d" else 1.0
    op, rhs_of = pb.elliptic_operator(x, y, gamma)
    assert len(op) == int(golden[f"{tag}/nterms"])
    # apply vs the reference, and vs the Kronecker matrix (test_acceptance.py:118-123)
    U = golden[f"{tag}/U"]
    AU = op.apply(U)
    assert relerr(AU, golden[f"{tag}/AU"]) <= 1e-12
    K = pb.to_kronecker(op)
    assert relerr(pb.unvec(K @ pb.vec(U), op.shape), AU) <= 1e-12
    rhs = rhs_of(golden[f"{tag}/F"])
    assert relerr(rhs, golden[f"{tag}/rhs"]) <= 1e-12
    direct = pb.solve_direct(op, rhs)
    assert relerr(direct.solution, golden[f"{tag}/direct"]) <= 1e-10
    if len(op) == 2:
        red = pb.solve_reduced(op, rhs)
        assert relerr(red.solution, golden[f"{tag}/reduced"]) <= 1e-10
        if f"{tag}/closed" in golden:
            F0 = golden[f"{tag}/F"].copy()
            F0[0, :] = F0[-1, :] = F0[:, 0] = F0[:, -1] = 0.0
            red0 = pb.solve_reduced(op, rhs_of(F0))
            assert relerr(red0.solution, golden[f"{tag}/reduced0"]) <= 1e-10
            closed = pb.solve_reduced_closed_form(gamma, pb.interior_values(F0, x, y), n)
            assert relerr(closed.solution, golden[f"{tag}/closed"]) <= 1e-10
            assert relerr(closed.solution, red0.solution) <= 1e-9  # the reference's own criterion
    if bc == "d":
        pre = pb.make_preconditioner("elliptic_square" if name == "square" else "elliptic_xnormal", x, y)
    else:
        pre = pb.make_preconditioner("identity", x, y)
    rep = pb.mo_pcg(op, rhs, precond=pre, stop=pb.relative_residual(1e-12), max_iter=5000)
    assert rep.stop_reason == "tolerance"
    assert relerr(rep.solution, golden[f"{tag}/pcg"]) <= 1e-10
    assert relerr(rep.solution, golden[f"{tag}/direct"]) <= 1e-9  # test_acceptance.py:154
    _, _, _, terms, orhs, pinv = desk_oracle(i)
    it, lo, hi = orc.iteration_envelope(terms, orhs(golden[f"{tag}/F"]), pinv, ("residual", 1e-12), max_iter=5000)
    ref_it = int(golden[f"{tag}/pcg_iters"])  # the reference's own run is one more realization
    lo, hi = min(lo, ref_it), max(hi, ref_it)
    assert abs(rep.iterations - ref_it) <= hi - lo + 1, (rep.iterations, ref_it, it, lo, hi)


@pytest.mark.parametrize("lumped", [False, True])
def test_parabolic_cap_matches_vector_pcg_iterate_by_iterate(lumped):
    """reference tests/test_solvers.py:249-269: tau = 5e-4 (mass-dominated,
    near-exact preconditioner), every MO-PCG iterate equals the vec-form
    PCG's; both on the device, and both against the oracle."""
    tau = 5e-4
    x, y = pb.build_direction_sets(pb.CAP_DOMAIN, 1, 8, pb.BCKind.DIRICHLET, lumped=True)
    op, _ = pb.parabolic_operator(x, y, 1.0, tau, lumped=lumped)
    pre = pb.make_preconditioner("parabolic", x, y, d_u=1.0, tau=tau, lumped=lumped)
    rhs = np.random.default_rng(1234).standard_normal(op.shape)
    stop = pb.relative_residual(1e-10)
    rep_m = pb.mo_pcg(op, rhs, precond=pre, stop=stop, record_iterates=True)
    rep_v = pb.vector_pcg(pb.to_kronecker(op), pb.vec(rhs), P=pre.as_kronecker(op.shape), stop=stop,
                          record_iterates=True)
    assert rep_m.iterations <= 12
    assert abs(rep_m.iterations - rep_v.iterations) <= 1
    for a, b in zip(rep_m.diagnostics["iterates"], rep_v.diagnostics["iterates"]):
        assert np.linalg.norm(pb.vec(a) - b) <= 1e-10 * max(np.linalg.norm(b), 1e-30)
    ox, oy = orc.direction_sets(orc.cap_domain(), 1, 8, orc.DIRICHLET, lumped=True)
    terms, _ = orc.parabolic_terms(ox, oy, 1.0, tau, lumped)
    opre = orc.LUPrecond(*orc.precond_factors("parabolic", ox, oy, d_u=1.0, tau=tau, lumped=lumped))
    ref = orc.mo_pcg(terms, rhs, opre.inverse, ("residual", 1e-10), record=True)
    assert rep_m.iterations == ref["iterations"]
    for a, b in zip(rep_m.diagnostics["iterates"], ref["iterates"]):
        assert relerr(a, b) <= 1e-10 if np.linalg.norm(b) > 0 else np.linalg.norm(a) == 0
