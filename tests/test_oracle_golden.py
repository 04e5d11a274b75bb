"""Pin the CPU oracle (oracle/) to golden vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle as orc
from _cases import (ASM_CASES, DESK_CASES, OBC, ODOMS, OP_CASES, cosine_source_rect, desk_oracle,
                    sine_source)
from conftest import relerr


@pytest.mark.parametrize("case", ASM_CASES, ids=str)
def test_assembly_matches_reference(golden, case):
    k, n, dn, bc = case
    x, y = orc.direction_sets(ODOMS[dn](), k, n, OBC[bc], lumped=(k == 1))
    tag = f"asm/{k}_{n}_{dn}_{bc}"
    for side, s in (("x", x), ("y", y)):
        for name, m in s["mats"].items():
            ref = golden[f"{tag}/{side}/{name}"]
            assert np.max(np.abs(m - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))), (side, name)
        for name, m in s.get("lumped", {}).items():
            ref = golden[f"{tag}/{side}/L_{name}"]
            assert np.max(np.abs(m - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))), (side, name)


@pytest.mark.parametrize("dn,bc", [("cap", "n"), ("square", "d"), ("jar", "n")])
def test_lumped_rectangular_grid(golden, dn, bc):
    x, y = orc.direction_sets(ODOMS[dn](), 1, (9, 6), OBC[bc], lumped=True)
    for side, s in (("x", x), ("y", y)):
        for name, m in s["lumped"].items():
            ref = golden[f"asml/{dn}_{bc}/{side}/{name}"]
            assert np.max(np.abs(m - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("i", range(len(OP_CASES)))
def test_operator_and_rhs_match_reference(golden, i):
    kind, k, n, dn, bc, p, lumped = OP_CASES[i]
    x, y = orc.direction_sets(ODOMS[dn](), k, n, OBC[bc], lumped=lumped)
    if kind == "ell":
        terms, rhs_of = orc.elliptic_terms(x, y, p, lumped)
    else:
        terms, rhs_of = orc.parabolic_terms(x, y, 1.0, p, lumped)
    tag = f"op/{i}"
    assert len(terms) == int(golden[f"{tag}/nterms"])
    assert relerr(orc.apply_terms(terms, golden[f"{tag}/U"]), golden[f"{tag}/AU"]) <= 1e-13
    assert relerr(rhs_of(golden[f"{tag}/F"]), golden[f"{tag}/rhs"]) <= 1e-13


def test_reduced_cfg1_type(golden):
    x, y = orc.direction_sets(orc.unit_square(), 1, 17, orc.DIRICHLET)
    terms, rhs_of = orc.elliptic_terms(x, y, 1.0)
    rhs = rhs_of(sine_source(17, 17, 1))
    assert relerr(rhs, golden["red1/rhs"]) <= 1e-14
    U, rel, cache = orc.reduced_solve(terms, rhs)
    assert relerr(U, golden["red1/U"]) <= 1e-12
    assert bool(cache["swapped"]) == bool(golden["red1/swapped"])
    assert rel <= 1e-12


def test_reduced_cfg2_type_swaps_pencils(golden):
    x, y = orc.direction_sets(orc.rect_domain(), 3, 12, orc.NEUMANN)
    terms, rhs_of = orc.elliptic_terms(x, y, 0.5)
    assert len(terms) == int(golden["red2/nterms"]) == 2
    rhs = rhs_of(cosine_source_rect(12, 2))
    assert relerr(rhs, golden["red2/rhs"]) <= 1e-14
    U, rel, cache = orc.reduced_solve(terms, rhs)
    assert bool(cache["swapped"]) and bool(golden["red2/swapped"])
    assert relerr(U, golden["red2/U"]) <= 1e-12


@pytest.mark.parametrize("tol_tag,tol", [("t12", 1e-12), ("t8", 1e-8)])
def test_mo_pcg_cfg3_type(golden, tol_tag, tol):
    x, y = orc.direction_sets(orc.wave_domain(), 2, 16, orc.DIRICHLET)
    terms, rhs_of = orc.elliptic_terms(x, y, 1.0)
    rhs = rhs_of(sine_source(16, 16, 3))
    assert relerr(rhs, golden["pcg3/rhs"]) <= 1e-14
    left, right, ln, rn = orc.precond_factors("elliptic_xnormal", x, y)
    assert [ln, rn] == list(golden["pcg3/names"])
    pre = orc.LUPrecond(left, right, ln, rn)
    assert relerr(pre.inverse(golden["pcg3/R"]), golden["pcg3/PinvR"]) <= 1e-13
    r = orc.mo_pcg(terms, rhs, pre.inverse, ("residual", tol), max_iter=5000, record=True)
    tag = f"pcg3/{tol_tag}"
    assert abs(r["iterations"] - int(golden[f"{tag}/iters"])) <= 1
    for a, b in zip(r["iterates"][:8], golden[f"{tag}/first8"]):
        assert relerr(a, b) <= 1e-10
    assert relerr(r["solution"], golden[f"{tag}/U"]) <= (1e-10 if tol < 1e-10 else 1e-7)


@pytest.mark.parametrize("tol_tag,tol", [("t12", 1e-12), ("t8", 1e-8)])
def test_imex_heat_cfg4_type(golden, tol_tag, tol):
    x, y = orc.direction_sets(orc.wave_domain(), 4, 8, orc.DIRICHLET)
    F = sine_source(8, 8, 4)
    assert relerr(F, golden["heat/F"]) == 0.0
    u0 = 1e-2 * np.random.default_rng(4).standard_normal((y["q"], x["q"]))
    assert np.array_equal(u0, golden["heat/u0"])
    tr = orc.imex_heat(orc.wave_domain(), x, y, 1.0, lambda u, X, Y, t: np.exp(-t) * F,
                       u0, 1e-3, 5e-3, rule="residual", tol=tol, max_iter=5000)
    assert np.all(np.abs(tr["iterations"] - golden[f"heat/{tol_tag}/iters"]) <= 1)
    assert relerr(tr["final"], golden[f"heat/{tol_tag}/U"]) <= (1e-10 if tol < 1e-10 else 1e-7)


@pytest.mark.parametrize("tag", ["tau", "t12"])
def test_imex_dib_cfg5_type(golden, tag):
    p = orc.dib_params(rho=400.0)
    assert p["D"] == pytest.approx(float(golden["dib/D"]), rel=1e-15)
    x, y = orc.direction_sets(orc.unit_square(), 1, 15, orc.NEUMANN, lumped=True)
    e0, t0 = orc.initial_fields((y["q"], x["q"]), 2e-3, 5)
    assert np.array_equal(e0 - 1e-3, golden["dib/eta0"])
    assert np.array_equal(t0 - 1e-3, golden["dib/theta0"])
    kin = (lambda u, v: orc.dib_rates(u, v, p)[0], lambda u, v: orc.dib_rates(u, v, p)[1])
    tau = 5e-3 / p["rho"]
    kw = dict(rule="residual", tol=1e-12, max_iter=2000) if tag == "t12" else {}
    tr = orc.imex_rds(x, y, 1.0, p["d_theta"], kin, p["rho"], (e0 - 1e-3, t0 - 1e-3), tau,
                      6 * tau, lumped=True, snapshot_every=2, **kw)
    assert np.array_equal(tr["iterations"], golden[f"dib/{tag}/iters"])
    assert [s[0] for s in tr["snapshots"]] == list(golden[f"dib/{tag}/snap_steps"])
    tolr = 1e-10 if tag == "t12" else 1e-8
    assert relerr(tr["final"][0], golden[f"dib/{tag}/U"]) <= tolr
    assert relerr(tr["final"][1], golden[f"dib/{tag}/V"]) <= tolr


def test_kinetics_and_initial_fields(golden):
    p = orc.dib_params(rho=400.0)
    f, g = orc.dib_rates(golden["kin/eta"], golden["kin/theta"], p)
    assert relerr(f, golden["kin/f"]) <= 1e-15 and relerr(g, golden["kin/g"]) <= 1e-15
    e, t = orc.initial_fields((6, 5), 1e-3, 7)
    assert np.array_equal(e, golden["init/eta"]) and np.array_equal(t, golden["init/theta"])


def test_known_answers():
    # reference tests: A=[4], M=[1/3] at N=2 (test_fem1d.py:59-62); Hadamard kernel (test_solvers.py:62-68)
    x, _ = orc.direction_sets(orc.unit_square(), 1, 2, orc.DIRICHLET)
    assert np.allclose(x["mats"]["A"], [[4.0]]) and np.allclose(x["mats"]["M"], [[1 / 3]])
    Z = np.diag([2.0, 3.0])
    U, _, _ = orc.reduced_solve([(Z, np.eye(2)), (np.eye(2), Z)], np.ones((2, 2)))
    assert np.allclose(U, [[1 / 4, 1 / 5], [1 / 5, 1 / 6]], atol=1e-14)


@pytest.mark.parametrize("gamma", [0, 1])
def test_closed_form_matches_reference(golden, gamma):
    tag = f"closed/g{gamma}"
    F = golden[f"{tag}/F"]
    U, res = orc.closed_form(float(gamma), F[1:-1, 1:-1], 16)
    assert relerr(U, golden[f"{tag}/U"]) <= 1e-13
    assert res <= 1e-13


@pytest.mark.parametrize("i", range(len(DESK_CASES)), ids=lambda i: str(DESK_CASES[i]))
def test_desk_matrix_matches_reference(golden, i):
    """reference tests/test_acceptance.py:109-148 on the oracle: apply,
    direct, reduced, closed form and MO-PCG against the reference's own
    outputs on the same seeded inputs."""
    k, n, name, bc = DESK_CASES[i]
    x, y, gamma, terms, rhs_of, pinv = desk_oracle(i)
    tag = f"desk/{i}"
    assert len(terms) == int(golden[f"{tag}/nterms"])
    assert relerr(orc.apply_terms(terms, golden[f"{tag}/U"]), golden[f"{tag}/AU"]) <= 1e-13
    rhs = rhs_of(golden[f"{tag}/F"])
    assert relerr(rhs, golden[f"{tag}/rhs"]) <= 1e-13
    direct = orc.direct_solve(terms, rhs)
    assert relerr(direct, golden[f"{tag}/direct"]) <= 1e-10
    if len(terms) == 2:
        U, _, _ = orc.reduced_solve(terms, rhs)
        assert relerr(U, golden[f"{tag}/reduced"]) <= 1e-10
        if f"{tag}/closed" in golden:
            F0 = golden[f"{tag}/F"].copy()
            F0[0, :] = F0[-1, :] = F0[:, 0] = F0[:, -1] = 0.0
            Uc, _ = orc.closed_form(gamma, F0[1:-1, 1:-1], n)
            assert relerr(Uc, golden[f"{tag}/closed"]) <= 1e-10
    it, lo, hi = orc.iteration_envelope(terms, rhs, pinv, ("residual", 1e-12), max_iter=5000)
    r = orc.mo_pcg(terms, rhs, pinv, ("residual", 1e-12), max_iter=5000)
    assert r["iterations"] == it and lo <= it <= hi
    assert abs(int(golden[f"{tag}/pcg_iters"]) - it) <= hi - lo + 1
    assert relerr(r["solution"], golden[f"{tag}/pcg"]) <= 1e-10
