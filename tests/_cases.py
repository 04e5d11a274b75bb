"""Shared seeded inputs of the BASELINE.json configurations,
restated for the tests so they do not depend on the product package."""

import numpy as np

import oracle as orc

ODOMS = {"square": orc.unit_square, "cap": orc.cap_domain, "jar": orc.jar_domain,
         "wave": orc.wave_domain, "rect": orc.rect_domain}
OBC = {"d": orc.DIRICHLET, "n": orc.NEUMANN}


def sine_source(N_x, N_y, seed):
    a, b, c = orc.seeded_modes(seed)
    xs = np.arange(N_x + 1) / N_x
    ys = np.arange(N_y + 1) / N_y
    return sum(c[m] * np.sin(b[m] * np.pi * ys)[:, None] * np.sin(a[m] * np.pi * xs)[None, :]
               for m in range(8))


def cosine_source_rect(N, seed):
    a, b, c = orc.seeded_modes(seed)
    X = 2.0 * np.arange(N + 1) / N
    Y = np.arange(N + 1) / N
    return sum(c[m] * np.cos(b[m] * np.pi * Y)[:, None] * np.cos(a[m] * np.pi * X / 2)[None, :]
               for m in range(8))


ASM_CASES = [(1, 8, "square", "d"), (2, 8, "cap", "n"), (3, 12, "jar", "d"),
             (4, 8, "wave", "d"), (3, 12, "rect", "n"), (2, 10, "wave", "n")]
OP_CASES = [("ell", 1, 8, "square", "d", 0.0, False), ("ell", 2, 8, "cap", "d", 0.0, False),
            ("ell", 3, 12, "jar", "n", 1.0, False), ("ell", 2, 10, "wave", "d", 1.0, False),
            ("ell", 1, 8, "cap", "n", 1.0, True), ("ell", 1, 8, "jar", "d", 0.0, True),
            ("ell", 3, 12, "rect", "n", 0.5, False),
            ("par", 4, 8, "wave", "d", 1e-3, False), ("par", 1, 9, "square", "n", 0.05, True),
            ("par", 2, 8, "cap", "n", 0.01, False)]


def desk_cases():
    """(k, N, domain, bc) of the reference's acceptance desk matrix
    (reference tests/conftest.py:12-22; same order as make_golden.py)."""
    out = []
    for k in (1, 2, 3, 4):
        for n in (8, 16, 24):
            if n % k:
                continue
            for name in ("square", "cap", "jar"):
                for bc in ("d", "n"):
                    out.append((k, n, name, bc))
    return out


DESK_CASES = desk_cases()


def desk_oracle(i):
    """The oracle's term list, rhs map and MO-PCG preconditioner of desk case
    i, built as reference tests/test_acceptance.py:112-148 builds them."""
    k, n, name, bc = DESK_CASES[i]
    x, y = orc.direction_sets(ODOMS[name](), k, n, OBC[bc], lumped=k == 1)
    gamma = 0.0 if bc == "d" else 1.0
    terms, rhs_of = orc.elliptic_terms(x, y, gamma)
    if bc == "d":
        pre = orc.LUPrecond(*orc.precond_factors("elliptic_square" if name == "square" else "elliptic_xnormal", x, y))
        pinv = pre.inverse
    else:
        pinv = None
    return x, y, gamma, terms, rhs_of, pinv


def wave_oracle(k, N, gamma=1.0, seed=3, lumped=False):
    """Oracle term list, seeded-sine rhs and elliptic_xnormal LU inverse of
    the cfg3-type problem (wave domain, Dirichlet) at any size."""
    ox, oy = orc.direction_sets(orc.wave_domain(), k, N, orc.DIRICHLET, lumped=lumped)
    terms, orhs = orc.elliptic_terms(ox, oy, gamma)
    Nx, Ny = (N, N) if np.isscalar(N) else N
    pre = orc.LUPrecond(*orc.precond_factors("elliptic_xnormal", ox, oy, lumped=lumped))
    return terms, orhs(sine_source(Nx, Ny, seed)), pre.inverse
