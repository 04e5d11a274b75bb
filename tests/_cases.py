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
