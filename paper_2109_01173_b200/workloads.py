"""The five BASELINE.json configurations expressed in the drop-in API.

Seeded synthetic inputs exactly as SURVEY App. A specifies (no dataset is
involved): ``rng = default_rng(seed)``; a, b = rng.integers(1, 17, 8) drawn in
that order, then c = rng.standard_normal(8); F is an 8-mode sine (or cosine)
product sampled on the full node grid.  Inadmissible sizes are replaced as
the survey prescribes (q = 2047 / 4095 instead of 2048 / 4096).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .fem1d import BCKind, build_direction_sets
from .geometry import SQUARE, DomainKind, DomainSpec, ProfileFn
from .models import InitialData, dib_kinetics_pair, dib_presets, initial_fields
from .operators import elliptic_operator, full_node_grid, parabolic_operator
from .solvers import make_preconditioner, relative_residual
from .timestepping import InnerSolver, SeparableSource, TimeGrid

WAVE = DomainSpec(DomainKind.XNORMAL, ProfileFn(
    lambda s: 1.0 + 0.3 * np.sin(2 * np.pi * np.asarray(s, float)),
    lambda s: 0.6 * np.pi * np.cos(2 * np.pi * np.asarray(s, float)), name="wave"), name="wave")
RECT2 = DomainSpec(DomainKind.XNORMAL, ProfileFn(
    lambda s: 2.0 * np.ones_like(np.asarray(s, float)),
    lambda s: np.zeros_like(np.asarray(s, float)), name="rect2"), name="rect")

FULL_N = {"cfg1": 257, "cfg2": 1023, "cfg3": 2048, "cfg4": 4096, "cfg5": 8191}


def seeded_modes(seed: int, n_modes: int = 8):
    rng = np.random.default_rng(seed)
    a = rng.integers(1, 17, n_modes)
    b = rng.integers(1, 17, n_modes)
    c = rng.standard_normal(n_modes)
    return a, b, c


def sine_source(N_x: int, N_y: int, seed: int) -> np.ndarray:
    """F[i, j] = sum_m c_m sin(b_m pi y_i) sin(a_m pi x_j) on reference nodes."""
    a, b, c = seeded_modes(seed)
    xs = np.arange(N_x + 1) / N_x
    ys = np.arange(N_y + 1) / N_y
    F = np.zeros((N_y + 1, N_x + 1))
    for m in range(8):
        F += c[m] * np.sin(b[m] * np.pi * ys)[:, None] * np.sin(a[m] * np.pi * xs)[None, :]
    return F


def cosine_source_rect(N: int, seed: int) -> np.ndarray:
    """F = sum_m c_m cos(a_m pi x / 2) cos(b_m pi y) at the physical nodes of [0,2]x[0,1]."""
    a, b, c = seeded_modes(seed)
    X = 2.0 * np.arange(N + 1) / N
    Y = np.arange(N + 1) / N
    F = np.zeros((N + 1, N + 1))
    for m in range(8):
        F += c[m] * np.cos(b[m] * np.pi * Y)[:, None] * np.cos(a[m] * np.pi * X / 2)[None, :]
    return F


@dataclass
class Workload:
    name: str
    N: int
    k: int
    x: object
    y: object
    op: object
    rhs_of: object
    rhs: np.ndarray | None = None
    precond: object = None
    stop: object = None
    extra: dict = field(default_factory=dict)

    @property
    def q(self):
        return self.op.shape


def cfg1(N: int | None = None) -> Workload:
    """Square, P1, Dirichlet, gamma = 1, reduced solve (configs[0])."""
    N = N or FULL_N["cfg1"]
    x, y = build_direction_sets(SQUARE, 1, N, BCKind.DIRICHLET)
    op, rhs_of = elliptic_operator(x, y, 1.0)
    return Workload("cfg1", N, 1, x, y, op, rhs_of, rhs_of(sine_source(N, N, 1)))


def cfg2(N: int | None = None) -> Workload:
    """[0,2]x[0,1], P3, Neumann, gamma = 0.5, reduced solve (configs[1])."""
    N = N or FULL_N["cfg2"]
    x, y = build_direction_sets(RECT2, 3, N, BCKind.NEUMANN)
    op, rhs_of = elliptic_operator(x, y, 0.5)
    return Workload("cfg2", N, 3, x, y, op, rhs_of, rhs_of(cosine_source_rect(N, 2)))


def cfg3(N: int | None = None, mode: str | None = None, tol: float = 1e-8) -> Workload:
    """Wave domain, P2, Dirichlet, gamma = 1, MO-PCG with the single-term
    elliptic_xnormal preconditioner, relative residual 1e-8 (configs[2])."""
    N = N or FULL_N["cfg3"]
    x, y = build_direction_sets(WAVE, 2, N, BCKind.DIRICHLET)
    op, rhs_of = elliptic_operator(x, y, 1.0)
    pre = make_preconditioner("elliptic_xnormal", x, y, mode=mode)
    return Workload("cfg3", N, 2, x, y, op, rhs_of, rhs_of(sine_source(N, N, 3)), pre,
                    relative_residual(tol))


def cfg4(N: int | None = None, mode: str | None = None, tol: float = 1e-8, steps: int = 100) -> Workload:
    """Heat on the wave domain, P4, Dirichlet, IMEX tau = 1e-3, 100 steps,
    source e^{-t} F, u0 = 1e-2 N(0,1) (configs[3])."""
    N = N or FULL_N["cfg4"]
    tau = 1e-3
    x, y = build_direction_sets(WAVE, 4, N, BCKind.DIRICHLET)
    op, rhs_of = parabolic_operator(x, y, 1.0, tau)
    pre = make_preconditioner("parabolic", x, y, d_u=1.0, tau=tau, mode=mode)
    F = sine_source(N, N, 4)
    u0 = 1e-2 * np.random.default_rng(4).standard_normal((y.q, x.q))
    src = SeparableSource(F, lambda t: float(np.exp(-t)))
    return Workload("cfg4", N, 4, x, y, op, rhs_of, None, pre, relative_residual(tol),
                    extra={"tau": tau, "grid": TimeGrid(tau, steps * tau), "source": src, "u0": u0,
                           "inner": InnerSolver(rule="residual", tol=tol, max_iter=100000, precond_mode=mode)})


def cfg5(N: int | None = None, mode: str | None = None, steps: int = 200) -> Workload:
    """Two-species DIB on the unit square, lumped P1, Neumann, rho = 400,
    d_theta = 20, tau_ref = 5e-3/400, reference tau rule (configs[4])."""
    N = N or FULL_N["cfg5"]
    p = dib_presets("spots_worms").replace(rho=400.0)
    tau = 5e-3 / p.rho
    x, y = build_direction_sets(SQUARE, 1, N, BCKind.NEUMANN, lumped=True)
    op, rhs_of = parabolic_operator(x, y, 1.0, tau, lumped=True)
    e0, t0 = initial_fields((y.q, x.q), InitialData(amplitude=2e-3, seed=5))
    return Workload("cfg5", N, 1, x, y, op, rhs_of, None, None, None,
                    extra={"params": p, "tau": tau, "grid": TimeGrid(tau, steps * tau),
                           "state0": (e0 - 1e-3, t0 - 1e-3), "kinetics": dib_kinetics_pair(p),
                           "inner": InnerSolver(precond_mode=mode, max_iter=100000)})


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


def physical_source_grid(w: Workload):
    return full_node_grid(WAVE, w.x, w.y)
