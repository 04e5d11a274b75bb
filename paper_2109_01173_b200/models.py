"""Two-species electrodeposition (DIB) kinetics, parameters and initial data
(models.py:19-126 of the reference).

``dib_kinetics`` is the entrywise host evaluation the reference exposes; the
IMEX driver evaluates the same polynomials on the device, fused into the
rhs pass, when it is handed a ``DIBKinetics`` pair (``dib_kinetics_pair``).
"""

from __future__ import annotations

from dataclasses import dataclass
from dataclasses import replace as _replace

import numpy as np

from .exceptions import ConfigError

EQUILIBRIUM = (0.0, 0.5)


def equilibrium_consistent_D(C: float, alpha: float, gamma_k: float) -> float:
    """D making (0, alpha) an equilibrium: g(0, alpha) = 0 (models.py:19-28)."""
    return C * (1 - alpha) * (1 - gamma_k * (1 - alpha)) / (alpha * (1 + gamma_k * alpha))


@dataclass(frozen=True)
class DIBParams:
    """Kinetics parameters; D slaved to C when unset (models.py:31-71)."""

    alpha: float = 0.5
    gamma_k: float = 0.2
    A1: float = 10.0
    A2: float = 30.0
    B: float = 25.0
    C: float = 7.0
    D: float | None = None
    k2: float = 2.5
    k3: float = 1.5
    d_theta: float = 20.0
    rho: float = 400.0

    def __post_init__(self):
        if self.D is None:
            object.__setattr__(self, "D", equilibrium_consistent_D(self.C, self.alpha, self.gamma_k))
        for name in ("alpha", "gamma_k", "A1", "A2", "B", "C", "D", "k2", "k3", "d_theta", "rho"):
            if getattr(self, name) <= 0:
                raise ConfigError(f"kinetics parameter {name} must be positive")
        if not 0 < self.alpha < 1:
            raise ConfigError("alpha must lie in (0, 1)")
        if not 0 < self.gamma_k < 1:
            raise ConfigError("gamma_k must lie in (0, 1)")

    def replace(self, **kw) -> "DIBParams":
        return _replace(self, **kw)

    def device_params(self) -> np.ndarray:
        """{alpha, gamma_k, A1, A2, B, C, D, k2, k3} for the fused device kernel."""
        return np.array([self.alpha, self.gamma_k, self.A1, self.A2, self.B, self.C, self.D,
                         self.k2, self.k3], dtype=float)


def dib_kinetics(eta, theta, p: DIBParams):
    """Entrywise rates (f, g) (models.py:74-82)."""
    eta = np.asarray(eta, dtype=float)
    theta = np.asarray(theta, dtype=float)
    f = p.A1 * (1.0 - theta) * eta - p.A2 * eta ** 3 - p.B * (theta - p.alpha)
    g = (p.C * (1.0 + p.k2 * eta) * (1.0 - theta) * (1.0 - p.gamma_k * (1.0 - theta))
         - p.D * theta * (1.0 + p.gamma_k * theta) * (1.0 + p.k3 * eta))
    return f, g


class DIBKinetics(tuple):
    """(f, g) pair of the DIB model that the IMEX driver recognises and
    evaluates on the device; still callable on the host like any pair."""

    def __new__(cls, params: DIBParams):
        f = lambda u, v: dib_kinetics(u, v, params)[0]  # noqa: E731
        g = lambda u, v: dib_kinetics(u, v, params)[1]  # noqa: E731
        obj = super().__new__(cls, (f, g))
        obj.params = params
        return obj


def dib_kinetics_pair(params: DIBParams) -> DIBKinetics:
    return DIBKinetics(params)


_PRESETS = {
    "spots_worms": DIBParams(A2=30.0, B=25.0, C=7.0),
    "holes": DIBParams(A2=1.0, B=30.0, C=3.0),
}


def dib_presets(name: str) -> DIBParams:
    try:
        return _PRESETS[name]
    except KeyError:
        raise ConfigError(f"unknown kinetics preset '{name}' (have: {sorted(_PRESETS)})") from None


@dataclass(frozen=True)
class InitialData:
    """Philox4x64-seeded perturbation of the equilibrium (models.py:103-115)."""

    amplitude: float = 1e-4
    seed: int = 20240

    def generator(self) -> np.random.Generator:
        return np.random.Generator(np.random.Philox(key=self.seed))


def initial_fields(shape, data: InitialData):
    """Equilibrium + amplitude * U[0,1) for both species (models.py:118-126)."""
    qy, qx = int(shape[0]), int(shape[1])
    if qy <= 0 or qx <= 0:
        raise ConfigError("grid dimensions must be positive")
    rng = data.generator()
    eta = EQUILIBRIUM[0] + data.amplitude * rng.random((qy, qx))
    theta = EQUILIBRIUM[1] + data.amplitude * rng.random((qy, qx))
    return eta, theta


def effective_domain_size(domain, rho: float) -> float:
    return float(rho) * domain.area()
