"""Small end-to-end exercise of every kernel family (a quick health check
after kernel changes; compute-sanitizer is not available on this pool):

    python tools/health_probe.py

cfg3-type MO-PCG in the three preconditioner modes (banded operator pass,
deferred U, DMMA GEMMs, SPIKE tiles and chains), a reduced solve, a native
DIB IMEX run with snapshots and a PGM frame — all at desk sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2109_01173_b200 as pb  # noqa: E402
from paper_2109_01173_b200.outputs import pgm_pixels  # noqa: E402

WAVE = pb.DomainSpec(pb.DomainKind.XNORMAL, pb.ProfileFn(
    lambda s: 1.0 + 0.3 * np.sin(2 * np.pi * np.asarray(s, float)),
    lambda s: 0.6 * np.pi * np.cos(2 * np.pi * np.asarray(s, float)), name="wave"))

N = int(os.environ.get("PROBE_N", "40"))
x, y = pb.build_direction_sets(WAVE, 2, N, pb.BCKind.DIRICHLET)
op, rhs_of = pb.elliptic_operator(x, y, 1.0)
rng = np.random.default_rng(0)
rhs = rng.standard_normal(op.shape)
for mode in ("inverse", "banded", "spectral"):
    pre = pb.make_preconditioner("elliptic_xnormal", x, y, mode=mode)
    r = pb.mo_pcg(op, rhs, precond=pre, stop=pb.relative_residual(1e-30), max_iter=12,
                  u0=1e-2 * rng.standard_normal(op.shape))
    print(mode, r.iterations, r.residual_history[-1])
xs, ys = pb.build_direction_sets(pb.SQUARE, 1, 33, pb.BCKind.DIRICHLET)
ops, rhs_s = pb.elliptic_operator(xs, ys, 1.0)
print("reduced", pb.solve_reduced(ops, rng.standard_normal(ops.shape)).residual_history[0])
p = pb.dib_presets("spots_worms").replace(rho=400.0)
xn, yn = pb.build_direction_sets(pb.SQUARE, 1, 23, pb.BCKind.NEUMANN, lumped=True)
e0, t0 = pb.initial_fields((yn.q, xn.q), pb.InitialData(amplitude=2e-3, seed=5))
tr = pb.imex_euler_rds(pb.SQUARE, xn, yn, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho, (e0, t0),
                       pb.TimeGrid(1.25e-5, 4 * 1.25e-5), lumped=True, snapshot_every=2)
print("rds", tr.iterations.tolist())
px, lohi = pgm_pixels(tr.final[0])
print("pgm", px.shape, lohi)
