"""Worker for the species-parallel IMEX tests (world size 2, gloo).

The step exchange, the ordered blow-up/convergence resolution and the
trajectory bookkeeping under test are the product's
(paper_2109_01173_b200.distributed.species_parallel_imex_rds).  On CPU the
local compute is a numpy stepper built from the oracle (test
infrastructure); on the GPU it is the product's CudaSpeciesStepper with the
state exchange staged through host memory."""

import os

import numpy as np
import torch
import torch.distributed as dist

import oracle as orc
import paper_2109_01173_b200 as pb
from paper_2109_01173_b200.distributed import SpeciesComm, species_parallel_imex_rds


def case(N=15, lumped=True):
    p = pb.dib_presets("spots_worms").replace(rho=400.0)
    x, y = pb.build_direction_sets(pb.SQUARE, 1, N, pb.BCKind.NEUMANN, lumped=lumped)
    e0, t0 = pb.initial_fields((y.q, x.q), pb.InitialData(amplitude=2e-3, seed=5))
    return p, x, y, (e0 - 1e-3, t0 - 1e-3), 5e-3 / p.rho


def oracle_kinetics(p):
    op = orc.dib_params(alpha=p.alpha, gamma_k=p.gamma_k, A1=p.A1, A2=p.A2, B=p.B, C=p.C, D=p.D,
                        k2=p.k2, k3=p.k3, d_theta=p.d_theta, rho=p.rho)
    return (lambda u, v: orc.dib_rates(u, v, op)[0], lambda u, v: orc.dib_rates(u, v, op)[1])


class OracleStepper:
    def __init__(self, N, blow):
        self.N, self.blow = N, blow

    def __call__(self, x, y, d, tau, rho, kinetics, inner, lumped, species):
        ox, oy = orc.direction_sets(orc.unit_square(), 1, self.N, orc.NEUMANN, lumped=True)
        self.terms, self.rhs_of = orc.parabolic_terms(ox, oy, d, tau, True)
        self.pre = orc.LUPrecond(*orc.precond_factors("parabolic_lumped", ox, oy, d_u=d, tau=tau, lumped=True))
        self.kin, self.species, self.tau, self.rho = kinetics, species, tau, rho
        self.rule = ("residual", tau if inner.rule == "tau" else inner.tol)
        self.max_iter = inner.max_iter
        return self

    def to_local(self, a):
        return torch.from_numpy(np.array(a, dtype=float, copy=True))

    def rhs(self, U, V):
        Uh, Vh = U.numpy(), V.numpy()
        W = (Uh if self.species == 0 else Vh) + self.tau * self.rho * np.asarray(self.kin[self.species](Uh, Vh))
        fin = np.isfinite(W)
        chk = (float(np.max(np.abs(W[fin]))) if fin.any() else 0.0, float((~fin).sum()))
        return self.rhs_of(W), chk

    def solve(self, rhs, warm):
        r = orc.mo_pcg(self.terms, rhs, self.pre.inverse, self.rule, u0=warm.numpy(), max_iter=self.max_iter)
        return torch.from_numpy(r["solution"]), r["iterations"], r["reason"] != "max_iter"

    def norms(self, A, B):
        a, b = A.numpy(), B.numpy()
        return [float(np.linalg.norm(a - b)), float(np.max(np.abs(a[np.isfinite(a)]), initial=0.0)),
                float((~np.isfinite(a)).sum()), float(np.linalg.norm(a))]

    def host(self, X):
        return X.numpy().copy()


class HostStagedSpeciesComm(SpeciesComm):
    """SpeciesComm over gloo for CUDA states (one GPU, ranks meet on the host)."""

    def exchange(self, own):
        parts = super().exchange(own.cpu())
        return [p.to(own.device) for p in parts]


def worker(rank, world, port, mode, out_dir, N, steps, blow):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, x, y, state0, tau = case(N)
        inner = pb.InnerSolver(rule="residual", tol=1e-12, max_iter=2000)
        if mode == "cpu":
            kin = oracle_kinetics(p)
            if blow:
                kin = (lambda u, v: 1e300 * (1.0 + u ** 2), kin[1]) if blow == "u" else \
                    (kin[0], lambda u, v: 1e300 * (1.0 + v ** 2))
            comm, factory = SpeciesComm("cpu"), OracleStepper(N, blow)
        else:
            torch.cuda.set_device(0)
            kin = pb.dib_kinetics_pair(p)
            comm, factory = HostStagedSpeciesComm("cpu"), None
        try:
            tr = species_parallel_imex_rds(pb.SQUARE, x, y, 1.0, p.d_theta, kin, p.rho, state0,
                                           pb.TimeGrid(tau, steps * tau), inner=inner, lumped=True,
                                           snapshot_every=2, comm=comm, stepper_factory=factory)
            np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=tr.final[0], V=tr.final[1],
                     iters=tr.iterations, incs=tr.increments, snaps=[s[0] for s in tr.snapshots],
                     steady=-1 if tr.steady_step is None else tr.steady_step, err="")
        except pb.BlowUpError as e:
            np.savez(os.path.join(out_dir, f"rank{rank}.npz"), err=f"blowup {e.step} {e.species}",
                     U=e.state[0], V=e.state[1])
    finally:
        dist.destroy_process_group()
