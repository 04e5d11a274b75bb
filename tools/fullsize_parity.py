"""Full-size parity with a fixed iteration budget (SURVEY §8 c: "At full size
for cfg3-5, compare against a fixed-iteration-budget reference run
(max_iter=K, same U0/rhs)").

    python tools/fullsize_parity.py [cfg3 cfg4 cfg5] [--K 10]

For each config: the step-0 system is built both in the product (device) and
in the oracle (the reference restated, numpy/scipy on the host), K MO-PCG
iterations are run on each with the stop rule disabled, and the relative
difference of the K-th iterate and of the residual histories is printed as one
JSON line.  cfg4/cfg5 use the IMEX step-0 right-hand side and warm start U0.
The oracle is the checker here (test infrastructure), never the measured path.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle as orc  # noqa: E402
import paper_2109_01173_b200 as pb  # noqa: E402
from paper_2109_01173_b200 import workloads as wl  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def case(name, K, modes):
    t0 = time.perf_counter()
    w = wl.CONFIGS[name]()
    N = w.N
    if name == "cfg3":
        ox, oy = orc.direction_sets(orc.wave_domain(), 2, N, orc.DIRICHLET)
        terms, orhs = orc.elliptic_terms(ox, oy, 1.0)
        opre = orc.LUPrecond(*orc.precond_factors("elliptic_xnormal", ox, oy))
        rhs, u0 = w.rhs, None
        systems = [(w.op, "elliptic_xnormal", {}, terms, opre, rhs, u0)]
    elif name == "cfg4":
        ex = w.extra
        ox, oy = orc.direction_sets(orc.wave_domain(), 4, N, orc.DIRICHLET)
        terms, orhs = orc.parabolic_terms(ox, oy, 1.0, ex["tau"])
        opre = orc.LUPrecond(*orc.precond_factors("parabolic", ox, oy, d_u=1.0, tau=ex["tau"]))
        u0 = ex["u0"]
        Wf = orc.expand_full(u0, ox, oy) + ex["tau"] * ex["source"].F  # step 0: t = 0
        rhs = orhs(Wf)
        systems = [(w.op, "parabolic", {"d_u": 1.0, "tau": ex["tau"]}, terms, opre, rhs, u0)]
    else:
        ex = w.extra
        p, tau = ex["params"], ex["tau"]
        ox, oy = orc.direction_sets(orc.unit_square(), 1, N, orc.NEUMANN, lumped=True)
        eta0, th0 = ex["state0"]
        op_p = orc.dib_params(alpha=p.alpha, gamma_k=p.gamma_k, A1=p.A1, A2=p.A2, B=p.B, C=p.C, D=p.D, k2=p.k2,
                              k3=p.k3, d_theta=p.d_theta, rho=p.rho)
        f, g = orc.dib_rates(eta0, th0, op_p)
        systems = []
        for d, S, rate in ((1.0, eta0, f), (p.d_theta, th0, g)):
            terms, orhs = orc.parabolic_terms(ox, oy, d, tau, True)
            opre = orc.LUPrecond(*orc.precond_factors("parabolic_lumped", ox, oy, d_u=d, tau=tau, lumped=True))
            op_d, _ = pb.parabolic_operator(w.x, w.y, d, tau, lumped=True)
            systems.append((op_d, "parabolic_lumped", {"d_u": d, "tau": tau, "lumped": True}, terms, opre,
                            orhs(S + tau * p.rho * rate), S))
    setup = time.perf_counter() - t0
    out = []
    for si, (op, kind, kw, terms, opre, rhs, u0) in enumerate(systems):
        t1 = time.perf_counter()
        ref = orc.mo_pcg(terms, rhs, opre.inverse, ("residual", 1e-30), u0=u0, max_iter=K)
        t_ref = time.perf_counter() - t1
        for mode in modes:
            pre = pb.make_preconditioner(kind, w.x, w.y, mode=mode, **kw)
            rep = pb.mo_pcg(op, rhs, precond=pre, stop=pb.relative_residual(1e-30), u0=u0, max_iter=K)
            h = np.asarray(ref["history"]) if "history" in ref else None
            line = {"workload": name, "system": si, "q": list(op.shape), "K": K, "mode": mode,
                    "rel_diff_iterate_K": rel(rep.solution, ref["solution"]),
                    "iterations": [rep.iterations, ref["iterations"]],
                    "oracle_s": t_ref, "setup_s": setup}
            if h is not None:
                m = min(len(h), len(rep.residual_history))
                line["max_rel_diff_residual_history"] = float(np.max(np.abs(rep.residual_history[:m] - h[:m]) /
                                                                    np.abs(h[:m])))
            print(json.dumps(line), flush=True)
            out.append(line)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["cfg3", "cfg4", "cfg5"])
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--modes", default="inverse,banded")
    a = ap.parse_args()
    Ks = {"cfg3": 10, "cfg4": 3, "cfg5": 2}
    for c in a.configs:
        case(c, a.K or Ks[c], a.modes.split(","))
