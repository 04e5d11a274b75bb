"""cProfile of a full IMEX run with the two-term preconditioner: python tools/imex_prof.py cfg4|cfg5 N steps"""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2109_01173_b200 as pb
from paper_2109_01173_b200 import workloads as wl
name = sys.argv[1]; N = int(sys.argv[2]); steps = int(sys.argv[3])
w = wl.CONFIGS[name](N=N, mode="inverse", steps=steps)
ex = w.extra
def run():
    if name == "cfg4":
        inner = pb.InnerSolver(rule="residual", tol=1e-8, max_iter=100000, precond="two_term")
        return pb.imex_euler_heat(wl.WAVE, w.x, w.y, 1.0, ex["source"], ex["u0"], ex["grid"], inner=inner)
    p = ex["params"]
    inner = pb.InnerSolver(max_iter=100000, precond="two_term")
    return pb.imex_euler_rds(pb.SQUARE, w.x, w.y, 1.0, p.d_theta, ex["kinetics"], p.rho, ex["state0"], ex["grid"], inner=inner, lumped=True)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable(); t0 = time.perf_counter()
tr = run(); torch.cuda.synchronize()
pr.disable(); print("total", time.perf_counter() - t0, "iters", tr.iterations)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
