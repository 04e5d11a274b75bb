#!/usr/bin/env python
"""MO-PCG DoF*iterations/s (fp64) on B200 — the BASELINE.json headline metric.

Workload (default): BASELINE configs[4] ("cfg5"), the config the metric is
quoted on at 1/2/4/8 GPUs and the largest that fits one B200: the two-species
DIB reaction-diffusion system on the unit square, lumped P1, Neumann,
N = 8191 (q = 8192 per species), spots_worms kinetics with rho = 400,
d_theta = 20, tau_ref = 5e-3/400, App. A initial state.  One "step" is one
IMEX step (timestepping.py:200-218) through the drop-in ``imex_euler_rds``
(native step loop): both species' fused kinetics+rhs pass, each species'
MO-PCG warm started from its state with the reference's single-term
preconditioner as two DMMA GEMMs (north star), the increment norms.  Each
solve runs a fixed inner budget of --iters-per-step iterations
(``InnerSolver(rule="budget")``: no stop test, so every step does the same
work).  DoF*it/s = q_y q_x * (MO-PCG iterations of both species) / seconds.

Printed (rank 0, one JSON line): value (states resident in HBM), e2e (numpy
states in from page-locked memory and out, H2D/D2H inside the timed
region), roofline of the dominant kernel (the 8192^3 DMMA GEMM of the
preconditioner, live CUDA events, against cuBLAS DGEMM measured in the same
run) and roofline_hbm of the banded MO-PCG pass and the R update at
q = 8192, cpu_baseline (the oracle port of the reference on the host cores:
both species' step-0 systems, 2 MO-PCG iterations each, SURVEY §8 d),
clocks, the banded-preconditioner (f1) alternative, and a short cfg3 block
(configs[2], MO-PCG elliptic, q = 2047).  Under torchrun (N > 1) the step
is split over the ranks (species-parallel at N = 2, species groups with
column-sharded MO-PCG at N = 4 / 8).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload cfg5|cfg3]
"""

from __future__ import annotations

import argparse
import json
import os
import signal
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MO-PCG DoF*iterations/s (fp64)"
UNIT = "DoF*iterations/s"
FP64_PEAK_FALLBACK = 35.48  # cuBLAS DGEMM 8192^3 measured on this pool (profiles/fp64_peaks_r01.log)
DATA = "synthetic (seeded App. A inputs: Philox initial state / 8-mode sine source; no dataset involved)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--workload", choices=["cfg5", "cfg3"], default="cfg5")
    ap.add_argument("--N", type=int, default=None, help="subintervals (default: the BASELINE size)")
    ap.add_argument("--iters-per-step", type=int, default=None,
                    help="MO-PCG budget per solve (cfg5: per species and step, default 20; cfg3: default 200)")
    ap.add_argument("--precond-mode", default="inverse", choices=["inverse", "spectral", "banded"])
    ap.add_argument("--strassen-levels", type=int, default=None,
                    help="Strassen levels of the inverse-form preconditioner products (default: the library's, "
                         "3 at q = 8192; 0 = classic GEMMs)")
    ap.add_argument("--no-classic", action="store_true", help="skip the classic-GEMM-schedule comparison block")
    ap.add_argument("--cpu-iters", type=int, default=2, help="oracle iterations per system in cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the banded-preconditioner (f1) measurement")
    ap.add_argument("--no-secondary", action="store_true", help="skip the cfg3 block of the cfg5 line")
    ap.add_argument("--no-full", action="store_true", help="cfg3: skip the full solves to 1e-8")
    ap.add_argument("--transposes", default="peer", choices=["peer", "nccl"],
                    help="cfg3 N > 1: preconditioner transposes over peer memory or NCCL all-to-alls")
    a = ap.parse_args()
    if a.iters_per_step is None:
        a.iters_per_step = 20 if a.workload == "cfg5" else 200
    if a.N is None:
        a.N = 8191 if a.workload == "cfg5" else 2048
    return a


# ------------------------------------------------------------------ clocks --
class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.25)
        self.proc.send_signal(signal.SIGTERM)
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        try:
            for line in open(self.path):
                f = [c.strip() for c in line.split(",")]
                if len(f) >= 8 and f[0].replace(".", "").isdigit():
                    rows.append(f)
        finally:
            os.unlink(self.path)
        if not rows:
            return out
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        out.update(sm_mhz=statistics.median(sm), sm_max_mhz=float(rows[0][1]), reasons=reasons,
                   samples=len(rows), power_w_max=max(float(r[2]) for r in rows if r[2] not in ("", "[N/A]")))
        return out


# ---------------------------------------------------------- host helpers ----
def host_stack() -> str:
    """numpy / scipy / BLAS of the host baseline (SURVEY §8 d protocol)."""
    import scipy
    blas = "BLAS unknown"
    try:
        from threadpoolctl import threadpool_info
        for lib in threadpool_info():
            if lib.get("user_api") == "blas":
                blas = f"{lib.get('internal_api')} {lib.get('version')} ({lib.get('num_threads')} threads)"
                break
    except Exception:
        pass
    return f"numpy {np.__version__}, scipy {scipy.__version__}, {blas}"


def cores() -> int:
    try:
        from threadpoolctl import threadpool_info
        for lib in threadpool_info():
            if lib.get("user_api") == "blas" and lib.get("num_threads"):
                return int(lib["num_threads"])
    except Exception:
        pass
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(k, "").isdigit():
            return int(os.environ[k])
    return os.cpu_count() or 1


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def hbm_peak():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        if mp.get("hbm_gbs"):
            return float(mp["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except (OSError, ValueError):
        pass
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def profile_json(name):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", name)))
    except (OSError, ValueError):
        return {}


# -------------------------------------------------------------- oracle legs --
def oracle_cfg5(N: int):
    """The two step-0 systems of cfg5 in the oracle (the reference restated:
    dense lumped-P1 assembly, dense term list, LU preconditioner), built
    exactly as imex_euler_rds's first step builds them (timestepping.py:
    184-209): rhs = M (S + tau rho kin(eta0, theta0)), warm start S."""
    import oracle as orc
    p = orc.dib_params(rho=400.0)  # spots_worms with D slaved to C (models.py:19-28, 85-90)
    tau = 5e-3 / p["rho"]
    x, y = orc.direction_sets(orc.unit_square(), 1, N, orc.NEUMANN, lumped=True)
    q = x["q"]
    e0, t0 = orc.initial_fields((q, q), 2e-3, 5)
    e0, t0 = e0 - 1e-3, t0 - 1e-3  # (0, 0.5) +- 1e-3
    f, g = orc.dib_rates(e0, t0, p)
    systems = []
    for d, S, rate in ((1.0, e0, f), (p["d_theta"], t0, g)):
        terms, rhs_of = orc.parabolic_terms(x, y, d, tau, True)
        pre = orc.LUPrecond(*orc.precond_factors("parabolic_lumped", x, y, d_u=d, tau=tau, lumped=True))
        systems.append((terms, pre, rhs_of(S + tau * p["rho"] * rate), S))
    return orc, systems, q


def oracle_cfg3(N: int):
    import oracle as orc
    x, y = orc.direction_sets(orc.wave_domain(), 2, N, orc.DIRICHLET)
    terms, rhs_of = orc.elliptic_terms(x, y, 1.0)
    pre = orc.LUPrecond(*orc.precond_factors("elliptic_xnormal", x, y))
    a, b, c = orc.seeded_modes(3)
    s = np.arange(N + 1) / N
    F = sum(c[m] * np.sin(b[m] * np.pi * s)[:, None] * np.sin(a[m] * np.pi * s)[None, :] for m in range(8))
    return orc, [(terms, pre, rhs_of(F), None)], x["q"]


def oracle_systems(workload: str, N: int):
    return oracle_cfg5(N) if workload == "cfg5" else oracle_cfg3(N)


def cpu_sample(workload: str, N: int, iters: int):
    """Time `iters` oracle MO-PCG iterations on each step-0 system (setup --
    assembly, terms, LU factorisation, initial residual and first
    preconditioner apply -- excluded; each iteration = operator apply,
    updates, preconditioner apply, as in the device loop)."""
    t0 = time.perf_counter()
    orc, systems, q = oracle_systems(workload, N)
    gens = [orc.pcg_iterations(terms, rhs, pre.inverse, u0=S) for terms, pre, rhs, S in systems]
    for gen in gens:  # the setup part (R0, Z0) of each solve
        next(gen)
    setup = time.perf_counter() - t0
    wall, n = 0.0, 0
    for gen in gens:
        for _ in range(iters):
            t1 = time.perf_counter()
            next(gen)
            wall += time.perf_counter() - t1
            n += 1
    return q * q * n / wall, wall, setup, n, len(systems)


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (the oracle port; the
    reference is pure Python and cannot travel to the GPU box) on the same
    workload, all host threads.  One step = one MO-PCG iteration of a
    step-0 system (cfg5 alternates the two species), continuing the same
    solve, so every timed step does exactly one iteration's work."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    t0 = time.perf_counter()
    orc, systems, q = oracle_systems(args.workload, args.N)
    gens = [orc.pcg_iterations(terms, rhs, pre.inverse, u0=S) for terms, pre, rhs, S in systems]
    for gen in gens:  # the setup part (R0, Z0) of each solve
        next(gen)
    k = 0
    for _ in range(args.warmup):
        next(gens[k % len(gens)])
        k += 1
    setup = time.perf_counter() - t0
    t1 = time.perf_counter()
    for _ in range(args.steps):
        next(gens[k % len(gens)])
        k += 1
    dt = time.perf_counter() - t1
    value = q * q * args.steps / dt
    wl_name = (f"cfg5 (BASELINE configs[4]) DIB two species, lumped P1 Neumann, N={args.N} q={q}"
               if args.workload == "cfg5" else
               f"cfg3 (BASELINE configs[2]) wave domain P2 Dirichlet, N={args.N} q={q}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": {"workload": wl_name, "step": "one MO-PCG iteration of a step-0 system"
                   + (" (species alternate)" if len(systems) > 1 else ""),
                   "parallelism": "host BLAS threads", "setup_s": round(setup, 1)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "port",
                         "sample": f"oracle restatement of sylfem mo_pcg (dense GEMM apply, LU preconditioner), "
                                   f"{args.steps} iterations after {args.warmup} warm-up iterations on the "
                                   f"step-0 system(s); setup excluded",
                         "host_stack": host_stack()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU pieces ----
def strassen_leaf(q: int, levels: int) -> int:
    """Leaf dimension of the Strassen schedule (odd shapes are padded to a multiple of 2^(levels+1))."""
    unit = 2 << levels
    return ((q + unit - 1) // unit * unit) >> levels


def gemm_roofline(q: int, levels: int = 0):
    """Dominant kernel: the q x q x q DMMA GEMM (C = A Bt^T), live CUDA
    events on the launching stream, against cuBLAS DGEMM 8192^3 measured in
    the same process."""
    import torch
    from paper_2109_01173_b200 import _native as nat
    L = nat.lib()
    ld = q + (q % 2)
    A = torch.randn(q, ld, dtype=torch.float64, device="cuda")
    B = torch.randn(q, ld, dtype=torch.float64, device="cuda")
    C = torch.empty(q, ld, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()

    def gemm():
        nat.check(L.sfb_dgemm_nt(A.data_ptr(), ld, B.data_ptr(), ld, q, q, q, C.data_ptr(), ld, s.cuda_stream))

    def timed(fn, reps):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / reps

    reps = max(3, min(20, int(2e12 / (2.0 * q ** 3))))
    t_gemm = timed(gemm, reps)
    del A, B, C
    n8 = 8192
    a8 = torch.randn(n8, n8, dtype=torch.float64, device="cuda")
    b8 = torch.randn(n8, n8, dtype=torch.float64, device="cuda")
    peak = 2.0 * n8 ** 3 / timed(lambda: a8 @ b8, 3) / 1e12
    cublas_same = None
    if q != n8:
        a = torch.randn(q, q, dtype=torch.float64, device="cuda")
        b = torch.randn(q, q, dtype=torch.float64, device="cuda")
        cublas_same = 2.0 * q ** 3 / timed(lambda: a @ b.T, reps) / 1e12
        del a, b
    else:
        cublas_same = peak
    del a8, b8
    torch.cuda.empty_cache()
    tf = 2.0 * q ** 3 / t_gemm / 1e12
    roof = {"bound": "tensor", "kernel": "dgemm_nt (DMMA.8x8x4 + TMA, stream-K)", "achieved": tf, "peak": peak,
            "unit": "TFLOP/s", "frac": tf / peak, "flops_per_launch": 2.0 * q ** 3, "launch_ms": t_gemm * 1e3,
            "peak_source": "cuBLAS DGEMM 8192^3 measured in this run", "cublas_same_shape_tflops": cublas_same}
    if levels > 0:
        # the dominant kernel of the Strassen schedule: one batched launch of the
        # seven leaf products (its own flops, not the algorithmic 2 q^3)
        h = strassen_leaf(q, levels)
        nb = 7 ** levels  # all leaf products of a preconditioner product are one strided-batch launch
        A = torch.randn(nb, h, h, dtype=torch.float64, device="cuda")
        B = torch.randn(nb, h, h, dtype=torch.float64, device="cuda")
        out = torch.empty(nb, h, h, dtype=torch.float64, device="cuda")

        def leaf():
            nat.check(L.sfb_dgemm_nt_batch(nb, A.data_ptr(), h, B.data_ptr(), h, h, h, h, out.data_ptr(), h, h * h,
                                           s.cuda_stream))

        t_leaf = timed(leaf, 10)
        tfl = 2.0 * nb * h ** 3 / t_leaf / 1e12
        roof = {"bound": "tensor",
                "kernel": f"dgemm_nt strided batch ({nb} x {h}^3 per launch: the leaf products of {levels} Strassen "
                          f"levels; DMMA.8x8x4 + rank-3 TMA maps, hybrid data-parallel + stream-K)",
                "achieved": tfl, "peak": peak, "unit": "TFLOP/s", "frac": tfl / peak,
                "flops_per_launch": 2.0 * nb * h ** 3, "launch_ms": t_leaf * 1e3,
                "launches_per_product": 1,
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run",
                "classic_gemm": {"kernel": "dgemm_nt, one q^3 product per launch", "achieved": tf, "frac": tf / peak,
                                 "launch_ms": t_gemm * 1e3, "flops_per_launch": 2.0 * q ** 3,
                                 "cublas_same_shape_tflops": cublas_same}}
        del A, B, out
        torch.cuda.empty_cache()
    return roof


def hbm_passes(op, pre, reps=20):
    """Banded MO-PCG pass and R update of one iteration, per launch, on the
    solver mo_pcg built for (op, pre) (SURVEY §8 d: 48 B/elem and 24 B/elem)."""
    import paper_2109_01173_b200 as pb
    pt = pb.solvers.pcg_pass_times(op, pre, reps=reps)
    peak, src = hbm_peak()
    qy, qx = op.shape
    ld = qx + (-qx % 32)
    n2 = qy * ld * 8  # the flat padded arrays the passes stream
    band = 6 * n2 / (pt["operator_ms"] * 1e-3) / 1e9
    upd = 3 * n2 / (pt["update_ms"] * 1e-3) / 1e9
    w = 2 * op.half_bandwidth + 1
    tr = profile_json("ncu_passes_r02.json")
    key = f"band_kernel<{len(op)},{w},PCG>@q{qy}"
    return {"bound": "hbm", "unit": "GB/s", "peak": peak, "peak_source": src, "q": [qy, qx],
            "banded_operator_pass": {
                "kernel": f"band_kernel<{len(op)} terms, W={w}> (LD_PCG)", "achieved": band, "frac": band / peak,
                "launch_ms": pt["operator_ms"], "algorithmic_bytes": 6 * n2,
                "traffic": tr.get(key, {}).get("dram_bytes_per_launch"),
                "note": "read Z, Q_prev, U; write Q, W, U (direction update, W = L(Q), <W,Q>, |Q|^2 and the "
                        "previous iteration's deferred U += alpha Q)"},
            "vector_update_pass": {
                "kernel": "pcg_rupdate_kernel", "achieved": upd, "frac": upd / peak, "launch_ms": pt["update_ms"],
                "algorithmic_bytes": 3 * n2,
                "traffic": tr.get(f"pcg_rupdate_kernel@q{qy}", {}).get("dram_bytes_per_launch"),
                "note": "read R, W; write R (+ |R|^2, stop test)"},
            "preconditioner_ms": pt["preconditioner_ms"]}


# ----------------------------------------------------------------- cfg5 -----
def cfg5_setup(args, mode):
    import paper_2109_01173_b200 as pb
    from paper_2109_01173_b200 import workloads as wl
    w = wl.cfg5(N=args.N, mode=mode)
    ex = w.extra
    p = ex["params"]
    inner = pb.InnerSolver(rule="budget", max_iter=args.iters_per_step, precond_mode=mode)
    run = dict(domain=pb.SQUARE, x=w.x, y=w.y, d_u=1.0, d_v=p.d_theta, kinetics=ex["kinetics"], rho=p.rho,
               inner=inner, lumped=True)
    return w, ex, run


def run_cfg5(args):
    import torch
    import paper_2109_01173_b200 as pb
    from paper_2109_01173_b200.timestepping import _step_system

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    K = args.iters_per_step
    if args.strassen_levels is not None:
        pb.set_strassen_levels(args.strassen_levels)
    t_setup = time.perf_counter()
    w, ex, run = cfg5_setup(args, args.precond_mode)
    qy, qx = w.op.shape
    tau = ex["tau"]
    grid1 = pb.TimeGrid(tau, tau)  # one IMEX step per call (the DIB system is autonomous)
    state = tuple(torch.from_numpy(np.ascontiguousarray(s)).cuda() for s in ex["state0"])

    if world == 1:
        def step(st, grid=grid1):
            return pb.imex_euler_rds(state0=st, grid=grid, **run)
    else:
        from paper_2109_01173_b200 import distributed as D
        if world == 2:
            def step(st, grid=grid1):
                return D.species_parallel_imex_rds(state0=st, grid=grid, **run)
        else:
            def step(st, grid=grid1):
                return D.grouped_imex_rds(state0=st, grid=grid, **run)

    # first step: builds the step systems (operators, dense preconditioner
    # inverses formed on the device, solver workspaces) -- reported as setup
    tr = step(state)
    barrier()
    setup_s = time.perf_counter() - t_setup
    if world == 1:
        state = tr.final
        for _ in range(max(args.warmup - 1, 0)):
            state = step(state).final
    elif args.warmup > 1:
        step(state, pb.TimeGrid(tau, (args.warmup - 1) * tau))
    barrier()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = 0
    if world == 1:
        for _ in range(args.steps):
            tr = step(state)
            state = tr.final
            its += int(np.sum(tr.iterations))
    else:
        # N > 1: the K steps in one driver call -- the states stay column-sharded
        # (or species-split) on the devices between steps; the per-rank setup
        # (block operators, inverses, process groups) is cached from the warm-up
        tr = step(state, pb.TimeGrid(tau, args.steps * tau))
        its = int(np.sum(tr.iterations))
    e1.record()
    barrier()
    clk = clocks.stop()
    elapsed = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    value = qy * qx * its / elapsed

    # ---- e2e: numpy states in (page-locked) / out through the drop-in driver ----
    e2e = None
    if not args.no_e2e:
        pinned = [torch.empty((qy, qx), dtype=torch.float64, pin_memory=True) for _ in range(2)]
        src = state if world == 1 else ex["state0"]
        for pbuf, s in zip(pinned, src):
            pbuf.copy_(s if isinstance(s, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(s)))
        hstate = tuple(pbuf.numpy() for pbuf in pinned)
        if world == 1:
            # warm: the page-locked result blocks enter the caching host allocator -- two steps, since a
            # step's inputs (the previous step's results) are still alive when its own results are allocated
            for _ in range(2):
                hstate = step(hstate).final
        barrier()
        e0.record()
        its_e = 0
        if world == 1:
            for _ in range(args.steps):
                tr = step(hstate)  # H2D of both states, D2H of both new states
                hstate = tr.final
                its_e += int(np.sum(tr.iterations))
            h2d = d2h = 2 * qy * qx * 8
            note = ("imex_euler_rds(state0 = numpy views of page-locked host arrays, one step per call); "
                    "the step systems are reused across calls (bounded step cache)")
        else:
            tr = step(hstate, pb.TimeGrid(tau, args.steps * tau))  # host states in, host states out
            its_e = int(np.sum(tr.iterations))
            h2d = 2 * qy * qx * 8 // args.steps  # each rank reads its part; averaged over the K steps
            d2h = sum(int(np.asarray(f).nbytes) for f in tr.final) // args.steps
            note = (f"{'species_parallel' if world == 2 else 'grouped'}_imex_rds(state0 = numpy page-locked host "
                    f"arrays, {args.steps} steps per call); bytes per step averaged over the call")
        e1.record()
        barrier()
        el = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        e2e = {"value": qy * qx * its_e / el, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "note": note}

    if rank != 0 or world > 1:
        line = None
        if rank == 0:
            line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
                    "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
                    "config": {"workload": cfg5_name(args, qy, qx), "iterations_per_step": 2 * K,
                               "parallelism": ("species-parallel (one species per GPU)" if world == 2 else
                                               f"2 species groups x {world // 2} column shards"),
                               "l2": "inputs larger than L2 (each q x q state is 537 MB)", "setup_s": setup_s},
                    "e2e": e2e, "clocks": clk,
                    # this library's kernels per rank in the timed region: species-parallel runs the
                    # single-GPU step of one species; the grouped driver per step rhs (1) + warm-start
                    # apply / residual / dots / start / xpby (5) + 2 preconditioner GEMMs, and per
                    # iteration apply, dots, update, 2 GEMMs, dots, control, xpby (8), + norms (1)
                    "gpu_launches": (args.steps * (4 + 2 + K * 4 + 1) if world == 2 else
                                     args.steps * (1 + 5 + 2 + K * 8 + 1)),
                    "roofline": None, "cpu_baseline": None}
            print(json.dumps(line), flush=True)
        dist.barrier()
        dist.destroy_process_group()
        return

    # ---- per-pass timing of the headline iteration (q = 8192) ----
    op_u, _, pre_u = _step_system(w.x, w.y, 1.0, tau, True, run["inner"])
    levels = pre_u.uses_strassen() if args.precond_mode == "inverse" else 0
    hbm = hbm_passes(op_u, pre_u)
    iter_ms = 1e3 * elapsed / args.steps / (2 * K)

    # ---- the same steps with the classic schedule (one q^3 DMMA GEMM per product) ----
    classic = None
    if levels > 0 and not args.no_classic:
        pb.clear_step_cache()
        del op_u, pre_u
        torch.cuda.empty_cache()
        prev_levels = pb.set_strassen_levels(0)
        stc = tuple(s.clone() for s in state)
        stc = step(stc).final
        barrier()
        e0.record()
        its_c = 0
        n_c = min(args.steps, 3)
        for _ in range(n_c):
            tr = step(stc)
            stc = tr.final
            its_c += int(np.sum(tr.iterations))
        e1.record()
        barrier()
        el_c = e0.elapsed_time(e1) / 1e3
        classic = {"value": qy * qx * its_c / el_c, "unit": UNIT, "steps": n_c, "ms_per_step": 1e3 * el_c / n_c,
                   "iteration_ms": 1e3 * el_c / its_c,
                   "note": "the same IMEX steps with each preconditioner product as one q^3 DMMA GEMM "
                           "(set_strassen_levels(0))"}
        del stc
        pb.clear_step_cache()
        pb.set_strassen_levels(prev_levels)
        torch.cuda.empty_cache()

    # ---- the same steps with the f1 banded preconditioner ----
    alt = None
    if not args.no_alt and args.precond_mode != "banded":
        wb, exb, runb = cfg5_setup(args, "banded")
        stb = tuple(s.clone() for s in state)
        stb = pb.imex_euler_rds(state0=stb, grid=grid1, **runb).final
        barrier()
        e0.record()
        its_b = 0
        for _ in range(args.steps):
            tr = pb.imex_euler_rds(state0=stb, grid=grid1, **runb)
            stb = tr.final
            its_b += int(np.sum(tr.iterations))
        e1.record()
        barrier()
        el_b = e0.elapsed_time(e1) / 1e3
        op_b, _, pre_b = _step_system(wb.x, wb.y, 1.0, tau, True, runb["inner"])
        alt = {"banded": {"value": qy * qx * its_b / el_b, "unit": UNIT, "ms_per_step": 1e3 * el_b / args.steps,
                          "iteration_ms": 1e3 * el_b / its_b, "roofline_hbm": hbm_passes(op_b, pre_b),
                          "note": "SURVEY §8 f1: the same preconditioner P_L U P_R applied by SPIKE-partitioned "
                                  "banded solves instead of dense-inverse GEMMs (parity-neutral, HBM-bound)"}}
        del stb
        pb.clear_step_cache()  # frees both species' solver workspaces of both forms

    del state
    torch.cuda.empty_cache()
    roof = gemm_roofline(qy, levels)
    n_gemm = 2 if args.precond_mode == "inverse" else (4 if args.precond_mode == "spectral" else 0)
    n_launch = n_gemm * roof.get("launches_per_product", 1)  # dominant-kernel launches per iteration
    tkey = f"q{strassen_leaf(qy, levels)}x{7 ** levels}" if levels > 0 else f"q{qy}"
    roof.update({"share_of_iteration": n_launch * roof["launch_ms"] / iter_ms if n_gemm else 0.0,
                 "iteration_ms": iter_ms,
                 "traffic": (profile_json("ncu_dgemm_r02.json").get(tkey) or {}).get("dram_bytes_per_launch")})
    if levels > 0:
        # the two dense products of one preconditioner application, as a whole
        h = strassen_leaf(qy, levels)
        # operand and assembly passes of the two products: (4^L + 7^L) leaf blocks in, out (+ R for <Z,R>)
        pass_bytes = (2 * 2 * (4 ** levels + 7 ** levels) + 4 ** levels) * h * h * 8.0
        pass_ms = hbm["preconditioner_ms"] - 2 * roof["launch_ms"]
        roof["preconditioner_application"] = {
            "passes": {"ms": pass_ms, "algorithmic_bytes": pass_bytes, "achieved": pass_bytes / (pass_ms * 1e-3) / 1e9,
                       "unit": "GB/s", "frac": pass_bytes / (pass_ms * 1e-3) / 1e9 / hbm["peak"],
                       "note": "strassen_operands_kernel + strassen_assemble_kernel of both products: the "
                               "application's time minus its two leaf launches"},
            "ms": hbm["preconditioner_ms"], "algorithmic_flops": 4.0 * qy ** 3,
            "algorithmic_tflops": 4.0 * qy ** 3 / (hbm["preconditioner_ms"] * 1e-3) / 1e12,
            "executed_flops": 4.0 * qy ** 3 * (7.0 / 8.0) ** levels,
            "note": f"{levels} Strassen levels: per product one pass forming the {7 ** levels} leaf operands of the "
                    f"variable factor, one strided-batch launch of the leaf products, one assembly pass"}
    if args.precond_mode == "banded":
        bp = hbm["banded_operator_pass"]
        roof = {"bound": "hbm", "kernel": bp["kernel"], "achieved": bp["achieved"], "peak": hbm["peak"],
                "unit": "GB/s", "frac": bp["frac"], "traffic": bp["traffic"], "launch_ms": bp["launch_ms"],
                "peak_source": hbm["peak_source"], "iteration_ms": iter_ms}

    cpu = None
    if not args.no_cpu_baseline:
        v, wall, setup, n_it, n_sys = cpu_sample("cfg5", args.N, args.cpu_iters)
        cpu = {"value": v, "unit": UNIT, "cores": cores(), "kind": "port",
               "sample": f"oracle restatement of sylfem mo_pcg (dense GEMM apply + LU preconditioner) on both cfg5 "
                         f"step-0 systems (rhs and warm start of imex_euler_rds's first step), {args.cpu_iters} "
                         f"iterations each ({n_it} iterations, {wall:.1f} s); setup {setup:.0f} s excluded",
               "host_stack": host_stack()}

    secondary = None
    if not args.no_secondary:
        secondary = cfg3_block(args)

    # kernels per IMEX step and species: rhs (1), warm-start apply (1) + R0 (1),
    # first preconditioner (n_pre), K x (banded pass + R update + preconditioner),
    # deferred U update (1), increment norms (1)
    n_pre = n_gemm if n_gemm else 5
    if levels > 0:
        n_pre = 2 * 3  # per product: leaf operands, leaf products, assembly
    per_species = 4 + n_pre + K * (2 + n_pre) + 1
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": {"workload": cfg5_name(args, qy, qx), "iterations_per_step": 2 * K,
                   "inner": f"InnerSolver(rule='budget', max_iter={K}, precond_mode='{args.precond_mode}') per species",
                   "preconditioner_mode": args.precond_mode,
                   "gemm_schedule": (f"{levels} Strassen levels: {7 ** levels} leaf products of "
                                     f"{strassen_leaf(qy, levels)}^3 per preconditioner product in one strided-batch "
                                     f"DMMA launch"
                                     if levels > 0 else "classic (one DMMA GEMM per product)"),
                   "l2": "inputs larger than L2 (each q x q state is 537 MB; 2 x (8 solver grids + 2 dense "
                         "inverses) = 10.7 GB resident" +
                         (", plus the Strassen operand sums and scratch)" if levels > 0 else ")"),
                   "parallelism": "single GPU", "setup_s": round(setup_s, 2)},
        "roofline": roof,
        "roofline_hbm": hbm,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": 2 * per_species * args.steps,
        "clocks": clk,
        "alt_preconditioner": alt,
        "classic_gemm_schedule": classic,
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)


def cfg5_name(args, qy, qx):
    return (f"cfg5 (BASELINE configs[4]): two-species DIB (spots_worms, rho=400, d_theta=20), unit square, "
            f"lumped P1, Neumann, N={args.N}, q={qy}x{qx} per species, IMEX tau_ref=1.25e-5, App. A initial "
            f"state; one step = one IMEX step (both species), {args.iters_per_step} MO-PCG iterations per "
            f"species solve, reference single-term preconditioner ({args.precond_mode})")


# ----------------------------------------------------------------- cfg3 -----
def cfg3_block(args, steps=5, K=200):
    """Secondary: cfg3 (configs[2]) MO-PCG, q = 2047, 200-iteration solves,
    plus the full solve to 1e-8 with the f1 preconditioner."""
    import torch
    import paper_2109_01173_b200 as pb
    from paper_2109_01173_b200 import workloads as wl
    w = wl.cfg3(N=2048, mode="inverse")
    op, pre = w.op, w.precond
    qy, qx = op.shape
    rhs = torch.from_numpy(w.rhs).cuda()
    stop = pb.fixed_budget()
    for _ in range(2):
        pb.mo_pcg(op, rhs, precond=pre, stop=stop, max_iter=K)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = sum(pb.mo_pcg(op, rhs, precond=pre, stop=stop, max_iter=K).iterations for _ in range(steps))
    e1.record()
    torch.cuda.synchronize()
    el = e0.elapsed_time(e1) / 1e3
    lv = pre.uses_strassen()
    sched = (f"2 dense products, each {7 ** lv} leaf products of {strassen_leaf(qy, lv)}^3 ({lv} Strassen levels) in "
             f"one strided-batch DMMA launch" if lv > 0 else "2 DMMA GEMMs")
    out = {"workload": "cfg3 (BASELINE configs[2]): wave domain, P2, Dirichlet, N=2048, q=2047x2047, 5-term "
                       f"operator, elliptic_xnormal preconditioner (inverse: {sched})",
           "value": qy * qx * its / el, "unit": UNIT, "iterations_per_step": K, "ms_per_step": 1e3 * el / steps}
    out["roofline_hbm"] = hbm_passes(op, pre)
    out["roofline"] = gemm_roofline(qy, lv)
    tkey = f"q{strassen_leaf(qy, lv)}x{7 ** lv}" if lv > 0 else f"q{qy}"
    out["roofline"]["traffic"] = (profile_json("ncu_dgemm_r02.json").get(tkey) or {}).get("dram_bytes_per_launch")
    if not args.no_full:
        pre_b = pb.make_preconditioner("elliptic_xnormal", w.x, w.y, mode="banded")
        pb.mo_pcg(op, rhs, precond=pre_b, stop=stop, max_iter=10)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rf = pb.mo_pcg(op, rhs, precond=pre_b, stop=pb.relative_residual(1e-8), max_iter=100000)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t1
        out["time_to_solution_banded"] = {"seconds": dt, "iterations": rf.iterations, "stop_reason": rf.stop_reason,
                                          "dof_it_per_s": qy * qx * rf.iterations / dt}
    return out


def run_cfg3(args):
    """cfg3 as the line's workload (round-1 headline): one MO-PCG solve of a
    fixed budget per step; N > 1 column-shards the solve."""
    import torch
    import paper_2109_01173_b200 as pb
    from paper_2109_01173_b200 import workloads as wl

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    t_setup = time.perf_counter()
    w = wl.cfg3(N=args.N, mode=args.precond_mode)
    op, pre = w.op, w.precond
    qy, qx = op.shape
    pre.native(op.shape)
    setup_s = time.perf_counter() - t_setup
    K = args.iters_per_step
    stop = pb.fixed_budget()
    rhs_d = torch.from_numpy(w.rhs).cuda()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    if world > 1:
        from paper_2109_01173_b200.distributed import Comm, CudaBackend, Layout, PeerTransposes, sharded_mo_pcg
        lay = Layout(qy, qx, world, rank)
        backend = CudaBackend(op, pre, lay)
        comm = Comm(lay, torch.device("cuda", local))
        peer = None
        if args.transposes == "peer":
            try:
                peer = PeerTransposes(lay, backend, sync="stream")
            except Exception as exc:  # noqa: BLE001
                log(f"peer transposes unavailable ({exc}); using NCCL all-to-alls")
        rhs_d = rhs_d[:, lay.c0:lay.c0 + lay.n].contiguous()
        w.rhs = np.ascontiguousarray(w.rhs[:, lay.c0:lay.c0 + lay.n])

        def step(rhs):
            return sharded_mo_pcg(backend, comm, rhs, stop=stop, max_iter=K,
                                  keep_on_device=not isinstance(rhs, np.ndarray), peer=peer)
    else:
        def step(rhs):
            return pb.mo_pcg(op, rhs, precond=pre, stop=stop, max_iter=K)

    for _ in range(max(args.warmup, 1)):
        step(rhs_d)
    barrier()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = sum(step(rhs_d).iterations for _ in range(args.steps))
    e1.record()
    barrier()
    clk = clocks.stop()
    elapsed = e0.elapsed_time(e1) / 1e3
    if dist is not None:
        t = torch.tensor([elapsed], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    value = qy * qx * its / elapsed
    e2e = None
    if not args.no_e2e:
        pinned = torch.empty(w.rhs.shape, dtype=torch.float64, pin_memory=True)
        pinned.copy_(torch.from_numpy(np.ascontiguousarray(w.rhs)))
        rhs_host = pinned.numpy()
        keep = step(rhs_host)
        keep = (keep, step(rhs_host))
        del keep
        barrier()
        e0.record()
        its_e = sum(step(rhs_host).iterations for _ in range(args.steps))
        e1.record()
        barrier()
        el = e0.elapsed_time(e1) / 1e3
        if dist is not None:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": qy * qx * its_e / el, "unit": UNIT, "h2d_bytes_per_step": int(w.rhs.size * 8),
               "d2h_bytes_per_step": int(w.rhs.size * 8 + (2 * K + 1) * 8)}
    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return
    lv = pre.uses_strassen() if (world == 1 and args.precond_mode == "inverse") else 0
    roof = gemm_roofline(qy, lv) if world == 1 else None
    hbm = hbm_passes(op, pre) if world == 1 else None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, wall, setup, n_it, _ = cpu_sample("cfg3", args.N, max(args.cpu_iters, 3))
        cpu = {"value": v, "unit": UNIT, "cores": cores(), "kind": "port",
               "sample": f"oracle restatement of sylfem mo_pcg on the same cfg3 system, {n_it} iterations "
                         f"({wall:.1f} s), setup {setup:.1f} s excluded", "host_stack": host_stack()}
    n_gemm = 2 if args.precond_mode == "inverse" else (4 if args.precond_mode == "spectral" else 0)
    n_pre = n_gemm if n_gemm else 5
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": {"workload": f"cfg3 (BASELINE configs[2]): wave domain, P2, Dirichlet, N={args.N}, "
                               f"q={qy}x{qx}, {len(op)}-term operator, MO-PCG with elliptic_xnormal "
                               f"preconditioner ({args.precond_mode})",
                   "iterations_per_step": K, "preconditioner_mode": args.precond_mode,
                   "l2": "inputs larger than L2", "setup_s": round(setup_s, 3),
                   "parallelism": f"column-sharded x{world}" if world > 1 else "single GPU"},
        "roofline": roof, "roofline_hbm": hbm, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": (2 + n_pre + 1 + (2 + n_pre) * K) * args.steps, "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "cfg5":
        run_cfg5(args)
    else:
        run_cfg3(args)


if __name__ == "__main__":
    main()
