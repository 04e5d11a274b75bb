#!/usr/bin/env python
"""MO-PCG DoF*iterations/s (fp64) on B200 — the BASELINE.json headline metric.

Workload (default): BASELINE configs[2] ("cfg3"): -Lap u + u = f on the wave
domain 0 <= x <= 1 + 0.3 sin(2 pi y), Dirichlet, MO-FEM P2 with N = 2048
(q = 2047; q = 2048 is inadmissible for P2/Dirichlet), the
5-term Sylvester operator and the single-term elliptic_xnormal preconditioner.
One "step" is one MO-PCG solve with a fixed budget of --iters-per-step
iterations (stop rule disabled so every step does the same work), run
through the drop-in API on device-resident inputs.  DoF*it/s = q_y q_x *
iterations / seconds.

Printed (rank 0, one JSON line): value (device-resident), e2e (host numpy
rhs in from page-locked memory, host solution out, H2D/D2H inside the timed
region), roofline of the dominant kernel (the FP64 DMMA GEMM of the
preconditioner) and roofline_hbm of the banded and update passes (live CUDA
events; DRAM traffic from the committed ncu captures), cpu_baseline (the
oracle port of the reference on the host cores, bounded sample), clocks,
the banded-preconditioner alternative and the full solve to 1e-8.
Under torchrun (N > 1) the same solve is column-sharded over the ranks.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
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
L2_BYTES = 126 * 1024 * 1024
FP64_PEAK_FALLBACK = 35.48  # cuBLAS DGEMM 8192^3 measured on this pool (profiles/fp64_peaks_r01.log)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--N", type=int, default=2048, help="subintervals of the cfg3 workload")
    # 200 iterations per solve: the solve's own setup (initial residual and first
    # preconditioner apply, ~1 ms) is amortised as in the real 13k-iteration solve
    ap.add_argument("--iters-per-step", type=int, default=200)
    ap.add_argument("--precond-mode", default="inverse", choices=["inverse", "spectral", "banded"])
    ap.add_argument("--cpu-iters", type=int, default=3, help="oracle iterations in the cpu_baseline sample")
    ap.add_argument("--ref-iters-per-step", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the banded-preconditioner (f1) measurement")
    ap.add_argument("--no-full", action="store_true", help="skip the full solve to 1e-8 (time to solution)")
    ap.add_argument("--transposes", default="peer", choices=["peer", "nccl"],
                    help="N > 1: preconditioner transposes over peer memory (P2P copies + the scatter GEMM) "
                         "or NCCL all-to-alls")
    return ap.parse_args()


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


# -------------------------------------------------------------- oracle leg --
def oracle_cfg3(N: int):
    """cfg3 in the oracle (the reference restated): dense factors, LU preconditioner."""
    import oracle as orc
    from paper_2109_01173_b200.workloads import sine_source
    x, y = orc.direction_sets(orc.wave_domain(), 2, N, orc.DIRICHLET)
    terms, rhs_of = orc.elliptic_terms(x, y, 1.0)
    pre = orc.LUPrecond(*orc.precond_factors("elliptic_xnormal", x, y))
    return orc, terms, rhs_of(sine_source(N, N, 3)), pre


def cpu_sample(N: int, iters: int):
    """Time `iters` oracle MO-PCG iterations on the step-0 system (setup excluded)."""
    t0 = time.perf_counter()
    orc, terms, rhs, pre = oracle_cfg3(N)
    setup = time.perf_counter() - t0
    r = orc.mo_pcg(terms, rhs, pre.inverse, ("residual", 1e-30), max_iter=iters)
    q = rhs.shape[0] * rhs.shape[1]
    return q * r["iterations"] / r["wall"], r["wall"], setup, r["iterations"]


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
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(k, "").isdigit():
            return int(os.environ[k])
    return os.cpu_count() or 1


# ---------------------------------------------------------------- dist ------
def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    world, rank, _ = dist_init(args)
    if rank != 0:
        return
    N, per = args.N, args.ref_iters_per_step
    orc, terms, rhs, pre = oracle_cfg3(N)
    q = rhs.shape[0] * rhs.shape[1]
    for _ in range(args.warmup):
        orc.mo_pcg(terms, rhs, pre.inverse, ("residual", 1e-30), max_iter=per)
    t0 = time.perf_counter()
    its = 0
    for _ in range(args.steps):
        its += orc.mo_pcg(terms, rhs, pre.inverse, ("residual", 1e-30), max_iter=per)["iterations"]
    dt = time.perf_counter() - t0
    value = q * its / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded 8-mode sine source, SURVEY App. A)",
        "config": {"workload": "cfg3 (BASELINE configs[2]) wave domain P2 Dirichlet, N=%d q=%d" % (N, N - 1),
                   "iterations_per_step": per, "parallelism": "host BLAS threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "port",
                         "sample": f"oracle restatement of sylfem mo_pcg (dense GEMM apply, LU preconditioner), "
                                   f"{per} iterations per step on the cfg3 step-0 system, setup excluded",
                         "host_stack": host_stack()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_native(args):
    import torch

    world, rank, local = dist_init(args)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")

    import paper_2109_01173_b200 as pb
    from paper_2109_01173_b200 import _native as nat
    from paper_2109_01173_b200 import workloads as wl

    t_setup = time.perf_counter()
    w = wl.cfg3(N=args.N, mode=args.precond_mode)
    op, pre = w.op, w.precond
    qy, qx = op.shape
    pre.native(op.shape)
    setup_s = time.perf_counter() - t_setup
    K_it = args.iters_per_step
    stop = pb.relative_residual(1e-30)  # fixed iteration budget per step
    rhs_d = torch.from_numpy(w.rhs).cuda()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    if world > 1:
        # column-sharded MO-PCG over NCCL (SURVEY §8 e): total work fixed -> strong scaling
        from paper_2109_01173_b200.distributed import Comm, CudaBackend, Layout, PeerTransposes, sharded_mo_pcg
        lay = Layout(qy, qx, world, rank)
        backend = CudaBackend(op, pre, lay)
        comm = Comm(lay, torch.device("cuda", local))
        peer = None
        if args.transposes == "peer":
            try:  # CUDA IPC between the ranks' GPUs; NCCL all-to-alls when peer mappings are unavailable
                peer = PeerTransposes(lay, backend, sync="stream")
            except Exception as exc:  # noqa: BLE001
                log(f"peer transposes unavailable ({exc}); using NCCL all-to-alls")
                args.transposes = "nccl"
        rhs_d = rhs_d[:, lay.c0:lay.c0 + lay.n].contiguous()
        w.rhs = np.ascontiguousarray(w.rhs[:, lay.c0:lay.c0 + lay.n])

        class _Rep:  # adapt the sharded report to the single-GPU fields used below
            def __init__(self, r, ms):
                self.iterations, self.diagnostics = r.iterations, {"device": {"loop_ms": ms}}

        def step(rhs):
            t1 = time.perf_counter()
            r = sharded_mo_pcg(backend, comm, rhs, stop=stop, max_iter=K_it,
                               keep_on_device=not isinstance(rhs, np.ndarray), peer=peer)
            return _Rep(r, 1e3 * (time.perf_counter() - t1))
    else:
        def step(rhs):
            return pb.mo_pcg(op, rhs, precond=pre, stop=stop, max_iter=K_it)

    for _ in range(max(args.warmup, 1)):
        rep = step(rhs_d)
    barrier()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = 0
    loop_ms = []
    for _ in range(args.steps):
        rep = step(rhs_d)
        its += rep.iterations
        loop_ms.append(rep.diagnostics["device"]["loop_ms"])
    e1.record()
    barrier()
    clk = clocks.stop()
    elapsed = e0.elapsed_time(e1) / 1e3
    if dist is not None:
        t = torch.tensor([elapsed], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    value = qy * qx * its / elapsed  # whole grid per iteration (sharded across ranks when world > 1)

    # ---- e2e through the drop-in API with host buffers ----
    e2e = None
    if not args.no_e2e:
        # the step's input lives in page-locked host memory (a numpy view of a
        # pinned buffer): the H2D inside the timed region is a DMA, not a staged copy
        pinned = torch.empty(w.rhs.shape, dtype=torch.float64, pin_memory=True)
        pinned.copy_(torch.from_numpy(np.ascontiguousarray(w.rhs)))
        rhs_host = pinned.numpy()
        # warm-up of the host path: two live results, so two page-locked result
        # blocks enter the caching host allocator (a timed step returns one
        # while the previous one is still referenced)
        keep = step(rhs_host)
        keep = (keep, step(rhs_host))
        del keep  # both blocks back in the cache before the timed steps
        barrier()
        e0.record()
        its_e = 0
        for _ in range(args.steps):
            rep_h = step(rhs_host)  # numpy in: H2D of rhs, D2H of solution + history
            its_e += rep_h.iterations
        e1.record()
        barrier()
        el = e0.elapsed_time(e1) / 1e3
        if dist is not None:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": qy * qx * its_e / el, "unit": UNIT,
               "h2d_bytes_per_step": int(qy * qx * 8),
               "d2h_bytes_per_step": int(qy * qx * 8 + (2 * K_it + 1) * 8)}

    # ---- the same workload with the f1 preconditioner (banded Cholesky,
    #      segmented solves): same operator, parity-neutral, HBM-bound ----
    alt = {}
    if world == 1 and not args.no_alt and args.precond_mode != "banded":
        pre_b = pb.make_preconditioner("elliptic_xnormal", w.x, w.y, mode="banded")
        pre_b.native(op.shape)
        for _ in range(max(args.warmup, 1)):
            pb.mo_pcg(op, rhs_d, precond=pre_b, stop=stop, max_iter=K_it)
        barrier()
        e0.record()
        its_b, lms = 0, []
        for _ in range(args.steps):
            rb = pb.mo_pcg(op, rhs_d, precond=pre_b, stop=stop, max_iter=K_it)
            its_b += rb.iterations
            lms.append(rb.diagnostics["device"]["loop_ms"])
        e1.record()
        barrier()
        el_b = e0.elapsed_time(e1) / 1e3
        alt["banded"] = {"value": qy * qx * its_b / el_b, "unit": UNIT, "ms_per_step": 1e3 * el_b / args.steps,
                         "iteration_ms": statistics.median(lms) / K_it,
                         "note": "SURVEY §8 f1: same preconditioner P_L U P_R applied by SPIKE-partitioned banded "
                                 "solves instead of dense-inverse GEMMs (parity-neutral)"}

    # ---- time to solution: the full cfg3 solve to the BASELINE tolerance 1e-8 ----
    tts = None
    if world == 1 and not args.no_full:
        tts = {}
        modes = [args.precond_mode] + ([] if args.no_alt or args.precond_mode == "banded" else ["banded"])
        for mode in modes:
            p_full = pre if mode == args.precond_mode else pre_b
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            rf = pb.mo_pcg(op, rhs_d, precond=p_full, stop=pb.relative_residual(1e-8), max_iter=100000)
            torch.cuda.synchronize()
            dt_full = time.perf_counter() - t1
            tts[mode] = {"seconds": dt_full, "iterations": rf.iterations, "stop_reason": rf.stop_reason,
                         "final_relative_residual": float(rf.residual_history[-1] / rf.residual_history[0]),
                         "dof_it_per_s": qy * qx * rf.iterations / dt_full}
        if not args.no_alt:
            # the north star's (lambda_i + mu_j) two-term spectral
            # preconditioner (opt-in; not the reference's, so iteration counts differ)
            t1 = time.perf_counter()
            pre2 = pb.two_term_preconditioner(op)
            pre2.native()
            setup2 = time.perf_counter() - t1
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            rf = pb.mo_pcg(op, rhs_d, precond=pre2, stop=pb.relative_residual(1e-8), max_iter=100000)
            torch.cuda.synchronize()
            dt_full = time.perf_counter() - t1
            tts["two_term_spectral"] = {
                "seconds": dt_full, "setup_s": setup2, "iterations": rf.iterations, "stop_reason": rf.stop_reason,
                "final_relative_residual": float(rf.residual_history[-1] / rf.residual_history[0]),
                "note": "opt-in f3 preconditioner (M1 x A + (B1+M3) x M exactly, 4 DMMA GEMMs per iteration)"}

    # ---- roofline of the dominant kernel: the DMMA GEMM (q x q x q) ----
    L = nat.lib()
    ldq = qy + (qy % 2)
    A = torch.randn(qy, ldq, dtype=torch.float64, device="cuda")
    B = torch.randn(qx, ldq, dtype=torch.float64, device="cuda")
    C = torch.empty(qy, ldq, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def gemm():
        nat.check(L.sfb_dgemm_nt(A.data_ptr(), ldq, B.data_ptr(), ldq, qy, qx, qy, C.data_ptr(), ldq, s))

    for _ in range(3):
        gemm()
    torch.cuda.synchronize()
    reps = 20
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    for _ in range(reps):
        gemm()
    g1.record()
    torch.cuda.synchronize()
    t_gemm = g0.elapsed_time(g1) / 1e3 / reps
    gemm_tf = 2.0 * qy * qx * qy / t_gemm / 1e12
    # cuBLAS DGEMM peak measured live on this box (the FP64 roofline denominator)
    n8 = 8192
    a8 = torch.randn(n8, n8, dtype=torch.float64, device="cuda")
    b8 = torch.randn(n8, n8, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a8 @ b8
    torch.cuda.synchronize()
    g0.record()
    for _ in range(3):
        a8 @ b8
    g1.record()
    torch.cuda.synchronize()
    peak = 2.0 * n8 ** 3 / (g0.elapsed_time(g1) / 1e3 / 3) / 1e12
    del a8, b8
    cublas_same = None
    try:
        Ad = A[:, :qy].contiguous()
        Bd = B[:, :qy].contiguous()
        for _ in range(2):
            Ad @ Bd.T
        torch.cuda.synchronize()
        g0.record()
        for _ in range(5):
            Ad @ Bd.T
        g1.record()
        torch.cuda.synchronize()
        cublas_same = 2.0 * qy * qx * qy / (g0.elapsed_time(g1) / 1e3 / 5) / 1e12
    except RuntimeError:
        pass
    n_gemm_per_iter = 2 if args.precond_mode == "inverse" else (4 if args.precond_mode == "spectral" else 0)
    iter_ms = statistics.median(loop_ms) / K_it
    share = (n_gemm_per_iter * t_gemm * 1e3) / iter_ms if n_gemm_per_iter else 0.0
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_dgemm_r01.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None

    # ---- HBM roofline of the memory-bound passes of the headline iteration
    #      (banded pass 32q^2 B incl. the direction update,
    #      vector update 48q^2 B), timed per launch on the solver's buffers ----
    hbm = None
    if world == 1 and op.banded:
        pt = pb.solvers.pcg_pass_times(op, pre, reps=20)
        hbm_peak, hbm_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
        try:
            mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            if mp.get("hbm_gbs"):
                hbm_peak, hbm_src = float(mp["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
        except (OSError, ValueError):
            pass
        n2 = qy * qx * 8
        # the banded iteration defers U += alpha Q into the next operator pass
        # (Q_prev is in shared memory there): operator pass 48 B, update pass 24 B
        band_gbs = 6 * n2 / (pt["operator_ms"] * 1e-3) / 1e9
        upd_gbs = 3 * n2 / (pt["update_ms"] * 1e-3) / 1e9
        ptraffic = {}
        try:
            ptraffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_passes_r01.json")))
        except (OSError, ValueError):
            pass
        hbm = {"bound": "hbm", "unit": "GB/s", "peak": hbm_peak, "peak_source": hbm_src,
               "banded_operator_pass": {
                   "kernel": f"band_kernel<{len(op)} terms, W={2 * op.half_bandwidth + 1}> (LD_PCG)",
                   "achieved": band_gbs, "frac": band_gbs / hbm_peak, "launch_ms": pt["operator_ms"],
                   "algorithmic_bytes": 6 * n2,
                   "traffic": ptraffic.get("band_kernel<5,5,PCG>", {}).get("dram_bytes_per_launch"),
                   "note": "read Z, Q_prev, U; write Q, W, U (the previous iteration's U += alpha Q rides along; "
                           "+ <W,Q>, |Q|^2); 2*T*W FMAs per element on the FP64 pipe"},
               "vector_update_pass": {
                   "kernel": "pcg_rupdate_kernel", "achieved": upd_gbs, "frac": upd_gbs / hbm_peak,
                   "launch_ms": pt["update_ms"], "algorithmic_bytes": 3 * n2,
                   "traffic": ptraffic.get("pcg_rupdate_kernel", {}).get("dram_bytes_per_launch"),
                   "note": "read R, W; write R (+ |R|^2, stop test)"},
               "preconditioner_ms": pt["preconditioner_ms"]}

    # ---- CPU baseline (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, wall, setup, n_it = cpu_sample(args.N, args.cpu_iters)
        cpu = {"value": v, "unit": UNIT, "cores": cores(), "kind": "port",
               "sample": f"oracle restatement of sylfem mo_pcg (dense GEMM apply + LU preconditioner) on the "
                         f"same cfg3 system, {n_it} iterations ({wall:.1f} s), setup {setup:.1f} s excluded",
               "host_stack": host_stack()}

    # per solve: init + first preconditioner (+ the deferred-U fixup of the banded
    # iteration); per iteration: operator pass, update, preconditioner
    n_pre = n_gemm_per_iter if n_gemm_per_iter else 5  # banded: 3 SPIKE tile passes + 2 interface chains
    # (the banded iteration's R update also sets the loop condition: no loop-control kernel)
    per_step_launches = 1 + n_pre + (1 if op.banded else 0) + ((2 if op.banded else 3) + n_pre) * K_it
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded 8-mode sine source, SURVEY App. A)",
            "config": {"workload": f"cfg3 (BASELINE configs[2]): wave domain, P2, Dirichlet, N={args.N}, "
                                   f"q={qy}x{qx}, {len(op)}-term operator, MO-PCG with elliptic_xnormal "
                                   f"preconditioner ({args.precond_mode})",
                       "iterations_per_step": K_it, "preconditioner_mode": args.precond_mode,
                       "l2": "inputs larger than L2 (8 grid buffers + 2 dense inverses = "
                             f"{(8 * qy * qx + qy * qy + qx * qx) * 8 / 2**20:.0f} MiB > 126 MiB)",
                       "parallelism": f"column-sharded x{world} (NCCL halo + allreduce; transposes: "
                                      f"{'P2P copies + GEMM-fused NVLink scatter' if args.transposes == 'peer' else 'NCCL all-to-all'})"
                       if world > 1 else "single GPU",
                       "setup_s": round(setup_s, 3)},
            "roofline": {"bound": "tensor", "kernel": "dgemm_nt (DMMA.8x8x4 + TMA)",
                         "achieved": gemm_tf, "peak": peak, "unit": "TFLOP/s", "frac": gemm_tf / peak,
                         "traffic": traffic, "flops_per_launch": 2.0 * qy * qx * qy,
                         "launch_ms": t_gemm * 1e3, "peak_source": "cuBLAS DGEMM 8192^3 measured in this run",
                         "cublas_same_shape_tflops": cublas_same,
                         "share_of_iteration": share, "iteration_ms": iter_ms},
            "roofline_hbm": hbm,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": per_step_launches * args.steps,
            "clocks": clk,
            "alt_preconditioner": alt or None,
            "time_to_solution": tts,
        }
        if args.precond_mode == "banded" and hbm:
            # no GEMM in this iteration: the dominant kernel is the banded MO-PCG pass
            bp = hbm["banded_operator_pass"]
            line["roofline"] = {"bound": "hbm", "kernel": bp["kernel"], "achieved": bp["achieved"],
                                "peak": hbm["peak"], "unit": "GB/s", "frac": bp["frac"], "traffic": bp["traffic"],
                                "algorithmic_bytes": bp["algorithmic_bytes"], "launch_ms": bp["launch_ms"],
                                "peak_source": hbm["peak_source"], "iteration_ms": iter_ms}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()
