#!/usr/bin/env python3
"""Benchmark: grid-point time-step solves per second of the FIDS march on B200.

Workload (default, BASELINE.json configs[2]): B independent instances per
GPU, n = 4096 unknowns (N_ref = 4097), M = 512 graded levels, gamma = 0.5,
alpha = 1.5, r = (2-gamma)/gamma, SOE tolerance 1e-12 (N_exp = 143),
Strang-preconditioned BiCGSTAB at tol 1e-12; per-instance seeded
kappa = exp(0.4 g(x)) (1 + 0.2 t), g = 8 random Fourier modes with
N(0, 1/k^2) coefficients; f = 8 random sine modes x (1 + t);
phi = (1 - x^2)^2 U[0.5, 2].  A "step" is one time level of the march over
the whole batch (fused SOE push + RHS kernel, then the fused level-solve
kernel).  value = (instances on all ranks) * n * K / max-over-ranks time.

Multi-GPU: one process per GPU (torchrun), B instances per rank (weak
scaling), no collective on the hot path; barrier + max-over-ranks timing.

--impl reference times the reference's CPU path — the oracle port of
tsfrac.run_fids (oracle/, numpy pocketfft + OpenBLAS, exactly the
reference's arithmetic) — on the host cores, one instance per worker
process, same levels, same metric.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "grid-point time-step solves/sec (B*N*M/s)"
UNIT = "grid-point solves/s"


def workload(args):
    if args.workload == "cfg2":
        wl = dict(name="configs[2] batched FIDS march", n=4096, M=512, gamma=0.5, alpha=1.5,
                  eps=1e-12, tol=1e-12, B=args.batch or 4096, cpu_levels=64)
    elif args.workload == "cfg0":
        wl = dict(name="configs[0] single FIDS march", n=1024, M=256, gamma=0.5, alpha=1.5,
                  eps=1e-12, tol=1e-12, B=args.batch or 1, cpu_levels=64)
    elif args.workload == "cfg1":
        wl = dict(name="configs[1] single FIDS march at paper-upper scale", n=16384, M=1024,
                  gamma=0.5, alpha=1.5, eps=1e-12, tol=1e-12, B=args.batch or 1, cpu_levels=64)
    elif args.workload == "cfg3":
        wl = dict(name="configs[3] large-N single FIDS march", n=1 << 20, M=256, gamma=0.7,
                  alpha=1.2, eps=1e-12, tol=1e-12, B=args.batch or 1, cpu_levels=4)
    else:
        raise SystemExit(f"unknown workload {args.workload}")
    if args.gamma:
        wl["gamma"] = args.gamma
    if args.alpha:
        wl["alpha"] = args.alpha
    return wl


def cfg0_fields(n):
    N = n + 1
    x = -1.0 + (2.0 / N) * np.arange(1, N)
    return x


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------------- CPU
def _cpu_worker(args):
    """Instances of the workload through the oracle port, one after another
    in this process; returns (wall seconds of levels (warmup, warmup+K] summed
    over the instances, iterations).  Runs in a SPAWNED process whose
    environment pins OpenBLAS/OpenMP to one thread before numpy loads
    (cpu_measure); threadpoolctl re-asserts it."""
    wl, bs, warmup, K = args
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    import oracle as O
    n = wl["n"]
    gam, alpha, M = wl["gamma"], wl["alpha"], wl["M"]
    r = (2.0 - gam) / gam
    N = n + 1
    t, tau = O.graded_mesh(M, r, 1.0)
    col, h, _ = O.ifl_column(alpha, 1.0 + alpha / 2.0, 1.0, N)
    xx = -1.0 + h * np.arange(1, N)
    _, symbol = O.toeplitz_symbol(col)
    lam = O.strang_eigs(col)
    G = math.exp(math.lgamma(1.0 - gam))
    s, w = O.soe_build(gam, wl["eps"], (1.0 / M) ** r, 1.0)
    wall = 0.0
    its = 0
    for b in bs:
        if wl.get("cfg2", True):
            from paper_2002_11978_b200 import workloads as WL
            x, kx, fx, u0 = WL.instance_fields(n, b, 1)
            kf = lambda xx, t, k=kx[0]: k * (1.0 + 0.2 * t)  # noqa: E731
            sf = lambda xx, t, f=fx[0]: f * (1.0 + t)  # noqa: E731
            phi = u0[0]
        else:
            kf = lambda xx, t: 1.0 + 0.5 * np.sin(np.pi * xx) * np.exp(-t)  # noqa: E731
            sf = lambda xx, t: (1.0 + t) * np.sin(np.pi * xx)  # noqa: E731
            phi = (1.0 - cfg0_fields(n) ** 2) ** 2
        u = np.asarray(phi, dtype=float)
        W = np.zeros((s.size, n))
        t0 = None
        for m in range(1, min(M, warmup + K) + 1):
            if m == warmup + 1:
                t0 = time.perf_counter()
            kap = kf(xx, t[m])
            f = sf(xx, t[m])
            u, _, out = O.fids_step(u, W, s, w, tau[m - 1], gam, G, kap, f, symbol, lam,
                                    wl["tol"])
            if m > warmup:
                its += out.iterations
        wall += time.perf_counter() - t0
    return wall, its


def host_info():
    """CPU model, core count and the numpy/scipy/BLAS versions of this host."""
    info = {"nproc": os.cpu_count()}
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    info["numpy"] = np.__version__
    try:
        import scipy
        info["scipy"] = scipy.__version__
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info
        blas = [d for d in threadpool_info() if d.get("user_api") == "blas"]
        if blas:
            info["blas"] = f"{blas[0].get('internal_api')} {blas[0].get('version')}"
    except Exception:
        pass
    return info


def cpu_measure(wl, warmup, K, workers, instances, cfg2=True):
    """Time `instances` instances (cfg2) or the single instance over `workers`
    spawned processes, each at ONE BLAS/OpenMP thread (set in the environment
    the children start with, so OpenBLAS sizes its pool to 1 before numpy
    loads).  value = instances * n * K / wall of the whole pool."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    wl = dict(wl, cfg2=cfg2)
    K = min(K, wl["M"] - warmup)
    if not cfg2:
        instances, workers = 1, 1
    workers = max(1, min(workers, instances))
    chunks = [list(range(i, instances, workers)) for i in range(workers)]
    saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS",
                                            "MKL_NUM_THREADS")}
    for k in saved:
        os.environ[k] = "1"
    try:
        with ProcessPoolExecutor(max_workers=workers,
                                 mp_context=mp.get_context("spawn")) as ex:
            list(ex.map(_cpu_worker, [(wl, [], 0, 1)] * workers))   # start-up, imports
            t0 = time.perf_counter()
            res = list(ex.map(_cpu_worker, [(wl, c, warmup, K) for c in chunks]))
            wall = time.perf_counter() - t0
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    # wall of the pool includes each worker's untimed warm-up levels: use the
    # sum of the timed level walls of the busiest worker instead
    busiest = max(r[0] for r in res)
    value = instances * wl["n"] * K / busiest
    return value, busiest, K, sum(r[1] for r in res) / (instances * K), wall


def cpu_sample_text(instances, workers, warmup, K, avg_its, cfg2):
    who = (f"{instances} configs[2] instances (global indices 0..{instances - 1}) over "
           f"{workers} spawned processes" if cfg2 else "the single instance (one process)")
    return (who + f", each process at 1 OpenBLAS/OpenMP thread, levels {warmup + 1}.."
            f"{warmup + K} via oracle/ (numpy pocketfft/OpenBLAS restatement of "
            f"tsfrac.run_fids, same arithmetic); avg iterations {avg_its:.2f}")


# ------------------------------------------------------------- launcher
def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n: int, argv=None, executable=None, script=None) -> int:
    """Run this script as `n` ranks, one process per GPU, with the environment
    torchrun would give them (RANK, LOCAL_RANK, WORLD_SIZE, MASTER_ADDR =
    127.0.0.1, MASTER_PORT); NCCL's INFO log (communicator / NVLS lines) goes
    to each rank's stderr.  Only rank 0 prints the JSON line.  Returns the
    largest exit code."""
    argv = sys.argv[1:] if argv is None else argv
    port = str(free_port())
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        procs.append(subprocess.Popen([executable or sys.executable,
                                       str(script or Path(__file__).resolve())] + list(argv),
                                      env=env))
    rcs = [p.wait() for p in procs]
    return max(rcs)


# --------------------------------------------------------------------- GPU
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=509)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", default="cfg2", choices=["cfg0", "cfg1", "cfg2", "cfg3"])
    ap.add_argument("--gamma", type=float, default=0.0, help="override the workload's gamma")
    ap.add_argument("--alpha", type=float, default=0.0, help="override the workload's alpha")
    ap.add_argument("--batch", type=int, default=0, help="instances per rank")
    ap.add_argument("--cpu-workers", type=int, default=0)
    ap.add_argument("--cpu-instances", type=int, default=0,
                    help="configs[2] instances timed by the CPU legs (default max(64, cores))")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-matvec", action="store_true",
                    help="skip the standalone Toeplitz-product measurement")
    ap.add_argument("--tol", type=float, default=0.0,
                    help="experiments only: override the Krylov tolerance (not a bench number)")
    args = ap.parse_args()
    wl = workload(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    warmup = max(3, args.warmup)
    cfg2 = args.workload == "cfg2"

    if args.impl == "reference":
        if rank != 0:
            return
        # batched configs[2]: >= 64 instances over every host core (one
        # process per core, 1 BLAS thread each); the single-instance configs
        # are one march in one process (the reference cannot split a march)
        ncpu = os.cpu_count() or 1
        workers = (args.cpu_workers or ncpu) if cfg2 else 1
        inst = max(64, workers) if cfg2 else 1
        if args.cpu_instances:
            inst = args.cpu_instances
        K = min(args.steps, wl["cpu_levels"])
        value, busiest, K, avg_its, pool_wall = cpu_measure(wl, warmup, K, workers, inst, cfg2)
        workers = min(workers, inst)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": K, "warmup": warmup,
            "ms_per_step": busiest / K * 1e3 / max(1, inst // workers),
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": {"workload": wl["name"], "instances_sampled": inst, "n": wl["n"],
                       "M": wl["M"], "gamma": wl["gamma"], "alpha": wl["alpha"],
                       "tol": wl["tol"], "avg_iterations": avg_its},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                             "sample": cpu_sample_text(inst, workers, warmup, K, avg_its, cfg2),
                             "host": host_info(), "pool_wall_s": pool_wall},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    if world == 1 and args.gpus > 1:
        # the driver may call `bench.py --gpus N` without torchrun: launch the
        # N ranks here (one process per GPU, torchrun's environment)
        raise SystemExit(spawn_ranks(args.gpus))

    import torch
    import paper_2002_11978_b200 as P
    from paper_2002_11978_b200 import _native
    from paper_2002_11978_b200.scheme import FidsMarch, _field_separable

    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        if args.gpus > 1 and dist.get_world_size() != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {dist.get_world_size()}")
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    n, M, gam, alpha, B = wl["n"], wl["M"], wl["gamma"], wl["alpha"], wl["B"]
    r = (2.0 - gam) / gam
    N = n + 1
    if cfg2:
        from paper_2002_11978_b200 import workloads as WL
        x, kx, fx, u0 = WL.instance_fields(n, rank * B, B)   # weak scaling: B per rank
        kap = P.SeparableField([np.ones(n)], lambda t: [1.0 + 0.2 * t])
        src = P.SeparableField([np.ones(n)], lambda t: [1.0 + t])
        kmodes, fmodes = kx[None], fx[None]
    else:
        x = cfg0_fields(n)
        kap = P.SeparableField([np.ones(n), 0.5 * np.sin(np.pi * x)], lambda t: [1.0, math.exp(-t)])
        src = P.SeparableField([np.sin(np.pi * x)], lambda t: [1.0 + t])
        u0 = np.repeat(((1.0 - x * x) ** 2)[None, :], B, axis=0)
        if args.workload == "cfg3" and (world > 1 or B > 1):
            # configs[3] as seeded copies: phi * U_b per global copy (workloads.copy_scales)
            from paper_2002_11978_b200 import workloads as WL
            u0 = u0 * WL.copy_scales(rank * B, B)[:, None]
        kmodes = fmodes = None
    mesh = P.build_mesh(M, r, 1.0)
    soe = P.build_soe(gam, wl["eps"], (1.0 / M) ** r, 1.0)
    kdev = _field_separable(kap, x, mesh.t, B, kmodes, dev)
    fdev = _field_separable(src, x, mesh.t, B, fmodes, dev)
    u0_d = torch.from_numpy(np.ascontiguousarray(u0)).to(dev)
    if args.tol > 0:
        wl["tol"] = args.tol
    march = FidsMarch(gam, alpha, 1.0, 1.0, M, r, N, soe, method=0, precond=1, tol=wl["tol"],
                      max_iters=None, B=B, kappa=kdev, source=fdev, u0=u0_d, device=local)
    K = args.steps

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # segments of at most M levels; a new march (state reset) starts when one ends
    def plan_levels(start_level, count):
        segs, lvl = [], start_level
        while count > 0:
            if lvl > M:
                segs.append(("reset", 0))
                lvl = 1
            take = min(count, M - lvl + 1)
            segs.append(("run", take))
            lvl += take
            count -= take
        return segs

    march.reset()
    march.run(warmup)
    barrier()
    nev = 3 * K
    events = [torch.cuda.Event(enable_timing=True) for _ in range(nev)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    t_start.record()
    ev_i = 0
    its_sum = 0
    launches = 0
    levels_done = []
    for kind, cnt in plan_levels(warmup + 1, K):
        if kind == "reset":
            march.reset()
            continue
        m0 = march.next_level
        march.run(cnt, events=events[ev_i: ev_i + 3 * cnt])
        ev_i += 3 * cnt
        levels_done.append((m0, march.next_level))
    t_end.record()
    barrier()
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    if dist is not None:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    iters = march.iters.cpu().numpy()
    large = n > 4096
    fused = os.environ.get("TSF_FUSE_SOE") == "1" and not large
    graph = (os.environ.get("TSF_SOLVE_GRAPH", "1") != "0" and not fused
             and os.environ.get("TSF_SOLVE_PERSIST") != "1")
    for m0, m1 in levels_done:
        its_sum += int(iters[m0 - 1: m1 - 1].sum())
        # launches per level (tsf_abi.cu tsf_fids_march): SOE push + RHS
        # kernel (level 1 only when fused), counter init, then
        #   single-CTA engine: begin + (v, t) phase pair per iteration,
        #   large-n engine: begin, scalar, spectrum + 23 kernels per iteration,
        # iterations launched in chunks of 4 until every instance finished
        mx = iters[m0 - 1: m1 - 1].max(axis=1)
        if large and graph:
            # tsf_large.cu large_solve: set, begin, scalar, spectrum, then one
            # graph whose WHILE body is the 17-kernel iteration chain + loop test
            launches += int(np.sum(4 + 18 * np.maximum(mx, 1)))
        elif large:    # host-driven chunks of 4 iterations, 17 kernels each
            launches += int(np.sum(4 + 17 * 4 * np.ceil(np.maximum(mx, 1) / 4.0)))
        elif (os.environ.get("TSF_HALF", "1") != "0" and n >= 512 and n & (n - 1) == 0
              and not fused and int(os.environ.get("TSF_PERSIST_MAX_B", "1000000000")) >= B):
            # half-length persistent solve: counter init + ONE kernel per level
            # (csrc/tsf_half.cuh k_krylov_persist_h, tsf_dispatch_impl.cuh solve_t)
            launches += 2 * (m1 - m0)
        elif graph:    # one graph per level, G instance-group branches each
            # set, begin, WHILE { v, t, test } (csrc/tsf_dispatch_impl.cuh
            # solve_graph; G = solve_groups(B): TSF_SOLVE_GROUPS, default 4 for B >= 1024)
            genv = int(os.environ.get("TSF_SOLVE_GROUPS", "0") or 0)
            ng = min(8, genv if genv > 0 else (4 if B >= 1024 else 1), B)
            bg = -(-B // ng)
            ng = -(-B // bg)
            lv = iters[m0 - 1: m1 - 1]
            for g in range(ng):
                mxg = lv[:, g * bg:(g + 1) * bg].max(axis=1)
                launches += int(np.sum(2 + 3 * np.maximum(mxg, 1)))
        else:
            launches += int(np.sum(2 + 2 * 4 * np.ceil(np.maximum(mx, 1) / 4.0)))
        launches += (m1 - m0) if not fused else (1 if m0 == 1 else 0)
        launches += 1 if (m1 == M + 1 and not fused) else 0
    status = march.status.cpu().numpy()
    if np.any(status != 0):
        raise SystemExit(f"solver failure in the timed region: status {np.unique(status)}")
    soe_ms = sum(events[3 * i].elapsed_time(events[3 * i + 1]) for i in range(K))
    solve_ms = sum(events[3 * i + 1].elapsed_time(events[3 * i + 2]) for i in range(K))
    nexp = soe.n_exp
    # algorithmic bytes: BiCGSTAB iteration 216 n per instance (SURVEY.md
    # §8(d)); SOE push + RHS (16 N_exp + 32) n per instance (W read+write;
    # u, u_prev, f-mode read; rhs write)
    Kb = getattr(march, "soe_block", 1)
    if Kb > 1 and not fused:
        # blocked SOE (csrc/tsf_soe.cuh): level m = mb+1 runs the W pass
        # (W read+write, du ring reads, u^{mb}, u^{mb-1}, G ring writes, f, rhs),
        # the other levels k_soe_level (u^{m-1}, u^{m-2}, du write, G read,
        # du^{mb+1..m-2} reads, f, rhs); bytes averaged over the timed levels
        def _soe_level_bytes(m):
            mb = Kb * ((m - 1) // Kb)
            if m - 1 == mb:
                ka = 0 if mb == 0 else Kb
                kn = min(Kb, M - mb)
                wb = 0 if (ka == 0) else 16 * nexp
                return (wb + 8 * max(ka - 1, 0) + 16 + 8 * max(kn - 1, 0) + 16) * n * B
            return (16 + 8 + 8 + 8 * (m - 2 - mb) + 16) * n * B
        lv = [m for m0, m1 in levels_done for m in range(m0, m1)]
        soe_bytes = sum(_soe_level_bytes(m) for m in lv) / max(len(lv), 1)
    else:
        soe_bytes = (16 * nexp + 32) * n * B
    krylov_bytes = 216 * n * its_sum / K
    solve_bytes = krylov_bytes + (soe_bytes if fused else 0)
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    half = os.environ.get("TSF_HALF", "1") != "0"   # half-length engines (tsf_half.cuh, tsf_hlarge.cuh)
    if large and half and n & (n - 1) == 0 and n >= int(os.environ.get("TSF_HLARGE_MIN_N", 1 << 13)):
        n1 = max(64, (n // 2) >> 11)   # tsf_large.cu large_plan_init, half geometry
        sname = (f"tsf large-n level solve, half-length transforms: k_hcol_fwd/k_hcol_inv<{n1}> "
                 f"+ k_hrow_strang/k_hrow_mv<{n // 2 // n1}> + k_lsc/k_lel_xr "
                 "(19 kernels per BiCGSTAB iteration)")
    elif large:
        n1 = max(64, n >> 12)   # tsf_large.cu large_plan_init
        sname = (f"tsf large-n level solve: k_lcol_fwd/k_lcol_inv<{n1}> + k_lrow<{n // n1}> "
                 "+ k_lsc/k_lel_* (17 kernels per BiCGSTAB iteration)")
    else:
        hk = half and n >= 512 and n & (n - 1) == 0 and not fused
        hp = hk and int(os.environ.get("TSF_PERSIST_MAX_B", "1000000000")) >= B
        sname = ((f"tsf level solve: k_krylov_persist_h<{n},1> (half-length transforms, one "
                  f"persistent {n // 16}-thread CTA per instance runs the whole BiCGSTAB solve)"
                  if hp else
                  f"tsf level solve: k_solve_begin_h + k_bicg_h<{n},1|2> (half-length "
                  f"transforms, {n // 16}-thread CTAs)" if hk else
                  f"tsf level solve: k_solve_begin + k_bicg_v/k_bicg_t<{n},1>")
                 + (" with fused SOE epilogue" if fused else "")
                 + (" (one CUDA graph per level: instance-group branches, each a conditional "
                    "WHILE loop)" if graph and not hp else ""))
    k_solve = {"name": sname, "avg_ms": solve_ms / K,
               "GBps": solve_bytes / (solve_ms / K * 1e-3) / 1e9,
               "iterations_per_launch": its_sum / K, "algorithmic_bytes": solve_bytes}
    k_soe = {"name": (f"tsf::k_soe_block + k_soe_level (blocked SOE, one W pass per {Kb} levels)"
                      if Kb > 1 and not fused else
                      "tsf::k_soe_push_rhs" + (" (level 1 only)" if fused else "")),
             "avg_ms": soe_ms / K,
             "GBps": (soe_bytes / (soe_ms / K * 1e-3) / 1e9) if not fused else None,
             "algorithmic_bytes": soe_bytes}
    dom = k_solve if solve_ms >= soe_ms else k_soe
    # ncu DRAM bytes of the same kernels, from a capture of THIS build only
    # (profiles/ncu_traffic.json, keyed by workload and the sha256 of the kernel
    # sources — nvcc output is not bit-reproducible — or of the library file;
    # tools/ncu_traffic.py writes it): per instance-iteration of the level solve
    traffic, traffic_src = None, "no ncu capture of this build for this workload"
    try:
        tr = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())[args.workload]
        if (tr.get("src_sha256") == _native.src_sha256() and "TSF_LIB" not in os.environ) or \
                tr.get("lib_sha256") == _native.lib_sha256():
            traffic = (tr["dram_bytes_per_instance_iteration"] * its_sum / K
                       if dom is k_solve else tr["soe_dram_bytes_per_level"] * B / tr["B"])
            traffic_src = (f"ncu dram__bytes_read+write of the same kernels ({tr['capture']}) "
                           "x this launch's instance-iterations")
    except Exception:
        traffic = None
    roof = {"kernel": dom["name"], "bound": "hbm", "achieved": dom["GBps"], "peak": hbm,
            "unit": "GB/s", "frac": dom["GBps"] / hbm, "traffic": traffic,
            "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": dom["algorithmic_bytes"], "peak_source": peak_src,
            "share_of_step": (solve_ms if dom is k_solve else soe_ms) / ms,
            "note": ("large-n level solve: four-step transforms through L2/HBM"
                     if large else
                     "level solve is transform (shared-memory latency / FP64) bound "
                     "(profiles/r02/half_ncu.md); an instance's vectors stay in L2 between "
                     "its iterations (persistent CTA); the SOE kernel alone runs at ~98% of "
                     "the HBM peak")}
    # FP64 view of the same launch: algorithmic flops per BiCGSTAB iteration
    # (SURVEY.md §8(d)): 2 Toeplitz products (5 L log2 L + L + 3n each: two
    # real length-L transforms), 2 Strang solves (5 n log2 n + 3n), ~20n
    # vector flops; against the measured FP64 FMA peak (profiles/
    # r01_fp64_peak.json, tools/probes/fp64_peak.cu)
    Lemb = 1 << max(5, (2 * n - 1 - 1).bit_length())
    it_flops = (2 * (5 * Lemb * math.log2(Lemb) + Lemb + 3 * n)
                + 2 * (5 * n * math.log2(n) + 3 * n) + 20 * n)
    fp64_peak = 36.8
    try:
        fp64_peak = float(json.loads((ROOT / "profiles" / "r01_fp64_peak.json").read_text())
                          ["fp64_fma_tflops"])
    except Exception:
        pass
    solve_flops = it_flops * its_sum / K
    roof["fp64"] = {"algorithmic_flops_per_launch": solve_flops,
                    "achieved_tflops": solve_flops / (solve_ms / K * 1e-3) / 1e12,
                    "peak_tflops": fp64_peak,
                    "frac": solve_flops / (solve_ms / K * 1e-3) / 1e12 / fp64_peak,
                    "peak_source": "measured DFMA peak, profiles/r01_fp64_peak.json",
                    "note": "algorithmic flops count real-input transforms; the half-length "
                            "engine (DESIGN.md §3.8) runs about these flops, the full-length "
                            "one (TSF_HALF=0, PCG, non-power-of-two n) ~2x"}
    value = world * B * n * K / (ms * 1e-3)

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        u0_h = torch.from_numpy(np.ascontiguousarray(u0)).pin_memory()
        km_h = None if kmodes is None else torch.from_numpy(np.ascontiguousarray(kmodes)).pin_memory()
        fm_h = None if fmodes is None else torch.from_numpy(np.ascontiguousarray(fmodes)).pin_memory()
        levels = min(M, warmup + K)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        # result buffers a caller of the API would hold: pinned, allocated once
        u_out = torch.empty((B, n), dtype=torch.float64).pin_memory()
        its_out = torch.empty((levels, B), dtype=march.iters.dtype).pin_memory()
        rel_out = torch.empty((levels, B), dtype=march.relres.dtype).pin_memory()
        barrier()
        e0.record()
        h2d = u0_h.numel() * 8
        march.u0.copy_(u0_h, non_blocking=True)
        if km_h is not None:
            kdev.modes.copy_(km_h, non_blocking=True)
            fdev.modes.copy_(fm_h, non_blocking=True)
            h2d += (km_h.numel() + fm_h.numel()) * 8
        ev[0].record()
        march.reset()
        ev[1].record()
        march.run(levels)
        ev[2].record()
        u_out.copy_(march.u_level(march.next_level - 1), non_blocking=True)
        its_out.copy_(march.iters[:levels], non_blocking=True)
        rel_out.copy_(march.relres[:levels], non_blocking=True)
        ev[3].record()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1)
        e2e_parts = {"h2d_ms": e0.elapsed_time(ev[0]), "reset_ms": ev[0].elapsed_time(ev[1]),
                     "march_ms": ev[1].elapsed_time(ev[2]), "d2h_ms": ev[2].elapsed_time(ev[3])}
        if dist is not None:
            tt = torch.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        d2h = u_out.numel() * 8 + its_out.numel() * 4 + rel_out.numel() * 8
        e2e = {"value": world * B * n * levels / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": h2d / levels, "d2h_bytes_per_step": d2h / levels,
               "levels": levels, "parts": e2e_parts,
               "note": "pinned host u0 + coefficient modes -> device, march levels "
                       f"1..{levels}, final u + per-level iterations/residuals -> pinned host "
                       "buffers; device events around the whole region"}

    # ---- standalone Toeplitz matvec throughput (configs[4] point at this n, B*n=2^26)
    mv = None
    if rank == 0 and n <= (1 << 20) and not args.no_matvec:
        col = P.build_ifl(1.5, 1.75, 1.0, n + 1).first_col
        op = P.build_toeplitz(col)
        Bm = (1 << 26) // n
        xm = torch.randn(Bm, n, dtype=torch.float64, device=dev)
        km = torch.rand(Bm, n, dtype=torch.float64, device=dev) * 1.5 + 0.5
        ym = torch.empty_like(xm)
        lib = _native.load()
        st = _native.stream_ptr()
        lib.tsf_toeplitz_matvec(op.plan.handle, Bm, xm.data_ptr(), ym.data_ptr(), km.data_ptr(), 2.0, st)
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(5):
            lib.tsf_toeplitz_matvec(op.plan.handle, Bm, xm.data_ptr(), ym.data_ptr(), km.data_ptr(),
                                    2.0, st)
        a1.record()
        torch.cuda.synchronize()
        t_mv = a0.elapsed_time(a1) / 5 * 1e-3
        gbs = 24.0 * n * Bm / t_mv / 1e9
        mv = {"n": n, "B": Bm, "GBps": gbs, "frac_hbm": gbs / hbm, "ms": t_mv * 1e3}
        del xm, km, ym

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ncpu = os.cpu_count() or 1
        workers = (args.cpu_workers or ncpu) if cfg2 else 1
        inst = (args.cpu_instances or max(64, workers)) if cfg2 else 1
        cw = min(K, wl["cpu_levels"])
        cval, cbusy, cK, cits, _ = cpu_measure(wl, warmup, cw, workers, inst, cfg2)
        cpu = {"value": cval, "unit": UNIT, "cores": min(workers, inst), "kind": "port",
               "sample": cpu_sample_text(inst, min(workers, inst), warmup, cK, cits, cfg2),
               "host": host_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": warmup, "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded per instance, SURVEY.md §8(d))",
            "config": {"workload": wl["name"], "instances_per_gpu": B, "global_batch": B * world,
                       "n": n, "M": M, "gamma": gam, "alpha": alpha, "r": r, "n_exp": nexp,
                       "tol": wl["tol"], "soe_eps": wl["eps"],
                       "levels_timed": [list(v) for v in levels_done],
                       "avg_iterations": its_sum / (K * B),
                       "l2": "inputs larger than L2: W is %.1f GB per GPU" % (B * nexp * n * 8 / 1e9),
                       "parallelism": f"instances sharded over {world} GPU(s), no collectives"}
            | ({"copies": "phi * U_b, U_b ~ U[0.5, 2] per global copy (workloads.copy_scales)"}
               if args.workload == "cfg3" and (world > 1 or B > 1) else {}),
            "roofline": roof,
            "kernels": {"soe_push_rhs": k_soe, "level_solve": k_solve},
            "toeplitz_matvec": mv,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        # the only collective of the path: gather the final levels (untimed)
        from paper_2002_11978_b200 import workloads as WL
        WL.gather_rows(march.u_level(march.next_level - 1))
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
