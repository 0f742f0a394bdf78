#!/usr/bin/env python3
"""BASELINE configs[4] kernel micro-sweep on one GPU.

Toeplitz matvec y = d x + kappa (A x) and Strang preconditioner solve
z = P^{-1} v for n = 2^10 .. 2^24 with B = 2^26 / n instances (IFL
generator at alpha = 1.5, kappa ~ U[0.5, 2], inputs N(0, 1), seeded), and
the SOE push + RHS kernel for N_exp in {16, 32, 64} at n = 4096.
Each line: algorithmic GB/s (matvec 24 B/point: x, kappa read, y write;
preconditioner 16 B/point; SOE (16 N_exp + 40) B/point) and the fraction
of the HBM peak in MEASURED_PEAKS.json.  CUDA-event timing, warm-up first.

    python tools/micro_sweep.py [--out profiles/r01_micro_sweep.json]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2002_11978_b200 as P  # noqa: E402
from paper_2002_11978_b200 import _native  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--min-log", type=int, default=10)
    ap.add_argument("--max-log", type=int, default=24)
    args = ap.parse_args()
    try:
        hbm = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        hbm = 6650.0
    try:   # measured DFMA peak (tools/probes/fp64_peak.cu)
        fp64 = float(json.loads((ROOT / "profiles" / "r01_fp64_peak.json").read_text())
                     ["fp64_fma_tflops"])
    except Exception:
        fp64 = 36.8
    lib = _native.load()
    st = _native.stream_ptr()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(20021978)
    rows = []
    total = 1 << 26
    for lg in range(args.min_log, args.max_log + 1):
        n = 1 << lg
        B = total // n
        col = P.build_ifl(1.5, 1.75, 1.0, n + 1).first_col
        op = P.build_toeplitz(col)
        plan = op.plan
        x = torch.randn(B, n, dtype=torch.float64, device=dev, generator=g)
        kap = torch.rand(B, n, dtype=torch.float64, device=dev, generator=g) * 1.5 + 0.5
        y = torch.empty_like(x)
        reps = 5
        t_mv = timed(lambda: _native.check(lib.tsf_toeplitz_matvec(
            plan.handle, B, x.data_ptr(), y.data_ptr(), kap.data_ptr(), 2.0, st)), reps)
        t_pc = timed(lambda: _native.check(lib.tsf_precond_solve(
            plan.handle, B, x.data_ptr(), y.data_ptr(), 2.0, 1.25, None, st)), reps)
        r = {"kernel": "toeplitz_matvec", "n": n, "B": B, "ms": t_mv * 1e3,
             "GBps": 24.0 * n * B / t_mv / 1e9}
        r["frac_hbm"] = r["GBps"] / hbm
        q = {"kernel": "precond_solve", "n": n, "B": B, "ms": t_pc * 1e3,
             "GBps": 16.0 * n * B / t_pc / 1e9}
        q["frac_hbm"] = q["GBps"] / hbm
        # FP64 roofline (SURVEY.md §8(d) algorithmic flops: two real length-L
        # transforms per product, two real length-n transforms per Strang
        # solve) and the binding roof t_roof = max(bytes/HBM, flops/FP64)
        L = 2 * n
        for row, flops, byts, t in ((r, 5 * L * np.log2(L) + L + 3 * n, 24.0 * n, t_mv),
                                    (q, 5 * n * np.log2(n) + 3 * n, 16.0 * n, t_pc)):
            row["TFLOPs"] = flops * B / t / 1e12
            row["frac_fp64"] = row["TFLOPs"] / fp64
            t_roof = max(byts * B / (hbm * 1e9), flops * B / (fp64 * 1e12))
            row["bound"] = "fp64" if flops * B / (fp64 * 1e12) > byts * B / (hbm * 1e9) else "hbm"
            row["frac_roof"] = t_roof / t
        rows += [r, q]
        print(json.dumps(r), flush=True)
        print(json.dumps(q), flush=True)
        del x, kap, y, op, plan
        from paper_2002_11978_b200 import toeplitz as _tz
        _tz._plans.clear()                     # free this size's workspaces
        torch.cuda.empty_cache()
    n, B = 4096, 4096
    for nexp in (16, 32, 64):
        W = torch.randn(B, nexp, n, dtype=torch.float64, device=dev, generator=g)
        u = torch.randn(B, n, dtype=torch.float64, device=dev, generator=g)
        up = torch.randn(B, n, dtype=torch.float64, device=dev, generator=g)
        f = torch.randn(B, n, dtype=torch.float64, device=dev, generator=g)
        rhs = torch.empty_like(u)
        tab = torch.rand(3, nexp, dtype=torch.float64, device=dev, generator=g)
        t = timed(lambda: _native.check(lib.tsf_soe_push_rhs(
            B, n, nexp, W.data_ptr(), u.data_ptr(), up.data_ptr(), 1e-3, tab[0].data_ptr(),
            tab[1].data_ptr(), tab[2].data_ptr(), 1, 0, 1, 2.0, 1.7, f.data_ptr(),
            rhs.data_ptr(), st)), 5)
        s = {"kernel": "soe_push_rhs", "n": n, "B": B, "n_exp": nexp, "ms": t * 1e3,
             "GBps": (16.0 * nexp + 40.0) * n * B / t / 1e9}
        s["frac_hbm"] = s["GBps"] / hbm
        rows.append(s)
        print(json.dumps(s), flush=True)
        del W
        torch.cuda.empty_cache()
    if args.out:
        Path(args.out).write_text(json.dumps({"hbm_peak_gbs": hbm, "fp64_peak_tflops": fp64,
                                              "rows": rows}, indent=1) + "\n")


if __name__ == "__main__":
    main()
