"""Full-size goldens for BASELINE configs[2] and configs[3] (TEST INFRASTRUCTURE).

Runs only in the build container (imports the read-only reference `tsfrac`
from /root/reference/pkg/src).  For each case it runs the UNMODIFIED
reference `run_fids` twice: once stock (numpy pocketfft) and once with only
its FFT engine swapped to scipy.fft (tsfrac.fourier.fft/ifft) — the
reference's own noise floor, exactly as oracle/engine_swap_floor.py does for
configs[1].  Per-level BiCGSTAB iterations are recorded by rebinding
`tsfrac.scheme.solve_bicgstab` (scheme.py:31, :136-138).

Outputs (tests/golden/):
  cfg2_many.npz     48 configs[2] instances (n = 4096, M = 512): per-level
                    iterations, u^64 and u^M (stock run)
  cfg2_floor.json   per instance and pooled: stock vs swapped within-±1
                    fraction, mean Δ, max |Δ|, rel-l2 of u^M
  cfg3.npz          configs[3] (n = 2^20, M = 256, γ = 0.7, α = 1.2): all
                    256 per-level iteration counts, u at levels 1/64/128/256
                    sub-sampled every 16th point plus its full l2 norm, and
                    projections of u^M onto 4 seeded N(0,1) vectors
  cfg3_floor.json   the same comparison for configs[3]

    OPENBLAS_NUM_THREADS=1 python oracle/gen_fullsize.py [--only cfg2|cfg3]
"""
from __future__ import annotations

import os

os.environ["OPENBLAS_NUM_THREADS"] = "1"
os.environ["OMP_NUM_THREADS"] = "1"

import argparse  # noqa: E402
import json  # noqa: E402
import multiprocessing as mp  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

# 48 configs[2] global instance indices: the two of cfg2.npz plus 46 drawn
# from a fixed seed over the whole batch of 4096
CFG2_INSTANCES = sorted({37, 200} | set(
    np.random.default_rng(2002_11978 + 2).choice(4096, 46, replace=False).tolist()))
CFG3_LEVELS = (1, 64, 128, 256)
CFG3_SUB = 16          # sub-sampling stride of the stored configs[3] levels
CFG3_PROJ_SEED = 33


def _reference(swap):
    """The reference with its FFT engine as given: False = stock numpy
    pocketfft; True / "scipy" = scipy.fft (note: scipy's complex ifft is
    bit-identical to numpy's, only real-input forward transforms differ);
    "exact" = the correctly rounded DFT (scipy.fft in long double, rounded
    once to double) — the most accurate engine there is, so its spread
    against the stock run is the floor ANY accurate second engine sees."""
    from gen_golden import _import_reference
    tsfrac = _import_reference()
    if swap:
        import numpy as _np
        import scipy.fft as sf
        import tsfrac.fourier as fourier
        import tsfrac.toeplitz as tz
        if swap == "exact":
            fourier.fft = lambda x: sf.fft(_np.asarray(x).astype(_np.clongdouble)).astype(_np.complex128)
            fourier.ifft = lambda x: sf.ifft(_np.asarray(x).astype(_np.clongdouble)).astype(_np.complex128)
        else:
            fourier.fft = lambda x: sf.fft(x)
            fourier.ifft = lambda x: sf.ifft(x)
        tz.fourier = fourier
    return tsfrac


def _cfg2_one(args):
    b, swap = args
    tsfrac = _reference(swap)
    from gen_golden import _march
    from paper_2002_11978_b200 import workloads as WL
    from tsfrac.scheme import ProblemSpec
    n, M = 4096, 512
    x, kx, fx, u0 = WL.instance_fields(n, b, 1)
    spec = ProblemSpec(gamma=0.5, alpha=1.5, l=1.0, T=1.0,
                       kappa=lambda xx, t, k=kx[0]: k * (1.0 + 0.2 * t),
                       source=lambda xx, t, f=fx[0]: f * (1.0 + t),
                       initial=lambda xx, u=u0[0]: u.copy())
    t0 = time.time()
    hist, rep, its, rel = _march(tsfrac, spec, M, 3.0, n + 1, 1e-12, 1e-12)
    print(f"cfg2 b{b} swap={swap} avg {its.mean():.2f} {time.time() - t0:.0f}s", flush=True)
    return b, swap, its, hist[64].copy(), hist[-1].copy()


def cfg3_fields():
    kappa = lambda x, t: 1.0 + 0.5 * np.sin(np.pi * x) * np.exp(-t)  # noqa: E731
    source = lambda x, t: (1.0 + t) * np.sin(np.pi * x)  # noqa: E731
    initial = lambda x: (1.0 - x * x) ** 2  # noqa: E731
    return kappa, source, initial


def cfg3_projectors(n: int) -> np.ndarray:
    return np.random.default_rng(CFG3_PROJ_SEED).standard_normal((4, n))


def _cfg3_one(swap):
    tsfrac = _reference(swap)
    from tsfrac.scheme import ProblemSpec, SolverOptions, run_fids
    n, M, g, a = 1 << 20, 256, 0.7, 1.2
    kappa, source, initial = cfg3_fields()
    spec = ProblemSpec(gamma=g, alpha=a, l=1.0, T=1.0, kappa=kappa, source=source,
                       initial=initial)
    # keep_history would hold (M+1) x 2^20 doubles (2.2 GB): keep the wanted
    # levels from the solver's own return value (scheme.py:288 u = solve(...))
    import tsfrac.scheme as sch
    keep = {}
    its_l = []
    orig = sch.solve_bicgstab

    def rec(*a, **k):
        x, rep = orig(*a, **k)
        its_l.append(rep.iterations)
        if len(its_l) in CFG3_LEVELS:
            keep[len(its_l)] = np.array(x, copy=True)
        return x, rep

    sch.solve_bicgstab = rec
    t0 = time.time()
    try:
        uM, rep = run_fids(spec, M, (2.0 - g) / g, n + 1, epsilon=1e-12,
                           options=SolverOptions(solver="pkrylov", tol=1e-12),
                           keep_history=False)
    finally:
        sch.solve_bicgstab = orig
    assert np.array_equal(keep[M], uM)
    its = np.array(its_l)
    print(f"cfg3 swap={swap} avg {its.mean():.2f} {time.time() - t0:.0f}s", flush=True)
    return swap, its, keep


def _rl2(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


def _stats(d):
    return {"within1": float(np.mean(np.abs(d) <= 1)), "within2": float(np.mean(np.abs(d) <= 2)),
            "mean_d": float(d.mean()), "max_abs_d": int(np.abs(d).max())}


def run_cfg2(pool):
    res = pool.map(_cfg2_one, [(b, s) for b in CFG2_INSTANCES for s in (False, True)])
    stock = {b: r for b, s, *r in res if not s}
    swap = {b: r for b, s, *r in res if s}
    out = {"instances": np.array(CFG2_INSTANCES)}
    floor = {}
    all_d = []
    for b in CFG2_INSTANCES:
        its, u64, uM = stock[b]
        out[f"b{b}_its"] = its
        out[f"b{b}_uM"] = uM
        out[f"b{b}_u64"] = u64
        d = swap[b][0] - its
        all_d.append(d)
        floor[f"b{b}"] = dict(_stats(d), rel_l2_uM=_rl2(swap[b][2], uM),
                              rel_l2_u64=_rl2(swap[b][1], u64))
    allD = np.concatenate(all_d)
    floor["pooled"] = dict(_stats(allD),
                           min_within1=min(v["within1"] for k, v in floor.items()),
                           max_rel_l2_uM=max(v["rel_l2_uM"] for k, v in floor.items()))
    np.savez_compressed(OUT / "cfg2_many.npz", **out)
    (OUT / "cfg2_floor.json").write_text(json.dumps(floor, indent=1) + "\n")
    print("cfg2 floor pooled", floor["pooled"], flush=True)


def run_cfg2_exact(pool):
    """cfg2_floor.json gains per-instance and pooled stats of the correctly
    rounded engine against the stock run (the realistic floor)."""
    g = np.load(OUT / "cfg2_many.npz")
    floor = json.loads((OUT / "cfg2_floor.json").read_text())
    res = pool.map(_cfg2_one, [(int(b), "exact") for b in g["instances"]])
    all_d = []
    ex = {}
    for b, _, its, u64, uM in res:
        d = its - g[f"b{b}_its"]
        all_d.append(d)
        ex[f"b{b}"] = dict(_stats(d), rel_l2_uM=_rl2(uM, g[f"b{b}_uM"]),
                           rel_l2_u64=_rl2(u64, g[f"b{b}_u64"]))
    D = np.concatenate(all_d)
    ex["pooled"] = dict(_stats(D), min_within1=min(v["within1"] for v in ex.values()),
                        max_rel_l2_uM=max(v["rel_l2_uM"] for v in ex.values()))
    floor["exact_engine"] = ex
    (OUT / "cfg2_floor.json").write_text(json.dumps(floor, indent=1) + "\n")
    print("cfg2 exact-engine floor pooled", ex["pooled"], flush=True)


def _cfg0_exact(_):
    tsfrac = _reference("exact")
    from gen_golden import _march
    from tsfrac.scheme import ProblemSpec
    kappa, source, initial = cfg3_fields()
    spec = ProblemSpec(gamma=0.5, alpha=1.5, l=1.0, T=1.0, kappa=kappa, source=source,
                       initial=initial)
    hist, rep, its, rel = _march(tsfrac, spec, 256, 3.0, 1025, 1e-12, 1e-12)
    return its, hist


def _cfg1_exact(ga):
    g, a = ga
    tsfrac = _reference("exact")
    from gen_golden import _march
    from tsfrac.scheme import ProblemSpec
    kappa, source, initial = cfg3_fields()
    spec = ProblemSpec(gamma=g, alpha=a, l=1.0, T=1.0, kappa=kappa, source=source,
                       initial=initial)
    t0 = time.time()
    hist, rep, its, rel = _march(tsfrac, spec, 1024, (2.0 - g) / g, 16385, 1e-12, 1e-12)
    print(f"cfg1 g{g} a{a} exact avg {its.mean():.2f} {time.time() - t0:.0f}s", flush=True)
    return its, hist[64].copy(), hist[-1].copy()


def run_cfg0_exact(pool):
    """march.npz's configs[0] run vs the correctly rounded engine ->
    cfg0_floor.json (per-level iterations, max rel-l2 over all levels)."""
    gm = np.load(OUT / "march.npz")
    its, hist = pool.map(_cfg0_exact, [0])[0]
    d = its - gm["cfg0_its"]
    rl = max(_rl2(hist[m], gm["cfg0_hist"][m]) for m in range(1, hist.shape[0]))
    out = {"exact_engine": dict(_stats(d), max_rel_l2=rl)}
    (OUT / "cfg0_floor.json").write_text(json.dumps(out, indent=1) + "\n")
    print("cfg0 exact-engine floor", out, flush=True)


def run_cfg1_exact(pool):
    """cfg1_floor.json gains, per (gamma, alpha), the correctly rounded
    engine's spread against the stock run (cfg1.npz)."""
    g1 = np.load(OUT / "cfg1.npz")
    floor = json.loads((OUT / "cfg1_floor.json").read_text())
    combos = [(g, a) for g in (0.3, 0.5, 0.8) for a in (0.5, 1.0, 1.5, 1.9)]
    for (g, a), (its, u64, uM) in zip(combos, pool.map(_cfg1_exact, combos)):
        tag = f"cfg1_g{int(g * 10)}_a{int(a * 10)}"
        d = its - g1[f"{tag}_its"]
        floor[tag]["exact_engine"] = dict(_stats(d), rel_l2_u64=_rl2(u64, g1[f"{tag}_u64"]),
                                          rel_l2_uM=_rl2(uM, g1[f"{tag}_uM"]))
        print(tag, floor[tag]["exact_engine"], flush=True)
    (OUT / "cfg1_floor.json").write_text(json.dumps(floor, indent=1) + "\n")


def _linalg_exact(i):
    """One linalg.npz case's Krylov solves through the reference with the
    correctly rounded engine: iterations of the preconditioned BiCGSTAB at
    tol 1e-10 / 1e-12 and of the unpreconditioned solve at 1e-10."""
    tsfrac = _reference("exact")
    from tsfrac.krylov import MatrixFreeOperator, solve_bicgstab
    from tsfrac.toeplitz import build_preconditioner, build_toeplitz
    from tsfrac.ifl import build_ifl  # noqa: F401
    g = np.load(OUT / "linalg.npz")
    col = g[f"tp{i}_col"]
    n = col.size
    op = build_toeplitz(col)
    shift = float(g[f"tp{i}_shift"][0])
    kap = g[f"tp{i}_kappa"]
    apply = lambda q: shift * q + kap * op.matvec(q)  # noqa: E731
    out = {}
    # build_preconditioner takes the IFL discretisation in the reference;
    # restate its use: Strang column of the first column (toeplitz.py:101-128)
    from tsfrac.toeplitz import CirculantPreconditioner, strang_first_column
    import tsfrac.fourier as fourier
    lam = fourier.fft(strang_first_column(col)).real
    total = shift + float(kap.mean()) * lam
    pc = CirculantPreconditioner(n=n, shift=shift, kappa_bar=float(kap.mean()), lam=lam,
                                 total_eigs=total)
    for tol in (10, 12):
        _, rep = solve_bicgstab(MatrixFreeOperator(n, apply), pc, g[f"tp{i}_bicg_{tol}_b"],
                                tol=10.0 ** -tol)
        out[f"bicg_{tol}"] = rep.iterations
    _, rep = solve_bicgstab(MatrixFreeOperator(n, apply), None, g[f"tp{i}_bicg_12_b"], tol=1e-10)
    out["plain"] = rep.iterations
    return i, out


def run_linalg_exact(pool):
    g = np.load(OUT / "linalg.npz")
    cases = [i for i in range(32) if f"tp{i}_col" in g]
    res = dict(pool.map(_linalg_exact, cases))
    (OUT / "linalg_exact.json").write_text(json.dumps({f"tp{i}": v for i, v in res.items()},
                                                      indent=1) + "\n")
    print("linalg exact", res, flush=True)


def run_cfg3_exact(pool):
    """cfg3_floor.json gains the correctly rounded engine's spread against
    the stock run (cfg3.npz): all 256 levels' iterations and the stored
    levels (sub-sampled rel-l2, as the GPU test measures them)."""
    g = np.load(OUT / "cfg3.npz")
    floor = json.loads((OUT / "cfg3_floor.json").read_text())
    swap, its, keep = pool.map(_cfg3_one, ["exact"])[0]
    ex = dict(_stats(its - g["its"]))
    for m in CFG3_LEVELS:
        ex[f"rel_l2_u{m}_sub"] = _rl2(keep[m][::CFG3_SUB], g[f"u{m}_sub"])
        ex[f"rel_l2_u{m}"] = ex[f"rel_l2_u{m}_sub"]
    floor["exact_engine"] = ex
    (OUT / "cfg3_floor.json").write_text(json.dumps(floor, indent=1) + "\n")
    print("cfg3 exact-engine floor", ex, flush=True)


def run_cfg3(pool):
    res = dict((s, (its, keep)) for s, its, keep in pool.map(_cfg3_one, [False, True]))
    its, keep = res[False]
    its_s, keep_s = res[True]
    n = 1 << 20
    P = cfg3_projectors(n)
    out = {"its": its, "levels": np.array(CFG3_LEVELS), "sub": np.array([CFG3_SUB]),
           "proj_seed": np.array([CFG3_PROJ_SEED])}
    floor = dict(_stats(its_s - its))
    for m in CFG3_LEVELS:
        u = keep[m]
        out[f"u{m}_sub"] = u[::CFG3_SUB].copy()
        out[f"u{m}_norm"] = np.array([np.linalg.norm(u)])
        out[f"u{m}_proj"] = P @ u
        floor[f"rel_l2_u{m}"] = _rl2(keep_s[m], u)
        floor[f"rel_l2_u{m}_sub"] = _rl2(keep_s[m][::CFG3_SUB], u[::CFG3_SUB])
    np.savez_compressed(OUT / "cfg3.npz", **out)
    (OUT / "cfg3_floor.json").write_text(json.dumps(floor, indent=1) + "\n")
    print("cfg3 floor", floor, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg2,cfg3")
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    args = ap.parse_args()
    ctx = mp.get_context("spawn")
    which = args.only.split(",")
    with ctx.Pool(args.workers) as pool:
        if "cfg3" in which:
            a3 = pool.map_async(_cfg3_one, [False, True])
        if "cfg2" in which:
            run_cfg2(pool)
        if "cfg2exact" in which:
            run_cfg2_exact(pool)
        if "linalgexact" in which:
            run_linalg_exact(pool)
        if "cfg3exact" in which:
            run_cfg3_exact(pool)
        if "cfg0exact" in which:
            run_cfg0_exact(pool)
        if "cfg1exact" in which:
            run_cfg1_exact(pool)
        if "cfg3" in which:
            res = a3.get()

            class _P:
                @staticmethod
                def map(fn, xs):
                    return res
            run_cfg3(_P)


if __name__ == "__main__":
    main()
