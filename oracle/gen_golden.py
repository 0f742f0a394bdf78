"""Generate the golden fixtures in tests/golden/ from the UPSTREAM reference.

TEST INFRASTRUCTURE ONLY.  Runs only in the build container, where the
read-only reference lives at /root/reference/pkg/src.  It imports `tsfrac`
itself (not the oracle), runs it on seeded inputs and stores inputs and
outputs; tests/test_oracle_golden.py then pins oracle/tsfrac_oracle.py to
these vectors, and the -m gpu tests compare the CUDA path with them.

Per-step Krylov iteration counts are captured by rebinding
`tsfrac.scheme.solve_bicgstab` (imported by name at scheme.py:31 and called
at scheme.py:136-138) to a recording wrapper, as SURVEY.md §8(c) describes.

Usage (OPENBLAS_NUM_THREADS=1 is forced below):
    python oracle/gen_golden.py [--big]
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import argparse  # noqa: E402
import math  # noqa: E402
import sys  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
SEED = 20240817  # the reference's own fixture seed, pkg/tests/conftest.py:5-7


def _import_reference():
    if not REF.is_dir():
        raise SystemExit("reference tree not present; fixtures are committed")
    sys.path.insert(0, str(REF))
    import tsfrac  # noqa: F401
    return tsfrac


class Recorder:
    def __init__(self, scheme_mod):
        self.mod = scheme_mod
        self.orig = scheme_mod.solve_bicgstab
        self.orig_cg = scheme_mod.solve_cg
        self.its, self.rel = [], []

    def __enter__(self):
        def wrap(fn):
            def inner(*a, **k):
                x, rep = fn(*a, **k)
                self.its.append(rep.iterations)
                self.rel.append(rep.final_relative_residual)
                return x, rep
            return inner
        self.mod.solve_bicgstab = wrap(self.orig)
        self.mod.solve_cg = wrap(self.orig_cg)
        return self

    def __exit__(self, *exc):
        self.mod.solve_bicgstab = self.orig
        self.mod.solve_cg = self.orig_cg


def cfg0_fields():
    """BASELINE.json configs[0] coefficient fields."""
    kappa = lambda x, t: 1.0 + 0.5 * np.sin(np.pi * x) * np.exp(-t)  # noqa: E731
    source = lambda x, t: (1.0 + t) * np.sin(np.pi * x)  # noqa: E731
    initial = lambda x: (1.0 - x * x) ** 2  # noqa: E731
    return kappa, source, initial


def gen_setup(tsfrac):
    from tsfrac.ifl import build_ifl
    from tsfrac.mesh import build_mesh, l1_weights
    from tsfrac.soe import build_soe

    out = {}
    # meshes + L1 rows (mesh.py:37-80)
    for tag, (M, r) in {"m8r2": (8, 2.0), "m256r3": (256, 3.0),
                        "m512r3": (512, 3.0), "m64r1": (64, 1.0)}.items():
        mesh = build_mesh(M, r, 1.0)
        out[f"mesh_{tag}_t"] = mesh.t
        out[f"mesh_{tag}_tau"] = mesh.tau
        for m in sorted({1, 2, M // 2, M}):
            out[f"mesh_{tag}_l1_g05_m{m}"] = l1_weights(mesh, 0.5, m).a
            out[f"mesh_{tag}_l1_g08_m{m}"] = l1_weights(mesh, 0.8, m).a
    # IFL columns (ifl.py:73-115)
    ifl_cases = [(1.5, 1.75, 1.0, 1025), (0.5, 1.25, 1.0, 65), (1.9, 1.95, 1.0, 64),
                 (1.2, 1.6, 1.0, 4097), (1.6, 2.0, 1.0, 33), (1.0, 1.5, 2.0, 17),
                 (1.5, 1.75, 1.0, 16385)]
    for i, (a, mu, l, N) in enumerate(ifl_cases):
        d = build_ifl(a, mu, l, N)
        out[f"ifl{i}_args"] = np.array([a, mu, l, N], dtype=float)
        out[f"ifl{i}_col"] = d.first_col
        out[f"ifl{i}_hscale"] = np.array([d.h, d.scale, d.c_norm])
    # SOE (soe.py:145-184): BASELINE configs and the reference test regimes
    soe_cases = {
        "cfg0": (0.5, 1e-12, (1.0 / 256) ** 3.0, 1.0),
        "cfg1_g03": (0.3, 1e-12, (1.0 / 1024) ** ((2 - 0.3) / 0.3), 1.0),
        "cfg1_g05": (0.5, 1e-12, (1.0 / 1024) ** 3.0, 1.0),
        "cfg1_g08": (0.8, 1e-12, (1.0 / 1024) ** ((2 - 0.8) / 0.8), 1.0),
        "cfg2": (0.5, 1e-12, (1.0 / 512) ** 3.0, 1.0),
        "cfg3": (0.7, 1e-12, (1.0 / 256) ** ((2 - 0.7) / 0.7), 1.0),
        "t_half": (0.5, 1e-10, 1e-4, 1.0),
        "t_ex2": (0.8, 1e-9, (1.0 / 2 ** 8) ** 3, 1.0),
        "t_pos": (0.3, 1e-8, 1e-3, 2.0),
    }
    for tag, (g, e, dl, T) in soe_cases.items():
        soe = build_soe(g, e, dl, T)
        out[f"soe_{tag}_args"] = np.array([g, e, dl, T])
        out[f"soe_{tag}_s"] = soe.nodes
        out[f"soe_{tag}_w"] = soe.weights
    return out


def gen_linear_algebra(tsfrac):
    from tsfrac.ifl import build_ifl
    from tsfrac.krylov import MatrixFreeOperator, solve_bicgstab, solve_cg
    from tsfrac.toeplitz import (build_preconditioner, build_toeplitz,
                                 precond_solve, strang_first_column,
                                 toeplitz_matvec)

    rng = np.random.default_rng(SEED)
    out = {}
    # Toeplitz matvec / Strang preconditioner on IFL columns, pow2 and not
    for i, (a, N) in enumerate([(1.5, 1025), (1.5, 4097), (0.5, 257), (1.9, 65),
                                (1.2, 64), (1.5, 101), (1.5, 17), (1.5, 8193)]):
        d = build_ifl(a, 1.0 + a / 2.0, 1.0, N)
        n = N - 1
        op = build_toeplitz(d.first_col)
        v = rng.standard_normal(n)
        kappa = rng.uniform(0.5, 2.0, n)
        shift = float(rng.uniform(1.0, 50.0))
        out[f"tp{i}_col"] = d.first_col
        out[f"tp{i}_v"] = v
        out[f"tp{i}_kappa"] = kappa
        out[f"tp{i}_shift"] = np.array([shift])
        if n <= 1024:
            out[f"tp{i}_spec"] = op.spectrum_embed
        out[f"tp{i}_Av"] = toeplitz_matvec(op, v)
        out[f"tp{i}_Mv"] = shift * v + kappa * op.matvec(v)
        p = build_preconditioner(d, shift, float(kappa.mean()))
        out[f"tp{i}_cs"] = strang_first_column(d.first_col)
        out[f"tp{i}_lam"] = p.lam
        out[f"tp{i}_total"] = p.total_eigs
        out[f"tp{i}_Pinv_v"] = precond_solve(p, v)
        # one full level solve (pkrylov branch, scheme.py:120-143)
        b = rng.standard_normal(n)
        apply = lambda q, s=shift, k=kappa, o=op: s * q + k * o.matvec(q)  # noqa: E731
        for tol in (1e-10, 1e-12):
            x, rep = solve_bicgstab(MatrixFreeOperator(n, apply), p, b, tol=tol)
            key = f"tp{i}_bicg_{int(-math.log10(tol))}"
            out[f"{key}_b"] = b
            out[f"{key}_x"] = x
            out[f"{key}_rep"] = np.array([rep.iterations, rep.final_relative_residual,
                                          float(rep.converged)])
        # CG on the x-independent variant (kappa constant)
        kc = float(kappa.mean())
        apply_c = lambda q, s=shift, k=kc, o=op: s * q + k * o.matvec(q)  # noqa: E731
        pc = build_preconditioner(d, shift, kc)
        x, rep = solve_cg(MatrixFreeOperator(n, apply_c), pc, b, tol=1e-12)
        out[f"tp{i}_cg_kc"] = np.array([kc])
        out[f"tp{i}_cg_x"] = x
        out[f"tp{i}_cg_rep"] = np.array([rep.iterations, rep.final_relative_residual,
                                         float(rep.converged)])
        # unpreconditioned ("krylov") solve
        x, rep = solve_bicgstab(MatrixFreeOperator(n, apply), None, b, tol=1e-10)
        out[f"tp{i}_plain_x"] = x
        out[f"tp{i}_plain_rep"] = np.array([rep.iterations, rep.final_relative_residual,
                                            float(rep.converged)])
    # SOE push / history term KATs on random state (soe.py:209-246)
    from tsfrac.soe import FastHistory, build_soe, fast_caputo_rhs, history_push
    soe = build_soe(0.5, 1e-12, (1.0 / 256) ** 3, 1.0)
    h = FastHistory.fresh(soe, 256)
    h.W[:] = rng.standard_normal(h.W.shape)
    out["push_W0"] = h.W.copy()
    du = rng.standard_normal(256)
    u_prev = rng.standard_normal(256)
    out["push_du"] = du
    out["push_uprev"] = u_prev
    out["push_tau"] = np.array([3.7e-4, 1.1e-2])
    out["push_rhs"] = fast_caputo_rhs(h, 12.5, u_prev, 0.5, 1.1e-2)
    history_push(h, du, 3.7e-4)
    out["push_W1"] = h.W.copy()
    return out


def _march(tsfrac, spec, M, r, N, eps, tol, solver="pkrylov", keep=True):
    from tsfrac.scheme import SolverOptions, run_fids
    with Recorder(tsfrac.scheme) as rec:
        hist, rep = run_fids(spec, M, r, N, epsilon=eps,
                             options=SolverOptions(solver=solver, tol=tol),
                             keep_history=keep)
    return hist, rep, np.array(rec.its), np.array(rec.rel)


def gen_marches(tsfrac):
    from tsfrac.scheme import ProblemSpec

    out = {}
    kappa, source, initial = cfg0_fields()
    # cfg0 at full size (BASELINE.json configs[0]): n=1024, M=256
    spec = ProblemSpec(gamma=0.5, alpha=1.5, l=1.0, T=1.0, kappa=kappa,
                       source=source, initial=initial)
    hist, rep, its, rel = _march(tsfrac, spec, 256, 3.0, 1025, 1e-12, 1e-12)
    out["cfg0_hist"] = hist
    out["cfg0_its"] = its
    out["cfg0_rel"] = rel
    out["cfg0_avg"] = np.array([rep.avg_iterations])
    # small marches: pow2 and non-pow2 n, both alphas regimes
    cases = {
        "s1": (0.5, 1.5, 64, 129, 1e-12),   # n=128
        "s2": (0.8, 1.9, 32, 65, 1e-10),    # n=64
        "s3": (0.3, 0.5, 48, 257, 1e-12),   # n=256
        "s4": (0.5, 1.5, 32, 64, 1e-12),    # n=63 (reference convention)
        "s5": (0.7, 1.2, 40, 513, 1e-12),   # n=512
    }
    for tag, (g, a, M, N, tol) in cases.items():
        spec = ProblemSpec(gamma=g, alpha=a, l=1.0, T=1.0, kappa=kappa,
                           source=source, initial=initial)
        r = (2.0 - g) / g
        hist, rep, its, rel = _march(tsfrac, spec, M, r, N, 1e-12, tol)
        out[f"{tag}_args"] = np.array([g, a, M, N, tol, r])
        out[f"{tag}_hist"] = hist
        out[f"{tag}_its"] = its
        out[f"{tag}_rel"] = rel
    # unpreconditioned + CG branches, small
    spec = ProblemSpec(gamma=0.5, alpha=1.5, l=1.0, T=1.0, kappa=kappa,
                       source=source, initial=initial)
    hist, rep, its, rel = _march(tsfrac, spec, 16, 3.0, 129, 1e-12, 1e-10, solver="krylov")
    out["plain_hist"], out["plain_its"] = hist, its
    spec_cg = ProblemSpec(gamma=0.5, alpha=1.5, l=1.0, T=1.0,
                          kappa=lambda x, t: np.full_like(x, 1.0 + 0.5 * t),
                          source=source, initial=initial, kappa_x_independent=True)
    hist, rep, its, rel = _march(tsfrac, spec_cg, 16, 3.0, 257, 1e-12, 1e-12)
    out["cg_hist"], out["cg_its"] = hist, its
    # zero data -> exactly zero (pkg/tests/test_scheme.py:29-34), pkrylov branch
    spec0 = ProblemSpec(gamma=0.5, alpha=1.5, l=1.0, T=1.0,
                        kappa=lambda x, t: np.ones_like(x),
                        source=lambda x, t: np.zeros_like(x),
                        initial=lambda x: np.zeros_like(x))
    hist, rep, its, rel = _march(tsfrac, spec0, 8, 2.0, 257, 1e-10, 1e-10)
    out["zero_hist"], out["zero_its"] = hist, its
    return out


def gen_dids(tsfrac):
    """run_dids (scheme.py:184-233): per-level history + iteration counts for
    pow2 / non-pow2 n and the dense branch, plus the FIDS march of the same
    case (the reference's FIDS-DIDS proximity criterion,
    pkg/tests/test_acceptance.py:141-166)."""
    from tsfrac.scheme import ProblemSpec, SolverOptions, run_dids
    kappa, source, initial = cfg0_fields()
    out = {}
    cases = {
        "d1": (0.5, 1.5, 64, 257, 1e-12, "pkrylov"),   # n=256
        "d2": (0.3, 1.2, 32, 101, 1e-12, "pkrylov"),   # n=100 (non-pow2)
        "d3": (0.8, 1.9, 24, 129, 1e-10, "krylov"),    # n=128 unpreconditioned
        "d4": (0.5, 1.5, 16, 65, 1e-12, "auto"),       # n=64 -> dense branch
    }
    for tag, (g, a, M, N, tol, solver) in cases.items():
        spec = ProblemSpec(gamma=g, alpha=a, l=1.0, T=1.0, kappa=kappa,
                           source=source, initial=initial)
        r = (2.0 - g) / g
        with Recorder(tsfrac.scheme) as rec:
            hist, rep = run_dids(spec, M, r, N, options=SolverOptions(solver=solver, tol=tol))
        out[f"{tag}_args"] = np.array([g, a, M, N, tol, r])
        out[f"{tag}_solver"] = np.array(solver)
        out[f"{tag}_hist"] = hist
        out[f"{tag}_its"] = np.array(rec.its, dtype=np.int64)
        out[f"{tag}_avg"] = np.array([rep.avg_iterations])
        out[f"{tag}_ops"] = rep.history_ops
        hf, _, _, _ = _march(tsfrac, spec, M, r, N, 1e-12, tol, solver=solver)
        out[f"{tag}_fids_hist"] = hf
    return out


def gen_cfg2(tsfrac):
    """Two configs[2] instances (global indices 37 and 200 of the seeded
    batch, paper_2002_11978_b200/workloads.py) at full size: n = 4096,
    M = 512, gamma = 0.5, alpha = 1.5, SOE eps 1e-12, tol 1e-12 — per-level
    iterations and u^M from the reference's own run_fids."""
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_2002_11978_b200 import workloads as WL
    from tsfrac.scheme import ProblemSpec
    out = {}
    n, M = 4096, 512
    for b in (37, 200):
        x, kx, fx, u0 = WL.instance_fields(n, b, 1)
        spec = ProblemSpec(gamma=0.5, alpha=1.5, l=1.0, T=1.0,
                           kappa=lambda xx, t, k=kx[0]: k * (1.0 + 0.2 * t),
                           source=lambda xx, t, f=fx[0]: f * (1.0 + t),
                           initial=lambda xx, u=u0[0]: u.copy())
        hist, rep, its, rel = _march(tsfrac, spec, M, 3.0, n + 1, 1e-12, 1e-12)
        out[f"b{b}_its"] = its
        out[f"b{b}_uM"] = hist[-1]
        out[f"b{b}_u64"] = hist[64]
    return out


def gen_big(tsfrac):
    """cfg1 (n=16384, M=1024) for all 12 (gamma, alpha): per-step its + u^M."""
    from concurrent.futures import ProcessPoolExecutor
    combos = [(g, a) for g in (0.3, 0.5, 0.8) for a in (0.5, 1.0, 1.5, 1.9)]
    out = {}
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        for (g, a), res in zip(combos, ex.map(_cfg1_one, combos)):
            tag = f"cfg1_g{int(g * 10)}_a{int(a * 10)}"
            out[f"{tag}_its"], out[f"{tag}_uM"], out[f"{tag}_u64"] = res
    return out


def _cfg1_one(ga):
    g, a = ga
    tsfrac = _import_reference()
    from tsfrac.scheme import ProblemSpec
    kappa, source, initial = cfg0_fields()
    spec = ProblemSpec(gamma=g, alpha=a, l=1.0, T=1.0, kappa=kappa,
                       source=source, initial=initial)
    hist, rep, its, rel = _march(tsfrac, spec, 1024, (2.0 - g) / g, 16385, 1e-12, 1e-12)
    return its, hist[-1], hist[64]


# Acceptance-gate runs (pkg/tests/test_acceptance.py:38-166): every scheme
# configuration of criteria 1-7 with the reference's own err_inf / average
# iterations / final level, plus the manufactured-problem functions
# (pkg/src/tsfrac/problems.py) tabulated for tests/test_problems.py.
ACCEPTANCE_RUNS = [
    # label, scheme, case, alpha, gamma, r, mu, M or None, N or None, q, eps, solver, tol
    ("c1_M128", "both", "example1", 1.5, 0.5, 2, None, 2 ** 7, None, 2, 1e-10, "auto", 1e-10),
    ("c1_M256", "both", "example1", 1.5, 0.5, 2, None, 2 ** 8, None, 2, 1e-10, "auto", 1e-10),
    ("c1_M512", "both", "example1", 1.5, 0.5, 2, None, 2 ** 9, None, 2, 1e-10, "auto", 1e-10),
    ("c1_M1024", "both", "example1", 1.5, 0.5, 2, None, 2 ** 10, None, 2, 1e-10, "auto", 1e-10),
    ("c2_M512", "dids", "example1", 1.6, 0.8, 3, 2.0, 2 ** 9, None, 2, 1e-10, "auto", 1e-10),
    ("c2_M1024", "dids", "example1", 1.6, 0.8, 3, 2.0, 2 ** 10, None, 2, 1e-10, "auto", 1e-10),
    ("c3_N8", "dids", "example1", 1.5, 0.8, 1, None, None, 8, 2, 1e-10, "auto", 1e-10),
    ("c3_N16", "dids", "example1", 1.5, 0.8, 1, None, None, 16, 2, 1e-10, "auto", 1e-10),
    ("c3_N32", "dids", "example1", 1.5, 0.8, 1, None, None, 32, 2, 1e-10, "auto", 1e-10),
    ("c3_N64", "dids", "example1", 1.5, 0.8, 1, None, None, 64, 2, 1e-10, "auto", 1e-10),
    ("c4_N9", "dids", "example2", 1.9, 0.8, 3, None, None, 9, 1.95, 1e-10, "auto", 1e-10),
    ("c4_N18", "dids", "example2", 1.9, 0.8, 3, None, None, 18, 1.95, 1e-10, "auto", 1e-10),
    ("c4_N36", "dids", "example2", 1.9, 0.8, 3, None, None, 36, 1.95, 1e-10, "auto", 1e-10),
    ("c4_N72", "dids", "example2", 1.9, 0.8, 3, None, None, 72, 1.95, 1e-10, "auto", 1e-10),
    ("c5_N256", "fids", "example2", 0.5, 0.5, 2, None, None, 2 ** 8, 1.25, 1e-9, "auto", 1e-10),
    ("c5_N512", "fids", "example2", 0.5, 0.5, 2, None, None, 2 ** 9, 1.25, 1e-9, "auto", 1e-10),
    ("c6_plain_N256", "fids", "example2", 1.9, 0.5, 2, None, None, 2 ** 8, 1.95, 1e-9, "krylov", 1e-10),
    ("c6_prec_N64", "fids", "example2", 1.9, 0.5, 2, None, None, 2 ** 6, 1.95, 1e-9, "pkrylov", 1e-10),
    ("c6_prec_N128", "fids", "example2", 1.9, 0.5, 2, None, None, 2 ** 7, 1.95, 1e-9, "pkrylov", 1e-10),
    ("c6_prec_N256", "fids", "example2", 1.9, 0.5, 2, None, None, 2 ** 8, 1.95, 1e-9, "pkrylov", 1e-10),
]


def gen_acceptance(tsfrac):
    import time

    from tsfrac.couplings import m_from_n, n_from_m
    from tsfrac.problems import make_case
    from tsfrac.scheme import SolverOptions, run_dids, run_fids

    out = {}
    xs = np.concatenate([np.linspace(-1.0, 1.0, 41), [-0.999, 0.3333, 0.999]])
    for i, (name, a, g) in enumerate([("example1", 1.5, 0.5), ("example1", 1.6, 0.8),
                                      ("example2", 1.9, 0.8), ("example2", 0.5, 0.5),
                                      ("example1", 1.5, 0.8), ("example2", 1.9, 0.5)]):
        case = make_case(name, a, g)
        out[f"fn{i}_args"] = np.array([a, g, case.s])
        out[f"fn{i}_name"] = np.array(name)
        out[f"fn{i}_x"] = xs
        out[f"fn{i}_initial"] = case.spec.initial(xs)
        for j, t in enumerate((0.0, 0.37, 1.0)):
            out[f"fn{i}_source_t{j}"] = case.spec.source(xs, t)
            out[f"fn{i}_exact_t{j}"] = case.spec.exact(xs, t)
            out[f"fn{i}_kappa_t{j}"] = case.spec.kappa(xs, t)
    labels = []
    for (label, scheme, name, a, g, r, mu, M, N, q, eps, solver, tol) in ACCEPTANCE_RUNS:
        if N is None:
            N = n_from_m(M, r, g, q)
        else:
            M = m_from_n(N, r, g, q)
        case = make_case(name, a, g)
        opts = SolverOptions(solver=solver, tol=tol)
        t0 = time.perf_counter()
        row = [M, N, np.nan, np.nan, np.nan, np.nan]
        if scheme in ("dids", "both"):
            h, rep = run_dids(case.spec, M, r, N, mu=mu, options=opts)
            row[2] = rep.err_inf
            out[f"acc_{label}_dids_uM"] = h[-1]
        if scheme in ("fids", "both"):
            with Recorder(tsfrac.scheme) as rec:
                h, rep = run_fids(case.spec, M, r, N, epsilon=eps, mu=mu, options=opts)
            row[3] = rep.err_inf
            row[4] = rep.avg_iterations
            out[f"acc_{label}_fids_uM"] = h[-1]
            if rec.its:
                out[f"acc_{label}_fids_its"] = np.array(rec.its, dtype=np.int64)
        row[5] = time.perf_counter() - t0
        out[f"acc_{label}"] = np.array(row, dtype=float)
        labels.append(label)
        print(label, row, flush=True)
    out["acc_labels"] = np.array(labels)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run cfg1 (minutes)")
    ap.add_argument("--only", default="", help="comma list of fixtures to regenerate "
                    "(setup,linalg,march,dids,cfg1,cfg2,acceptance); default all but cfg1/cfg2")
    args = ap.parse_args()
    tsfrac = _import_reference()
    OUT.mkdir(parents=True, exist_ok=True)
    if args.only:
        gens = {"setup": gen_setup, "linalg": gen_linear_algebra, "march": gen_marches,
                "dids": gen_dids, "cfg1": gen_big, "cfg2": gen_cfg2,
                "acceptance": gen_acceptance}
        for name in args.only.split(","):
            np.savez_compressed(OUT / f"{name}.npz", **gens[name](tsfrac))
            print(name, (OUT / f"{name}.npz").stat().st_size)
        return
    np.savez_compressed(OUT / "setup.npz", **gen_setup(tsfrac))
    np.savez_compressed(OUT / "linalg.npz", **gen_linear_algebra(tsfrac))
    np.savez_compressed(OUT / "march.npz", **gen_marches(tsfrac))
    np.savez_compressed(OUT / "dids.npz", **gen_dids(tsfrac))
    if args.big:
        np.savez_compressed(OUT / "cfg1.npz", **gen_big(tsfrac))
    meta = {"numpy": np.__version__, "seed": SEED,
            "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS")}
    import scipy
    meta["scipy"] = scipy.__version__
    (OUT / "README.md").write_text(
        "Golden vectors produced by `python oracle/gen_golden.py` from the upstream\n"
        "reference (`/root/reference/pkg/src/tsfrac`, read-only, build container only).\n\n"
        + "\n".join(f"- {k}: {v}" for k, v in meta.items()) + "\n")
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
