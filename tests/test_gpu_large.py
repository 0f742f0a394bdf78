"""GPU parity of the large-n (four-step) engine, n = 2^13 .. 2^24.

Same bars as test_gpu_parity.py: matvec / preconditioner within 1e-13
relative (max-abs / max) of the oracle, level solves within the reference's
own FFT-engine-swap floor, the BASELINE configs[1] march (n = 16384,
M = 1024, tol 1e-12) against the reference goldens (tests/golden/cfg1.npz).
"""

import math

import numpy as np
import pytest

import oracle as O
from tsf_testlib import cfg0_fields, golden, rel_err, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2002_11978_b200 as P  # noqa: E402


def _col(n, alpha=1.5):
    return O.ifl_column(alpha, 1.0 + alpha / 2.0, 1.0, n + 1)[0]


def _grid(n):
    return -1.0 + (2.0 / (n + 1)) * np.arange(1, n + 1)


def _kappa(n, seed=0):
    rng = np.random.default_rng(seed)
    x = _grid(n)
    return 1.0 + 0.5 * rng.uniform(0.2, 1.0) * np.sin(np.pi * x) ** 2


# configs[4] spans n = 2^10..2^24: the four-step engine's sizes up to the top
@pytest.mark.parametrize("n", [8192, 16384, 65536, 1 << 20, 1 << 22, 1 << 24])
def test_large_matvec_vs_oracle(n):
    rng = np.random.default_rng(n)
    col = _col(n)
    v = rng.standard_normal(n)
    L, sym = O.toeplitz_symbol(col)
    want = O.toeplitz_apply(sym, v)
    op = P.build_toeplitz(col)
    got = P.toeplitz_matvec(op, v)
    assert rel_err(got, want) <= 1e-13
    kap = _kappa(n, 1)
    got = P.toeplitz_matvec(op, v, kappa=kap, shift=37.5)
    assert rel_err(got, 37.5 * v + kap * want) <= 1e-13


def test_large_matvec_batched_and_unit_vector():
    n = 8192
    rng = np.random.default_rng(3)
    col = rng.standard_normal(n) / (1.0 + np.arange(n))
    op = P.build_toeplitz(col)
    e1 = np.zeros(n)
    e1[0] = 1.0
    out = P.toeplitz_matvec(op, e1)                       # A e1 = first column
    assert np.max(np.abs(out - col)) <= 1e-13 * np.abs(col).max()
    V = rng.standard_normal((3, n))
    got = P.toeplitz_matvec(op, V)
    L, sym = O.toeplitz_symbol(col)
    for b in range(3):
        assert rel_err(got[b], O.toeplitz_apply(sym, V[b])) <= 1e-13


@pytest.mark.parametrize("n", [8192, 65536, 1 << 20, 1 << 22, 1 << 24])
def test_large_precond_vs_oracle(n):
    rng = np.random.default_rng(n + 1)
    col = _col(n)
    shift, kbar = 41.0, 1.3
    p = P.build_preconditioner(col, shift, kbar)
    total = shift + kbar * O.strang_eigs(col)
    v = rng.standard_normal(n)
    got = P.precond_solve(p, v)
    assert rel_err(got, O.precond_apply(total, v)) <= 1e-13


def _level(n, seed, shift=36.0):
    col = _col(n)
    kap = _kappa(n, seed)
    rng = np.random.default_rng(seed + 100)
    x = _grid(n)
    b = np.sin(np.pi * x) * (1.0 + 0.1 * rng.standard_normal(n))
    return col, kap, shift, b


def _oracle_solve(col, kap, shift, b, tol, pc=True):
    L, sym = O.toeplitz_symbol(col)
    total = shift + float(kap.mean()) * O.strang_eigs(col)
    apply = lambda q: shift * q + kap * O.toeplitz_apply(sym, q)  # noqa: E731
    ps = (lambda q: O.precond_apply(total, q)) if pc else None
    return O.bicgstab(apply, ps, b, tol=tol)


@pytest.mark.parametrize("n", [8192, 16384])
@pytest.mark.parametrize("tol", [1e-10, 1e-12])
def test_large_level_solve_vs_oracle(n, tol):
    col, kap, shift, b = _level(n, n)
    xo, out = _oracle_solve(col, kap, shift, b, tol)
    op = P.build_toeplitz(col)
    lev = P.LevelOperator(op, shift, kap)
    pc = P.build_preconditioner(col, shift, float(kap.mean()))
    x, rep = P.solve_bicgstab(lev, pc, b, tol=tol)
    assert rep.converged and out.converged
    # reference engine-swap floor at these tolerances (test_gpu_parity.py)
    assert abs(rep.iterations - out.iterations) <= (2 if tol == 1e-10 else 3), \
        (rep.iterations, out.iterations)
    assert rep.final_relative_residual < tol
    assert rel_l2(x, xo) <= (1e-8 if tol == 1e-10 else 1e-10)


@pytest.mark.parametrize("tol", [1e-10, 1e-12])
def test_large_level_solve_at_rounding_floor(tol):
    """n = 2^18: the TRUE residual of the reference's own solve stagnates at
    ~8e-10 (cond x eps) whatever tol asks, so the recursive-residual
    iteration count is rounding noise: numpy vs scipy.fft give 27 vs 25
    (tol 1e-10) and 30 vs 31 (1e-12) iterations and solutions 5.8e-10 apart
    (measured with oracle/; the GPU box's own oracle run gives 23 / 24 with a
    different BLAS thread count).  Gate: true residual and solution at that
    floor, iterations within 30% at tol 1e-10 (at 1e-12, below the attainable
    true residual, the count is noise: 24 vs 32 seen)."""
    n = 1 << 18
    col, kap, shift, b = _level(n, n)
    xo, out = _oracle_solve(col, kap, shift, b, tol)
    lev = P.LevelOperator(P.build_toeplitz(col), shift, kap)
    pc = P.build_preconditioner(col, shift, float(kap.mean()))
    x, rep = P.solve_bicgstab(lev, pc, b, tol=tol)
    assert rep.converged and rep.final_relative_residual < tol
    L, sym = O.toeplitz_symbol(col)
    true_res = np.linalg.norm(b - (shift * x + kap * O.toeplitz_apply(sym, x))) / np.linalg.norm(b)
    assert true_res <= 1e-8, true_res
    assert rel_l2(x, xo) <= 1e-8
    if tol == 1e-10:   # at 1e-12 (below the true-residual floor) the count is noise
        assert abs(rep.iterations - out.iterations) <= max(3, 0.3 * out.iterations)


def test_large_unpreconditioned_solve():
    n = 8192
    col, kap, shift, b = _level(n, 5, shift=2e4)
    xo, out = _oracle_solve(col, kap, shift, b, 1e-10, pc=False)
    lev = P.LevelOperator(P.build_toeplitz(col), shift, kap)
    x, rep = P.solve_bicgstab(lev, None, b, tol=1e-10)
    assert rep.converged and out.converged
    assert abs(rep.iterations - out.iterations) <= max(2, out.iterations // 10)
    assert rel_l2(x, xo) <= 1e-8


def test_large_zero_rhs_and_max_iters():
    n = 8192
    col, kap, shift, b = _level(n, 9)
    lev = P.LevelOperator(P.build_toeplitz(col), shift, kap)
    pc = P.build_preconditioner(col, shift, float(kap.mean()))
    x, rep = P.solve_bicgstab(lev, pc, np.zeros(n))
    assert rep.converged and rep.iterations == 0
    np.testing.assert_array_equal(x, 0.0)
    x, rep = P.solve_bicgstab(lev, pc, b, tol=1e-16, max_iters=2)
    assert not rep.converged and rep.iterations == 2


def test_large_batched_solve_equals_single():
    n = 8192
    col = _col(n)
    shift = 36.0
    op = P.build_toeplitz(col)
    rows = []
    for s in range(3):
        _, kap, _, b = _level(n, 20 + s)
        rows.append((kap, b))
    K = np.stack([k for k, _ in rows])
    Bm = np.stack([b for _, b in rows])
    pc = P.build_preconditioner(col, shift, 1.2)
    lev = P.LevelOperator(op, shift, K)
    X, reps = P.solve_bicgstab(lev, pc, Bm, tol=1e-12)
    for s, (kap, b) in enumerate(rows):
        lev1 = P.LevelOperator(op, shift, kap)
        x1, rep1 = P.solve_bicgstab(lev1, pc, b, tol=1e-12)
        np.testing.assert_array_equal(X[s], x1)
        assert reps[s].iterations == rep1.iterations


_CFG1 = [(g, a) for g in (0.3, 0.5, 0.8) for a in (0.5, 1.0, 1.5, 1.9)]


@pytest.mark.parametrize("gam,alpha", _CFG1)
def test_cfg1_march_vs_reference(gam, alpha):
    """BASELINE configs[1] (n = 16384, M = 1024, tol 1e-12) vs the reference.

    Gate = the reference's own floor on this config: the stock run against
    the same code with only its FFT engine swapped (numpy -> scipy.fft),
    tests/golden/cfg1_floor.json from oracle/engine_swap_floor.py.  At
    alpha >= 1.5 that floor is well below the north star's +-1 / 1e-10 (e.g.
    73% within +-1 and 2.6e-9 rel-l2 at gamma=0.5, alpha=1.9): tol 1e-12 sits
    at the rounding floor of these systems, so any second FFT moves it.
    """
    import json
    from pathlib import Path
    g = golden("cfg1")
    floor = json.loads((Path(__file__).parent / "golden" / "cfg1_floor.json").read_text())
    tag = f"cfg1_g{int(gam * 10)}_a{int(alpha * 10)}"
    fl = floor[tag]
    k, f, phi = cfg0_fields()
    spec = P.ProblemSpec(gamma=gam, alpha=alpha, l=1.0, T=1.0, kappa=k, source=f, initial=phi)
    hist, rep = P.run_fids(spec, 1024, (2.0 - gam) / gam, 16385, epsilon=1e-12,
                           options=P.SolverOptions(solver="pkrylov", tol=1e-12))
    d = rep.iterations - g[f"{tag}_its"]
    frac = float(np.mean(np.abs(d) <= 1))
    e64 = rel_l2(hist[64], g[f"{tag}_u64"])
    eM = rel_l2(hist[-1], g[f"{tag}_uM"])
    print(f"{tag}: within+-1 {frac:.3f} (floor {fl['within1']:.3f}) mean d {d.mean():+.3f} "
          f"e64 {e64:.2e} eM {eM:.2e} (floor {fl['rel_l2_uM']:.2e})")
    assert frac >= min(0.95, fl["within1"] - 0.05)
    # no systematic bias: mean delta within 3 standard errors (or 0.1)
    assert abs(d.mean()) <= max(0.1, 3.0 * d.std() / math.sqrt(d.size)), (d.mean(), d.std())
    assert e64 <= max(1e-10, 10 * fl["rel_l2_u64"])
    assert eM <= max(1e-10, 10 * fl["rel_l2_uM"])


@pytest.mark.parametrize("n", [5000, 12289, 70001])
def test_large_nonpow2_matvec_and_precond(n):
    """n not a power of two: vectors zero-padded to the transform length
    L/2 of the reference's own embedding (toeplitz.py:39-41)."""
    rng = np.random.default_rng(n)
    col = _col(n)
    v = rng.standard_normal(n)
    L, sym = O.toeplitz_symbol(col)
    op = P.build_toeplitz(col)
    kap = _kappa(n, 3)
    got = P.toeplitz_matvec(op, v, kappa=kap, shift=11.0)
    assert rel_err(got, 11.0 * v + kap * O.toeplitz_apply(sym, v)) <= 1e-13
    p = P.build_preconditioner(col, 41.0, 1.3)
    total = 41.0 + 1.3 * O.strang_eigs(col)
    assert rel_err(P.precond_solve(p, v), O.precond_apply(total, v)) <= 1e-13


def test_large_nonpow2_level_solves():
    n = 10000
    col, kap, shift, b = _level(n, 77)
    lev = P.LevelOperator(P.build_toeplitz(col), shift, kap)
    for pc_on in (True, False):
        tol = 1e-10
        xo, out = _oracle_solve(col, kap, shift, b, tol, pc=pc_on)
        pc = P.build_preconditioner(col, shift, float(kap.mean())) if pc_on else None
        x, rep = P.solve_bicgstab(lev, pc, b, tol=tol)
        assert rep.converged and out.converged
        assert abs(rep.iterations - out.iterations) <= max(2, out.iterations // 5), \
            (pc_on, rep.iterations, out.iterations)
        assert rel_l2(x, xo) <= 1e-8


@pytest.mark.parametrize("n,pc_on", [(16384, True), (16384, False), (65536, True)])
def test_large_cg_vs_oracle(n, pc_on):
    """Fused PCG of the four-step engine (krylov.py:43-85) against the oracle."""
    col, kap, shift, b = _level(n, 5 + n)
    kc = float(kap.mean())
    L, sym = O.toeplitz_symbol(col)
    total = shift + kc * O.strang_eigs(col)
    apply = lambda q: shift * q + kc * O.toeplitz_apply(sym, q)  # noqa: E731
    ps = (lambda q: O.precond_apply(total, q)) if pc_on else None
    xo, out = O.cg(apply, ps, b, tol=1e-10, max_iters=5000)
    lev = P.LevelOperator(P.build_toeplitz(col), shift, np.full(n, kc))
    pc = P.build_preconditioner(col, shift, kc) if pc_on else None
    x, rep = P.solve_cg(lev, pc, b, tol=1e-10, max_iters=5000)
    assert rep.converged == out.converged
    assert abs(rep.iterations - out.iterations) <= max(2, out.iterations // 10), \
        (rep.iterations, out.iterations)
    assert rel_l2(x, xo) <= 1e-8
