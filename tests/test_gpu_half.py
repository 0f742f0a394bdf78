"""GPU parity of the half-length transform engine (csrc/tsf_half.cuh): its two
building blocks alone against the oracle (toeplitz.py:131-136 and
toeplitz.py:51-63 + scheme.py:129-130), and the level solve it drives against
the full-length engine (TSF_HALF=0 in a subprocess) and the oracle.

Tolerances: 1e-13 relative (max-abs / max) for one Strang solve; the Toeplitz
product of a Strang output inherits that solve's rounding through the stored
spectrum, amplified by the symbol, so it is compared at
2e-12 against the oracle applied to the device's own output; the level solve
within +-2 iterations and 1e-10 relative l2 of the oracle.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from tsf_testlib import rel_err, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2002_11978_b200 as P  # noqa: E402
from paper_2002_11978_b200 import _native  # noqa: E402
from paper_2002_11978_b200 import workloads as WL  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def _setup(n, alpha=1.5):
    col, _, _ = O.ifl_column(alpha, 1 + alpha / 2, 1.0, n + 1)
    _, sym = O.toeplitz_symbol(col)
    lam = O.strang_eigs(col)
    return col, sym, lam


@pytest.mark.parametrize("n", [512, 1024, 2048, 4096])
def test_half_blocks_vs_oracle(n):
    col, sym, lam = _setup(n)
    op = P.build_toeplitz(col)
    P.build_preconditioner(col, 1.0, 1.0)   # the plan's Strang tables
    B = 3
    rng = np.random.default_rng(n)
    x = rng.standard_normal((B, n))
    x[1] = np.cos(np.pi * np.linspace(-1, 1, n)) ** 2          # smooth
    kap = rng.uniform(0.5, 2.0, (B, n))
    shift = 37.5
    total = np.stack([shift + kap[b].mean() * lam for b in range(B)])
    F = 1.0 / total
    F = 0.5 * (F + np.roll(F[:, ::-1], 1, axis=1)) / n
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    xd, Fd, kd = dev(x), dev(F), dev(kap)
    hs = torch.zeros(B, n // 2 + 1, 2, dtype=torch.float64, device="cuda")
    z = torch.empty_like(xd)
    lib = _native.load()
    _native.check(lib.tsf_half_debug(op.plan.handle, 0, B, xd.data_ptr(), Fd.data_ptr(), 0.0,
                                     hs.data_ptr(), z.data_ptr(), _native.stream_ptr()))
    zz = z.cpu().numpy()
    for b in range(B):
        want = O.precond_apply(total[b], x[b])
        assert rel_err(zz[b], want) <= 1e-13, (n, b)
    h = hs.cpu().numpy().view(np.complex128).reshape(B, n // 2 + 1)
    want_h = (np.fft.fft(x, axis=1) * F)[:, :n // 2 + 1]
    assert rel_err(h, want_h) <= 1e-13
    y = torch.empty_like(xd)
    _native.check(lib.tsf_half_debug(op.plan.handle, 1, B, z.data_ptr(), kd.data_ptr(), shift,
                                     hs.data_ptr(), y.data_ptr(), _native.stream_ptr()))
    yy = y.cpu().numpy()
    for b in range(B):
        want = shift * zz[b] + kap[b] * O.toeplitz_apply(sym, zz[b])
        assert rel_err(yy[b], want) <= 2e-12, (n, b)


def _solve_script(n, B):
    return f"""
import sys, numpy as np
sys.path.insert(0, {str(ROOT)!r}); sys.path.insert(0, {str(ROOT / 'tests')!r})
import oracle as O, paper_2002_11978_b200 as P
from paper_2002_11978_b200 import workloads as WL
n, B = {n}, {B}
col, _, _ = O.ifl_column(1.5, 1.75, 1.0, n + 1)
op = P.build_toeplitz(col)
x, kx, fx, u0 = WL.instance_fields(n, 0, B)
shift = 411.0
its = []
xs = []
for b in range(B):
    lev = P.LevelOperator(op, shift, kx[b])
    pc = P.build_preconditioner(col, shift, float(kx[b].mean()))
    rhs = fx[b] + shift * u0[b]
    xb, rep = P.solve_bicgstab(lev, pc, rhs, tol=1e-12)
    assert rep.converged
    its.append(rep.iterations); xs.append(xb)
np.savez(sys.argv[1], its=np.array(its), x=np.stack(xs))
"""


@pytest.mark.parametrize("n", [1024, 4096])
def test_half_level_solve_vs_full_engine_and_oracle(n, tmp_path):
    B = 4
    out = {}
    for tag, half in (("half", "1"), ("full", "0")):
        f = tmp_path / f"{tag}.npz"
        env = dict(os.environ, TSF_HALF=half)
        subprocess.run([sys.executable, "-c", _solve_script(n, B), str(f)], check=True, env=env)
        out[tag] = np.load(f)
    col, sym, lam = _setup(n)
    x, kx, fx, u0 = WL.instance_fields(n, 0, B)
    shift = 411.0
    for b in range(B):
        rhs = fx[b] + shift * u0[b]
        total = shift + float(kx[b].mean()) * lam
        xr, rep = O.bicgstab(lambda q: shift * q + kx[b] * O.toeplitz_apply(sym, q),
                             lambda q: O.precond_apply(total, q), rhs, tol=1e-12)
        for tag in ("half", "full"):
            assert abs(int(out[tag]["its"][b]) - rep.iterations) <= 2, (tag, b)
            assert rel_l2(out[tag]["x"][b], xr) <= 1e-10, (tag, b)
        assert rel_l2(out["half"]["x"][b], out["full"]["x"][b]) <= 1e-10


def test_half_control_flow_edges():
    """The reference's control flow on the half-length kernels (n = 1024):
    max_iters exhaustion (krylov.py:100), zero right-hand side (krylov.py:
    109-111), non-positive kappa (scheme.py:156-160)."""
    n = 1024
    col, sym, lam = _setup(n)
    x, kx, fx, u0 = WL.instance_fields(n, 0, 1)
    lev = P.LevelOperator(P.build_toeplitz(col), 411.0, kx[0])
    pc = P.build_preconditioner(col, 411.0, float(kx[0].mean()))
    rhs = fx[0] + 411.0 * u0[0]
    xs, rep = P.solve_bicgstab(lev, pc, rhs, tol=1e-15, max_iters=1)
    assert not rep.converged and rep.iterations == 1
    xs, rep = P.solve_bicgstab(lev, pc, np.zeros(n))
    assert rep.converged and rep.iterations == 0
    np.testing.assert_array_equal(xs, 0.0)
    spec = P.ProblemSpec(gamma=0.5, alpha=1.5, l=1.0, T=1.0,
                         kappa=lambda x, t: np.where(x > 0, 1.0, -1.0),
                         source=lambda x, t: np.zeros_like(x),
                         initial=lambda x: (1 - x * x) ** 2)
    with pytest.raises(ValueError, match="kappa"):
        P.run_fids(spec, 4, 1.0, n + 1, options=P.SolverOptions(solver="pkrylov"))


def test_half_large_control_flow_edges():
    """Same on the half-length four-step kernels (n = 2^15)."""
    n = 1 << 15
    col, sym, lam = _setup(n)
    xg = WL.grid(n)
    kap = 1.0 + 0.5 * np.sin(np.pi * xg)
    lev = P.LevelOperator(P.build_toeplitz(col), 411.0, kap)
    pc = P.build_preconditioner(col, 411.0, float(kap.mean()))
    rhs = np.sin(np.pi * xg) + 411.0 * (1 - xg * xg) ** 2
    xs, rep = P.solve_bicgstab(lev, pc, rhs, tol=1e-15, max_iters=2)
    assert not rep.converged and rep.iterations == 2
    xs, rep = P.solve_bicgstab(lev, pc, np.zeros(n))
    assert rep.converged and rep.iterations == 0
    total = 411.0 + float(kap.mean()) * lam
    xr, ref = O.bicgstab(lambda q: 411.0 * q + kap * O.toeplitz_apply(sym, q),
                         lambda q: O.precond_apply(total, q), rhs, tol=1e-12)
    xs, rep = P.solve_bicgstab(lev, pc, rhs, tol=1e-12)
    assert rep.converged and abs(rep.iterations - ref.iterations) <= 2
    assert rel_l2(xs, xr) <= 1e-10


@pytest.mark.parametrize("n,B", [(1024, 4), (4096, 3), (512, 300)])
def test_half_persistent_kernel_bit_identical(n, B):
    """The half-length engine runs the whole solve in one persistent kernel
    per instance (k_krylov_persist_h: the same phase bodies in a loop, its hot
    vectors in shared memory); its results must equal the phase kernels' bit
    for bit (TSF_PERSIST_MAX_B=0 in a subprocess).  (512, 300): more CTAs than
    SMs, so finished instances' SMs are back-filled."""
    import tempfile
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for tag, mb in (("persist", "1000000"), ("phases", "0")):
            f = Path(td) / f"{tag}.npz"
            env = dict(os.environ, TSF_PERSIST_MAX_B=mb)
            subprocess.run([sys.executable, "-c", _solve_script(n, B), str(f)], check=True, env=env)
            out[tag] = {k: v.copy() for k, v in np.load(f).items()}
    np.testing.assert_array_equal(out["persist"]["its"], out["phases"]["its"])
    np.testing.assert_array_equal(out["persist"]["x"], out["phases"]["x"])
