"""CPU check of the half-length transform algebra (csrc/tsf_half.cuh,
tsf_hlarge.cuh) through its numpy emulation (tools/half_probe.py Engine):
the Strang solve and the Toeplitz product of toeplitz.py:51-63 / 131-136
computed with ONE complex transform of length n/2 each must equal the
oracle's full-length results to rounding, for both sub-transform backends."""
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle as O

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
from half_probe import Engine  # noqa: E402


@pytest.mark.parametrize("n", [64, 1024, 8192])
@pytest.mark.parametrize("kind", ["eng", "half"])
@pytest.mark.parametrize("backend", ["numpy", "ld"])
def test_half_structure_matches_oracle(n, kind, backend):
    col, _, _ = O.ifl_column(1.5, 1.75, 1.0, n + 1)
    _, sym = O.toeplitz_symbol(col)
    lam = O.strang_eigs(col)
    rng = np.random.default_rng(n)
    p = rng.standard_normal(n)
    total = 3.0 + 1.2 * lam
    e = Engine(kind, backend, sym, n)
    q = e.pc(p, total)
    qr = O.precond_apply(total, p)
    assert np.linalg.norm(q - qr) <= 1e-14 * np.linalg.norm(qr) * np.log2(n)
    # product of the Strang output: even bins from the stored spectrum
    y = e.mv(q)
    yr = O.toeplitz_apply(sym, q)
    assert np.linalg.norm(y - yr) <= 1e-12 * np.linalg.norm(yr)
    # product of an arbitrary vector: no stored spectrum
    x = rng.standard_normal(n)
    y2 = e.mv(x)
    y2r = O.toeplitz_apply(sym, x)
    assert np.linalg.norm(y2 - y2r) <= 1e-14 * np.linalg.norm(y2r) * np.log2(n)


def test_half_structure_level_solve_iterations():
    """The reference's BiCGSTAB control flow over the half-length structure
    converges like the reference's own arithmetic (tools/half_probe.py)."""
    n = 1024
    col, _, _ = O.ifl_column(1.5, 1.75, 1.0, n + 1)
    _, sym = O.toeplitz_symbol(col)
    lam = O.strang_eigs(col)
    x = -1.0 + (2.0 / (n + 1)) * np.arange(1, n + 1)
    kap = 1.0 + 0.5 * np.sin(np.pi * x)
    rhs = np.sin(np.pi * x) + 411.0 * (1 - x * x) ** 2
    shift = 411.0
    total = shift + float(kap.mean()) * lam
    xr, ref = O.bicgstab(lambda q: shift * q + kap * O.toeplitz_apply(sym, q),
                         lambda q: O.precond_apply(total, q), rhs, tol=1e-12)
    e = Engine("half", "numpy", sym, n)
    xh, out = O.bicgstab(lambda q: shift * q + kap * e.mv(q), lambda q: e.pc(q, total), rhs,
                         tol=1e-12)
    assert out.converged and abs(out.iterations - ref.iterations) <= 2
    assert np.linalg.norm(xh - xr) <= 1e-10 * np.linalg.norm(xr)
