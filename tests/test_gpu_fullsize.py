"""Parity at BASELINE.json's full sizes.

configs[2] (n = 4096, M = 512) for a 256-instance batch of the seeded
workload: two instances against the reference's own full-size goldens
(tests/golden/cfg2.npz), and size-independent properties of the whole batch:
  * position invariance — the same instances marched as a different batch
    give bit-identical u^M and iteration counts (each CTA is deterministic);
  * exact homogeneity — doubling f and u^0 doubles u^M bit for bit with the
    same iteration counts (every operation is linear; scaling by 2 is exact).
configs[3] (n = 2^20): the first levels against the oracle.

Gates for the goldens come from the reference's engine-swap floor on these
two instances (numpy -> scipy.fft, measured on the CPU): ±1 iteration on 75-77%
of levels, max |Δ| 4-6, u^M within 1.9e-12.
"""

import math

import numpy as np
import pytest

import oracle as O
from tsf_testlib import golden, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2002_11978_b200 as P  # noqa: E402
from paper_2002_11978_b200 import workloads as WL  # noqa: E402
from paper_2002_11978_b200.scheme import FidsMarch, _field_separable  # noqa: E402

N_, M_ = 4096, 512


def _march(b0, B, fscale=1.0):
    gam, alpha = 0.5, 1.5
    r = (2 - gam) / gam
    x, kx, fx, u0 = WL.instance_fields(N_, b0, B)
    kap = P.SeparableField([np.ones(N_)], lambda t: [1.0 + 0.2 * t])
    src = P.SeparableField([np.ones(N_)], lambda t: [1.0 + t])
    mesh = P.build_mesh(M_, r, 1.0)
    soe = P.build_soe(gam, 1e-12, (1.0 / M_) ** r, 1.0)
    dev = torch.device("cuda:0")
    kd = _field_separable(kap, x, mesh.t, B, kx[None], dev)
    fd = _field_separable(src, x, mesh.t, B, (fscale * fx)[None], dev)
    m = FidsMarch(gam, alpha, 1.0, 1.0, M_, r, N_ + 1, soe, method=0, precond=1, tol=1e-12,
                  max_iters=None, B=B, kappa=kd, source=fd,
                  u0=torch.from_numpy(np.ascontiguousarray(fscale * u0)).to(dev), device=0,
                  private_plan=True)
    m.run()
    res = m.result()
    assert np.all(res.status == 0)
    out = res.u_final.cpu().numpy().copy(), res.iterations.copy()
    del m, res
    torch.cuda.empty_cache()
    return out


@pytest.fixture(scope="module")
def batch():
    return _march(0, 256)


def test_cfg2_full_size_vs_reference_goldens(batch):
    uB, itB = batch
    g = golden("cfg2")
    for b in (37, 200):
        ref_its, ref_u = g[f"b{b}_its"], g[f"b{b}_uM"]
        d = itB[:, b] - ref_its
        assert rel_l2(uB[b], ref_u) <= 1e-10
        assert np.mean(np.abs(d) <= 1) >= 0.70, (b, np.unique(d, return_counts=True))
        assert np.max(np.abs(d)) <= 8 and abs(d.mean()) <= 0.3, (b, d.mean())


def test_cfg2_full_size_position_invariance(batch):
    uB, itB = batch
    u2, it2 = _march(37, 16)      # instances 37..52 as their own batch
    np.testing.assert_array_equal(u2, uB[37:53])
    np.testing.assert_array_equal(it2, itB[:, 37:53])


def test_cfg2_full_size_exact_homogeneity(batch):
    uB, itB = batch
    u2, it2 = _march(0, 32, fscale=2.0)
    np.testing.assert_array_equal(it2, itB[:, :32])
    np.testing.assert_array_equal(u2, 2.0 * uB[:32])


def test_cfg3_first_levels_vs_oracle():
    """configs[3] size (n = 2^20, M = 256, gamma = 0.7, alpha = 1.2): levels
    1..3 of run_fids's device march against the oracle's fids_step."""
    n, M, gam, alpha = 1 << 20, 256, 0.7, 1.2
    r = (2 - gam) / gam
    N = n + 1
    kappa = lambda xx, t: 1.0 + 0.5 * np.sin(np.pi * xx) * np.exp(-t)  # noqa: E731
    source = lambda xx, t: (1.0 + t) * np.sin(np.pi * xx)  # noqa: E731
    x = WL.grid(n)
    kap = P.SeparableField([np.ones(n), 0.5 * np.sin(np.pi * x)], lambda t: [1.0, math.exp(-t)])
    src = P.SeparableField([np.sin(np.pi * x)], lambda t: [1.0 + t])
    mesh = P.build_mesh(M, r, 1.0)
    soe = P.build_soe(gam, 1e-12, (1.0 / M) ** r, 1.0)
    dev = torch.device("cuda:0")
    u0 = (1.0 - x * x) ** 2
    m = FidsMarch(gam, alpha, 1.0, 1.0, M, r, N, soe, method=0, precond=1, tol=1e-12,
                  max_iters=None, B=1, kappa=_field_separable(kap, x, mesh.t, 1, None, dev),
                  source=_field_separable(src, x, mesh.t, 1, None, dev),
                  u0=torch.from_numpy(u0[None, :].copy()).to(dev), hist_B=1, device=0)
    levels = 3
    m.run(levels)
    torch.cuda.synchronize()
    hist = m.hist[: levels + 1, 0].cpu().numpy()
    its = m.iters[:levels, 0].cpu().numpy()
    # oracle, same levels
    t, tau = O.graded_mesh(M, r, 1.0)
    col, h, _ = O.ifl_column(alpha, 1.0 + alpha / 2.0, 1.0, N)
    _, symbol = O.toeplitz_symbol(col)
    lam = O.strang_eigs(col)
    G = math.exp(math.lgamma(1.0 - gam))
    s, w = soe.nodes, soe.weights
    W = np.zeros((s.size, n))
    u = u0.copy()
    for k in range(1, levels + 1):
        u, _, out = O.fids_step(u, W, s, w, tau[k - 1], gam, G, kappa(x, t[k]), source(x, t[k]),
                                symbol, lam, 1e-12)
        assert rel_l2(hist[k], u) <= 1e-10, k
        assert abs(int(its[k - 1]) - out.iterations) <= 2, (k, its[k - 1], out.iterations)
