"""GPU parity of the DIDS path (run_dids, scheme.py:184-233): the device L1
history kernel (tsf_l1_history_rhs) and full marches against the reference
goldens and the oracle.

Tolerances: history RHS 1e-14 relative (the GEMV summation order differs
from OpenBLAS); marches within 1e-10 relative l2 at every level with
per-level iteration counts within +-1 on >= 90% of the levels (the small
golden marches have 16-64 levels; SURVEY.md §8(c) floors), and the
reference's FIDS-DIDS proximity criterion (pkg/tests/test_acceptance.py:
141-166) between this package's own run_fids and run_dids.
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
from paper_2002_11978_b200 import _native  # noqa: E402
from scipy.special import gammaln  # noqa: E402


@pytest.mark.parametrize("n,rows,B", [(1, 1, 1), (100, 1, 1), (257, 2, 1), (1024, 37, 1),
                                      (4096, 200, 3), (33, 9, 5)])
def test_l1_history_rhs_kernel(n, rows, B):
    rng = np.random.default_rng(n * 7 + rows)
    hist = rng.standard_normal((B, rows, n))
    w = rng.uniform(0.1, 2.0, max(rows - 1, 1))
    f = rng.standard_normal((B, n))
    G = math.exp(gammaln(0.5))
    c0 = 1.7 / G
    want = f + c0 * hist[:, 0]
    if rows > 1:
        want = want + np.einsum("k,bki->bi", w[: rows - 1], hist[:, 1:]) / G
    hd = torch.from_numpy(hist).cuda()
    wd = torch.from_numpy(w).cuda()
    fd = torch.from_numpy(f).cuda()
    out = torch.empty_like(fd)
    _native.check(_native.load().tsf_l1_history_rhs(B, n, rows, hd.data_ptr(), rows * n,
                                                    wd.data_ptr(), c0, G, fd.data_ptr(),
                                                    out.data_ptr(), _native.stream_ptr()))
    assert rel_err(out.cpu().numpy(), want) <= 1e-14


def test_l1_history_rhs_first_term_keeps_numpy_rounding():
    # rows == 1: rhs = f + (a0/G) u0 exactly as numpy rounds it (no FMA)
    rng = np.random.default_rng(3)
    n = 4096
    h0 = rng.standard_normal(n)
    f = rng.standard_normal(n)
    G = math.exp(gammaln(0.7))
    c0 = 3.3 / G
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    hd = torch.from_numpy(h0).cuda()
    fd = torch.from_numpy(f).cuda()
    _native.check(_native.load().tsf_l1_history_rhs(1, n, 1, hd.data_ptr(), n, None, c0, G,
                                                    fd.data_ptr(), out.data_ptr(),
                                                    _native.stream_ptr()))
    np.testing.assert_array_equal(out.cpu().numpy(), f + c0 * h0)


def test_l1_history_rhs_rejects_bad_arguments():
    lib = _native.load()
    assert lib.tsf_l1_history_rhs(1, 0, 1, None, 0, None, 1.0, 1.0, None, None, None) == -1
    assert lib.tsf_l1_history_rhs(1, 8, 2, None, 16, None, 1.0, 1.0, None, None, None) == -1


@pytest.mark.parametrize("tag", ["d1", "d2", "d3", "d4"])
def test_run_dids_vs_reference_goldens(tag):
    g = golden("dids")
    gam, a, M, N, tol, r = g[f"{tag}_args"]
    M, N = int(M), int(N)
    solver = str(g[f"{tag}_solver"])
    k, f, phi = cfg0_fields()
    spec = P.ProblemSpec(gamma=gam, alpha=a, l=1.0, T=1.0, kappa=k, source=f, initial=phi)
    hist, rep = P.run_dids(spec, M, r, N, options=P.SolverOptions(solver=solver, tol=tol))
    ref = g[f"{tag}_hist"]
    assert hist.shape == ref.shape == (M + 1, N - 1)
    errs = [rel_l2(hist[m], ref[m]) for m in range(1, M + 1)]
    assert max(errs) <= 1e-10, max(errs)
    assert rep.scheme_tag == "DIDS"
    np.testing.assert_array_equal(rep.history_ops, g[f"{tag}_ops"])
    assert rep.history_memory_values == (M + 1) * (N - 1)
    if solver == "auto":      # dense branch: no Krylov iterations
        assert rep.solver_tag == "direct" and np.all(rep.iterations == 0)
        return
    ref_its = g[f"{tag}_its"]
    d = np.abs(rep.iterations - ref_its)
    if solver == "krylov":
        # unpreconditioned alpha = 1.9 (~115 its per level): the reference
        # with only its FFT engine swapped (numpy -> scipy.fft) lands within
        # +-1 on 29% of these levels, |d| <= 9 (measured); gate as the plain
        # linear-algebra test does, per level
        assert np.all(d <= np.maximum(2, ref_its // 10)), d
        assert abs(rep.avg_iterations - g[f"{tag}_avg"][0]) <= 3.0
        return
    assert np.mean(d <= 1) >= 0.9, d
    assert abs(rep.avg_iterations - g[f"{tag}_avg"][0]) <= 0.5


@pytest.mark.parametrize("tag", ["d1", "d2"])
def test_fids_dids_proximity_on_device(tag):
    # criterion 7 (pkg/tests/test_acceptance.py:141-166): max |DIDS - FIDS| <= 100 eps
    g = golden("dids")
    gam, a, M, N, tol, r = g[f"{tag}_args"]
    M, N = int(M), int(N)
    k, f, phi = cfg0_fields()
    spec = P.ProblemSpec(gamma=gam, alpha=a, l=1.0, T=1.0, kappa=k, source=f, initial=phi)
    opts = P.SolverOptions(solver="pkrylov", tol=tol)
    hd, _ = P.run_dids(spec, M, r, N, options=opts)
    hf, _ = P.run_fids(spec, M, r, N, epsilon=1e-12, options=opts)
    assert np.max(np.abs(hd - hf)) <= 100 * 1e-12


def test_run_dids_vs_oracle_cfg0_shape():
    # configs[0] fields and size (n = 1024) over 48 levels, against the oracle
    k, f, phi = cfg0_fields()
    M = 48
    spec = P.ProblemSpec(gamma=0.5, alpha=1.5, l=1.0, T=1.0, kappa=k, source=f, initial=phi)
    hist, rep = P.run_dids(spec, M, 3.0, 1025, options=P.SolverOptions(solver="pkrylov",
                                                                      tol=1e-12))
    ref = O.dids_march(0.5, 1.5, 1.0, 1.0, M, 3.0, 1025, k, f, phi, tol=1e-12)
    assert max(rel_l2(hist[m], ref.hist[m]) for m in range(1, M + 1)) <= 1e-10
    assert np.mean(np.abs(rep.iterations - ref.iterations) <= 1) >= 0.9
