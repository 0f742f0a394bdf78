"""The reference's acceptance gate re-run through the device solvers.

Every scheme criterion of pkg/tests/test_acceptance.py:38-166 (criteria 1-7:
temporal and spatial convergence of FIDS and DIDS on the manufactured
problems, the low-alpha branch, the preconditioner benefit and the FIDS-DIDS
proximity) is executed with this package's run_fids / run_dids on the B200,
on the reference's exact grids (couplings.n_from_m / m_from_n), and checked
twice:

* against the reference test's own pinned numbers and tolerances (errors
  within 2%, rates within 0.05, iteration windows), and
* against the reference itself run on the same configuration
  (tests/golden/acceptance.npz, `python oracle/gen_golden.py --only
  acceptance`): err_inf within 1e-6 relative, final level within 1e-9
  relative l2 (direct solves: 1e-12), average iterations within the
  engine-swap floor (±1 per level on average for preconditioned solves, 10%
  for the unpreconditioned one).
"""

import math

import numpy as np
import pytest

from tsf_testlib import golden, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2002_11978_b200 import SolverOptions, run_dids, run_fids  # noqa: E402
from harness.couplings import m_from_n, n_from_m  # noqa: E402
from harness.problems import make_case  # noqa: E402


def _ref(label):
    g = golden("acceptance")
    row = g[f"acc_{label}"]
    return {"M": int(row[0]), "N": int(row[1]), "err_dids": row[2], "err_fids": row[3],
            "avg_its": row[4], "dids_uM": g.get(f"acc_{label}_dids_uM"),
            "fids_uM": g.get(f"acc_{label}_fids_uM")}


def _check_against_reference(label, scheme, hist, rep, direct):
    ref = _ref(label)
    err = rep.err_inf
    want = ref[f"err_{scheme}"]
    assert err == pytest.approx(want, rel=1e-6), f"{label} {scheme}: {err} vs ref {want}"
    uM = np.asarray(hist[-1])
    tol = 1e-12 if direct else 1e-9
    assert rel_l2(uM, ref[f"{scheme}_uM"]) <= tol, label
    return err


def _fids(label, case, M, r, N, eps, mu=None, solver="auto", tol=1e-10):
    h, rep = run_fids(case.spec, M, r, N, epsilon=eps, mu=mu,
                      options=SolverOptions(solver=solver, tol=tol))
    direct = solver == "direct" or (solver == "auto" and N - 1 <= 128)
    _check_against_reference(label, "fids", h, rep, direct)
    return h, rep


def _dids(label, case, M, r, N, mu=None):
    h, rep = run_dids(case.spec, M, r, N, mu=mu)
    _check_against_reference(label, "dids", h, rep, N - 1 <= 128)
    return h, rep


def test_criterion_01_temporal_convergence_smooth():
    """test_acceptance.py:38-55 — alpha 1.5, (r, gamma) = (2, 0.5), both schemes."""
    expected = {2 ** 7: 4.363e-3, 2 ** 8: 1.964e-3, 2 ** 9: 9.497e-4, 2 ** 10: 4.542e-4}
    case = make_case("example1", 1.5, 0.5)
    for M, want in expected.items():
        N = n_from_m(M, 2, 0.5, 2)
        _, rd = _dids(f"c1_M{M}", case, M, 2, N)
        _, rf = _fids(f"c1_M{M}", case, M, 2, N, 1e-10)
        assert rd.err_inf == pytest.approx(want, rel=0.02)
        assert rf.err_inf == pytest.approx(want, rel=0.02)


def test_criterion_02_temporal_convergence_mu2():
    """test_acceptance.py:58-69 — alpha 1.6, mu = 2, (r, gamma) = (3, 0.8)."""
    case = make_case("example1", 1.6, 0.8)
    errs = {}
    for M in (2 ** 9, 2 ** 10):
        N = n_from_m(M, 3, 0.8, 2)
        _, rep = _dids(f"c2_M{M}", case, M, 3, N, mu=2.0)
        errs[M] = rep.err_inf
    assert errs[2 ** 10] == pytest.approx(9.389e-5, rel=0.02)
    assert math.log2(errs[2 ** 9] / errs[2 ** 10]) == pytest.approx(1.285, abs=0.05)


def test_criterion_03_spatial_convergence_smooth():
    """test_acceptance.py:72-86 — alpha 1.5, (r, gamma) = (1, 0.8), N = 8..64."""
    case = make_case("example1", 1.5, 0.8)
    errs = []
    for N in (8, 16, 32, 64):
        M = m_from_n(N, 1, 0.8, 2)
        _, rep = _dids(f"c3_N{N}", case, M, 1, N)
        errs.append(rep.err_inf)
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    for got, want in zip(rates, (2.166, 2.136, 2.112)):
        assert got == pytest.approx(want, abs=0.05)


def test_criterion_04_spatial_reduced_regularity():
    """test_acceptance.py:89-102 — example2, alpha 1.9, (r, gamma) = (3, 0.8)."""
    case = make_case("example2", 1.9, 0.8)
    errs = []
    for N in (9, 18, 36, 72):
        M = m_from_n(N, 3, 0.8, 1.95)
        _, rep = _dids(f"c4_N{N}", case, M, 3, N)
        errs.append(rep.err_inf)
    assert errs[-1] == pytest.approx(1.135e-3, rel=0.02)
    for i in range(3):
        assert math.log2(errs[i] / errs[i + 1]) == pytest.approx(2.03, abs=0.05)


def test_criterion_05_low_alpha_branch():
    """test_acceptance.py:105-116 — example2, alpha 0.5, FIDS at eps 1e-9 (device
    BiCGSTAB: n = 255 and 511 are non-power-of-two, Strang preconditioner
    applied through the Toeplitz engine)."""
    case = make_case("example2", 0.5, 0.5)
    errs = {}
    for N in (2 ** 8, 2 ** 9):
        M = m_from_n(N, 2, 0.5, 1.25)
        _, rep = _fids(f"c5_N{N}", case, M, 2, N, 1e-9)
        errs[N] = rep.err_inf
        assert abs(rep.avg_iterations - _ref(f"c5_N{N}")["avg_its"]) <= 1.0
    assert errs[2 ** 9] == pytest.approx(2.115e-4, rel=0.02)
    assert math.log2(errs[2 ** 8] / errs[2 ** 9]) == pytest.approx(1.232, abs=0.05)


def test_criterion_06_preconditioner_benefit():
    """test_acceptance.py:119-138 — (r, gamma, alpha) = (2, 0.5, 1.9), mu = 1.95,
    tol 1e-10: unpreconditioned ~198 iterations per level, preconditioned ~8
    independent of N."""
    g = golden("acceptance")
    if "acc_c6_plain_N256" not in g:
        pytest.skip("criterion-6 reference runs not in the fixture")
    case = make_case("example2", 1.9, 0.5)

    def avg_its(label, N, solver):
        M = m_from_n(N, 2, 0.5, 1.95)
        _, rep = _fids(label, case, M, 2, N, 1e-9, solver=solver, tol=1e-10)
        return rep.avg_iterations

    plain = avg_its("c6_plain_N256", 2 ** 8, "krylov")
    assert 160.0 <= plain <= 240.0
    assert plain == pytest.approx(_ref("c6_plain_N256")["avg_its"], rel=0.10)
    prec = {}
    for N in (2 ** 6, 2 ** 7, 2 ** 8):
        prec[N] = avg_its(f"c6_prec_N{N}", N, "pkrylov")
        assert 6.0 <= prec[N] <= 12.0
        assert abs(prec[N] - _ref(f"c6_prec_N{N}")["avg_its"]) <= 1.0
    assert max(prec.values()) - min(prec.values()) <= 2.0


def test_criterion_07_fids_dids_proximity():
    """test_acceptance.py:141-166 — every criterion 1-5 configuration with
    M <= 2^8: max |DIDS - FIDS| <= 100 eps at eps = 1e-10, both on the device."""
    eps = 1e-10
    configs = []
    for M in (2 ** 7, 2 ** 8):
        configs.append(("example1", 1.5, 0.5, 2, None, M, n_from_m(M, 2, 0.5, 2)))
    configs.append(("example1", 1.6, 0.8, 3, 2.0, 2 ** 8, n_from_m(2 ** 8, 3, 0.8, 2)))
    for N in (8, 16):
        configs.append(("example1", 1.5, 0.8, 1, None, m_from_n(N, 1, 0.8, 2), N))
    for N in (9, 18, 36):
        configs.append(("example2", 1.9, 0.8, 3, None, m_from_n(N, 3, 0.8, 1.95), N))
    configs.append(("example2", 0.5, 0.5, 2, None, m_from_n(2 ** 6, 2, 0.5, 1.25), 2 ** 6))
    for name, alpha, gamma, r, mu, M, N in configs:
        assert M <= 2 ** 8
        case = make_case(name, alpha, gamma)
        h_d, _ = run_dids(case.spec, M, r, N, mu=mu)
        h_f, _ = run_fids(case.spec, M, r, N, epsilon=eps, mu=mu)
        diff = float(np.max(np.abs(np.asarray(h_d) - np.asarray(h_f))))
        assert diff <= 100.0 * eps, f"{name} M={M} N={N}: {diff:.2e}"


def test_foreign_problem_spec_is_accepted():
    """A spec object of another package (the reference's own ProblemSpec) works:
    the drivers read its fields by name (CLI backend switch)."""
    from types import SimpleNamespace

    case = make_case("example1", 1.5, 0.5)
    sp = case.spec
    foreign = SimpleNamespace(gamma=sp.gamma, alpha=sp.alpha, l=sp.l, T=sp.T, kappa=sp.kappa,
                              source=sp.source, initial=sp.initial, exact=sp.exact,
                              kappa_x_independent=False)
    M = 2 ** 7
    N = n_from_m(M, 2, 0.5, 2)
    h0, r0 = run_fids(sp, M, 2, N, epsilon=1e-10)
    h1, r1 = run_fids(foreign, M, 2, N, epsilon=1e-10)
    np.testing.assert_array_equal(np.asarray(h0), np.asarray(h1))
    assert r0.err_inf == r1.err_inf
    _, d0 = run_dids(sp, M, 2, N)
    _, d1 = run_dids(foreign, M, 2, N)
    assert d0.err_inf == d1.err_inf
