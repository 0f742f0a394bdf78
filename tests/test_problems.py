"""Host-side manufactured problems and couplings (problems.py, couplings.py)
against values produced by the reference itself (tests/golden/acceptance.npz,
`python oracle/gen_golden.py --only acceptance`).

The source, exact solution, initial bump and diffusivity keep the reference's
evaluation order, so they are compared bit for bit; the couplings must
regenerate the acceptance grids (M, N) exactly.
"""

import numpy as np
import pytest

from tsf_testlib import golden

from harness import couplings, problems


def _fn_cases():
    g = golden("acceptance")
    return sorted({k.split("_")[0] for k in g if k.startswith("fn")})


def test_problem_functions_bit_identical():
    g = golden("acceptance")
    cases = _fn_cases()
    assert len(cases) >= 6
    for c in cases:
        a, gam, s = g[f"{c}_args"]
        name = str(g[f"{c}_name"])
        case = problems.make_case(name, float(a), float(gam))
        assert case.s == int(s)
        x = g[f"{c}_x"]
        np.testing.assert_array_equal(case.spec.initial(x), g[f"{c}_initial"])
        for j, t in enumerate((0.0, 0.37, 1.0)):
            np.testing.assert_array_equal(case.spec.source(x, t), g[f"{c}_source_t{j}"])
            np.testing.assert_array_equal(case.spec.exact(x, t), g[f"{c}_exact_t{j}"])
            np.testing.assert_array_equal(case.spec.kappa(x, t), g[f"{c}_kappa_t{j}"])


def test_acceptance_grids_from_couplings():
    """n_from_m / m_from_n regenerate every (M, N) of the acceptance runs."""
    from oracle.gen_golden import ACCEPTANCE_RUNS

    g = golden("acceptance")
    for (label, _, _, _, gam, r, _, M, N, q, *_rest) in ACCEPTANCE_RUNS:
        want_M, want_N = g[f"acc_{label}"][:2]
        if N is None:
            N = couplings.n_from_m(M, r, gam, q)
        else:
            M = couplings.m_from_n(N, r, gam, q)
        assert (M, N) == (int(want_M), int(want_N)), label


def test_problem_errors_match_reference():
    with pytest.raises(KeyError):
        problems.make_case("example3", 1.5, 0.5)
    with pytest.raises(ValueError):
        problems.hypergeom_terminating(0.5, 0, 0.1)
    with pytest.raises(ValueError):
        problems.exact_ifl_of_bump(3, 1.5, 1.5)
    with pytest.raises(ValueError):
        problems.example_source("example1", 3, 1.5, 0.5, 0.0, -1.0)
    with pytest.raises(ValueError):
        couplings.n_from_m(0, 2, 0.5, 2)
    with pytest.raises(ValueError):
        couplings.m_from_n(1, 2, 0.5, 2)
    assert problems.make_case("example2", 1.5, 0.5, s=4).s == 1
    assert problems.make_case("example1", 1.5, 0.5, s=2).s == 2
    # scalar in, scalar out (problems.py:49-52, 75, 85)
    assert isinstance(problems.hypergeom_terminating(0.5, 2, 0.25), float)
    assert isinstance(problems.exact_ifl_of_bump(2, 1.5, 0.25), float)
    assert problems.make_case("example1", 1.5, 0.5).spec.exact(1.0, 0.5) == 0.0


def test_rate_and_temporal_exponent():
    assert couplings.temporal_exponent(2, 0.5) == 1.0
    assert couplings.temporal_exponent(3, 0.8) == pytest.approx(1.2)
    assert couplings.rate(4.0, 1.0) == 2.0
