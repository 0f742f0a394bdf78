"""Product host setup (mesh, L1, IFL column, SOE, Strang column) against the
reference goldens — the setup is the reference's own numpy path restated."""

import numpy as np
import pytest

import paper_2002_11978_b200 as P
from tsf_testlib import golden, rel_err


@pytest.mark.parametrize("tag,M,r", [("m8r2", 8, 2.0), ("m256r3", 256, 3.0), ("m64r1", 64, 1.0)])
def test_mesh_l1(tag, M, r):
    g = golden("setup")
    mesh = P.build_mesh(M, r, 1.0)
    np.testing.assert_array_equal(mesh.t, g[f"mesh_{tag}_t"])
    for m in sorted({1, 2, M // 2, M}):
        assert rel_err(P.l1_weights(mesh, 0.5, m).a, g[f"mesh_{tag}_l1_g05_m{m}"]) <= 1e-13


def test_ifl_columns():
    g = golden("setup")
    i = 0
    while f"ifl{i}_args" in g:
        a, mu, l, N = g[f"ifl{i}_args"]
        d = P.build_ifl(a, mu, l, int(N))
        assert rel_err(d.first_col, g[f"ifl{i}_col"]) <= 1e-13
        i += 1


@pytest.mark.parametrize("tag", ["cfg0", "cfg1_g03", "cfg1_g05", "cfg1_g08", "cfg2", "cfg3",
                                 "t_half", "t_ex2", "t_pos"])
def test_soe(tag):
    g = golden("setup")
    gam, eps, delta, T = g[f"soe_{tag}_args"]
    soe = P.build_soe(gam, eps, delta, T)
    assert soe.n_exp == g[f"soe_{tag}_s"].size
    assert rel_err(soe.nodes, g[f"soe_{tag}_s"]) <= 1e-13
    assert rel_err(soe.weights, g[f"soe_{tag}_w"]) <= 1e-13


def test_soe_errors():
    with pytest.raises(P.SoeConstructionError):
        P.build_soe(0.5, 1e-10, 1.0, 1.0)
    with pytest.raises(P.SoeConstructionError):
        P.build_soe(0.5, 1e-10, 1e-7, 1.0, node_cap=20)
    with pytest.raises(ValueError):
        P.build_soe(1.5, 1e-10, 1e-3, 1.0)


def test_strang_column_kats():
    # pkg/tests/test_toeplitz.py:63-75
    np.testing.assert_array_equal(P.strang_first_column(np.array([10.0, 20, 30, 40, 50])),
                                  [10.0, 20.0, 30.0, 30.0, 20.0])
    np.testing.assert_array_equal(P.strang_first_column(np.array([1.0, 2, 3, 4])),
                                  [1.0, 2.0, 3.0, 2.0])
    with pytest.raises(ValueError):
        P.strang_first_column(np.array([1.0]))


def test_select_solver():
    assert P.select_solver(64) == "direct"
    assert P.select_solver(512) == "pkrylov"
    assert P.select_solver(512, P.SolverOptions(solver="krylov")) == "krylov"


def test_separable_field_matches_numpy_expression():
    x = np.linspace(-1, 1, 1025)[1:-1]
    fld = P.SeparableField([np.ones_like(x), 0.5 * np.sin(np.pi * x)],
                           lambda t: [1.0, float(np.exp(-t))])
    for t in (0.0, 0.25, 1.0):
        np.testing.assert_array_equal(fld(x, t), 1.0 + 0.5 * np.sin(np.pi * x) * np.exp(-t))


def test_device_entry_points_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2002_11978_b200 import _native
    with pytest.raises(_native.NativeError):
        P.toeplitz_matvec(P.build_toeplitz(np.array([2.0, -1.0, 0.0])), np.ones(3))
