"""Pin the CPU oracle (oracle/tsfrac_oracle.py) to the upstream reference's
golden vectors (tests/golden/, written by oracle/gen_golden.py).

Bit-exactness is expected where the oracle performs the same numpy
operations in the same order as the reference; tolerances below 1e-15
relative are used only where BLAS dot ordering may differ between hosts.
"""

import math

import numpy as np
import pytest

import oracle as O
from tsf_testlib import cfg0_fields as _cfg0_fields, golden, rel_err as _rel


class TestSetupPins:
    @pytest.mark.parametrize("tag,M,r", [("m8r2", 8, 2.0), ("m256r3", 256, 3.0),
                                         ("m512r3", 512, 3.0), ("m64r1", 64, 1.0)])
    def test_mesh_and_l1(self, tag, M, r):
        g = golden("setup")
        t, tau = O.graded_mesh(M, r, 1.0)
        np.testing.assert_array_equal(t, g[f"mesh_{tag}_t"])
        np.testing.assert_array_equal(tau, g[f"mesh_{tag}_tau"])
        for m in sorted({1, 2, M // 2, M}):
            for gam, key in ((0.5, "g05"), (0.8, "g08")):
                a = O.l1_weight_row(t, tau, gam, m)
                assert _rel(a, g[f"mesh_{tag}_l1_{key}_m{m}"]) <= 1e-13
                assert a[-1] == O.last_l1_weight(tau[m - 1], gam)

    def test_ifl_columns(self):
        g = golden("setup")
        i = 0
        while f"ifl{i}_args" in g:
            a, mu, l, N = g[f"ifl{i}_args"]
            col, h, scale = O.ifl_column(a, mu, l, int(N))
            assert _rel(col, g[f"ifl{i}_col"]) <= 1e-13
            assert h == g[f"ifl{i}_hscale"][0]
            i += 1
        assert i >= 5

    @pytest.mark.parametrize("tag", ["cfg0", "cfg1_g03", "cfg1_g05", "cfg1_g08",
                                     "cfg2", "cfg3", "t_half", "t_ex2", "t_pos"])
    def test_soe_nodes_weights(self, tag):
        g = golden("setup")
        gam, eps, delta, T = g[f"soe_{tag}_args"]
        s, w = O.soe_build(gam, eps, delta, T)
        assert s.size == g[f"soe_{tag}_s"].size
        assert _rel(s, g[f"soe_{tag}_s"]) <= 1e-13
        assert _rel(w, g[f"soe_{tag}_w"]) <= 1e-13

    def test_soe_sizes_match_survey(self):
        # N_exp = 131 / 239 / 155 / 104 / 143 / 101
        g = golden("setup")
        sizes = {k: g[f"soe_{k}_s"].size for k in
                 ("cfg0", "cfg1_g03", "cfg1_g05", "cfg1_g08", "cfg2", "cfg3")}
        assert sizes == {"cfg0": 131, "cfg1_g03": 239, "cfg1_g05": 155,
                         "cfg1_g08": 104, "cfg2": 143, "cfg3": 101}


class TestLinearAlgebraPins:
    def _cases(self):
        g = golden("linalg")
        i = 0
        while f"tp{i}_col" in g:
            yield i, g
            i += 1

    def test_toeplitz_and_preconditioner(self):
        for i, g in self._cases():
            col, v = g[f"tp{i}_col"], g[f"tp{i}_v"]
            L, spec = O.toeplitz_symbol(col)
            if f"tp{i}_spec" in g:
                np.testing.assert_array_equal(spec, g[f"tp{i}_spec"])
            np.testing.assert_array_equal(O.toeplitz_apply(spec, v), g[f"tp{i}_Av"])
            np.testing.assert_array_equal(O.strang_column(col), g[f"tp{i}_cs"])
            lam = O.strang_eigs(col)
            np.testing.assert_array_equal(lam, g[f"tp{i}_lam"])
            shift = g[f"tp{i}_shift"][0]
            kap = g[f"tp{i}_kappa"]
            total = shift + float(kap.mean()) * lam
            np.testing.assert_array_equal(total, g[f"tp{i}_total"])
            np.testing.assert_array_equal(O.precond_apply(total, v), g[f"tp{i}_Pinv_v"])

    def test_bicgstab_cg_plain(self):
        for i, g in self._cases():
            col = g[f"tp{i}_col"]
            _, spec = O.toeplitz_symbol(col)
            lam = O.strang_eigs(col)
            shift = g[f"tp{i}_shift"][0]
            kap = g[f"tp{i}_kappa"]
            total = shift + float(kap.mean()) * lam
            apply = lambda q: shift * q + kap * O.toeplitz_apply(spec, q)  # noqa: E731
            for tol in (10, 12):
                key = f"tp{i}_bicg_{tol}"
                x, out = O.bicgstab(apply, lambda q: O.precond_apply(total, q),
                                    g[f"{key}_b"], tol=10.0 ** -tol)
                its, rel, conv = g[f"{key}_rep"]
                assert out.iterations == int(its) and out.converged == bool(conv)
                assert _rel(x, g[f"{key}_x"]) <= 1e-14
            kc = g[f"tp{i}_cg_kc"][0]
            tot_c = shift + kc * lam
            x, out = O.cg(lambda q: shift * q + kc * O.toeplitz_apply(spec, q),
                          lambda q: O.precond_apply(tot_c, q), g[f"tp{i}_bicg_12_b"],
                          tol=1e-12)
            assert out.iterations == int(g[f"tp{i}_cg_rep"][0])
            assert _rel(x, g[f"tp{i}_cg_x"]) <= 1e-14
            x, out = O.bicgstab(apply, None, g[f"tp{i}_bicg_12_b"], tol=1e-10)
            assert out.iterations == int(g[f"tp{i}_plain_rep"][0])
            assert _rel(x, g[f"tp{i}_plain_x"]) <= 1e-13

    def test_soe_push_and_history_term(self):
        g = golden("linalg")
        s, w = O.soe_build(0.5, 1e-12, (1.0 / 256) ** 3, 1.0)
        W = g["push_W0"].copy()
        tau_push, tau_rhs = g["push_tau"]
        H = O.soe_history_term(W, s, w, tau_rhs)
        rhs = (12.5 * g["push_uprev"] - H) / math.exp(math.lgamma(0.5))
        assert _rel(rhs, g["push_rhs"]) <= 1e-14
        O.soe_push(W, s, g["push_du"], tau_push)
        np.testing.assert_array_equal(W, g["push_W1"])


class TestMarchPins:
    @pytest.mark.parametrize("tag", ["s1", "s2", "s3", "s4", "s5"])
    def test_small_marches(self, tag):
        g = golden("march")
        gam, a, M, N, tol, r = g[f"{tag}_args"]
        rec = O.fids_march(gam, a, 1.0, 1.0, int(M), r, int(N), *_cfg0_fields(),
                           epsilon=1e-12, tol=tol)
        np.testing.assert_array_equal(rec.iterations, g[f"{tag}_its"])
        assert _rel(rec.hist, g[f"{tag}_hist"]) <= 1e-13

    def test_cfg0_full(self):
        g = golden("march")
        rec = O.fids_march(0.5, 1.5, 1.0, 1.0, 256, 3.0, 1025, *_cfg0_fields(),
                           epsilon=1e-12, tol=1e-12)
        np.testing.assert_array_equal(rec.iterations, g["cfg0_its"])
        assert _rel(rec.hist, g["cfg0_hist"]) <= 1e-13
        assert rec.nodes.size == 131

    def test_zero_data_exactly_zero(self):
        g = golden("march")
        rec = O.fids_march(0.5, 1.5, 1.0, 1.0, 8, 2.0, 257,
                           lambda x, t: np.ones_like(x), lambda x, t: np.zeros_like(x),
                           lambda x: np.zeros_like(x), epsilon=1e-10, tol=1e-10)
        np.testing.assert_array_equal(rec.hist, g["zero_hist"])
        assert np.all(rec.iterations == 0)

    def test_unpreconditioned_and_cg(self):
        g = golden("march")
        k, f, phi = _cfg0_fields()
        rec = O.fids_march(0.5, 1.5, 1.0, 1.0, 16, 3.0, 129, k, f, phi,
                           epsilon=1e-12, tol=1e-10, precondition=False)
        np.testing.assert_array_equal(rec.iterations, g["plain_its"])
        assert _rel(rec.hist, g["plain_hist"]) <= 1e-12
        rec = O.fids_march(0.5, 1.5, 1.0, 1.0, 16, 3.0, 257,
                           lambda x, t: np.full_like(x, 1.0 + 0.5 * t), f, phi,
                           epsilon=1e-12, tol=1e-12, use_cg=True)
        np.testing.assert_array_equal(rec.iterations, g["cg_its"])
        assert _rel(rec.hist, g["cg_hist"]) <= 1e-13


class TestDidsPins:
    """run_dids (scheme.py:184-233) restated by oracle.dids_march."""

    @pytest.mark.parametrize("tag", ["d1", "d2", "d3"])
    def test_dids_marches(self, tag):
        g = golden("dids")
        gam, a, M, N, tol, r = g[f"{tag}_args"]
        solver = str(g[f"{tag}_solver"])
        rec = O.dids_march(gam, a, 1.0, 1.0, int(M), r, int(N), *_cfg0_fields(), tol=tol,
                           precondition=solver == "pkrylov")
        np.testing.assert_array_equal(rec.iterations, g[f"{tag}_its"])
        assert _rel(rec.hist, g[f"{tag}_hist"]) <= 1e-13
        assert rec.iterations.sum() / M == g[f"{tag}_avg"][0]
        np.testing.assert_array_equal(g[f"{tag}_ops"], np.arange(1, int(M) + 1) * (int(N) - 1))

    @pytest.mark.parametrize("tag", ["d1", "d2", "d3", "d4"])
    def test_fids_dids_proximity_in_the_goldens(self, tag):
        # the reference's criterion 7 (pkg/tests/test_acceptance.py:141-166),
        # here at SOE eps 1e-12: |DIDS - FIDS| <= 100 eps
        g = golden("dids")
        assert np.max(np.abs(g[f"{tag}_hist"] - g[f"{tag}_fids_hist"])) <= 100 * 1e-12


def test_cfg2_full_size_instances_pin_the_oracle():
    """Two configs[2] instances at full size (n = 4096, M = 512): the oracle
    reproduces the reference's per-level iterations and u^M bit for bit."""
    from paper_2002_11978_b200 import workloads as WL
    g = golden("cfg2")
    b = 37
    x, kx, fx, u0 = WL.instance_fields(4096, b, 1)
    rec = O.fids_march(0.5, 1.5, 1.0, 1.0, 512, 3.0, 4097,
                       lambda xx, t: kx[0] * (1.0 + 0.2 * t), lambda xx, t: fx[0] * (1.0 + t),
                       lambda xx: u0[0], epsilon=1e-12, tol=1e-12, keep_history=False)
    np.testing.assert_array_equal(rec.iterations, g[f"b{b}_its"])
    np.testing.assert_array_equal(rec.hist, g[f"b{b}_uM"])
