"""Parity at BASELINE.json's full sizes.

configs[2] (n = 4096, M = 512): 48 instances of the seeded batch (global
indices in tests/golden/cfg2_many.npz, oracle/gen_fullsize.py) marched as one
batch against the reference's own full-size runs, gated at the reference's
floor on the SAME instances (tests/golden/cfg2_floor.json: the unmodified
reference with its FFT engine replaced by the correctly rounded DFT — pooled
±1 on 80.5% of levels, per instance 56-100%, max |Δ| 9, u^M within 9e-12;
see the test's docstring for why the scipy.fft swap understates it); plus
size-independent properties of a 256-instance batch:
  * position invariance — the same instances marched as a different batch
    give bit-identical u^M and iteration counts (each CTA is deterministic);
  * exact homogeneity — doubling f and u^0 doubles u^M bit for bit with the
    same iteration counts (every operation is linear; scaling by 2 is exact).
configs[3] (n = 2^20, M = 256): the whole march against the reference's run
(tests/golden/cfg3.npz: all 256 per-level iteration counts, u at levels
1/64/128/256 sub-sampled every 16th point, its l2 norm and four seeded
projections), gated at that config's engine-swap floor (cfg3_floor.json).
"""

import math

import numpy as np
import pytest

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


def _march_instances(idx):
    """The configs[2] instances with the given GLOBAL indices as one batch."""
    gam, alpha = 0.5, 1.5
    r = (2 - gam) / gam
    parts = [WL.instance_fields(N_, int(b), 1) for b in idx]
    x = parts[0][0]
    kx = np.concatenate([p[1] for p in parts])
    fx = np.concatenate([p[2] for p in parts])
    u0 = np.concatenate([p[3] for p in parts])
    B = len(idx)
    kap = P.SeparableField([np.ones(N_)], lambda t: [1.0 + 0.2 * t])
    src = P.SeparableField([np.ones(N_)], lambda t: [1.0 + t])
    mesh = P.build_mesh(M_, r, 1.0)
    soe = P.build_soe(gam, 1e-12, (1.0 / M_) ** r, 1.0)
    dev = torch.device("cuda:0")
    m = FidsMarch(gam, alpha, 1.0, 1.0, M_, r, N_ + 1, soe, method=0, precond=1, tol=1e-12,
                  max_iters=None, B=B, kappa=_field_separable(kap, x, mesh.t, B, kx[None], dev),
                  source=_field_separable(src, x, mesh.t, B, fx[None], dev),
                  u0=torch.from_numpy(np.ascontiguousarray(u0)).to(dev), device=0,
                  private_plan=True)
    m.run(64)
    u64 = m.u_level(64).cpu().numpy().copy()
    m.run()
    res = m.result()
    assert np.all(res.status == 0)
    out = u64, res.u_final.cpu().numpy().copy(), res.iterations.copy()
    del m, res
    torch.cuda.empty_cache()
    return out


def test_cfg2_full_size_vs_reference_goldens():
    """48 configs[2] instances vs the reference (cfg2_many.npz), gated at the
    reference's own floor on the same instances (cfg2_floor.json).

    Two floors are committed, both the UNMODIFIED reference with only its FFT
    engine replaced (oracle/gen_fullsize.py):
      * scipy.fft: pooled ±1 on 98.5% of levels — but scipy's complex ifft is
        bit-identical to numpy's, so this only perturbs the real-input forward
        transforms and understates what a second engine sees;
      * the correctly rounded DFT (long double, rounded once): pooled ±1 on
        80.5%, mean Δ -0.05, max |Δ| 9, per instance 56-100%, u^M within
        9e-12 — the floor of ANY accurate second engine, and the gate here.
    """
    import json
    from pathlib import Path
    g = golden("cfg2_many")
    floor = json.loads((Path(__file__).parent / "golden" / "cfg2_floor.json").read_text())
    ex = floor["exact_engine"]
    idx = g["instances"]
    u64, uM, its = _march_instances(idx)
    all_d, rows = [], []
    for i, b in enumerate(idx):
        fl = ex[f"b{b}"]
        d = its[:, i] - g[f"b{b}_its"]
        all_d.append(d)
        frac = float(np.mean(np.abs(d) <= 1))
        e64 = rel_l2(u64[i], g[f"b{b}_u64"])
        eM = rel_l2(uM[i], g[f"b{b}_uM"])
        rows.append((int(b), frac, fl["within1"], int(np.abs(d).max()), e64, eM))
        # solution: within 10x the exact engine's distance on this instance (or 1e-10)
        assert e64 <= max(1e-10, 10 * fl["rel_l2_u64"]), (b, e64)
        assert eM <= max(1e-10, 10 * fl["rel_l2_uM"]), (b, eM)
    rows.sort(key=lambda r: r[1])
    for r in rows[:6]:
        print("cfg2 b%d: within+-1 %.3f (exact-engine floor %.3f) max|d| %d e64 %.2e eM %.2e" % r)
    D = np.concatenate(all_d)
    pooled = float(np.mean(np.abs(D) <= 1))
    print(f"cfg2 x{len(idx)} pooled: within+-1 {pooled:.4f} (exact-engine floor "
          f"{ex['pooled']['within1']:.4f}, scipy-swap {floor['pooled']['within1']:.4f}) mean d "
          f"{D.mean():+.4f} (floor {ex['pooled']['mean_d']:+.4f}) max|d| {np.abs(D).max()} "
          f"(floor {ex['pooled']['max_abs_d']})")
    # which instances sit at the rounding floor differs between any two
    # engines: per instance the bar is the floor's worst instance with margin
    assert rows[0][1] >= ex["pooled"]["min_within1"] - 0.2, rows[0]
    assert np.abs(D).max() <= 2 * max(2, ex["pooled"]["max_abs_d"])
    assert pooled >= ex["pooled"]["within1"] - 0.03
    assert abs(D.mean()) <= max(0.1, 3.0 * D.std() / math.sqrt(D.size)), (D.mean(), D.std())


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


def test_cfg3_full_march_vs_reference():
    """configs[3] (n = 2^20, M = 256, gamma = 0.7, alpha = 1.2): all 256 levels
    of run_fids's device march against the reference's own run
    (cfg3.npz), gated at the engine-swap floor of the same run (cfg3_floor.json)."""
    import json
    from pathlib import Path
    g = golden("cfg3")
    floor = json.loads((Path(__file__).parent / "golden" / "cfg3_floor.json").read_text())
    n, M, gam, alpha = 1 << 20, 256, 0.7, 1.2
    r = (2 - gam) / gam
    x = WL.grid(n)
    kap = P.SeparableField([np.ones(n), 0.5 * np.sin(np.pi * x)], lambda t: [1.0, math.exp(-t)])
    src = P.SeparableField([np.sin(np.pi * x)], lambda t: [1.0 + t])
    mesh = P.build_mesh(M, r, 1.0)
    soe = P.build_soe(gam, 1e-12, (1.0 / M) ** r, 1.0)
    dev = torch.device("cuda:0")
    u0 = (1.0 - x * x) ** 2
    m = FidsMarch(gam, alpha, 1.0, 1.0, M, r, n + 1, soe, method=0, precond=1, tol=1e-12,
                  max_iters=None, B=1, kappa=_field_separable(kap, x, mesh.t, 1, None, dev),
                  source=_field_separable(src, x, mesh.t, 1, None, dev),
                  u0=torch.from_numpy(u0[None, :].copy()).to(dev), device=0)
    sub = int(g["sub"][0])
    Pj = np.random.default_rng(int(g["proj_seed"][0])).standard_normal((4, n))
    done = 0
    for lv in g["levels"]:
        m.run(int(lv) - done)
        done = int(lv)
        u = m.u_level(done)[0].cpu().numpy()
        e_sub = rel_l2(u[::sub], g[f"u{lv}_sub"])
        nref = float(g[f"u{lv}_norm"][0])
        e_norm = abs(np.linalg.norm(u) - nref) / nref
        e_proj = float(np.max(np.abs(Pj @ u - g[f"u{lv}_proj"]))) / (nref * math.sqrt(n))
        # the reference against itself with another FFT engine (scipy swap
        # and, when generated, the correctly rounded DFT): 9e-13 at level 1,
        # 4.5e-10 at level 256 — the march's drift at n = 2^20
        fl_u = max(floor[f"rel_l2_u{lv}"], floor.get("exact_engine", {}).get(f"rel_l2_u{lv}", 0.0))
        tol_u = max(1e-10, 10 * fl_u)
        print(f"cfg3 level {lv}: sub rel-l2 {e_sub:.2e} norm {e_norm:.2e} proj {e_proj:.2e} "
              f"(floor {floor[f'rel_l2_u{lv}']:.2e})")
        assert e_sub <= tol_u and e_norm <= tol_u and e_proj <= tol_u, lv
    res = m.result()
    assert np.all(res.status == 0)
    d = res.iterations[:, 0] - g["its"]
    frac = float(np.mean(np.abs(d) <= 1))
    print(f"cfg3: within+-1 {frac:.3f} (floor {floor['within1']:.3f}) mean d {d.mean():+.3f} "
          f"(floor {floor['mean_d']:+.3f}) max|d| {np.abs(d).max()} (floor {floor['max_abs_d']})")
    ex = floor.get("exact_engine", floor)
    # second-structure floors (tools/cfg3_structure_floor.py: the reference's
    # control flow with this repo's transform structures emulated in numpy)
    sf = Path(__file__).parent / "golden" / "cfg3_structure_floor.json"
    st_floor = min(v["within1"] for v in json.loads(sf.read_text()).values()) if sf.exists() else 1.0
    assert frac >= min(0.95, min(floor["within1"], ex["within1"], st_floor) - 0.05)
    # bias: MORE iterations than the reference would mean a less accurate
    # engine (gate: 0.1 or three standard errors); the device takes slightly
    # FEWER at this size (-0.11 with the per-level SOE schedule, -0.18 with
    # the blocked one; the numpy structure floors: +0.02 / -0.02) with the
    # solution inside the floor at every stored level — bounded, not gated tight
    assert d.mean() <= max(0.1, 3.0 * d.std() / math.sqrt(d.size)), (d.mean(), d.std())
    assert d.mean() >= -0.3, d.mean()
    assert np.max(np.abs(d)) <= 2 * max(2, floor["max_abs_d"], ex["max_abs_d"])
