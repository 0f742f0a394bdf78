"""Quick device timing probe (CUDA events) for the first kernels."""
import sys, time, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2002_11978_b200 as P
from paper_2002_11978_b200 import _native, toeplitz as TZ

def ev_time(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3

lib = _native.load()
for n in (1024, 2048, 4096):
    d = P.build_ifl(1.5, 1.75, 1.0, n + 1)
    op = P.build_toeplitz(d.first_col)
    B = (1 << 26) // n
    x = torch.randn(B, n, dtype=torch.float64, device="cuda")
    k = torch.rand(B, n, dtype=torch.float64, device="cuda") * 1.5 + 0.5
    y = torch.empty_like(x)
    pl = op.plan
    st = _native.stream_ptr()
    t = ev_time(lambda: lib.tsf_toeplitz_matvec(pl.handle, B, x.data_ptr(), y.data_ptr(), k.data_ptr(), 3.0, st))
    gbs = 24.0 * n * B / t / 1e9
    t2 = ev_time(lambda: lib.tsf_precond_solve(pl.handle, B, x.data_ptr(), y.data_ptr(), 3.0, 1.2, None, st))
    gbs2 = 16.0 * n * B / t2 / 1e9
    print(f"n={n} B={B}: matvec {t*1e3:.3f} ms {gbs:.0f} GB/s | precond {t2*1e3:.3f} ms {gbs2:.0f} GB/s", flush=True)

# SOE push+rhs at N_exp=143, n=4096, B=512
n, nexp, B = 4096, 143, 512
W = torch.randn(B, nexp, n, dtype=torch.float64, device="cuda")
u = torch.randn(B, n, dtype=torch.float64, device="cuda"); up = torch.randn_like(u); rhs = torch.empty_like(u)
tab = torch.rand(3, nexp, dtype=torch.float64, device="cuda")
st = _native.stream_ptr()
t = ev_time(lambda: lib.tsf_soe_push_rhs(B, n, nexp, W.data_ptr(), u.data_ptr(), up.data_ptr(), 1e-3, tab[0].data_ptr(), tab[1].data_ptr(), tab[2].data_ptr(), 1, 0, 1, 2.0, 1.7, u.data_ptr(), rhs.data_ptr(), st))
print(f"soe push+rhs nexp={nexp} n={n} B={B}: {t*1e3:.3f} ms  {(16*nexp+40)*n*B/t/1e9:.0f} GB/s", flush=True)
del W

# batched march, cfg2-shaped, small M
n, M, Bm = 4096, 12, 1024
N = n + 1
x = -1.0 + (2.0 / N) * np.arange(1, N)
rng = np.random.default_rng(0)
kx = np.exp(0.4 * rng.standard_normal((Bm, 1)) * np.sin(np.pi * x)[None, :])
fx = rng.standard_normal((Bm, 1)) * np.sin(np.pi * x)[None, :]
u0 = (1 - x * x) ** 2 * rng.uniform(0.5, 2.0, (Bm, 1))
kap = P.SeparableField([np.ones(n)], lambda t: [1.0 + 0.2 * t])
src = P.SeparableField([np.ones(n)], lambda t: [1.0 + t])
t0 = time.perf_counter()
uB, rep = P.run_fids_batched(0.5, 1.5, M, 3.0, N, kap, src, u0, kappa_modes=kx[None], source_modes=fx[None],
                             epsilon=1e-12, options=P.SolverOptions(solver="pkrylov", tol=1e-12))
t1 = time.perf_counter()
its = rep["iterations"]
print(f"batched march B={Bm} n={n} M={M}: {t1-t0:.2f} s wall incl setup, its mean {its.mean():.2f} max {its.max()}", flush=True)
