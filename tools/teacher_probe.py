"""Teacher-forced parity probe on configs[0]: each level is solved on the
device from the reference's own (u^{m-1}, W^{m-1}); prints the iteration
delta distribution next to the end-to-end one."""
import sys, math
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import oracle as O
from tsf_testlib import golden, cfg0_fields
import paper_2002_11978_b200 as P
from scipy.special import gammaln

g = golden("march")
hist_ref, its_ref = g["cfg0_hist"], g["cfg0_its"]
gam, a, M, N = 0.5, 1.5, 256, 1025
n = N - 1
t, tau = O.graded_mesh(M, 3.0, 1.0)
col, h, _ = O.ifl_column(a, 1.0 + a / 2, 1.0, N)
x = -1.0 + h * np.arange(1, N)
s, w = O.soe_build(gam, 1e-12, (1.0 / M) ** 3.0, 1.0)
G = math.exp(gammaln(1 - gam))
kf, ff, _ = cfg0_fields()
op = P.build_toeplitz(col)
W = np.zeros((s.size, n))
tf = []
for m in range(1, M + 1):
    if m > 1:
        O.soe_push(W, s, hist_ref[m - 1] - hist_ref[m - 2], tau[m - 2])
    amm = O.last_l1_weight(tau[m - 1], gam)
    kap = kf(x, t[m])
    rhs = ff(x, t[m]) + (amm * hist_ref[m - 1] - O.soe_history_term(W, s, w, tau[m - 1])) / G
    shift = amm / G
    pc = P.build_preconditioner(col, shift, float(kap.mean()))
    u, rep = P.solve_bicgstab(P.LevelOperator(op, shift, kap), pc, rhs, tol=1e-12)
    tf.append(rep.iterations)
tf = np.array(tf)
d = tf - its_ref
print("teacher-forced: within1 %.4f mean %.3f" % (np.mean(np.abs(d) <= 1), d.mean()), np.unique(d, return_counts=True))
spec = P.ProblemSpec(gamma=gam, alpha=a, l=1.0, T=1.0, kappa=kf, source=ff, initial=cfg0_fields()[2])
hist, rep = P.run_fids(spec, M, 3.0, N, epsilon=1e-12, options=P.SolverOptions(solver="pkrylov", tol=1e-12))
d = rep.iterations - its_ref
print("end-to-end:     within1 %.4f mean %.3f" % (np.mean(np.abs(d) <= 1), d.mean()), np.unique(d, return_counts=True))
print("relres last steps", rep.relres[-5:])
