"""Wave-efficiency probe of the batched level solve (configs[2] shape):
runs a short march, then from the per-level, per-instance iteration counts
estimates how many CTA slots each phase launch spends on finished instances
(every launch covers all B instances; finished ones exit at once)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import paper_2002_11978_b200 as P
from paper_2002_11978_b200 import workloads as WL
from paper_2002_11978_b200.scheme import FidsMarch, _field_separable

n, M, B, levels = 4096, 512, int(sys.argv[1]) if len(sys.argv) > 1 else 4096, 40
gam, alpha = 0.5, 1.5
r = (2 - gam) / gam
x, kx, fx, u0 = WL.instance_fields(n, 0, B)
kap = P.SeparableField([np.ones(n)], lambda t: [1.0 + 0.2 * t])
src = P.SeparableField([np.ones(n)], lambda t: [1.0 + t])
mesh = P.build_mesh(M, r, 1.0)
soe = P.build_soe(gam, 1e-12, (1.0 / M) ** r, 1.0)
dev = torch.device("cuda:0")
kd = _field_separable(kap, x, mesh.t, B, kx[None], dev)
fd = _field_separable(src, x, mesh.t, B, fx[None], dev)
march = FidsMarch(gam, alpha, 1.0, 1.0, M, r, n + 1, soe, method=0, precond=1, tol=1e-12,
                  max_iters=None, B=B, kappa=kd, source=fd, u0=torch.from_numpy(u0).to(dev),
                  device=0)
march.reset()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * levels)]
march.run(levels, events=ev)
torch.cuda.synchronize()
its = march.iters[:levels].cpu().numpy()
sms = torch.cuda.get_device_properties(0).multi_processor_count
tot_work, tot_slots, done_ctas = 0.0, 0.0, 0
for m in range(levels):
    it = its[m]
    mx = int(it.max())
    for k in range(1, mx + 1):
        active = int(np.sum(it >= k))
        tot_work += active
        tot_slots += np.ceil(active / sms) * sms
        done_ctas += B - active
solve_ms = [ev[3 * i + 1].elapsed_time(ev[3 * i + 2]) for i in range(levels)]
print(f"B={B} levels={levels} mean its {its.mean():.2f} max-mean per level "
      f"{np.mean(its.max(axis=1) - its.mean(axis=1)):.2f}")
print(f"wave efficiency (active CTAs / full waves) {tot_work / tot_slots:.3f}; "
      f"finished-instance CTAs launched per level {done_ctas / levels:.0f} "
      f"(x2 phases); solve ms/level {np.mean(solve_ms[4:]):.3f}")
