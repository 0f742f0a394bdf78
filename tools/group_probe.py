"""Concurrency probe: the configs[2] batch split into G groups, each a
FidsMarch with a private plan on its own stream, marched level by level
round-robin (no host sync).  Prints ms per level for G = 1, 2, 4, 8."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import paper_2002_11978_b200 as P
from paper_2002_11978_b200 import workloads as WL
from paper_2002_11978_b200.scheme import FidsMarch, _field_separable

n, M, B = 4096, 512, 4096
gam, alpha = 0.5, 1.5
r = (2 - gam) / gam
levels = int(sys.argv[1]) if len(sys.argv) > 1 else 60
x, kx, fx, u0 = WL.instance_fields(n, 0, B)
kap = P.SeparableField([np.ones(n)], lambda t: [1.0 + 0.2 * t])
src = P.SeparableField([np.ones(n)], lambda t: [1.0 + t])
mesh = P.build_mesh(M, r, 1.0)
soe = P.build_soe(gam, 1e-12, (1.0 / M) ** r, 1.0)
dev = torch.device("cuda:0")
for G in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2", "4", "8"])]:
    marches, streams = [], []
    bg = B // G
    for g in range(G):
        sl = slice(g * bg, (g + 1) * bg)
        kd = _field_separable(kap, x, mesh.t, bg, kx[None, sl], dev)
        fd = _field_separable(src, x, mesh.t, bg, fx[None, sl], dev)
        marches.append(FidsMarch(gam, alpha, 1.0, 1.0, M, r, n + 1, soe, method=0, precond=1,
                                 tol=1e-12, max_iters=None, B=bg, kappa=kd, source=fd,
                                 u0=torch.from_numpy(np.ascontiguousarray(u0[sl])).to(dev),
                                 device=0, private_plan=True))
        streams.append(torch.cuda.Stream(dev))
    for mh in marches:
        mh.reset()
    torch.cuda.synchronize()
    for mh, st in zip(marches, streams):     # warm-up: 3 levels each
        mh.run(3, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_event(e0)
    for _ in range(levels):
        for mh, st in zip(marches, streams):
            mh.run(1, stream=st)
    for s in streams:
        e = torch.cuda.Event()
        e.record(s)
        torch.cuda.current_stream().wait_event(e)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / levels
    its = np.concatenate([mh.iters[3:3 + levels].cpu().numpy() for mh in marches], axis=1)
    print(f"G={G}: {ms:.3f} ms/level over levels 4..{3 + levels}, mean its {its.mean():.3f}",
          flush=True)
    del marches
    torch.cuda.empty_cache()
