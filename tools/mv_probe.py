"""Probe: standalone large-n matvec timing in a fresh process vs after a march."""
import sys, json, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2002_11978_b200 as P
from paper_2002_11978_b200 import _native

def mv_time(n, B, reps=5):
    col = P.build_ifl(1.5, 1.75, 1.0, n + 1).first_col
    op = P.build_toeplitz(col)
    x = torch.randn(B, n, dtype=torch.float64, device="cuda")
    k = torch.rand(B, n, dtype=torch.float64, device="cuda") + 0.5
    y = torch.empty_like(x)
    lib = _native.load(); st = _native.stream_ptr()
    f = lambda: _native.check(lib.tsf_toeplitz_matvec(op.plan.handle, B, x.data_ptr(), y.data_ptr(), k.data_ptr(), 2.0, st))
    f(); torch.cuda.synchronize()
    out = []
    for r in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); out.append(a.elapsed_time(b))
    return out

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
print("fresh B=64", mv_time(n, (1 << 26) // n))
print("B=1", mv_time(n, 1))
print("B=8", mv_time(n, 8))
print("again B=64", mv_time(n, (1 << 26) // n))
