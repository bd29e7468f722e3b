"""Time pf_rayleigh_ritz with n = p (so it is dominated by the Jacobi solve)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1904_10585_b200 import Context

for p in (16, 32, 64, 128):
    n = p
    rng = np.random.default_rng(p)
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = (q * rng.standard_normal(n)) @ q.T
    A = torch.tensor(0.5 * (A + A.T)).cuda()
    U = torch.eye(n, dtype=torch.float64).cuda()
    ctx = Context(n, p, 4)
    V = torch.empty((n, p), dtype=torch.float64, device="cuda")
    th = torch.empty(p, dtype=torch.float64, device="cuda")
    for _ in range(3):
        ctx.rayleigh_ritz(A, U, V, th)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.rayleigh_ritz(A, U, V, th)
    e1.record()
    torch.cuda.synchronize()
    d = ctx.diagnostics()
    ms = e0.elapsed_time(e1) / 10
    print(f"p={p}: RR {ms*1e3:.1f} us, sweeps {d['jacobi_sweeps']}, per sweep {ms*1e3/max(d['jacobi_sweeps'],1):.1f} us, "
          f"per round {ms*1e3/max(d['jacobi_sweeps'],1)/(p-1):.2f} us")
