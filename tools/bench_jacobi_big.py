"""Time the p = 512 cooperative Jacobi (jacobi_big_kernel) through pf_rayleigh_ritz on a PF_TF32
context with n = p (no preceding filter: full EVD of a random symmetric H)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1904_10585_b200 import Context, PF_TF32

for p in (256, 512):
    n = p
    rng = np.random.default_rng(p)
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = (q * rng.standard_normal(n)) @ q.T
    A = torch.tensor(0.5 * (A + A.T), dtype=torch.float32).cuda()
    U = torch.eye(n, dtype=torch.float32).cuda()
    ctx = Context(n, p, 4, dtype=PF_TF32)
    V = torch.empty((p, n), dtype=torch.float32, device="cuda")
    th = torch.empty(p, dtype=torch.float64, device="cuda")
    for _ in range(2):
        ctx.rayleigh_ritz(A, U, V, th)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ctx.rayleigh_ritz(A, U, V, th)
    e1.record()
    torch.cuda.synchronize()
    d = ctx.diagnostics()
    ms = e0.elapsed_time(e1) / 3
    print(f"grid {os.environ.get('PF_JB_GRID', '64')} p={p}: RR {ms:.2f} ms, sweeps {d['jacobi_sweeps']}, "
          f"per round {ms * 1e3 / max(d['jacobi_sweeps'], 1) / (p - 1):.2f} us", flush=True)
