"""Times pf_orth (CholeskyQR2: Gram, p x p Cholesky + inverse, Y R^{-1}, twice) on an n x p fp64
block -- the orthonormalisation step a3.  Development tool: PF_CHOL_BIG=1 selects the 32-column
panel Cholesky for p >= 64."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1904_10585_b200 import Context

for n, p in ((16384, 64), (32768, 128)):
    g = torch.Generator(device="cuda").manual_seed(0)
    Y0 = torch.randn((n, p), dtype=torch.float64, device="cuda", generator=g)
    Y0 = Y0 * torch.logspace(0, 4, p, dtype=torch.float64, device="cuda")[None, :]
    Y = Y0.clone()
    ctx = Context(n, p, 4)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ctx.orth(Y, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20):
            Y.copy_(Y0)
            ctx.orth(Y, st)
        e1.record(st)
    torch.cuda.synchronize()
    err = torch.linalg.norm(Y.T @ Y - torch.eye(p, dtype=torch.float64, device="cuda")).item()
    print(f"n={n} p={p}: orth {e0.elapsed_time(e1) / 20 * 1e3:.1f} us (incl. an 8 MB copy), "
          f"||Q^T Q - I|| = {err:.2e}", flush=True)
