"""Time the fused rank-p rebuild + PFAM update (pf_admm_step, K7) at config-3 size on its own:
python tools/bench_update.py [n] [p] [fuse(1|0)] [reps].  Development measurement (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from pfinputs import CONFIGS, reduced, pfam_problem
from paper_1904_10585_b200._lib import Context, PF_FP64_I8, PF_FP64


def main(n=16384, p=64, fuse=1, reps=10):
    cfg = reduced(CONFIGS[3], n=n, p=p)
    prob = pfam_problem(cfg)
    rs = np.random.default_rng(0)
    V = torch.from_numpy(np.linalg.qr(rs.standard_normal((n, p)))[0]).cuda()
    f = torch.from_numpy(np.abs(rs.standard_normal(p)) * 30.0).cuda()
    g = torch.Generator(device="cuda").manual_seed(1)
    Z = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g) * 1e-2
    Z = (Z + Z.T) * 0.5
    adj = torch.from_numpy(np.ascontiguousarray(prob["adj_bits"]).view(np.int32)).cuda()
    deg = torch.from_numpy(prob["deg"]).cuda()
    obj = torch.zeros(2, dtype=torch.float64, device="cuda")
    c = Context(n, p, 4, dtype=PF_FP64_I8 if fuse else PF_FP64)
    for _ in range(2):
        c.admm_step(V, f, 1.0, adj, deg, Z, obj)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c.admm_step(V, f, 1.0, adj, deg, Z, obj)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byt = 8 * n * n * (1.5 if fuse == 0 else 1.5) + (7 * n * n if fuse else 0)
    print(f"n={n} p={p} fuse={fuse}: {ms:.3f} ms per update, {byt / ms / 1e6:.0f} GB/s algorithmic")


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
