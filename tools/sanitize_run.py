"""Small runs of every hot-path kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): python tools/sanitize_run.py [quick].  Reduced configs 1-4 (fp64 DMMA K1,
int8-digit K1-i8 with the fused PFAM digits, K7 PFPG / PFAM, Jacobi p <= 128, Cholesky variants,
Lanczos) and a reduced config 5 (TF32 K1t, cooperative Jacobi / panel Cholesky, Newton-Schulz).
No oracle: the parity suite checks the numbers; this only drives the kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from pfinputs import CONFIGS, reduced
from paper_1904_10585_b200 import run


def main(quick=False):
    cases = [reduced(CONFIGS[1], iters=2),
             reduced(CONFIGS[2], n=520, iters=2, dtype="f64i8"),
             reduced(CONFIGS[3], n=700, iters=2, edge_prob=0.1, dtype="f64i8"),
             reduced(CONFIGS[3], n=650, p=16, d=4, iters=2, edge_prob=0.1),
             reduced(CONFIGS[4], n=600, p=128, d=3, iters=2),
             reduced(CONFIGS[5], n=1024, p=128, nbig=20, nrefl=8, d=4, iters=2),
             reduced(CONFIGS[5], n=1024, p=128, nbig=20, nrefl=8, d=4, iters=2, rr_ns=True)]
    if quick:
        cases = cases[1:3] + cases[5:6]
    for cfg in cases:
        out = run(cfg)
        torch.cuda.synchronize()
        print(cfg.name, cfg.n, cfg.p, cfg.dtype, "ok", out["status"]["names"], flush=True)


if __name__ == "__main__":
    main("quick" in sys.argv)
