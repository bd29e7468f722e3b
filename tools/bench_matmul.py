"""Times the filter GEMM alone through pf_matmul (out = A Y, fp64 dtypes) on a symmetric Gaussian
A: per-launch kernel time (pf_profile events around the GEMM launch) and the whole call (digit
split of Y included; the split of A is done once, as in an iteration).  Development tool.

  python tools/bench_matmul.py [--n 16384] [--p 64] [--slices 7] [--reps 20]   (--slices 0: DMMA)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--p", type=int, default=64)
    ap.add_argument("--slices", type=int, nargs="+", default=[7, 6, 0])
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_1904_10585_b200._lib import Context, PF_FP64_I8

    n, p = args.n, args.p
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    A = A + A.T
    Y = torch.randn((n, p), dtype=torch.float64, device="cuda", generator=g)
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    c = Context(n, p, 4, dtype=PF_FP64_I8)
    for S in args.slices:
        c.set_i8_slices(S)
        with torch.cuda.stream(st):
            c.matmul(A, Y, out, st)                      # split A (once), warm up
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(st)
            c.invalidate()
            c.matmul(A, Y, out, st)                      # A split + Y split + GEMM
            e1.record(st)
            c.profile(True)
            for _ in range(args.reps):
                c.matmul(A, Y, out, st)
            e2.record(st)
        torch.cuda.synchronize()
        gemm_ms, launches = c.profile_read(st)
        c.profile(False)
        k_ms = gemm_ms / launches
        call_ms = e1.elapsed_time(e2) / args.reps
        split_ms = e0.elapsed_time(e1) - call_ms
        print(json.dumps({
            "n": n, "p": p, "path": "int8 digits S=%d" % S if S else "fp64 DMMA",
            "gemm_ms": k_ms, "gemm_fp64_equiv_tflops": 2.0 * n * n * p / k_ms / 1e9,
            "a_bytes_per_pass": (S if S else 8) * n * n,
            "a_gbps": (S if S else 8) * n * n / k_ms / 1e6,
            "call_ms": call_ms, "a_split_ms": split_ms}), flush=True)


if __name__ == "__main__":
    main()
