"""PFSVT measurement (NEXT-3): the matrix completion runs of tab:SVT-MKL on one
GPU to the SVT stopping rule, d = 1.  Reports iterations, recovered rank, mse, seconds to
convergence (problem generation excluded), ms per iteration, and the CSR filter product's
per-launch time with its gathered bytes (nnz x p x 8 from L2) and streamed bytes (nnz x 12).

  python tools/bench_svt.py [--cases svt1k svt5k svt10k]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", nargs="+", default=["svt1k", "svt5k", "svt10k"])
    ap.add_argument("--adapt", type=int, default=0,
                    help="1: NEXT-2 adaptive block size (p_k from svp_{k-1} + 5, reading R27)")
    args = ap.parse_args()
    import numpy as np
    import torch
    from pfinputs import NEXT_CONFIGS, svt_problem
    from paper_1904_10585_b200 import SVTSolver

    for name in args.cases:
        cfg = NEXT_CONFIGS[name]
        if args.adapt:
            from pfinputs import reduced
            cfg = reduced(cfg, svt_adapt=True)
        t0 = time.time()
        prob = svt_problem(cfg)
        gen_s = time.time() - t0
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            s = SVTSolver(cfg, prob, stream=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 0
        with torch.cuda.stream(st):
            e0.record(st)
            while it < cfg.iters:
                s.step()
                it += 1
                if s.residual() <= cfg.svt_tol:     # host read per iteration (the stop rule)
                    break
            e1.record(st)
        torch.cuda.synchronize()
        total_ms = e0.elapsed_time(e1)
        # one CSR filter product timed alone
        ptr, col, x = s.row_ptr, s.col, s.x
        p_final = s.p
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        out = torch.empty_like(s.Q)                 # the filter's own buffers live in libpf now
        with torch.cuda.stream(st):
            for _ in range(3):
                s.ctx.spmm(ptr, col, x, s.Q, out, stream=st)
            ev[0].record(st)
            for _ in range(20):
                s.ctx.spmm(ptr, col, x, s.Q, out, stream=st)
            ev[1].record(st)
        torch.cuda.synchronize()
        spmm_ms = ev[0].elapsed_time(ev[1]) / 20
        nnz = int(prob["b"].size)
        U, sv, V = s.factors()
        M = prob["ML"] @ prob["MR"].T
        mse = float(np.linalg.norm((U * sv) @ V.T - M) / np.linalg.norm(M))
        print(json.dumps({
            "case": f"{name}: m=n={cfg.n}, SR={cfg.sr}, r={cfg.r}, p={cfg.p}, d={cfg.d}, nnz={nnz}"
                    + (", adaptive p (R27)" if args.adapt else ""),
            "p_final": p_final,
            "iters": it, "svp": int(s.svp.item()), "res": s.residual(), "mse": mse,
            "seconds_to_converge": total_ms / 1e3, "ms_per_iter": total_ms / it,
            "spmm_ms": spmm_ms,
            "spmm_gather_gbps": nnz * p_final * 8 / spmm_ms / 1e6,
            "spmm_stream_gbps": nnz * 12 / spmm_ms / 1e6,
            "host_generation_s": gen_s}), flush=True)
        del s
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
