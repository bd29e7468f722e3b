"""Config 5 measurement (BASELINE configs[4]): fp32 storage, TF32 tcgen05 filter, n = 65536,
p = 512, d in {4, 8, 16}, 1 GPU.  Not the bench line (bench.py measures the metric's workload,
config 3); this records the TF32 path's numbers for profiles/.

  python tools/bench_cfg5.py [--n 65536] [--p 512] [--d 4 8 16] [--steps 3] [--passes 3]

A step = filter (d TF32 GEMM passes + re-bases + CholeskyQR2) + Rayleigh-Ritz (one more GEMM
pass, Gram, 512 x 512 Jacobi) + spectral operator, on the resident fp32 iterate; the workload
noise A <- fl32(A + E_k) between steps is timed separately.  CUDA events on the
launching stream; the Chebyshev-step GEMM is timed per launch inside libpf (pf_profile).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--p", type=int, default=512)
    ap.add_argument("--d", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--ns", type=int, default=1,
                    help="1: Rayleigh-Ritz spectral operator by Newton-Schulz (pf_rr_ns, R26)")
    ap.add_argument("--passes", type=int, default=0,
                    help="uniform TF32 passes (1..3); 0 = the config's schedule (reading R18)")
    args = ap.parse_args()
    import numpy as np
    import torch
    from pfinputs import CONFIGS, reduced, cfg5_problem
    from paper_1904_10585_b200 import Solver
    from paper_1904_10585_b200._lib import kernel_launches

    t0 = time.time()
    base = reduced(CONFIGS[5], n=args.n, p=args.p)
    A0 = cfg5_problem(base)
    gen_s = time.time() - t0
    stream = torch.cuda.Stream()
    Adev = None
    for d in args.d:
        cfg = reduced(base, d=d, rr_ns=bool(args.ns))
        with torch.cuda.stream(stream):
            if Adev is None:
                buf = torch.empty((cfg.n, (cfg.n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
                buf[:, :cfg.n].copy_(torch.from_numpy(A0))
                Adev = buf[:, :cfg.n]
            A = Adev.clone() if False else Adev
            s = Solver(cfg, problem={"_dev": {"A0": A}}, stream=stream)
            if args.passes:
                s.ctx.set_tf32_passes(args.passes)
            s.step()                      # k = 0: Lanczos + warm-up sweeps (untimed)
            s.perturb_hash(0)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4 * args.steps)]
        s.ctx.profile(True)
        l0 = kernel_launches()
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                e[4 * i].record(stream)
                s.step()
                e[4 * i + 1].record(stream)
                e[4 * i + 2].record(stream)
                s.perturb_hash(s.k)
                e[4 * i + 3].record(stream)
        torch.cuda.synchronize()
        launches = kernel_launches() - l0
        step_ms = [e[4 * i].elapsed_time(e[4 * i + 1]) for i in range(args.steps)]
        pert_ms = [e[4 * i + 2].elapsed_time(e[4 * i + 3]) for i in range(args.steps)]
        gemm_ms, gemm_n = s.ctx.profile_read(stream)
        s.ctx.profile(False)
        diag = s.ctx.diagnostics(stream)
        st = s.ctx.status(stream)
        n, p = cfg.n, cfg.p
        ms = float(np.mean(step_ms))
        gemm_avg = gemm_ms / max(gemm_n, 1)
        flops_pass = 2.0 * n * n * p
        rank = int(s.rank.item())
        out = {
            "config": f"config 5 sweep, n={n}, p={p}, d={d}, fp32 storage, tcgen05 TF32 filter "
                      + (f"{args.passes}xTF32 every pass" if args.passes else
                         f"schedule: {cfg.tf32_early}xTF32 steps 1..{d - cfg.tf32_tail}, "
                         f"3xTF32 last {cfg.tf32_tail} steps + RR") +
                      (", RR spectral operator by Newton-Schulz" if args.ns else ", RR by Jacobi")
                      + ", 1 GPU",
            "ns_iters_last": int(s.ns_it.item()) if args.ns else None,
            "it_per_s": 1e3 / ms, "ms_per_step": ms, "step_ms": step_ms,
            "filter_tflops": 2.0 * d * n * n * p / (ms / 1e3) / 1e12,
            "gemm_avg_ms": gemm_avg, "gemm_launches": gemm_n,
            "gemm_algorithmic_tflops": flops_pass / (gemm_avg / 1e3) / 1e12,
            "gemm_passes_per_step": None if not args.passes else args.passes,
            "gemm_share_of_step": gemm_ms / sum(step_ms),
            "perturb_ms": float(np.mean(pert_ms)),
            "perturb_gbps": 2 * 4.0 * n * n / (np.mean(pert_ms) / 1e3) / 1e9,
            "kernel_launches_per_step": launches / args.steps,
            "jacobi_sweeps_last": diag["jacobi_sweeps"], "rank_last": rank,
            "status": st["names"], "rebases": st["rebases"],
            "host_generation_s": gen_s,
        }
        print(json.dumps(out), flush=True)
        del s
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
