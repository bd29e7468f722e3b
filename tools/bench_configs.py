"""Per-config measurement of the fp64 path (BASELINE configs[0..3] = our configs 1-4), 1 GPU.
Not the bench line (bench.py measures the metric's workload, config 3); this records every
fp64 config's iterations/s, filter TFLOP/s and the Chebyshev-step GEMM's per-launch time for
profiles/.

  python tools/bench_configs.py [--configs 1 2 4] [--steps 20] [--warmup 3]

A step = one iteration of the config's mode (Lanczos refresh as scheduled, filter, CholeskyQR2,
Rayleigh-Ritz, spectral operator, update); configs 1's noise A <- A + E_k is host-generated and
is not in the timed region (its E_k are pre-uploaded and added between timed steps, the add timed
separately).  CUDA events on the launching stream; GEMM launches timed inside libpf (pf_profile).
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
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--graphs", type=int, default=1, help="1: replay the captured iteration body")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f64i8"])
    ap.add_argument("--slices", type=int, default=7)
    args = ap.parse_args()
    import numpy as np
    import torch
    from pfinputs import CONFIGS, cfg1_noise
    from paper_1904_10585_b200 import Solver
    from paper_1904_10585_b200.solver import _dev
    from paper_1904_10585_b200._lib import kernel_launches

    for cid in args.configs:
        cfg = CONFIGS[cid]
        if args.dtype != cfg.dtype:
            from pfinputs import reduced
            cfg = reduced(cfg, dtype=args.dtype)
        n, p, d = cfg.n, cfg.p, cfg.d
        t0 = time.time()
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            s = Solver(cfg, stream=stream, graphs=bool(args.graphs))
            if args.dtype == "f64i8":
                s.ctx.set_i8_slices(args.slices)
            sweep = cfg.mode in ("sweep_psd", "sweep_soft")
            noise = [_dev(cfg1_noise(cfg, k)) for k in range(args.warmup + args.steps)] \
                if sweep else None
            for k in range(args.warmup):
                s.step()
                if sweep:
                    s.perturb(noise[k])
            for k in range(s.k, s.k + args.steps):
                if k % cfg.lanczos_every == 0:
                    s.lanczos_vector(k)
        torch.cuda.synchronize()
        setup_s = time.time() - t0
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
        s.ctx.profile(True)
        l0 = kernel_launches()
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                ev[2 * i].record(stream)
                s.step()
                ev[2 * i + 1].record(stream)
                if sweep:
                    s.perturb(noise[args.warmup + i])
        torch.cuda.synchronize()
        launches = kernel_launches() - l0
        if s.graphs:       # replays launch the captured kernels without passing the host counter
            launches += args.steps * max(s.graph_launches.values())
        step_ms = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.steps)]
        gemm_ms, gemm_n = s.ctx.profile_read(stream)
        share = gemm_ms / sum(step_ms)
        if s.graphs:
            # the graphs were captured with profiling off: time the GEMM launches on a few eager
            # steps (same kernels), its share against those steps' own time
            s.graphs = False
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.ctx.profile_read(stream)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(5):
                    s.step()
                e1.record(stream)
            torch.cuda.synchronize()
            gemm_ms, gemm_n = s.ctx.profile_read(stream)
            share = gemm_ms / e0.elapsed_time(e1)
            s.graphs = True
        s.ctx.profile(False)
        st = s.ctx.status(stream)
        ms = float(np.mean(step_ms))
        gemm_avg = gemm_ms / max(gemm_n, 1)
        out = {
            "config": f"config {cid}: {cfg.name}, mode {cfg.mode}, n={n}, p={p}, d={d}, "
                      + ("fp64 DMMA" if args.dtype == "f64" else f"fp64 via int8 digits S={args.slices}")
                      + ", 1 GPU"
                      + (", CUDA-graph body" if s.graphs else ", eager launches"),
            "it_per_s": 1e3 / ms, "ms_per_step": ms,
            "ms_per_step_median": float(np.median(step_ms)),
            "filter_tflops_per_step_time": 2.0 * d * n * n * p / (ms / 1e3) / 1e12,
            "gemm_avg_ms": gemm_avg, "gemm_launches": gemm_n,
            "gemm_algorithmic_tflops": 2.0 * n * n * p / (gemm_avg / 1e3) / 1e12,
            "gemm_algorithmic_gbps": 8.0 * n * n / (gemm_avg / 1e3) / 1e9,
            "gemm_share_of_step": share,
            "kernel_launches_per_step": (launches - (args.steps if sweep else 0)) / args.steps,
            "rank_last": int(s.rank.item()), "status": st["names"], "rebases": st["rebases"],
            "setup_s": setup_s,
        }
        print(json.dumps(out), flush=True)
        del s
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
