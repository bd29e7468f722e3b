"""bench.py -- PFAM iterations/s and poly-filter TFLOP/s on config 3 (n = 16384, p = 64, d = 8).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3]

A step is one whole iteration of the hot path: interval (Lanczos
refresh every 10 iterations, as it falls), Chebyshev filter (d fp64 DMMA GEMM passes),
CholeskyQR2, Rayleigh-Ritz (one more GEMM pass + Jacobi), spectral operator, and the fused
rank-p rebuild + PFAM update of the 2 GiB iterate.  Inputs are synthetic and
larger than L2 (the iterate is 2 GiB), so no L2 flush is needed between steps.

N > 1 (torchrun): configs 1-3 do not shard: every rank runs an independent
replica (seed + rank), value = sum of per-rank throughput over the max-over-ranks time.
`--impl reference` times the CPU oracle (oracle/) on the host cores on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "poly-filter TFLOP/s and PFPG/PFAM iterations/s at n=16384, 1/2/4/8 B200"
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


def peaks() -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            try:
                sm, mx, pw, rs = [x.strip() for x in line.split(",")]
                self.samples.append((float(sm), float(mx), float(pw), int(rs, 16)))
            except Exception:
                pass

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        s = self.samples
        if not s:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [x for x in s if x[2] > 200] or s
        bits = 0
        for x in loaded:
            bits |= x[3]
        return {"sm_mhz": statistics.median(x[0] for x in loaded),
                "sm_max_mhz": max(x[1] for x in s),
                "power_w_max": max(x[2] for x in s),
                "samples": len(s),
                "reasons": [v for k, v in REASONS.items() if bits & k and k != 0x1]}


def bench_cfg(cfg_id: int):
    from pfinputs import bench_config
    return bench_config(cfg_id)


# ============================================================================ our arm
def run_ours(args, rank: int, world: int, local_rank: int) -> dict | None:
    import torch
    import torch.distributed as dist
    from pfinputs import reduced
    from paper_1904_10585_b200 import Solver
    from paper_1904_10585_b200._lib import kernel_launches

    torch.cuda.set_device(local_rank)
    cfg = bench_cfg(args.config)
    if world > 1:
        cfg = reduced(cfg, seed=cfg.seed + rank)          # independent replica per rank
    if args.path == "i8":
        cfg = reduced(cfg, dtype="f64i8")                 # fp64 via exact int8 products (K1-i8)
    n, p, d = cfg.n, cfg.p, cfg.d
    stream = torch.cuda.Stream()
    from pfinputs import pfam_problem
    prob = pfam_problem(cfg)                              # host data, shared with the DMMA leg
    with torch.cuda.stream(stream):
        # iterations k >= 1 replay a captured CUDA graph of the iteration body (both buffer
        # parities are captured during the warm-up, W >= 3)
        s = Solver(cfg, problem=prob, stream=stream, graphs=True)
        for _ in range(max(3, args.warmup)):
            s.step()
        # pre-stage the Lanczos start vectors the timed steps will use (host->device, untimed)
        for k in range(s.k, s.k + args.steps):
            if k % cfg.lanczos_every == 0:
                s.lanczos_vector(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = kernel_launches()
    r0 = s.replayed_launches
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            s.step()
        e1.record(stream)
    torch.cuda.synchronize()
    launches = kernel_launches() - l0 + s.replayed_launches - r0
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    # per-launch time of the dominant kernel: the graphs hold no profiling events, so a few eager
    # steps (the same kernels) run with pf_profile on, after the timed region
    s.graphs = False
    s.ctx.profile(True)
    ep0, ep1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        ep0.record(stream)
        for _ in range(5):
            s.step()
        ep1.record(stream)
    torch.cuda.synchronize()
    gemm_ms, gemm_n = s.ctx.profile_read(stream)
    upd_ms, upd_n = s.ctx.profile_read_update(stream)
    gemm_share = gemm_ms / ep0.elapsed_time(ep1)
    upd_share = upd_ms / ep0.elapsed_time(ep1)
    s.ctx.profile(False)
    s.graphs = True
    status = s.ctx.status(stream)
    obj = s.objective()

    # ---------------------------------------------------------------- end to end
    e2e = run_e2e(cfg, args, stream)
    # the same workload on the fp64 DMMA filter GEMM (PF_FP64), for comparison
    dmma = run_dmma(cfg, prob, args, stream) if args.path == "i8" else None

    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    if rank != 0:
        return None
    per_step_ms = ms_max / args.steps
    value = world * args.steps / (ms_max / 1e3)
    flops_gemm = 2.0 * n * n * p                      # algorithmic flops of one Chebyshev step
    gemm_avg_ms = gemm_ms / max(gemm_n, 1)
    achieved = flops_gemm / (gemm_avg_ms / 1e3) / 1e12
    pk = peaks()
    fp64_peak = pk.get("fp64_dmma_tflops")
    peak_src = "MEASURED_PEAKS.json fp64_dmma_tflops"
    if fp64_peak is None:
        fp64_peak = 37.1
        peak_src = "measured on this pool by tools/probe/peaks.cu (profiles/r01_probe_peaks.log): " \
                   "fp64 DMMA m16n8k4 37.1 TF/s at 1965 MHz; MEASURED_PEAKS.json has no fp64 entry"
    traffic = None
    tfile = "i8_gemm_traffic.json" if args.path == "i8" else "gemm_traffic.json"
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", tfile)))
        if tr.get("n") == n and tr.get("p") == p:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    if args.path == "i8":
        # K1-i8: S = 7 digit slices, S (S + 1) / 2 = 28 exact int8 slice products per Chebyshev
        # step; peak = measured dense bf16 x 2 (int8 : bf16 = 2 : 1 nominal, B200_PROFILING.md)
        S = 7
        ops = 2.0 * n * n * p * S * (S + 1) / 2
        i8_peak = 2.0 * pk.get("bf16_tflops", 1618.6)
        kname = ("cheb_gemm_i8_kernel<7,64> (tcgen05 kind::i8" if os.environ.get("PF_I8PAIR") == "0"
                 else "cheb_gemm_i8p_kernel (CTA pairs, tcgen05.mma.cta_group::2 kind::i8, M = 256")
        roof = {"bound": "tensor", "kernel": kname + ", exact digit products, fp64 level "
                "combination)",
                "achieved": ops / (gemm_avg_ms / 1e3) / 1e12, "peak": i8_peak, "unit": "TOPS",
                "frac": ops / (gemm_avg_ms / 1e3) / 1e12 / i8_peak, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json bf16_tflops x 2 (nominal int8:bf16); the "
                               "burst int8 rate measured by tools/probe/mma_i8_rate.cu is "
                               "16372 ops/clk/SM = 4.76 POPS at 1965 MHz",
                "algorithmic_per_launch": {"int8_ops": ops, "fp64_flops": flops_gemm,
                                           "bytes": 7.0 * n * n},
                "hbm_frac": 7.0 * n * n / (gemm_avg_ms / 1e3) / 1e9 / pk.get("hbm_gbs", 6550.4),
                "fp64_equivalent_tflops": achieved,
                "fp64_equivalent_vs_dmma_peak": achieved / fp64_peak,
                "avg_launch_ms": gemm_avg_ms, "launches": gemm_n, "share_of_step": gemm_share}
    else:
        roof = {"bound": "tensor", "kernel": "cheb_gemm_kernel<64> (fp64 DMMA)",
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": traffic,
                "peak_source": peak_src,
                "algorithmic_per_launch": {"flops": flops_gemm, "bytes": 8.0 * n * n},
                "avg_launch_ms": gemm_avg_ms, "launches": gemm_n,
                "share_of_step": gemm_share}
    # the PFAM update (pf_admm_step, HBM-bound): Z_old upper triangle read, Z_new written in full,
    # the digit slices of Z_new (fused, i8 path), V and V' rows, the upper adjacency bits
    upd_roof = None
    if upd_n:
        fused = args.path == "i8" and os.environ.get("PF_FUSE_DIGITS", "1") != "0"
        k7i8 = fused and p == 64 and os.environ.get("PF_K7I8", "1") != "0"
        # Z_new written in full, or (upper-block storage, pf_set_z_upper) on and above the
        # 128 x 128 diagonal blocks only
        zup = bool(getattr(s, "z_upper", False))
        zw = 8.0 * n * (n + 128) / 2 if zup else 8.0 * n * n
        # digit slices of Z_new: every tile, or (the filter reads the lower tiles as the stored
        # upper ones transposed: PF_I8T / PF_I8SYM) the upper tiles and the
        # 256 x 256 diagonal super-blocks only
        half = k7i8 and world == 1 and (os.environ.get("PF_I8T", "1") != "0" or
                                        os.environ.get("PF_I8SYM") == "1")
        dw = (7.0 * n * (n + 256) / 2 if half else 7.0 * n * n) if fused else 0.0
        ubytes = 8.0 * n * (n + 1) / 2 + zw + dw + 2 * 8.0 * n * p + n * n / 16.0
        uavg = upd_ms / upd_n
        utraffic = None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "update_traffic.json")))
            if tr.get("n") == n and tr.get("p") == p and tr.get("kernel_i8") == k7i8:
                utraffic = tr["dram_bytes_per_launch"]
        except Exception:
            pass
        upd_roof = {"bound": "hbm",
                    "kernel": ("rebuild_i8_kernel (W from tcgen05 kind::i8 digit products, "
                               "TMA-staged update)") if k7i8 else "rebuild_kernel<P> (fp64 DMMA)",
                    "achieved": ubytes / (uavg / 1e3) / 1e9, "peak": pk.get("hbm_gbs", 6550.4),
                    "unit": "GB/s",
                    "frac": ubytes / (uavg / 1e3) / 1e9 / pk.get("hbm_gbs", 6550.4),
                    "traffic": utraffic, "algorithmic_bytes_per_launch": ubytes,
                    "avg_launch_ms": uavg, "launches": upd_n, "share_of_step": upd_share,
                    "z_storage": "upper blocks (pf_set_z_upper)" if zup else "full",
                    "digit_tiles": "upper tiles + diagonal super-blocks (K1-i8p reads the rest "
                                   "transposed)" if half else "all",
                    "timed": "events around pf_admm_step (row bounds + splits + update kernel)"}
    filter_flops_per_step = 2.0 * d * n * n * p
    cpu = cpu_baseline(cfg, args) if (world == 1 and not args.no_cpu) else None
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "it/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": per_step_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 (int8-digit emulation, S=7)" if args.path == "i8" else "f64",
        "data": "synthetic (BASELINE configs[2] recipe, DESIGN.md §3)",
        "config": {"workload": f"config 3: PFAM max-cut SDP, n={n}, p={p}, d={d}, G(n,{cfg.edge_prob})",
                   "n": n, "p": p, "d": d, "lanczos_every": cfg.lanczos_every,
                   "rayleigh_ritz": "matrix form: F = P_+(H) = H when H is positive definite "
                                    "(Cholesky test), else Newton-Schulz / Jacobi; update "
                                    "W = Q F Q^T (DESIGN.md R30)" if cfg.rr_ns else
                                    "Jacobi eigendecomposition",
                   "lambda_min": (f"warm-started {cfg.lanczos_warm}-step Lanczos refresh every "
                                  f"{cfg.lanczos_every} iterations (R29)") if cfg.lanczos_warm
                                 else f"{cfg.lanczos_steps}-step seeded Lanczos (R5)",
                   "filter_gemm": "fp64 from exact int8 tensor-core products of 7-bit digit "
                                  "slices (PF_FP64_I8, S=7)" if args.path == "i8" else
                                  "fp64 DMMA (PF_FP64)",
                   "iterate_storage": ("symmetric Z in upper-block storage: the update writes Z_new "
                                       "on and above the 128 x 128 diagonal blocks (every reader on "
                                       "this path reads only those), plus all digit slices "
                                       "(pf_set_z_upper)") if getattr(s, "z_upper", False)
                                      else "full symmetric Z",
                   "cuda_graphs": "iteration body replayed (k >= 1)",
                   "l2": "inputs larger than L2 (2 GiB fp64 iterate re-read every pass)",
                   "parallelism": "replicas" if world > 1 else "1 GPU"},
        "filter_tflops": world * filter_flops_per_step * args.steps / (ms_max / 1e3) / 1e12,
        "roofline": roof,
        "update_roofline": upd_roof,
        "clocks": clk,
        "gpu_launches": launches,
        "e2e": e2e,
        "device_status": status["names"],
        "objective_last": obj,
    }
    if dmma is not None:
        out["fp64_dmma_path"] = dmma
    if cpu is not None:
        out["cpu_baseline"] = cpu
    return out


def run_dmma(cfg, prob, args, stream) -> dict:
    """The same timed loop on the fp64 DMMA filter GEMM (dtype PF_FP64), same problem data."""
    import torch
    from pfinputs import reduced
    from paper_1904_10585_b200 import Solver
    c64 = reduced(cfg, dtype="f64")
    with torch.cuda.stream(stream):
        s = Solver(c64, problem=prob, stream=stream, graphs=True)
        for _ in range(max(3, args.warmup)):
            s.step()
        for k in range(s.k, s.k + args.steps):
            if k % c64.lanczos_every == 0:
                s.lanczos_vector(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            s.step()
        e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # its dominant kernel against the fp64 DMMA peak (eager profiled steps, as for the main arm)
    s.graphs = False
    s.ctx.profile(True)
    with torch.cuda.stream(stream):
        for _ in range(3):
            s.step()
    torch.cuda.synchronize()
    gms, gn = s.ctx.profile_read(stream)
    s.ctx.profile(False)
    g_avg = gms / max(gn, 1)
    tflops = 2.0 * c64.n * c64.n * c64.p / (g_avg / 1e3) / 1e12
    pk = peaks().get("fp64_dmma_tflops", 37.1)
    out = {"value": args.steps / (ms / 1e3), "unit": "it/s", "ms_per_step": ms / args.steps,
           "what": "same workload and timing, filter GEMM on fp64 DMMA (PF_FP64)",
           "roofline": {"bound": "tensor", "kernel": "cheb_gemm_kernel<64> (fp64 DMMA)",
                        "achieved": tflops, "peak": pk, "unit": "TFLOP/s", "frac": tflops / pk,
                        "avg_launch_ms": g_avg,
                        "peak_source": "fp64 DMMA m16n8k4 measured on this pool "
                                       "(profiles/r01_probe_peaks.log)"}}
    del s
    torch.cuda.empty_cache()
    return out


def run_e2e(cfg, args, stream) -> dict:
    """End to end through the public API from host-resident problem data:
    pinned H2D of the graph bitmask, degrees and U0 + (W + K) iterations with a D2H read of the
    objective every iteration + D2H of the final factors (V, f); it/s over K counted steps.
    The context (the library's scratch, like a BLAS handle) is created before the timed region;
    everything that depends on the problem -- upload, solver state, graph capture -- is inside."""
    import numpy as np
    import torch
    from pfinputs import initial_block, lanczos_start, pfam_problem
    from paper_1904_10585_b200 import Solver
    prob = pfam_problem(cfg)
    host = {"adj_bits": torch.from_numpy(prob["adj_bits"].view(np.int32)).pin_memory(),
            "deg": torch.from_numpy(prob["deg"]).pin_memory(),
            "U0": torch.from_numpy(initial_block(cfg)).pin_memory()}
    # the configured job: config 3 is a 100-iteration solve (BASELINE.json configs[2]), so the
    # fixed costs of a solve (k = 0 with its warm-up sweeps and 20-step Lanczos, graph capture,
    # uploads) are spread over the job's own length, not over the bench's timed-step count
    K = max(args.steps + args.warmup, cfg.iters)
    # seeded Lanczos start vectors the run uses (only k = 0 when refreshes are warm-started, R29)
    v0 = {k: torch.from_numpy(lanczos_start(cfg, k)).pin_memory()
          for k in range(K) if k % cfg.lanczos_every == 0 and (k == 0 or cfg.lanczos_warm <= 0)}
    obj_host = torch.empty((K, 2), dtype=torch.float64).pin_memory()
    from paper_1904_10585_b200._lib import Context, PF_FP64, PF_FP64_I8
    ctx = Context(cfg.n, cfg.p, cfg.d, dtype=PF_FP64_I8 if cfg.dtype == "f64i8" else PF_FP64)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    h2d = d2h = 0
    with torch.cuda.stream(stream):
        e0.record(stream)
        dev = {k: v.cuda(non_blocking=True) for k, v in host.items()}
        h2d += sum(v.numel() * v.element_size() for v in host.values())
        s = Solver(cfg, problem={"adj_bits": None, "deg": None, "t": cfg.t, "_dev": dev},
                   stream=stream, graphs=True, ctx=ctx)
        for k in range(K):
            if k in v0:
                s._v0[k] = v0[k].cuda(non_blocking=True)
                h2d += v0[k].numel() * 8
            s.step()
            obj_host[k].copy_(s.obj, non_blocking=True)
            d2h += 16
        Vh = s.ritz.to("cpu", non_blocking=True)
        # the factors of X_k: (V, f), or (Q, F) for the matrix-form Rayleigh-Ritz (R30)
        fh = (s.F if s.last_ns else s.f).to("cpu", non_blocking=True)
        d2h += Vh.numel() * 8 + fh.numel() * 8
        e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return {"value": K / (ms / 1e3),
            "unit": "it/s", "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": d2h / K,
            "iterations": K, "ms_total": ms,
            "what": "the configured solve (cfg.iters iterations, at least warmup + steps) from "
                    "host data on a pre-created context: H2D problem + U0, solver state, every "
                    "iteration (graph capture included), per-iteration objective D2H, final "
                    "factors D2H"}


# ============================================================================ CPU oracle
def cpu_baseline(cfg, args, budget_iters: int = 3) -> dict:
    """The oracle as it stands (oracle.run) on the host cores: iterations 1..budget_iters of
    the same config after its k = 0 iteration; setup (problem, dense C) untimed."""
    import numpy as np
    import oracle
    stamps = []
    t0 = [None]

    def prog(rec):
        stamps.append(time.perf_counter())

    t_start = time.perf_counter()
    oracle.run(cfg, iters=budget_iters + 1, record_factors=False, progress=prog)
    per = (stamps[-1] - stamps[0]) / budget_iters
    cores = len(os.sched_getaffinity(0))
    return {"value": 1.0 / per, "unit": "it/s", "cores": cores, "kind": "oracle",
            "sample": f"config 3 full size, oracle iterations k=1..{budget_iters} (k=0 and "
                      f"setup untimed); numpy/OpenBLAS fp64 on {cores} host threads",
            "wall_s": time.perf_counter() - t_start}


def run_reference(args, rank: int, world: int) -> dict | None:
    if rank != 0:
        return None
    cfg = bench_cfg(args.config)
    K = max(1, min(args.steps, 3))
    import oracle
    stamps = []
    oracle.run(cfg, iters=K + 1, record_factors=False,
               progress=lambda rec: stamps.append(time.perf_counter()))
    per = (stamps[-1] - stamps[0]) / K
    cores = len(os.sched_getaffinity(0))
    v = 1.0 / per
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "it/s", "n_gpus": world,
            "steps": K, "warmup": 1, "ms_per_step": per * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE configs[2] recipe)",
            "config": {"workload": f"config 3: PFAM max-cut SDP, n={cfg.n}, p={cfg.p}, d={cfg.d}"},
            "cpu_baseline": {"value": v, "unit": "it/s", "cores": cores, "kind": "oracle",
                             "sample": f"oracle iterations k=1..{K} of config 3 (k=0 untimed)"},
            "e2e": {"value": v, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--path", default="i8", choices=["i8", "dmma"],
                    help="filter GEMM: fp64 via exact int8 products (default) or fp64 DMMA")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        out = run_ours(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
