"""Per-phase timing of the config-3 iteration (CUDA events around each C-ABI call) and the
Jacobi sweep counts; development diagnostics, not the bench."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from pfinputs import CONFIGS, reduced
from paper_1904_10585_b200 import Solver


def main(cfg_id=3, iters=14, **over):
    cfg = CONFIGS[cfg_id]
    if over:
        cfg = reduced(cfg, **over)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        s = Solver(cfg, stream=st)
    ctx = s.ctx
    names = ["lanczos", "interval", "filter", "rr", "spectral", "update"]
    for k in range(iters):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        with torch.cuda.stream(st):
            ev[0].record(st)
            if k == 0 or (s.psd and k % cfg.lanczos_every == 0):
                if cfg.lanczos_warm > 0 and k > 0:
                    ctx.lanczos(s.A, None, cfg.lanczos_warm, s.lohi, st)
                else:
                    ctx.lanczos(s.A, s.lanczos_vector(k), cfg.lanczos_steps, s.lohi, st)
            ev[1].record(st)
            if s.psd:
                ctx.interval_psd(s.lohi, cfg.eta, s.interval, st)
            else:
                ctx.interval_soft(s.thr, cfg.eta, s.interval, st)
            ev[2].record(st)
            for _ in range(cfg.warmup if k == 0 else 1):
                ctx.filter(s.A, s.U, s.interval, 1, cfg.rho_max, st)
            ev[3].record(st)
            if cfg.rr_ns:   # matrix-form spectral operator (R26 / R30), update W = Q F Q^T
                if s.F is None:
                    s.F = torch.empty((cfg.p, cfg.p), dtype=torch.float64, device="cuda")
                    s.ns_it = torch.zeros(1, dtype=torch.int32, device="cuda")
                ctx.rr_ns(s.A, s.U, s.op, s.thr, s.F, s.rank, s.ns_it, st)
                ev[4].record(st)
                ev[5].record(st)
                if cfg.mode == "pfam":
                    ctx.admm_step_f(s.U, s.F, cfg.t, s.adj, s.deg, s.A, s.obj, st)
                ev[6].record(st)
                s.k += 1
                torch.cuda.synchronize()
                ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(names))]
                print(f"k={k:3d} " + " ".join(f"{n}={m:7.3f}" for n, m in zip(names, ms)) +
                      f" total={sum(ms):7.3f} ms  ns_iters={int(s.ns_it.item())} rank={int(s.rank.item())}",
                      flush=True)
                continue
            ctx.rayleigh_ritz(s.A, s.U, s.V, s.theta, st)
            ev[4].record(st)
            ctx.spectral_op(s.op, s.thr, s.theta, s.f, s.rank, st)
            ev[5].record(st)
            if cfg.mode == "pfpg":
                ctx.prox_step(s.V, s.f, cfg.tau, s.mu, s.omega, s.W, s.A, s.obj, st)
            elif cfg.mode == "pfam":
                ctx.admm_step(s.V, s.f, cfg.t, s.adj, s.deg, s.A, s.obj, st)
            ev[6].record(st)
            s.ritz = s.V
            s.U, s.V = s.V, s.U
            s.k += 1
        torch.cuda.synchronize()
        dg = ctx.diagnostics(st)
        ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(names))]
        print(f"k={k:3d} " + " ".join(f"{n}={m:7.3f}" for n, m in zip(names, ms)) +
              f" total={sum(ms):7.3f} ms  jacobi_sweeps={dg['jacobi_sweeps']} rank={int(s.rank.item())}",
              flush=True)


if __name__ == "__main__":
    # diag_step.py <cfg> <iters> [dtype]  (dtype f64i8 = the bench's int8-digit filter)
    # diag_step.py <cfg> <iters> [dtype] [field=value ...] (Config overrides, e.g. lanczos_warm=8)
    kw = {"dtype": sys.argv[3]} if len(sys.argv) > 3 else {}
    for a in sys.argv[4:]:
        k, v = a.split("=")
        kw[k] = type(getattr(CONFIGS[int(sys.argv[1])], k))(v)
    main(*[int(a) for a in sys.argv[1:3]], **kw)
