"""Per-step device times of the bench loop (config 3, the bench's method and CUDA graphs), eager
vs graphs: python tools/step_times.py [steps] [graphs 0|1]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from pfinputs import bench_config, reduced, pfam_problem
from paper_1904_10585_b200 import Solver


def main(steps=24, graphs=1):
    cfg = reduced(bench_config(3), dtype="f64i8")
    prob = pfam_problem(cfg)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        s = Solver(cfg, problem=prob, stream=st, graphs=bool(graphs))
        for _ in range(3):
            s.step()
        for k in range(s.k, s.k + steps):
            if k % cfg.lanczos_every == 0:
                s.lanczos_vector(k)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    with torch.cuda.stream(st):
        ev[0].record(st)
        for i in range(steps):
            s.step()
            ev[i + 1].record(st)
    torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    print("graphs" if graphs else "eager", " ".join(f"{m:.3f}" for m in ms))
    print("mean", sum(ms) / steps)
    # re-base steps per iteration (span-exact Y R^-1 re-basing of the filter, reading R7)
    s.ctx.status(st)
    rb = []
    for _ in range(12):
        with torch.cuda.stream(st):
            s.step()
        rb.append(s.ctx.status(st)["rebases"])
    print("rebases per iteration (next 12):", rb)


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
