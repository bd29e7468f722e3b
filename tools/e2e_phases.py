"""Phase times of the bench's end-to-end solve (bench.run_e2e's structure): solver construction
from pinned host data, k = 0 (Lanczos + warm-up sweeps), the two graph-capturing iterations, and
the steady graph replays.  Development tool: python tools/e2e_phases.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from pfinputs import bench_config, initial_block, pfam_problem
    from paper_1904_10585_b200 import Solver
    from paper_1904_10585_b200._lib import Context, PF_FP64_I8
    cfg = bench_config(3)
    cfg = type(cfg)(**{**cfg.__dict__, "dtype": "f64i8"})
    prob = pfam_problem(cfg)
    host = {"adj_bits": torch.from_numpy(prob["adj_bits"].view(np.int32)).pin_memory(),
            "deg": torch.from_numpy(prob["deg"]).pin_memory(),
            "U0": torch.from_numpy(initial_block(cfg)).pin_memory()}
    ctx = Context(cfg.n, cfg.p, cfg.d, dtype=PF_FP64_I8)
    st = torch.cuda.Stream()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    with torch.cuda.stream(st):
        ev[0].record(st)
        dev = {k: v.cuda(non_blocking=True) for k, v in host.items()}
        s = Solver(cfg, problem={"adj_bits": None, "deg": None, "t": cfg.t, "_dev": dev},
                   stream=st, graphs=True, ctx=ctx)
        ev[1].record(st)
        s.step()                      # k = 0
        ev[2].record(st)
        s.step()                      # k = 1: capture graph A
        s.step()                      # k = 2: capture graph B
        ev[3].record(st)
        for _ in range(20):
            s.step()
        ev[4].record(st)
    torch.cuda.synchronize()
    names = ["setup", "k=0", "k=1,2 (captures)", "20 replays"]
    for i, nm in enumerate(names):
        print(f"{nm:18s} {ev[i].elapsed_time(ev[i + 1]):8.2f} ms")


if __name__ == "__main__":
    main()
