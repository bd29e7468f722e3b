"""Accuracy / speed of TF32 precision schedules (reading R18) on config 5: full-size k = 0
against the closed form Q soft(Lambda) Q^T, a reduced p = 512 trajectory against the oracle, and
the full-size step time.  Development evidence for the default schedule; not a test."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
from pfinputs import (CONFIGS, reduced, cfg5_problem, cfg5_spectrum, cfg5_reflectors,
                      cfg5_basis_columns)
from paper_1904_10585_b200 import Solver, run

SCHED = [tuple(int(x) for x in a.split(',')) for a in sys.argv[1:]] or [(3, 0), (1, 2)]


def reduced_errs(early, tail, ref):
    cfg = reduced(CONFIGS[5], n=4096, p=512, nbig=200, nrefl=32, iters=3, tf32_early=early,
                  tf32_tail=tail)
    got = run(cfg)["records"]
    return [O.lowrank_diff_fro(g["V"], g["f"], r["V"], r["f"]) / O.lowrank_fro(r["V"], r["f"])
            for g, r in zip(got, ref)]


def main():
    ref = O.run(reduced(CONFIGS[5], n=4096, p=512, nbig=200, nrefl=32, iters=3))["records"]
    base = reduced(CONFIGS[5], iters=4)
    A0 = cfg5_problem(base)
    lam = cfg5_spectrum(base)
    Vh, T = cfg5_reflectors(base)
    big = np.where(np.abs(lam) > base.theta)[0]
    fex = np.sign(lam[big]) * (np.abs(lam[big]) - base.theta)
    Qb = cfg5_basis_columns(Vh, T, big)
    den = O.lowrank_fro(Qb, fex)
    buf = torch.empty((base.n, base.n), dtype=torch.float32, device="cuda")
    for early, tail in SCHED:
        cfg = reduced(base, tf32_early=early, tf32_tail=tail)
        buf.copy_(torch.from_numpy(A0))
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            s = Solver(cfg, problem={"_dev": {"A0": buf}}, stream=st)
            s.step()
        torch.cuda.synchronize()
        f = s.f.cpu().numpy()
        keep = f != 0
        err0 = O.lowrank_diff_fro(s.ritz_factors()[:, keep], f[keep], Qb, fex) / den
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(2):
                s.step()
            e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 2
        red = reduced_errs(early, tail, ref)
        print(json.dumps({"early_passes": early, "exact_tail": tail, "fullsize_k0_err": err0,
                          "reduced_p512_errs": red, "ms_per_step_d8": ms}), flush=True)
        del s
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
