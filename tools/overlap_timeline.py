"""Config-5 row-block split on ONE GPU through the loopback communicator (pf_create_loop): per
rank, the time of a Chebyshev-filter call (d GEMM steps, each gathering Y_j) with the slab-wise
overlapped gather (PF_OVERLAP=1) and with one all-gather before one GEMM (PF_OVERLAP=0), plus the
time of the gathers alone (the same copies, no GEMM).  python tools/overlap_timeline.py [n] [p] [W]
The W ranks share one GPU, so the absolute times are not W-GPU times; the comparison shows how
much of the gather the overlapped schedule hides behind the GEMM on each rank's stream."""
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1904_10585_b200._lib import Context, Loopback, PF_TF32


def one(n, p, W, d, overlap, reps=3):
    os.environ["PF_OVERLAP"] = "1" if overlap else "0"
    hub = Loopback(W)
    res = [None] * W

    def worker(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c = Context(n, p, d, rank=r, world=W, dtype=PF_TF32, loop=hub)
            nl = c.n_local
            g = torch.Generator(device="cuda").manual_seed(r)
            A = torch.randn((nl, n), dtype=torch.float32, device="cuda", generator=g) * 0.01
            U = torch.randn((p, nl), dtype=torch.float32, device="cuda", generator=g)
            iv = torch.tensor([-1.0, 1.0], dtype=torch.float64, device="cuda")
            c.orth(U, st)
            c.filter(A, U, iv, 1, 1e30, st)  # warm-up (rho_max huge: no re-base)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                c.filter(A, U, iv, 1, 1e30, st)
            e1.record(st)
            e1.synchronize()
            res[r] = {"filter_ms": e0.elapsed_time(e1) / reps}
            if overlap:
                c.profile(True)
                c.filter(A, U, iv, 1, 1e30, st)
                tl = c.overlap_timeline(st)
                c.profile(False)
                arr, beg, end = tl[:W], tl[W:2 * W], tl[2 * W:]
                # exposed: time a slab GEMM could not start because its slab had not landed
                exposed = sum(max(0.0, arr[s] - end[s - 1]) for s in range(1, W))
                res[r].update(last_step_ms=end[-1], arrival_ms=arr, gemm_begin_ms=beg,
                              gemm_end_ms=end, exposed_gather_ms=exposed)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(W)]
    [t.start() for t in th]
    [t.join() for t in th]
    return res


def main(n=32768, p=512, W=2, d=8):
    out = {"n": n, "p": p, "world": W, "d": d,
           "filter_ms_overlap": one(n, p, W, d, True),
           "filter_ms_single_gather": one(n, p, W, d, False)}
    print(json.dumps(out))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
