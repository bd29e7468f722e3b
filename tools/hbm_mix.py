"""HBM bandwidth by traffic mix on this B200 (CUDA events, best of 10): write-only (fill), read-only
(sum), copy (read + write 1:1).  The PFAM update is ~23% reads / 77% writes; its roofline
denominator is the measured copy bandwidth (MEASURED_PEAKS.json), this shows where write-heavy
traffic actually saturates.  python tools/hbm_mix.py"""
import torch


def best(fn, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


n = 1 << 29  # 4 GiB of fp64
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
a.fill_(1.0)
b.fill_(2.0)
torch.cuda.synchronize()
gb = n * 8 / 1e9
t = best(lambda: a.fill_(3.0))
print(f"write-only (fill): {gb / t * 1e3:.0f} GB/s")
t = best(lambda: a.sum())
print(f"read-only (sum):   {gb / t * 1e3:.0f} GB/s")
t = best(lambda: b.copy_(a))
print(f"copy (r+w):        {2 * gb / t * 1e3:.0f} GB/s")
