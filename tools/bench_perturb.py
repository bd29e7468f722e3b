import sys, torch
sys.path.insert(0, '/root/repo')
from paper_1904_10585_b200._lib import Context, PF_TF32
n = 16384
ctx = Context(n, 64, 4, dtype=PF_TF32)
A = torch.zeros((n, n), dtype=torch.float32, device="cuda")
ctx.perturb_hash(A, 0, 1, 1e-3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(5):
    ctx.perturb_hash(A, 0, k, 1e-3)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"perturb n={n}: {ms:.3f} ms, {8.0*n*n/ms/1e6:.0f} GB/s")
