import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_10585_b200 import Context
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = torch.randn(n, n, dtype=torch.float64, device="cuda"); A = A + A.T
ctx = Context(n, 64, 8)
v0 = torch.randn(n, dtype=torch.float64, device="cuda")
lohi = torch.zeros(2, dtype=torch.float64, device="cuda")
for _ in range(2):
    ctx.lanczos(A, v0, 20, lohi)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    ctx.lanczos(A, v0, 20, lohi)
e1.record(); torch.cuda.synchronize()
print(f"lanczos n={n}: {e0.elapsed_time(e1)/3:.3f} ms per 20-step refresh", lohi.cpu().numpy())
