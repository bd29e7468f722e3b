import os, time, json, subprocess, torch
print("cores", len(os.sched_getaffinity(0)), os.cpu_count())
print(subprocess.run(["nvidia-smi","--query-gpu=name,clocks.sm,clocks.max.sm,power.limit","--format=csv"],capture_output=True,text=True).stdout)
dev = torch.device("cuda:0")
for n, p in [(16384, 64), (4096, 32), (32768, 128), (16384, 16)]:
    A = torch.randn(n, n, dtype=torch.float64, device=dev); Y = torch.randn(n, p, dtype=torch.float64, device=dev)
    for _ in range(3): Z = A @ Y
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): Z = A @ Y
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cuBLAS DGEMM n={n} p={p}: {ms:.3f} ms  {2*n*n*p/ms/1e9:.2f} TFLOP/s  {8*n*n/ms/1e6:.0f} GB/s")
    del A
n = 8192
A = torch.randn(n, n, dtype=torch.float64, device=dev)
for _ in range(2): Z = A @ A
torch.cuda.synchronize(); t = time.time()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): Z = A @ A
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"cuBLAS DGEMM square 8192: {2*n**3/ms/1e9:.2f} TFLOP/s")
import numpy as np
a = np.random.rand(4096, 4096); b = np.random.rand(4096, 64)
t = time.time(); 
for _ in range(5): c = a @ b
print("host numpy GEMV-ish 4096x4096x64 GFLOP/s", 5*2*4096*4096*64/(time.time()-t)/1e9)
a = np.random.rand(4096, 4096)
t = time.time(); c = a @ a; print("host numpy 4096^3 GFLOP/s", 2*4096**3/(time.time()-t)/1e9)
