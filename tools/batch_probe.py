import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2510_03421_b200 as P
from paper_2510_03421_b200 import workloads as W
A = W.c1()
for i in range(3): P.glynn_batch(A)
t = time.perf_counter(); 
for i in range(10): P.glynn_batch(A)
print("host batch 64x12x12", (time.perf_counter()-t)/10*1e3, "ms")
dA = torch.tensor(A, device='cuda')
for i in range(3): P.glynn_batch(dA)
torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record(); 
for i in range(10): P.glynn_batch(dA)
e1.record(); torch.cuda.synchronize(); print("device batch 64x12x12", e0.elapsed_time(e1)/10, "ms")
for n in (8, 10, 12):
    B = np.random.default_rng(0).uniform(-1,1,(100000, n, n))
    dB = torch.tensor(B, device='cuda'); P.glynn_batch(dB); torch.cuda.synchronize()
    e0.record(); 
    for i in range(5): P.glynn_batch(dB)
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/5
    print(f"device batch 1e5 x {n}x{n}", ms, "ms", 1e5*2**(n-1)*2*n/(ms*1e-3)/1e12, "Tops")
for name, A in (("c2a", W.c2a()), ("c2b", W.c2b())):
    dA = torch.tensor(A, device='cuda'); P.opt_batch(dA); torch.cuda.synchronize()
    e0.record()
    for i in range(10): P.opt_batch(dA)
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/10
    print(f"device opt_batch {name} 1e6: {ms:.4f} ms  {1e6/(ms*1e-3):.3e} matrices/s  {A.nbytes/(ms*1e-3)/1e9:.0f} GB/s")
    ts = []
    for _ in range(3):
        t = time.perf_counter(); P.opt_batch(A); ts.append(time.perf_counter() - t)
    print(f"host opt_batch {name}: " + ", ".join(f"{x*1e3:.1f}" for x in ts) + " ms")
