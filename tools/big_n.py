import sys, time, torch, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2206_05466_b200 as zt
from paper_2206_05466_b200.integrator import midpoint_step_raw
n = int(sys.argv[1])
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
w = 0.5 * (a - a.conj().T); del a
w -= torch.trace(w) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
p = zt.solve_stream(w, op)
back = zt.apply_laplacian(p, op=op)
print("roundtrip", float((back - w).norm() / w.norm()))
w = p / torch.linalg.norm(p); del p, back
c0 = zt.casimirs(w, 3)
torch.cuda.synchronize(); t0 = time.perf_counter()
out, k, r, _ = midpoint_step_raw(w, 0.0025, 1e-12, 10, op)
torch.cuda.synchronize(); t1 = time.perf_counter()
out2, k2, r2, _ = midpoint_step_raw(out, 0.0025, 1e-12, 10, op)
torch.cuda.synchronize(); t2 = time.perf_counter()
c1 = zt.casimirs(out2, 3)
print(f"N={n} iters={k},{k2} step1 {t1-t0:.3f}s step2 {t2-t1:.3f}s C2 drift {abs(c1[1]-c0[1])/abs(c0[1]):.2e} C3 drift {abs(c1[2]-c0[2])/abs(c0[2]):.2e} skew {zt.skewness_residual(out2):.2e} mem {torch.cuda.max_memory_allocated()/1e9:.1f} GB")
