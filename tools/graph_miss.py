import sys, time, torch
sys.path.insert(0, "/root/repo")
import paper_2206_05466_b200 as zt
from paper_2206_05466_b200.integrator import midpoint_step_raw
n = 2048
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
r = 0.5 * (a - a.conj().T); r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
w = zt.solve_stream(r, op); w /= torch.linalg.norm(w)
bufs = [torch.empty_like(w) for _ in range(12)]
for i in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    midpoint_step_raw(w, 0.005, 1e-12, 10, op, out=bufs[i])
    torch.cuda.synchronize(); t1 = time.perf_counter()
    midpoint_step_raw(w, 0.005, 1e-12, 10, op, out=bufs[i])
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"miss {1e3*(t1-t0):.2f} ms  hit {1e3*(t2-t1):.2f} ms")
