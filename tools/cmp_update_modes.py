"""Run 5 cfg-4-recipe steps and save (W, [(iterations, residual)]) -- run once
with ZT_SEP_UPDATE=0 and once without to check the two update paths agree
bitwise: python tools/cmp_update_modes.py N out.pt"""
import sys, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2206_05466_b200 as zt
from paper_2206_05466_b200.integrator import midpoint_step_raw
n = int(sys.argv[1]); dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
r = 0.5 * (a - a.conj().T); r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
w = zt.solve_stream(r, op); w /= torch.linalg.norm(w)
its = []
for _ in range(5):
    w, k, res, _ = midpoint_step_raw(w, 0.005, 1e-12, 10, op)
    its.append((k, res))
torch.save((w.cpu(), its), sys.argv[2])
