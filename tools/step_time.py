"""Device time per midpoint step at the cfg-4 workload (N=2048 default) through
the C ABI, plus iteration counts; experiment helper (env switches apply)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200.integrator import midpoint_step_raw  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
h = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
r = 0.5 * (a - a.conj().T)
r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
w = zt.solve_stream(r, op)
w /= torch.linalg.norm(w)
nxt = torch.empty_like(w)
for _ in range(3):
    nxt, k, res, _ = midpoint_step_raw(w, h, 1e-12, 10, op, out=nxt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
its = []
cur, spare = w, nxt
e0.record()
for _ in range(steps):
    out, k, res, _ = midpoint_step_raw(cur, h, 1e-12, 10, op, out=spare)
    its.append(k)
    cur, spare = out, cur
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
print(f"{os.environ.get('TAG', '')} N={n} ms/step={ms:.3f} steps/s={1e3 / ms:.2f} iters={sorted(set(its))} "
      f"|W|={float(torch.linalg.norm(cur)):.15f}")
