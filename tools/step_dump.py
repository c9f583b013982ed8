"""Experiment helper: run S steps of the cfg-4 workload from the seeded W0 and
save W_S (to compare library variants bitwise): python tools/step_dump.py OUT.npy [N] [S]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200.integrator import midpoint_step_raw  # noqa: E402

out = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
r = 0.5 * (a - a.conj().T)
r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
w = zt.solve_stream(r, op)
w /= torch.linalg.norm(w)
nxt = torch.empty_like(w)
for _ in range(steps):
    nxt, k, res, _ = midpoint_step_raw(w, 0.005, 1e-12, 10, op, out=nxt)
    w, nxt = nxt, w
np.save(out, w.cpu().numpy())
