"""Run the batched stream solve a few times (profiling target): python tools/solve_once.py N [reps]"""
import sys
import os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05466_b200 as zt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(8, n, n, dtype=torch.complex128, device="cuda", generator=g) / n
w = 0.5 * (a - a.conj().transpose(1, 2))
w -= torch.diagonal(w, dim1=1, dim2=2).mean(-1)[:, None, None] * torch.eye(n, device="cuda", dtype=torch.complex128)
op = zt.build_operator(n)
for _ in range(reps):
    p = zt.solve_stream_batched(w, op)
torch.cuda.synchronize()
print("ok", float(p.abs().sum()))
