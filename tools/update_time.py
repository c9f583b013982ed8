"""Time one fused update (solve + planes + k_zupdate) by running midpoint
steps with tol = 1e300 (one fixed-point iteration + the final update = 2
updates per step).  Experiment helper for kernel variants."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200.integrator import midpoint_step_raw  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
w = 0.5 * (a - a.conj().T)
w -= torch.trace(w) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
out = torch.empty_like(w)
for _ in range(3):
    midpoint_step_raw(w, 0.005, 1e300, 10, op, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    midpoint_step_raw(w, 0.005, 1e300, 10, op, out=out)
e1.record()
torch.cuda.synchronize()
print(os.environ.get("TAG", ""), f"N={n} ms/update={e0.elapsed_time(e1) / 40:.4f}")
