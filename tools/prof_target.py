"""Small fixed workload for ncu captures: solve (batch 8) and both GEMM
algorithms at N=2048, a few launches each."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_05466_b200 as zt
from paper_2206_05466_b200 import integrator as I

what = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda:0")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(8, n, n, dtype=torch.complex128, device=dev, generator=g) / n
w = (0.5 * (a - a.conj().transpose(-1, -2))).contiguous()
op = zt.build_operator(n)
if what in ("all", "solve"):
    for _ in range(3):
        zt.solve_stream_batched(w, op)
if what in ("all", "gemm"):
    x, y = w[0].contiguous(), w[1].contiguous()
    c = torch.empty_like(x)
    for algo in (0, 1):
        for _ in range(2):
            I.zgemm(x, y, c, algo)
torch.cuda.synchronize()
print("done")
