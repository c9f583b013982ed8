"""Per-kernel CUDA-event averages (solve / full fused update / final update)
over cfg-4 steps, via the library's profiling slots; experiment helper for
kernel variants (ZT_LIB_PATH)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200 import _lib  # noqa: E402
from paper_2206_05466_b200.integrator import midpoint_step_raw  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
r = 0.5 * (a - a.conj().T)
r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
w = zt.solve_stream(r, op)
w /= torch.linalg.norm(w)
out = torch.empty_like(w)
lib = _lib.lib
def step(x, out):
    try:
        return midpoint_step_raw(x, 0.005, 1e-12, 10, op, out=out)[0]
    except zt.FixedPointError:  # timing-only kernel variants
        return out


for _ in range(3):
    step(w, out)
torch.cuda.synchronize()
lib.zt_profile_read(None, None, 1)
lib.zt_profile_enable(1)
x = w
for _ in range(steps):
    y = step(x, out)
    x, out = y, x
torch.cuda.synchronize()
lib.zt_profile_enable(0)
pms = (ctypes.c_double * 3)()
pcnt = (ctypes.c_int64 * 3)()
lib.zt_profile_read(ctypes.cast(pms, ctypes.c_void_p), ctypes.cast(pcnt, ctypes.c_void_p), 1)
avg = [pms[i] / max(1, pcnt[i]) for i in range(3)]
print(f"{os.environ.get('TAG', '')} N={n} solve={avg[0]*1e3:.1f}us full={avg[1]:.4f}ms final={avg[2]:.4f}ms "
      f"counts={list(pcnt)}")
