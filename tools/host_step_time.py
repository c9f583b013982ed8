"""Where the time goes in the host-result step: device step alone, step +
one full D2H copy, and the progressive host step (zt_midpoint_step_host)."""
import sys, os, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200.integrator import midpoint_step_raw  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
r = 0.5 * (a - a.conj().T); r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
op = zt.build_operator(n, dev)
w = zt.solve_stream(r, op); w /= torch.linalg.norm(w)
host = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
out = torch.empty_like(w)


def run(mode, K=20):
    for _ in range(3):
        midpoint_step_raw(w, 0.005, 1e-12, 10, op, out=out, host_out=host if mode == "prog" else None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        if mode == "prog":
            midpoint_step_raw(w, 0.005, 1e-12, 10, op, out=out, host_out=host)
        else:
            midpoint_step_raw(w, 0.005, 1e-12, 10, op, out=out)
            if mode == "copy":
                host.copy_(out, non_blocking=True)
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / K * 1e3


for mode in ("device", "copy", "prog", "device", "prog"):
    print(f"{mode:7s} {run(mode):.3f} ms/step", flush=True)
