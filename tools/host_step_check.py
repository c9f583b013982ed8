"""zt_midpoint_step_host (progressive final update + overlapped block copies)
against zt_midpoint_step: W_{n+1} on the host and on the device bitwise equal
to the plain step, over several steps and sizes."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200.integrator import midpoint_step_raw  # noqa: E402

dev = torch.device("cuda:0")
for n in [int(a) for a in sys.argv[1:]] or [2048, 1000, 130, 64, 5]:
    g = torch.Generator(device=dev).manual_seed(n)
    a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
    r = 0.5 * (a - a.conj().T); r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
    op = zt.build_operator(n, dev)
    w = zt.solve_stream(r, op); w /= torch.linalg.norm(w)
    host = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
    x1 = w.clone(); x2 = w.clone()
    worst = 0.0
    for step in range(4):
        y1, k1, r1, _ = midpoint_step_raw(x1, 0.005, 1e-12, 10, op)
        y2, k2, r2, _ = midpoint_step_raw(x2, 0.005, 1e-12, 10, op, host_out=host)
        torch.cuda.synchronize()
        dh = float((host.to(dev) - y1).abs().max())
        dd = float((y2 - y1).abs().max())
        worst = max(worst, dh, dd)
        if dh or dd:
            bad = ((y2 - y1).abs() > 0).nonzero()
            badh = ((host.to(dev) - y1).abs() > 0).nonzero()
            print(f"  step {step}: dd={dd} dh={dh} nbad_dev={bad.shape[0]} nbad_host={badh.shape[0]} "
                  f"rows {bad[:, 0].min().item() if bad.numel() else -1}..{bad[:, 0].max().item() if bad.numel() else -1} "
                  f"cols {bad[:, 1].min().item() if bad.numel() else -1}..{bad[:, 1].max().item() if bad.numel() else -1} "
                  f"first {bad[:4].tolist()}", flush=True)
        assert (k1, r1) == (k2, r2), (n, step, k1, k2, r1, r2)
        x1, x2 = y1, y2
    print(f"N={n} host/device max|diff| vs plain step = {worst}", flush=True)
