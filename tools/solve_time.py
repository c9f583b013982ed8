"""Time the batched stream solve (batch 8, L2 flushed) for the library at
ZT_LIB_PATH; prints one line per N.  Experiment helper."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05466_b200 as zt  # noqa: E402

HBM = 6552.0
flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
out = []
for n in [int(x) for x in (sys.argv[1:] or ["1024", "2048", "4096"])]:
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(8, n, n, dtype=torch.complex128, device="cuda", generator=g) / n
    w = 0.5 * (a - a.conj().transpose(1, 2))
    del a
    w -= torch.diagonal(w, dim1=1, dim2=2).mean(-1)[:, None, None] * torch.eye(n, device="cuda", dtype=torch.complex128)
    op = zt.build_operator(n)
    p = zt.solve_stream_batched(w, op)
    ref = torch.load(f"/tmp/ref_{n}.pt") if os.path.exists(f"/tmp/ref_{n}.pt") else None
    if ref is None:
        torch.save(p, f"/tmp/ref_{n}.pt")
        err = 0.0
    else:
        err = float((p - ref).norm() / ref.norm())
    ts = []
    for _ in range(15):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        zt.solve_stream_batched(w, op)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts)[2:-2]
    ms = sum(ts) / len(ts)
    out.append(f"N={n} {ms*1e3:7.1f}us {8*24*n*n/ms/1e6/HBM:.3f} relF_vs_first={err:.1e}")
    del w, p
print(os.environ.get("ZT_LIB_PATH", "default"), " | ".join(out))
