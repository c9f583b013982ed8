"""One-rank symmetric-memory sharded step: the device-driven graph path vs the
eager peer path vs the single-GPU step (parity and ms per step).  Experiment
helper: python tools/sharded_graph_check.py [N] [steps]"""
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05466_b200.integrator import midpoint_step_raw  # noqa: E402
from paper_2206_05466_b200.sharded import DeviceBackend, PeerShardedStepper  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda:0")
s = socket.socket()
s.bind(("127.0.0.1", 0))
os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
s.close()
dist.init_process_group("nccl", device_id=dev)
be = DeviceBackend(n, dev)
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g) / n
r = 0.5 * (a - a.conj().T)
r -= torch.trace(r) / n * torch.eye(n, device=dev, dtype=torch.complex128)
from paper_2206_05466_b200 import solve_stream  # noqa: E402
w0 = solve_stream(r, be.op)
w0 /= torch.linalg.norm(w0)
h = 0.005


def run(step, w, k):
    its = []
    for _ in range(k):
        w, it = step(w)
        its.append(it)
    return [w], its


def single(w):
    o, k, _, _ = midpoint_step_raw(w, h, 1e-12, 10, be.op)
    return o, k


res = {}
for name, mk in [("single", None), ("eager", False), ("graph", True)]:
    if mk is None:
        fn = single
    else:
        stp = PeerShardedStepper(n, be, graph=mk)
        fn = (lambda st: (lambda w: (lambda o: (o[0], o[1]))(st.midpoint_step(w, h))))(stp)
    run(fn, w0, 3)  # warm-up (graph capture)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    outs, its = run(fn, w0, steps)
    e1.record()
    torch.cuda.synchronize()
    res[name] = (outs[-1], its, e0.elapsed_time(e1) / steps)
ref = res["single"][0]
for name, (o, its, ms) in res.items():
    err = float((o - ref).norm() / ref.norm())
    print(f"N={n} {name:6s} ms/step={ms:.3f} steps/s={1e3 / ms:.1f} iters={sorted(set(its))} relF_vs_single={err:.2e}"
          f" bitwise_vs_eager={bool(torch.equal(o, res['eager'][0])) if 'eager' in res else None}")
dist.destroy_process_group()
