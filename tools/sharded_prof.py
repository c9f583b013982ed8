"""Profiling target: a few one-rank sharded steps in eager or graph mode
(python tools/sharded_prof.py N eager|graph steps)."""
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05466_b200 import solve_stream  # noqa: E402
from paper_2206_05466_b200.sharded import DeviceBackend, PeerShardedStepper  # noqa: E402

n = int(sys.argv[1])
mode = sys.argv[2]
steps = int(sys.argv[3])
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
w = solve_stream(r, be.op)
w /= torch.linalg.norm(w)
st = PeerShardedStepper(n, be, graph=(mode == "graph"))
for _ in range(2):
    w, k, _ = st.midpoint_step(w, 0.005)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(steps):
    w, k, _ = st.midpoint_step(w, 0.005)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
dist.destroy_process_group()
