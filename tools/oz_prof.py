"""One zt_oz_zgemm at N (profiling target)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05466_b200 import _lib  # noqa: E402
lib = _lib.lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
A = torch.from_numpy(rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).to(dev)
B = torch.from_numpy(rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).to(dev)
C = torch.zeros_like(A)
ws = torch.empty(lib.zt_oz_workspace_bytes(n), dtype=torch.uint8, device=dev)
for _ in range(2):
    rc = lib.zt_oz_zgemm(n, A.data_ptr(), n, B.data_ptr(), n, mode, C.data_ptr(), n, 0, ws.data_ptr(), ws.numel(),
                    torch.cuda.current_stream().cuda_stream)
    assert rc == 0, (rc, lib.zt_last_error())
torch.cuda.synchronize()
print("ok")
