"""Experiment: does an issue-bound Ozaki pass (reconstruction / row
conversion) overlap with the tensor-bound residue GEMM when both run on
different streams?  Times each alone and both concurrently (N = 2048)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05466_b200 import _lib  # noqa: E402

lib = _lib.lib
dev = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
nm = lib.zt_oz_moduli(None, 0)
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randint(-44, 45, (nm, 2, n, n), dtype=torch.int8, device=dev, generator=g)
b = torch.randint(-44, 45, (nm, 2, n, n), dtype=torch.int8, device=dev, generator=g)
r = torch.empty(nm, 2, n, n, dtype=torch.int8, device=dev)
r2 = torch.randint(0, 89, (nm, 2, n, n), dtype=torch.uint8, device=dev, generator=g)
sh = torch.zeros(n, dtype=torch.int32, device=dev)
c = torch.empty(n, n, dtype=torch.complex128, device=dev)
x = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g)
planes = torch.empty(nm, 2, n, n, dtype=torch.int8, device=dev)
sh2 = torch.empty(n, dtype=torch.int32, device=dev)
kb = lib.zt_oz_bits(n)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def gemm(s):
    assert lib.zt_oz_modgemm(nm, n, n, n, a.data_ptr(), b.data_ptr(), r.data_ptr(), 0, s.cuda_stream) == 0


def recon(s):
    assert lib.zt_oz_reconstruct(n, n, r2.data_ptr(), sh.data_ptr(), sh.data_ptr(), ctypes.c_void_p(c.data_ptr()), n,
                                 None, 0, 0, None, 0, 0, ctypes.c_void_p(s.cuda_stream)) == 0


def conv(s):
    assert lib.zt_oz_convert_rows(n, n, ctypes.c_void_p(x.data_ptr()), n, 0, 0, kb, ctypes.c_void_p(planes.data_ptr()),
                                  ctypes.c_void_p(sh2.data_ptr()), None, ctypes.c_void_p(s.cuda_stream)) == 0


def timed(work, reps=10):
    for _ in range(2):
        work()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        work()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


out = {"N": n}
out["gemm"] = timed(lambda: gemm(s1))
out["recon_x4"] = timed(lambda: [recon(s2) for _ in range(4)])
out["conv_x3"] = timed(lambda: [conv(s2) for _ in range(3)])
out["gemm+recon_x4"] = timed(lambda: (gemm(s1), [recon(s2) for _ in range(4)]))
out["gemm+conv_x3"] = timed(lambda: (gemm(s1), [conv(s2) for _ in range(3)]))
print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in out.items()}))
