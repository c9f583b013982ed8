"""Time zt_oz_modgemm (all moduli, full and lower-tile modes) with CUDA
events, and the whole complex product zt_oz_zgemm.

ops = 2 * 2 * nmod * N^3 int8 ops per full residue product (two real
products U, V per modulus); `equiv_TF` = the 8 N^3 algorithmic FP64 flop of
one complex product over the measured time.

usage: python tools/oz_modgemm_time.py [N ...]   (default 2048 4096)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05466_b200 import _lib  # noqa: E402

lib = _lib.lib
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
nm = lib.zt_oz_moduli(None, 0)


def timed(fn, k=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


for n in [int(a) for a in sys.argv[1:]] or [2048, 4096]:
    g = torch.Generator(device=dev).manual_seed(0)
    a = torch.randint(-44, 45, (nm, 2, n, n), dtype=torch.int8, device=dev, generator=g)
    b = torch.randint(-44, 45, (nm, 2, n, n), dtype=torch.int8, device=dev, generator=g)
    r = torch.empty(nm, 2, n, n, dtype=torch.int8, device=dev)
    out = {"N": n, "nmod": nm}
    for lower in (0, 1):
        us = timed(lambda: lib.zt_oz_modgemm(nm, n, n, n, a.data_ptr(), b.data_ptr(), r.data_ptr(), lower,
                                              st.cuda_stream))
        mt = n // 256
        frac = 1.0 if not lower else (mt * (mt + 1) / 2) / (mt * mt)
        ops = 2.0 * 2 * nm * n * n * n * frac
        key = "lower" if lower else "full"
        out[f"{key}_us"] = round(us, 1)
        out[f"{key}_TOPS"] = round(ops / us / 1e6, 1)
    del a, b, r
    x = torch.randn(n, n, dtype=torch.complex128, device=dev)
    y = torch.randn(n, n, dtype=torch.complex128, device=dev)
    c = torch.empty_like(x)
    ws = torch.empty(lib.zt_oz_workspace_bytes(n), dtype=torch.uint8, device=dev)
    us = timed(lambda: lib.zt_oz_zgemm(n, x.data_ptr(), n, y.data_ptr(), n, 0, c.data_ptr(), n, 0, ws.data_ptr(),
                                        ws.numel(), st.cuda_stream))
    out["zgemm_us"] = round(us, 1)
    out["zgemm_equiv_TF"] = round(8.0 * n**3 / us / 1e6, 1)
    print(json.dumps(out), flush=True)
