"""Time zt_oz_modgemm (all moduli, full and lower-tile modes) for the
single-CTA and the CTA-pair residue-GEMM kernels with CUDA events.

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
for n in [int(a) for a in sys.argv[1:]] or [2048, 4096]:
    g = torch.Generator(device=dev).manual_seed(0)
    a = torch.randint(-60, 61, (nm, 3, n, n), dtype=torch.int8, device=dev, generator=g)
    b = torch.randint(-60, 61, (nm, 2, n, n), dtype=torch.int8, device=dev, generator=g)
    r = torch.empty(nm, 2, n, n, dtype=torch.int8, device=dev)
    out = {"N": n}
    ref = {}
    for cta in (1, 2):
        assert lib.zt_oz_set_cta(cta) == 0
        for lower in (0, 1):
            for _ in range(3):
                assert lib.zt_oz_modgemm(nm, n, n, n, a.data_ptr(), b.data_ptr(), r.data_ptr(), lower,
                                         st.cuda_stream) == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k = 10
            e0.record()
            for _ in range(k):
                lib.zt_oz_modgemm(nm, n, n, n, a.data_ptr(), b.data_ptr(), r.data_ptr(), lower, st.cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / k * 1e3
            ops = 2.0 * 4 * nm * n * n * n * (1.0 if not lower else 0.5625)
            out[f"cta{cta}_{'lower' if lower else 'full'}_us"] = round(us, 1)
            out[f"cta{cta}_{'lower' if lower else 'full'}_TOPS"] = round(ops / us / 1e6, 1)
            if lower:
                m = (torch.arange(n, device=dev)[:, None] // 128) >= (torch.arange(n, device=dev)[None, :] // 128)
                cur = r[:, :, m].clone()
            else:
                cur = r.clone()
            if (lower, ) in ref:
                out[f"same_{'lower' if lower else 'full'}"] = bool(torch.equal(ref[(lower, )], cur))
            else:
                ref[(lower, )] = cur
    lib.zt_oz_set_cta(0)
    print(json.dumps(out), flush=True)
