"""Quick device timings (CUDA events) of the three hot kernels + one step."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2206_05466_b200 as zt
from paper_2206_05466_b200 import integrator as I

dev = torch.device("cuda:0")


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def rand_skew(n, b=None, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    shape = (n, n) if b is None else (b, n, n)
    a = torch.randn(shape, dtype=torch.complex128, device=dev, generator=g) / n
    w = 0.5 * (a - a.conj().transpose(-1, -2))
    return w.contiguous()


for n in (1024, 2048, 4096):
    w = rand_skew(n, 8)
    op = zt.build_operator(n)
    ms = timeit(lambda: zt.solve_stream_batched(w, op))
    print(json.dumps({"op": "solve_b8", "n": n, "ms": round(ms, 4), "GBps_24N2": round(8 * 24 * n * n / ms / 1e6, 1)}))
    del w
for n in (2048, 4096):
    a = rand_skew(n, seed=1); b = rand_skew(n, seed=2); c = torch.empty_like(a)
    for algo in (0, 1):
        ms = timeit(lambda: I.zgemm(a, b, c, algo), reps=5)
        print(json.dumps({"op": "zgemm", "algo": ["3M", "4M"][algo], "n": n, "ms": round(ms, 3), "eff_tflops": round(8 * n**3 / ms / 1e9, 2)}))
    ms = timeit(lambda: torch.matmul(a, b, out=c), reps=5)
    print(json.dumps({"op": "zgemm_cublas", "n": n, "ms": round(ms, 3), "tflops": round(8 * n**3 / ms / 1e9, 2)}))
n = 2048
r = rand_skew(n, seed=0)
r = r - torch.diagonal(r).mean() * torch.eye(n, dtype=r.dtype, device=dev)
op = zt.build_operator(n)
w0 = zt.solve_stream(r)
w0 = w0 / torch.linalg.norm(w0)
x = w0.clone()
out = torch.empty_like(x)
its = []
def step():
    global x, out
    y, k, res, _ = I.midpoint_step_raw(x, 0.005, 1e-12, 10, op, out=out)
    its.append(k)
    x, out = y, x
ms = timeit(step, reps=10)
print(json.dumps({"op": "step", "n": n, "ms": round(ms, 3), "steps_per_s": round(1000 / ms, 2), "iters": its[-5:]}))
