import json, sys
import torch
sys.path.insert(0, ".")
import paper_2206_05466_b200 as zt
from paper_2206_05466_b200 import integrator as I
dev = torch.device("cuda:0")
def timeit(fn, reps=5, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for n in (2048, 4096):
    a = torch.randn(n, n, dtype=torch.complex128, device=dev); b = torch.randn(n, n, dtype=torch.complex128, device=dev)
    c = torch.empty_like(a)
    for algo, name in ((0, "3M"), (1, "4M")):
        ms = timeit(lambda: I.zgemm(a, b, c, algo))
        dm = {0: 6, 1: 8}[algo]
        print(json.dumps({"n": n, "algo": name, "ms": round(ms, 3), "eff_tf": round(8 * n**3 / ms / 1e9, 2), "dmma_tf": round(dm * n**3 / ms / 1e9, 2)}))
