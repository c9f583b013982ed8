"""Library comparison bar: cuBLAS ZGEMM / DGEMM throughput via torch.matmul (CUDA events)."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda:0")
for dt, name, fl in [(torch.complex128, "zgemm", 8), (torch.float64, "dgemm", 2)]:
    for n in (2048, 4096, 8192):
        a = torch.randn(n, n, dtype=dt, device=dev)
        b = torch.randn(n, n, dtype=dt, device=dev)
        c = torch.empty(n, n, dtype=dt, device=dev)
        for _ in range(3):
            torch.matmul(a, b, out=c)
        torch.cuda.synchronize()
        reps = 10 if n < 8192 else 4
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            torch.matmul(a, b, out=c)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"lib": name, "n": n, "ms": round(ms, 3), "tflops": round(fl * n**3 / ms / 1e9, 2)}))
        del a, b, c
