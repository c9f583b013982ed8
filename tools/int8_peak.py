"""Measured INT8 tensor-core peak on this B200 (the roofline denominator for
the Ozaki-II residue GEMM): cuBLASLt int8 GEMM (torch._int_mm) at 8192^3,
best of 10 (burst) and back to back for ~4 s (sustained), with the SM clock
sampled under load.  One JSON line."""
import json, subprocess, threading, time
import torch

dev = torch.device("cuda:0")
n = 8192
a = torch.randint(-64, 64, (n, n), dtype=torch.int8, device=dev)
b = torch.randint(-64, 64, (n, n), dtype=torch.int8, device=dev)
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
clk = []
stop = False


def sample():
    while not stop:
        try:
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                                 capture_output=True, text=True, timeout=5).stdout.strip()
            clk.append(float(out.splitlines()[0]))
        except Exception:
            pass
        time.sleep(0.2)


th = threading.Thread(target=sample); th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time(); it = 0
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        torch._int_mm(a, b)
    it += 20
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
stop = True; th.join()
ms = e0.elapsed_time(e1) / it
ops = 2.0 * n ** 3
print(json.dumps({"what": "cuBLASLt int8 GEMM (torch._int_mm) 8192^3", "burst_tops": ops / best / 1e9,
                  "sustained_tops": ops / ms / 1e9, "sm_mhz_samples": sorted(clk)[len(clk) // 2] if clk else None}))
