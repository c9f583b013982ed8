"""Op-level measurements for BASELINE configs 2 and 3 (device-resident,
CUDA events, L2 flushed between timed launches by a 256 MB write):

cfg 2  stream solve, batch of 8 random_admissible(N, default_rng(0), 1/N) draws,
       N in {1024, 2048, 4096}: time, algorithmic 24 N^2 B per matrix -> GB/s,
       fraction of MEASURED_PEAKS hbm_gbs; parity relF vs the CPU oracle (N=1024
       all 8, larger N first matrix).
cfg 3  commutator C = PW - WP (a = P W, C = a - a^H) and sandwich
       S = (I - hP/2) W (I + hP/2), h = 0.01, P then W drawn from
       random_admissible(N, default_rng(0), 1/N), N in {2048, 4096, 8192}:
       algorithmic 8 N^3 / 16 N^3 flop -> TF/s vs the measured DMMA peak;
       cuBLAS ZGEMM (torch.matmul) timed beside; parity vs numpy at N=2048.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200 import _lib  # noqa: E402
from oracle import zeitlin_oracle as zo  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)
try:
    HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    HBM = 6650.0
PEAK = max(json.loads(l)["tflops"] for l in open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.jsonl"))
           if '"dmma' in l)


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


def cfg2():
    for n in (1024, 2048, 4096):
        rng = np.random.default_rng(0)
        ws = [zo.random_admissible(n, rng, 1.0 / n) for _ in range(8)]
        w = torch.from_numpy(np.stack(ws)).to(dev)
        op = zt.build_operator(n)
        p = zt.solve_stream_batched(w, op)
        checks = range(8) if n == 1024 else range(1)
        err = max(np.linalg.norm(p[k].cpu().numpy() - zo.solve_stream(ws[k])) / np.linalg.norm(zo.solve_stream(ws[k]))
                  for k in checks)
        ms = timed(lambda: zt.solve_stream_batched(w, op))
        gbs = 8 * 24 * n * n / (ms * 1e-3) / 1e9
        print(json.dumps({"cfg": 2, "op": "stream_solve_batch8", "N": n, "ms": round(ms, 4), "GBps_alg": round(gbs, 1),
                          "frac_hbm": round(gbs / HBM, 3), "relF_vs_oracle": err}), flush=True)
        del w, p


def cfg3():
    h = 0.01
    for n in (2048, 4096, 8192):
        rng = np.random.default_rng(0)
        pn = zo.random_admissible(n, rng, 1.0 / n)
        wn = zo.random_admissible(n, rng, 1.0 / n)
        P, W = torch.from_numpy(pn).to(dev), torch.from_numpy(wn).to(dev)
        C = torch.empty_like(P); S = torch.empty_like(P); work = torch.empty_like(P)
        s = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
        com = lambda: _lib.check(_lib.lib.zt_commutator(n, P.data_ptr(), W.data_ptr(), C.data_ptr(), work.data_ptr(), s()))  # noqa: E731
        sand = lambda: _lib.check(_lib.lib.zt_sandwich(n, P.data_ptr(), W.data_ptr(), h, S.data_ptr(), work.data_ptr(), s()))  # noqa: E731
        com(); sand(); torch.cuda.synchronize()
        rec = {}
        if n == 2048:
            a = pn @ wn
            cref = a - a.conj().T
            sref = wn - 0.5 * h * (a - a.conj().T) - 0.25 * h * h * (a @ pn)
            rec["relF_commutator"] = float(np.linalg.norm(C.cpu().numpy() - cref) / np.linalg.norm(cref))
            rec["relF_sandwich"] = float(np.linalg.norm(S.cpu().numpy() - sref) / np.linalg.norm(sref))
        reps = 5 if n < 8192 else 2
        mc = timed(com, reps, 2)
        msw = timed(sand, reps, 2)
        mcb = timed(lambda: torch.matmul(P, W, out=work), reps, 2)
        print(json.dumps({"cfg": 3, "N": n, "commutator_ms": round(mc, 3),
                          "commutator_TFs_alg": round(8 * n**3 / mc / 1e9, 2),
                          "sandwich_ms": round(msw, 3), "sandwich_TFs_alg": round(16 * n**3 / msw / 1e9, 2),
                          "frac_dmma_peak_sandwich": round(16 * n**3 / msw / 1e9 / PEAK, 3),
                          "cublas_zgemm_ms": round(mcb, 3), "cublas_TFs": round(8 * n**3 / mcb / 1e9, 2),
                          "dmma_peak_TFs": PEAK, **rec}), flush=True)
        del P, W, C, S, work


if __name__ == "__main__":
    which = sys.argv[1:] or ["2", "3"]
    if "2" in which:
        cfg2()
    if "3" in which:
        cfg3()
