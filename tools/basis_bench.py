"""Spectral basis on the device: compute_basis,
extract and project times at N in {512, 1024, 2048} (CUDA events), bytes
moved vs HBM, and the CPU restatement of compute_basis / extract (scipy
LAPACK per block, numpy GEMVs; the reference's algorithm) timed beside at
N <= 1024.  One JSON line per N."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2206_05466_b200 import basis as B  # noqa: E402
from oracle import zeitlin_oracle as zo  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6552.0) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6552.0


def ev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in [int(x) for x in (sys.argv[1:] or ["512", "1024", "2048"])]:
    rec = {"op": "basis", "N": n}
    b = B.compute_basis(n)
    vbytes = 8.0 * b.data.numel()
    rec["basis_GB"] = vbytes / 1e9
    rec["compute_basis_ms"] = ev_time(lambda: B.compute_basis(n, align_oracle=False), 2)
    w = torch.from_numpy(zo.random_admissible(n, np.random.default_rng(1), 1.0 / n)).cuda()
    rec["extract_ms"] = ev_time(lambda: B.extract_packed(w, b))
    rec["extract_GBps"] = vbytes / (rec["extract_ms"] * 1e-3) / 1e9
    rec["extract_frac_hbm"] = rec["extract_GBps"] / HBM
    pos, neg = B.extract_packed(w, b)
    rec["project_ms"] = ev_time(lambda: B.project_packed(pos, None, b))
    rec["project_GBps"] = vbytes / (rec["project_ms"] * 1e-3) / 1e9
    back = B.project_packed(pos, None, b)
    rec["roundtrip_max_abs_err"] = float((back - w).abs().max() / w.abs().max())
    if n <= 1024:
        t0 = time.perf_counter()
        vecs = zo.basis_vectors(n)
        rec["cpu_compute_basis_s"] = time.perf_counter() - t0
        wn = w.cpu().numpy()
        t0 = time.perf_counter()
        zo.extract(wn, vecs)
        rec["cpu_extract_s"] = time.perf_counter() - t0
        mine = b.vectors
        rec["max_abs_diff_vs_lapack_up_to_sign"] = float(max(
            np.max(np.abs(a * np.sign(np.einsum("ij,ij->j", a, r)) - r)) for a, r in zip(mine, vecs)))
        rec["cpu_cores"] = len(os.sched_getaffinity(0))
    print(json.dumps(rec), flush=True)
    del b, w, pos, neg, back
    torch.cuda.empty_cache()
