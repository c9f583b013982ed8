"""BASELINE cfg 4 in full: N = 2048, smooth W0, h = 0.005, 200 steps on the
device and with the CPU oracle from the same W0 (numpy/OpenBLAS on all host
cores): per-step iteration counts, relF(W_200), Casimir C2/C3 and energy
drift of both, the drifts also sampled every SAMPLE steps along both
trajectories (same evaluator for both: the oracle's) so the comparison is
not a single roundoff-level sample.  One JSON line (profiles/r02_cfg4_full.json)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200.integrator import midpoint_step_raw  # noqa: E402
from oracle import zeitlin_oracle as zo  # noqa: E402

N, H, STEPS = 2048, 0.005, int(sys.argv[1]) if len(sys.argv) > 1 else 200
SAMPLE = 20
dev = torch.device("cuda:0")
r = zo.random_admissible(N, np.random.default_rng(0), 1.0 / N)
op = zt.build_operator(N, dev)
w0 = zt.solve_stream(torch.from_numpy(r).to(dev), op)
w0 = w0 / torch.linalg.norm(w0)
w0n = w0.cpu().numpy()
# device
x, spare, its, gsamp = w0.clone(), torch.empty_like(w0), [], []
gpu_s = 0.0
for s in range(STEPS):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, k, _, _ = midpoint_step_raw(x, H, 1e-12, 10, op, out=spare)
    torch.cuda.synchronize()
    gpu_s += time.perf_counter() - t0
    its.append(k)
    x, spare = out, x
    if (s + 1) % SAMPLE == 0:
        gsamp.append(x.cpu().numpy())
# oracle
oop = zo.build_operator(N)
ref, rits, rsamp = w0n.copy(), [], []
cpu_s = 0.0
for s in range(STEPS):
    t0 = time.perf_counter()
    ref, k, _ = zo.midpoint_step(ref, H, op=oop)
    cpu_s += time.perf_counter() - t0
    rits.append(k)
    if (s + 1) % SAMPLE == 0:
        rsamp.append(ref.copy())
xn = x.cpu().numpy()
c0, h0 = zo.casimirs(w0n, 3), zo.hamiltonian(w0n, oop)


def drift(w):
    c = zo.casimirs(w, 3)
    return {"C2": abs(c[1] - c0[1]) / abs(c0[1]), "C3": abs(c[2] - c0[2]) / abs(c0[2]),
            "H": abs(zo.hamiltonian(w, oop) - h0) / abs(h0)}


def along(samples):
    d = [drift(w) for w in samples]
    return {k: {"max": max(e[k] for e in d), "rms": float(np.sqrt(np.mean([e[k] ** 2 for e in d]))),
                "samples": [e[k] for e in d]} for k in ("C2", "C3", "H")}


print(json.dumps({
    "cfg": 4, "N": N, "h": H, "steps": STEPS,
    "iterations_identical": its == rits, "iterations": sorted(set(its)),
    "relF_W_final": float(np.linalg.norm(xn - ref) / np.linalg.norm(ref)),
    "drift_gpu": drift(xn), "drift_oracle": drift(ref),
    "drift_along_gpu": along(gsamp), "drift_along_oracle": along(rsamp), "sample_every": SAMPLE,
    "gpu_s": gpu_s, "cpu_s": cpu_s, "cpu_cores": len(os.sched_getaffinity(0)),
}))
