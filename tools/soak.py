"""Long device-resident run at the cfg-4 recipe: K steps through the C ABI,
Casimirs C2, C3 and the energy H sampled every S steps (relative drift from
step 0), iteration counts, exact skew-Hermitian structure kept.  Robustness
evidence (python tools/soak.py [steps] [every] [N])."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200.diagnostics import hamiltonian  # noqa: E402
from paper_2206_05466_b200.integrator import casimirs, midpoint_step_raw  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
every = int(sys.argv[2]) if len(sys.argv) > 2 else 200
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
h = 0.005
dev = torch.device("cuda:0")
from bench import cfg4_initial_numpy  # noqa: E402

op = zt.build_operator(n, dev)
w = zt.solve_stream(torch.from_numpy(cfg4_initial_numpy(n)).to(dev), op)
w = w / torch.linalg.norm(w)


def meters(x):
    c = casimirs(x, 3)
    return float(c[1]), float(c[2]), float(hamiltonian(x, op))


c2_0, c3_0, h_0 = meters(w)
spare = torch.empty_like(w)
its, rows = [], []
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for s in range(1, steps + 1):
    out, k, _, _ = midpoint_step_raw(w, h, 1e-12, 10, op, out=spare)
    its.append(k)
    w, spare = out, w
    if s % every == 0:
        c2, c3, hh = meters(w)
        skew = float((w + w.conj().T).abs().max())
        rows.append({"step": s, "dC2": abs(c2 - c2_0) / abs(c2_0), "dC3": abs(c3 - c3_0) / max(abs(c3_0), 1e-300),
                     "dH": abs(hh - h_0) / abs(h_0), "max|W+W^H|": skew,
                     "finite": bool(torch.isfinite(torch.view_as_real(w)).all())})
t1.record()
torch.cuda.synchronize()
print(json.dumps({"N": n, "h": h, "steps": steps, "iterations": sorted(set(its)), "samples": rows,
                  "wall_ms_incl_meters": t0.elapsed_time(t1)}))
