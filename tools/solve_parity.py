"""relF of the device stream solve vs the CPU oracle (dpttrf factors) at
several N, on random_admissible(N, default_rng(0), 1/N) and the smooth cfg-4
recipe; prints the worst per-N value."""
import json, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2206_05466_b200 as zt
from oracle import zeitlin_oracle as zo
for n in (200, 512, 1024, 2048, 4096):
    rng = np.random.default_rng(0)
    w = zo.random_admissible(n, rng, 1.0 / n)
    s = zo.smooth_initial(n) if n <= 2048 else None
    out = {}
    for name, x in (("white", w), ("smooth", s)):
        if x is None:
            continue
        p = zt.solve_stream(torch.from_numpy(x).cuda()).cpu().numpy()
        r = zo.solve_stream(x, check=False)
        out[name] = float(np.linalg.norm(p - r) / np.linalg.norm(r))
    print(json.dumps({"n": n, **out}), flush=True)
