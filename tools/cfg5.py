"""BASELINE cfg 5 on one GPU: N = 4096 and 8192, smooth initial vorticity
(lap^-1 of random_admissible(N, default_rng(0), 1/N), unit Frobenius norm),
h = 0.0025.  Times the single-GPU step (one CUDA graph per step) and the
row-block sharded code path on a one-rank NCCL group, and checks the first
steps against the CPU oracle (same W0) for parity: identical iteration
counts, relF(W) <= 1e-10.  One JSON line per N to stdout.

    python tools/cfg5.py [--steps 50] [--oracle-steps 2] [--n 4096 8192]
"""
import argparse
import json
import os
import socket
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2206_05466_b200 as zt  # noqa: E402
from paper_2206_05466_b200.integrator import midpoint_step_raw  # noqa: E402
from oracle import zeitlin_oracle as zo  # noqa: E402

H, TOL, MAX_ITER = 0.0025, 1e-12, 10


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--oracle-steps", type=int, default=2)
    ap.add_argument("--n", type=int, nargs="+", default=[4096, 8192])
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
    s.close()
    import torch.distributed as dist
    from paper_2206_05466_b200.sharded import DeviceBackend, PeerShardedStepper, ShardedStepper

    dist.init_process_group("nccl", device_id=dev)
    for n in args.n:
        rec = {"cfg": 5, "N": n, "h": H, "gpus": 1}
        r = zo.random_admissible(n, np.random.default_rng(0), 1.0 / n)
        op = zt.build_operator(n, dev)
        w0 = zt.solve_stream(torch.from_numpy(r).to(dev), op)
        w0 = w0 / torch.linalg.norm(w0)
        # parity: the first oracle steps from the same W0
        t0 = time.perf_counter()
        ref = w0.cpu().numpy()
        oop = zo.build_operator(n)
        x = w0.clone()
        kr_all, k_all = [], []
        for _ in range(args.oracle_steps):
            ref, kr, _ = zo.midpoint_step(ref, H, TOL, MAX_ITER, op=oop)
            x, k, _, _ = midpoint_step_raw(x, H, TOL, MAX_ITER, op)
            kr_all.append(kr)
            k_all.append(k)
        rec["oracle_s_per_step"] = (time.perf_counter() - t0) / max(1, args.oracle_steps)
        rec["parity"] = {"steps": args.oracle_steps, "iters_gpu": k_all, "iters_oracle": kr_all,
                         "relF": float(np.linalg.norm(x.cpu().numpy() - ref) / np.linalg.norm(ref))}
        del oop
        # single-GPU fused step
        cur, spare = w0.clone(), torch.empty_like(w0)
        for _ in range(2):
            cur2, _, _, _ = midpoint_step_raw(cur, H, TOL, MAX_ITER, op, out=spare)
            cur, spare = cur2, cur
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = []
        e0.record()
        for _ in range(args.steps):
            out, k, _, _ = midpoint_step_raw(cur, H, TOL, MAX_ITER, op, out=spare)
            its.append(k)
            cur, spare = out, cur
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        kbar = float(np.mean(its))
        c0, c1 = zt.casimirs(w0, 3), zt.casimirs(cur, 3)
        h0, h1 = zt.hamiltonian(w0, op), zt.hamiltonian(cur, op)
        rec["single_gpu"] = {"ms_per_step": ms, "steps_per_s": 1e3 / ms, "steps": args.steps,
                             "iterations": sorted(set(its)),
                             "TFLOPs_alg": 16.0 * n**3 * (kbar + 1) / (ms * 1e-3) / 1e12,
                             "drift": {"C2": abs(c1[1] - c0[1]) / abs(c0[1]), "C3": abs(c1[2] - c0[2]) / abs(c0[2]),
                                       "H": abs(h1 - h0) / abs(h0)}}
        del cur, spare
        # the sharded code paths on a one-rank group (collectives / peer stores executed)
        be = DeviceBackend(n, dev)
        ns = max(2, min(args.steps, 10))
        for name, st in (("sharded_peer_g1", PeerShardedStepper(n, be)),
                         ("sharded_nccl_g1", ShardedStepper(n, be, force_collectives=True))):
            rows = w0.clone()
            rows, _, _ = st.midpoint_step(rows, H, TOL, MAX_ITER)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(ns):
                rows, k, _ = st.midpoint_step(rows, H, TOL, MAX_ITER)
            e1.record()
            torch.cuda.synchronize()
            rec[name] = {"ms_per_step": e0.elapsed_time(e1) / ns, "steps": ns}
            del st
        print(json.dumps(rec), flush=True)
        del rows, w0, be
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
