"""Host logic of the row-block sharded step (cfg 5) on world size 2 over gloo.

The collectives (all-gather of X, all-to-all of the a tiles for (a^H)_R,
all-reduce max of the residual) and the row-block algebra are the product
code (paper_2206_05466_b200/sharded.py); only the per-rank compute is a CPU
stand-in built on the oracle, injected here as the test backend.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import zeitlin_oracle as zo


class CpuBackend:
    device = torch.device("cpu")

    def solve(self, x_full):
        return torch.from_numpy(zo.solve_stream(x_full.numpy(), check=False))

    def validate(self, x_full):
        zo.validate_vorticity(x_full.numpy())

    def gemm_rows(self, p_rows, x_full):
        return p_rows @ x_full

    def gemm_block(self, a_rows, b_full, c0, mc):
        return a_rows @ b_full[:, c0:c0 + mc]

    def update_rows(self, a_rows, p, ah_rows, base, xprev, hh, qq):
        out = base + hh * (a_rows - ah_rows) + qq * (a_rows @ p)
        res = float((out - xprev).abs().max()) if xprev is not None else 0.0
        return out, res


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, h, steps, max_iter, q, grid=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_05466_b200.sharded import BlockShardedStepper, ShardedStepper  # noqa: WPS433

        w = torch.from_numpy(zo.smooth_initial(n))
        if grid is None:
            st = ShardedStepper(n, CpuBackend())
            rows = w[st.r0:st.r0 + st.m].clone()
        else:
            st = BlockShardedStepper(n, CpuBackend(), grid=grid if grid != "auto" else None)
            rows = st.block(w)
        iters = []
        for _ in range(steps):
            rows, k, _ = st.midpoint_step(rows, h, max_iter=max_iter)
            iters.append(k)
        full = st.all_gather_rows(rows)
        if rank == 0:
            q.put(("ok", full.numpy(), iters))
    except Exception as e:  # report to the parent
        if rank == 0:
            q.put(("err", type(e).__name__, getattr(e, "iterations", None)))
    finally:
        dist.destroy_process_group()


def _run(world, n, h, steps, max_iter=10, grid=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, h, steps, max_iter, q, grid)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    return out


@pytest.mark.parametrize("world,n", [(2, 16), (2, 24), (4, 16)])
def test_sharded_step_matches_oracle(world, n):
    status, full, iters = _run(world, n, h=0.01, steps=3)
    assert status == "ok"
    w = zo.smooth_initial(n)
    ref_iters = []
    for _ in range(3):
        w, k, _ = zo.midpoint_step(w, 0.01)
        ref_iters.append(k)
    assert iters == ref_iters
    assert np.linalg.norm(full - w) / np.linalg.norm(w) <= 1e-13


@pytest.mark.parametrize("world,n,grid", [(2, 16, (1, 2)), (2, 16, (2, 1)), (4, 16, "auto"), (4, 24, (1, 4))])
def test_block_sharded_step_matches_oracle(world, n, grid):
    """2-D block layout (BlockShardedStepper): block all-gathers of X and a,
    block products, the (a^H) block from the gathered a; identical iteration
    counts and W after 3 steps against the oracle."""
    status, full, iters = _run(world, n, h=0.01, steps=3, grid=grid)
    assert status == "ok", (status, full)
    w = zo.smooth_initial(n)
    ref_iters = []
    for _ in range(3):
        w, k, _ = zo.midpoint_step(w, 0.01)
        ref_iters.append(k)
    assert iters == ref_iters
    err = np.linalg.norm(full - w) / np.linalg.norm(w)
    assert err <= 1e-13, (err, np.abs(full - w).max(axis=1))


def test_block_sharded_non_convergence_raises():
    status, name, iters = _run(4, 16, h=0.5, steps=1, max_iter=1, grid="auto")
    assert status == "err" and name == "FixedPointError" and iters == 1


def test_block_grid_and_shapes():
    from paper_2206_05466_b200.sharded import BlockShardedStepper, block_grid

    assert [block_grid(g) for g in (1, 2, 4, 8)] == [(1, 1), (1, 2), (2, 2), (2, 4)]
    st = BlockShardedStepper(12, CpuBackend())  # no process group: one 1 x 1 block
    assert (st.mr, st.mc, st.r0, st.c0) == (12, 12, 0, 0)
    with pytest.raises(ValueError, match="process grid"):
        BlockShardedStepper(12, CpuBackend(), grid=(1, 2))


def test_sharded_non_convergence_raises():
    status, name, iters = _run(2, 16, h=0.5, steps=1, max_iter=1)
    assert status == "err" and name == "FixedPointError" and iters == 1


def test_sharded_requires_divisible_n():
    from paper_2206_05466_b200.sharded import ShardedStepper

    class FakeGroup:
        pass

    # single process (no process group): world = 1, any N divides
    st = ShardedStepper(10, CpuBackend())
    assert st.m == 10 and st.r0 == 0


def test_residual_bit_pattern_max():
    """The peer path reduces residuals as int64 bit patterns of non-negative
    doubles (one host read per update): the max is the max double, NaN wins
    and reads back as inf (never converged, integrator.py:131)."""
    from paper_2206_05466_b200.sharded import _local_max

    def bits(v):
        return torch.tensor([v], dtype=torch.float64).view(torch.int64)

    assert _local_max([bits(1e-13), bits(3e-12), bits(0.0)]) == 3e-12
    assert _local_max([bits(2.5e-14)]) == 2.5e-14
    assert _local_max([bits(1e-13), bits(float("nan"))]) == float("inf")
