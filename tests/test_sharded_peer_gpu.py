"""Peer-fused sharded step (sharded.py: collectives as epilogue stores into
the other ranks' buffers) on the library's step product (the INT8 Ozaki-II
GEMM by default; a subprocess runs the DMMA variant).  G virtual ranks on one GPU run the algorithm
phase by phase (every kernel's inputs are complete before it starts; no rank
waits on another), and must reproduce the single-GPU step; the symmetric-
memory path runs on a one-rank NCCL group."""

import numpy as np
import pytest
import torch
from conftest import relf

from oracle import zeitlin_oracle as zo

pytestmark = pytest.mark.gpu


def _virtual_ranks(n, world, dev):
    from paper_2206_05466_b200.sharded import DeviceBackend, OzPeerRank, PeerRank

    be = DeviceBackend(n, dev)
    cls = OzPeerRank if be.oz else PeerRank
    m = n // world
    xf = [torch.zeros((n, n), dtype=torch.complex128, device=dev) for _ in range(world)]
    ac = [torch.zeros((n, m), dtype=torch.complex128, device=dev) for _ in range(world)]
    br = [torch.full((m, n), float("nan"), dtype=torch.complex128, device=dev) for _ in range(world)]
    xp = torch.tensor([t.data_ptr() for t in xf], dtype=torch.int64, device=dev)
    ap = torch.tensor([t.data_ptr() for t in ac], dtype=torch.int64, device=dev)
    bp = [t.data_ptr() for t in br]
    return [cls(n, world, g, be, xf[g], ac[g], xp, ap, br[g], bp) for g in range(world)]


@pytest.mark.parametrize("n,world", ((256, 2), (512, 4), (384, 3), (512, 8), (640, 5), (768, 6), (300, 3), (200, 4), (210, 6)))
def test_virtual_ranks_match_single_gpu(n, world):
    from paper_2206_05466_b200.integrator import midpoint_step_raw
    from paper_2206_05466_b200.laplacian import build_operator
    from paper_2206_05466_b200.sharded import peer_midpoint_step

    dev = torch.device("cuda:0")
    w = torch.from_numpy(zo.smooth_initial(n)).to(dev)
    ranks = _virtual_ranks(n, world, dev)
    m = n // world
    rows = [w[g * m:(g + 1) * m].contiguous() for g in range(world)]
    ref = w
    op = build_operator(n, dev)
    for _ in range(3):
        rows, k, r = peer_midpoint_step(ranks, rows, 0.005)
        ref, kr, _, _ = midpoint_step_raw(ref, 0.005, 1e-12, 10, op)
        assert k == kr
    got = torch.cat(rows).cpu().numpy()
    assert relf(got, ref.cpu().numpy()) <= 1e-13
    # the gathered iterate (the converged W~, updated in place and broadcast)
    # is identical on every rank, and the balanced GEMM-2 blocks tile b_R
    # exactly (b rows started as NaN)
    for rk in ranks:
        assert torch.equal(rk.xfull, ranks[0].xfull)
        assert not torch.isnan(torch.view_as_real(rk.brows)).any()
    work = [sum(nr * nc for _, nr, _, nc, _ in rk.blocks()) for rk in ranks]
    m = n // world
    # (G+1)/2 blocks each; odd m splits the G/2 pair into m//2 and m - m//2
    assert max(work) - min(work) <= m and abs(sum(work) / world - m * m * (world + 1) / 2) <= m


def test_virtual_ranks_errors_and_nonconvergence():
    from paper_2206_05466_b200.integrator import FixedPointError
    from paper_2206_05466_b200.sharded import peer_midpoint_step

    dev = torch.device("cuda:0")
    n, world = 128, 2
    ranks = _virtual_ranks(n, world, dev)
    w = torch.from_numpy(zo.random_admissible(n, np.random.default_rng(1), 1.0)).to(dev)
    rows = [w[:64].contiguous(), w[64:].contiguous()]
    with pytest.raises(ValueError):
        peer_midpoint_step(ranks, rows, -1.0)
    with pytest.raises(FixedPointError) as e:
        peer_midpoint_step(ranks, rows, 0.5, max_iter=1)
    assert e.value.iterations == 1 and e.value.residual > 1e-14


def _one_rank_group(dev):
    import os
    import socket

    import torch.distributed as dist

    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
        s.close()
        dist.init_process_group("nccl", device_id=dev)


@pytest.mark.parametrize("graph", [False, True])
def test_symmetric_memory_path_one_rank(graph):
    """One-rank NCCL group with torch symmetric memory: the eager peer path
    and the device-driven graph path (fixed point as a conditional WHILE
    node, residual exchanged by peer stores, input gate in the graph) over
    two consecutive steps (the second replays the captured graph)."""
    import torch.distributed as dist

    from paper_2206_05466_b200.integrator import midpoint_step_raw
    from paper_2206_05466_b200.sharded import DeviceBackend, PeerShardedStepper

    dev = torch.device("cuda:0")
    _one_rank_group(dev)
    try:
        n = 256
        be = DeviceBackend(n, dev)
        st = PeerShardedStepper(n, be, graph=graph)
        assert st.graph == graph
        w = torch.from_numpy(zo.smooth_initial(n)).to(dev)
        ref = w
        cur = w.clone()
        for _ in range(2):
            cur, k, _ = st.midpoint_step(cur, 0.005)
            ref, kr, _, _ = midpoint_step_raw(ref, 0.005, 1e-12, 10, be.op)
            assert k == kr and relf(cur.cpu().numpy(), ref.cpu().numpy()) <= 1e-13
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", (200, 300))
def test_graph_path_ragged_sizes(n):
    """The device-driven graph step at sizes that are not multiples of the
    256-row residue tiles or of the 64-row solve chunks, replayed over three
    steps against the single-GPU step."""
    import torch.distributed as dist

    from paper_2206_05466_b200.integrator import midpoint_step_raw
    from paper_2206_05466_b200.sharded import DeviceBackend, PeerShardedStepper

    dev = torch.device("cuda:0")
    _one_rank_group(dev)
    try:
        be = DeviceBackend(n, dev)
        st = PeerShardedStepper(n, be, graph=True)
        w = torch.from_numpy(zo.random_admissible(n, np.random.default_rng(n), 1.0 / n)).to(dev)
        ref, cur = w, w.clone()
        for _ in range(3):
            cur, k, _ = st.midpoint_step(cur, 0.01)
            ref, kr, _, _ = midpoint_step_raw(ref, 0.01, 1e-12, 10, be.op)
            assert k == kr and relf(cur.cpu().numpy(), ref.cpu().numpy()) <= 1e-13
    finally:
        dist.destroy_process_group()


def test_graph_path_matches_eager_and_raises():
    """The graph path is bitwise the eager peer path; a non-skew input raises
    StructureError from the in-graph gate and a capped fixed point raises
    FixedPointError with the iteration count, as the reference does."""
    import torch.distributed as dist

    from paper_2206_05466_b200.integrator import FixedPointError
    from paper_2206_05466_b200.laplacian import StructureError
    from paper_2206_05466_b200.sharded import DeviceBackend, PeerShardedStepper

    dev = torch.device("cuda:0")
    _one_rank_group(dev)
    try:
        n = 256
        be = DeviceBackend(n, dev)
        ge, gg = PeerShardedStepper(n, be, graph=False), PeerShardedStepper(n, be, graph=True)
        w = torch.from_numpy(zo.random_admissible(n, np.random.default_rng(3), 1.0 / n)).to(dev)
        oe, ke, re = ge.midpoint_step(w.clone(), 0.01)
        og, kg, rg = gg.midpoint_step(w.clone(), 0.01)
        assert ke == kg and re == rg and torch.equal(oe, og)
        bad = w.clone()
        bad[0, 1] += 1.0
        with pytest.raises(StructureError, match="skew-Hermitian"):
            gg.midpoint_step(bad, 0.01)
        big = torch.from_numpy(zo.random_admissible(n, np.random.default_rng(1), 1.0)).to(dev)
        with pytest.raises(FixedPointError) as e:
            gg.midpoint_step(big, 0.5, max_iter=1)
        assert e.value.iterations == 1 and e.value.residual > 1e-14
        # the graph path still steps correctly after the errors
        og2, kg2, _ = gg.midpoint_step(w.clone(), 0.01)
        assert kg2 == ke and torch.equal(og2, oe)
    finally:
        dist.destroy_process_group()


def test_virtual_ranks_default_product_is_int8():
    from paper_2206_05466_b200.sharded import DeviceBackend, OzPeerRank

    dev = torch.device("cuda:0")
    assert DeviceBackend(256, dev).oz
    assert isinstance(_virtual_ranks(256, 2, dev)[0], OzPeerRank)


def test_virtual_ranks_native_dmma_variant():
    """ZT_GEMM_ALGO=3m in a fresh process: the DMMA sharded kernels still
    reproduce the single-GPU step."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import torch\n"
        "from test_sharded_peer_gpu import test_virtual_ranks_match_single_gpu as t\n"
        "t(512, 4); t(300, 3)\n"
        "print('ok')\n"
    )
    env = dict(os.environ, ZT_GEMM_ALGO="3m", PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests")]))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
