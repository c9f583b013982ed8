"""GPU checks of the sharded-step building blocks: rectangular DMMA GEMM,
row-block update (on the library's step product), the INT8 building blocks
(row / column conversions of sub-blocks, reconstruction with scatter and
mirror) against numpy, and the ShardedStepper over a single-rank NCCL group
(exercises the real collective calls) against the oracle."""

import os
import socket

import numpy as np
import pytest
from conftest import relf

from oracle import zeitlin_oracle as zo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


@pytest.mark.parametrize("m,n,k", [(64, 128, 128), (17, 33, 65), (256, 1024, 1024), (5, 3, 2), (512, 512, 200)])
def test_zgemm_rect(m, n, k):
    from paper_2206_05466_b200 import _lib

    rng = np.random.default_rng(m + n + k)
    a = rng.normal(size=(m, k)) + 1j * rng.normal(size=(m, k))
    b = rng.normal(size=(k, n)) + 1j * rng.normal(size=(k, n))
    da, db = dev(a), dev(b)
    c = torch.empty((m, n), dtype=torch.complex128, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib.zt_zgemm_rect(m, n, k, da.data_ptr(), k, db.data_ptr(), n, c.data_ptr(), n, 0, s))
    assert relf(c.cpu().numpy(), a @ b) <= 1e-14


@pytest.mark.parametrize("m,n", [(64, 256), (100, 300), (512, 512)])
def test_update_rows(m, n):
    from paper_2206_05466_b200.sharded import DeviceBackend

    rng = np.random.default_rng(m * n)
    c = lambda *s: rng.normal(size=s) + 1j * rng.normal(size=s)  # noqa: E731
    a, ah, base, xp = c(m, n), c(m, n), c(m, n), c(m, n)
    p = zo.random_admissible(n, rng, 1.0)  # the step's P is skew-Hermitian (the INT8 path reads it as skew-B)
    be = DeviceBackend(n, torch.device("cuda"))
    out, res = be.update_rows(dev(a), dev(p), dev(ah), dev(base), dev(xp), 0.003, -2e-6)
    want = base + 0.003 * (a - ah) + (-2e-6) * (a @ p)
    assert relf(out.cpu().numpy(), want) <= 1e-15
    assert abs(res - np.max(np.abs(want - xp))) <= 1e-15 * np.max(np.abs(want - xp))


@pytest.fixture(scope="module", autouse=True)
def _teardown_pg():
    yield
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("force", [False, True])
def test_sharded_stepper_single_rank_nccl(force):
    import torch.distributed as dist

    from paper_2206_05466_b200.sharded import DeviceBackend, ShardedStepper

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    n = 256
    st = ShardedStepper(n, DeviceBackend(n, torch.device("cuda", 0)), force_collectives=force)
    w = zo.smooth_initial(n)
    x = dev(w)
    ref = w
    for _ in range(2):
        x, k, _ = st.midpoint_step(x, 0.005)
        ref, kr, _ = zo.midpoint_step(ref, 0.005)
        assert k == kr
    assert relf(x.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("m,n,c0,mc", [(128, 256, 128, 128), (100, 300, 40, 130), (256, 512, 0, 512),
                                        (512, 1024, 256, 256)])
def test_gemm_block(m, n, c0, mc):
    """DeviceBackend.gemm_block (2-D layout): rows times a column block of a
    full matrix read in place, on the INT8 product, against numpy."""
    from paper_2206_05466_b200.sharded import DeviceBackend

    rng = np.random.default_rng(m + n + c0)
    a = (rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))) / n
    b = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / n
    be = DeviceBackend(n, torch.device("cuda", 0))
    got = be.gemm_block(dev(a), dev(b), c0, mc).cpu().numpy()
    assert got.shape == (m, mc)
    assert relf(got, a @ b[:, c0:c0 + mc]) <= 1e-14


@pytest.mark.parametrize("force", [False, True])
def test_block_stepper_single_rank_nccl(force):
    import torch.distributed as dist

    from paper_2206_05466_b200.sharded import BlockShardedStepper, DeviceBackend

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    n = 256
    st = BlockShardedStepper(n, DeviceBackend(n, torch.device("cuda", 0)), force_collectives=force)
    w = zo.smooth_initial(n)
    x = st.block(dev(w))
    ref = w
    for _ in range(2):
        x, k, _ = st.midpoint_step(x, 0.005)
        ref, kr, _ = zo.midpoint_step(ref, 0.005)
        assert k == kr
    assert relf(st.all_gather_blocks(x).cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("n,world", [(256, 2), (256, 4), (384, 8)])
def test_block_stepper_thread_ranks(n, world):
    """The 2-D block layout on G ranks of one GPU, one host thread per rank:
    the block all-gathers and the residual all-reduce are host-side
    exchanges between the threads (no kernel waits on another rank's), the
    block products and the solve run on the device backend.  Identical
    iteration counts and W within 1e-12 of the oracle after 2 steps."""
    import threading

    from paper_2206_05466_b200.sharded import BlockShardedStepper, DeviceBackend, block_grid

    pr, pc = block_grid(world)
    bar = threading.Barrier(world)
    box: dict = {}

    class ThreadRank(BlockShardedStepper):
        def __init__(self, rank):
            self.world, self.rank, self.force, self.group = world, rank, True, None
            self.n, self.pr, self.pc = n, pr, pc
            self.mr, self.mc = n // pr, n // pc
            self.br, self.bc = divmod(rank, pc)
            self.r0, self.c0 = self.br * self.mr, self.bc * self.mc
            self.backend = DeviceBackend(n, torch.device("cuda", 0))

        def _exchange(self, v):
            box[self.rank] = v
            bar.wait()
            got = [box[g] for g in range(world)]
            bar.wait()
            return got

        def all_gather_blocks(self, blk):
            torch.cuda.synchronize()
            g = torch.cat(self._exchange(blk.contiguous()))
            return g.reshape(pr, pc, self.mr, self.mc).permute(0, 2, 1, 3).reshape(n, n)

        all_gather_rows = all_gather_blocks

        def all_reduce_max(self, v):
            return max(self._exchange(v))

    w = zo.smooth_initial(n)
    wd = dev(w)
    out, errs = [None] * world, []

    def run(rank):
        try:
            st = ThreadRank(rank)
            x = st.block(wd)
            ks = []
            for _ in range(2):
                x, k, _ = st.midpoint_step(x, 0.005)
                ks.append(k)
            out[rank] = (st.all_gather_blocks(x), ks)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            bar.abort()

    th = [threading.Thread(target=run, args=(g,)) for g in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    ref, kref = w, []
    for _ in range(2):
        ref, k, _ = zo.midpoint_step(ref, 0.005)
        kref.append(k)
    for full, ks in out:
        assert ks == kref
        assert relf(full.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("m,n,c0,nc", [(64, 256, 0, 256), (100, 300, 40, 130), (256, 512, 256, 256)])
def test_oz_building_blocks(m, n, c0, nc):
    """zt_oz_convert_rows / _cols + zt_oz_modgemm + zt_oz_reconstruct: a_R = P_R X
    with the column blocks scattered to peer buffers, and a block a_R P[:, C]
    of a skew-Hermitian P (rows C as skew-B planes) with its -conj^T mirror."""
    from paper_2206_05466_b200 import _lib

    lib = _lib.lib
    rng = np.random.default_rng(m + n)
    pad = lambda x: (x + 255) // 256 * 256  # noqa: E731
    s = torch.cuda.current_stream().cuda_stream
    d = torch.device("cuda")
    P = zo.random_admissible(n, rng, 1.0)
    P[np.diag_indices(n)] += 1e-3 * rng.normal(size=n)  # real diagonal part: taken as is
    X = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    A = rng.normal(size=(m, n)) + 1j * rng.normal(size=(m, n))
    kb = lib.zt_oz_bits(n)

    def planes(rows, cols):
        return torch.empty(lib.zt_oz_plane_bytes(rows, cols), dtype=torch.uint8, device=d)

    ap, sa = planes(m, n), torch.empty(pad(m), dtype=torch.int32, device=d)
    bx, sx = planes(n, n), torch.empty(pad(n), dtype=torch.int32, device=d)
    cm = torch.empty(pad(n), dtype=torch.int64, device=d)
    dA, dX, dP = dev(A), dev(X), dev(P)
    _lib.check(lib.zt_oz_convert_rows(m, n, dA.data_ptr(), n, 0, 0, kb, ap.data_ptr(), sa.data_ptr(), None, s))
    _lib.check(lib.zt_oz_convert_cols(n, n, dX.data_ptr(), n, kb, bx.data_ptr(), sx.data_ptr(), cm.data_ptr(), s))
    r = planes(m, n)
    _lib.check(lib.zt_oz_modgemm(17, pad(m), pad(n), pad(n), ap.data_ptr(), bx.data_ptr(), r.data_ptr(), 0, s))
    # scatter: column block h (width mloc) into peer h's n x mloc buffer at rows r0 + i
    mloc, r0 = 50, 7
    nblk = -(-n // mloc)
    peers = [torch.zeros((r0 + m, mloc), dtype=torch.complex128, device=d) for _ in range(nblk)]
    ptrs = torch.tensor([t.data_ptr() for t in peers], dtype=torch.int64, device=d)
    c = torch.zeros((m, n), dtype=torch.complex128, device=d)
    _lib.check(lib.zt_oz_reconstruct(m, n, r.data_ptr(), sa.data_ptr(), sx.data_ptr(), c.data_ptr(), n,
                                     ptrs.data_ptr(), mloc, r0, None, n, 0, s))
    ref = A @ X
    got = c.cpu().numpy()
    assert relf(got, ref) <= 1e-15
    for h, t in enumerate(peers):
        w = min(mloc, n - h * mloc)
        np.testing.assert_array_equal(t[r0:, :w].cpu().numpy(), got[:, h * mloc:h * mloc + w])
    # block a P[:, C] from rows C of P in the skew-B layout, mirrored
    bp, sb = planes(nc, n), torch.empty(pad(nc), dtype=torch.int32, device=d)
    _lib.check(lib.zt_oz_convert_rows(nc, n, dP.data_ptr() + c0 * n * 16, n, 1, c0, kb, bp.data_ptr(),
                                      sb.data_ptr(), None, s))
    r2 = planes(m, nc)
    _lib.check(lib.zt_oz_modgemm(17, pad(m), pad(nc), pad(n), ap.data_ptr(), bp.data_ptr(), r2.data_ptr(), 0, s))
    blk = torch.zeros((m, nc), dtype=torch.complex128, device=d)
    mir = torch.zeros((nc, m), dtype=torch.complex128, device=d)
    _lib.check(lib.zt_oz_reconstruct(m, nc, r2.data_ptr(), sa.data_ptr(), sb.data_ptr(), blk.data_ptr(), nc,
                                     None, 1, 0, mir.data_ptr(), m, 0, s))
    want = A @ P[:, c0:c0 + nc]
    b = blk.cpu().numpy()
    assert relf(b, want) <= 1e-15
    np.testing.assert_array_equal(mir.cpu().numpy(), -b.conj().T)


def test_oz_lower_block_mirrors_into_itself():
    """Lower-mode residue GEMM + zt_oz_reconstruct(lower=1, mirror=the block):
    a skew-Hermitian diagonal block b = a P (a = P X with skew P, X) from its
    lower 256-tiles equals the full product up to round-off, exactly
    skew-Hermitian off the diagonal tiles."""
    from paper_2206_05466_b200 import _lib

    lib = _lib.lib
    n = 600
    rng = np.random.default_rng(3)
    pad = lambda x: (x + 255) // 256 * 256  # noqa: E731
    s = torch.cuda.current_stream().cuda_stream
    d = torch.device("cuda")
    P = zo.random_admissible(n, rng, 1.0)
    X = zo.random_admissible(n, rng, 1.0)
    A = P @ X
    kb = lib.zt_oz_bits(n)
    ap = torch.empty(lib.zt_oz_plane_bytes(n, n), dtype=torch.uint8, device=d)
    bp = torch.empty_like(ap)
    r = torch.empty_like(ap)
    sa, sb = (torch.empty(pad(n), dtype=torch.int32, device=d) for _ in range(2))
    dA, dP = dev(A), dev(P)
    _lib.check(lib.zt_oz_convert_rows(n, n, dA.data_ptr(), n, 0, 0, kb, ap.data_ptr(), sa.data_ptr(), None, s))
    _lib.check(lib.zt_oz_convert_rows(n, n, dP.data_ptr(), n, 1, 0, kb, bp.data_ptr(), sb.data_ptr(), None, s))
    _lib.check(lib.zt_oz_modgemm(17, pad(n), pad(n), pad(n), ap.data_ptr(), bp.data_ptr(), r.data_ptr(), 1, s))
    c = torch.full((n, n), float("nan"), dtype=torch.complex128, device=d)
    _lib.check(lib.zt_oz_reconstruct(n, n, r.data_ptr(), sa.data_ptr(), sb.data_ptr(), c.data_ptr(), n, None, 1, 0,
                                     c.data_ptr(), n, 1, s))
    got = c.cpu().numpy()
    assert not np.isnan(got.real).any()
    assert relf(got, A @ P) <= 1e-15
    off = (np.arange(n)[:, None] // 256) != (np.arange(n)[None, :] // 256)
    assert np.array_equal(got[off], (-got.conj().T)[off])
