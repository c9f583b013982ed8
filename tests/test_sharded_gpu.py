"""GPU checks of the sharded-step building blocks: rectangular DMMA GEMM,
row-block update epilogue, and the ShardedStepper over a single-rank NCCL
group (exercises the real collective calls) against the oracle."""

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
    a, p, ah, base, xp = c(m, n), c(n, n), c(m, n), c(m, n), c(m, n)
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
