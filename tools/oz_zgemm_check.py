"""zt_oz_zgemm (FP64 complex GEMM emulated on INT8 tensor cores) vs numpy and
vs an extended-precision reference; native DMMA zt_zgemm beside it."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05466_b200 import _lib  # noqa: E402
from paper_2206_05466_b200.integrator import zgemm  # noqa: E402
from oracle import zeitlin_oracle as zo  # noqa: E402

lib = _lib.lib
dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream


def oz(a, b, bmode=0, lower=0):
    n = a.shape[0]
    ws = torch.empty(lib.zt_oz_workspace_bytes(n), dtype=torch.uint8, device=dev)
    c = torch.zeros_like(a)
    rc = lib.zt_oz_zgemm(n, a.data_ptr(), n, b.data_ptr(), n, bmode, c.data_ptr(), n, lower, ws.data_ptr(),
                         ws.numel(), st)
    torch.cuda.synchronize()
    assert rc == 0, (rc, lib.zt_last_error())
    return c, ws


def relf(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


for n in (130, 256, 512):
    rng = np.random.default_rng(n)
    A = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    B = zo.random_admissible(n, rng, 1.0 / n)
    B[np.diag_indices(n)] += 1e-3 * rng.normal(size=n)  # real diagonal part (as the solve's P)
    # exact-ish reference in extended precision
    Al, Bl = A.astype(np.clongdouble), B.astype(np.clongdouble)
    ref = (Al @ Bl).astype(np.complex128) if n <= 256 else A @ B
    ad, bd = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
    c0, _ = oz(ad, bd, 0)
    c1, _ = oz(ad, bd, 1)
    cn = zgemm(ad, bd).cpu().numpy()
    print(f"N={n}: oz(general B) relF {relf(c0.cpu().numpy(), ref):.2e}  oz(skew B) {relf(c1.cpu().numpy(), ref):.2e}  "
          f"native DMMA {relf(cn, ref):.2e}  numpy {relf(A @ B, ref):.2e}", flush=True)
    cl, _ = oz(ad, bd, 1, lower=1)
    m = np.tril(np.ones((n, n), bool))
    blk = (np.arange(n)[:, None] // 128) >= (np.arange(n)[None, :] // 128)
    print(f"   lower tiles equal to full: {bool(np.array_equal(cl.cpu().numpy()[blk], c1.cpu().numpy()[blk]))}")

n = 2048
rng = np.random.default_rng(0)
A = torch.from_numpy(rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).to(dev)
B = torch.from_numpy(zo.random_admissible(n, rng, 1.0 / n)).to(dev)
c, ws = oz(A, B, 0)
print(f"N=2048 oz vs numpy relF {relf(c.cpu().numpy(), A.cpu().numpy() @ B.cpu().numpy()):.2e}")
for mode in (0, 1):
    for _ in range(2):
        lib.zt_oz_zgemm(n, A.data_ptr(), n, B.data_ptr(), n, mode, c.data_ptr(), n, 0, ws.data_ptr(), ws.numel(), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        lib.zt_oz_zgemm(n, A.data_ptr(), n, B.data_ptr(), n, mode, c.data_ptr(), n, 0, ws.data_ptr(), ws.numel(), st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"oz_zgemm N=2048 bmode={mode}: {ms*1e3:.0f} us = {8*n**3/ms/1e9:.1f} TF algorithmic", flush=True)
for _ in range(2):
    zgemm(A, B, out=c)
e0.record()
for _ in range(10):
    zgemm(A, B, out=c)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"native DMMA zgemm N=2048: {ms*1e3:.0f} us = {8*n**3/ms/1e9:.1f} TF", flush=True)
