"""Quantized spherical Laplacian on B200: drop-in for ``zeitlin.laplacian``.

Same public names and semantics as the reference module
(/root/reference/pkg/src/zeitlin/laplacian.py:46-59); the O(N^2) stream
solve and the stencil run as sm_100a kernels (``csrc/zt_solve.cu``) through
the C ABI.  Inputs may be ``torch.cuda`` complex128 tensors (zero-copy,
device-resident — the fast path) or numpy arrays (copied to the current CUDA
device at the API edge and returned as numpy, so unmodified reference
callers work).  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib

__all__ = [
    "VorticityMatrix",
    "LaplacianBlock",
    "LaplacianOperator",
    "StructureError",
    "build_block",
    "build_operator",
    "apply_laplacian",
    "solve_stream",
    "skewness_residual",
    "trace_residual",
    "validate_vorticity",
    "spectral_norm",
]

VorticityMatrix = torch.Tensor
STRUCTURE_TOL = 1e-10  # laplacian.py:68


class StructureError(ValueError):
    """An input matrix violates a structural invariant (laplacian.py:71-72)."""


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------
def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _dev_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    d = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
    return torch.cuda.current_device() if d.index is None else d.index


def _to_device(w):
    """(contiguous complex128 CUDA tensor, was_numpy)."""
    if isinstance(w, torch.Tensor):
        if w.dim() != 2 or w.shape[0] != w.shape[1]:
            raise ValueError(f"expected a square matrix, got shape {tuple(w.shape)}")
        if not w.is_cuda:
            raise ValueError("tensor inputs must live on a CUDA device (no CPU fallback)")
        if w.dtype != torch.complex128:
            w = w.to(torch.complex128)
        return w.contiguous(), False
    a = np.asarray(w)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {a.shape}")
    a = np.ascontiguousarray(a, dtype=np.complex128)
    # stream-ordered copy: asynchronous when the array is pinned (results of
    # this module are, so a state fed back step after step is DMA'd directly);
    # every public call synchronises before returning, so the caller may
    # reuse the array afterwards
    return torch.from_numpy(a).to(torch.device("cuda", torch.cuda.current_device()), non_blocking=True), True


def _out(t: torch.Tensor, as_numpy: bool):
    """Device result -> the caller's type.  numpy results land in pinned host
    memory (torch's caching host allocator recycles the blocks once the caller
    drops them), so the copy runs at full DMA rate without page faults, and a
    result fed back as the next input is pinned too (direct DMA on the way in)."""
    if not as_numpy:
        return t
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


_ws_local = threading.local()


def workspace(device: torch.device, key: str, nbytes: int) -> torch.Tensor:
    """Per-thread reusable device workspace (cf. laplacian.py:232-248)."""
    store = getattr(_ws_local, "store", None)
    if store is None:
        store = _ws_local.store = {}
    k = (device.index, key)
    buf = store.get(k)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        store[k] = buf
    return buf


# ---------------------------------------------------------------------------
# blocks (host, closed form; laplacian.py:129-176)
# ---------------------------------------------------------------------------
def _block_entries(n_total: int, m: int):
    s = (n_total - 1) / 2.0
    i = np.arange(n_total - m, dtype=np.float64)
    diag = 2.0 * (s * (2.0 * i + 1.0 + m) - i * (i + m))
    i = i[:-1]
    off = -np.sqrt((i + m + 1.0) * (n_total - 1.0 - i - m)) * np.sqrt((i + 1.0) * (n_total - 1.0 - i))
    return diag, off


@dataclass(frozen=True)
class LaplacianBlock:
    """Tridiagonal restriction of the positive operator to diagonal m."""

    n_total: int
    m: int
    diag: np.ndarray
    offdiag: np.ndarray

    @property
    def size(self) -> int:
        return self.n_total - self.m

    def eigenvalues(self) -> np.ndarray:
        l = np.arange(self.m, self.n_total, dtype=np.float64)
        return l * (l + 1.0)

    def to_dense(self) -> np.ndarray:
        a = np.diag(self.diag)
        if self.offdiag.size:
            a += np.diag(self.offdiag, 1) + np.diag(self.offdiag, -1)
        return a


def build_block(n_total: int, m: int) -> LaplacianBlock:
    if n_total < 2:
        raise ValueError(f"matrix truncation must be at least 2, got {n_total}")
    if not 0 <= m <= n_total - 1:
        raise ValueError(f"diagonal index m={m} out of range for N={n_total}")
    d, o = _block_entries(n_total, m)
    return LaplacianBlock(n_total, m, d, o)


# ---------------------------------------------------------------------------
# operator (laplacian.py:179-219, 319-322)
# ---------------------------------------------------------------------------
class LaplacianOperator:
    """Per-(N, device) operator: LDL^T carry tables resident in HBM.

    Immutable after construction and shareable across threads/streams.
    """

    def __init__(self, n: int, device=None):
        if n < 2:
            raise ValueError(f"matrix truncation must be at least 2, got {n}")
        dev = torch.device("cuda", _dev_index(device))
        self.n = n
        self.device = dev
        h = ctypes.c_void_p()
        check(lib.zt_op_create(n, dev.index, ctypes.byref(h)))
        self._h = h.value

    @property
    def handle(self) -> int:
        return self._h

    def factors(self):
        """Reference-layout (linv, dinv) sheared tables (laplacian.py:213-215)."""
        n = self.n
        linv = np.zeros((n, n))
        dinv = np.zeros((n, n))
        check(lib.zt_op_factors(self._h, linv.ctypes.data, dinv.ctypes.data))
        return linv, dinv

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib.zt_op_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None


_op_cache: dict = {}
_op_lock = threading.Lock()


def build_operator(n: int, device=None) -> LaplacianOperator:
    """Cached operator per (N, device) (laplacian.py:319-322, LRU of 8)."""
    dev = _dev_index(device)
    key = (n, dev)
    with _op_lock:
        op = _op_cache.get(key)
        if op is None:
            if len(_op_cache) >= 8:
                _op_cache.pop(next(iter(_op_cache)))
            op = _op_cache[key] = LaplacianOperator(n, dev)
        return op


def _resolve(op, w) -> LaplacianOperator:
    """laplacian.py:325-333.

    ``op`` may be any operator object with an ``n`` attribute: unmodified
    reference callers pass the reference's own ``zeitlin.laplacian.
    LaplacianOperator`` (driver.py:290, 396; diagnostics.py:62), which holds
    host tables only.  Such an operator (or one of ours built for another
    device) is mapped to the cached device operator for (N, the matrix's
    device); the size check and its message are the reference's.
    """
    n = w.shape[0]
    if op is None:
        return build_operator(n, w.device)
    op_n = getattr(op, "n", None)
    if op_n is None:
        raise TypeError(f"expected a LaplacianOperator, got {type(op).__name__}")
    if op_n != n:
        raise ValueError(f"operator size {op_n} does not match matrix size {n}")
    if not isinstance(op, LaplacianOperator) or op.device != w.device:
        return build_operator(n, w.device)
    return op


# ---------------------------------------------------------------------------
# structure residuals (laplacian.py:75-126)
# ---------------------------------------------------------------------------
def _residuals(wd: torch.Tensor):
    n = wd.shape[0]
    out = torch.empty(3, dtype=torch.float64, device=wd.device)
    ws = workspace(wd.device, "resid", lib.zt_resid_workspace_bytes(n))
    check(lib.zt_residuals_ws(n, wd.data_ptr(), n, out.data_ptr(), ws.data_ptr(), _stream_ptr(wd.device)))
    return out.tolist()


def skewness_residual(w) -> float:
    """||W + W^H||_F / ||W||_F (laplacian.py:75-96)."""
    wd, _ = _to_device(w)
    return float(_residuals(wd)[0])


def trace_residual(w) -> float:
    """|Tr W| / ||W||_F (laplacian.py:99-104)."""
    wd, _ = _to_device(w)
    return float(_residuals(wd)[1])


def validate_vorticity(w, tol: float = STRUCTURE_TOL) -> None:
    """Raise StructureError unless w is square, skew-Hermitian, traceless."""
    shape = tuple(w.shape)
    if len(shape) != 2 or shape[0] != shape[1]:
        raise StructureError(f"expected a square matrix, got shape {shape}")
    wd, _ = _to_device(w)
    sk, tr, _ = _residuals(wd)
    if sk > tol:
        raise StructureError(f"matrix is not skew-Hermitian: residual {sk:.3e} > {tol:.1e}")
    if tr > tol:
        raise StructureError(f"matrix is not traceless: residual {tr:.3e} > {tol:.1e}")


def spectral_norm(w) -> float:
    """Largest |eigenvalue| of iW (laplacian.py:119-126); init-time only."""
    wd, _ = _to_device(w)
    eigs = torch.linalg.eigvalsh(1j * wd)
    return float(eigs.abs().max())


# ---------------------------------------------------------------------------
# apply / solve
# ---------------------------------------------------------------------------
def apply_laplacian(w, sign: int = -1, op: LaplacianOperator | None = None):
    """Blockwise quantized Laplacian (laplacian.py:341-367); lower triangle read."""
    if sign not in (-1, 1):
        raise ValueError("sign must be -1 or +1")
    wd, as_np = _to_device(w)
    op = _resolve(op, wd)
    n = op.n
    y = torch.empty_like(wd)
    check(lib.zt_apply_laplacian(op.handle, wd.data_ptr(), n, 0, y.data_ptr(), n, 0, sign, 1,
                                 _stream_ptr(wd.device)))
    return _out(y, as_np)


def solve_stream(w, op: LaplacianOperator | None = None, check: bool = True,
                 tol: float = STRUCTURE_TOL, use_jit: bool = True):
    """Solve lap(P) = W in O(N^2) (laplacian.py:370-431).

    ``use_jit`` is accepted and ignored (there is one device path).
    """
    wd, as_np = _to_device(w)
    op = _resolve(op, wd)
    if check:
        sk, tr, _ = _residuals(wd)
        if tr > tol:
            raise StructureError(
                f"input is not traceless (residual {tr:.3e} > {tol:.1e}); "
                "the main-diagonal system is inconsistent"
            )
        if sk > tol:
            raise StructureError(f"input is not skew-Hermitian (residual {sk:.3e} > {tol:.1e})")
    p = _solve_device(wd, op)
    return _out(p, as_np)


def _solve_device(wd: torch.Tensor, op: LaplacianOperator, out: torch.Tensor | None = None):
    n = op.n
    p = torch.empty_like(wd) if out is None else out
    ws = workspace(wd.device, "solve", lib.zt_solve_workspace_bytes(n, 1))
    _lib.check(lib.zt_stream_solve_ws(op.handle, wd.data_ptr(), n, 0, p.data_ptr(), n, 0, 1,
                                      ws.data_ptr(), ws.numel(), _stream_ptr(wd.device)))
    return p


def solve_stream_batched(w: torch.Tensor, op: LaplacianOperator | None = None) -> torch.Tensor:
    """Batched stream solve over a (B, N, N) CUDA tensor (config 2)."""
    if w.dim() != 3 or w.shape[1] != w.shape[2]:
        raise ValueError("expected a (B, N, N) stack")
    w = w.contiguous()
    b = w.shape[0]
    op = _resolve(op, w[0])
    n = op.n
    p = torch.empty_like(w)
    ws = workspace(w.device, "solve_b", lib.zt_solve_workspace_bytes(n, b))
    check(lib.zt_stream_solve_ws(op.handle, w.data_ptr(), n, n * n, p.data_ptr(), n, n * n, b,
                                 ws.data_ptr(), ws.numel(), _stream_ptr(w.device)))
    return p


