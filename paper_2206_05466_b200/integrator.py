"""Isospectral midpoint integrator on B200: drop-in for ``zeitlin.integrator``.

Same names, arguments, error types and bookkeeping as the reference
(/root/reference/pkg/src/zeitlin/integrator.py:34-210).  The whole fixed
point — stream solves, the two complex128 products per update (3M DMMA
GEMMs, the second one only on the lower triangle because a P = P X P is
skew-Hermitian), the commutator update and the entrywise residual max —
stays in HBM and runs as sm_100a kernels behind ``zt_fixed_point`` /
``zt_midpoint_step``; the host reads back one 8-byte residual per iteration
to take the same stop decision as integrator.py:129-132.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from ._lib import lib
from .laplacian import (
    LaplacianOperator,
    StructureError,
    _resolve,
    _stream_ptr,
    _to_device,
    _out,
    solve_stream,
    spectral_norm,
    workspace,
)

__all__ = [
    "StepperState",
    "StepInfo",
    "FixedPointError",
    "fixed_point_solve",
    "midpoint_step",
    "midpoint_step_info",
    "casimirs",
    "casimirs_from_spectrum",
    "commutator_scale",
    "default_time_step",
]


class FixedPointError(RuntimeError):
    """The inner iteration failed to reach tolerance (integrator.py:48-54)."""

    def __init__(self, message: str, residual: float, iterations: int):
        super().__init__(message)
        self.residual = residual
        self.iterations = iterations


@dataclass
class StepperState:
    """One simulation state (integrator.py:57-72); ``w`` may be a CUDA tensor."""

    w: object
    h: float
    time: float = 0.0
    step_index: int = 0
    tol: float = 1e-12
    max_iter: int = 10
    comm_scale: float = 1.0


@dataclass
class StepInfo:
    iterations: int
    consistency_error: float | None = None
    residual: float | None = None


def commutator_scale(n: int) -> float:
    """n^{3/2} / sqrt(16 pi) (integrator.py:81-83)."""
    return n**1.5 / math.sqrt(16.0 * math.pi)


def default_time_step(w, op: LaplacianOperator | None = None) -> float:
    """0.1 / ||lap^{-1} W||_2 (integrator.py:86-93)."""
    p_norm = spectral_norm(solve_stream(w, op))
    if p_norm == 0.0:
        return 0.1
    return 0.1 / p_norm


def _params(h, tol, max_iter):
    if h < 0.0:
        raise ValueError(f"time-step must be nonnegative, got {h}")
    if tol <= 0.0:
        raise ValueError(f"tolerance must be positive, got {tol}")
    if max_iter < 1:
        raise ValueError(f"max_iter must be at least 1, got {max_iter}")


def _step_ws(op: LaplacianOperator, device: torch.device) -> torch.Tensor:
    return workspace(device, "step", lib.zt_step_workspace_bytes(op.n))


def _raise(rc: int, iters: int, residual: float):
    if rc == _lib.ZT_ENOCONV:
        raise FixedPointError(_lib.last_error(), residual=residual, iterations=iters)
    _lib.check(rc, structure_error=StructureError)


def fixed_point_solve(w_n, h: float, tol: float = 1e-12, max_iter: int = 10,
                      op: LaplacianOperator | None = None):
    """Solve the implicit midpoint relation for W~ (integrator.py:96-138)."""
    _params(h, tol, max_iter)
    wd, as_np = _to_device(w_n)
    op = _resolve(op, wd)
    wt = torch.empty_like(wd)
    ws = _step_ws(op, wd.device)
    it, res = ctypes.c_int(0), ctypes.c_double(0.0)
    rc = lib.zt_fixed_point(op.handle, wd.data_ptr(), wt.data_ptr(), float(h), float(tol), int(max_iter),
                            ws.data_ptr(), ws.numel(), ctypes.byref(it), ctypes.byref(res),
                            _stream_ptr(wd.device))
    if rc:
        _raise(rc, it.value, res.value)
    return _out(wt, as_np), it.value


def midpoint_step_raw(w: torch.Tensor, h_eff: float, tol: float, max_iter: int,
                      op: LaplacianOperator, out: torch.Tensor | None = None,
                      check_consistency: bool = False, host_out: torch.Tensor | None = None):
    """Device fast path: W_{n+1} into ``out`` (fresh if None); returns
    (w_next, iterations, last_residual, consistency).  ``host_out`` (pinned
    CPU complex128, N x N) also receives W_{n+1}, copied block by block while
    the step's last GEMM still runs (zt_midpoint_step_host)."""
    w_next = torch.empty_like(w) if out is None else out
    ws = _step_ws(op, w.device)
    it, res, cons = ctypes.c_int(0), ctypes.c_double(0.0), ctypes.c_double(0.0)
    if host_out is not None and not check_consistency:
        if host_out.shape != w.shape or host_out.dtype != torch.complex128 or host_out.is_cuda:
            raise ValueError("host_out must be a CPU complex128 tensor shaped like w")
        rc = lib.zt_midpoint_step_host(op.handle, w.data_ptr(), w_next.data_ptr(), host_out.data_ptr(),
                                       float(h_eff), float(tol), int(max_iter), ws.data_ptr(), ws.numel(),
                                       ctypes.byref(it), ctypes.byref(res), _stream_ptr(w.device))
        if rc:
            _raise(rc, it.value, res.value)
        return w_next, it.value, res.value, None
    rc = lib.zt_midpoint_step(op.handle, w.data_ptr(), w_next.data_ptr(), float(h_eff), float(tol),
                              int(max_iter), ws.data_ptr(), ws.numel(), ctypes.byref(it),
                              ctypes.byref(res), ctypes.byref(cons) if check_consistency else None,
                              _stream_ptr(w.device))
    if rc:
        _raise(rc, it.value, res.value)
    return w_next, it.value, res.value, (cons.value if check_consistency else None)


def midpoint_step_info(state: StepperState, op: LaplacianOperator | None = None,
                       check_consistency: bool = False):
    """Advance one step; report inner-iteration statistics (integrator.py:141-171)."""
    h = state.h * state.comm_scale
    _params(h, state.tol, state.max_iter)
    wd, as_np = _to_device(state.w)
    op = _resolve(op, wd)
    if as_np and not check_consistency:
        # numpy in, numpy out: W_{n+1} lands in a pinned block (torch's caching
        # host allocator) through the overlapped block copies
        host = torch.empty(wd.shape, dtype=torch.complex128, pin_memory=True)
        _, iters, res, cons = midpoint_step_raw(wd, h, state.tol, state.max_iter, op, host_out=host)
        w_out = host.numpy()
    else:
        w_next, iters, res, cons = midpoint_step_raw(wd, h, state.tol, state.max_iter, op,
                                                     check_consistency=check_consistency)
        w_out = _out(w_next, as_np)
    new_state = replace(
        state,
        w=w_out,
        time=state.time + state.h,
        step_index=state.step_index + 1,
    )
    return new_state, StepInfo(iterations=iters, consistency_error=cons, residual=res)


def midpoint_step(state: StepperState, op: LaplacianOperator | None = None) -> StepperState:
    """Advance the state by one step (integrator.py:174-177)."""
    new_state, _ = midpoint_step_info(state, op)
    return new_state


def zgemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None, algo: int = 0):
    """C = A @ B on the sm_100a DMMA kernel (complex128, square)."""
    n = a.shape[0]
    c = torch.empty_like(a) if out is None else out
    _lib.check(lib.zt_zgemm(n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, algo,
                            _stream_ptr(a.device)))
    return c


def casimirs(w, k_max: int) -> np.ndarray:
    """Tr(W^k) as reals, k = 1..k_max (integrator.py:180-210), on device."""
    wd, _ = _to_device(w)
    n = wd.shape[0]
    if not 1 <= k_max <= n:
        raise ValueError(f"k_max={k_max} out of range 1..{n}")
    half = (k_max + 1) // 2
    powers = [wd]
    for _ in range(half - 1):
        powers.append(zgemm(powers[-1], wd))
    out = np.empty(k_max)
    for k in range(1, k_max + 1):
        if k == 1:
            t = complex(torch.diagonal(wd).sum().item())
        else:
            a, b = (k + 1) // 2, k // 2
            t = complex((powers[a - 1] * powers[b - 1].T).sum().item())
        out[k - 1] = t.real if k % 2 == 0 else ((-1j) ** k * t).real
    return out


def casimirs_from_spectrum(eigenvalues, k_max: int) -> np.ndarray:
    """integrator.py:213-220."""
    eigs = np.asarray(eigenvalues, dtype=np.complex128)
    out = np.empty(k_max)
    for k in range(1, k_max + 1):
        t = np.sum(eigs**k)
        out[k - 1] = t.real if k % 2 == 0 else ((-1j) ** k * t).real
    return out
