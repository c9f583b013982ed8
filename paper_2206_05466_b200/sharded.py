"""Row-block sharded isospectral step over G ranks (BASELINE cfg 5).

The reference is single-process; the paper distributes the dense
products with ScaLAPACK and moves diagonal pieces between ranks for the
stream solve.  On one NVSwitch box the solve is
cheap enough to run redundantly, which removes the diagonal redistribution
(SURVEY.md §8(e)).  Per fixed-point iteration (integrator.py:125-132) rank g,
owning rows R_g (N/G of them) of W_n and of the iterate X:

    X      = all_gather(X_R)                      NCCL all-gather
    P      = lap^{-1} X                          redundant, full (N x N)
    a_R    = P_R X                                local GEMM (N/G x N x N)
    (a^H)_R from the N/G x N/G tiles a[R_j, R_g]  NCCL all-to-all
    X_R'   = W_R + (h/2)(a_R - (a^H)_R) + (h^2/4) a_R P   GEMM + fused epilogue
    r      = all_reduce_max(max|X_R' - X_R|)      NCCL all-reduce (1 double)

and the final update (integrator.py:154-158) is the same with base X_R and
coefficient -(h^2/4).  Every rank takes the identical stop decision.

Compute goes through a backend object; the product backend
(`DeviceBackend`) runs the sm_100a kernels of libzt.so; tests inject a CPU
backend to check the decomposition with gloo on world size 2.
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist


class DeviceBackend:
    """sm_100a kernels through the C ABI (stream solve, rectangular DMMA GEMM,
    row-block update epilogue with residual)."""

    def __init__(self, n: int, device: torch.device):
        from . import _lib
        from .laplacian import _stream_ptr, build_operator, workspace

        self._lib = _lib
        self.n = n
        self.device = device
        self.op = build_operator(n, device)
        self._ws = workspace
        self._stream = _stream_ptr
        self._flag = torch.zeros(1, dtype=torch.int64, device=device)

    def solve(self, x_full: torch.Tensor) -> torch.Tensor:
        from .laplacian import _solve_device

        return _solve_device(x_full, self.op)

    def validate(self, x_full: torch.Tensor) -> None:
        from .laplacian import validate_vorticity

        validate_vorticity(x_full)

    def gemm_rows(self, p_rows: torch.Tensor, x_full: torch.Tensor) -> torch.Tensor:
        m, n = p_rows.shape
        out = torch.empty((m, n), dtype=torch.complex128, device=self.device)
        self._lib.check(self._lib.lib.zt_zgemm_rect(m, n, n, p_rows.data_ptr(), n, x_full.data_ptr(), n,
                                                    out.data_ptr(), n, 0, self._stream(self.device)))
        return out

    def update_rows(self, a_rows, p, ah_rows, base, xprev, hh, qq):
        m, n = a_rows.shape
        out = torch.empty_like(a_rows)
        self._flag.zero_()
        self._lib.check(self._lib.lib.zt_zgemm_update_rows(
            m, n, a_rows.data_ptr(), p.data_ptr(), ah_rows.data_ptr(), base.data_ptr(),
            xprev.data_ptr() if xprev is not None else None, out.data_ptr(), n, hh, qq,
            self._flag.data_ptr(), self._stream(self.device)))
        bits = int(self._flag.item())
        res = torch.tensor([bits], dtype=torch.int64).view(torch.float64).item()
        return out, res


class ShardedStepper:
    """Midpoint step with W distributed by row blocks over `group`."""

    def __init__(self, n: int, backend, group=None, force_collectives: bool = False):
        self.group = group
        # force_collectives: run the NCCL/gloo calls even on one rank (tests)
        self.force = force_collectives and dist.is_initialized()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if n % self.world:
            raise ValueError(f"N={n} must be divisible by the number of ranks {self.world}")
        self.n = n
        self.m = n // self.world
        self.r0 = self.rank * self.m
        self.backend = backend

    # -- collectives -------------------------------------------------------
    def all_gather_rows(self, x_rows: torch.Tensor) -> torch.Tensor:
        if self.world == 1 and not self.force:
            return x_rows
        full = torch.empty((self.n, self.n), dtype=x_rows.dtype, device=x_rows.device)
        dist.all_gather_into_tensor(torch.view_as_real(full), torch.view_as_real(x_rows.contiguous()),
                                    group=self.group)
        return full

    def ah_rows(self, a_rows: torch.Tensor) -> torch.Tensor:
        """Rows R_g of a^H from the tiles a[R_j, R_g] held by every rank j."""
        m, g = self.m, self.world
        if g == 1 and not self.force:
            return a_rows.conj().transpose(0, 1).contiguous()
        send = a_rows.reshape(m, g, m).permute(1, 0, 2).contiguous()  # block j = a[R_g, R_j]
        recv = torch.empty_like(send)
        dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send), group=self.group)
        a_col = recv.reshape(self.n, m)  # a[:, R_g] (block j = a[R_j, R_g])
        return a_col.conj().transpose(0, 1).contiguous()

    def all_reduce_max(self, v: float) -> float:
        if self.world == 1 and not self.force:
            return v
        if v != v:
            v = math.inf  # NaN -> never converged (integrator.py:131 semantics)
        t = torch.tensor([v], dtype=torch.float64, device=self._coll_device())
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def _coll_device(self):
        be = dist.get_backend(self.group)
        return torch.device("cpu") if be == "gloo" else self.backend.device

    # -- one update ---------------------------------------------------------
    def _update(self, x_rows, base_rows, hh, qq, residual: bool, validate: bool = False):
        x_full = self.all_gather_rows(x_rows)
        if validate:
            # input gate of fixed_point_solve (integrator.py:121, laplacian.py:107-116)
            self.backend.validate(x_full)
        p = self.backend.solve(x_full)
        p_rows = p[self.r0:self.r0 + self.m].contiguous()
        a_rows = self.backend.gemm_rows(p_rows, x_full)
        ah = self.ah_rows(a_rows)
        new_rows, res = self.backend.update_rows(a_rows, p, ah, base_rows, x_rows if residual else None, hh, qq)
        return new_rows, res

    def fixed_point(self, w_rows, h, tol=1e-12, max_iter=10):
        """integrator.py:96-138 on row blocks; returns (W~_R, iterations, residual)."""
        if h < 0.0:
            raise ValueError(f"time-step must be nonnegative, got {h}")
        if tol <= 0.0:
            raise ValueError(f"tolerance must be positive, got {tol}")
        if max_iter < 1:
            raise ValueError(f"max_iter must be at least 1, got {max_iter}")
        hh, qq = 0.5 * h, 0.25 * h * h
        x = w_rows
        r = math.inf
        for k in range(1, max_iter + 1):
            x, r_local = self._update(x, w_rows, hh, qq, residual=True, validate=(k == 1))
            r = self.all_reduce_max(r_local)
            if r <= tol:
                return x, k, r
        from .integrator import FixedPointError

        raise FixedPointError(
            f"fixed-point iteration did not reach tol={tol:.1e} in {max_iter} iterations "
            f"(last residual {r:.3e})", residual=r, iterations=max_iter)

    def midpoint_step(self, w_rows, h, tol=1e-12, max_iter=10):
        """integrator.py:141-171 on row blocks: (W_{n+1}_R, iterations, residual)."""
        wt, k, r = self.fixed_point(w_rows, h, tol, max_iter)
        out, _ = self._update(wt, wt, 0.5 * h, -0.25 * h * h, residual=False)
        return out, k, r
