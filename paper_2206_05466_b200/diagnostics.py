"""Sample-time parity meters on device (diagnostics.py:60-63 of the reference)."""

from __future__ import annotations

import torch

from .laplacian import LaplacianOperator, _to_device, solve_stream


def hamiltonian(w, op: LaplacianOperator | None = None) -> float:
    """H = -1/2 Re Tr(W^H P), P = lap^{-1} W (diagnostics.py:60-63)."""
    wd, _ = _to_device(w)
    p = solve_stream(wd, op)
    return -0.5 * float(torch.vdot(wd.reshape(-1), p.reshape(-1)).real)
