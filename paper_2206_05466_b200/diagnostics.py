"""Sample-time parity meters on device (diagnostics.py:60-63 of the reference)
and the reference's drift records (diagnostics.py:36-110; host arithmetic on
the k_max Casimir values, which come from the device)."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .laplacian import LaplacianOperator, _to_device, solve_stream


def hamiltonian(w, op: LaplacianOperator | None = None) -> float:
    """H = -1/2 Re Tr(W^H P), P = lap^{-1} W (diagnostics.py:60-63)."""
    wd, _ = _to_device(w)
    p = solve_stream(wd, op)
    return -0.5 * float(torch.vdot(wd.reshape(-1), p.reshape(-1)).real)


#: diagnostics.py:38-40: baselines below this are treated as zero and the
#: drift for that Casimir is reported as an absolute error (flagged).
CASIMIR_BASELINE_FLOOR = 1e-14


@dataclass
class DiagnosticsRecord:
    """diagnostics.py:43-57: one sample of the conserved-quantity diagnostics;
    ``casimir_rel_err[j]`` is |C_k(t) - C_k(0)| / |C_k(0)| for k = j + 2 (the
    absolute error for k in ``casimir_abs_fallback``)."""

    time: float
    casimir_rel_err: np.ndarray | None = None
    casimir_abs_fallback: tuple[int, ...] = ()
    hamiltonian: float | None = None
    mean_energy: float | None = None
    spectrum: np.ndarray | None = field(default=None, repr=False)


def _drift(base: np.ndarray, ck) -> np.ndarray:
    denom = np.where(np.abs(base) < CASIMIR_BASELINE_FLOOR, 1.0, np.abs(base))
    return np.abs(np.asarray(ck, dtype=np.float64)[1:] - base) / denom


def casimir_drift(series) -> list[DiagnosticsRecord]:
    """diagnostics.py:86-110: drift of C_2..C_kmax against the first entry of
    a [(time, casimirs(w, k_max)), ...] series."""
    if not series:
        return []
    _, c0 = series[0]
    c0 = np.asarray(c0, dtype=np.float64)
    if c0.size < 2:
        raise ValueError("series must carry Casimirs up to k >= 2")
    base = c0[1:]
    fallback = tuple(k + 2 for k in np.flatnonzero(np.abs(base) < CASIMIR_BASELINE_FLOOR))
    return [DiagnosticsRecord(time=t, casimir_rel_err=_drift(base, ck), casimir_abs_fallback=fallback)
            for t, ck in series]
