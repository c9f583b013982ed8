"""B200-native isospectral time-step hot path (arXiv 2206.05466).

Drop-in for the reference package's step / stream-solve API
(/root/reference/pkg/src/zeitlin/__init__.py:27-48): the same names, backed
by hand-written sm_100a kernels in ``libzt.so`` (C ABI: include/zt.h).
"""

from .basis import (
    DeviceBasis,
    HarmonicCoefficients,
    QuantizedBasis,
    compute_basis,
    energy_spectrum,
    evaluate_on_grid,
    extract,
    hamiltonian_from_coeffs,
    load_basis,
    project,
    save_basis,
    threej,
    wigner_basis_oracle,
)
from .diagnostics import CASIMIR_BASELINE_FLOOR, DiagnosticsRecord, casimir_drift, hamiltonian
from .driver import (
    EXIT_CONFIG,
    EXIT_IO,
    EXIT_OK,
    EXIT_SOLVER,
    Checkpoint,
    ConfigError,
    DeviceRun,
    FileFormatError,
    SimConfig,
    SolverError,
    random_initial_condition,
    read_checkpoint,
    read_grid,
    write_checkpoint,
    run,
    write_grid,
)
from .integrator import (
    FixedPointError,
    StepInfo,
    StepperState,
    casimirs,
    casimirs_from_spectrum,
    commutator_scale,
    default_time_step,
    fixed_point_solve,
    midpoint_step,
    midpoint_step_info,
)
from .laplacian import (
    LaplacianBlock,
    LaplacianOperator,
    StructureError,
    apply_laplacian,
    build_block,
    build_operator,
    skewness_residual,
    solve_stream,
    solve_stream_batched,
    spectral_norm,
    trace_residual,
    validate_vorticity,
)

__all__ = [
    "FixedPointError", "StepInfo", "StepperState", "casimirs", "casimirs_from_spectrum",
    "commutator_scale", "default_time_step", "fixed_point_solve", "midpoint_step",
    "midpoint_step_info", "LaplacianBlock", "LaplacianOperator", "StructureError",
    "apply_laplacian", "build_block", "build_operator", "skewness_residual", "solve_stream",
    "solve_stream_batched", "spectral_norm", "trace_residual", "validate_vorticity", "hamiltonian",
    "Checkpoint", "DeviceRun", "FileFormatError", "read_checkpoint", "write_checkpoint",
    "DeviceBasis", "HarmonicCoefficients", "QuantizedBasis", "compute_basis", "energy_spectrum", "extract",
    "hamiltonian_from_coeffs", "load_basis", "project", "save_basis", "threej", "wigner_basis_oracle",
    "evaluate_on_grid", "random_initial_condition", "read_grid", "write_grid",
    "CASIMIR_BASELINE_FLOOR", "DiagnosticsRecord", "casimir_drift", "EXIT_OK", "EXIT_CONFIG", "EXIT_SOLVER",
    "EXIT_IO", "ConfigError", "SimConfig", "SolverError", "run",
]
