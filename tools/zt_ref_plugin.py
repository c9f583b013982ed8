"""pytest plugin: run the reference's OWN test files, unmodified, against the
B200 drop-in (SURVEY.md §8(b) "Behavioural contract").

Loaded with ``-p zt_ref_plugin`` so it is imported before collection; it
imports the reference package ``zeitlin`` (installed under baseline/_ref by
tools/stage_reference.sh, which also stages the reference's tests there) and
rebinds the hot-path names to ``paper_2206_05466_b200`` — the module
attributes and the names other reference modules bound at import time
(diagnostics.py:27, driver.py:38-45), exactly what INTEGRATION.md §2 tells a
maintainer to do.  Basis, formats, CLI and the driver loop stay the
reference's CPU code; only the per-step path runs on the GPU.

    PYTHONPATH=baseline/_ref:baseline/_ref/zeitlin_tests:tools:. \\
        python -m pytest -p zt_ref_plugin baseline/_ref/zeitlin_tests/test_laplacian.py ...
"""

from __future__ import annotations

import zeitlin.diagnostics as D
import zeitlin.driver as R
import zeitlin.integrator as I
import zeitlin.laplacian as L

import paper_2206_05466_b200 as zt

CALLS: dict[str, int] = {}


def _counted(name, fn):
    def wrapper(*args, **kwargs):
        CALLS[name] = CALLS.get(name, 0) + 1
        return fn(*args, **kwargs)

    wrapper.__name__ = getattr(fn, "__name__", name)
    wrapper.__doc__ = fn.__doc__
    return wrapper


# cached per (N, device) like the reference's (laplacian.py:319-322); the
# reference's tests check `build_operator(16) is build_operator(16)`
_build_operator = _counted("build_operator", zt.build_operator)
_solve_stream = _counted("solve_stream", zt.solve_stream)
_apply = _counted("apply_laplacian", zt.apply_laplacian)
_fps = _counted("fixed_point_solve", zt.fixed_point_solve)
_msi = _counted("midpoint_step_info", zt.midpoint_step_info)
_ms = _counted("midpoint_step", zt.midpoint_step)

PATCHES = [
    (L, "build_operator", _build_operator),
    (L, "solve_stream", _solve_stream),
    (L, "apply_laplacian", _apply),
    (L, "validate_vorticity", zt.validate_vorticity),
    (L, "skewness_residual", zt.skewness_residual),
    (L, "trace_residual", zt.trace_residual),
    (L, "StructureError", zt.StructureError),
    (I, "solve_stream", _solve_stream),
    (I, "validate_vorticity", zt.validate_vorticity),
    (I, "fixed_point_solve", _fps),
    (I, "midpoint_step_info", _msi),
    (I, "midpoint_step", _ms),
    (I, "FixedPointError", zt.FixedPointError),
    (I, "casimirs", _counted("casimirs", zt.casimirs)),
    (D, "solve_stream", _solve_stream),
    (R, "midpoint_step_info", _msi),
    (R, "build_operator", _build_operator),
    (R, "FixedPointError", zt.FixedPointError),
]
for mod, name, fn in PATCHES:
    setattr(mod, name, fn)


def pytest_report_header(config):
    return "zt_ref_plugin: zeitlin hot path rebound to paper_2206_05466_b200 (sm_100a)"


def pytest_terminal_summary(terminalreporter):
    calls = ", ".join(f"{k}={v}" for k, v in sorted(CALLS.items()))
    terminalreporter.write_line(f"zt_ref_plugin intercepted calls: {calls}")


def pytest_configure(config):
    # the reference registers these in its pyproject.toml (pkg/pyproject.toml:27-31)
    config.addinivalue_line("markers", "slow: long-running conservation and scaling runs")
    config.addinivalue_line("markers", "acceptance: top-level acceptance criteria")
