"""Pin the CPU oracle against golden vectors produced by the reference itself.

The goldens come from tests/golden/make_golden.py (runs the reference
``zeitlin`` package from /root/reference).  These checks make the oracle a
trusted checker for the GPU parity tests.
"""

import numpy as np
import pytest
from conftest import load_golden, relf

from oracle import zeitlin_oracle as zo

SOLVE_NS = (2, 3, 5, 8, 17, 40, 64, 97)


@pytest.mark.parametrize("n", SOLVE_NS)
def test_solve_and_apply_match_reference(n, golden):
    g = golden("solve_small.npz")
    w = g[f"W_{n}"]
    assert relf(zo.solve_stream(w), g[f"P_{n}"]) <= 1e-14
    # the stencil is evaluated in the reference's exact operation order
    np.testing.assert_array_equal(zo.apply_laplacian(w), g[f"A_{n}"])
    np.testing.assert_array_equal(zo.apply_laplacian(w, sign=1), g[f"Ap_{n}"])


def test_operator_tables_bit_identical(golden):
    g = golden("solve_small.npz")
    op = zo.OracleOperator(17)
    np.testing.assert_array_equal(op.linv, g["linv_17"])
    np.testing.assert_array_equal(op.dinv, g["dinv_17"])
    np.testing.assert_array_equal(op.stencil_diag, g["sdiag_17"])
    np.testing.assert_array_equal(op.stencil_off, g["soff_17"])


def test_known_answers(golden):
    k = golden("known.npz")
    assert np.max(np.abs(zo.solve_stream(k["W5"]) - k["P5_pinv"])) <= 1e-11
    np.testing.assert_allclose(k["casimir_diag"], [0.0, -2.0, 0.0, 2.0], atol=1e-15)
    wd = 1j * np.diag([1.0, -1.0, 0.0, 0.0]).astype(complex)
    np.testing.assert_allclose(zo.casimirs(wd, 4), k["casimir_diag"], atol=1e-15)
    d, o = zo.block_entries(2, 0)
    np.testing.assert_array_equal(d, k["b20_diag"])
    np.testing.assert_array_equal(o, k["b20_off"])
    d, o = zo.block_entries(3, 1)
    np.testing.assert_array_equal(d, k["b31_diag"])
    np.testing.assert_array_equal(o, k["b31_off"])  # sqrt(2)*sqrt(2), 1 ulp off -2


def test_cfg1_steps_match_reference(golden):
    g = golden("cfg1.npz")
    w = g["W0"]
    w0 = zo.random_admissible(128, np.random.default_rng(0), 1.0 / 128)
    np.testing.assert_array_equal(w, w0)  # generator reproducible here
    iters = []
    for s in range(10):
        w, k, _ = zo.midpoint_step(w, 0.01)
        iters.append(k)
        if s == 0:
            assert relf(w, g["W1"]) <= 1e-14
    assert iters == list(g["iters"])
    assert relf(w, g["W10"]) <= 1e-13
    np.testing.assert_allclose(zo.casimirs(w, 3), g["casimirs"][-1], rtol=1e-12, atol=1e-15)
    assert abs(zo.hamiltonian(w) - g["H"][-1]) <= 1e-14 * abs(g["H"][-1])


def test_cfg4_recipe_n64_matches_reference(golden):
    g = golden("cfg4_n64.npz")
    w = zo.smooth_initial(64)
    assert relf(w, g["W0"]) <= 1e-14
    iters = []
    for _ in range(20):
        w, k, _ = zo.midpoint_step(w, 0.005)
        iters.append(k)
    assert iters == list(g["iters"])
    assert relf(w, g["W20"]) <= 1e-12


def test_fixed_point_residual_trace(golden):
    g = golden("cfg1.npz")
    tr = []
    zo.fixed_point_solve(g["W0"], 0.01, trace=tr)
    ref = g["fp_residuals_step1"]
    np.testing.assert_allclose(tr[: len(ref)], ref, rtol=1e-6)


def test_oracle_errors():
    w = zo.random_admissible(8, np.random.default_rng(3))
    with pytest.raises(zo.OracleStructureError):
        zo.solve_stream(w + 1e-3j * np.eye(8))
    with pytest.raises(ValueError, match="does not match"):
        zo.apply_laplacian(w, op=zo.build_operator(6))
    with pytest.raises(zo.OracleFixedPointError) as e:
        zo.fixed_point_solve(w / 4, 0.05, tol=1e-14, max_iter=1)
    assert e.value.iterations == 1 and e.value.residual > 1e-14


def test_closed_form_ldlt_matches_dpttrf():
    """The pivots of every m >= 1 block are the integers (k+m+1)(N-1-k) and
    L_k = -sqrt((N-1-k-m)(k+1) / ((k+m+1)(N-1-k))): the GPU solve uses this
    closed form; LAPACK dpttrf (laplacian.py:208) reproduces it to rounding."""
    import scipy.linalg.lapack as lapack

    for n in (17, 128, 512):
        for m in range(1, n - 1):
            dm, em = zo.block_entries(n, m)
            d, e, info = lapack.dpttrf(dm, em)
            k = np.arange(n - m, dtype=np.float64)
            np.testing.assert_allclose(d, (k + m + 1) * (n - 1 - k), rtol=4e-15)
            kk = k[:-1]
            lex = -np.sqrt((n - 1 - kk - m) / (kk + m + 1)) * np.sqrt((kk + 1) / (n - 1 - kk))
            np.testing.assert_allclose(e, lex, rtol=4e-15)


def _split_vectors(flat, n):
    out, off = [], 0
    for m in range(n):
        sz = (n - m) * (n - max(m, 1))
        out.append(flat[off:off + sz].reshape(n - m, n - max(m, 1)))
        off += sz
    return out


@pytest.mark.parametrize("n", (2, 3, 5, 8, 9, 16, 17, 33, 48))
def test_basis_oracle_pinned(n):
    """The basis restatement reproduces the reference's vectors bit for bit
    (3j-aligned signs at n <= 16, the sign rule above), and extract/project
    its transforms (basis.py:119-165, 276-331)."""
    g = load_golden("basis.npz")
    ref = _split_vectors(g[f"vec_{n}"], n)
    mine = zo.basis_vectors(n)
    if n > 16:
        for a, b in zip(mine, ref):
            np.testing.assert_array_equal(a, b)
    mine = zo.align_with(mine, ref)
    for a, b in zip(mine, ref):
        np.testing.assert_array_equal(a, b)
    p, q = zo.extract(g[f"W_{n}"], ref)
    np.testing.assert_array_equal(p, g[f"pos_{n}"])
    np.testing.assert_array_equal(q, g[f"neg_{n}"])
    np.testing.assert_array_equal(zo.project(g[f"cpos_{n}"], g[f"cneg_{n}"], ref), g[f"P_{n}"])


@pytest.mark.parametrize("n,h", ((64, 0.005), (128, 0.01), (256, 0.005)))
def test_final_update_identity(n, h):
    """The device step's final update W_n + h (a - a^H) (zt_api.cu final_update)
    equals the reference's sandwich form W~ + (h/2)(a - a^H) - (h^2/4) a P~
    (integrator.py:154-158) at the converged fixed point: the (h^2/4) a P
    terms cancel; what remains is the fixed point's last correction times
    h |P|, below round-off at these tolerances."""
    w = zo.smooth_initial(n)
    op = zo.build_operator(n)
    wt, k = zo.fixed_point_solve(w, h, op=op)
    p = zo.solve_stream(wt, op, check=False)  # W~ is traceless only to ~1e-8
    a = p @ wt
    sandwich = wt + 0.5 * h * (a - a.conj().T) - 0.25 * h * h * (a @ p)
    comm = w + h * (a - a.conj().T)
    assert relf(comm, sandwich) <= 1e-15


def test_bench_arms_print_the_same_config():
    """bench.py: both arms' `config` is the workload description only
    (identical dicts, so a driver comparing them sees the same workload)."""
    import bench

    a = bench.bench_config([2, 2, 2])
    b = bench.bench_config([2])
    assert a == b
    assert set(a) == {"workload", "N", "h", "tol", "max_iter", "init", "iterations_per_step"}


def test_bench_stdout_is_one_json_line(tmp_path):
    """bench.py's stdout carries exactly one JSON line even when a library
    writes to fd 1 during the run (NCCL prints its version banner there when
    the box sets NCCL_DEBUG): claim_stdout() points fd 1 at stderr and emit()
    writes the line to the original stdout."""
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import os, sys; sys.argv = ['bench.py']; sys.path.insert(0, %r)\n"
        "import bench\n"
        "bench.claim_stdout()\n"
        "os.write(1, b'NCCL version 0.0.0+test\\n')\n"
        "print('a library notice')\n"
        "bench.emit({'metric': 'm', 'value': 1.5})\n" % ROOT
    )
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert len(lines) == 1 and __import__("json").loads(lines[0]) == {"metric": "m", "value": 1.5}
    assert "NCCL version 0.0.0+test" in r.stderr and "a library notice" in r.stderr
