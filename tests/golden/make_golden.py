"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src); the outputs are committed as small .npz fixtures so
the GPU box, which has no /root/reference, can check against them:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Contents (all complex128 C-order unless noted):
  solve_small.npz   per N in SOLVE_NS: W (random_admissible, seed 1000+N),
                    P = solve_stream(W), A = apply_laplacian(W) (sign -1),
                    plus the reference operator's factor tables at N=17
  cfg1.npz          BASELINE cfg 1: N=128, W0 = random_admissible(128,
                    default_rng(0), 1/128), h=0.01, 10 steps: W1, W10,
                    iterations per step, fixed-point residual traces of step 1,
                    casimirs(w,3) and hamiltonian at every step
  cfg4_n64.npz      cfg 4 recipe at N=64 (smooth W0, h=0.005), 20 steps: W20,
                    per-step iterations, C2/C3/H series
  known.npz         known answers: pinv-oracle P at N=5, casimirs of
                    i*diag(1,-1,0,0), blocks N=2 m=0 / N=3 m=1
  basis.npz         per N in BASIS_NS: reference basis vectors (all m, the
                    QuantizedBasis layout, concatenated), extract of
                    random_admissible(N, default_rng(500+N), 1) (packed pos/neg),
                    its energy spectrum, project of random real coefficients
                    (test_basis.py:20-32 generator, default_rng(700+N))
  grids.npz         diagnostics.evaluate_on_grid of random real coefficients at
                    (N, n_lat, n_lon, l_max) = (16, 9, 14, -), (40, 33, 64, 20),
                    (100, 50, 80, 99)
  init.npz          driver.random_initial_condition(SimConfig(n, seed, l_min,
                    l_max), compute_basis(n)) at N = 9, 12, 16 (oracle-aligned)
  modes.npz         inputs of the reference's integrator property tests
                    (test_integrator.py) built with its spherical-harmonic basis
                    (out of scope here): single modes (N=8 l=4 m=1, N=9 l=2 m=0),
                    normalized states (N=32, N=16, N=8, N=128), the rigid-rotation
                    state (N=16) and the basis matrix T_{5,3} used to extract the
                    advected coefficient, plus the reference's own results
  runs.npz          driver.run(SimConfig(...)) output directories for the
                    test_driver.py configurations RUNS (text of diagnostics.csv,
                    run_meta.json and the final spectrum csv as uint8 arrays,
                    the final checkpoint's W and the final grid field)
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from conftest import casimir_laplacian_dense, random_admissible  # noqa: E402
from zeitlin import diagnostics, integrator, laplacian  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SOLVE_NS = (2, 3, 5, 8, 17, 40, 64, 97)


def solve_small():
    d = {}
    for n in SOLVE_NS:
        w = random_admissible(n, np.random.default_rng(1000 + n), 1.0 / n)
        d[f"W_{n}"] = w
        d[f"P_{n}"] = laplacian.solve_stream(w)
        d[f"A_{n}"] = laplacian.apply_laplacian(w)
        d[f"Ap_{n}"] = laplacian.apply_laplacian(w, sign=1)
    op = laplacian.build_operator(17)
    d["linv_17"] = op._solve_linv
    d["dinv_17"] = op._solve_dinv
    d["sdiag_17"] = op._stencil_diag
    d["soff_17"] = op._stencil_off
    np.savez_compressed(os.path.join(OUT, "solve_small.npz"), **d)


def run_steps(w0, h, steps, keep=()):
    st = integrator.StepperState(w=w0.copy(), h=h)
    iters, c, hh, kept = [], [], [], {}
    c.append(integrator.casimirs(st.w, 3))
    hh.append(diagnostics.hamiltonian(st.w))
    for s in range(1, steps + 1):
        st, info = integrator.midpoint_step_info(st)
        iters.append(info.iterations)
        c.append(integrator.casimirs(st.w, 3))
        hh.append(diagnostics.hamiltonian(st.w))
        if s in keep:
            kept[s] = st.w.copy()
    return st, np.array(iters), np.array(c), np.array(hh), kept


def fp_trace(w0, h):
    """Residuals of every fixed-point iterate, by re-running with max_iter=k."""
    res = []
    for k in range(1, 11):
        try:
            integrator.fixed_point_solve(w0, h, max_iter=k)
            break
        except integrator.FixedPointError as e:
            res.append(e.residual)
    return np.array(res)


def cfg1():
    n = 128
    w0 = random_admissible(n, np.random.default_rng(0), 1.0 / n)
    st, iters, c, hh, kept = run_steps(w0, 0.01, 10, keep=(1,))
    np.savez_compressed(
        os.path.join(OUT, "cfg1.npz"),
        W0=w0, W1=kept[1], W10=st.w, iters=iters, casimirs=c, H=hh,
        fp_residuals_step1=fp_trace(w0, 0.01),
    )


def cfg4_n64():
    n = 64
    r = random_admissible(n, np.random.default_rng(0), 1.0 / n)
    w0 = laplacian.solve_stream(r)
    w0 /= np.linalg.norm(w0)
    st, iters, c, hh, _ = run_steps(w0, 0.005, 20)
    np.savez_compressed(
        os.path.join(OUT, "cfg4_n64.npz"), W0=w0, W20=st.w, iters=iters, casimirs=c, H=hh
    )


def known():
    n = 5
    w = random_admissible(n, np.random.default_rng(5), 1.0)
    basis = np.eye(n * n, dtype=complex).reshape(n * n, n, n)
    op_dense = np.stack([casimir_laplacian_dense(e).ravel() for e in basis], axis=1)
    p_pinv = (np.linalg.pinv(op_dense) @ w.ravel()).reshape(n, n)
    wd = 1j * np.diag([1.0, -1.0, 0.0, 0.0]).astype(complex)
    b20 = laplacian.build_block(2, 0)
    b31 = laplacian.build_block(3, 1)
    np.savez_compressed(
        os.path.join(OUT, "known.npz"),
        W5=w, P5_pinv=p_pinv, P5_ref=laplacian.solve_stream(w),
        casimir_diag=integrator.casimirs(wd, 4),
        b20_diag=b20.diag, b20_off=b20.offdiag, b31_diag=b31.diag, b31_off=b31.offdiag,
    )


def modes():
    from test_basis import random_real_field_coeffs
    from zeitlin.basis import HarmonicCoefficients, compute_basis, extract, project

    def single(n, l, m, amp):
        c = HarmonicCoefficients.zeros(n)
        c.set(l, m, amp)
        c.enforce_reality()
        return project(c, compute_basis(n))

    def normalized(n, seed, l_hi=None):
        rng = np.random.default_rng(seed)
        c = random_real_field_coeffs(n, rng, l_lo=2, l_hi=l_hi or min(n - 2, 10))
        w = project(c, compute_basis(n))
        return w / laplacian.spectral_norm(w)

    d = {}
    d["mode_8_4_1"] = single(8, 4, 1, 0.9 - 0.3j)
    d["mode_9_2_0"] = single(9, 2, 0, 1.1)
    d["norm32"] = normalized(32, 11)
    d["norm16"] = normalized(16, 12)
    d["norm8"] = normalized(8, 13, l_hi=4)
    d["norm128"] = normalized(128, 14, l_hi=20)
    # rigid rotation (test_integrator.py:190-218)
    n = 16
    basis = compute_basis(n)
    c = HarmonicCoefficients.zeros(n)
    c.set(1, 0, 1.3)
    c.set(5, 3, 1e-6)
    c.enforce_reality()
    w = project(c, basis)
    d["rot16"] = w
    # T_{5,3}: the coefficient is Tr(T^H W) for the trace-orthonormal basis;
    # recover the linear functional by probing extract with unit matrices
    f = np.zeros((n, n), dtype=complex)
    for i in range(n):
        for j in range(n):
            e = np.zeros((n, n), dtype=complex)
            e[i, j] = 1.0
            f[i, j] = extract(e, basis).get(5, 3)
    d["extract_5_3"] = f  # coefficient = sum(f * W)
    st = integrator.StepperState(w=w.copy(), h=1e-3, tol=1e-14, max_iter=60)
    for _ in range(1000):
        st = integrator.midpoint_step(st)
    d["rot16_after_1000"] = st.w
    d["rot16_time"] = np.array(st.time)
    np.savez_compressed(os.path.join(OUT, "modes.npz"), **d)


BASIS_NS = (2, 3, 5, 8, 9, 16, 17, 33, 48)


def basis():
    """Reference basis vectors (sign rule / oracle alignment), extract of an
    admissible W, project of real coefficients, energy spectrum (basis.py)."""
    from test_basis import random_real_field_coeffs
    from zeitlin.basis import compute_basis, extract, project
    from zeitlin.diagnostics import energy_spectrum

    d = {}
    for n in BASIS_NS:
        b = compute_basis(n)
        d[f"vec_{n}"] = np.concatenate([v.ravel() for v in b.vectors])
        w = random_admissible(n, np.random.default_rng(500 + n), 1.0)
        c = extract(w, b)
        d[f"W_{n}"] = w
        d[f"pos_{n}"] = np.concatenate(c.pos)
        d[f"neg_{n}"] = np.concatenate(c.neg)
        d[f"E_{n}"] = energy_spectrum(c)
        cr = random_real_field_coeffs(n, np.random.default_rng(700 + n))
        d[f"cpos_{n}"] = np.concatenate(cr.pos)
        d[f"cneg_{n}"] = np.concatenate(cr.neg)
        d[f"P_{n}"] = project(cr, b)
    np.savez_compressed(os.path.join(OUT, "basis.npz"), **d)
    from zeitlin.basis import save_basis

    save_basis(os.path.join(OUT, "basis_n5.zeb"), compute_basis(5))  # formats.py:83-89


def initial_conditions():
    """driver.random_initial_condition at oracle-aligned sizes (basis signs match)."""
    from zeitlin.basis import compute_basis
    from zeitlin.driver import SimConfig, random_initial_condition

    d = {}
    for n, seed, lo, hi in ((12, 5, 2, 6), (16, 20260809, 1, 15), (9, 3, 2, 8)):
        cfg = SimConfig(n=n, steps=0, seed=seed, l_min=lo, l_max=hi)
        d[f"W_{n}_{seed}_{lo}_{hi}"] = random_initial_condition(cfg, compute_basis(n))
    np.savez_compressed(os.path.join(OUT, "init.npz"), **d)


def grids():
    """diagnostics.evaluate_on_grid of random real coefficients (input pinned)."""
    from test_basis import random_real_field_coeffs
    from zeitlin.diagnostics import evaluate_on_grid

    d = {}
    for n, nlat, nlon, lmax in ((16, 9, 14, None), (40, 33, 64, 20), (100, 50, 80, 99)):
        c = random_real_field_coeffs(n, np.random.default_rng(900 + n))
        d[f"pos_{n}"] = np.concatenate(c.pos)
        d[f"neg_{n}"] = np.concatenate(c.neg)
        d[f"grid_{n}"] = evaluate_on_grid(c, nlat, nlon, l_max=lmax)
    np.savez_compressed(os.path.join(OUT, "grids.npz"), **d)
    from zeitlin.formats import write_grid

    write_grid(os.path.join(OUT, "grid_n16.zgd"), d["grid_16"], 0.375)  # formats.py:163-168


def checkpoint():
    """A ZCK1 file written by the reference's own writer (formats.py:130-143)."""
    from zeitlin.formats import Checkpoint, write_checkpoint

    w = random_admissible(8, np.random.default_rng(8), 0.5)
    cp = Checkpoint(step_index=37, time=0.185, n=8, seed=1234, rng_state=b'{"state": 1}', w=w)
    write_checkpoint(os.path.join(OUT, "ck_n8.zck"), cp)
    np.save(os.path.join(OUT, "ck_n8_w.npy"), w)


#: (name, SimConfig kwargs): test_driver.py:176-248 configurations
RUNS = (
    ("resume", dict(n=12, steps=40, h=1e-3, l_min=2, l_max=6, sample_every=10, checkpoint_every=20, seed=7)),
    ("auto_h", dict(n=8, steps=2, l_max=5, seed=1)),
    ("cadence", dict(n=8, steps=25, h=1e-3, l_max=5, sample_every=10, checkpoint_every=20, seed=1)),
    ("grid", dict(n=10, steps=5, h=1e-3, l_max=6, sample_every=5, seed=4)),
)


def runs():
    """The reference's run loop end to end (driver.py:259-410)."""
    import tempfile
    from pathlib import Path

    from zeitlin.driver import SimConfig, run
    from zeitlin.formats import read_checkpoint, read_grid

    d = {}
    for name, kw in RUNS:
        with tempfile.TemporaryDirectory() as tmp:
            assert run(SimConfig(output_dir=tmp, **kw)) == 0
            out, last = Path(tmp), kw["steps"]
            for key, fname in (("diag", "diagnostics.csv"), ("meta", "run_meta.json"),
                               ("spec", f"spectrum_{last:08d}.csv")):
                d[f"{name}_{key}"] = np.frombuffer((out / fname).read_bytes(), dtype=np.uint8)
            d[f"{name}_w"] = read_checkpoint(out / f"checkpoint_{last:08d}.zck").w
            d[f"{name}_grid"], _ = read_grid(out / f"grid_{last:08d}.bin")
    np.savez_compressed(os.path.join(OUT, "runs.npz"), **d)


if __name__ == "__main__":
    runs()
    grids()
    initial_conditions()
    basis()
    checkpoint()
    modes()
    solve_small()
    cfg1()
    cfg4_n64()
    known()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
