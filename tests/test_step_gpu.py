"""GPU parity of the isospectral step (fixed point + final update) and the
complex128 DMMA GEMM against the oracle and the reference goldens."""

import numpy as np
import pytest
from conftest import relf

from oracle import zeitlin_oracle as zo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def zt():
    import paper_2206_05466_b200 as m

    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


@pytest.mark.parametrize("n", (1, 2, 3, 8, 17, 63, 64, 65, 100, 128, 256, 333))
@pytest.mark.parametrize("algo", (0, 1))
def test_zgemm_vs_numpy(zt, n, algo):
    rng = np.random.default_rng(n)
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    b = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    c = zt.integrator.zgemm(dev(a), dev(b), algo=algo).cpu().numpy()
    assert relf(c, a @ b) <= 1e-14


def test_cfg1_ten_steps_match_reference(zt, golden):
    g = golden("cfg1.npz")
    st = zt.StepperState(w=dev(g["W0"]), h=0.01)
    iters = []
    for s in range(10):
        st, info = zt.midpoint_step_info(st)
        iters.append(info.iterations)
        if s == 0:
            assert relf(st.w.cpu().numpy(), g["W1"]) <= 1e-12
    assert iters == list(g["iters"])
    w = st.w.cpu().numpy()
    assert relf(w, g["W10"]) <= 1e-10
    c = zt.casimirs(st.w, 3)
    c0 = g["casimirs"][0]
    # drift no larger than the reference's (with a round-off floor)
    ref_drift = np.abs(g["casimirs"][-1] - c0)
    assert np.all(np.abs(c[1:] - c0[1:]) <= np.maximum(ref_drift[1:], 1e-13 * np.abs(c0[1:])))
    h = zt.hamiltonian(st.w)
    assert abs(h - g["H"][0]) <= max(abs(g["H"][-1] - g["H"][0]), 1e-13 * abs(g["H"][0]))


def test_cfg4_recipe_n64(zt, golden):
    g = golden("cfg4_n64.npz")
    st = zt.StepperState(w=dev(g["W0"]), h=0.005)
    iters = []
    for _ in range(20):
        st, info = zt.midpoint_step_info(st)
        iters.append(info.iterations)
    assert iters == list(g["iters"])
    assert relf(st.w.cpu().numpy(), g["W20"]) <= 1e-10


def test_zero_step_is_exact(zt):
    w = zo.random_admissible(8, np.random.default_rng(0))
    wt, it = zt.fixed_point_solve(w, h=0.0)
    assert it == 1
    np.testing.assert_array_equal(wt, w)


def test_errors(zt):
    w = zo.random_admissible(8, np.random.default_rng(1))
    with pytest.raises(zt.StructureError):
        zt.fixed_point_solve(w + 0.01 * np.eye(8), h=1e-3)
    with pytest.raises(ValueError):
        zt.fixed_point_solve(w, h=-1.0)
    with pytest.raises(ValueError):
        zt.fixed_point_solve(w, h=1e-3, tol=0.0)
    with pytest.raises(ValueError):
        zt.fixed_point_solve(w, h=1e-3, max_iter=0)
    w16 = zo.random_admissible(16, np.random.default_rng(2))
    w16 /= np.max(np.abs(np.linalg.eigvalsh(1j * w16)))
    with pytest.raises(zt.FixedPointError) as e:
        zt.fixed_point_solve(w16, h=0.05, tol=1e-14, max_iter=1)
    assert e.value.residual > 1e-14 and e.value.iterations == 1


def test_zero_state_and_bookkeeping(zt):
    st = zt.StepperState(w=np.zeros((6, 6), dtype=complex), h=1e-2)
    out = zt.midpoint_step(st)
    assert np.all(out.w == 0.0)
    assert out.step_index == 1 and abs(out.time - 1e-2) < 1e-15


def test_consistency_and_comm_scale(zt):
    w = zo.smooth_initial(12)
    st = zt.StepperState(w=w, h=1e-3, tol=1e-13)
    _, info = zt.midpoint_step_info(st, check_consistency=True)
    assert info.consistency_error <= 1e-12
    a = zt.midpoint_step(zt.StepperState(w=w.copy(), h=1e-3, comm_scale=4.0)).w
    b = zt.midpoint_step(zt.StepperState(w=w.copy(), h=4e-3, comm_scale=1.0)).w
    np.testing.assert_allclose(a, b, atol=1e-14)


# 1024 and 1280 run the fused update with a split-K tail (3 and 2 K-slices on
# 148 SMs: 392 = 2*148 + 96 and 610 = 4*148 + 18 work units)
@pytest.mark.parametrize("n", (200, 512, 1024, 1280))
def test_step_vs_oracle_midsize(zt, n):
    w = zo.smooth_initial(n)
    ref = w
    x = dev(w)
    for _ in range(3):
        ref, kr, _ = zo.midpoint_step(ref, 0.005)
        x, k, _, _ = zt.integrator.midpoint_step_raw(x, 0.005, 1e-12, 10, zt.build_operator(n))
        assert k == kr
    assert relf(x.cpu().numpy(), ref) <= 1e-12


def test_casimirs_match_oracle(zt):
    w = zo.random_admissible(16, np.random.default_rng(3))
    for k in (2, 5, 9):
        np.testing.assert_allclose(zt.casimirs(dev(w), k), zo.casimirs(w, k), rtol=1e-12, atol=1e-12)


def test_cfg4_full_size_steps_vs_oracle(zt):
    """BASELINE cfg 4 at its full size (N = 2048, h = 0.005): 3 steps against
    the oracle — identical iteration counts, relF(W) <= 1e-10, Casimir C2/C3
    and energy drift no larger than the oracle's (floor 1e-13 relative)."""
    n = 2048
    w = zo.smooth_initial(n)
    c0, h0 = zo.casimirs(w, 3), zo.hamiltonian(w)
    x = dev(w)
    c0_gpu, h0_gpu = zt.casimirs(x, 3), zt.hamiltonian(x)
    op = zt.build_operator(n)
    ref = w
    for _ in range(3):
        ref, kr, _ = zo.midpoint_step(ref, 0.005, op=zo.build_operator(n))
        x, k, _, _ = zt.integrator.midpoint_step_raw(x, 0.005, 1e-12, 10, op)
        assert k == kr
    got = x.cpu().numpy()
    assert relf(got, ref) <= 1e-10
    c_ref, c_gpu = zo.casimirs(ref, 3), zt.casimirs(x, 3)
    floor = 1e-13
    for j in (1, 2):  # each run's drift with its own evaluator
        assert abs(c_gpu[j] - c0_gpu[j]) <= max(abs(c_ref[j] - c0[j]), floor * abs(c0[j]))
    assert abs(zt.hamiltonian(x) - h0_gpu) <= max(abs(zo.hamiltonian(ref) - h0), floor * abs(h0))


@pytest.mark.parametrize("n", (2048,))
def test_long_run_structure_full_size(zt, n):
    """Size-independent invariants over 20 device steps at N = 2048: skew and
    trace residuals stay at round-off, C2 (= -||W||_F^2) is conserved."""
    w = zo.smooth_initial(n)
    x = dev(w)
    op = zt.build_operator(n)
    c2_0 = zt.casimirs(x, 2)[1]
    for _ in range(20):
        x, k, _, _ = zt.integrator.midpoint_step_raw(x, 0.005, 1e-12, 10, op)
        assert k == 2
    assert zt.skewness_residual(x) <= 1e-13
    assert zt.trace_residual(x) <= 1e-13
    assert abs(zt.casimirs(x, 2)[1] - c2_0) <= 1e-12 * abs(c2_0)


@pytest.mark.parametrize("n", (2048, 4096, 8192))
def test_cfg3_commutator_and_sandwich_full_size(zt, n):
    """BASELINE cfg 3 at every size it names (P then W from
    random_admissible(N, rng(0), 1/N), h = 0.01) through the DEFAULT product
    (the INT8 Ozaki-II GEMM, as in the step): C = a - a^H and
    S = W - (h/2)(a - a^H) - (h^2/4) a P with a = P W (integrator.py:127-129)
    against numpy/OpenBLAS, relF <= 1e-14; C exactly skew-Hermitian."""
    from paper_2206_05466_b200 import _lib

    h = 0.01
    rng = np.random.default_rng(0)
    pn = zo.random_admissible(n, rng, 1.0 / n)
    wn = zo.random_admissible(n, rng, 1.0 / n)
    P, W = dev(pn), dev(wn)
    C, S, work = torch.empty_like(P), torch.empty_like(P), torch.empty_like(P)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib.zt_commutator(n, P.data_ptr(), W.data_ptr(), C.data_ptr(), work.data_ptr(), s))
    _lib.check(_lib.lib.zt_sandwich(n, P.data_ptr(), W.data_ptr(), h, S.data_ptr(), work.data_ptr(), s))
    a = pn @ wn
    cref = a - a.conj().T
    c = C.cpu().numpy()
    assert relf(c, cref) <= 1e-14
    assert np.array_equal(c, -c.conj().T)
    sref = wn - 0.5 * h * cref - 0.25 * h * h * (a @ pn)
    assert relf(S.cpu().numpy(), sref) <= 1e-14


@pytest.mark.parametrize("n", [5, 64, 130, 1000])
def test_host_result_step_bitwise(n):
    """zt_midpoint_step_host (progressive final update, W_{n+1} copied to the
    host block by block while the last GEMM runs) == the plain step, on the
    host and on the device, step after step; errors still raise (no hang)."""
    from paper_2206_05466_b200 import FixedPointError, build_operator
    from paper_2206_05466_b200.integrator import midpoint_step_raw

    dev = torch.device("cuda:0")
    w0 = torch.from_numpy(zo.random_admissible(n, np.random.default_rng(n), 1.0 / n)).to(dev)
    op = build_operator(n, dev)
    host = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
    x1, x2 = w0, w0.clone()
    for _ in range(3):
        y1, k1, r1, _ = midpoint_step_raw(x1, 0.01, 1e-12, 10, op)
        y2, k2, r2, _ = midpoint_step_raw(x2, 0.01, 1e-12, 10, op, host_out=host)
        assert (k1, r1) == (k2, r2)
        assert torch.equal(y1, y2)
        assert torch.equal(y1.cpu(), host)
        x1, x2 = y1, y2
    with pytest.raises(FixedPointError):
        midpoint_step_raw(x2, 0.5, 1e-14, 1, op, host_out=host)
    # the numpy drop-in goes through it and returns pinned-backed arrays
    from paper_2206_05466_b200 import StepperState, midpoint_step_info

    st, info = midpoint_step_info(StepperState(w=x1.cpu().numpy(), h=0.01))
    assert isinstance(st.w, np.ndarray) and np.array_equal(st.w, midpoint_step_raw(x1, 0.01, 1e-12, 10, op)[0].cpu().numpy())


@pytest.mark.parametrize("n,recipe", [(130, "random"), (300, "smooth"), (1024, "smooth")])
def test_fixed_point_solve_h_positive_vs_oracle(zt, n, recipe):
    """Public fixed_point_solve (integrator.py:96-138) at h > 0: W~ and the
    iteration count against the oracle's fixed point from the same W_n."""
    w = zo.random_admissible(n, np.random.default_rng(n), 1.0 / n) if recipe == "random" else zo.smooth_initial(n)
    h = 0.01 if recipe == "random" else 0.005
    ref, kref = zo.fixed_point_solve(w, h)
    got, k = zt.fixed_point_solve(dev(w), h)
    assert k == kref
    assert relf(got.cpu().numpy(), ref) <= 1e-12
    # numpy in -> numpy out, same numbers
    got_np, k2 = zt.fixed_point_solve(w, h)
    assert k2 == k and isinstance(got_np, np.ndarray)
    np.testing.assert_array_equal(got_np, got.cpu().numpy())


class _ForeignOperator:
    """Duck-typed stand-in for the reference's zeitlin.laplacian.LaplacianOperator
    (host tables only; laplacian.py:179-219): what the unmodified driver passes
    (driver.py:290, 396; diagnostics.py:62)."""

    def __init__(self, n):
        self.n = n
        self._solve_linv = np.zeros((n, n))
        self._solve_dinv = np.zeros((n, n))


def test_foreign_operator_object(zt):
    """The drop-in accepts the reference's own operator object: the driver's
    exact calls midpoint_step_info(state, ref_op) and hamiltonian(w, ref_op)
    with a numpy state give the same numbers as op=None; a size mismatch keeps
    the reference's ValueError text."""
    n = 96
    w = zo.smooth_initial(n)
    op = _ForeignOperator(n)
    st = zt.StepperState(w=w.copy(), h=0.005)
    a, ia = zt.midpoint_step_info(st, op)
    b, ib = zt.midpoint_step_info(st)
    assert ia.iterations == ib.iterations
    np.testing.assert_array_equal(a.w, b.w)
    assert zt.hamiltonian(w, op) == zt.hamiltonian(w)
    np.testing.assert_array_equal(zt.solve_stream(w, op), zt.solve_stream(w))
    np.testing.assert_array_equal(zt.apply_laplacian(w, op=op), zt.apply_laplacian(w))
    wt, k = zt.fixed_point_solve(w, 0.005, op=op)
    assert k == ib.iterations
    with pytest.raises(ValueError, match="does not match"):
        zt.midpoint_step_info(st, _ForeignOperator(n + 1))
    try:  # the real reference class when the reference install travelled with the repo
        import sys
        from conftest import ROOT
        import os

        ref_path = os.path.join(ROOT, "baseline", "_ref")
        if os.path.isdir(os.path.join(ref_path, "zeitlin")) and ref_path not in sys.path:
            sys.path.append(ref_path)
        from zeitlin.laplacian import LaplacianOperator as RefOp
    except Exception:
        return
    np.testing.assert_array_equal(zt.midpoint_step_info(st, RefOp(n))[0].w, b.w)


@pytest.mark.parametrize("n,steps", [(4096, 2), (8192, 1)])
def test_cfg5_sizes_on_default_path_vs_oracle(zt, n, steps):
    """BASELINE cfg 5 sizes (smooth recipe, h = 0.0025) on the default INT8
    product path against the CPU oracle from the same W0: identical iteration
    counts, relF(W) <= 1e-10, Casimir C2/C3 and energy drift no larger than
    the oracle's (floor 1e-13 relative)."""
    w = zo.smooth_initial(n)
    oop = zo.build_operator(n)
    x = dev(w)
    op = zt.build_operator(n)
    # drift of each run measured with its own evaluator (device casimirs /
    # hamiltonian for the GPU run, numpy for the oracle run)
    c0_ref, h0_ref = zo.casimirs(w, 3), zo.hamiltonian(w, op=oop)
    c0_gpu, h0_gpu = zt.casimirs(x, 3), zt.hamiltonian(x)
    ref = w
    for _ in range(steps):
        ref, kr, _ = zo.midpoint_step(ref, 0.0025, op=oop)
        x, k, _, _ = zt.integrator.midpoint_step_raw(x, 0.0025, 1e-12, 10, op)
        assert k == kr
    assert relf(x.cpu().numpy(), ref) <= 1e-10
    c_ref, c_gpu = zo.casimirs(ref, 3), zt.casimirs(x, 3)
    floor = 1e-13
    for j in (1, 2):
        assert abs(c_gpu[j] - c0_gpu[j]) <= max(abs(c_ref[j] - c0_ref[j]), floor * abs(c0_ref[j]))
    h_drift = abs(zt.hamiltonian(x) - h0_gpu)
    assert h_drift <= max(abs(zo.hamiltonian(ref, op=oop) - h0_ref), floor * abs(h0_ref))


def test_eager_and_graph_steps_bitwise(zt):
    """zt_set_graph(0) (eager launches, one read-back per iteration) and the
    CUDA-graph step give bitwise identical W_{n+1}, iterations and residual."""
    from paper_2206_05466_b200 import _lib

    n = 300
    x = dev(zo.smooth_initial(n))
    op = zt.build_operator(n)
    y1, k1, r1, _ = zt.integrator.midpoint_step_raw(x, 0.005, 1e-12, 10, op)
    prev = _lib.lib.zt_set_graph(0)
    try:
        y2, k2, r2, _ = zt.integrator.midpoint_step_raw(x, 0.005, 1e-12, 10, op)
    finally:
        _lib.lib.zt_set_graph(prev)
    assert (k1, r1) == (k2, r2)
    assert torch.equal(y1, y2)


def test_gate_rejects_before_the_fixed_point(zt):
    """A W_n that fails the input gate raises StructureError with the
    reference's text on both the graph and the eager path."""
    n = 64
    w = zo.random_admissible(n, np.random.default_rng(9), 1.0 / n)
    bad = w + 0.01 * np.eye(n)
    op = zt.build_operator(n)
    from paper_2206_05466_b200 import _lib

    for mode in (1, 0):
        prev = _lib.lib.zt_set_graph(mode)
        try:
            with pytest.raises(zt.StructureError, match="traceless|skew"):
                zt.integrator.midpoint_step_raw(dev(bad), 0.005, 1e-12, 10, op)
            y, k, _, _ = zt.integrator.midpoint_step_raw(dev(w), 0.005, 1e-12, 10, op)
            assert k >= 1
        finally:
            _lib.lib.zt_set_graph(prev)


def test_exact_skew_is_preserved_and_not_required(zt):
    """From a W_n that is exactly skew-Hermitian off the diagonal (the
    reference's generator and every solve output are), each step's W_{n+1}
    is exactly skew off the diagonal too (the update and final passes write
    mirror pairs as exact negated conjugates, like the reference's own
    a - a^H); a W_n that is skew only to round-off still matches the oracle."""
    n = 333
    w = zo.smooth_initial(n)
    off = ~np.eye(n, dtype=bool)
    assert np.array_equal(w[off], (-w.conj().T)[off])
    op = zt.build_operator(n)
    x = dev(w)
    ref = w
    for _ in range(3):
        x, k, _, _ = zt.integrator.midpoint_step_raw(x, 0.005, 1e-12, 10, op)
        ref, kr, _ = zo.midpoint_step(ref, 0.005)
        assert k == kr
        got = x.cpu().numpy()
        assert np.array_equal(got[off], (-got.conj().T)[off])
    assert relf(got, ref) <= 1e-12
    # skew to round-off only: perturb a few upper entries by 1e-15 relative
    w2 = w.copy()
    rng = np.random.default_rng(7)
    for _ in range(20):
        i, j = sorted(rng.choice(n, 2, replace=False))
        w2[i, j] += 1e-15 * abs(w2[i, j]) * (1 + 1j)
    assert not np.array_equal(w2[off], (-w2.conj().T)[off])
    y, k2, _, _ = zt.integrator.midpoint_step_raw(dev(w2), 0.005, 1e-12, 10, op)
    ref2, kr2, _ = zo.midpoint_step(w2, 0.005)
    assert k2 == kr2 and relf(y.cpu().numpy(), ref2) <= 1e-12
