"""Dynamics properties of the device step, mirroring the reference's own
integrator tests (test_integrator.py:89-218) on inputs generated with the
reference's spherical-harmonic basis (tests/golden/modes.npz)."""

import math

import numpy as np
import pytest
from conftest import relf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def zt():
    import paper_2206_05466_b200 as m

    return m


@pytest.fixture(scope="module")
def modes(golden):
    return golden("modes.npz")


@pytest.fixture(scope="module")
def golden():
    from conftest import load_golden

    return load_golden


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def run(zt, w, h, steps, **kw):
    st = zt.StepperState(w=dev(w), h=h, **kw)
    iters = []
    for _ in range(steps):
        st, info = zt.midpoint_step_info(st)
        iters.append(info.iterations)
    return st, iters


@pytest.mark.parametrize("key,h", [("mode_8_4_1", 1e-2), ("mode_9_2_0", 5e-3)])
def test_single_modes_are_steady(zt, modes, key, h):
    w = modes[key]
    st, _ = run(zt, w, h, 1, tol=1e-14, max_iter=60)
    assert np.max(np.abs(st.w.cpu().numpy() - w)) <= 1e-12


def test_isospectrality_200_steps(zt, modes):
    w = modes["norm32"]
    eig0 = np.sort(np.linalg.eigvalsh(1j * w))
    st, _ = run(zt, w, 1e-3, 200, tol=1e-12)
    eig1 = np.sort(np.linalg.eigvalsh(1j * st.w.cpu().numpy()))
    assert np.max(np.abs(eig1 - eig0)) <= 10.0 * 1e-12
    assert zt.skewness_residual(st.w) <= 1e-12
    assert zt.trace_residual(st.w) <= 1e-12


def test_casimir_and_energy_500_steps(zt, modes):
    w = modes["norm16"]
    c0 = zt.casimirs(dev(w), 5)
    h0 = zt.hamiltonian(dev(w))
    st, _ = run(zt, w, 1e-3, 500)
    c1 = zt.casimirs(st.w, 5)
    assert np.max(np.abs(c1[1:] - c0[1:]) / np.abs(c0[1:])) <= 1e-10
    assert abs(zt.hamiltonian(st.w) - h0) / abs(h0) <= 1e-6


def test_quick_convergence_n128(zt, modes):
    _, iters = run(zt, modes["norm128"], 2e-4, 20)
    assert max(iters) <= 3


def test_midpoint_relation(zt, modes):
    st = zt.StepperState(w=dev(modes["norm8"]), h=1e-3, tol=1e-13)
    _, info = zt.midpoint_step_info(st, check_consistency=True)
    assert info.consistency_error <= 1e-12


def test_order_of_accuracy(zt, modes):
    w0 = modes["norm8"]
    horizon = 0.4

    def advance(h):
        st = zt.StepperState(w=dev(w0), h=h, tol=1e-13, max_iter=80)
        for _ in range(round(horizon / h)):
            st = zt.midpoint_step(st)
        return st.w.cpu().numpy()

    ref = advance(horizon / 512)
    hs = [horizon / 8, horizon / 16, horizon / 32]
    errs = [np.linalg.norm(advance(h) - ref) for h in hs]
    slope = np.polyfit(np.log(hs), np.log(errs), 1)[0]
    assert 1.7 <= slope <= 2.3


def test_rigid_rotation_exact_rate(zt, modes):
    """Independent dynamics oracle (test_integrator.py:190-218): a degree-1
    zonal state rotates the (5, 3) mode at rate -a kappa m (1/2 - 1/(l(l+1)))."""
    n, a, eps, l, m = 16, 1.3, 1e-6, 5, 3
    st, _ = run(zt, modes["rot16"], 1e-3, 1000, tol=1e-14, max_iter=60)
    kappa = math.sqrt(12.0 / (n * (n**2 - 1.0)))
    rate = -a * kappa * m * (0.5 - 1.0 / (l * (l + 1.0)))
    w = st.w.cpu().numpy()
    got = np.sum(modes["extract_5_3"] * w)
    want = eps * np.exp(1j * rate * st.time)
    assert abs(np.angle(got / want)) <= 1e-7
    assert abs(abs(got) - eps) / eps <= 1e-12
    # and the state itself against the reference's own 1000-step run
    assert relf(w, modes["rot16_after_1000"]) <= 1e-10
    assert abs(st.time - float(modes["rot16_time"])) <= 1e-12
