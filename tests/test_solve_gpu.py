"""GPU parity of the stream solve / apply / residual kernels vs the oracle
(itself pinned to the reference) and the reference's golden vectors."""

import numpy as np
import pytest
from conftest import relf

from oracle import zeitlin_oracle as zo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SOLVE_NS = (2, 3, 5, 8, 17, 40, 64, 97)


@pytest.fixture(scope="module")
def zt():
    import paper_2206_05466_b200 as m

    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


@pytest.mark.parametrize("n", SOLVE_NS)
def test_solve_matches_reference_golden(zt, golden, n):
    g = golden("solve_small.npz")
    p = zt.solve_stream(dev(g[f"W_{n}"])).cpu().numpy()
    assert relf(p, g[f"P_{n}"]) <= 1e-13


@pytest.mark.parametrize("n", SOLVE_NS)
def test_apply_bit_identical_to_reference(zt, golden, n):
    g = golden("solve_small.npz")
    w = dev(g[f"W_{n}"])
    np.testing.assert_array_equal(zt.apply_laplacian(w).cpu().numpy(), g[f"A_{n}"])
    np.testing.assert_array_equal(zt.apply_laplacian(w, sign=1).cpu().numpy(), g[f"Ap_{n}"])


def test_operator_factors_bit_identical_to_dpttrf(zt, golden):
    g = golden("solve_small.npz")
    linv, dinv = zt.build_operator(17).factors()
    np.testing.assert_array_equal(linv, g["linv_17"])
    np.testing.assert_array_equal(dinv, g["dinv_17"])


@pytest.mark.parametrize("n", (31, 32, 33, 63, 64, 65, 96, 127, 128, 129, 200, 256, 300, 513))
def test_solve_vs_oracle_ragged_sizes(zt, n):
    w = zo.random_admissible(n, np.random.default_rng(n), 1.0 / n)
    p = zt.solve_stream(dev(w)).cpu().numpy()
    assert relf(p, zo.solve_stream(w)) <= 1e-13
    a = zt.apply_laplacian(dev(w)).cpu().numpy()
    np.testing.assert_array_equal(a, zo.apply_laplacian(w))


@pytest.mark.parametrize("n", (16, 64, 128, 1000))
def test_roundtrip(zt, n):
    w = dev(zo.random_admissible(n, np.random.default_rng(7 + n)))
    p = zt.solve_stream(w)
    assert (torch.linalg.norm(zt.apply_laplacian(p) - w) / torch.linalg.norm(w)).item() <= 1e-10
    w2 = zt.solve_stream(zt.apply_laplacian(w))
    assert (torch.linalg.norm(w2 - w) / torch.linalg.norm(w)).item() <= 1e-10


def test_zero_and_structure(zt):
    z = torch.zeros(5, 5, dtype=torch.complex128, device="cuda")
    assert bool((zt.solve_stream(z) == 0).all())
    assert bool((zt.apply_laplacian(torch.zeros(6, 6, dtype=torch.complex128, device="cuda")) == 0).all())
    w = dev(zo.random_admissible(32, np.random.default_rng(1)))
    p = zt.solve_stream(w)
    assert zt.skewness_residual(p) <= 1e-12
    assert zt.trace_residual(p) <= 1e-12


def test_gates_and_errors(zt):
    w = zo.random_admissible(8, np.random.default_rng(2))
    with pytest.raises(zt.StructureError, match="traceless"):
        zt.solve_stream(dev(w + 1e-3j * np.eye(8)))
    p = zt.solve_stream(dev(w + 1e-3j * np.eye(8)), check=False)
    assert zt.trace_residual(p) <= 1e-12
    w2 = w.copy()
    w2[2, 3] += 0.1
    with pytest.raises(zt.StructureError, match="skew"):
        zt.solve_stream(dev(w2))
    with pytest.raises(ValueError, match="does not match"):
        zt.apply_laplacian(dev(zo.random_admissible(5, np.random.default_rng(0))), op=zt.build_operator(6))
    with pytest.raises(ValueError, match="square"):
        zt.apply_laplacian(torch.zeros(3, 4, dtype=torch.complex128, device="cuda"))
    with pytest.raises(ValueError):
        zt.apply_laplacian(dev(w), sign=2)
    assert zt.build_operator(16) is zt.build_operator(16)


def test_apply_reads_lower_triangle_only(zt):
    rng = np.random.default_rng(9)
    w = zo.random_admissible(9, rng)
    c = w.copy()
    c[np.triu_indices(9, k=1)] = rng.normal(size=36)
    np.testing.assert_array_equal(zt.apply_laplacian(dev(w)).cpu().numpy(),
                                  zt.apply_laplacian(dev(c)).cpu().numpy())
    np.testing.assert_array_equal(zt.solve_stream(dev(w)).cpu().numpy(),
                                  zt.solve_stream(dev(c), check=False).cpu().numpy())


def test_numpy_in_numpy_out(zt):
    w = zo.random_admissible(12, np.random.default_rng(4))
    p = zt.solve_stream(w)
    assert isinstance(p, np.ndarray)
    assert relf(p, zo.solve_stream(w)) <= 1e-13


def test_residuals_match_oracle(zt):
    w = zo.random_admissible(100, np.random.default_rng(5))
    w2 = w + 1e-6 * np.random.default_rng(6).normal(size=w.shape)
    for x in (w, w2, w + 1e-4j * np.eye(100)):
        assert abs(zt.skewness_residual(dev(x)) - zo.skewness_residual(x)) <= 1e-12 * max(1, zo.skewness_residual(x))
        assert abs(zt.trace_residual(dev(x)) - zo.trace_residual(x)) <= 1e-14 + 1e-12 * zo.trace_residual(x)


@pytest.mark.parametrize("n", (1024,))
def test_batched_solve_cfg2_shape(zt, n):
    rng = np.random.default_rng(0)
    ws = [zo.random_admissible(n, rng, 1.0 / n) for _ in range(3)]
    p = zt.solve_stream_batched(dev(np.stack(ws))).cpu().numpy()
    for k in range(3):
        assert relf(p[k], zo.solve_stream(ws[k])) <= 1e-12


@pytest.mark.parametrize("n", (2048, 4096))
def test_cfg2_full_size_batch(zt, n):
    """BASELINE cfg 2 at full size: 8 successive random_admissible(N, rng(0),
    1/N) draws.  Matrix 0 against the oracle; every matrix through the
    size-independent round trip lap(P) = W (test_laplacian.py:116-124) and
    bit-identical to its own single-matrix solve."""
    rng = np.random.default_rng(0)
    ws = np.stack([zo.random_admissible(n, rng, 1.0 / n) for _ in range(8)])
    wd = dev(ws)
    op = zt.build_operator(n)
    p = zt.solve_stream_batched(wd, op)
    assert relf(p[0].cpu().numpy(), zo.solve_stream(ws[0])) <= 1e-12
    for k in range(8):
        back = zt.apply_laplacian(p[k], op=op)
        assert float((back - wd[k]).norm() / wd[k].norm()) <= 1e-10
        if k in (0, 7):
            assert torch.equal(zt.solve_stream(wd[k], op), p[k])
    del p, wd
    torch.cuda.empty_cache()
