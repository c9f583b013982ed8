"""FP64-accurate complex GEMM on the INT8 tensor cores (Ozaki scheme II,
csrc/zt_oz.cu), the step's default product: the tcgen05 kind::i8 residue
GEMM against exact int64 arithmetic, the reconstructed complex128 product
against an extended-precision reference (no less accurate than the native
FP64 DMMA product; componentwise bound per row / column scale), the
skew-Hermitian B layout, the lower-tile mode, NaN / Inf propagation; and
the native DMMA step (ZT_GEMM_ALGO=3m) still matching the reference's cfg 1
run (the step parity tests run on the default path)."""

import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest
import torch
from conftest import ROOT, relf

from oracle import zeitlin_oracle as zo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2206_05466_b200 import _lib

    return _lib.lib


def _moduli(lib):
    buf = (ctypes.c_int * 32)()
    k = lib.zt_oz_moduli(ctypes.cast(buf, ctypes.c_void_p), 32)
    return [buf[i] for i in range(k)]


def _iotas(lib):
    buf = (ctypes.c_int * 32)()
    k = lib.zt_oz_iotas(ctypes.cast(buf, ctypes.c_void_p), 32)
    return [buf[i] for i in range(k)]


def test_moduli_split_gaussian_integers(lib):
    """Every modulus is odd with a square root of -1 (prime factors = 1 mod 4),
    pairwise coprime, product >= 2^124; operand bits KB with 2 K 2^(2 KB) < M / 2:
    55 up to K = 4096, 54 up to K = 2^14."""
    import math

    P, I = _moduli(lib), _iotas(lib)
    assert len(P) == len(I) == 17
    for p, io in zip(P, I):
        assert p % 2 == 1 and p <= 241 and (io * io + 1) % p == 0
    for x in range(len(P)):
        for y in range(x + 1, len(P)):
            assert math.gcd(P[x], P[y]) == 1
    assert sum(math.log2(p) for p in P) >= 124.0
    lg = sum(math.log2(p) for p in P)
    for k, kb in ((256, 56), (2048, 55), (4096, 55), (8192, 54), (16384, 54)):
        assert lib.zt_oz_bits(k) == kb
        assert 1 + math.log2(k) + 2 * kb < lg - 1  # |Re C|, |Im C| <= 2 K 2^(2 KB) < M / 2


@pytest.mark.parametrize("nmod,mp,np_,kp,lower", [(1, 256, 256, 128, 0), (3, 256, 512, 384, 0), (17, 256, 256, 256, 0),
                                                  (2, 512, 512, 256, 1), (4, 768, 768, 128, 1),
                                                  (5, 1024, 1024, 256, 1), (3, 768, 512, 640, 0),
                                                  # odd tile counts, more / fewer tiles than CTA pairs
                                                  (17, 1024, 1280, 256, 0), (17, 1280, 1280, 128, 1),
                                                  (1, 2048, 2048, 128, 0)])
def test_residue_gemm_exact(lib, nmod, mp, np_, kp, lower):
    """R_j = ((U + V) + k_j, (U - V) + k_j) mod p_j with U = A+ B+^T, V = A- B-^T,
    exactly, on the CTA-pair (cta_group::2) tcgen05 kind::i8 kernel; the
    lower mode fills the 256-tiles on or below the diagonal."""
    P = _moduli(lib)
    rng = np.random.default_rng(nmod * 7 + mp)
    a = np.stack([rng.integers(-(P[j] // 2), P[j] // 2 + 1, (2, mp, kp)) for j in range(nmod)]).astype(np.int8)
    b = np.stack([rng.integers(-(P[j] // 2), P[j] // 2 + 1, (2, np_, kp)) for j in range(nmod)]).astype(np.int8)
    dev = torch.device("cuda:0")
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    r = torch.zeros(nmod, 2, mp, np_, dtype=torch.int8, device=dev)
    rc = lib.zt_oz_modgemm(nmod, mp, np_, kp, ad.data_ptr(), bd.data_ptr(), r.data_ptr(), lower,
                           torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    rh = r.cpu().numpy().view(np.uint8).astype(np.int64)
    a64, b64 = a.astype(np.int64), b.astype(np.int64)
    mask = ((np.arange(mp)[:, None] // 256) >= (np.arange(np_)[None, :] // 256)) if lower else np.ones((mp, np_), bool)
    for j in range(nmod):
        p, k = P[j], P[j] // 2
        u = a64[j, 0] @ b64[j, 0].T
        v = a64[j, 1] @ b64[j, 1].T
        for ref, got in ((u + v, rh[j, 0]), (u - v, rh[j, 1])):
            assert np.all((np.mod(ref + k - got, p) == 0)[mask])
            assert np.all((got[mask] >= 0) & (got[mask] < p))


def test_residue_gemm_rejects_bad_shapes(lib):
    s = torch.cuda.current_stream().cuda_stream
    t = torch.zeros(1 << 20, dtype=torch.int8, device="cuda")
    assert lib.zt_oz_modgemm(1, 128, 256, 128, t.data_ptr(), t.data_ptr(), t.data_ptr(), 0, s) != 0
    assert lib.zt_oz_modgemm(18, 256, 256, 128, t.data_ptr(), t.data_ptr(), t.data_ptr(), 0, s) != 0
    assert lib.zt_oz_modgemm(1, 256, 256, 64, t.data_ptr(), t.data_ptr(), t.data_ptr(), 0, s) != 0


def _oz(lib, a, b, bmode=0, lower=0):
    n = a.shape[0]
    ws = torch.empty(lib.zt_oz_workspace_bytes(n), dtype=torch.uint8, device=a.device)
    c = torch.zeros_like(a)
    rc = lib.zt_oz_zgemm(n, a.data_ptr(), n, b.data_ptr(), n, bmode, c.data_ptr(), n, lower, ws.data_ptr(),
                         ws.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert rc == 0
    return c.cpu().numpy()


@pytest.mark.parametrize("n", [5, 130, 256])
def test_complex_product_accuracy(lib, n):
    """relF vs an extended-precision product <= 4e-16 and no worse than the
    native FP64 DMMA product; the skew-B layout gives the same product."""
    from paper_2206_05466_b200.integrator import zgemm

    rng = np.random.default_rng(n)
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    b = zo.random_admissible(n, rng, 1.0 / n)
    b[np.diag_indices(n)] += 1e-3 * rng.normal(size=n)  # the solve's P has a real diagonal part
    ref = (a.astype(np.clongdouble) @ b.astype(np.clongdouble)).astype(np.complex128)
    dev = torch.device("cuda:0")
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    c0, c1 = _oz(lib, ad, bd, 0), _oz(lib, ad, bd, 1)
    native = zgemm(ad, bd).cpu().numpy()
    assert relf(c0, ref) <= 4e-16
    assert relf(c0, ref) <= relf(native, ref) * 1.05
    np.testing.assert_array_equal(c0, c1)
    cl = _oz(lib, ad, bd, 1, lower=1)
    blk = (np.arange(n)[:, None] // 128) >= (np.arange(n)[None, :] // 128)
    np.testing.assert_array_equal(cl[blk], c1[blk])


@pytest.mark.parametrize("n", [2048, 4096])
def test_complex_product_accuracy_full_size(lib, n):
    """The step's sizes: a P X-shaped product (P the solve of a random
    skew-Hermitian field, X skew-Hermitian) at N = 2048 / 4096, checked on 16
    rows against an extended-precision (x87 80-bit) product of those rows:
    relF <= 4e-16 and no worse than the native FP64 DMMA product's rows."""
    from paper_2206_05466_b200.integrator import zgemm

    rng = np.random.default_rng(n + 1)
    x = zo.random_admissible(n, rng, 1.0 / n)
    p = zo.random_admissible(n, rng, 1.0 / n)
    dev = torch.device("cuda:0")
    ad, bd = torch.from_numpy(p).to(dev), torch.from_numpy(x).to(dev)
    c = _oz(lib, ad, bd)
    native = zgemm(ad, bd).cpu().numpy()
    rows = np.sort(rng.choice(n, 16, replace=False))
    ref = (p[rows].astype(np.clongdouble) @ x.astype(np.clongdouble)).astype(np.complex128)
    e_oz, e_dmma = relf(c[rows], ref), relf(native[rows], ref)
    print(f"N={n}: oz relF {e_oz:.2e}, native DMMA {e_dmma:.2e} (16 rows)")
    assert e_oz <= 4e-16
    assert e_oz <= e_dmma * 1.05


def test_zero_and_scaled_inputs(lib):
    """Zero rows/columns (shift 0) stay exact zeros; the power-of-two scaling
    makes the product equivariant to 2^k rescaling of either operand."""
    n = 200
    rng = np.random.default_rng(3)
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    b = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    a[7] = 0
    b[:, 11] = 0
    dev = torch.device("cuda:0")
    c = _oz(lib, torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev))
    assert np.all(c[7] == 0) and np.all(c[:, 11] == 0)
    c2 = _oz(lib, torch.from_numpy(a * 2.0**-300).to(dev), torch.from_numpy(b * 2.0**40).to(dev))
    np.testing.assert_array_equal(c2, c * 2.0**-260)


def test_extreme_row_scales(lib):
    """Rows / columns whose maxima span the whole binary64 range (subnormal to
    ~1e300): the two-factor power-of-two scaling keeps them exact, so each
    scaled row of the product equals the unscaled product row times the same
    power of two (bitwise), and tiny rows far below the rest do not lose
    accuracy (row scaling is per row)."""
    n = 256
    rng = np.random.default_rng(5)
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    b = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    dev = torch.device("cuda:0")
    c = _oz(lib, torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev))
    rows = {3: -1060, 17: -1000, 40: -600, 99: 900, 150: 1000}  # 2^-1060: subnormal entries
    cols = {5: -1000, 77: 980}
    a2, b2 = a.copy(), b.copy()
    for i, e in rows.items():
        a2[i] = a[i] * 2.0**e
    for j, e in cols.items():
        b2[:, j] = b[:, j] * 2.0**e
    c2 = _oz(lib, torch.from_numpy(a2).to(dev), torch.from_numpy(b2).to(dev))
    for i, e in rows.items():
        for j in range(n):
            ej = e + cols.get(j, 0)
            if -1000 <= ej <= 1000 and e > -1060:  # results stay normal: exactly the scaled product
                assert c2[i, j] == c[i, j] * 2.0**ej, (i, j)
    # subnormal inputs: the row is still computed from its own scale (relative accuracy of
    # the subnormal entries themselves, ~2^-1074 absolute)
    ref = (a2[3].astype(np.clongdouble) @ b2.astype(np.clongdouble)).astype(np.complex128)
    sub = np.ones(n, bool)
    sub[77] = False  # column 77 (x 2^980) lifts row 3 back into the normal range
    assert np.abs(c2[3, sub] - ref[sub]).max() <= 2.0**-1072
    assert abs(c2[3, 77] - ref[77]) <= 4e-16 * abs(ref[77])
    fin = np.ones((n, n), bool)
    fin[[99, 150], 77] = False  # 2^1880, 2^1980: the true product overflows (inf, as numpy)
    assert np.all(np.isfinite(c2[fin])) and np.all(np.isinf(c2[~fin]))


def test_native_dmma_step_still_matches_reference():
    """ZT_GEMM_ALGO=3m (native FP64 DMMA products) in a fresh process: cfg 1
    W10 and iteration counts against the reference's golden run."""
    code = (
        "import numpy as np, torch\n"
        "from conftest import load_golden, relf\n"
        "import paper_2206_05466_b200 as zt\n"
        "g = load_golden('cfg1.npz')\n"
        "st = zt.StepperState(w=torch.from_numpy(g['W0']).cuda(), h=0.01)\n"
        "its = []\n"
        "for _ in range(10):\n"
        "    st, info = zt.midpoint_step_info(st)\n"
        "    its.append(info.iterations)\n"
        "assert its == list(g['iters']), its\n"
        "print(relf(st.w.cpu().numpy(), g['W10']))\n"
    )
    env = dict(os.environ, ZT_GEMM_ALGO="3m", PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests")]))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 1e-10


def test_nan_and_inf_propagate(lib):
    """A row of A holding a NaN / a column of B holding an infinity gives a
    NaN row / column of C (as numpy's NaN / inf); every other entry is the
    product of the clean matrices, bitwise (row / column scales are local)."""
    n = 300
    rng = np.random.default_rng(11)
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    b = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    dev = torch.device("cuda:0")
    clean = _oz(lib, torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev))
    a2, b2 = a.copy(), b.copy()
    a2[3, 5] = complex(np.nan, 0.0)
    b2[7, 9] = complex(0.0, np.inf)
    c = _oz(lib, torch.from_numpy(a2).to(dev), torch.from_numpy(b2).to(dev))
    assert np.all(np.isnan(c[3].real)) and np.all(np.isnan(c[3].imag))
    assert np.all(~np.isfinite(c[:, 9]))
    keep = np.ones((n, n), bool)
    keep[3] = False
    keep[:, 9] = False
    np.testing.assert_array_equal(c[keep], clean[keep])
    # skew-B layout and the lower-tile mode flag the same way
    cs = _oz(lib, torch.from_numpy(a2).to(dev), torch.from_numpy(b2).to(dev), bmode=1)
    assert np.all(np.isnan(cs[3].real))


def test_intra_row_dynamic_range_bound(lib):
    """Rows of A whose entries span 1e-20 .. 1 (and columns of B likewise):
    the Ozaki-II product scales each row / column so its largest entry has KB
    integer bits (zt_oz_bits: 56 at K = 256), so an entry is kept to 2^-KB of
    its ROW maximum, not of itself; entries below rowmax * 2^-KB are rounded
    away (native DGEMM keeps them).  The error is therefore bounded per row /
    column,
        |C~ - C|_ij <= sqrt2 2^-KB (rowmax_i(A) sum_k |B_kj| + colmax_j(B) sum_k |A_ik|) + 2u |C_ij|,
    which this test checks entrywise against an extended-precision product,
    together with the normwise error."""
    from paper_2206_05466_b200.integrator import zgemm

    n = 256
    rng = np.random.default_rng(21)
    scale_a = 10.0 ** (-20.0 * rng.random((n, n)))
    scale_b = 10.0 ** (-20.0 * rng.random((n, n)))
    a = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) * scale_a
    b = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) * scale_b
    dev = torch.device("cuda:0")
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    c = _oz(lib, ad, bd)
    ref = (a.astype(np.clongdouble) @ b.astype(np.clongdouble)).astype(np.complex128)
    u = 2.0**-53
    q = 2.0 ** -lib.zt_oz_bits(n)
    rowmax = np.maximum(np.abs(a.real), np.abs(a.imag)).max(axis=1)
    colmax = np.maximum(np.abs(b.real), np.abs(b.imag)).max(axis=0)
    bound = np.sqrt(2) * q * (rowmax[:, None] * np.abs(b).sum(axis=0)[None, :]
                              + colmax[None, :] * np.abs(a).sum(axis=1)[:, None]) * 1.01 + 2 * u * np.abs(ref)
    err = np.abs(c - ref)
    assert np.all(err <= bound), float(np.max(err / bound))
    native = zgemm(ad, bd).cpu().numpy()
    print(f"intra-row range: oz relF {relf(c, ref):.2e}, native DMMA {relf(native, ref):.2e}")
    assert relf(c, ref) <= 2e-15
    assert relf(native, ref) <= 2e-15
