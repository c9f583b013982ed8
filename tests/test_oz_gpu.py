"""FP64-accurate complex GEMM on the INT8 tensor cores (Ozaki scheme II,
csrc/zt_oz.cu), the step's default product: the tcgen05 kind::i8 residue
GEMM against exact int64 arithmetic, the reconstructed complex128 product
against an extended-precision reference (no less accurate than the native
FP64 DMMA product), the skew-Hermitian B layout and the lower-tile mode; and
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


@pytest.mark.parametrize("nmod,mp,np_,kp,lower", [(1, 128, 256, 64, 0), (3, 256, 512, 320, 0), (16, 256, 256, 256, 0),
                                                  (2, 512, 512, 192, 1), (4, 768, 768, 128, 1),
                                                  (5, 1024, 1024, 256, 1), (3, 768, 512, 448, 0)])
@pytest.mark.parametrize("cta", [1, 2])
def test_residue_gemm_exact(lib, nmod, mp, np_, kp, lower, cta):
    """R_j = (A_re B_re^T + A_-im B_im^T, A_re B_im^T + A_im B_re^T) + p_j // 2 mod p_j, exactly,
    for the single-CTA 128 x 256 kernel and the CTA-pair (cta_group::2) kernel (Re and Im as
    separate 256 x 256 real tiles with K doubled)."""
    assert lib.zt_oz_set_cta(cta) == 0
    try:
        _check_residue_gemm(lib, nmod, mp, np_, kp, lower)
    finally:
        lib.zt_oz_set_cta(0)


def test_set_cta_rejects_bad_values(lib):
    assert lib.zt_oz_set_cta(3) != 0
    assert lib.zt_oz_set_cta(-1) != 0


def _check_residue_gemm(lib, nmod, mp, np_, kp, lower):
    P = _moduli(lib)
    rng = np.random.default_rng(nmod * 7 + mp)
    a = np.stack([rng.integers(-(P[j] // 2), P[j] // 2 + 1, (3, mp, kp)) for j in range(nmod)]).astype(np.int8)
    b = np.stack([rng.integers(-(P[j] // 2), P[j] // 2 + 1, (2, np_, kp)) for j in range(nmod)]).astype(np.int8)
    dev = torch.device("cuda:0")
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    r = torch.zeros(nmod, 2, mp, np_, dtype=torch.int8, device=dev)
    rc = lib.zt_oz_modgemm(nmod, mp, np_, kp, ad.data_ptr(), bd.data_ptr(), r.data_ptr(), lower,
                           torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    rh = r.cpu().numpy().view(np.uint8).astype(np.int64)
    a64, b64 = a.astype(np.int64), b.astype(np.int64)
    mask = ((np.arange(mp)[:, None] // 128) >= (np.arange(np_)[None, :] // 128)) if lower else np.ones((mp, np_), bool)
    for j in range(nmod):
        re = a64[j, 0] @ b64[j, 0].T + a64[j, 2] @ b64[j, 1].T
        im = a64[j, 0] @ b64[j, 1].T + a64[j, 1] @ b64[j, 0].T
        for ref, got in ((re, rh[j, 0]), (im, rh[j, 1])):
            # epilogue residues: (product + p // 2) mod p as unsigned bytes in [0, p)
            assert np.all((np.mod(ref + P[j] // 2 - got, P[j]) == 0)[mask])
            assert np.all((got[mask] >= 0) & (got[mask] < P[j]))


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
