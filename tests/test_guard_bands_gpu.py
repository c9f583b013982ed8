"""Out-of-bounds writes through the C ABI (include/zt.h), found without a
sanitizer: every caller-owned output and workspace sits inside a larger
allocation filled with a byte pattern, is given to the library at exactly the
size the header states (workspaces: the *_workspace_bytes value; outputs with
a padded leading dimension and batch stride), and afterwards the guard bands
before and after it, the pad columns of every row and the gaps between batch
entries must still hold the pattern.  Ragged sizes (not multiples of any
tile) as in the reference's known-answer tests (test_laplacian.py:79, 162;
test_acceptance.py:110).  Results are compared with the public Python path
(contiguous buffers) bit for bit, so a padded layout cannot change a value."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import zeitlin_oracle as zo

pytestmark = pytest.mark.gpu

PAT = 0xA5
GUARD = 1 << 16  # bytes on either side (a multiple of the 512 B allocation alignment)
SIZES = [2, 3, 13, 97, 130, 257, 300, 513]


class Guarded:
    """`nbytes` of device memory with pattern-filled bands on both sides."""

    def __init__(self, nbytes, dev, fill=PAT):
        self.nbytes = int(nbytes)
        self.pad = (-self.nbytes) % 16
        self.raw = torch.full((2 * GUARD + self.nbytes + self.pad,), fill, dtype=torch.uint8, device=dev)

    @property
    def ptr(self):
        return self.raw.data_ptr() + GUARD

    def body(self, dtype=torch.uint8):
        return self.raw[GUARD:GUARD + self.nbytes].view(dtype)

    def assert_intact(self, what):
        lo = self.raw[:GUARD]
        hi = self.raw[GUARD + self.nbytes:]
        assert bool((lo == PAT).all()), f"{what}: write before the buffer"
        assert bool((hi == PAT).all()), f"{what}: write past the buffer ({self.nbytes} bytes)"


def matrix_view(g, n, ld, batch=1, stride=None):
    """complex128 views (batch of n x n inside rows of length ld) of a Guarded."""
    stride = n * ld if stride is None else stride
    flat = g.body(torch.complex128)
    return [flat[b * stride:b * stride + n * ld].view(n, ld) for b in range(batch)]


def assert_pads_untouched(g, n, ld, batch, stride, what, cols=None):
    """pad columns [cols, ld) of each of the n rows (cols = n unless given) and
    the gaps between batch entries"""
    cols = n if cols is None else cols
    by = g.body().view(-1, 16)  # one row of 16 bytes per complex element
    mask = torch.ones(by.shape[0], dtype=torch.bool, device=by.device)
    for b in range(batch):
        mask[b * stride:b * stride + n * ld].view(n, ld)[:, :cols] = False
    bad = mask & (by != PAT).any(dim=1)
    assert not bool(bad.any()), f"{what}: pad element {int(bad.nonzero()[0])} overwritten"


@pytest.fixture(scope="module")
def zt():
    import paper_2206_05466_b200 as z

    return z


@pytest.fixture(scope="module")
def lib():
    from paper_2206_05466_b200 import _lib

    return _lib.lib


def _stream(dev):
    return torch.cuda.current_stream(dev).cuda_stream


def _w(n, seed=0, batch=1):
    rng = np.random.default_rng(seed)
    return [zo.random_admissible(n, rng, 1.0 / n) for _ in range(batch)]


@pytest.mark.parametrize("n", SIZES)
def test_solve_and_apply_padded_outputs(zt, lib, n):
    dev = torch.device("cuda:0")
    batch, ld = 2, n + 3
    stride = n * ld + 5
    ws_np = _w(n, 1, batch)
    w = torch.from_numpy(np.stack(ws_np)).to(dev)
    op = zt.build_operator(n, dev)
    out = Guarded(16 * ((batch - 1) * stride + n * ld), dev)
    wsb = lib.zt_solve_workspace_bytes(n, batch)
    ws = Guarded(wsb, dev)
    rc = lib.zt_stream_solve_ws(op.handle, w.data_ptr(), n, n * n, out.ptr, ld, stride, batch, ws.ptr, wsb,
                                _stream(dev))
    assert rc == 0
    torch.cuda.synchronize()
    out.assert_intact("zt_stream_solve_ws output")
    ws.assert_intact("zt_stream_solve_ws workspace")
    assert_pads_untouched(out, n, ld, batch, stride, "zt_stream_solve_ws")
    views = matrix_view(out, n, ld, batch, stride)
    for b in range(batch):
        assert torch.equal(views[b][:, :n], zt.solve_stream(w[b], op, check=False))
    # stencil application, both signs, padded rows
    for sign in (-1, 1):
        y = Guarded(16 * ((batch - 1) * stride + n * ld), dev)
        rc = lib.zt_apply_laplacian(op.handle, w.data_ptr(), n, n * n, y.ptr, ld, stride, sign, batch, _stream(dev))
        assert rc == 0
        torch.cuda.synchronize()
        y.assert_intact("zt_apply_laplacian output")
        assert_pads_untouched(y, n, ld, batch, stride, "zt_apply_laplacian")
        yv = matrix_view(y, n, ld, batch, stride)
        for b in range(batch):
            assert torch.equal(yv[b][:, :n], zt.apply_laplacian(w[b], sign, op))


@pytest.mark.parametrize("n", SIZES)
def test_residuals_exact_workspace(zt, lib, n):
    dev = torch.device("cuda:0")
    w = torch.from_numpy(_w(n, 2)[0]).to(dev)
    out = Guarded(3 * 8, dev)
    wsb = lib.zt_resid_workspace_bytes(n)
    ws = Guarded(wsb, dev)
    assert lib.zt_residuals_ws(n, w.data_ptr(), n, out.ptr, ws.ptr, _stream(dev)) == 0
    torch.cuda.synchronize()
    out.assert_intact("zt_residuals_ws output")
    ws.assert_intact("zt_residuals_ws workspace")
    got = out.body(torch.float64).cpu().numpy()
    assert abs(got[2] - np.linalg.norm(w.cpu().numpy())) <= 1e-13 * got[2]
    assert got[0] <= 1e-14 and got[1] <= 1e-14


@pytest.mark.parametrize("graph", [1, 0])
@pytest.mark.parametrize("n", SIZES)
def test_step_exact_workspace(zt, lib, n, graph):
    dev = torch.device("cuda:0")
    h = 0.01
    w = torch.from_numpy(_w(n, 3)[0]).to(dev)
    op = zt.build_operator(n, dev)
    prev = lib.zt_set_graph(graph)
    try:
        ref_state, info = zt.midpoint_step_info(zt.StepperState(w=w, h=h), op)
        wt_ref, k_ref = zt.fixed_point_solve(w, h, op=op)
        nxt = Guarded(16 * n * n, dev)
        wsb = lib.zt_step_workspace_bytes(n)
        ws = Guarded(wsb, dev)
        it, res, cons = ctypes.c_int(0), ctypes.c_double(0.0), ctypes.c_double(0.0)
        rc = lib.zt_midpoint_step(op.handle, w.data_ptr(), nxt.ptr, h, 1e-12, 10, ws.ptr, wsb, ctypes.byref(it),
                                  ctypes.byref(res), None, _stream(dev))
        assert rc == 0
        torch.cuda.synchronize()
        nxt.assert_intact("zt_midpoint_step output")
        ws.assert_intact("zt_midpoint_step workspace")
        assert it.value == info.iterations
        assert torch.equal(nxt.body(torch.complex128).view(n, n), ref_state.w)
        # with the consistency output (one more epilogue output into the workspace)
        ws2 = Guarded(wsb, dev)
        nxt2 = Guarded(16 * n * n, dev)
        rc = lib.zt_midpoint_step(op.handle, w.data_ptr(), nxt2.ptr, h, 1e-12, 10, ws2.ptr, wsb, ctypes.byref(it),
                                  ctypes.byref(res), ctypes.byref(cons), _stream(dev))
        assert rc == 0
        torch.cuda.synchronize()
        nxt2.assert_intact("zt_midpoint_step (consistency) output")
        ws2.assert_intact("zt_midpoint_step (consistency) workspace")
        assert cons.value <= 1e-12
        # the fixed point alone
        wt = Guarded(16 * n * n, dev)
        ws3 = Guarded(wsb, dev)
        rc = lib.zt_fixed_point(op.handle, w.data_ptr(), wt.ptr, h, 1e-12, 10, ws3.ptr, wsb, ctypes.byref(it),
                                ctypes.byref(res), _stream(dev))
        assert rc == 0
        torch.cuda.synchronize()
        wt.assert_intact("zt_fixed_point output")
        ws3.assert_intact("zt_fixed_point workspace")
        assert it.value == k_ref
        assert torch.equal(wt.body(torch.complex128).view(n, n), wt_ref)
    finally:
        lib.zt_set_graph(prev)


@pytest.mark.parametrize("n", SIZES)
def test_products_padded_outputs(zt, lib, n):
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(4)
    a_np = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    b_np = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    a, b = torch.from_numpy(a_np).to(dev), torch.from_numpy(b_np).to(dev)
    want = a_np @ b_np
    scale = np.abs(a_np) @ np.abs(b_np)
    ld = n + 2
    # the step's default product (INT8 residue GEMM), exact-size workspace
    c = Guarded(16 * n * ld, dev)
    wsb = lib.zt_oz_workspace_bytes(n)
    ws = Guarded(wsb, dev)
    rc = lib.zt_oz_zgemm(n, a.data_ptr(), n, b.data_ptr(), n, 0, c.ptr, ld, 0, ws.ptr, wsb, _stream(dev))
    assert rc == 0
    torch.cuda.synchronize()
    c.assert_intact("zt_oz_zgemm output")
    ws.assert_intact("zt_oz_zgemm workspace")
    assert_pads_untouched(c, n, ld, 1, n * ld, "zt_oz_zgemm")
    got = matrix_view(c, n, ld)[0][:, :n].cpu().numpy()
    assert float(np.max(np.abs(got - want) / scale)) <= 4e-16
    # the native FP64 DMMA product
    for algo in (0, 1):
        c2 = Guarded(16 * n * ld, dev)
        rc = lib.zt_zgemm(n, a.data_ptr(), n, b.data_ptr(), n, c2.ptr, ld, algo, _stream(dev))
        assert rc == 0
        torch.cuda.synchronize()
        c2.assert_intact("zt_zgemm output")
        assert_pads_untouched(c2, n, ld, 1, n * ld, "zt_zgemm")
        got = matrix_view(c2, n, ld)[0][:, :n].cpu().numpy()
        assert float(np.max(np.abs(got - want) / scale)) <= 1e-14


@pytest.mark.parametrize("m,n,nc", [(3, 13, 5), (97, 300, 130), (130, 257, 257), (300, 513, 64)])
def test_oz_building_blocks_exact_buffers(lib, m, n, nc):
    """The sharded step's building blocks (zt_oz_convert_rows / _cols,
    zt_oz_modgemm, zt_oz_reconstruct with its peer scatter and mirror) on
    buffers of exactly the documented sizes: plane sets of
    zt_oz_plane_bytes, pad(rows) shifts, pad(ncols) column-maximum words,
    m x n outputs with padded rows, N x mloc scatter targets."""
    from paper_2206_05466_b200 import _lib

    dev = torch.device("cuda:0")
    s = _stream(dev)
    rng = np.random.default_rng(m * n)
    pad = lambda x: (x + 255) // 256 * 256  # noqa: E731
    A = rng.normal(size=(m, n)) + 1j * rng.normal(size=(m, n))
    X = rng.normal(size=(n, nc)) + 1j * rng.normal(size=(n, nc))
    dA, dX = torch.from_numpy(A).to(dev), torch.from_numpy(X).to(dev)
    kb = lib.zt_oz_bits(n)
    ap, sa = Guarded(lib.zt_oz_plane_bytes(m, n), dev), Guarded(4 * pad(m), dev)
    ap2 = Guarded(lib.zt_oz_plane_bytes(m, n), dev)
    bx, sx, cm = Guarded(lib.zt_oz_plane_bytes(nc, n), dev), Guarded(4 * pad(nc), dev), Guarded(8 * pad(nc), dev)
    _lib.check(lib.zt_oz_convert_rows(m, n, dA.data_ptr(), n, 0, 0, kb, ap.ptr, sa.ptr, None, s))
    _lib.check(lib.zt_oz_convert_cols(n, nc, dX.data_ptr(), nc, kb, bx.ptr, sx.ptr, cm.ptr, s))
    r = Guarded(lib.zt_oz_plane_bytes(m, nc), dev)
    _lib.check(lib.zt_oz_modgemm(17, pad(m), pad(nc), pad(n), ap.ptr, bx.ptr, r.ptr, 0, s))
    ldc, mloc, r0 = nc + 1, 50, 7
    nblk = -(-nc // mloc)
    c = Guarded(16 * m * ldc, dev)
    peers = [Guarded(16 * (r0 + m) * mloc, dev) for _ in range(nblk)]
    ptrs = torch.tensor([t.ptr for t in peers], dtype=torch.int64, device=dev)
    mir = Guarded(16 * nc * (m + 2), dev)
    _lib.check(lib.zt_oz_reconstruct(m, nc, r.ptr, sa.ptr, sx.ptr, c.ptr, ldc, ptrs.data_ptr(), mloc, r0,
                                     mir.ptr, m + 2, 0, s))
    # mode 2 of the row conversion writes two plane sets from one read
    if m == n:
        _lib.check(lib.zt_oz_convert_rows(m, n, dA.data_ptr(), n, 2, 0, kb, ap.ptr, sa.ptr, ap2.ptr, s))
    torch.cuda.synchronize()
    for g, what in ((ap, "A planes"), (sa, "row shifts"), (bx, "B planes"), (sx, "column shifts"),
                    (cm, "column maxima"), (r, "residues"), (c, "C"), (mir, "mirror"), (ap2, "second plane set")):
        g.assert_intact(what)
    for t in peers:
        t.assert_intact("scatter target")
    assert_pads_untouched(c, m, ldc, 1, m * ldc, "zt_oz_reconstruct C", cols=nc)
    assert_pads_untouched(mir, nc, m + 2, 1, nc * (m + 2), "zt_oz_reconstruct mirror", cols=m)
    got = c.body(torch.complex128).view(m, ldc)[:, :nc].cpu().numpy()
    want = A @ X
    assert float(np.max(np.abs(got - want) / (np.abs(A) @ np.abs(X)))) <= 4e-16
    np.testing.assert_array_equal(mir.body(torch.complex128).view(nc, m + 2)[:, :m].cpu().numpy(), -got.conj().T)
    for h, t in enumerate(peers):
        w = min(mloc, nc - h * mloc)
        tv = t.body(torch.complex128).view(r0 + m, mloc)
        np.testing.assert_array_equal(tv[r0:, :w].cpu().numpy(), got[:, h * mloc:h * mloc + w])
        assert bool((t.body().view(r0 + m, mloc * 16)[:r0] == PAT).all()), "rows above r0 overwritten"
        if w < mloc:
            assert bool((t.body().view(r0 + m, mloc, 16)[:, w:] == PAT).all()), "columns past the block overwritten"


def _nan_padded(x, ld, dev):
    """x (rows x cols complex128) inside rows of length ld; every pad element
    and both guard bands are all-ones bytes (NaN as a double): a read outside
    the matrix that reaches a result turns it into NaN."""
    rows, cols = x.shape
    g = Guarded(16 * rows * ld, dev, fill=0xFF)
    g.body(torch.complex128).view(rows, ld)[:, :cols] = x
    return g


@pytest.mark.parametrize("n", SIZES)
def test_inputs_read_inside_their_bounds(zt, lib, n):
    """Inputs with padded leading dimensions whose pads and surroundings are
    NaN: the results equal the contiguous-input results bit for bit (the
    solve and the stencil also ignore a NaN strict upper triangle,
    laplacian.py:370-431 reads the lower triangle only)."""
    dev = torch.device("cuda:0")
    s = _stream(dev)
    op = zt.build_operator(n, dev)
    w = torch.from_numpy(_w(n, 5)[0]).to(dev)
    wl = w.clone()
    wl[torch.triu(torch.ones(n, n, dtype=torch.bool, device=dev), 1)] = complex(float("nan"), float("nan"))
    ld = n + 3
    gw = _nan_padded(wl, ld, dev)
    p = torch.empty_like(w)
    wsb = lib.zt_solve_workspace_bytes(n, 1)
    ws = Guarded(wsb, dev)
    assert lib.zt_stream_solve_ws(op.handle, gw.ptr, ld, 0, p.data_ptr(), n, 0, 1, ws.ptr, wsb, s) == 0
    assert torch.equal(p, zt.solve_stream(w, op, check=False))
    for sign in (-1, 1):
        y = torch.empty_like(w)
        assert lib.zt_apply_laplacian(op.handle, gw.ptr, ld, 0, y.data_ptr(), n, 0, sign, 1, s) == 0
        assert torch.equal(y, zt.apply_laplacian(w, sign, op))
    # residuals of a padded matrix
    gfull = _nan_padded(w, ld, dev)
    out, out2 = torch.empty(3, dtype=torch.float64, device=dev), torch.empty(3, dtype=torch.float64, device=dev)
    assert lib.zt_residuals(n, gfull.ptr, ld, out.data_ptr(), s) == 0
    assert lib.zt_residuals(n, w.data_ptr(), n, out2.data_ptr(), s) == 0
    assert torch.equal(out, out2)
    # products with padded operands
    rng = np.random.default_rng(6)
    a = torch.from_numpy(rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).to(dev)
    b = torch.from_numpy(rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).to(dev)
    ga, gb = _nan_padded(a, n + 1, dev), _nan_padded(b, n + 5, dev)
    wsz = lib.zt_oz_workspace_bytes(n)
    wk = torch.empty(wsz, dtype=torch.uint8, device=dev)
    c1, c2 = torch.empty_like(a), torch.empty_like(a)
    assert lib.zt_oz_zgemm(n, ga.ptr, n + 1, gb.ptr, n + 5, 0, c1.data_ptr(), n, 0, wk.data_ptr(), wsz, s) == 0
    assert lib.zt_oz_zgemm(n, a.data_ptr(), n, b.data_ptr(), n, 0, c2.data_ptr(), n, 0, wk.data_ptr(), wsz, s) == 0
    assert torch.equal(c1, c2)
    for algo in (0, 1):
        assert lib.zt_zgemm(n, ga.ptr, n + 1, gb.ptr, n + 5, c1.data_ptr(), n, algo, s) == 0
        assert lib.zt_zgemm(n, a.data_ptr(), n, b.data_ptr(), n, c2.data_ptr(), n, algo, s) == 0
        assert torch.equal(c1, c2)
