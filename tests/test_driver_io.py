"""ZCK1 checkpoint format compatibility with the reference (formats.py:116-156)
against a file written by the reference's own writer (tests/golden/ck_n8.zck)."""

import os

import numpy as np
import pytest
import torch
from conftest import GOLDEN


def test_reader_parses_reference_checkpoint():
    from paper_2206_05466_b200.driver import read_checkpoint

    cp = read_checkpoint(os.path.join(GOLDEN, "ck_n8.zck"), device="cpu")
    w = np.load(os.path.join(GOLDEN, "ck_n8_w.npy"))
    assert (cp.step_index, cp.time, cp.n, cp.seed, cp.rng_state) == (37, 0.185, 8, 1234, b'{"state": 1}')
    np.testing.assert_array_equal(cp.w.numpy(), w)


def test_writer_is_byte_identical_to_reference(tmp_path):
    from paper_2206_05466_b200.driver import Checkpoint, write_checkpoint

    w = torch.from_numpy(np.load(os.path.join(GOLDEN, "ck_n8_w.npy")))
    path = tmp_path / "x.zck"
    write_checkpoint(path, Checkpoint(37, 0.185, 8, 1234, b'{"state": 1}', w))
    assert path.read_bytes() == open(os.path.join(GOLDEN, "ck_n8.zck"), "rb").read()


def test_reader_rejects_corruption(tmp_path):
    from paper_2206_05466_b200.driver import FileFormatError, read_checkpoint

    raw = open(os.path.join(GOLDEN, "ck_n8.zck"), "rb").read()
    for bad in (b"ZCK2" + raw[4:], raw[:-1], raw + b"\0"):
        p = tmp_path / "bad.zck"
        p.write_bytes(bad)
        with pytest.raises(FileFormatError):
            read_checkpoint(p, device="cpu")


def test_basis_cache_matches_reference_format(tmp_path):
    """ZEB1 basis cache (formats.py:83-113): a file written by the reference's
    save_basis parses to its vectors, and writing them back is byte-identical."""
    from paper_2206_05466_b200.basis import load_basis, save_basis
    from paper_2206_05466_b200.driver import FileFormatError

    src = os.path.join(GOLDEN, "basis_n5.zeb")
    b = load_basis(src, device="cpu")
    g = np.load(os.path.join(GOLDEN, "basis.npz"))
    np.testing.assert_array_equal(b.data.numpy(), g["vec_5"])
    out = tmp_path / "b.zeb"
    save_basis(out, b)
    assert out.read_bytes() == open(src, "rb").read()
    raw = open(src, "rb").read()
    for bad in (b"ZEB2" + raw[4:], raw[:-8], raw + b"\0"):
        p = tmp_path / "bad.zeb"
        p.write_bytes(bad)
        with pytest.raises(FileFormatError):
            load_basis(p, device="cpu")


def test_grid_snapshot_matches_reference_format(tmp_path):
    """ZGD1 grid files (formats.py:163-181) both ways."""
    from paper_2206_05466_b200.driver import FileFormatError, read_grid, write_grid

    src = os.path.join(GOLDEN, "grid_n16.zgd")
    field, t = read_grid(src)
    np.testing.assert_array_equal(field, np.load(os.path.join(GOLDEN, "grids.npz"))["grid_16"])
    assert t == 0.375
    out = tmp_path / "g.zgd"
    write_grid(out, field, t)
    assert out.read_bytes() == open(src, "rb").read()
    raw = open(src, "rb").read()
    for bad in (b"ZGD2" + raw[4:], raw[:-8], raw + b"\0"):
        p = tmp_path / "bad.zgd"
        p.write_bytes(bad)
        with pytest.raises(FileFormatError):
            read_grid(p)


@pytest.mark.parametrize("kwargs", [
    dict(n=1, steps=1), dict(n=8, steps=-1), dict(n=8, steps=1, h=0.0), dict(n=8, steps=1, l_min=1),
    dict(n=8, steps=1, l_max=8), dict(n=8, steps=1, l_min=6, l_max=5), dict(n=8, steps=1, tol=0.0),
    dict(n=8, steps=1, max_iter=0), dict(n=8, steps=1, sample_every=0), dict(n=8, steps=1, k_max=1),
    dict(n=8, steps=1, seed=-1), dict(n=8, steps=1, comm_scale=0.0), dict(n=8, steps=1, threads=-1),
])
def test_simconfig_validate_rejects(kwargs):
    """test_driver.py:91-109 (driver.py:97-122)."""
    from paper_2206_05466_b200.driver import ConfigError, SimConfig

    with pytest.raises(ConfigError):
        SimConfig(**{"l_max": 5, **kwargs}).validate()
    SimConfig(n=8, steps=1, l_max=5).validate()


def test_invalid_config_exits_2(tmp_path):
    """test_driver.py:111-113: validation precedes any device work."""
    from paper_2206_05466_b200.driver import EXIT_CONFIG, SimConfig, run

    assert run(SimConfig(n=8, steps=1, l_max=20, output_dir=str(tmp_path))) == EXIT_CONFIG
    assert not any(tmp_path.iterdir())


def test_casimir_drift_records():
    """diagnostics.py:86-110: relative drift against the first entry, absolute
    below the 1e-14 baseline floor (flagged)."""
    from paper_2206_05466_b200 import DiagnosticsRecord, casimir_drift

    assert casimir_drift([]) == []
    c0 = np.array([0.0, -2.0, 1e-16, 4.0])
    recs = casimir_drift([(0.0, c0), (0.5, np.array([0.0, -2.0 + 2e-12, 3e-16, 4.0]))])
    assert all(isinstance(r, DiagnosticsRecord) for r in recs)
    assert recs[1].time == 0.5 and recs[1].casimir_abs_fallback == (3,)
    np.testing.assert_allclose(recs[1].casimir_rel_err, [1e-12, 2e-16, 0.0], rtol=1e-3, atol=1e-30)
    np.testing.assert_array_equal(recs[0].casimir_rel_err, [0.0, 0.0, 0.0])
    with pytest.raises(ValueError):
        casimir_drift([(0.0, np.array([1.0]))])
