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
