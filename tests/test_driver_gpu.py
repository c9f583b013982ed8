"""Device run loop: sample/checkpoint cadence, parity of the checkpointed state
with the reference run (cfg 4 recipe at N=64), and the resume contract of
/root/reference/pkg/tests/test_driver.py:231-248 (a run resumed from a
checkpoint reproduces the uninterrupted run byte for byte)."""

import json

import numpy as np
import pytest
import torch
from conftest import load_golden, relf

pytestmark = pytest.mark.gpu


def _run(out, w0, steps, **kw):
    from paper_2206_05466_b200 import DeviceRun, StepperState

    run = DeviceRun(StepperState(w=torch.from_numpy(w0).cuda(), h=0.005), out, k_max=3,
                    sample_every=10, checkpoint_every=20, seed=7, rng_state=b'{"s": 0}', **kw)
    run.start()
    run.advance(steps)
    return run


def test_run_matches_reference_and_resumes_bitwise(tmp_path):
    from paper_2206_05466_b200 import DeviceRun, read_checkpoint

    g = load_golden("cfg4_n64.npz")
    full = _run(tmp_path / "full", g["W0"], 40)
    names = sorted(p.name for p in (tmp_path / "full").iterdir())
    assert names == ["checkpoint_00000000.zck", "checkpoint_00000020.zck", "checkpoint_00000040.zck",
                     "diagnostics.csv", "run_meta.json"]
    cp20 = read_checkpoint(tmp_path / "full" / "checkpoint_00000020.zck")
    assert (cp20.step_index, cp20.n, cp20.seed, cp20.rng_state) == (20, 64, 7, b'{"s": 0}')
    assert relf(cp20.w.cpu().numpy(), g["W20"]) < 1e-12

    rows = (tmp_path / "full" / "diagnostics.csv").read_text().splitlines()
    assert rows[0] == "time,H,K,C2_rel,C3_rel"
    assert len(rows) == 1 + 5  # t = 0, 10, 20, 30, 40 steps
    t, h_val, k_val, c2, c3 = (float(x) for x in rows[3].split(","))
    assert t == pytest.approx(20 * 0.005, abs=1e-15)
    assert h_val == pytest.approx(g["H"][20], rel=1e-12) and k_val == h_val
    c0 = g["casimirs"][0]
    assert abs(c2 - abs(g["casimirs"][20][1] - c0[1]) / abs(c0[1])) < 1e-12
    assert c2 < 1e-12 and c3 < 1e-10

    part = _run(tmp_path / "part", g["W0"], 20)
    assert (tmp_path / "part" / "checkpoint_00000020.zck").read_bytes() == \
        (tmp_path / "full" / "checkpoint_00000020.zck").read_bytes()
    del part
    res = DeviceRun.resume(tmp_path / "part" / "checkpoint_00000020.zck", tmp_path / "part",
                           k_max=3, sample_every=10, checkpoint_every=20)
    res.advance(40)
    for f in ("diagnostics.csv", "checkpoint_00000040.zck"):
        assert (tmp_path / "part" / f).read_bytes() == (tmp_path / "full" / f).read_bytes(), f


def test_resume_truncates_later_rows_and_checks_config(tmp_path):
    from paper_2206_05466_b200 import DeviceRun

    g = load_golden("cfg4_n64.npz")
    _run(tmp_path / "o", g["W0"], 40)
    cp = tmp_path / "o" / "checkpoint_00000020.zck"
    run = DeviceRun.resume(cp, tmp_path / "o", k_max=3, sample_every=10, checkpoint_every=20)
    assert len((tmp_path / "o" / "diagnostics.csv").read_text().splitlines()) == 1 + 3
    assert run.state.step_index == 20
    with pytest.raises(ValueError):
        DeviceRun.resume(cp, tmp_path / "o", k_max=4)
    meta = json.loads((tmp_path / "o" / "run_meta.json").read_text())
    meta["seed"] = 8
    (tmp_path / "o" / "run_meta.json").write_text(json.dumps(meta))
    with pytest.raises(ValueError):
        DeviceRun.resume(cp, tmp_path / "o", k_max=3)
    with pytest.raises(ValueError):
        DeviceRun.resume(cp, tmp_path / "missing", k_max=3)


def test_run_with_device_basis_writes_spectra(tmp_path):
    """With a device basis the run writes spectrum_<step>.csv (driver.py:368-372)
    and K = sum_l E(l), equal to the trace-form H (diagnostics.py:8-12); the
    resumed run still reproduces every file byte for byte."""
    from paper_2206_05466_b200 import DeviceRun, StepperState, compute_basis

    g = load_golden("cfg4_n64.npz")
    b = compute_basis(64)

    def go(out, steps):
        run = DeviceRun(StepperState(w=torch.from_numpy(g["W0"]).cuda(), h=0.005), out, k_max=3,
                        sample_every=10, checkpoint_every=10, seed=1, basis=b, write_grid=True)
        run.start()
        run.advance(steps)

    go(tmp_path / "a", 20)
    rows = [r.split(",") for r in (tmp_path / "a" / "diagnostics.csv").read_text().splitlines()[1:]]
    for r in rows:
        assert float(r[2]) == pytest.approx(float(r[1]), rel=1e-12)
    sp = (tmp_path / "a" / "spectrum_00000020.csv").read_text().splitlines()
    assert sp[0] == "l,E_l" and len(sp) == 64 and sp[1].startswith("1,")
    go(tmp_path / "b", 10)
    DeviceRun.resume(tmp_path / "b" / "checkpoint_00000010.zck", tmp_path / "b", k_max=3, sample_every=10,
                     checkpoint_every=10, basis=b, write_grid=True).advance(20)
    from paper_2206_05466_b200.driver import read_grid

    field, t = read_grid(tmp_path / "a" / "grid_00000020.bin")
    assert field.shape == (126, 252) and t == pytest.approx(0.1, abs=1e-15)
    for f in ("diagnostics.csv", "spectrum_00000020.csv", "grid_00000020.bin", "checkpoint_00000020.zck"):
        assert (tmp_path / "b" / f).read_bytes() == (tmp_path / "a" / f).read_bytes(), f
