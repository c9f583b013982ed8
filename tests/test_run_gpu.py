"""`run(SimConfig)` — the reference's run loop (driver.py:259-410) on the device
path — against the reference's own output directories (tests/golden/runs.npz,
written by the reference's `run` for the test_driver.py configurations), plus
the behaviour test_driver.py:176-265 asserts: cadence, auto time step,
grid/spectrum consistency, exit codes 2/3/4, and a resumed run reproducing the
uninterrupted run's diagnostics and spectrum byte for byte."""

import json

import numpy as np
import pytest
from conftest import load_golden, relf

pytestmark = pytest.mark.gpu

RUNS = {
    "resume": dict(n=12, steps=40, h=1e-3, l_min=2, l_max=6, sample_every=10, checkpoint_every=20, seed=7),
    "auto_h": dict(n=8, steps=2, l_max=5, seed=1),
    "cadence": dict(n=8, steps=25, h=1e-3, l_max=5, sample_every=10, checkpoint_every=20, seed=1),
    "grid": dict(n=10, steps=5, h=1e-3, l_max=6, sample_every=5, seed=4),
}


def _rows(text):
    lines = text.strip().splitlines()
    return lines[0].split(","), np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])


@pytest.fixture(scope="module")
def golden():
    return load_golden("runs.npz")


@pytest.mark.parametrize("name", sorted(RUNS))
def test_run_matches_reference_output(tmp_path, golden, name):
    from paper_2206_05466_b200 import run
    from paper_2206_05466_b200.driver import SimConfig, read_checkpoint, read_grid

    kw = RUNS[name]
    out = tmp_path / "o"
    assert run(SimConfig(output_dir=str(out), **kw)) == 0
    last = kw["steps"]
    text = lambda key: bytes(golden[f"{name}_{key}"]).decode()  # noqa: E731

    # run_meta.json: same keys; h and the Casimir baseline as hex floats
    mine, ref = json.loads((out / "run_meta.json").read_text()), json.loads(text("meta"))
    assert mine.keys() == ref.keys()
    assert (mine["version"], mine["n"], mine["seed"], mine["k_max"]) == (ref["version"], ref["n"], ref["seed"], ref["k_max"])
    h_m, h_r = float.fromhex(mine["h"]), float.fromhex(ref["h"])
    if "h" in kw:
        assert h_m == h_r
    else:  # default_time_step = 0.1 / ||lap^-1 W0||_2 (integrator.py:86-93)
        assert h_m == pytest.approx(h_r, rel=1e-12)
    cb_m = np.array([float.fromhex(v) for v in mine["casimir_baseline"]])
    cb_r = np.array([float.fromhex(v) for v in ref["casimir_baseline"]])
    np.testing.assert_allclose(cb_m, cb_r, rtol=1e-12, atol=1e-14)  # C1 = tr W is round-off

    # diagnostics.csv: same header and sample times; H, K to 1e-12; Casimir
    # drifts are round-off on both sides (floor 1e-13)
    hm, dm = _rows((out / "diagnostics.csv").read_text())
    hr, dr = _rows(text("diag"))
    assert hm == hr and dm.shape == dr.shape
    np.testing.assert_allclose(dm[:, 0], dr[:, 0], rtol=1e-12, atol=0)
    np.testing.assert_allclose(dm[:, 1:3], dr[:, 1:3], rtol=1e-11)
    assert np.all(dm[:, 3:] <= np.maximum(dr[:, 3:], 1e-13))

    # the final spectrum, state and grid
    sm, sr = _rows((out / f"spectrum_{last:08d}.csv").read_text()), _rows(text("spec"))
    assert sm[0] == sr[0] == ["l", "E_l"]
    np.testing.assert_allclose(sm[1], sr[1], rtol=1e-10, atol=1e-16)
    w = read_checkpoint(out / f"checkpoint_{last:08d}.zck").w.cpu().numpy()
    assert relf(w, golden[f"{name}_w"]) <= 1e-12
    field, _ = read_grid(out / f"grid_{last:08d}.bin")
    ref_field = golden[f"{name}_grid"]
    np.testing.assert_allclose(field, ref_field, atol=1e-11 * np.max(np.abs(ref_field)), rtol=0)


def test_zero_steps_writes_initial_sample_only(tmp_path):
    from paper_2206_05466_b200.driver import SimConfig, run

    out = tmp_path / "o"
    assert run(SimConfig(n=8, steps=0, h=1e-3, l_max=5, output_dir=str(out), seed=1)) == 0
    header, rows = _rows((out / "diagnostics.csv").read_text())
    assert header == ["time", "H", "K", "C2_rel", "C3_rel", "C4_rel", "C5_rel"]
    assert rows.shape[0] == 1 and rows[0, 0] == 0.0
    assert (out / "spectrum_00000000.csv").exists()
    assert (out / "checkpoint_00000000.zck").exists()
    assert (out / "grid_00000000.bin").exists()


def test_cadence_includes_final(tmp_path):
    from paper_2206_05466_b200.driver import SimConfig, run

    out = tmp_path / "o"
    assert run(SimConfig(output_dir=str(out), **RUNS["cadence"])) == 0
    _, rows = _rows((out / "diagnostics.csv").read_text())
    assert [round(t / 1e-3) for t in rows[:, 0]] == [0, 10, 20, 25]
    assert sorted(p.name for p in out.glob("checkpoint_*.zck")) == [
        "checkpoint_00000000.zck", "checkpoint_00000020.zck", "checkpoint_00000025.zck"]


def test_exit_codes(tmp_path):
    from paper_2206_05466_b200.driver import EXIT_CONFIG, EXIT_IO, EXIT_SOLVER, SimConfig, run

    # test_driver.py:224-229: one iteration at tol 1e-14 cannot converge
    assert run(SimConfig(n=12, steps=5, h=0.5, l_max=6, max_iter=1, tol=1e-14,
                         output_dir=str(tmp_path / "s"), seed=1)) == EXIT_SOLVER
    # test_driver.py:260-263
    assert run(SimConfig(n=8, steps=1, h=1e-3, l_max=5, output_dir=str(tmp_path), seed=1),
               resume=str(tmp_path / "nope.zck")) == EXIT_IO
    # test_driver.py:250-258: the checkpoint's N / seed must match
    base = dict(n=10, h=1e-3, l_max=6, sample_every=10, checkpoint_every=10)
    out = tmp_path / "o"
    assert run(SimConfig(steps=10, output_dir=str(out), seed=3, **base)) == 0
    cp = str(out / "checkpoint_00000010.zck")
    assert run(SimConfig(steps=20, output_dir=str(out), seed=4, **base), resume=cp) == EXIT_CONFIG
    assert run(SimConfig(n=12, steps=20, h=1e-3, l_max=6, output_dir=str(out), seed=3), resume=cp) == EXIT_CONFIG
    assert run(SimConfig(steps=20, output_dir=str(out), seed=3, **{**base, "h": 2e-3}), resume=cp) == EXIT_CONFIG


def test_resume_reproduces_stream(tmp_path):
    """test_driver.py:231-248, plus the checkpoints and grids."""
    from paper_2206_05466_b200.driver import SimConfig, run

    base = {k: v for k, v in RUNS["resume"].items() if k != "steps"}
    full, part = tmp_path / "full", tmp_path / "part"
    assert run(SimConfig(steps=40, output_dir=str(full), **base)) == 0
    assert run(SimConfig(steps=20, output_dir=str(part), **base)) == 0
    assert run(SimConfig(steps=40, output_dir=str(part), **base),
               resume=str(part / "checkpoint_00000020.zck")) == 0
    for fname in ("diagnostics.csv", "spectrum_00000040.csv", "checkpoint_00000040.zck", "grid_00000040.bin",
                  "run_meta.json"):
        assert (part / fname).read_bytes() == (full / fname).read_bytes(), fname
