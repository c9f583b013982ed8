"""Device-resident run loop, on-device sample-time diagnostics and ZCK1
checkpoints (the caller of the hot path and its
on-disk state format).

The reference's driver (/root/reference/pkg/src/zeitlin/driver.py:284-410)
copies W to the host at every sample; here W stays in HBM for the whole run:
the step is one CUDA graph per step, and the sample-time quantities are
computed on the device — Casimirs C_2..C_kmax (integrator.py:180-210, DMMA
GEMMs), the energy H (diagnostics.py:60-63, stream solve + vdot) and their
drift (diagnostics.py:86-110).  Only checkpoints leave the device.

Checkpoints use the reference's ZCK1 layout byte for byte
(formats.py:116-156): magic "ZCK1", `<IIQdQI` = version, N, step, time, seed,
rng-blob length, the rng blob, then the N^2 complex128 entries in
column-major order — produced by a device-side transpose before the single
device-to-host copy.  Runs are bitwise deterministic, so a run resumed from a
checkpoint reproduces the uninterrupted run's checkpoints and diagnostics
byte for byte (the reference's test_driver.py:231-248 contract).

With a device basis (`basis.compute_basis`) each sample
also extracts the coefficients on the device and writes the reference's
`spectrum_<step>.csv` (rows l, E_l) with K = sum_l E(l)
(driver.py:357-372) and, with `write_grid`, the ZGD1 grid snapshot of the
field (rank 4, driver.py:373-375); without one, K is the trace-form energy H,
equal to it up to round-off (diagnostics.py:8-12).  Out of scope: the config
file and CLI.
"""

from __future__ import annotations

import json
import struct
import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .basis import (
    HarmonicCoefficients,
    energy_spectrum_packed,
    evaluate_on_grid_packed,
    extract_packed,
    project_packed,
)
from .diagnostics import casimir_drift, hamiltonian
from .integrator import FixedPointError, StepperState, casimirs, default_time_step, midpoint_step_raw
from .laplacian import build_operator

CHECKPOINT_MAGIC = b"ZCK1"
GRID_MAGIC = b"ZGD1"
FORMAT_VERSION = 1


class FileFormatError(ValueError):
    """formats.py:49-50."""


EXIT_OK = 0      # driver.py:61-64: run() exit codes
EXIT_CONFIG = 2
EXIT_SOLVER = 3
EXIT_IO = 4


class ConfigError(ValueError):
    """Invalid or inconsistent run configuration (driver.py:67-68)."""


class SolverError(RuntimeError):
    """The inner iteration failed during a run; carries the step index (driver.py:71-72)."""


@dataclass
class SimConfig:
    """Run parameters (driver.py:75-122); ``h=None`` selects the advective-limit
    default.  ``threads`` and ``deterministic`` are accepted: device runs are
    bitwise deterministic at any setting."""

    n: int
    steps: int
    h: float | None = None
    tol: float = 1e-12
    max_iter: int = 10
    seed: int = 0
    l_min: int = 2
    l_max: int = 20
    sample_every: int = 5000
    checkpoint_every: int = 10000
    output_dir: str = "out"
    threads: int = 0
    comm_scale: float = 1.0
    k_max: int = 5
    deterministic: bool = False
    write_grid: bool = True
    basis_cache: str | None = None

    def validate(self) -> None:
        checks = (
            (self.n >= 2, f"n must be at least 2, got {self.n}"),
            (self.steps >= 0, f"steps must be nonnegative, got {self.steps}"),
            (self.h is None or self.h > 0.0, f"h must be positive, got {self.h}"),
            (2 <= self.l_min <= self.l_max <= self.n - 1,
             f"need 2 <= l_min <= l_max <= n-1, got l_min={self.l_min}, l_max={self.l_max}, n={self.n}"),
            (self.tol > 0.0, f"tol must be positive, got {self.tol}"),
            (self.max_iter >= 1, f"max_iter must be at least 1, got {self.max_iter}"),
            (self.sample_every >= 1 and self.checkpoint_every >= 1,
             "sample_every and checkpoint_every must be at least 1"),
            (0 <= self.seed < 2**64, f"seed must fit in 64 bits, got {self.seed}"),
            (2 <= self.k_max <= self.n, f"k_max={self.k_max} out of range 2..{self.n}"),
            (self.threads >= 0, f"threads must be nonnegative, got {self.threads}"),
            (self.comm_scale > 0.0, f"comm_scale must be positive, got {self.comm_scale}"),
        )
        for ok, msg in checks:
            if not ok:
                raise ConfigError(msg)


def _log(msg: str) -> None:
    print(f"[zeitlin] {msg}", file=sys.stderr, flush=True)


def format_float(x: float) -> str:
    """%.17g, formats.py:55-56."""
    return f"{float(x):.17g}"


@dataclass
class Checkpoint:
    step_index: int
    time: float
    n: int
    seed: int
    rng_state: bytes
    w: torch.Tensor  # on device


def _atomic_write(path: Path, payload: bytes) -> None:
    tmp = path.with_name(path.name + ".tmp")
    tmp.write_bytes(payload)
    tmp.replace(path)


def write_checkpoint(path, cp: Checkpoint) -> None:
    """ZCK1 writer (formats.py:130-143): column-major body from a device transpose."""
    n = cp.w.shape[0]
    header = CHECKPOINT_MAGIC + struct.pack(
        "<IIQdQI", FORMAT_VERSION, n, cp.step_index, cp.time, cp.seed, len(cp.rng_state))
    body = cp.w.transpose(0, 1).contiguous().cpu().numpy().astype("<c16").tobytes()
    _atomic_write(Path(path), header + cp.rng_state + body)


def read_checkpoint(path, device=None) -> Checkpoint:
    """ZCK1 reader (formats.py:146-156) onto the device."""
    with open(path, "rb") as fh:
        if fh.read(4) != CHECKPOINT_MAGIC:
            raise FileFormatError(f"{path}: bad magic, expected {CHECKPOINT_MAGIC!r}")
        head = fh.read(36)
        if len(head) != 36:
            raise FileFormatError("truncated file while reading header")
        version, n, step, time, seed, blob_len = struct.unpack("<IIQdQI", head)
        if version != FORMAT_VERSION:
            raise FileFormatError(f"{path}: unsupported version {version}")
        rng_state = fh.read(blob_len)
        raw = fh.read(16 * n * n)
        if len(rng_state) != blob_len or len(raw) != 16 * n * n:
            raise FileFormatError("truncated file while reading state entries")
        if fh.read(1):
            raise FileFormatError(f"{path}: trailing bytes after state entries")
    wt = torch.from_numpy(np.frombuffer(raw, dtype="<c16").reshape(n, n).copy())
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    w = wt.to(dev).transpose(0, 1).contiguous()  # column-major on disk (device transpose)
    return Checkpoint(step_index=step, time=time, n=n, seed=seed, rng_state=rng_state, w=w)


def write_grid(path, field: np.ndarray, time: float) -> None:
    """ZGD1 snapshot (formats.py:163-168): header, then n_lat x n_lon <f8."""
    if field.ndim != 2:
        raise ValueError(f"grid field must be 2-D, got shape {field.shape}")
    n_lat, n_lon = field.shape
    header = GRID_MAGIC + struct.pack("<IId", n_lat, n_lon, time)
    _atomic_write(Path(path), header + np.ascontiguousarray(field, dtype="<f8").tobytes())


def read_grid(path) -> tuple[np.ndarray, float]:
    """ZGD1 reader (formats.py:171-181)."""
    with open(path, "rb") as fh:
        if fh.read(4) != GRID_MAGIC:
            raise FileFormatError(f"{path}: bad magic, expected {GRID_MAGIC!r}")
        head = fh.read(16)
        if len(head) != 16:
            raise FileFormatError("truncated file while reading header")
        n_lat, n_lon, time = struct.unpack("<IId", head)
        if n_lat < 2 or n_lon < 2:
            raise FileFormatError(f"{path}: invalid grid shape {n_lat} x {n_lon}")
        raw = fh.read(8 * n_lat * n_lon)
        if len(raw) != 8 * n_lat * n_lon:
            raise FileFormatError("truncated file while reading grid samples")
        if fh.read(1):
            raise FileFormatError(f"{path}: trailing bytes after grid samples")
    return np.frombuffer(raw, dtype="<f8").reshape(n_lat, n_lon).copy(), time


def _drift_row(c0: np.ndarray, ck: np.ndarray) -> np.ndarray:
    """diagnostics.py:86-110 for one sample: |C_k - C_k(0)| / |C_k(0)|, k >= 2,
    absolute error where the baseline is below 1e-14."""
    return casimir_drift([(0.0, c0), (0.0, ck)])[1].casimir_rel_err


def random_initial_condition(cfg, basis, rng: np.random.Generator | None = None) -> torch.Tensor:
    """driver.py:196-225: band-limited random field, unit spectral norm.

    `cfg` needs n, l_min, l_max, seed (the reference's SimConfig works).
    Magnitudes uniform in [0.8, 1.2], uniform random phase (m = 0: real with
    a random sign), drawn m ascending then l ascending so a seed pins the
    coefficients bitwise; negative orders from the reality condition.  The
    field is assembled on the device with the device basis; above N = 16 the
    basis phase convention may differ from the reference's LAPACK-rounding
    signs (basis.py:27-30), so the same seed gives the same coefficients but
    not necessarily the same matrix there.
    """
    from .laplacian import spectral_norm

    n, l_min, l_max = cfg.n, cfg.l_min, cfg.l_max
    if l_max >= n:
        raise ConfigError(f"l_max={l_max} must be below n={n}")
    if rng is None:
        rng = np.random.default_rng(cfg.seed)
    coeffs = HarmonicCoefficients.zeros(n)
    for m in range(l_max + 1):
        lo = max(l_min, m, 1)
        if lo > l_max:
            continue
        count = l_max - lo + 1
        amps = rng.uniform(0.8, 1.2, count)
        if m == 0:
            vals = amps * np.where(rng.random(count) < 0.5, -1.0, 1.0) + 0j
        else:
            vals = amps * np.exp(2j * np.pi * rng.random(count))
        first = lo - max(m, 1)
        coeffs.pos[m][first:first + count] = vals
    coeffs.enforce_reality()
    pos, _ = coeffs.packed(basis.data.device)
    w = project_packed(pos, None, basis)
    return w / spectral_norm(w)


class DeviceRun:
    """Device-resident time stepping with sample / checkpoint cadence
    (driver.py:357-410 without the basis-dependent outputs)."""

    def __init__(self, state: StepperState, output_dir, k_max: int = 3, sample_every: int = 10,
                 checkpoint_every: int = 100, seed: int = 0, rng_state: bytes = b"",
                 baseline: np.ndarray | None = None, basis=None, write_grid: bool = False):
        w = state.w if isinstance(state.w, torch.Tensor) else torch.from_numpy(np.asarray(state.w))
        if not w.is_cuda:
            w = w.to(torch.device("cuda", torch.cuda.current_device()))
        self.w = w.to(torch.complex128).contiguous()
        self.spare = torch.empty_like(self.w)
        self.state = state
        self.n = self.w.shape[0]
        self.op = build_operator(self.n, self.w.device)
        self.out = Path(output_dir)
        self.out.mkdir(parents=True, exist_ok=True)
        self.k_max = k_max
        self.sample_every = sample_every
        self.checkpoint_every = checkpoint_every
        self.seed = seed
        self.rng_state = rng_state
        self.baseline = casimirs(self.w, k_max) if baseline is None else np.asarray(baseline)
        self.diag_path = self.out / "diagnostics.csv"
        self.meta_path = self.out / "run_meta.json"
        self.iterations: list[int] = []
        if basis is not None and basis.n != self.n:
            raise ValueError(f"basis is for N={basis.n}, state has N={self.n}")
        self.basis = basis
        self.write_grid = write_grid and basis is not None
        self.log = False

    # -- files ---------------------------------------------------------------
    def start(self) -> None:
        """Fresh run: metadata, header, the t = 0 sample and checkpoint (driver.py:336-392)."""
        meta = {"version": 1, "n": self.n, "seed": self.seed, "h": float(self.state.h).hex(),
                "k_max": self.k_max, "casimir_baseline": [float(c).hex() for c in self.baseline]}
        self.meta_path.write_text(json.dumps(meta, indent=1) + "\n")
        header = ",".join(["time", "H", "K"] + [f"C{k}_rel" for k in range(2, self.k_max + 1)])
        self.diag_path.write_text(header + "\n")
        self.sample()
        self.checkpoint()

    @classmethod
    def resume(cls, checkpoint_path, output_dir, k_max=3, sample_every=10, checkpoint_every=100,
               tol=1e-12, max_iter=10, comm_scale=1.0, basis=None, write_grid=False):
        """Resume from a ZCK1 checkpoint and the run's run_meta.json (driver.py:300-334)."""
        out = Path(output_dir)
        meta_path, diag_path = out / "run_meta.json", out / "diagnostics.csv"
        if not meta_path.exists():
            raise ConfigError(f"resume requires {meta_path} from the original run directory")
        if not diag_path.exists():
            raise FileFormatError(f"{diag_path}: missing diagnostics file for resume")
        meta = json.loads(meta_path.read_text())
        cp = checkpoint_path if isinstance(checkpoint_path, Checkpoint) else read_checkpoint(checkpoint_path)
        if meta.get("n") != cp.n or meta.get("seed") != cp.seed:
            raise ConfigError(f"{meta_path} does not match checkpoint (N={cp.n}, seed={cp.seed})")
        h = float.fromhex(meta["h"])
        baseline = np.array([float.fromhex(s) for s in meta["casimir_baseline"]])
        if baseline.size != k_max:
            raise ConfigError(f"{meta_path} stores k_max={baseline.size}, asked for {k_max}")
        st = StepperState(w=cp.w, h=h, time=cp.time, step_index=cp.step_index, tol=tol,
                          max_iter=max_iter, comm_scale=comm_scale)
        run = cls(st, out, k_max=k_max, sample_every=sample_every, checkpoint_every=checkpoint_every,
                  seed=cp.seed, rng_state=cp.rng_state, baseline=baseline, basis=basis, write_grid=write_grid)
        # drop diagnostics rows after the resume point (driver.py:241-252)
        lines = run.diag_path.read_text().splitlines()
        kept = [lines[0]] + [ln for ln in lines[1:]
                             if ln and float(ln.split(",", 1)[0]) <= cp.time + 0.5 * h]
        run.diag_path.write_text("\n".join(kept) + "\n")
        return run

    def sample(self) -> float:
        """On-device Casimirs and energy at the current state (driver.py:357-376)."""
        ck = casimirs(self.w, self.k_max)
        h_val = hamiltonian(self.w, self.op)
        k_val = h_val
        if self.basis is not None:
            pos, neg = extract_packed(self.w, self.basis)
            energy = energy_spectrum_packed(pos, neg, self.basis).cpu().numpy()
            k_val = float(energy.sum())
            lines = ["l,E_l"] + [f"{l},{format_float(energy[l])}" for l in range(1, self.n)]
            _atomic_write(self.out / f"spectrum_{self.state.step_index:08d}.csv", ("\n".join(lines) + "\n").encode())
            if self.write_grid:
                # driver.py:355, 373-375: l_render = min(N-1, 512) on a 2L x 4L grid
                lr = min(self.n - 1, 512)
                field = evaluate_on_grid_packed(self.n, pos, 2 * lr, 4 * lr, l_max=lr).cpu().numpy()
                write_grid(self.out / f"grid_{self.state.step_index:08d}.bin", field, self.state.time)
        row = [format_float(self.state.time), format_float(h_val), format_float(k_val)]
        row += [format_float(v) for v in _drift_row(self.baseline, ck)]
        with open(self.diag_path, "a", encoding="utf-8") as fh:
            fh.write(",".join(row) + "\n")
        return h_val

    def checkpoint(self) -> Path:
        path = self.out / f"checkpoint_{self.state.step_index:08d}.zck"
        write_checkpoint(path, Checkpoint(self.state.step_index, self.state.time, self.n, self.seed,
                                          self.rng_state, self.w))
        return path

    # -- stepping ------------------------------------------------------------
    def advance(self, steps: int) -> None:
        """Step to `steps` (absolute step index), sampling / checkpointing at cadence."""
        st = self.state
        h_eff = st.h * st.comm_scale
        while st.step_index < steps:
            try:
                nxt, k, _, _ = midpoint_step_raw(self.w, h_eff, st.tol, st.max_iter, self.op, out=self.spare)
            except FixedPointError as exc:  # driver.py:394-399
                raise SolverError(f"step {st.step_index + 1}: {exc} (residual {exc.residual:.3e})") from exc
            self.w, self.spare = nxt, self.w
            st.time = st.time + st.h
            st.step_index += 1
            self.iterations.append(k)
            final = st.step_index == steps
            if st.step_index % self.sample_every == 0 or final:
                h_val = self.sample()
                if self.log:
                    _log(f"step {st.step_index}/{steps} t={st.time:.6g} H={h_val:.9e} iters={k}")
            if st.step_index % self.checkpoint_every == 0 or final:
                self.checkpoint()
        st.w = self.w


def run(cfg: SimConfig, resume: str | None = None) -> int:
    """driver.py:259-281: execute a run; returns a process exit code (0 ok,
    2 configuration, 3 solver, 4 I/O).  The loop is `DeviceRun` (W stays in
    HBM; samples and checkpoints computed on the device)."""
    try:
        cfg.validate()
    except ConfigError as exc:
        _log(f"configuration error: {exc}")
        return EXIT_CONFIG
    try:
        _run_inner(cfg, resume)
    except ConfigError as exc:
        _log(f"configuration error: {exc}")
        return EXIT_CONFIG
    except (SolverError, FixedPointError) as exc:
        _log(f"solver failure: {exc}")
        return EXIT_SOLVER
    except (OSError, FileFormatError) as exc:
        _log(f"I/O failure: {exc}")
        return EXIT_IO
    return EXIT_OK


def _run_inner(cfg: SimConfig, resume: str | None) -> None:
    """driver.py:284-410 on the device."""
    from .basis import compute_basis, load_basis

    out = Path(cfg.output_dir)
    out.mkdir(parents=True, exist_ok=True)
    meta_path = out / "run_meta.json"
    lap = build_operator(cfg.n)
    if cfg.basis_cache:
        basis = load_basis(cfg.basis_cache)
        if basis.n != cfg.n:
            raise ConfigError(f"basis cache is for N={basis.n}, configuration asks for N={cfg.n}")
    else:
        basis = compute_basis(cfg.n)
    common = dict(k_max=cfg.k_max, sample_every=cfg.sample_every, checkpoint_every=cfg.checkpoint_every,
                  basis=basis, write_grid=cfg.write_grid)
    if resume is not None:
        cp = read_checkpoint(resume)
        if cp.n != cfg.n:
            raise ConfigError(f"checkpoint is for N={cp.n}, configuration asks for N={cfg.n}")
        if cp.seed != cfg.seed:
            raise ConfigError(f"checkpoint seed {cp.seed} differs from configured {cfg.seed}")
        if not meta_path.exists():
            raise ConfigError(f"resume requires {meta_path} from the original run directory")
        meta = json.loads(meta_path.read_text())
        if meta.get("n") != cfg.n or meta.get("seed") != cfg.seed:
            raise ConfigError(f"{meta_path} does not match this configuration")
        h = float.fromhex(meta["h"])
        if cfg.h is not None and cfg.h != h:
            raise ConfigError(f"configured h={cfg.h} differs from the original run's h={h}; "
                              "a resumed run must keep its time-step")
        if len(meta["casimir_baseline"]) != cfg.k_max:
            raise ConfigError(f"{meta_path} stores k_max={len(meta['casimir_baseline'])}, configured {cfg.k_max}")
        dr = DeviceRun.resume(cp, out, tol=cfg.tol, max_iter=cfg.max_iter, comm_scale=cfg.comm_scale,
                              **common)
        _log(f"resumed from {resume} at step {cp.step_index} (t={cp.time:g})")
    else:
        rng = np.random.default_rng(cfg.seed)
        w0 = random_initial_condition(cfg, basis, rng)
        h = cfg.h if cfg.h is not None else default_time_step(w0, lap)
        st = StepperState(w=w0, h=h, tol=cfg.tol, max_iter=cfg.max_iter, comm_scale=cfg.comm_scale)
        blob = json.dumps(rng.bit_generator.state).encode("utf-8")
        dr = DeviceRun(st, out, seed=cfg.seed, rng_state=blob, **common)
        _log(f"N={cfg.n} steps={cfg.steps} h={h:g} seed={cfg.seed}")
        dr.start()
    dr.log = True
    dr.advance(cfg.steps)
