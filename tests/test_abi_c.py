"""The boundary from plain C: tests/abi_c/zt_c_consumer.c includes
include/zt.h as C99 (no C++, no torch), links libzt.so, and drives the path
with cudaMalloc'ed buffers — what a cgo / JNI / FFI stub on the reference
side would do.  CPU: it compiles warning-free and links
against every entry point it names.  GPU: it runs (round trip
lap(lap^-1 W) = W, one midpoint step with the consistency output, the gate's
and the argument checks' status codes)."""

import os
import shutil
import subprocess

import pytest
from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "abi_c", "zt_c_consumer.c")
PKG = os.path.join(ROOT, "paper_2206_05466_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _compile(out):
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), SRC, "-L", PKG, "-lzt", "-L", os.path.join(CUDA, "lib64"),
           "-lcudart", "-lm", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no gcc")
def test_header_is_c99_and_links(tmp_path):
    exe = _compile(str(tmp_path / "zt_c_consumer"))
    assert os.path.getsize(exe) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 97, 300])
def test_c_consumer_runs(tmp_path, n):
    exe = _compile(str(tmp_path / "zt_c_consumer"))
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = os.pathsep.join([PKG, os.path.join(CUDA, "lib64"), env.get("LD_LIBRARY_PATH", "")])
    r = subprocess.run([exe, str(n)], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "zt_c_consumer ok" in r.stdout
