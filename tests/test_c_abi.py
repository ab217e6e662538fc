"""The drop-in boundary is a plain C ABI: tests/c_abi/pgx_c_smoke.c is
compiled with gcc against include/pgx.h and linked with libpgx.so -- no
Python, no torch on that side.  CPU: host-only entry points (version,
size queries, error codes and messages).  GPU: a full connected_components
run through the C ABI, checked against the oracle (values and
per-superstep counts)."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_2010_01542_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_abi", "pgx_c_smoke.c")
LIBDIR = os.path.join(ROOT, "paper_2010_01542_b200")  # the in-tree libpgx.so
CUDA = "/usr/local/cuda"


def _build(tmp_path, gpu: bool):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path / ("smoke_gpu" if gpu else "smoke_host"))
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           SRC, "-o", exe, "-L", LIBDIR, "-lpgx", f"-Wl,-rpath,{LIBDIR}"]
    if gpu:
        cmd[1:1] = ["-DPGX_SMOKE_GPU", "-I", f"{CUDA}/include"]
        cmd += ["-L", f"{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{CUDA}/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_program_host_entry_points(tmp_path):
    exe = _build(tmp_path, gpu=False)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == f"host ok abi={_lib.PGX_ABI_VERSION}"


@pytest.mark.gpu
def test_c_program_runs_components_on_the_gpu(tmp_path):
    exe = _build(tmp_path, gpu=True)
    out = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    lines = dict(l.split(" ", 1) for l in out.stdout.strip().splitlines())
    off = np.array([0, 2, 4, 6, 8, 10, 12], np.int64)
    tgt = np.array([1, 2, 0, 2, 0, 1, 4, 5, 3, 5, 3, 4], np.int32)
    want = O.run_cc(6, off, tgt)
    assert [int(x) for x in lines["labels"].split()] == want.values.tolist() == [0, 0, 0, 3, 3, 3]
    assert lines["steps"] == f"{want.superstep_count} cap 0"
    assert [int(x) for x in lines["active"].split()] == want.active_counts
    assert [int(x) for x in lines["sent"].split()] == want.messages_sent
