"""The C-ABI from plain C (tests/capi/capi_demo.c): builds with gcc against
include/clifford_b200.h and libclifford_b200.so only -- no Python, torch or CUDA
headers in the caller. CPU: compiles, links and runs the host-only checks
(version, error contract, blade products). GPU: the conv (fp32 mode, host
buffers) against the program's own fp64 direct convolution and the activation."""

import os
import subprocess

import pytest

from paper_2507_01040_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    _lib.load()  # the library is built
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = str(tmp_path_factory.mktemp("capi") / "capi_demo")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "capi", "capi_demo.c"), "-o", exe, "-L", libdir, "-lclifford_b200",
           f"-Wl,-rpath,{libdir}", "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_capi_from_c_host_only(demo):
    r = subprocess.run([demo, "--host-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "capi_demo ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_capi_from_c_gpu(demo):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    r = subprocess.run([demo], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "capi_demo ok" in r.stdout, r.stdout + r.stderr
