"""Build libclifford_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2507_01040_b200.build [--force]

Plain nvcc (no torch extension machinery): the product is a C-ABI shared
library (include/clifford_b200.h) loaded through ctypes. cudart is linked
statically; the driver API (TMA descriptor encoding) is reached through
cudaGetDriverEntryPoint, so the .so needs nothing beyond libcuda at run time.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libclifford_b200.so")
# diagnostic build: identical kernels plus the CL_* A/B timing switches and the
# CL_DBG_FLIP_COEFF fault injection read from the environment (internal.h
# CL_ENV); used by tests/test_gpu_variants.py and tools/ through CL_LIB_PATH
LIB_AB = os.path.join(LIBDIR, "libclifford_b200_ab.so")
# the C-ABI registered as PyTorch operators (torch.ops.clifford_b200.*): the
# binding the Python layer uses; it dlopens LIB (or LIB_AB) at load time
TORCH_OPS = os.path.join(LIBDIR, "libclifford_b200_torch.so")
TORCH_SRC = os.path.join(HERE, "csrc_torch", "clifford_ops.cpp")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", f"-I{ROOT}/include", "-Xptxas", "-v"]
# extra -D switches for A/B builds of tools/ (e.g. CL_NVCC_DEFS="-DCL_X3_EPI_GROUPS=3"); empty in the product build
FLAGS += os.environ.get("CL_NVCC_DEFS", "").split()


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "clifford_b200.h"),
                                                                TORCH_SRC]


def up_to_date() -> bool:
    for lib in (LIB, LIB_AB, TORCH_OPS):
        if not os.path.exists(lib):
            return False
        t = os.path.getmtime(lib)
        if any(os.path.getmtime(d) > t for d in deps()):
            return False
    return True


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    variants = [(LIB, os.path.join(LIBDIR, "obj"), []),
                (LIB_AB, os.path.join(LIBDIR, "obj_ab"), ["-DCL_AB_SWITCHES"])]
    for _, objdir, _ in variants:
        os.makedirs(objdir, exist_ok=True)

    def compile_one(job):
        src, objdir, defs = job
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *defs, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and not defs:
            sys.stderr.write(r.stderr)
        return obj

    # longest translation units first (conv_tc.cu dominates)
    srcs = sorted(sources(), key=lambda p: -os.path.getsize(p))
    jobs = [(src, objdir, defs) for src in srcs for _, objdir, defs in variants]
    with ThreadPoolExecutor(max_workers=min(len(jobs) + 1, max(2, os.cpu_count() or 1))) as ex:
        ops = ex.submit(build_torch_ops)
        objs = list(ex.map(compile_one, jobs))
        ops.result()
    for lib, objdir, _ in variants:
        mine = [o for o in objs if os.path.dirname(o) == objdir]
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *mine, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def build_torch_ops() -> str:
    """g++ against the installed torch's headers and libraries (no nvcc: the
    extension only forwards tensors and the current stream to the C-ABI)."""
    import torch
    tdir = os.path.dirname(torch.__file__)
    inc = [os.path.join(tdir, "include"), os.path.join(tdir, "include", "torch", "csrc", "api", "include"),
           os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "include")]
    libdir = os.path.join(tdir, "lib")
    abi = int(getattr(torch._C, "_GLIBCXX_USE_CXX11_ABI", 1))
    # the system g++: a CXX wrapper that links libstdc++ statically (as /opt/gcc's
    # does here) gives the extension a private std::string / exception runtime,
    # and a c10::Error thrown across it into torch then crashes
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else os.environ.get("CXX", "g++")
    cmd = [cxx, "-O2", "-std=c++17", "-fPIC", "-shared", f"-D_GLIBCXX_USE_CXX11_ABI={abi}",
           *[f"-I{d}" for d in inc], TORCH_SRC, "-o", TORCH_OPS, f"-L{libdir}", "-lc10", "-lc10_cuda", "-ltorch_cpu",
           "-ltorch", f"-Wl,-rpath,{libdir}", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"torch ops build failed:\n{r.stdout}\n{r.stderr}")
    return TORCH_OPS


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
