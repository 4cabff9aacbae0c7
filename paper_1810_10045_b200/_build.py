"""Build liblmscale.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_1810_10045_b200._build        # or __graft_entry__.build()

Links NCCL 2.28 from the nvidia-nccl wheel that torch itself loads, with an
rpath to it, so the process has exactly one libnccl.so.2.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblmscale.so")
LIB_CHECKED = os.path.join(PKG, "liblmscale_checked.so")  # device bounds checks compiled in
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl as nn
    base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "lmscale.h"), __file__]


def up_to_date(path: str = LIB) -> bool:
    if not os.path.exists(path):
        return False
    t = os.path.getmtime(path)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """checked: the LMSCALE_DEVICE_CHECKS build (bounds asserts in the kernels)
    as liblmscale_checked.so; load it with LMSCALE_LIB=<path>."""
    out = LIB_CHECKED if checked else LIB
    if not force and up_to_date(out):
        return out
    inc, lib = nccl_dirs()
    nvcc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc, "-O3", "-std=c++17", "-lineinfo", *ARCH, "-shared", "-Xcompiler", "-fPIC",
           *(["-DLMSCALE_DEVICE_CHECKS"] if checked else []),
           "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
           "-I", os.path.join(ROOT, "include"), "-I", inc,
           *sources(), "-L", lib, "-l:libnccl.so.2", f"-Xlinker", f"-rpath={lib}",
           "-o", tmp]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                checked="--checked" in sys.argv))
