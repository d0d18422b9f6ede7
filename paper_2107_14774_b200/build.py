"""Build the in-tree sm_100a shared library liblbm_cuboid.so (the C ABI of
include/lbm_cuboid.h) with nvcc.  Links the NCCL that PyTorch ships (same
soname, rpath to its directory) so one NCCL instance serves the process."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblbm_cuboid.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    try:
        import nvidia.nccl  # noqa: PLC0415

        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except ImportError:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(ROOT, "include", "lbm_cuboid.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile liblbm_cuboid.so (or, with out/defines, a kernel variant)."""
    target = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    inc, libdir = nccl_dirs()
    tmp = target + f".tmp{os.getpid()}"
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-I", inc,
           *[f"-D{d}" for d in defines], os.path.join(CSRC, "lbm_cuboid.cu"), "-o", tmp,
           "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building liblbm_cuboid.so")
    with open(target + ".ptxas.log" if out else os.path.join(PKG, "ptxas.log"), "w") as fh:
        fh.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
