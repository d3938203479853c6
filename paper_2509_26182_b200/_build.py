"""Build the in-tree CUDA extension ``libswarmsched_b200.so`` (sm_100a only).

The library is a plain C-ABI shared object (no torch / pybind types): nvcc
compiles every ``csrc/*.cu`` with ``-fmad=false`` so fp64 results keep the
reference's separately-rounded IEEE operations (SURVEY.md hazard H1).
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libswarmsched_b200.so")
CSRC_NCCL = os.path.join(HERE, "csrc_nccl")
LIB_NCCL = os.path.join(HERE, "libswarmsched_b200_nccl.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def nccl_dirs():
    """(include dir, lib dir) of the NCCL that torch loads (the nvidia-nccl wheel), so the exchange library and
    torch share one libnccl.so.2 in the process."""
    try:
        import nvidia.nccl as nn
        base = os.path.dirname(nn.__file__) if getattr(nn, "__file__", None) else list(nn.__path__)[0]
    except ImportError:
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    return os.path.join(base, "include"), os.path.join(base, "lib")


def build_nccl(force: bool = False) -> str:
    """libswarmsched_b200_nccl.so: the Phase-1 argmax and chain gather over NCCL (include/swarmsched_b200_nccl.h)."""
    srcs = sorted(glob.glob(os.path.join(CSRC_NCCL, "*.cu")))
    hdr = os.path.join(HERE, "..", "include", "swarmsched_b200_nccl.h")
    if not force and os.path.exists(LIB_NCCL) and all(os.path.getmtime(p) <= os.path.getmtime(LIB_NCCL)
                                                       for p in srcs + [hdr]):
        return LIB_NCCL
    inc, libdir = nccl_dirs()
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB_NCCL + ".tmp"
    cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-I", inc, *srcs,
           "-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir, "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed on the NCCL exchange library")
    os.replace(tmp, LIB_NCCL)
    return LIB_NCCL


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "swarmsched_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    objs = []
    for src in sources():
        obj = os.path.join(CSRC, os.path.basename(src)[:-3] + ".o")
        cmd = [nvcc, *ARCH, *FLAGS, "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(res.stderr)
        objs.append(obj)
    tmp = LIB + ".tmp"
    res = subprocess.run([nvcc, *ARCH, "-shared", "-o", tmp, *objs], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    for obj in objs:
        os.remove(obj)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))
    print(build_nccl(force=True))
