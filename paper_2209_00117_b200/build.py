"""Build libvd.so in-tree with nvcc for sm_100a (no GPU needed: nvcc cross-compiles)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", "vd.cu")]
DEPS = SRC + [os.path.join(PKG, "csrc", "vd_kernels.cuh"), os.path.join(ROOT, "include", "vd.h")]
LIB = os.path.join(PKG, "libvd.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    import nvidia.nccl  # the NCCL headers shipped with torch's wheel; only nccl.h is used
    return os.path.join(list(nvidia.nccl.__path__)[0], "include")


def nvcc_cmd(out: str = LIB, extra: list[str] | None = None) -> list[str]:
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    return [nvcc, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
            # shared cudart: in a torch process the already-loaded libcudart.so.12 is reused; the
            # rpath finds the toolkit's copy when libvd is loaded on its own
            "-cudart", "shared", "-Xlinker", "-rpath=/usr/local/cuda/lib64",
            "-I", os.path.join(ROOT, "include"), "-I", _nccl_include(),
            "-o", out, *SRC, "-ldl", *(extra or [])]


def build(force: bool = False, verbose: bool = False) -> str:
    newest = max(os.path.getmtime(p) for p in DEPS)
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = nvcc_cmd(tmp)
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
