"""Build libvd.so in-tree with nvcc for sm_100a (no GPU needed: nvcc cross-compiles)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# vd.cu (host runtime + C ABI + the non-pass kernels) and one translation unit per jump-pass
# kernel family (vd_launch_*.cu), compiled in parallel and linked into one shared library
SRC = [os.path.join(PKG, "csrc", f) for f in ("vd.cu", "vd_launch_sk_small_a.cu", "vd_launch_sk_small_b.cu",
                                               "vd_launch_sk_mid_a.cu", "vd_launch_sk_mid_b.cu", "vd_launch_sk_large_a.cu",
                                               "vd_launch_sk_large_b.cu", "vd_launch_remap.cu", "vd_launch_fast.cu",
                                               "vd_launch_wide.cu", "vd_launch_wsk.cu")]
DEPS = SRC + [os.path.join(PKG, "csrc", "vd_kernels.cuh"), os.path.join(PKG, "csrc", "vd_launch.h"),
              os.path.join(ROOT, "include", "vd.h")]
LIB = os.path.join(PKG, "libvd.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    import nvidia.nccl  # the NCCL headers shipped with torch's wheel; only nccl.h is used
    return os.path.join(list(nvidia.nccl.__path__)[0], "include")


def _nvcc() -> str:
    return os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def compile_cmd(src: str, obj: str, extra: list[str] | None = None) -> list[str]:
    return [_nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-c",
            "-I", os.path.join(ROOT, "include"), "-I", _nccl_include(), "-o", obj, src, *(extra or [])]


def link_cmd(objs: list[str], out: str) -> list[str]:
    # shared cudart: in a torch process the already-loaded libcudart.so.12 is reused; the
    # rpath finds the toolkit's copy when libvd is loaded on its own
    return [_nvcc(), *ARCH, "-shared", "-cudart", "shared", "-Xlinker", "-rpath=/usr/local/cuda/lib64",
            "-o", out, *objs, "-ldl"]


def compile_all(out: str, extra: list[str] | None = None, verbose: bool = False) -> None:
    """Compile every translation unit in parallel (one nvcc per file), then link `out`."""
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    with tempfile.TemporaryDirectory(prefix="vdbuild") as tmp:
        objs = [os.path.join(tmp, os.path.basename(s) + ".o") for s in SRC]
        cmds = [compile_cmd(s, o, extra) for s, o in zip(SRC, objs)]
        if verbose:
            for c in cmds:
                print(" ".join(c), file=sys.stderr)
        with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
            for r in list(ex.map(lambda c: subprocess.run(c), cmds)):
                if r.returncode != 0:
                    raise subprocess.CalledProcessError(r.returncode, r.args)
        subprocess.run(link_cmd(objs, out), check=True)


def build(force: bool = False, verbose: bool = False) -> str:
    newest = max(os.path.getmtime(p) for p in DEPS)
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    compile_all(tmp, verbose=verbose)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
