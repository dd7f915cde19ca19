"""CPU oracle for the dJFA hot path (arXiv 2209.00117) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  It shares no code with the CUDA path
(paper_2209_00117_b200/), which never imports it.

The arithmetic lives in vd_oracle.c (plain C, uint64 distances, OpenMP over output
rows); this module only builds it with gcc and marshals numpy arrays through ctypes.
Each wrapper names the paper passage its C function follows.

Pins (tests/test_oracle_*.py, run with -m "not gpu"): Eq. 2's printed example, SPEC's
schedule examples, scipy's exact Euclidean distance transform, the literal Algorithm-1
scatter formulation, hand-worked golden diagrams (tests/golden/), closed-form special
cases and invariants.  See DESIGN.md §4 for the pin of every function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

EMPTY = 0xFFFFFFFF
METRICS = {"euclid": 0, "manhattan": 1}  # P:172-173 (dJFAe / dJFAm)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vd_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc -O2 -fopenmp (seconds).  Returns its path."""
    up_to_date = (
        os.path.exists(_LIB_PATH)
        and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)
        and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(os.path.join(_HERE, "vd_oracle.h"))
    )
    if force or not up_to_date:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.run(
            ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wextra",
             "-o", tmp, _SRC],
            check=True,
        )
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        u32, u64, i32, p = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        sig = {
            "or_pack": (u32, [u32, u32]),
            "or_jfa_schedule": (i32, [u32, u32, p, i32]),
            "or_djfa_schedule": (i32, [u32, u64, u32, u32, p, i32]),
            "or_exact_brute": (None, [u32, u64, p, p]),
            "or_exact_bucketed": (i32, [u32, u64, p, u32, p]),
            "or_init": (None, [u32, u64, p, p]),
            "or_pass": (None, [u32, u32, p, p]),
            "or_jfa": (i32, [u32, u64, p, u32, p]),
            "or_move": (None, [u32, u64, p, p, p]),
            "or_djfa_step": (i32, [u32, u64, p, p, u32, u32, p, p]),
            "or_match_count": (u64, [u64, p, p]),
            "or_label_hash": (u64, [u64, p]),
            "or_num_threads": (i32, []),
            "or_pass_v": (None, [u32, u32, i32, i32, p, p]),
            "or_exact_brute_m": (None, [u32, u64, p, i32, p]),
            "or_jfa_v": (i32, [u32, u64, p, u32, i32, i32, p]),
            "or_djfa_step_v": (i32, [u32, u64, p, p, u32, u32, i32, i32, p, p]),
            "or_stf": (i32, [u32, u64, p, i32, p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


def _seeds(xy) -> np.ndarray:
    xy = np.ascontiguousarray(xy, dtype=np.uint16).reshape(-1)
    assert xy.size % 2 == 0
    return xy


def pack(x: int, y: int) -> int:
    """Label of the seed at (x, y): (y << 16) | x (R-1)."""
    return int(_load().or_pack(x, y))


def jfa_schedule(N: int, extras: int = 0) -> list[int]:
    """Eq. 2 k-list, + `extras` k=1 passes."""
    ks = np.zeros(64, dtype=np.uint32)
    n = _load().or_jfa_schedule(N, extras, _ptr(ks), 64)
    if n < 0:
        raise ValueError("bad N")
    return [int(v) for v in ks[:n]]


def djfa_schedule(N: int, s: int, d_max: int, extras: int = 0) -> list[int]:
    """Eq. 3-4 delta-list, exact integer form (R-7)."""
    ks = np.zeros(64, dtype=np.uint32)
    n = _load().or_djfa_schedule(N, s, d_max, extras, _ptr(ks), 64)
    if n < 0:
        raise ValueError("bad arguments")
    return [int(v) for v in ks[:n]]


def exact_brute(N: int, xy, metric: str = "euclid") -> np.ndarray:
    """Eq. 1 by brute force over all seeds; (N, N) uint32 labels.
    metric: "euclid" (default) or "manhattan" (dJFAm)."""
    xy = _seeds(xy)
    out = np.empty((N, N), dtype=np.uint32)
    _load().or_exact_brute_m(N, xy.size // 2, _ptr(xy), METRICS[metric], _ptr(out))
    return out


def exact(N: int, xy, bucket: int | None = None) -> np.ndarray:
    """Eq. 1 via bucketed ring search; equals exact_brute (tested)."""
    xy = _seeds(xy)
    s = xy.size // 2
    if bucket is None:
        bucket = max(1, int(round((N * N / max(s, 1)) ** 0.5)))
    out = np.empty((N, N), dtype=np.uint32)
    rc = _load().or_exact_bucketed(N, s, _ptr(xy), bucket, _ptr(out))
    if rc != 0:
        raise MemoryError("or_exact_bucketed failed")
    return out


def init(N: int, xy) -> np.ndarray:
    """All EMPTY, each seed pixel holds its own label."""
    xy = _seeds(xy)
    G = np.empty((N, N), dtype=np.uint32)
    _load().or_init(N, xy.size // 2, _ptr(xy), _ptr(G))
    return G


def jump_pass(G: np.ndarray, k: int, metric: str = "euclid", vn: bool = False) -> np.ndarray:
    """One gather pass with step k over Table 1; returns a new array.
    vn: Von Neumann neighbourhood (the 4 axis offsets)."""
    G = np.ascontiguousarray(G, dtype=np.uint32)
    N = G.shape[0]
    assert G.shape == (N, N)
    out = np.empty_like(G)
    _load().or_pass_v(N, k, METRICS[metric], int(bool(vn)), _ptr(G), _ptr(out))
    return out


def jfa(N: int, xy, extras: int = 0, metric: str = "euclid", vn_waves: int = 0) -> np.ndarray:
    """Full JFA: init + passes of jfa_schedule(N, extras); the first vn_waves passes use
    the Von Neumann neighbourhood ("Von Neumann alone ... even for JFA")."""
    xy = _seeds(xy)
    G = np.empty((N, N), dtype=np.uint32)
    n = _load().or_jfa_v(N, xy.size // 2, _ptr(xy), extras, METRICS[metric], vn_waves, _ptr(G))
    if n < 0:
        raise ValueError("or_jfa failed")
    return G


def stf(N: int, xy, metric: str = "euclid"):
    """Standard Flooding: k = 1 Moore passes until no pixel is EMPTY (R-22).
    Returns (G, passes)."""
    xy = _seeds(xy)
    G = np.empty((N, N), dtype=np.uint32)
    n = _load().or_stf(N, xy.size // 2, _ptr(xy), METRICS[metric], _ptr(G))
    if n < 0:
        raise ValueError("or_stf failed")
    return G, n


def move(N: int, xy_old, disp) -> np.ndarray:
    """SimulateParticles: clamp(old + disp) per axis (R-10, R-4)."""
    xy_old = _seeds(xy_old)
    disp = np.ascontiguousarray(disp, dtype=np.int16).reshape(-1)
    assert disp.size == xy_old.size
    out = np.empty_like(xy_old)
    _load().or_move(N, xy_old.size // 2, _ptr(xy_old), _ptr(disp), _ptr(out))
    return out


def djfa_step(N: int, xy_old, disp, d_max: int, G: np.ndarray, extras: int = 0, metric: str = "euclid",
              vn_waves: int = 0, inplace: bool = False):
    """One dJFA time step (Alg. 1; R-9).  Returns (G_new, xy_new, passes).
    metric "manhattan" = dJFAm; vn_waves = Von Neumann waves first.
    inplace: advance the caller's C-contiguous uint32 array G itself instead of a copy
    (saves one N*N copy of host memory at 65536^2; the arithmetic is the same)."""
    xy_old = _seeds(xy_old)
    disp = np.ascontiguousarray(disp, dtype=np.int16).reshape(-1)
    assert disp.size == xy_old.size
    if inplace:
        assert G.dtype == np.uint32 and G.flags["C_CONTIGUOUS"] and G.flags["WRITEABLE"]
    else:
        G = np.array(G, dtype=np.uint32, copy=True, order="C")
    xy_new = np.empty_like(xy_old)
    n = _load().or_djfa_step_v(N, xy_old.size // 2, _ptr(xy_old), _ptr(disp), d_max, extras, METRICS[metric],
                               vn_waves, _ptr(G), _ptr(xy_new))
    if n == -3:
        raise ValueError("previous diagram is incomplete or holds non-seed labels")
    if n < 0:
        raise ValueError("or_djfa_step failed")
    return G, xy_new, n


def match_count(a: np.ndarray, b: np.ndarray) -> int:
    """Eq. 5 numerator."""
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    assert a.shape == b.shape
    return int(_load().or_match_count(a.size, _ptr(a), _ptr(b)))


def similarity(a: np.ndarray, b: np.ndarray) -> float:
    """Eq. 5: 100 * matching pixels / total pixels."""
    return 100.0 * match_count(a, b) / a.size


def label_hash(G: np.ndarray) -> int:
    """Order-independent u64 checksum: sum_p fmix32((uint32)(p * 0x9E3779B9) ^ label[p])."""
    G = np.ascontiguousarray(G, dtype=np.uint32)
    return int(_load().or_label_hash(G.size, _ptr(G)))


def num_threads() -> int:
    return int(_load().or_num_threads())
