"""paper_2209_00117_b200 -- Python binding of libvd (include/vd.h), the B200 (sm_100a)
implementation of the dJFA hot path of arXiv 2209.00117 ("GPU Voronoi Diagrams for
Random Moving Seeds").

Argument marshalling only: every step of the path (seed stamping, jump passes, the dJFA
move / forward map / remap, Eq. 5 similarity, the label hash) runs in libvd's CUDA
kernels.  There is no CPU fallback: if libvd.so is missing or no GPU is present, the
calls raise.  PyTorch is used only for device memory, streams and process groups
(callers may pass torch tensors, host or CUDA, and torch's current stream).

The function names are the C ABI's (vd_create, vd_jfa, vd_djfa_step, vd_similarity, ...);
`VoronoiDiagram` wraps a handle.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "VDError", "load_library", "library_path", "VoronoiDiagram", "EMPTY",
    "vd_config", "vd_halo_plan_t", "vd_create", "vd_destroy", "vd_jfa", "vd_move_seeds",
    "vd_djfa_step", "vd_djfa_step_hash", "vd_stf", "vd_get_labels_into", "vd_similarity", "vd_similarity_host", "vd_label_hash", "vd_get_labels",
    "vd_get_seeds", "vd_band", "vd_last_passes", "vd_last_packed_passes", "vd_synchronize", "vd_set_pass_timing",
    "vd_pass_timing", "vd_pass_times", "vd_launch_count", "vd_schedule_jfa", "vd_schedule_djfa",
    "vd_halo_plan", "vd_nccl_unique_id", "vd_status_str", "vd_set_labels", "vd_pass", "vd_peer_export",
    "vd_peer_attach", "vd_peer_status", "vd_label_hash_async", "EXPORTED_SYMBOLS",
]

EMPTY = 0xFFFFFFFF
_PKG = os.path.dirname(os.path.abspath(__file__))
# Always the in-tree build.  Kernel-variant experiments (scripts/time_variants.py) load
# another build explicitly with _load_variant(path); no environment variable redirects the
# product binding.
_LIB_PATH = os.path.join(_PKG, "libvd.so")
_lib = None

VD_OK, VD_ERR_ARG, VD_ERR_RANGE, VD_ERR_STATE, VD_ERR_CUDA, VD_ERR_NCCL, VD_ERR_OOM = 0, -1, -2, -3, -4, -5, -6


class VDError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        name = _lib.vd_status_str(status).decode() if _lib is not None else str(status)
        super().__init__(f"{where}: {name}" + (f" ({detail})" if detail else ""))


class vd_config(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("extra_passes", ctypes.c_uint32),
        ("virtual_shards", ctypes.c_uint32),
        ("metric", ctypes.c_uint32),
        ("vn_waves", ctypes.c_uint32),
        ("jfa_vn_waves", ctypes.c_uint32),
        ("peer_halos", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32 * 2),
    ]


class vd_halo_plan_t(ctypes.Structure):
    _fields_ = [
        ("recv_top_rank", ctypes.c_int32),
        ("recv_bot_rank", ctypes.c_int32),
        ("halo_rows", ctypes.c_uint32),
        ("top_row0", ctypes.c_int64),
        ("bot_row0", ctypes.c_int64),
        ("send_top_row0", ctypes.c_uint32),
        ("send_bot_row0", ctypes.c_uint32),
    ]


H = ctypes.c_void_p
P = ctypes.c_void_p
_SIGS = {
    "vd_config_init": (None, [ctypes.POINTER(vd_config)]),
    "vd_nccl_unique_id": (ctypes.c_int32, [P]),
    "vd_create": (ctypes.c_int32, [ctypes.POINTER(H), ctypes.c_uint32, ctypes.c_uint64, P, ctypes.POINTER(vd_config)]),
    "vd_jfa": (ctypes.c_int32, [H]),
    "vd_stf": (ctypes.c_int32, [H, ctypes.POINTER(ctypes.c_uint32)]),
    "vd_move_seeds": (ctypes.c_int32, [H, P]),
    "vd_djfa_step": (ctypes.c_int32, [H, P, ctypes.c_uint32]),
    "vd_djfa_step_hash": (ctypes.c_int32, [H, P, ctypes.c_uint32, P]),
    "vd_similarity": (ctypes.c_int32, [H, H, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]),
    "vd_similarity_host": (ctypes.c_int32, [H, P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)]),
    "vd_label_hash": (ctypes.c_int32, [H, ctypes.POINTER(ctypes.c_uint64)]),
    "vd_label_hash_async": (ctypes.c_int32, [H, P]),
    "vd_get_labels": (ctypes.c_int32, [H, P]),
    "vd_get_seeds": (ctypes.c_int32, [H, P]),
    "vd_band": (ctypes.c_int32, [H, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]),
    "vd_last_passes": (ctypes.c_int32, [H, ctypes.POINTER(ctypes.c_uint32)]),
    "vd_last_packed_passes": (ctypes.c_int32, [H, ctypes.POINTER(ctypes.c_uint32)]),
    "vd_synchronize": (ctypes.c_int32, [H]),
    "vd_set_pass_timing": (ctypes.c_int32, [H, ctypes.c_int]),
    "vd_pass_timing": (ctypes.c_int32, [H, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64),
                                        ctypes.POINTER(ctypes.c_uint64)]),
    "vd_pass_times": (ctypes.c_int32, [H, P, P, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]),
    "vd_launch_count": (ctypes.c_int32, [H, ctypes.POINTER(ctypes.c_uint64)]),
    "vd_schedule_jfa": (ctypes.c_int32, [ctypes.c_uint32, ctypes.c_uint32, P, ctypes.c_uint32,
                                         ctypes.POINTER(ctypes.c_uint32)]),
    "vd_schedule_djfa": (ctypes.c_int32, [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, P,
                                          ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]),
    "vd_halo_plan": (ctypes.c_int32, [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.POINTER(vd_halo_plan_t)]),
    "vd_set_labels": (ctypes.c_int32, [H, P]),
    "vd_pass": (ctypes.c_int32, [H, ctypes.c_uint32, ctypes.c_uint32]),
    "vd_peer_export": (ctypes.c_int32, [H, P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "vd_peer_attach": (ctypes.c_int32, [H, P, ctypes.c_size_t]),
    "vd_peer_status": (ctypes.c_int32, [H, ctypes.POINTER(ctypes.c_uint32)]),
    "vd_destroy": (None, [H]),
    "vd_status_str": (ctypes.c_char_p, [ctypes.c_int32]),
    "vd_last_error": (ctypes.c_char_p, [H]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)


def library_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libvd.so (built by paper_2209_00117_b200.build / __graft_entry__.build()).
    Raises if it is missing: there is no fallback implementation."""
    return _load(_LIB_PATH)


def _load_variant(path: str):
    """Experiments only (scripts/time_variants.py): bind a variant build of libvd instead of
    the in-tree one.  Must be called before anything else loads the library."""
    if _lib is not None:
        raise RuntimeError("libvd is already loaded")
    return _load(os.path.abspath(path))


def _load(path: str):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libvd.so not found at {path}: run `python -m paper_2209_00117_b200.build` "
                           "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(st: int, where: str, h=None):
    if st != VD_OK:
        detail = ""
        if h is not None:
            msg = _lib.vd_last_error(h)
            detail = msg.decode() if msg else ""
        raise VDError(st, where, detail)


def _addr(a, dtype, count: int):
    """(pointer, keepalive) for a numpy array or a torch tensor (host or CUDA)."""
    if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):
        import torch
        want = {np.uint16: torch.uint16, np.int16: torch.int16, np.uint32: torch.uint32}[dtype]
        if a.dtype != want or not a.is_contiguous() or a.numel() != count:
            raise ValueError(f"expected a contiguous {want} tensor of {count} elements")
        return ctypes.c_void_p(a.data_ptr()), a
    arr = np.ascontiguousarray(a, dtype=dtype).reshape(-1)
    if arr.size != count:
        raise ValueError(f"expected {count} elements, got {arr.size}")
    return ctypes.c_void_p(arr.ctypes.data), arr


# ------------------------------------------------------------------ raw ABI (same names)

def vd_nccl_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.vd_nccl_unique_id(buf), "vd_nccl_unique_id")
    return buf.raw


METRICS = {"euclid": 0, "manhattan": 1}  # VD_METRIC_* (dJFAe / dJFAm)
VD_PASS_VON_NEUMANN = 1


def vd_create(N: int, seeds_xy, *, device: int = -1, stream: int | None = None, rank: int = 0, world: int = 1,
              nccl_id: bytes | None = None, extra_passes: int = 0, virtual_shards: int = 0, metric: str = "euclid",
              vn_waves: int = 0, jfa_vn_waves: int = 0, peer_halos: bool = False):
    lib = load_library()
    s = (seeds_xy.numel() if hasattr(seeds_xy, "numel") else np.asarray(seeds_xy).size) // 2
    ptr, keep = _addr(seeds_xy, np.uint16, 2 * s)
    cfg = vd_config()
    lib.vd_config_init(ctypes.byref(cfg))
    cfg.device = device
    cfg.stream = stream
    cfg.rank, cfg.world = rank, world
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        cfg.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    cfg.extra_passes = extra_passes
    cfg.virtual_shards = virtual_shards
    cfg.metric = METRICS[metric]
    cfg.vn_waves = vn_waves
    cfg.jfa_vn_waves = jfa_vn_waves
    cfg.peer_halos = 1 if peer_halos else 0
    h = H()
    _check(lib.vd_create(ctypes.byref(h), N, s, ptr, ctypes.byref(cfg)), "vd_create")
    del keep, idbuf
    return h


def vd_destroy(h) -> None:
    if h:
        load_library().vd_destroy(h)


def vd_jfa(h) -> None:
    _check(load_library().vd_jfa(h), "vd_jfa", h)


def vd_stf(h) -> int:
    n = ctypes.c_uint32()
    _check(load_library().vd_stf(h, ctypes.byref(n)), "vd_stf", h)
    return n.value


def vd_move_seeds(h, disp_xy, s: int) -> None:
    ptr, keep = _addr(disp_xy, np.int16, 2 * s)
    _check(load_library().vd_move_seeds(h, ptr), "vd_move_seeds", h)
    del keep


def vd_djfa_step(h, disp_xy, d_max: int, s: int) -> None:
    ptr, keep = _addr(disp_xy, np.int16, 2 * s)
    _check(load_library().vd_djfa_step(h, ptr, d_max), "vd_djfa_step", h)
    del keep


def vd_djfa_step_hash(h, disp_xy, d_max: int, s: int, pinned_out: int) -> None:
    """vd_djfa_step + the new diagram's label checksum into pinned host memory at pinned_out
    (e.g. a pinned torch.int64 tensor's data_ptr()); enqueue only."""
    ptr, keep = _addr(disp_xy, np.int16, 2 * s)
    _check(load_library().vd_djfa_step_hash(h, ptr, d_max, ctypes.c_void_p(pinned_out)), "vd_djfa_step_hash", h)
    del keep


def vd_set_labels(h, labels: np.ndarray) -> None:
    arr = np.ascontiguousarray(labels, dtype=np.uint32)
    _check(load_library().vd_set_labels(h, ctypes.c_void_p(arr.ctypes.data)), "vd_set_labels", h)


def vd_peer_export(h) -> bytes:
    lib = load_library()
    n = ctypes.c_size_t()
    _check(lib.vd_peer_export(h, None, 0, ctypes.byref(n)), "vd_peer_export", h)
    buf = ctypes.create_string_buffer(n.value)
    _check(lib.vd_peer_export(h, ctypes.cast(buf, ctypes.c_void_p), n.value, ctypes.byref(n)), "vd_peer_export", h)
    return buf.raw[:n.value]


def vd_peer_attach(h, blobs: list[bytes]) -> None:
    """blobs: every rank's vd_peer_export() result, in rank order."""
    each = len(blobs[0])
    allb = ctypes.create_string_buffer(b"".join(blobs), each * len(blobs))
    _check(load_library().vd_peer_attach(h, ctypes.cast(allb, ctypes.c_void_p), each), "vd_peer_attach", h)


def vd_peer_status(h) -> bool:
    t = ctypes.c_uint32()
    _check(load_library().vd_peer_status(h, ctypes.byref(t)), "vd_peer_status", h)
    return bool(t.value)


def vd_pass(h, k: int, von_neumann: bool = False) -> None:
    _check(load_library().vd_pass(h, k, VD_PASS_VON_NEUMANN if von_neumann else 0), "vd_pass", h)


def vd_similarity(h, ref) -> tuple[float, int]:
    pct, m = ctypes.c_double(), ctypes.c_uint64()
    _check(load_library().vd_similarity(h, ref, ctypes.byref(pct), ctypes.byref(m)), "vd_similarity", h)
    return pct.value, m.value


def vd_similarity_host(h, ref_labels: np.ndarray) -> tuple[float, int]:
    ref = np.ascontiguousarray(ref_labels, dtype=np.uint32)
    pct, m = ctypes.c_double(), ctypes.c_uint64()
    _check(load_library().vd_similarity_host(h, ctypes.c_void_p(ref.ctypes.data), ctypes.byref(pct),
                                             ctypes.byref(m)), "vd_similarity_host", h)
    return pct.value, m.value


def vd_label_hash(h) -> int:
    v = ctypes.c_uint64()
    _check(load_library().vd_label_hash(h, ctypes.byref(v)), "vd_label_hash", h)
    return v.value


def vd_label_hash_async(h, pinned_ptr: int) -> None:
    """Enqueue the checksum; it lands at pinned_ptr (page-locked host memory) asynchronously."""
    _check(load_library().vd_label_hash_async(h, ctypes.c_void_p(pinned_ptr)), "vd_label_hash_async", h)


def vd_band(h) -> tuple[int, int]:
    r0, n = ctypes.c_uint32(), ctypes.c_uint32()
    _check(load_library().vd_band(h, ctypes.byref(r0), ctypes.byref(n)), "vd_band", h)
    return r0.value, n.value


def vd_get_labels(h, N: int) -> np.ndarray:
    _, rows = vd_band(h)
    out = np.empty((rows, N), dtype=np.uint32)
    _check(load_library().vd_get_labels(h, ctypes.c_void_p(out.ctypes.data)), "vd_get_labels", h)
    return out


def vd_get_labels_into(h, ptr: int) -> None:
    """vd_get_labels into caller memory at address ptr (e.g. a pinned torch tensor's
    data_ptr(), rows x N uint32 of this handle's band)."""
    _check(load_library().vd_get_labels(h, ctypes.c_void_p(ptr)), "vd_get_labels", h)


def vd_get_seeds(h, s: int) -> np.ndarray:
    out = np.empty(2 * s, dtype=np.uint16)
    _check(load_library().vd_get_seeds(h, ctypes.c_void_p(out.ctypes.data)), "vd_get_seeds", h)
    return out


def vd_last_passes(h) -> int:
    v = ctypes.c_uint32()
    _check(load_library().vd_last_passes(h, ctypes.byref(v)), "vd_last_passes", h)
    return v.value


def vd_last_packed_passes(h) -> int:
    v = ctypes.c_uint32()
    _check(load_library().vd_last_packed_passes(h, ctypes.byref(v)), "vd_last_packed_passes", h)
    return v.value


def vd_synchronize(h) -> None:
    _check(load_library().vd_synchronize(h), "vd_synchronize", h)


def vd_set_pass_timing(h, enable: bool) -> None:
    _check(load_library().vd_set_pass_timing(h, int(enable)), "vd_set_pass_timing", h)


def vd_pass_timing(h) -> tuple[float, int, int]:
    ms, n, px = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64()
    _check(load_library().vd_pass_timing(h, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(px)),
           "vd_pass_timing", h)
    return ms.value, n.value, px.value


def vd_pass_times(h) -> list[tuple[int, float]]:
    """(k, ms) of every timed jump pass since the last vd_pass_timing (no reset)."""
    lib = load_library()
    n = ctypes.c_uint32()
    _check(lib.vd_pass_times(h, None, None, 0, ctypes.byref(n)), "vd_pass_times", h)
    ms = np.zeros(n.value, dtype=np.float32)
    ks = np.zeros(n.value, dtype=np.uint32)
    _check(lib.vd_pass_times(h, ctypes.c_void_p(ms.ctypes.data), ctypes.c_void_p(ks.ctypes.data), n.value,
                             ctypes.byref(n)), "vd_pass_times", h)
    return [(int(k), float(t)) for k, t in zip(ks, ms)]


def vd_launch_count(h) -> int:
    v = ctypes.c_uint64()
    _check(load_library().vd_launch_count(h, ctypes.byref(v)), "vd_launch_count", h)
    return v.value


def vd_schedule_jfa(N: int, extras: int = 0) -> list[int]:
    ks = (ctypes.c_uint32 * 64)()
    n = ctypes.c_uint32()
    _check(load_library().vd_schedule_jfa(N, extras, ks, 64, ctypes.byref(n)), "vd_schedule_jfa")
    return list(ks[: n.value])


def vd_schedule_djfa(N: int, s: int, d_max: int, extras: int = 0) -> list[int]:
    ks = (ctypes.c_uint32 * 64)()
    n = ctypes.c_uint32()
    _check(load_library().vd_schedule_djfa(N, s, d_max, extras, ks, 64, ctypes.byref(n)), "vd_schedule_djfa")
    return list(ks[: n.value])


def vd_halo_plan(N: int, world: int, rank: int, k: int) -> dict:
    p = vd_halo_plan_t()
    _check(load_library().vd_halo_plan(N, world, rank, k, ctypes.byref(p)), "vd_halo_plan")
    return {f: getattr(p, f) for f, _ in vd_halo_plan_t._fields_}


def vd_status_str(st: int) -> str:
    return load_library().vd_status_str(st).decode()


# ------------------------------------------------------------------ convenience wrapper

class VoronoiDiagram:
    """One diagram context (vd_create ... vd_destroy).

    >>> vd = VoronoiDiagram(N, seeds_xy)        # seeds: uint16 x0,y0,x1,y1,...
    >>> vd.jfa()                                # full JFA (Eq. 2 schedule)
    >>> vd.djfa_step(disp_xy, d_max)            # one dJFA time step (Alg. 1)
    >>> vd.similarity(other)                    # Eq. 5, percent
    """

    def __init__(self, N: int, seeds_xy, **cfg):
        self.N = int(N)
        self.s = (seeds_xy.numel() if hasattr(seeds_xy, "numel") else np.asarray(seeds_xy).size) // 2
        self.h = vd_create(self.N, seeds_xy, **cfg)

    def close(self):
        if self.h:
            vd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def jfa(self):
        vd_jfa(self.h)

    def stf(self) -> int:
        return vd_stf(self.h)

    def move_seeds(self, disp_xy):
        vd_move_seeds(self.h, disp_xy, self.s)

    def djfa_step(self, disp_xy, d_max: int):
        vd_djfa_step(self.h, disp_xy, d_max, self.s)

    def similarity(self, other: "VoronoiDiagram") -> float:
        return vd_similarity(self.h, other.h)[0]

    def match_count(self, other: "VoronoiDiagram") -> int:
        return vd_similarity(self.h, other.h)[1]

    def similarity_host(self, ref_labels) -> float:
        return vd_similarity_host(self.h, ref_labels)[0]

    def label_hash(self) -> int:
        return vd_label_hash(self.h)

    def set_labels(self, labels):
        vd_set_labels(self.h, labels)

    def attach_peers(self, group=None):
        """Peer halos across processes: all-gather the IPC blobs over `group` (torch.distributed,
        any backend) and attach the neighbouring bands (vd_peer_attach)."""
        import torch.distributed as dist
        blobs = [None] * dist.get_world_size(group)
        dist.all_gather_object(blobs, vd_peer_export(self.h), group=group)
        vd_peer_attach(self.h, blobs)

    def peer_timed_out(self) -> bool:
        return vd_peer_status(self.h)

    def jump_pass(self, k: int, von_neumann: bool = False):
        vd_pass(self.h, k, von_neumann)

    def labels(self) -> np.ndarray:
        return vd_get_labels(self.h, self.N)

    def seeds(self) -> np.ndarray:
        return vd_get_seeds(self.h, self.s)

    def band(self) -> tuple[int, int]:
        return vd_band(self.h)

    def last_passes(self) -> int:
        return vd_last_passes(self.h)

    def last_packed_passes(self) -> int:
        return vd_last_packed_passes(self.h)

    def synchronize(self):
        vd_synchronize(self.h)

    def set_pass_timing(self, enable: bool):
        vd_set_pass_timing(self.h, enable)

    def pass_timing(self):
        return vd_pass_timing(self.h)

    def pass_times(self):
        return vd_pass_times(self.h)

    def launch_count(self) -> int:
        return vd_launch_count(self.h)
