"""Thin ctypes binding of libfastrs.so (include/fastrs.h) — argument marshalling only.

Every step of the computation runs in the CUDA kernels behind the C ABI; this module only
turns torch CUDA tensors into raw device pointers + the current stream, sizes and caches
the device workspace, and maps status codes to exceptions.  There is no CPU fallback: if
the library cannot be loaded, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

from . import _build

BORDER_BACKGROUND = 1
DETERMINISTIC = 2
ASYNC = 4
HOST_IO = 8
FORCE_FALLBACK = 16  # run the dilation with the atomic sparse-table kernel (cross-check)
APPROX_LT = 256  # approximate local thickness (FASTRS_APPROX_LT)
NO_LIST_STAGING = 1024  # test hook: K5a list overflow takes the regather pass instead of staging
NO_COVER_CUT = 2048  # test hook: K5a keeps every reaching ball (no cover cut)
EXACT_PRUNE = 4096  # K4 tests every |s|^2 <= 12 offset class (the exact kept set)
TILE_RECORD_WORDS = 20  # FASTRS_TILE_RECORD_WORDS: u32 per tile record of slab_pack_tiles

STAGES = ("edt_x", "edt_y", "edt_z", "prune", "dilate", "metrics", "epilogue", "gather")

_STATUS = {0: "OK", 1: "EINVAL", 2: "ENOSITE", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "EINTERNAL"}

_lock = threading.Lock()
_lib = None


class FastrsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fastrs {_STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = _STATUS.get(code, str(code))


class _Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("volume", "n_shell", "max_lt2", "mean_lt", "max_lt",
                                               "shell_mean_lt", "axis_a", "axis_cb")]


class _Diag(ctypes.Structure):
    _fields_ = [("status_bits", ctypes.c_uint32), ("dmax", ctypes.c_uint32), ("n_fg", ctypes.c_uint64),
                ("n_kept", ctypes.c_uint64), ("n_intervals", ctypes.c_uint64),
                ("sum_scale_log2", ctypes.c_int32), ("n_fallback", ctypes.c_uint32),
                ("n_rounds_extra", ctypes.c_uint32), ("n_regathers", ctypes.c_uint32),
                ("max_group_list", ctypes.c_uint32), ("sum_group_list", ctypes.c_uint64),
                ("n_painted", ctypes.c_uint64), ("n_covering", ctypes.c_uint64),
                ("n_staged", ctypes.c_uint32), ("n_deferred", ctypes.c_uint32),
                ("n_col_slow", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class _SlabInfo(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("h", ctypes.c_int64), ("H", ctypes.c_int64), ("dxy_max", ctypes.c_uint32),
                ("dmax", ctypes.c_uint32), ("bytes_sent", ctypes.c_uint64), ("bytes_received", ctypes.c_uint64)]


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load libfastrs.so (built in-tree).  Raises if it cannot be built or loaded."""
    global _lib
    with _lock:
        if _lib is None:
            if build_if_missing and not _build.up_to_date():
                _build.build()
            if not os.path.exists(_build.SO):
                raise ImportError(f"libfastrs.so missing at {_build.SO}; run __graft_entry__.build()")
            lib = ctypes.CDLL(_build.SO)
            vp, i64, i32, u32, ci, cd, sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32,
                                              ctypes.c_int, ctypes.c_double, ctypes.c_size_t)
            lib.fastrs_workspace_bytes.argtypes = [vp, ci, i64, i32, u32, ctypes.POINTER(sz)]
            lib.fastrs_edt_sq.argtypes = [vp, vp, ci, i64, u32, vp, vp, sz, vp]
            lib.fastrs_local_thickness.argtypes = [vp, vp, ci, i64, u32, vp, vp, vp, sz, vp]
            lib.fastrs_sphericity_roundness.argtypes = [vp, vp, ci, i64, i32, u32, vp, vp, vp, vp, sz, vp]
            lib.fastrs_sphericity_roundness_host.argtypes = [vp, vp, ci, i64, i32, u32, vp, vp, vp, sz, vp]
            lib.fastrs_read_diagnostics.argtypes = [vp, ctypes.POINTER(_Diag), vp]
            lib.fastrs_profile.argtypes = [ci]
            lib.fastrs_profile.restype = None
            lib.fastrs_profile_read.argtypes = [vp, vp, ci]
            lib.fastrs_last_error.restype = ctypes.c_char_p
            lib.fastrs_release.restype = None
            for n in ("spheroid_area", "ramanujan_perimeter", "sphericity_3d", "sphericity_2d"):
                f = getattr(lib, "fastrs_" + n)
                f.argtypes = [cd, cd]
                f.restype = cd
            lib.fastrs_slab_workspace_bytes.argtypes = [vp, ctypes.POINTER(sz)]
            lib.fastrs_slab_edt_xy.argtypes = [vp, vp, vp, i32, u32, vp, vp, vp, sz, vp]
            lib.fastrs_slab_edt_z.argtypes = [vp, vp, i64, i64, i64, i64, u32, vp, vp, vp, sz, vp]
            lib.fastrs_slab_reduce.argtypes = [vp, vp, vp, i64, i64, i64, u32, i32, u32, vp, vp, vp, vp, vp, vp,
                                               sz, vp]
            lib.fastrs_metrics_from_partials.argtypes = [vp, vp, vp, vp, vp, i64, ci, i64, u32, vp, vp, vp, vp,
                                                         sz, vp]
            lib.fastrs_slab_prune.argtypes = [vp, vp, i64, i64, u32, vp, sz, vp]
            lib.fastrs_slab_pack_tiles.argtypes = [vp, vp, i64, i64, vp, vp, vp, vp]
            lib.fastrs_slab_unpack_tiles.argtypes = [vp, vp, i64, i64, vp, vp, vp]
            lib.fastrs_slab_dilate.argtypes = [vp, vp, vp, i64, i64, i64, u32, i32, u32, vp, vp, vp, vp, vp, vp, sz, vp]
            lib.fastrs_nccl_available.argtypes = []
            lib.fastrs_nccl_unique_id.argtypes = [vp]
            lib.fastrs_comm_init.argtypes = [vp, ci, ci, ctypes.POINTER(vp)]
            lib.fastrs_comm_destroy.argtypes = [vp]
            lib.fastrs_slab_partition.argtypes = [i64, ci, vp]
            lib.fastrs_slab_halo_plan.argtypes = [vp, ci, i64, i64, vp, i64, ctypes.POINTER(i64)]
            lib.fastrs_slab_call_workspace_bytes.argtypes = [vp, i64, i64, ci, ci, i32, i64, u32, ctypes.POINTER(sz)]
            lib.fastrs_sphericity_roundness_slab.argtypes = [vp, vp, i64, i64, i32, u32, i64, vp, vp, vp,
                                                             ctypes.POINTER(_SlabInfo), vp, vp, sz, vp]
            lib.fastrs_ccl_workspace_bytes.argtypes = [vp, ci, i64, ctypes.POINTER(sz)]
            lib.fastrs_label_components.argtypes = [vp, vp, ci, i64, ci, vp, vp, vp, sz, vp]
            lib.fastrs_wl_workspace_bytes.argtypes = [i64, i32, ctypes.POINTER(sz)]
            lib.fastrs_sphericity_wl.argtypes = [vp, vp, ci, i64, i32, vp, vp, vp, vp, sz, vp]
            lib.fastrs_mc_workspace_bytes.argtypes = [i64, i32, ctypes.POINTER(sz)]
            lib.fastrs_mc_measure.argtypes = [vp, vp, ci, i64, i32, vp, vp, vp, sz, vp]
            lib.fastrs_touches_edge.argtypes = [vp, vp, ci, i64, i32, vp, u32, vp]
            lib.fastrs_filter_objects.argtypes = [vp, vp, vp, vp, i64, i64, u32, vp]
            for n in ("workspace_bytes", "edt_sq", "local_thickness", "sphericity_roundness",
                      "sphericity_roundness_host", "read_diagnostics", "profile_read", "slab_workspace_bytes",
                      "slab_edt_xy", "slab_edt_z", "slab_reduce", "metrics_from_partials", "touches_edge",
                      "filter_objects", "nccl_available", "nccl_unique_id", "comm_init", "comm_destroy",
                      "slab_partition", "slab_halo_plan", "slab_call_workspace_bytes", "slab_prune",
                      "slab_pack_tiles", "slab_unpack_tiles", "slab_dilate",
                      "sphericity_roundness_slab", "ccl_workspace_bytes", "label_components",
                      "wl_workspace_bytes", "sphericity_wl", "mc_workspace_bytes", "mc_measure"):
                getattr(lib, "fastrs_" + n).restype = ci
            _lib = lib
    return _lib


def _check(rc: int):
    if rc != 0:
        raise FastrsError(rc, load().fastrs_last_error().decode(errors="replace"))


def _geometry(shape, ndim, batch):
    shape = tuple(int(s) for s in shape)
    if ndim is None:
        if len(shape) not in (2, 3):
            raise ValueError("pass ndim= for batched input")
        ndim = len(shape)
    if len(shape) == ndim:
        b = 1
    elif len(shape) == ndim + 1:
        b = shape[0]
    else:
        raise ValueError(f"labels of shape {shape} do not match ndim={ndim}")
    if batch is not None and batch != b:
        raise ValueError("batch does not match the labels' shape")
    dims = (ctypes.c_int64 * ndim)(*shape[-ndim:])
    return ndim, b, dims


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def workspace_bytes(shape, ndim=None, max_label=0, flags=0) -> int:
    ndim, b, dims = _geometry(shape, ndim, None)
    out = ctypes.c_size_t(0)
    _check(load().fastrs_workspace_bytes(dims, ndim, b, int(max_label), flags, ctypes.byref(out)))
    return out.value


_ws_cache: dict = {}


def workspace(nbytes: int, device) -> torch.Tensor:
    """Cached per-device workspace (grown on demand; 256-byte aligned by the allocator)."""
    device = torch.device(device)
    key = device.index if device.index is not None else torch.cuda.current_device()
    t = _ws_cache.get(key)
    if t is None or t.numel() < nbytes:
        _ws_cache.pop(key, None)
        t = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = t
    return t


def _labels_arg(labels: torch.Tensor) -> torch.Tensor:
    if not isinstance(labels, torch.Tensor) or not labels.is_cuda:
        raise TypeError("labels must be a CUDA torch.Tensor (use sphericity_roundness_host for host arrays)")
    if labels.dtype != torch.int32:
        raise TypeError("labels must be int32")
    return labels.contiguous()


def edt_sq(labels: torch.Tensor, ndim=None, flags=BORDER_BACKGROUND, out=None, ws=None) -> torch.Tensor:
    """Exact squared label-aware EDT (int32 tensor holding the uint32 D; 0 on background)."""
    labels = _labels_arg(labels)
    ndim, b, dims = _geometry(labels.shape, ndim, None)
    if out is None:
        out = torch.empty_like(labels)
    nb = workspace_bytes(labels.shape, ndim, 0, flags)
    ws = workspace(nb, labels.device) if ws is None else ws
    _check(load().fastrs_edt_sq(labels.data_ptr(), dims, ndim, b, flags, out.data_ptr(), ws.data_ptr(),
                                ws.numel(), _stream(labels.device)))
    return out


def local_thickness(labels: torch.Tensor, ndim=None, flags=BORDER_BACKGROUND, lt2=True, lt=False, ws=None):
    """Exact local thickness.  Returns LT^2 (int32 tensor), the float32 radius, or both."""
    labels = _labels_arg(labels)
    ndim, b, dims = _geometry(labels.shape, ndim, None)
    o2 = torch.empty_like(labels) if lt2 else None
    o1 = torch.empty(labels.shape, dtype=torch.float32, device=labels.device) if lt else None
    nb = workspace_bytes(labels.shape, ndim, 0, flags)
    ws = workspace(nb, labels.device) if ws is None else ws
    _check(load().fastrs_local_thickness(labels.data_ptr(), dims, ndim, b, flags,
                                         None if o2 is None else o2.data_ptr(),
                                         None if o1 is None else o1.data_ptr(), ws.data_ptr(), ws.numel(),
                                         _stream(labels.device)))
    if lt2 and lt:
        return o2, o1
    return o2 if lt2 else o1


def sphericity_roundness(labels: torch.Tensor, max_label=None, ndim=None, flags=BORDER_BACKGROUND,
                         stats=False, ws=None, out=None) -> dict:
    """Per-object sphericity and roundness (float64 tensors of batch*max_label entries,
    index b*max_label + label-1).  With stats=True also the per-label statistics."""
    labels = _labels_arg(labels)
    ndim, b, dims = _geometry(labels.shape, ndim, None)
    if max_label is None:
        max_label = max(1, int(labels.max().item()))
    M = b * max_label
    dev = labels.device
    res = out if out is not None else {}
    if "sphericity" not in res:
        res["sphericity"] = torch.empty(M, dtype=torch.float64, device=dev)
        res["roundness"] = torch.empty(M, dtype=torch.float64, device=dev)
    st = None
    if stats:
        for k, dt in (("volume", torch.int64), ("n_shell", torch.int64), ("max_lt2", torch.int32),
                      ("mean_lt", torch.float64), ("max_lt", torch.float64), ("shell_mean_lt", torch.float64),
                      ("axis_a", torch.float64), ("axis_cb", torch.float64)):
            if k not in res:
                res[k] = torch.empty(M, dtype=dt, device=dev)
        st = _Stats(*[res[n].data_ptr() for n, _ in _Stats._fields_])
    nb = workspace_bytes(labels.shape, ndim, max_label, flags)
    ws = workspace(nb, dev) if ws is None else ws
    _check(load().fastrs_sphericity_roundness(labels.data_ptr(), dims, ndim, b, int(max_label), flags,
                                              res["sphericity"].data_ptr(), res["roundness"].data_ptr(),
                                              None if st is None else ctypes.byref(st), ws.data_ptr(),
                                              ws.numel(), _stream(dev)))
    return res


def sphericity_roundness_host(labels, max_label: int, ndim=None, flags=BORDER_BACKGROUND, device="cuda",
                              ws=None, out=None):
    """End-to-end entry point with HOST buffers: labels (numpy or pinned CPU tensor) are
    copied to the device inside the C call; results come back as numpy float64 arrays."""
    if isinstance(labels, torch.Tensor):
        if labels.is_cuda or labels.dtype != torch.int32:
            raise TypeError("labels must be a CPU int32 tensor or numpy array")
        ptr, shape = labels.data_ptr(), labels.shape
    else:
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        ptr, shape = labels.ctypes.data, labels.shape
    ndim, b, dims = _geometry(shape, ndim, None)
    M = b * max_label
    if out is None:
        out = (np.empty(M), np.empty(M))
    nb = workspace_bytes(shape, ndim, max_label, flags | HOST_IO)
    dev = torch.device(device)
    ws = workspace(nb, dev) if ws is None else ws
    _check(load().fastrs_sphericity_roundness_host(ptr, dims, ndim, b, int(max_label), flags,
                                                   out[0].ctypes.data, out[1].ctypes.data, ws.data_ptr(),
                                                   ws.numel(), _stream(dev)))
    return out


def diagnostics(ws: torch.Tensor) -> dict:
    d = _Diag()
    _check(load().fastrs_read_diagnostics(ws.data_ptr(), ctypes.byref(d), _stream(ws.device)))
    return {n: getattr(d, n) for n, _ in _Diag._fields_}


def last_workspace(device=None) -> torch.Tensor:
    device = torch.device(device or "cuda")
    key = device.index if device.index is not None else torch.cuda.current_device()
    return _ws_cache[key]


def profile(enable: bool):
    load().fastrs_profile(1 if enable else 0)


def profile_read() -> tuple[dict, int]:
    ms = (ctypes.c_double * len(STAGES))()
    calls = ctypes.c_int64(0)
    load().fastrs_profile_read(ms, ctypes.byref(calls), len(STAGES))
    return {s: ms[i] for i, s in enumerate(STAGES)}, calls.value


# ------------------------------------------------------------------------------------------
# z-slab phases (include/fastrs.h "multi-GPU z-slab path"); slab.py orchestrates them
# ------------------------------------------------------------------------------------------

PARTIAL_KEYS = ("vol", "n_shell", "sum_lt", "sum_shell_lt", "max_lt2")


def _dims3(shape):
    return (ctypes.c_int64 * 3)(*[int(v) for v in shape])


def slab_workspace(dims_ext, device) -> torch.Tensor:
    out = ctypes.c_size_t(0)
    _check(load().fastrs_slab_workspace_bytes(_dims3(dims_ext), ctypes.byref(out)))
    return workspace(out.value, device)


def workspace_for_slab(dims_ext, device) -> torch.Tensor:
    """A fresh (uncached) slab-phase workspace: the kept-centre halo phases keep tile data in it
    between calls, one per (virtual) rank."""
    out = ctypes.c_size_t(0)
    _check(load().fastrs_slab_workspace_bytes(_dims3(dims_ext), ctypes.byref(out)))
    return torch.empty(out.value, dtype=torch.uint8, device=device)


def _ptr_or_none(t):
    return None if t is None else t.data_ptr()


def slab_edt_xy(labels: torch.Tensor, labels_below, max_label: int, flags=BORDER_BACKGROUND, ws=None):
    """Phase A: x/y passes of the own slab.  Returns (packed int32 [nz,Y,X], dxy_max int32[1])."""
    labels = _labels_arg(labels)
    packed = torch.empty_like(labels)
    dxy = torch.zeros(1, dtype=torch.int32, device=labels.device)
    ws = slab_workspace(labels.shape, labels.device) if ws is None else ws
    below = None if labels_below is None else _labels_arg(labels_below)
    _check(load().fastrs_slab_edt_xy(labels.data_ptr(), _ptr_or_none(below), _dims3(labels.shape), int(max_label),
                                     flags, packed.data_ptr(), dxy.data_ptr(), ws.data_ptr(), ws.numel(),
                                     _stream(labels.device)))
    return packed, dxy


def slab_edt_z(packed_ext: torch.Tensor, own_lo: int, own_hi: int, z_ext0: int, Z: int, flags=BORDER_BACKGROUND,
               out=None, ws=None):
    """Phase B: z pass over the h-extended slab.  Returns (D int32 [own_hi-own_lo,Y,X], dmax int32[1])."""
    packed_ext = packed_ext.contiguous()
    _, Y, X = packed_ext.shape
    d = torch.empty((own_hi - own_lo, Y, X), dtype=torch.int32, device=packed_ext.device) if out is None else out
    dmax = torch.zeros(1, dtype=torch.int32, device=packed_ext.device)
    ws = slab_workspace(packed_ext.shape, packed_ext.device) if ws is None else ws
    _check(load().fastrs_slab_edt_z(packed_ext.data_ptr(), _dims3(packed_ext.shape), own_lo, own_hi, z_ext0, Z,
                                    flags, d.data_ptr(), dmax.data_ptr(), ws.data_ptr(), ws.numel(),
                                    _stream(packed_ext.device)))
    return d, dmax


def slab_reduce(labels: torch.Tensor, d_ext: torch.Tensor, own_lo: int, own_hi: int, Z: int, dmax_global: int,
                max_label: int, flags=BORDER_BACKGROUND, ws=None) -> dict:
    """Phase C: prune + dilation + shell + partial per-label sums of the own slab.  Returns
    int64 tensors vol, n_shell (max_label), sum_lt, sum_shell_lt (2*max_label: the hi | lo words
    of the 2^-32 fixed-point sums; u64 bit patterns) and int32 max_lt2."""
    labels = _labels_arg(labels)
    d_ext = d_ext.contiguous()
    dev = labels.device
    part = {k: torch.empty(max_label * (2 if k.startswith("sum") else 1), dtype=torch.int64, device=dev)
            for k in PARTIAL_KEYS[:4]}
    part["max_lt2"] = torch.empty(max_label, dtype=torch.int32, device=dev)
    ws = slab_workspace(d_ext.shape, dev) if ws is None else ws
    _check(load().fastrs_slab_reduce(labels.data_ptr(), d_ext.data_ptr(), _dims3(d_ext.shape), own_lo, own_hi, Z,
                                     int(dmax_global), int(max_label), flags,
                                     *[part[k].data_ptr() for k in PARTIAL_KEYS], ws.data_ptr(), ws.numel(),
                                     _stream(dev)))
    return part


def _new_partials(max_label: int, dev) -> dict:
    part = {k: torch.empty(max_label * (2 if k.startswith("sum") else 1), dtype=torch.int64, device=dev)
            for k in PARTIAL_KEYS[:4]}
    part["max_lt2"] = torch.empty(max_label, dtype=torch.int32, device=dev)
    return part


def slab_prune(d_ext: torch.Tensor, own_lo: int, own_hi: int, ws: torch.Tensor, flags=BORDER_BACKGROUND):
    """Phase C1 (kept-centre halo): K4 on the own tile layers of the extended slab into `ws`."""
    d_ext = d_ext.contiguous()
    _check(load().fastrs_slab_prune(d_ext.data_ptr(), _dims3(d_ext.shape), own_lo, own_hi, flags, ws.data_ptr(),
                                    ws.numel(), _stream(d_ext.device)))


def slab_pack_tiles(ws: torch.Tensor, dims_ext, tz_a: int, tz_b: int):
    """K4 outputs of tile layers [tz_a, tz_b) of `ws`: (records int32 [tiles*12], centres int64 [n])."""
    dev = ws.device
    Y, X = int(dims_ext[1]), int(dims_ext[2])
    tiles = (tz_b - tz_a) * ((Y + 7) // 8) * ((X + 31) // 32)
    rec = torch.empty(tiles * TILE_RECORD_WORDS, dtype=torch.int32, device=dev)
    ent = torch.empty(tiles * 2048, dtype=torch.int64, device=dev)
    n = torch.zeros(1, dtype=torch.int64, device=dev)
    _check(load().fastrs_slab_pack_tiles(ws.data_ptr(), _dims3(dims_ext), tz_a, tz_b, rec.data_ptr(), ent.data_ptr(),
                                         n.data_ptr(), _stream(dev)))
    return rec, ent[:int(n.item())].clone()


def slab_unpack_tiles(ws: torch.Tensor, dims_ext, tz_a: int, tz_b: int, rec: torch.Tensor, ent: torch.Tensor):
    ent = ent if ent.numel() else torch.zeros(1, dtype=torch.int64, device=ws.device)
    _check(load().fastrs_slab_unpack_tiles(ws.data_ptr(), _dims3(dims_ext), tz_a, tz_b, rec.data_ptr(),
                                           ent.data_ptr(), _stream(ws.device)))


def slab_dilate(labels: torch.Tensor, d_ext: torch.Tensor, own_lo: int, own_hi: int, Z: int, dmax_global: int,
                max_label: int, ws: torch.Tensor, flags=BORDER_BACKGROUND) -> dict:
    """Phase C2 (kept-centre halo): K5 on the own tiles from the tile data in `ws` -> partials."""
    labels = _labels_arg(labels)
    d_ext = d_ext.contiguous()
    part = _new_partials(int(max_label), labels.device)
    _check(load().fastrs_slab_dilate(labels.data_ptr(), d_ext.data_ptr(), _dims3(d_ext.shape), own_lo, own_hi, Z,
                                     int(dmax_global), int(max_label), flags,
                                     *[part[k].data_ptr() for k in PARTIAL_KEYS], ws.data_ptr(), ws.numel(),
                                     _stream(labels.device)))
    return part


def metrics_from_partials(part: dict, ndim: int, nscale: int, dmax_global: int, stats=False, ws=None) -> dict:
    """Phase D: closed forms per label from (reduced) partials."""
    dev = part["vol"].device
    M = part["vol"].numel()
    res = {"sphericity": torch.empty(M, dtype=torch.float64, device=dev),
           "roundness": torch.empty(M, dtype=torch.float64, device=dev)}
    st = None
    if stats:
        for k, dt in (("volume", torch.int64), ("n_shell", torch.int64), ("max_lt2", torch.int32),
                      ("mean_lt", torch.float64), ("max_lt", torch.float64), ("shell_mean_lt", torch.float64),
                      ("axis_a", torch.float64), ("axis_cb", torch.float64)):
            res[k] = torch.empty(M, dtype=dt, device=dev)
        st = _Stats(*[res[n].data_ptr() for n, _ in _Stats._fields_])
    ws = workspace(256, dev) if ws is None else ws
    _check(load().fastrs_metrics_from_partials(*[part[k].contiguous().data_ptr() for k in PARTIAL_KEYS], M, ndim,
                                               int(nscale), int(dmax_global), res["sphericity"].data_ptr(),
                                               res["roundness"].data_ptr(), None if st is None else ctypes.byref(st),
                                               ws.data_ptr(), ws.numel(), _stream(dev)))
    return res


EDGE_SKIP_ZLO, EDGE_SKIP_ZHI = 32, 64


def touches_edge(labels: torch.Tensor, max_label: int, ndim=None, flags: int = 0) -> torch.Tensor:
    """uint8 flags (batch*max_label): 1 where a label has an element on its item's grid boundary
    (fastrs_touches_edge).  flags: EDGE_SKIP_ZLO / EDGE_SKIP_ZHI for a
    z-slab whose first / last slice is not a face of the whole volume."""
    labels = _labels_arg(labels)
    ndim, b, dims = _geometry(labels.shape, ndim, None)
    out = torch.empty(b * int(max_label), dtype=torch.uint8, device=labels.device)
    _check(load().fastrs_touches_edge(labels.data_ptr(), dims, ndim, b, int(max_label), out.data_ptr(), int(flags),
                                      _stream(labels.device)))
    return out


def filter_objects(res: dict, min_volume=None, edge=None) -> dict:
    """The paper's analysis filters, in place on a result dict of sphericity_roundness(stats=True
    when min_volume is given): NaN metrics for labels with volume < min_volume and,
    with edge = touches_edge(...), for labels on the grid boundary."""
    sph, rnd = res["sphericity"], res["roundness"]
    vol = None
    if min_volume is not None:
        if "volume" not in res:
            raise ValueError("min_volume needs the stats of sphericity_roundness(stats=True)")
        vol = res["volume"]
    _check(load().fastrs_filter_objects(sph.data_ptr(), rnd.data_ptr(), None if vol is None else vol.data_ptr(),
                                        None if edge is None else edge.data_ptr(), sph.numel(),
                                        int(min_volume or 0), 0, _stream(sph.device)))
    return res


def spheroid_area(a, c):
    return load().fastrs_spheroid_area(a, c)


def ramanujan_perimeter(a, b):
    return load().fastrs_ramanujan_perimeter(a, b)


def sphericity_3d(V, mean_lt):
    return load().fastrs_sphericity_3d(V, mean_lt)


def sphericity_2d(A, mean_lt):
    return load().fastrs_sphericity_2d(A, mean_lt)


def release():
    load().fastrs_release()


# ------------------------------------------------------------------------------------------
# multi-GPU z-slab call with NCCL inside the library (include/fastrs.h
# fastrs_sphericity_roundness_slab); slab.py builds the communicator
# ------------------------------------------------------------------------------------------

SLAB_TRANSPOSE = 128
SLAB_DENSE_HALO = 512


def nccl_available() -> bool:
    return bool(load().fastrs_nccl_available())


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().fastrs_nccl_unique_id(buf))
    return buf.raw


class Comm:
    """An NCCL communicator owned by libfastrs (fastrs_comm_init on the current device)."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        self.handle = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        _check(load().fastrs_comm_init(buf, int(nranks), int(rank), ctypes.byref(self.handle)))
        self.nranks, self.rank = int(nranks), int(rank)

    def close(self):
        if self.handle:
            _check(load().fastrs_comm_destroy(self.handle))
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slab_partition(Z: int, nranks: int) -> list:
    b = (ctypes.c_int64 * (nranks + 1))()
    _check(load().fastrs_slab_partition(int(Z), int(nranks), b))
    return [(int(b[i]), int(b[i + 1])) for i in range(nranks)]


def slab_halo_plan(slabs, w: int, Z: int) -> list:
    """(src, dst, side, a, b) transfers of the library's halo plan (side 'lo' / 'hi')."""
    P = len(slabs)
    bd = (ctypes.c_int64 * (P + 1))(*([s[0] for s in slabs] + [slabs[-1][1]]))
    n = ctypes.c_int64(0)
    _check(load().fastrs_slab_halo_plan(bd, P, int(w), int(Z), None, 0, ctypes.byref(n)))
    ent = (ctypes.c_int64 * (5 * n.value))()
    _check(load().fastrs_slab_halo_plan(bd, P, int(w), int(Z), ent, n.value, ctypes.byref(n)))
    return [(int(ent[5 * i]), int(ent[5 * i + 1]), "lo" if ent[5 * i + 2] == 0 else "hi", int(ent[5 * i + 3]),
             int(ent[5 * i + 4])) for i in range(n.value)]


def sphericity_roundness_slab(labels_slab: torch.Tensor, z0: int, Z: int, max_label: int, comm: Comm,
                              flags=BORDER_BACKGROUND, halo_cap: int = 64, stats=False, out=None, ws=None) -> dict:
    """Collective over `comm`: per-object sphericity / roundness of the volume whose z-slab
    [z0, z0 + nz) this rank holds (fastrs_sphericity_roundness_slab: NCCL inside the library).
    flags | SLAB_TRANSPOSE selects the all-to-all transpose z pass.  A halo wider than
    halo_cap is retried once with the width the library reported.  Returns the results of all
    labels and "slab_info"."""
    labels_slab = _labels_arg(labels_slab)
    dev = labels_slab.device
    M = int(max_label)
    res = out if out is not None else {"sphericity": torch.empty(M, dtype=torch.float64, device=dev),
                                       "roundness": torch.empty(M, dtype=torch.float64, device=dev)}
    st = None
    if stats:
        for k, dt in (("volume", torch.int64), ("n_shell", torch.int64), ("max_lt2", torch.int32),
                      ("mean_lt", torch.float64), ("max_lt", torch.float64), ("shell_mean_lt", torch.float64),
                      ("axis_a", torch.float64), ("axis_cb", torch.float64)):
            res[k] = torch.empty(M, dtype=dt, device=dev)
        st = _Stats(*[res[n].data_ptr() for n, _ in _Stats._fields_])
    dims = _dims3(labels_slab.shape)
    info = _SlabInfo()
    for attempt in range(2):
        nb = ctypes.c_size_t(0)
        _check(load().fastrs_slab_call_workspace_bytes(dims, int(z0), int(Z), comm.nranks, comm.rank, M,
                                                       int(halo_cap), int(flags), ctypes.byref(nb)))
        w = workspace(nb.value, dev) if ws is None else ws
        rc = load().fastrs_sphericity_roundness_slab(labels_slab.data_ptr(), dims, int(z0), int(Z), M, int(flags),
                                                     int(halo_cap), res["sphericity"].data_ptr(),
                                                     res["roundness"].data_ptr(),
                                                     None if st is None else ctypes.byref(st), ctypes.byref(info),
                                                     comm.handle, w.data_ptr(), w.numel(), _stream(dev))
        if rc == 3 and attempt == 0 and "exceeds halo_cap" in load().fastrs_last_error().decode():
            msg = load().fastrs_last_error().decode()
            halo_cap = int(msg.split("= ")[1].split()[0]) + 8  # the width the library reported
            continue
        _check(rc)
        break
    res["slab_info"] = {k: int(getattr(info, k)) for k, _ in _SlabInfo._fields_}
    res["slab_info"]["halo_cap"] = int(halo_cap)
    return res


# ------------------------------------------------------------------------------------------
# analysis protocol (include/fastrs.h "analysis protocol around the hot path")
# ------------------------------------------------------------------------------------------

def label_components(mask: torch.Tensor, connectivity=None, ndim=None):
    """Connected components of a binary mask (fastrs_label_components): (int32 labels, int64
    per-item counts).  connectivity 4 / 8 (2D, default 8), 6 / 18 / 26 (3D, default 26)."""
    m = (mask != 0).to(torch.uint8).contiguous() if mask.dtype != torch.uint8 else mask.contiguous()
    ndim, b, dims = _geometry(m.shape, ndim, None)
    conn = connectivity or (8 if ndim == 2 else 26)
    nb = ctypes.c_size_t(0)
    _check(load().fastrs_ccl_workspace_bytes(dims, ndim, b, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=m.device)
    out = torch.empty(m.shape, dtype=torch.int32, device=m.device)
    counts = torch.zeros(b, dtype=torch.int64, device=m.device)
    _check(load().fastrs_label_components(m.data_ptr(), dims, ndim, b, int(conn), out.data_ptr(), counts.data_ptr(),
                                          ws.data_ptr(), ws.numel(), _stream(m.device)))
    return out, counts


def sphericity_wl(labels: torch.Tensor, max_label: int) -> dict:
    """Eq. 3 width/length sphericity of a 2D label image or a batch [B][Y][X] (fastrs_sphericity_wl):
    dict swl, d1, d2 (float64, batch*max_label)."""
    labels = _labels_arg(labels)
    ndim, b, dims = _geometry(labels.shape, 2, None)
    M = b * int(max_label)
    out = {k: torch.empty(M, dtype=torch.float64, device=labels.device) for k in ("swl", "d1", "d2")}
    nb = ctypes.c_size_t(0)
    _check(load().fastrs_wl_workspace_bytes(b, int(max_label), ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=labels.device)
    _check(load().fastrs_sphericity_wl(labels.data_ptr(), dims, 2, b, int(max_label), out["swl"].data_ptr(),
                                       out["d1"].data_ptr(), out["d2"].data_ptr(), ws.data_ptr(), ws.numel(),
                                       _stream(labels.device)))
    return out


def mc_measure(labels: torch.Tensor, max_label: int, ndim=None) -> dict:
    """S_MC baseline (fastrs_mc_measure): dict measure (perimeter 2D / surface area 3D) and
    sphericity_mc, float64, batch*max_label."""
    labels = _labels_arg(labels)
    ndim, b, dims = _geometry(labels.shape, ndim, None)
    M = b * int(max_label)
    out = {k: torch.empty(M, dtype=torch.float64, device=labels.device) for k in ("measure", "sphericity_mc")}
    nb = ctypes.c_size_t(0)
    _check(load().fastrs_mc_workspace_bytes(b, int(max_label), ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=labels.device)
    _check(load().fastrs_mc_measure(labels.data_ptr(), dims, ndim, b, int(max_label), out["measure"].data_ptr(),
                                    out["sphericity_mc"].data_ptr(), ws.data_ptr(), ws.numel(),
                                    _stream(labels.device)))
    return out
