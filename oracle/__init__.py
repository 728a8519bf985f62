"""CPU oracle of the paper's definitions — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2504_05808_b200``) never imports it and shares no code with it.

Thin ctypes wrapper over ``oracle/liboracle.so`` (built from ``oracle/oracle.cpp`` with
g++; see that file's header for what is computed and which paper passage each step
follows).  Inputs are numpy arrays; all outputs are fresh numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")
_SRCS = [_SRC, os.path.join(_HERE, "oracle_analysis.cpp")]
_lock = threading.Lock()
_lib = None

BORDER_BACKGROUND = 1

STATUS = {0: "OK", 1: "EINVAL", 2: "ENOSITE", 6: "EINTERNAL"}


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle returned {STATUS.get(code, code)}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so in-tree (plain g++ -O2; building the checker is not using it)."""
    if force or not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(s) for s in _SRCS):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread",
                               *_SRCS, "-o", _SO + ".tmp"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_SO)
            vp, i64, i32, u32, ci, cd = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                          ctypes.c_uint32, ctypes.c_int, ctypes.c_double)
            lib.fastrs_oracle_edt_sq.argtypes = [vp, vp, ci, i64, u32, vp, ci]
            lib.fastrs_oracle_edt_sq.restype = ci
            lib.fastrs_oracle_fields.argtypes = [vp, vp, ci, i64, i32, u32, vp, vp, vp, ci]
            lib.fastrs_oracle_fields.restype = ci
            lib.fastrs_oracle_sphericity_roundness.argtypes = [vp, vp, ci, i64, i32, u32] + [vp] * 10 + [ci]
            lib.fastrs_oracle_sphericity_roundness.restype = ci
            lib.fastrs_oracle_label_components.argtypes = [vp, vp, ci, i64, ci, vp, vp]
            lib.fastrs_oracle_label_components.restype = ci
            lib.fastrs_oracle_sphericity_wl.argtypes = [vp, vp, ci, i64, i32, vp, vp, vp]
            lib.fastrs_oracle_sphericity_wl.restype = ci
            lib.fastrs_oracle_mc_measure.argtypes = [vp, vp, ci, i64, i32, vp, vp]
            lib.fastrs_oracle_mc_measure.restype = ci
            for name in ("spheroid_area", "ramanujan_perimeter", "sphericity_3d", "sphericity_2d"):
                f = getattr(lib, "fastrs_oracle_" + name)
                f.argtypes = [cd, cd]
                f.restype = cd
            _lib = lib
    return _lib


def _geom(labels: np.ndarray, ndim: int | None, batch: int | None):
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    if ndim is None:
        ndim = labels.ndim
    if batch is None:
        batch = 1 if labels.ndim == ndim else labels.shape[0]
    dims = np.ascontiguousarray(labels.shape[-ndim:], dtype=np.int64)
    return labels, ndim, int(batch), dims


def _p(a):
    return None if a is None else a.ctypes.data


def edt_sq(labels, flags=BORDER_BACKGROUND, ndim=None, batch=None, nthreads=0) -> np.ndarray:
    """Exact squared label-aware EDT, uint32, 0 on background."""
    labels, ndim, batch, dims = _geom(labels, ndim, batch)
    out = np.zeros(labels.shape, np.uint32)
    st = _load().fastrs_oracle_edt_sq(_p(labels), _p(dims), ndim, batch, flags, _p(out), nthreads)
    if st:
        raise OracleError(st)
    return out


def fields(labels, max_label=None, flags=BORDER_BACKGROUND, ndim=None, batch=None, nthreads=0):
    """Return (D, LT^2, shell) full-grid fields (uint32, uint32, uint8)."""
    labels, ndim, batch, dims = _geom(labels, ndim, batch)
    if max_label is None:
        max_label = max(1, int(labels.max(initial=0)))
    d2 = np.zeros(labels.shape, np.uint32)
    lt2 = np.zeros(labels.shape, np.uint32)
    sh = np.zeros(labels.shape, np.uint8)
    st = _load().fastrs_oracle_fields(_p(labels), _p(dims), ndim, batch, max_label, flags,
                                      _p(d2), _p(lt2), _p(sh), nthreads)
    if st:
        raise OracleError(st)
    return d2, lt2, sh


def sphericity_roundness(labels, max_label=None, flags=BORDER_BACKGROUND, ndim=None, batch=None,
                         label_mask=None, nthreads=0) -> dict:
    """Per-object metrics; arrays of batch*max_label entries, index b*max_label + label-1."""
    labels, ndim, batch, dims = _geom(labels, ndim, batch)
    if max_label is None:
        max_label = max(1, int(labels.max(initial=0)))
    M = batch * max_label
    out = dict(sphericity=np.empty(M), roundness=np.empty(M), volume=np.empty(M, np.int64),
               n_shell=np.empty(M, np.int64), max_lt2=np.empty(M, np.uint32), mean_lt=np.empty(M),
               shell_mean_lt=np.empty(M), axis_a=np.empty(M), axis_cb=np.empty(M))
    mask = None
    if label_mask is not None:
        mask = np.ascontiguousarray(label_mask, dtype=np.uint8).reshape(-1)
        assert mask.size == M
    st = _load().fastrs_oracle_sphericity_roundness(
        _p(labels), _p(dims), ndim, batch, int(max_label), flags,
        *[_p(out[k]) for k in ("sphericity", "roundness", "volume", "n_shell", "max_lt2", "mean_lt",
                               "shell_mean_lt", "axis_a", "axis_cb")],
        _p(mask), nthreads)
    if st:
        raise OracleError(st)
    return out


def spheroid_area(a: float, c: float) -> float:
    return _load().fastrs_oracle_spheroid_area(a, c)


def ramanujan_perimeter(a: float, b: float) -> float:
    return _load().fastrs_oracle_ramanujan_perimeter(a, b)


def sphericity_3d(V: float, mean_lt: float) -> float:
    return _load().fastrs_oracle_sphericity_3d(V, mean_lt)


def sphericity_2d(A: float, mean_lt: float) -> float:
    return _load().fastrs_oracle_sphericity_2d(A, mean_lt)


def touches_edge(labels, max_label, ndim=None, batch=None) -> np.ndarray:
    """Edge objects, the plain definition (SPEC.md:212 remove_edge_objects: "any label whose
    support touches a grid boundary"; "Edge cells are removed"): uint8 flags,
    batch*max_label entries, 1 where the label occurs on the first or last index of any axis of
    its item.  Labels outside 1..max_label are ignored."""
    labels, ndim, batch, dims = _geom(labels, ndim, batch)
    items = labels.reshape((batch,) + tuple(int(d) for d in dims))
    out = np.zeros(batch * int(max_label), np.uint8)
    for b in range(batch):
        it = items[b]
        for ax in range(ndim):
            for idx in (0, it.shape[ax] - 1):
                face = np.take(it, idx, axis=ax)
                for L in np.unique(face):
                    if 1 <= L <= max_label:
                        out[b * max_label + L - 1] = 1
    return out


def filter_objects(res: dict, min_volume=None, edge=None) -> dict:
    """The paper's analysis filters on an oracle result dict (copies): NaN sphericity/roundness
    where volume < min_volume (PAPER.md:274, SPEC.md:219 filter_small) or edge[i] != 0."""
    out = dict(res)
    drop = np.zeros(res["sphericity"].shape, bool)
    if min_volume is not None:
        drop |= res["volume"] < min_volume
    if edge is not None:
        drop |= np.asarray(edge) != 0
    for k in ("sphericity", "roundness"):
        v = np.array(res[k], dtype=np.float64)
        v[drop] = np.nan
        out[k] = v
    return out


def label_components(mask, connectivity=None, ndim=None, batch=None):
    """Connected components of a binary mask (oracle_analysis.cpp): int32 labels 1..K per item in
    row-major first-encounter order, and the per-item counts.  connectivity: 4 / 8 (2D, default
    8), 6 / 18 / 26 (3D, default 26)."""
    m = np.ascontiguousarray(np.asarray(mask) != 0, dtype=np.uint8)
    ndim = m.ndim if ndim is None else ndim
    batch = (1 if m.ndim == ndim else m.shape[0]) if batch is None else batch
    dims = np.ascontiguousarray(m.shape[-ndim:], dtype=np.int64)
    if connectivity is None:
        connectivity = 8 if ndim == 2 else 26
    out = np.zeros(m.shape, np.int32)
    counts = np.zeros(batch, np.int64)
    st = _load().fastrs_oracle_label_components(_p(m), _p(dims), ndim, batch, int(connectivity), _p(out),
                                                _p(counts))
    if st:
        raise OracleError(st)
    return out, counts


def sphericity_wl(labels, max_label=None, batch=None):
    """Eq. 3 width-to-length sphericity (2D): dict of swl, d1, d2 (batch*max_label)."""
    labels, ndim, batch, dims = _geom(labels, 2, batch)
    if max_label is None:
        max_label = max(1, int(labels.max(initial=0)))
    M = batch * max_label
    out = dict(swl=np.empty(M), d1=np.empty(M), d2=np.empty(M))
    st = _load().fastrs_oracle_sphericity_wl(_p(labels), _p(dims), 2, batch, int(max_label), _p(out["swl"]),
                                             _p(out["d1"]), _p(out["d2"]))
    if st:
        raise OracleError(st)
    return out


def mc_measure(labels, max_label=None, ndim=None, batch=None):
    """S_MC baseline: per-label marching-squares perimeter (2D) / marching-tetrahedra surface area
    (3D) and the sphericity from it (Eq. 2 / Eq. 1): dict measure, sphericity_mc."""
    labels, ndim, batch, dims = _geom(labels, ndim, batch)
    if max_label is None:
        max_label = max(1, int(labels.max(initial=0)))
    M = batch * max_label
    out = dict(measure=np.empty(M), sphericity_mc=np.empty(M))
    st = _load().fastrs_oracle_mc_measure(_p(labels), _p(dims), ndim, batch, int(max_label), _p(out["measure"]),
                                          _p(out["sphericity_mc"]))
    if st:
        raise OracleError(st)
    return out
