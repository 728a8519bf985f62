"""Seeded synthetic label grids (test and bench scaffolding, shared by both sides).

Holds none of the method's arithmetic: it only draws shape parameters with
``numpy.random.default_rng(seed)`` and rasterises them through ``libsynth.so``
(``synth/synth.cpp``).  The five workloads are BASELINE.json ``configs[0..4]``
(C1..C5), re-parametrised where the stated size distributions contradict the stated
packing; the full recipe is in DESIGN.md ("Input recipe").

Also provides the closed-form check shapes (digital disk / sphere / blocks / bars)
and random tiny label grids used by the property tests.
"""
from __future__ import annotations

import ctypes
import hashlib
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_SRC = os.path.join(_HERE, "synth.cpp")
_lock = threading.Lock()
_lib = None

NPARAM = 13


def build(force: bool = False) -> str:
    """Compile libsynth.so in-tree (g++)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O3", "-march=x86-64-v2", "-std=c++17", "-shared", "-fPIC", "-pthread",
               _SRC, "-o", _SO + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_SO)
            lib.synth_place.restype = ctypes.c_int
            lib.synth_place.argtypes = [
                ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int,
                ctypes.c_void_p, ctypes.c_void_p]
            lib.synth_cells.restype = None
            lib.synth_cells.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
            _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --------------------------------------------------------------------------------------
# closed-form check shapes (centre-inclusion rasterisation)
# --------------------------------------------------------------------------------------

def disk(r: int, canvas: int | None = None, label: int = 1) -> np.ndarray:
    """Digital disk {x^2+y^2 <= r^2} centred on a pixel of a canvas with margin."""
    n = canvas or 2 * r + 5
    c = n // 2
    y, x = np.mgrid[0:n, 0:n]
    out = np.zeros((n, n), np.int32)
    out[(y - c) ** 2 + (x - c) ** 2 <= r * r] = label
    return out


def sphere(r: int, canvas: int | None = None, label: int = 1) -> np.ndarray:
    n = canvas or 2 * r + 5
    c = n // 2
    z, y, x = np.mgrid[0:n, 0:n, 0:n]
    out = np.zeros((n, n, n), np.int32)
    out[(z - c) ** 2 + (y - c) ** 2 + (x - c) ** 2 <= r * r] = label
    return out


def ellipse(a: float, b: float, canvas=None, label: int = 1) -> np.ndarray:
    """Axis-aligned ellipse, semi-axis a along x and b along y."""
    ny = canvas[0] if canvas else int(2 * math.ceil(b) + 5)
    nx = canvas[1] if canvas else int(2 * math.ceil(a) + 5)
    cy, cx = ny // 2, nx // 2
    y, x = np.mgrid[0:ny, 0:nx]
    out = np.zeros((ny, nx), np.int32)
    out[((x - cx) / a) ** 2 + ((y - cy) / b) ** 2 <= 1.0] = label
    return out


def spheroid(a: float, c: float, label: int = 1) -> np.ndarray:
    """Axis-aligned spheroid: semi-axes a (x, y) and c (z)."""
    nz = int(2 * math.ceil(c) + 5)
    nx = int(2 * math.ceil(a) + 5)
    z, y, x = np.mgrid[0:nz, 0:nx, 0:nx]
    out = np.zeros((nz, nx, nx), np.int32)
    out[((x - nx // 2) / a) ** 2 + ((y - nx // 2) / a) ** 2 + ((z - nz // 2) / c) ** 2 <= 1.0] = label
    return out


def random_labels(shape, nlabels: int, seed: int, fill: float = 0.6, blob: int = 1) -> np.ndarray:
    """Tiny random label grid with touching labels (property tests).

    Each element is background with probability 1-fill, else one of 1..nlabels; with
    blob>1 the labels are drawn on a coarse grid and upsampled so runs are longer.
    """
    rng = np.random.default_rng(seed)
    coarse = tuple(max(1, -(-s // blob)) for s in shape)
    lab = rng.integers(1, nlabels + 1, size=coarse).astype(np.int32)
    fgm = rng.random(coarse) < fill
    lab[~fgm] = 0
    for ax in range(len(shape)):
        lab = np.repeat(lab, blob, axis=ax)
    lab = lab[tuple(slice(0, s) for s in shape)]
    return np.ascontiguousarray(lab)


# --------------------------------------------------------------------------------------
# BASELINE.json configs C1..C5
# --------------------------------------------------------------------------------------

def _quat(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _place(shape3, is2d, params, labels, seed, max_tries=10000):
    lib = _load()
    Z, Y, X = shape3
    grid = np.zeros((Z, Y, X), np.int32)
    n = params.shape[0]
    placed = np.zeros(n, np.int32)
    scale = np.zeros(n, np.float64)
    params = np.ascontiguousarray(params, np.float64)
    labels = np.ascontiguousarray(labels, np.int32)
    lib.synth_place(_ptr(grid), Z, Y, X, int(is2d), n, _ptr(params), _ptr(labels),
                    int(seed) & (2**64 - 1), max_tries, _ptr(placed), _ptr(scale))
    return grid, placed, scale


def _objects3d(rng, r_eq, aspect, rough_frac):
    n = len(r_eq)
    p = np.zeros((n, NPARAM))
    a = r_eq * aspect ** (-1.0 / 3.0)
    c = aspect * a
    p[:, 0] = a
    p[:, 1] = a
    p[:, 2] = c
    p[:, 3:7] = _quat(rng, n)
    rough = rng.random(n) < rough_frac
    p[:, 7] = np.where(rough, rng.uniform(0.10, 0.30, n), 0.0)
    p[:, 8] = rng.integers(0, 2**31, n)
    return p


def make_config(i: int, seed: int | None = None, batch: int | None = None, images: tuple | None = None):
    """Return (labels, info) for BASELINE.json config C{i} (i in 1..5).

    labels: int32, C order; 2D (Y,X) for C1, 3D (Z,Y,X) for C2..C4, (B,Y,X) for C5.
    info: dict(config, seed, ndim, batch, max_label, n_objects, fill, sha256).
    ``batch`` overrides the number of C5 images (default 256); ``images=(i0, i1)`` rasterises
    only images [i0, i1) of that seeded batch (identical to the same slice of the whole batch:
    the per-rank shard of the multi-GPU bench).
    """
    seed = i if seed is None else seed
    rng = np.random.default_rng(seed)
    if i == 1:
        # 20 ellipses, semi-axes ~U[5,30], uniform angle; disc r=20 at (128,128) = label 21
        n = 20
        p = np.zeros((n + 1, NPARAM))
        p[0, 0:2] = 20.0
        p[0, 8] = 1
        p[0, 9:12] = (0, 128, 128)
        p[0, 12] = 1
        p[1:, 0] = rng.uniform(5, 30, n)
        p[1:, 1] = rng.uniform(5, 30, n)
        p[1:, 3] = rng.uniform(0, math.pi, n)
        p[1:, 8] = rng.integers(0, 2**31, n)
        order = 1 + np.argsort(-(p[1:, 0] * p[1:, 1]), kind="stable")
        params = np.concatenate([p[:1], p[order]])
        labels = np.concatenate([[n + 1], np.arange(1, n + 1)]).astype(np.int32)
        grid, placed, _ = _place((1, 256, 256), True, params, labels, seed)
        lab = grid[0]
        ndim, B, max_label = 2, 1, n + 1
    elif i == 2:
        # 50 spheroids, a~U[4,20], aspect~U[0.3,3]; sphere r=15 at (64,64,64) = label 51
        n = 50
        a = rng.uniform(4, 20, n)
        asp = rng.uniform(0.3, 3.0, n)
        p = np.zeros((n, NPARAM))
        p[:, 0] = a
        p[:, 1] = a
        p[:, 2] = asp * a
        p[:, 3:7] = _quat(rng, n)
        p[:, 8] = rng.integers(0, 2**31, n)
        chk = np.zeros((1, NPARAM))
        chk[0, 0:3] = 15.0
        chk[0, 3] = 1.0
        chk[0, 9:12] = 64
        chk[0, 12] = 1
        order = np.argsort(-(p[:, 0] * p[:, 1] * p[:, 2]), kind="stable")
        params = np.concatenate([chk, p[order]])
        labels = np.concatenate([[n + 1], np.arange(1, n + 1)]).astype(np.int32)
        grid, placed, _ = _place((128, 128, 128), False, params, labels, seed)
        lab = grid
        ndim, B, max_label = 3, 1, n + 1
    elif i in (3, 4):
        if i == 3:
            # 2000 particles, r_eq log-uniform [4,30], aspect U[0.3,3], half rough
            n, dim = 2000, 512
            r_eq = np.exp(rng.uniform(math.log(4), math.log(30), n))
        else:
            # ~20000 particles, r_eq truncated power law p(r) ~ r^-1.7 on [3,40]
            n, dim = 20000, 1024
            k = 1.7
            u = rng.random(n)
            lo, hi = 3.0 ** (1 - k), 40.0 ** (1 - k)
            r_eq = (lo + u * (hi - lo)) ** (1.0 / (1 - k))
        asp = rng.uniform(0.3, 3.0, n)
        p = _objects3d(rng, r_eq, asp, 0.5)
        order = np.argsort(-r_eq, kind="stable")
        params = p[order]
        labels = np.arange(1, n + 1, dtype=np.int32)
        grid, placed, _ = _place((dim, dim, dim), False, params, labels, seed, max_tries=2000)
        lab = grid
        ndim, B, max_label = 3, 1, n
    elif i == 5:
        # B images 2048^2, ~500 touching cells each, semi-axes U[8,60], noise U[0,0.2]
        B = 256 if batch is None else batch
        ncell, dim = 500, 2048
        p = np.zeros((B * ncell, NPARAM))
        p[:, 0] = rng.uniform(8, 60, B * ncell)
        p[:, 1] = rng.uniform(8, 60, B * ncell)
        p[:, 3] = rng.uniform(0, math.pi, B * ncell)
        p[:, 7] = rng.uniform(0.0, 0.20, B * ncell)
        p[:, 8] = rng.integers(0, 2**31, B * ncell)
        p[:, 10] = rng.uniform(0, dim, B * ncell)
        p[:, 11] = rng.uniform(0, dim, B * ncell)
        p[:, 12] = 1
        if images is not None:  # a shard [i0, i1) of the seeded B-image batch (same draws)
            i0, i1 = images
            p = p[i0 * ncell:i1 * ncell]
            B = i1 - i0
        lab = np.empty((B, dim, dim), np.int32)
        _load().synth_cells(_ptr(lab), B, dim, dim, ncell, _ptr(np.ascontiguousarray(p)))
        ndim, max_label = 2, ncell
    else:
        raise ValueError(f"unknown config C{i}")
    info = describe(lab, ndim=ndim, batch=B, max_label=max_label)
    info.update(config=f"C{i}", seed=seed)
    return lab, info


def make_count_volume(seed: int = 6, n: int = 15503, dim: int = 400):
    """Synthetic stand-in for the paper's object-count experiment volume (a 400^3
    uCT scan with 15 503 objects of 27 to ~130 000 voxels): n
    spheroids / rough grains, r_eq on a truncated power law p(r) ~ r^-3 between the radii of 27
    and 130 000 voxel spheres (expected fill ~21 %), aspect U[0.3, 3], half rough; largest
    placed first, >= 1 voxel gaps.  Objects that do not fit are left out (info["n_objects"])."""
    rng = np.random.default_rng(seed)
    k = 3.0
    r_lo, r_hi = (3 * 27 / (4 * math.pi)) ** (1 / 3), (3 * 130000 / (4 * math.pi)) ** (1 / 3)
    u = rng.random(n)
    lo, hi = r_lo ** (1 - k), r_hi ** (1 - k)
    r_eq = (lo + u * (hi - lo)) ** (1.0 / (1 - k))
    asp = rng.uniform(0.3, 3.0, n)
    p = _objects3d(rng, r_eq, asp, 0.5)
    order = np.argsort(-r_eq, kind="stable")
    labels = np.arange(1, n + 1, dtype=np.int32)
    grid, placed, _ = _place((dim, dim, dim), False, p[order], labels, seed, max_tries=2000)
    info = describe(grid, ndim=3, batch=1, max_label=n)
    info.update(config="count-volume", seed=seed)
    return grid, info


def describe(lab: np.ndarray, ndim: int, batch: int, max_label: int) -> dict:
    counts = np.bincount(lab.reshape(-1), minlength=max_label + 1)
    fg = int(lab.size - counts[0])
    flat = lab.reshape(-1)
    # full hash for small grids; a strided-sample hash (every 4099th element) for large ones
    h = hashlib.sha256((flat if flat.size <= 2**26 else flat[::4099]).tobytes()).hexdigest()
    return dict(ndim=ndim, batch=batch, max_label=int(max_label), n_elements=int(lab.size),
                fill=fg / lab.size, n_labels_present=int((counts[1:] > 0).sum()),
                sha256=h, sha256_kind="full" if flat.size <= 2**26 else "strided-4099")
