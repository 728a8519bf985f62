"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/fastrs.h
declares (no GPU needed: only host-side entry points are called)."""
from __future__ import annotations

import ctypes
import math
import os
import re
import subprocess

import pytest

from paper_2504_05808_b200 import _build
from paper_2504_05808_b200 import fastrs as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fastrs.h")).read()
    return sorted(set(re.findall(r"FASTRS_API[^;(]*?\b(fastrs_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("fastrs_workspace_bytes", "fastrs_edt_sq", "fastrs_local_thickness", "fastrs_sphericity_roundness",
              "fastrs_sphericity_roundness_host", "fastrs_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = F.load()
    for n in _declared():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", _build.SO], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fastrs_\w+)", out))
    assert set(_declared()) == exported


def test_built_for_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.SO], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_workspace_bytes_host_only():
    nb = F.workspace_bytes((128, 128, 128), 3, 51, 0)
    # two N*4 EDT buffers + per-tile centre slots (8 B/element) at least
    assert nb >= 128 ** 3 * 16
    nb_io = F.workspace_bytes((128, 128, 128), 3, 51, F.HOST_IO)
    assert nb_io >= nb + 128 ** 3 * 4
    with pytest.raises(F.FastrsError) as e:
        F.workspace_bytes((4, 4, 4, 4), 4, 1, 0)
    assert e.value.name == "EINVAL"
    with pytest.raises(F.FastrsError):
        F.workspace_bytes((0, 4), 2, 1, 0)
    with pytest.raises(F.FastrsError):
        F.workspace_bytes((20000, 4), 2, 1, 0)


def test_null_labels_rejected_before_any_device_work():
    lib = F.load()
    dims = (ctypes.c_int64 * 2)(4, 4)
    rc = lib.fastrs_edt_sq(None, dims, 2, 1, 1, None, None, 0, None)
    assert rc == 1
    assert b"NULL" in lib.fastrs_last_error()


def test_host_math_matches_oracle_closed_forms():
    import oracle
    for a, c in [(1, 1), (2, 1), (1, 2), (3.5, 0.2), (0.2, 3.5), (20.02, 19.98), (5, 5 + 1e-9)]:
        assert F.spheroid_area(a, c) == pytest.approx(oracle.spheroid_area(a, c), rel=1e-13)
    for a, b in [(1, 1), (2, 1), (3, 1), (10, 0.5)]:
        assert F.ramanujan_perimeter(a, b) == pytest.approx(oracle.ramanujan_perimeter(a, b), rel=1e-14)
    for V, a in [(14147, 15.03329637837291), (1.0, 1.0), (8309, 8.4), (1e6, 40.0)]:
        assert F.sphericity_3d(V, a) == pytest.approx(oracle.sphericity_3d(V, a), rel=1e-13)
    for A, a in [(1257, math.sqrt(401)), (1.0, 1.0), (5000, 20.0)]:
        assert F.sphericity_2d(A, a) == pytest.approx(oracle.sphericity_2d(A, a), rel=1e-13)
