"""Pins of the analysis-protocol oracle (oracle/oracle_analysis.cpp; SURVEY.md §8(f) NEXT-2 and
NEXT-4): connected components against scipy.ndimage.label and SPEC.md's examples; Eq. 3
width/length sphericity against the exact covariance of rasterised rectangles and SPEC.md's
ellipse; the S_MC perimeter / surface area against closed forms derived by hand from the
construction (single pixel / voxel, rectangles, boxes) and against the analytic circle /
sphere."""
from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.ndimage as ndi

import oracle


# ---- connected components --------------------------------

@pytest.mark.parametrize("ndim,conn,rank", [(2, 4, 1), (2, 8, 2), (3, 6, 1), (3, 18, 2), (3, 26, 3)])
def test_ccl_matches_scipy(ndim, conn, rank):
    rng = np.random.default_rng(conn)
    st = ndi.generate_binary_structure(ndim, rank)
    for _ in range(20):
        shape = tuple(int(v) for v in rng.integers(3, 24 if ndim == 2 else 10, ndim))
        m = rng.random(shape) < rng.uniform(0.2, 0.7)
        want, n = ndi.label(m, structure=st)  # raster-order first-encounter numbering
        got, counts = oracle.label_components(m, conn)
        np.testing.assert_array_equal(got, want)
        assert counts[0] == n


def test_ccl_spec_examples_and_batch():
    diag = np.array([[1, 0], [0, 1]])
    assert oracle.label_components(diag, 4)[1][0] == 2
    assert oracle.label_components(diag, 8)[1][0] == 1
    assert oracle.label_components(np.zeros((4, 5)), 8)[1][0] == 0
    rng = np.random.default_rng(3)
    b = rng.random((3, 9, 11)) < 0.5
    got, counts = oracle.label_components(b, 8, ndim=2)
    for i in range(3):
        one, c = oracle.label_components(b[i], 8)
        np.testing.assert_array_equal(got[i], one)
        assert counts[i] == c[0]
    with pytest.raises(oracle.OracleError):
        oracle.label_components(diag, 6)


# ---- Eq. 3 width / length sphericity -------------------

def test_wl_rectangles_exact():
    """An axis-aligned w x h rectangle of pixels: var_x = (w^2 - 1)/12, var_y = (h^2 - 1)/12
    (discrete uniform), so d = 4 sqrt(var) exactly."""
    for w, h in ((10, 4), (7, 7), (31, 2), (1, 9)):
        lab = np.zeros((h + 4, w + 6), np.int32)
        lab[2:2 + h, 3:3 + w] = 1
        r = oracle.sphericity_wl(lab, 1)
        vx, vy = (w * w - 1) / 12, (h * h - 1) / 12
        d1, d2 = 4 * math.sqrt(max(vx, vy)), 4 * math.sqrt(min(vx, vy))
        assert r["d1"][0] == pytest.approx(d1, rel=1e-12) and r["d2"][0] == pytest.approx(d2, rel=1e-12, abs=1e-12)
        assert r["swl"][0] == pytest.approx(d2 / d1, rel=1e-12, abs=1e-12)


def test_wl_spec_examples():
    yy, xx = np.mgrid[-40:41, -40:41]
    t = math.radians(30)
    u, v = xx * math.cos(t) + yy * math.sin(t), -xx * math.sin(t) + yy * math.cos(t)
    ell = ((u / 30.0) ** 2 + (v / 15.0) ** 2 <= 1).astype(np.int32)  # 60 x 30, rotated
    assert abs(oracle.sphericity_wl(ell, 1)["swl"][0] - 0.5) < 0.03
    disk = ((xx ** 2 + yy ** 2) <= 400).astype(np.int32)
    assert abs(oracle.sphericity_wl(disk, 1)["swl"][0] - 1.0) < 0.01
    px = np.zeros((3, 3), np.int32)
    px[1, 1] = 2
    r = oracle.sphericity_wl(px, 2)
    assert r["swl"][1] == 1.0 and np.isnan(r["swl"][0])


# ---- S_MC: marching squares perimeter, marching cubes area -------------

def test_marching_squares_closed_forms():
    px = np.zeros((3, 3), np.int32)
    px[1, 1] = 1
    assert oracle.mc_measure(px)["measure"][0] == pytest.approx(2 * math.sqrt(2), rel=1e-14)  # diamond
    for w, h in ((10, 10), (3, 7), (1, 5)):
        lab = np.zeros((h + 2, w + 2), np.int32)
        lab[1:1 + h, 1:1 + w] = 1
        # straight cells along the sides (w - 1 + h - 1 per pair) and 4 corners cut by sqrt(2)/2
        want = 2 * (w - 1) + 2 * (h - 1) + 4 * math.sqrt(0.5)
        assert oracle.mc_measure(lab)["measure"][0] == pytest.approx(want, rel=1e-14)
    # objects on the grid border are closed by the background outside
    full = np.ones((5, 4), np.int32)
    assert oracle.mc_measure(full)["measure"][0] == pytest.approx(2 * 4 + 2 * 3 + 4 * math.sqrt(0.5), rel=1e-14)


def test_marching_cubes_closed_forms():
    vox = np.zeros((3, 3, 3), np.int32)
    vox[1, 1, 1] = 1
    # 8 corner cubes, each an equilateral triangle of side sqrt(1/2): an octahedron of area sqrt(3)
    assert oracle.mc_measure(vox)["measure"][0] == pytest.approx(math.sqrt(3), rel=1e-14)
    for a, b, c in ((2, 2, 2), (26, 22, 16), (1, 3, 5)):
        lab = np.zeros((a + 2, b + 2, c + 2), np.int32)
        lab[1:1 + a, 1:1 + b, 1:1 + c] = 1
        # face cubes: unit squares; edge cubes: sqrt(1/2) x 1 rectangles; 8 corner triangles
        want = (2 * ((a - 1) * (b - 1) + (b - 1) * (c - 1) + (a - 1) * (c - 1))
                + 4 * ((a - 1) + (b - 1) + (c - 1)) * math.sqrt(0.5) + math.sqrt(3))
        assert oracle.mc_measure(lab)["measure"][0] == pytest.approx(want, rel=1e-13), (a, b, c)


def test_mc_against_analytic_shapes():
    yy, xx = np.mgrid[-60:61, -60:61]
    disk = ((xx ** 2 + yy ** 2) <= 2500).astype(np.int32)
    p = oracle.mc_measure(disk)["measure"][0]
    assert 2 * math.pi * 50 < p < 2 * math.pi * 50 * 1.07  # the digital boundary's corners
    z, y, x = np.mgrid[-22:23, -22:23, -22:23]
    sph = ((x ** 2 + y ** 2 + z ** 2) <= 400).astype(np.int32)
    r = oracle.mc_measure(sph)
    assert 4 * math.pi * 400 < r["measure"][0] < 4 * math.pi * 400 * 1.10
    assert 0.90 < r["sphericity_mc"][0] < 1.0
    # translation invariance; two labels measured independently
    two = np.zeros((60, 60, 60), np.int32)
    two[5:50, 5:50, 5:50][sph[:, :, :] > 0] = 1
    two[48:52, 50:55, 40:58] = 2
    rr = oracle.mc_measure(two)
    assert rr["measure"][0] == pytest.approx(r["measure"][0], rel=1e-14)
