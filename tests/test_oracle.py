"""Pins for the CPU oracle (runs without a GPU).

The oracle is checked against things other than itself: brute-force definitions on tiny
grids (tests/_refs.py), scipy's EDT on separated labels, SPEC worked examples
(tests/golden/spec_examples.txt), lattice-count closed forms for the digital disk and
sphere, numeric surface-of-revolution integrals, complete elliptic integrals, and
invariants (SURVEY.md §8(c) "What pins each part").
"""
from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.integrate
import scipy.ndimage
import scipy.special

import oracle
import synth
from tests import _refs

BB = oracle.BORDER_BACKGROUND


# ------------------------------------------------------------------------------------------
# EDT
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("border", [True, False])
@pytest.mark.parametrize("seed", range(30))
def test_edt_matches_bruteforce_random_touching(seed, border):
    """Label-aware EDT == brute force over all sites."""
    shape = (10, 11) if seed % 2 == 0 else (6, 7, 5)
    lab = synth.random_labels(shape, nlabels=3, seed=seed, fill=0.75, blob=1 + seed % 3)
    ref = _refs.brute_edt_sq(lab, border)
    if (ref < 0).any():
        with pytest.raises(oracle.OracleError):
            oracle.edt_sq(lab, flags=BB if border else 0)
        return
    got = oracle.edt_sq(lab, flags=BB if border else 0)
    np.testing.assert_array_equal(got.astype(np.int64), ref)


def test_edt_bigger_crop_uses_separable_path():
    """Crops > 4096 elements take the separable O(len^2) path; still equal to brute force."""
    lab = synth.random_labels((20, 20, 14), nlabels=2, seed=7, fill=0.9, blob=5)
    lab[:] = np.where(lab > 0, 1, 0)
    ref = _refs.brute_edt_sq(lab, True)
    np.testing.assert_array_equal(oracle.edt_sq(lab).astype(np.int64), ref)


@pytest.mark.parametrize("seed", range(6))
def test_edt_matches_scipy_on_separated_labels(seed):
    """On a single label, the label-aware EDT is the binary EDT of the padded mask
    (library routine: scipy.ndimage.distance_transform_edt), squared and rounded."""
    rng = np.random.default_rng(seed)
    mask = scipy.ndimage.binary_opening(rng.random((40, 37, 23)) < 0.7, iterations=1)
    lab = mask.astype(np.int32)
    padded = np.pad(mask, 1)
    ref = np.rint(scipy.ndimage.distance_transform_edt(padded) ** 2).astype(np.int64)[1:-1, 1:-1, 1:-1]
    np.testing.assert_array_equal(oracle.edt_sq(lab).astype(np.int64), ref)


def test_edt_invariants_on_c1():
    lab, info = synth.make_config(1)
    D = oracle.edt_sq(lab).astype(np.int64)
    fg = lab > 0
    assert (D[fg] >= 1).all() and (D[~fg] == 0).all()
    # 1-Lipschitz in d = sqrt(D) across face neighbours of the same label
    d = np.sqrt(D)
    for ax in (0, 1):
        same = (np.diff(lab, axis=ax) == 0) & fg[(slice(None),) * ax + (slice(1, None),)]
        assert (np.abs(np.diff(d, axis=ax))[same] <= 1 + 1e-12).all()


def test_enosite_without_border():
    lab = np.ones((4, 5), np.int32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.edt_sq(lab, flags=0)
    assert e.value.code == 2
    # with the border as background the same grid is fine
    assert oracle.edt_sq(lab, flags=BB).max() == 4  # centre row of a 4x5 grid: min(2,3)^2


def test_invalid_label():
    lab = np.zeros((4, 4), np.int32)
    lab[1, 1] = 7
    with pytest.raises(oracle.OracleError) as e:
        oracle.sphericity_roundness(lab, max_label=3)
    assert e.value.code == 1


# ------------------------------------------------------------------------------------------
# LT and shell
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("border", [True, False])
@pytest.mark.parametrize("seed", range(20))
def test_lt_matches_bruteforce_all_balls(seed, border):
    shape = (12, 13) if seed % 2 == 0 else (7, 8, 6)
    lab = synth.random_labels(shape, nlabels=2, seed=100 + seed, fill=0.8, blob=2 + seed % 2)
    D = _refs.brute_edt_sq(lab, border)
    if (D < 0).any():
        pytest.skip("no site")
    d2, lt2, sh = oracle.fields(lab, flags=BB if border else 0)
    np.testing.assert_array_equal(d2.astype(np.int64), D)
    np.testing.assert_array_equal(lt2.astype(np.int64), _refs.brute_lt_sq(lab, D))
    np.testing.assert_array_equal(sh.astype(bool), _refs.brute_shell(lab, border))
    # shell <=> D == 1 (SURVEY.md §8(c) pin table: proved equivalence)
    np.testing.assert_array_equal(sh.astype(bool), d2 == 1)


def test_spec_worked_examples():
    cases = _refs.load_spec_examples()
    for name, c in cases.items():
        if name == "block3x3x3":
            continue
        lab = c["labels"].astype(np.int32)
        d2, lt2, sh = oracle.fields(lab)
        np.testing.assert_array_equal(d2, c["d2"], err_msg=name)
        if "lt2" in c:
            np.testing.assert_array_equal(lt2, c["lt2"], err_msg=name)
        if "shell" in c:
            np.testing.assert_array_equal(sh, c["shell"], err_msg=name)
        if "shell_mean_lt" in c:
            r = oracle.sphericity_roundness(lab)
            assert r["shell_mean_lt"][0] == pytest.approx(c["shell_mean_lt"], rel=0, abs=1e-15)
    c = cases["block3x3x3"]
    lab = np.zeros(c["shape"], np.int32)
    lab[1:4, 1:4, 1:4] = 1
    d2, lt2, sh = oracle.fields(lab)
    assert d2[2, 2, 2] == c["centre_d2"]
    assert (lt2[lab > 0] == c["lt2_all"]).all()
    assert int(sh.sum()) == c["n_shell"]


def test_digital_disk_r20():
    g = _refs.load_closed_forms()["digital_disk_r20"]
    lab = synth.disk(20)
    # independent lattice count (Gauss circle problem, brute count)
    assert sum(1 for x in range(-20, 21) for y in range(-20, 21) if x * x + y * y <= 400) == g["area"]
    d2, lt2, sh = oracle.fields(lab)
    assert int(d2.max()) == g["max_d2"] == 20 * 20 + 1
    assert (lt2[lab > 0] == g["lt2_all"]).all()
    assert int(sh.sum()) == g["n_shell_4conn"]
    r = oracle.sphericity_roundness(lab)
    assert r["volume"][0] == g["area"]
    assert r["mean_lt"][0] == pytest.approx(math.sqrt(401), rel=1e-15)
    assert r["sphericity"][0] == pytest.approx(g["sphericity"], rel=1e-11)
    assert r["roundness"][0] == pytest.approx(1.0, abs=4e-16)


def test_digital_sphere_r15():
    g = _refs.load_closed_forms()["digital_sphere_r15"]
    lab = synth.sphere(15)
    n = sum(1 for x in range(-15, 16) for y in range(-15, 16) for z in range(-15, 16)
            if x * x + y * y + z * z <= 225)
    assert n == g["volume"]
    d2, lt2, sh = oracle.fields(lab)
    assert int(d2.max()) == g["max_d2"] and int((d2 == d2.max()).sum()) == 1
    assert (lt2[lab > 0] == g["lt2_all"]).all()
    assert int(sh.sum()) == g["n_shell_6conn"]
    r = oracle.sphericity_roundness(lab)
    assert r["sphericity"][0] == pytest.approx(g["sphericity"], rel=1e-11)
    assert r["roundness"][0] == pytest.approx(1.0, abs=4e-16)


def test_one_element_objects():
    """1-element objects: D=1, LT=1, R=1 (reading c15); 3D one voxel: c = 3/(4 pi) < a
    exercises the oblate branch."""
    lab = np.zeros((5, 5, 5), np.int32)
    lab[2, 2, 2] = 1
    r = oracle.sphericity_roundness(lab)
    assert r["volume"][0] == 1 and r["max_lt2"][0] == 1 and r["roundness"][0] == 1.0
    assert r["axis_cb"][0] == pytest.approx(3 / (4 * math.pi))
    assert r["sphericity"][0] == pytest.approx(
        math.pi ** (1 / 3) * 6 ** (2 / 3) / _spheroid_area_numeric(1.0, 3 / (4 * math.pi)), rel=1e-9)


# ------------------------------------------------------------------------------------------
# closed forms (Eqs. 1, 2, 6-11)
# ------------------------------------------------------------------------------------------

def _spheroid_area_numeric(a, c):
    """Surface of revolution of x = a sin t, z = c cos t (independent of Eqs. 6-7)."""
    f = lambda t: 2 * math.pi * a * math.sin(t) * math.sqrt((a * math.cos(t)) ** 2 + (c * math.sin(t)) ** 2)
    return scipy.integrate.quad(f, 0, math.pi, epsabs=0, epsrel=1e-13, limit=200)[0]


def _ellipse_perimeter_exact(a, b):
    a, b = max(a, b), min(a, b)
    return 4 * a * scipy.special.ellipe(1 - (b / a) ** 2)


@pytest.mark.parametrize("a,c", [(1, 1), (2, 1), (1, 2), (3, 1.5), (1, 0.3), (1, 3), (5, 5.0000001),
                                 (5, 4.9999999), (1, 1e-3), (1e-3, 1), (20.02, 19.98)])
def test_spheroid_area_vs_numeric_integral(a, c):
    assert oracle.spheroid_area(a, c) == pytest.approx(_spheroid_area_numeric(a, c), rel=1e-10)


def test_spheroid_area_spec_values():
    g = _refs.load_closed_forms()["spheroid_area"]
    for a, c, v in g["cases"]:
        assert oracle.spheroid_area(a, c) == pytest.approx(v, rel=g["rel_tol_spec"])
    assert oracle.spheroid_area(1, 1) == 4 * math.pi
    # continuity at c = a
    for s in (1 + 1e-6, 1 - 1e-6, 1 + 1e-12, 1 - 1e-12):
        assert oracle.spheroid_area(1, s) == pytest.approx(_spheroid_area_numeric(1, s), rel=1e-12)


@pytest.mark.parametrize("a,b", [(1, 1), (2, 1), (3, 1), (4, 1), (1, 2), (10, 9.5), (7, 1.5)])
def test_ramanujan_vs_elliptic_integral(a, b):
    exact = _ellipse_perimeter_exact(a, b)
    got = oracle.ramanujan_perimeter(a, b)
    assert got <= exact * (1 + 1e-15)  # Ramanujan I never overestimates
    h = ((a - b) / (a + b)) ** 2
    # Ramanujan I agrees with the exact series pi(a+b)(1 + h/4 + h^2/64 + h^3/256 + ...)
    # through h^2; its error starts at pi(a+b) h^3/512.  Bound with twice that term.
    assert exact - got <= math.pi * (a + b) * h ** 3 / 256 + 1e-12


def test_ramanujan_spec_values():
    g = _refs.load_closed_forms()["ramanujan_perimeter"]
    for a, b, v in g["cases"]:
        assert oracle.ramanujan_perimeter(a, b) == pytest.approx(v, rel=g["rel_tol_vs_exact"])
    assert oracle.ramanujan_perimeter(1, 1) == pytest.approx(2 * math.pi, rel=1e-15)


@pytest.mark.parametrize("a,c", [(1, 2), (2, 1), (1, 3), (3, 1), (1, 1), (2.5, 0.7), (0.4, 3.3)])
def test_sphericity_3d_continuum(a, c):
    """Eq. 1 with the spheroid model: for V = 4/3 pi a^2 c and mean_lt = a, the model
    spheroid IS the body, so S = (36 pi V^2)^(1/3) / area (numeric integral)."""
    V = 4 / 3 * math.pi * a * a * c
    want = (36 * math.pi * V * V) ** (1 / 3) / _spheroid_area_numeric(a, c)
    assert oracle.sphericity_3d(V, a) == pytest.approx(want, rel=1e-10)
    assert oracle.sphericity_3d(V, a) <= 1 + 4 * 2.2e-16


def test_sphericity_continuum_named_values():
    g = _refs.load_closed_forms()["continuum_sphericity"]
    assert oracle.sphericity_3d(4 / 3 * math.pi * 2, 1.0) == pytest.approx(g["prolate_1to2"], abs=1e-6)
    # A = 2 pi, mean_lt 1 -> b = 2 -> ellipse 1:2
    assert oracle.sphericity_2d(2 * math.pi, 1.0) == pytest.approx(g["ellipse_2to1"], abs=5e-4)
    exact = 2 * math.sqrt(math.pi * 2 * math.pi) / _ellipse_perimeter_exact(2, 1)
    assert oracle.sphericity_2d(2 * math.pi, 1.0) == pytest.approx(exact, rel=1e-4)
    assert oracle.sphericity_3d(4 / 3 * math.pi * 8, 2.0) == pytest.approx(1.0, rel=1e-15)
    assert oracle.sphericity_2d(math.pi * 9, 3.0) == pytest.approx(1.0, rel=1e-15)


def test_sphericity_scale_covariance_and_monotonicity():
    for s in (0.5, 2.0, 7.0):
        assert oracle.sphericity_3d(s ** 3 * 100.0, s * 2.0) == pytest.approx(oracle.sphericity_3d(100.0, 2.0), rel=1e-13)
        assert oracle.sphericity_2d(s ** 2 * 100.0, s * 3.0) == pytest.approx(oracle.sphericity_2d(100.0, 3.0), rel=1e-13)
    # fixed area, growing elongation -> strictly decreasing 2D sphericity
    A = 100.0
    vals = [oracle.sphericity_2d(A, a) for a in np.linspace(math.sqrt(A / math.pi), 1.0, 12)]
    assert all(x > y for x, y in zip(vals, vals[1:]))


# ------------------------------------------------------------------------------------------
# invariants on the configs
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("cfg", [1, 2])
def test_invariants_on_configs(cfg):
    lab, info = synth.make_config(cfg)
    ml = info["max_label"]
    d2, lt2, sh = oracle.fields(lab, max_label=ml)
    r = oracle.sphericity_roundness(lab, max_label=ml)
    fg = lab > 0
    assert int(r["volume"].sum()) == int(fg.sum())
    assert (lt2[fg].astype(np.int64) >= d2[fg]).all()
    np.testing.assert_array_equal(sh.astype(bool), d2 == 1)
    for L in range(1, ml + 1):
        m = lab == L
        if not m.any():
            continue
        assert lt2[m].max() == d2[m].max() == r["max_lt2"][L - 1]
        assert lt2[m].min() >= d2[m].min()
    ok = r["volume"] > 0
    assert ((r["roundness"][ok] > 0) & (r["roundness"][ok] <= 1 + 4 * 2.2e-16)).all()
    assert (r["sphericity"][ok] <= 1 + 4 * 2.2e-16).all()
    # the closed-form check object (label ml) is the digital disk r=20 / sphere r=15
    g = _refs.load_closed_forms()["digital_disk_r20" if cfg == 1 else "digital_sphere_r15"]
    assert r["sphericity"][ml - 1] == pytest.approx(g["sphericity"], rel=1e-11)
    assert r["roundness"][ml - 1] == pytest.approx(1.0, abs=4e-16)


def test_survey_regression_values():
    """Values the survey computed with its own implementation of the same definitions
    (SURVEY.md §8(c) "Regression expectations"): ellipse 60x30, prolate 10x10x20."""
    r = oracle.sphericity_roundness(synth.ellipse(60, 30))
    assert r["mean_lt"][0] == pytest.approx(29.03358, abs=1e-5)
    assert math.sqrt(r["max_lt2"][0]) == pytest.approx(30.01666, abs=1e-5)
    assert r["shell_mean_lt"][0] == pytest.approx(25.98295, abs=1e-5)
    assert r["sphericity"][0] == pytest.approx(0.902880, abs=1e-6)
    assert r["roundness"][0] == pytest.approx(0.865618, abs=1e-6)
    r = oracle.sphericity_roundness(synth.spheroid(10, 20))
    assert r["volume"][0] == 8309
    assert r["sphericity"][0] == pytest.approx(0.915768, abs=1e-6)
    assert r["roundness"][0] == pytest.approx(0.926893, abs=1e-6)


def test_label_mask_and_absent_labels():
    lab, info = synth.make_config(1)
    ml = info["max_label"] + 3  # labels 22..24 absent -> NaN
    mask = np.zeros(ml, np.uint8)
    mask[[0, 5, 20]] = 1
    full = oracle.sphericity_roundness(lab, max_label=ml)
    part = oracle.sphericity_roundness(lab, max_label=ml, label_mask=mask)
    for i in range(ml):
        if mask[i]:
            assert part["sphericity"][i] == full["sphericity"][i]
        else:
            assert math.isnan(part["sphericity"][i])
    assert np.isnan(full["sphericity"][21:]).all() and (full["volume"][21:] == 0).all()


def test_batch_items_independent():
    a = synth.make_config(1)[0]
    b = synth.disk(20, canvas=256)
    stack = np.stack([a, b])
    r = oracle.sphericity_roundness(stack, max_label=21, ndim=2)
    ra = oracle.sphericity_roundness(a, max_label=21)
    np.testing.assert_array_equal(r["sphericity"][:21], ra["sphericity"])
    assert r["sphericity"][21] == pytest.approx(0.999999085802, rel=1e-11)


def test_touches_edge_spec_examples():
    """SPEC.md:215-218 remove_edge_objects examples, and the same rule on every face in 3D,
    per batch item."""
    a = np.zeros((5, 6), np.int32)
    a[0, 2] = 1  # a single object touching row 0
    assert oracle.touches_edge(a, 1).tolist() == [1]
    b = np.zeros((5, 6), np.int32)
    b[2, 2:4] = 1  # interior object only
    assert oracle.touches_edge(b, 1).tolist() == [0]
    c = b.copy()
    c[3:5, 5] = 2  # one interior + one edge object -> one label remains
    flags = oracle.touches_edge(c, 2)
    assert flags.tolist() == [0, 1] and int((flags == 0).sum()) == 1
    v = np.zeros((4, 5, 6), np.int32)
    v[1:3, 1:4, 1:5] = 1
    v[3, 2, 2] = 2  # last z slice
    v[1, 2, 0] = 3  # first x column
    v[2, 4, 3] = 4  # last y row
    v[2, 2, 2] = 5  # interior
    assert oracle.touches_edge(v, 5).tolist() == [0, 1, 1, 1, 0]
    batch = np.stack([b, c])  # per item: label 2 of item 1 touches, nothing in item 0
    assert oracle.touches_edge(batch, 2, ndim=2).tolist() == [0, 0, 0, 1]
    assert oracle.touches_edge(np.full((1, 1), 7), 6).tolist() == [0] * 6  # label > max_label ignored


def test_filter_objects_small_and_edge():
    """SPEC.md:220-224 filter_small examples through the result filter: min_volume 1 is the
    identity; a 27-voxel object is removed at 1000; a threshold above every object removes all."""
    lab = np.zeros((12, 12, 12), np.int32)
    lab[2:5, 2:5, 2:5] = 1  # 27 voxels
    lab[6:11, 6:11, 6:11] = 2  # 125 voxels
    res = oracle.sphericity_roundness(lab, max_label=2)
    same = oracle.filter_objects(res, min_volume=1)
    np.testing.assert_array_equal(same["sphericity"], res["sphericity"])
    f = oracle.filter_objects(res, min_volume=1000)
    assert np.isnan(f["sphericity"]).all() and np.isnan(f["roundness"]).all()
    g = oracle.filter_objects(res, min_volume=100)
    assert np.isnan(g["sphericity"][0]) and g["sphericity"][1] == res["sphericity"][1]
    h = oracle.filter_objects(res, edge=np.array([0, 1], np.uint8))
    assert h["roundness"][0] == res["roundness"][0] and np.isnan(h["roundness"][1])
