"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): bit-exact for squared distances, LT^2, counts and shell
masks; float64 sphericity / roundness within 1e-5 relative (the derivation of the much
tighter actual error is in DESIGN.md "Tolerances": the fixed-point LT sums err by
<= V * 2^-(s+1) absolute, s >= 20).
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from tests import _refs

pytestmark = pytest.mark.gpu

RTOL = 1e-5


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2504_05808_b200 import fastrs
    fastrs.load()
    return fastrs


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def compare_metrics(got: dict, want: dict, where=""):
    g = {k: v.cpu().numpy() for k, v in got.items()}
    np.testing.assert_array_equal(g["volume"], want["volume"], err_msg=where)
    np.testing.assert_array_equal(g["n_shell"], want["n_shell"], err_msg=where)
    np.testing.assert_array_equal(g["max_lt2"].view(np.uint32), want["max_lt2"], err_msg=where)
    present = want["volume"] > 0
    assert np.isnan(g["sphericity"][~present]).all() and np.isnan(g["roundness"][~present]).all()
    for k in ("sphericity", "roundness", "mean_lt", "shell_mean_lt", "axis_cb"):
        np.testing.assert_allclose(g[k][present], want[k][present], rtol=RTOL, atol=0, err_msg=f"{where} {k}")


def full_check(F, lab, flags, ndim=None, max_label=None, fields=True):
    """D, LT^2 and all per-label outputs vs the oracle."""
    ndim = ndim or lab.ndim
    ml = max_label or max(1, int(lab.max()))
    t = _dev(lab)
    if fields:
        d2, lt2, sh = oracle.fields(lab, max_label=ml, flags=flags, ndim=ndim)
        np.testing.assert_array_equal(_u32(F.edt_sq(t, ndim=ndim, flags=flags)), d2)
        np.testing.assert_array_equal(_u32(F.local_thickness(t, ndim=ndim, flags=flags)), lt2)
        np.testing.assert_array_equal(_u32(F.local_thickness(t, ndim=ndim, flags=flags | F.FORCE_FALLBACK)), lt2)
        lt_f = F.local_thickness(t, ndim=ndim, flags=flags, lt2=False, lt=True).cpu().numpy()
        np.testing.assert_array_equal(lt_f, np.sqrt(lt2.astype(np.float64)).astype(np.float32))
    got = F.sphericity_roundness(t, max_label=ml, ndim=ndim, flags=flags, stats=True)
    want = oracle.sphericity_roundness(lab, max_label=ml, flags=flags, ndim=ndim)
    compare_metrics(got, want)
    return got, want


# ------------------------------------------------------------------------------------------
# tiny random grids: touching labels, ragged sizes, both border modes
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("border", [1, 0])
@pytest.mark.parametrize("seed", range(40))
def test_random_tiny(F, seed, border):
    rng = np.random.default_rng(seed)
    if seed % 2:
        shape = tuple(int(v) for v in rng.integers(3, 40, 3))
    else:
        shape = tuple(int(v) for v in rng.integers(3, 150, 2))
    lab = synth.random_labels(shape, nlabels=int(rng.integers(1, 6)), seed=seed, fill=float(rng.uniform(0.3, 0.95)),
                              blob=int(rng.integers(1, 6)))
    try:
        oracle.edt_sq(lab, flags=border)
    except oracle.OracleError as e:
        assert e.code == 2
        with pytest.raises(F.FastrsError) as ge:
            F.edt_sq(_dev(lab), flags=border)
        assert ge.value.name == "ENOSITE"
        return
    if lab.max() == 0:
        lab[0, 0] = 1
    full_check(F, lab, border)


@pytest.mark.parametrize("border", [1, 0])
@pytest.mark.parametrize("shape", [(5, 128), (3, 1152), (6, 2048), (4, 5, 256), (3, 4, 1024), (2, 3, 1152)])
def test_k1_segment_form(F, shape, border):
    """K1's segment form (X % 128 == 0: per-lane 32-element segments, 1024-element blocks, carries
    between blocks; 1152 = one full block + a partial one) against the oracle's EDT and against
    the warp-sweep form (FASTRS_K1_WARP) bit for bit, on runs short and long."""
    for k, (nl, blob) in enumerate([(6, 1), (3, 9), (2, 40)]):
        lab = synth.random_labels(shape, nlabels=nl, seed=sum(shape) + 7 * k + border, fill=0.7, blob=blob)
        lab.flat[0] = 0  # a site in every case (no ENOSITE without the border flag)
        if lab.max() == 0:
            lab.flat[1] = 1
        t = _dev(lab)
        got = _u32(F.edt_sq(t, flags=border))
        np.testing.assert_array_equal(got, oracle.edt_sq(lab, flags=border))
        os.environ["FASTRS_K1_WARP"] = "1"
        try:
            warp_form = _u32(F.edt_sq(t, flags=border))
        finally:
            del os.environ["FASTRS_K1_WARP"]
        np.testing.assert_array_equal(got, warp_form)


@pytest.mark.parametrize("border", [1, 0])
@pytest.mark.parametrize("seed", range(12))
def test_envelope_column_pass(F, seed, border):
    """The exact lower-envelope column pass (K2/K3 fix-up for the CTAs the 16-bit scan cannot
    finish) forced on EVERY CTA (FASTRS_COL_FH_ALL): D element by element against the oracle on
    random touching-label grids, ragged sizes, both border modes, short and long runs."""
    rng = np.random.default_rng(1000 + seed)
    shape = tuple(int(v) for v in rng.integers(3, 60, 3)) if seed % 2 else tuple(int(v) for v in rng.integers(3, 300, 2))
    lab = synth.random_labels(shape, nlabels=int(rng.integers(1, 6)), seed=seed, fill=float(rng.uniform(0.3, 0.95)),
                              blob=int(rng.integers(1, 12)))
    lab.flat[0] = 0
    if lab.max() == 0:
        lab.flat[1] = 1
    try:
        want = oracle.edt_sq(lab, flags=border)
    except oracle.OracleError as e:
        assert e.code == 2
        return
    t = _dev(lab)
    os.environ["FASTRS_COL_FH_ALL"] = "1"
    try:
        got = _u32(F.edt_sq(t, flags=border))
        lt2 = _u32(F.local_thickness(t, flags=border))
    finally:
        del os.environ["FASTRS_COL_FH_ALL"]
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(lt2, _u32(F.local_thickness(t, flags=border)))


def test_envelope_column_pass_large_objects(F):
    """Objects far wider than the staged window (radius 95 sphere, a 150 x 60 ellipse and
    touching neighbours): the envelope pass against scipy's EDT, and against the windowed 32-bit
    scan (FASTRS_COL_WINDOWED) bit for bit."""
    import scipy.ndimage
    lab = synth.sphere(95, canvas=200)
    lab[150:, :, :] = np.where(lab[150:, :, :] > 0, 2, 0)  # cut the cap off as a touching label
    yy, xx = np.ogrid[:400, :700]
    ell = (((yy - 200) / 150.0) ** 2 + ((xx - 350) / 330.0) ** 2 <= 1).astype(np.int32)
    for img in (lab, ell):
        t = _dev(img)
        got = _u32(F.edt_sq(t))
        os.environ["FASTRS_COL_WINDOWED"] = "1"
        try:
            win = _u32(F.edt_sq(t))
        finally:
            del os.environ["FASTRS_COL_WINDOWED"]
        np.testing.assert_array_equal(got, win)
        if img.max() == 1:
            ref = np.rint(scipy.ndimage.distance_transform_edt(np.pad(img > 0, 1)) ** 2).astype(np.uint32)
            np.testing.assert_array_equal(got, ref[(slice(1, -1),) * img.ndim])


def _edt_env(F, t, env, flags=1, ndim=None):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        got = _u32(F.edt_sq(t, flags=flags, ndim=ndim))
        d = F.diagnostics(F.last_workspace())
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    return got, d


def test_column_slow_list(F):
    """K2/K3 elements whose scan leaves the staged window go to a list scanned by a separate kernel
    with batched L2 reads (round 2c): D against scipy / the oracle, bit-identical to the in-line
    32-bit scan (FASTRS_COL_INLINE), and with a 3-entry list (FASTRS_COL_SLOW_CAP) whose overflow
    takes the in-line scan; n_col_slow > 0 shows the list was used."""
    import scipy.ndimage
    yy, xx = np.ogrid[:300, :520]
    ell = (((yy - 150) / 120.0) ** 2 + ((xx - 260) / 250.0) ** 2 <= 1).astype(np.int32)
    zz, yy3, xx3 = np.ogrid[:420, :130, :130]  # a z cylinder of radius 60: K3 scans cross segment ends
    sph = (((yy3 - 65) ** 2 + (xx3 - 65) ** 2 <= 60 ** 2) & (zz >= 5) & (zz < 400)).astype(np.int32)
    del zz, yy3, xx3
    blobs = synth.random_labels((500, 480), nlabels=3, seed=11, fill=0.9, blob=120)
    blobs.flat[0] = 0
    for img, border in ((ell, 1), (sph, 1), (sph, 0), (blobs, 1), (blobs, 0)):
        t = _dev(img)
        got, d = _edt_env(F, t, {})
        if img is not blobs:
            assert d["n_col_slow"] > 0, d
        inline, d_in = _edt_env(F, t, {"FASTRS_COL_INLINE": "1"}, flags=border)
        assert d_in["n_col_slow"] == 0
        got, _ = _edt_env(F, t, {}, flags=border)
        np.testing.assert_array_equal(got, inline)
        capped, d_cap = _edt_env(F, t, {"FASTRS_COL_SLOW_CAP": "3"}, flags=border)
        assert d_cap["n_col_slow"] > 3
        np.testing.assert_array_equal(capped, inline)
        if img.max() == 1 and border == 1:
            ref = np.rint(scipy.ndimage.distance_transform_edt(np.pad(img > 0, 1)) ** 2).astype(np.uint32)
            np.testing.assert_array_equal(got, ref[(slice(1, -1),) * img.ndim])
        elif img is blobs:
            np.testing.assert_array_equal(got, oracle.edt_sq(img, flags=border))


@pytest.mark.parametrize("shape", [(1, 1), (1, 77), (77, 1), (2, 3, 1), (1, 1, 1), (9, 1, 40), (33, 65),
                                   (17, 9, 33), (8, 8, 32), (8, 64, 64), (3, 16384)])
def test_ragged_and_degenerate_shapes(F, shape):
    lab = synth.random_labels(shape, nlabels=3, seed=sum(shape), fill=0.7, blob=3)
    if lab.max() == 0:
        lab.flat[0] = 1
    full_check(F, lab, 1)


def test_closed_form_objects(F):
    cf = _refs.load_closed_forms()
    # LT sums are exact fixed-point integers of terms rounded to 2^-s (s = 32 here): the
    # means carry <= 2^-(s+1) absolute error, i.e. ~1e-11 relative at lt ~ 15-20
    got, _ = full_check(F, synth.disk(20), 1)
    assert got["sphericity"][0].item() == pytest.approx(cf["digital_disk_r20"]["sphericity"], rel=1e-9)
    assert got["roundness"][0].item() == pytest.approx(1.0, abs=1e-9)
    got, _ = full_check(F, synth.sphere(15), 1)
    assert got["sphericity"][0].item() == pytest.approx(cf["digital_sphere_r15"]["sphericity"], rel=1e-9)
    assert got["roundness"][0].item() == pytest.approx(1.0, abs=1e-9)
    assert int(got["max_lt2"][0]) == 226 and int(got["n_shell"][0]) == 2262


def test_spec_examples(F):
    for name, c in _refs.load_spec_examples().items():
        if "labels" not in c:
            continue
        lab = c["labels"].astype(np.int32)
        np.testing.assert_array_equal(_u32(F.edt_sq(_dev(lab))), c["d2"], err_msg=name)
        if "lt2" in c:
            np.testing.assert_array_equal(_u32(F.local_thickness(_dev(lab))), c["lt2"], err_msg=name)


def test_large_balls_beyond_table_and_halo(F):
    """Objects whose D exceeds the staged column halo (32^2) and the 3D containment-table cap
    (8192 -> radius > 90): exercises the global-memory window fallback and never-pruned
    centres.  Too big for the all-balls oracle, so pinned by closed forms instead: the EDT
    of a single label is scipy's binary EDT of the padded mask, and a digital disk/sphere of
    radius r centred on an element has D(centre) = r^2 + 1 and LT^2 = r^2 + 1 everywhere
    (the centre ball covers the whole object)."""
    import scipy.ndimage
    # r = 300: D = 90001 > 65535 sends every tile to the atomic sparse-table kernel (u32 values)
    for lab, r in ((synth.disk(150, canvas=311), 150), (synth.sphere(95, canvas=193), 95),
                   (synth.disk(300, canvas=605), 300)):
        t = _dev(lab)
        ref = np.rint(scipy.ndimage.distance_transform_edt(np.pad(lab > 0, 1)) ** 2).astype(np.uint32)
        ref = ref[(slice(1, -1),) * lab.ndim]
        np.testing.assert_array_equal(_u32(F.edt_sq(t)), ref)
        lt2 = _u32(F.local_thickness(t))
        assert (lt2[lab > 0] == r * r + 1).all() and (lt2[lab == 0] == 0).all()
        got = F.sphericity_roundness(t, max_label=1, stats=True)
        assert got["roundness"][0].item() == 1.0
        assert int(got["volume"][0]) == int((lab > 0).sum())


def test_big_bucket_scatter_rounds(F):
    """Large objects (radii 32-50, Dmax > 1536): thousands of nearly tangent kept balls of similar D
    reach a tile group.  The cover cut (the largest reaching ball contains the group's foreground)
    drops them; without it (NO_COVER_CUT) one D bucket overflows the gather's shared list and its
    sort range, and K5a writes that bucket by exact-D scatter rounds (count, prefix sum, scatter)
    instead of handing the group to the atomic fallback.  LT^2 element by element against the fallback kernel (an independent
    dilation: per-tile reverse sparse tables), D against scipy's EDT (labels separated by
    background), the centre-ball closed form LT^2 = r^2 + 1 in the core of the big sphere, and the
    per-label outputs of both paths."""
    import scipy.ndimage
    Z, Y, X = 224, 160, 160
    z, y, x = np.ogrid[:Z, :Y, :X]
    lab = np.zeros((Z, Y, X), np.int32)
    big = (z - 64) ** 2 + (y - 80) ** 2 + (x - 80) ** 2 <= 50 ** 2
    small = (z - 140) ** 2 + (y - 80) ** 2 + (x - 80) ** 2 <= 32 ** 2  # overlaps the big one: a dumbbell
    lab[big | small] = 1
    other = (z - 180) ** 2 + (y - 124) ** 2 + (x - 118) ** 2 <= 34 ** 2  # 2 voxels clear of the dumbbell
    lab[other & ~(big | small)] = 2
    lab[(z - 190) ** 2 + (y - 40) ** 2 + (x - 40) ** 2 <= 12 ** 2] = 3
    t = _dev(lab)
    ref = np.rint(scipy.ndimage.distance_transform_edt(np.pad(lab > 0, 1)) ** 2).astype(np.uint32)[1:-1, 1:-1, 1:-1]
    sep = scipy.ndimage.binary_dilation(lab == 2) & (lab == 1)
    assert not sep.any()  # label 2 does not touch label 1: the binary EDT is the label-aware one
    np.testing.assert_array_equal(_u32(F.edt_sq(t)), ref)
    lt2 = _u32(F.local_thickness(t))
    d = F.diagnostics(F.last_workspace())
    assert d["n_fallback"] == 0, d
    # without the cover cut every reaching ball is listed: one D bucket overflows -> scatter rounds
    lt2_long = _u32(F.local_thickness(t, flags=1 | F.NO_COVER_CUT))
    d_long = F.diagnostics(F.last_workspace())
    assert d_long["n_fallback"] == 0 and d_long["n_rounds_extra"] > 0, d_long
    assert d_long["sum_group_list"] > d["sum_group_list"], (d_long, d)
    lt2_fb = _u32(F.local_thickness(t, flags=1 | F.FORCE_FALLBACK))
    np.testing.assert_array_equal(lt2, lt2_fb)
    np.testing.assert_array_equal(lt2_long, lt2_fb)
    core = (z - 64) ** 2 + (y - 80) ** 2 + (x - 80) ** 2 <= 20 ** 2
    assert (lt2[core & (lab == 1)] == 50 * 50 + 1).all()
    fg = lab > 0
    assert (lt2[fg] >= ref[fg]).all() and (lt2[~fg] == 0).all()
    got = F.sphericity_roundness(t, max_label=3, stats=True)
    want = F.sphericity_roundness(t, max_label=3, stats=True, flags=1 | F.FORCE_FALLBACK)
    for k in ("volume", "n_shell", "max_lt2", "sphericity", "roundness", "mean_lt", "shell_mean_lt"):
        assert torch.equal(got[k], want[k]), k


def test_dilation_waves_on_a_full_pool(F):
    """A candidate pool too small for the gather (FASTRS_POOL_DIV shrinks it) defers tile groups to
    later waves of K5a + K5b over the reused pool (only the last wave's overflow goes to the atomic
    fallback): results bit-identical to the default call, LT^2 equal to the oracle's on C2."""
    for cfg, div in ((2, 40), (3, 24)):
        lab, info = synth.make_config(cfg)
        ml = info["max_label"]
        t = _dev(lab)
        want = F.sphericity_roundness(t, max_label=ml, stats=True)
        lt_want = F.local_thickness(t)
        os.environ["FASTRS_POOL_DIV"] = str(div)
        try:
            got = F.sphericity_roundness(t, max_label=ml, stats=True)
            d = F.diagnostics(F.last_workspace())
            lt_got = F.local_thickness(t)
        finally:
            del os.environ["FASTRS_POOL_DIV"]
        assert d["n_deferred"] > 0, d
        assert torch.equal(lt_got, lt_want)
        for k in ("volume", "n_shell", "max_lt2", "mean_lt", "shell_mean_lt", "sphericity", "roundness"):
            np.testing.assert_array_equal(got[k].cpu().numpy(), want[k].cpu().numpy(), err_msg=k)  # (NaN == NaN)
        if cfg == 2:
            np.testing.assert_array_equal(_u32(lt_got), oracle.fields(lab, max_label=ml, flags=1)[1])


def test_empty_and_single_element_objects(F):
    lab = np.zeros((20, 21, 22), np.int32)
    r = F.sphericity_roundness(_dev(lab), max_label=3)
    assert torch.isnan(r["sphericity"]).all()
    lab[3, 4, 5] = 2
    lab[10, 10, 10] = 3
    lab[10, 10, 11] = 1  # touching another label
    full_check(F, lab, 1, max_label=5)
    full_check(F, lab, 0, max_label=5)


def test_errors(F):
    lab = np.zeros((8, 8), np.int32)
    lab[2, 2] = 9
    with pytest.raises(F.FastrsError) as e:
        F.sphericity_roundness(_dev(lab), max_label=4)
    assert e.value.name == "EINVAL"
    lab[2, 2] = -1
    with pytest.raises(F.FastrsError) as e:
        F.edt_sq(_dev(lab))
    assert e.value.name == "EINVAL"
    with pytest.raises(F.FastrsError) as e:
        F.edt_sq(_dev(np.ones((5, 6, 7), np.int32)), flags=0)
    assert e.value.name == "ENOSITE"


def test_batched_items_are_independent(F):
    a = synth.random_labels((3, 40, 50), nlabels=4, seed=3, fill=0.8, blob=4)
    full_check(F, a, 1, ndim=2)
    b = synth.random_labels((2, 12, 20, 33), nlabels=4, seed=4, fill=0.8, blob=3)
    full_check(F, b, 1, ndim=3)
    # X % 4 == 0: K4 stages its tiles through the 4D TMA tensor map (batch as the 4th dim)
    c = synth.random_labels((3, 19, 21, 36), nlabels=5, seed=6, fill=0.8, blob=3)
    full_check(F, c, 1, ndim=3)
    # a batch equals its items run one by one
    t = _dev(a)
    rb = F.sphericity_roundness(t, max_label=4, ndim=2)["roundness"].cpu().numpy().reshape(3, 4)
    for i in range(3):
        ri = F.sphericity_roundness(_dev(a[i]), max_label=4)["roundness"].cpu().numpy()
        np.testing.assert_array_equal(rb[i], ri)


# ------------------------------------------------------------------------------------------
# BASELINE.json configs
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("cfg", [1, 2])
def test_config_full(F, cfg):
    lab, info = synth.make_config(cfg)
    got, want = full_check(F, lab, 1, max_label=info["max_label"])
    cf = _refs.load_closed_forms()["digital_disk_r20" if cfg == 1 else "digital_sphere_r15"]
    i = info["max_label"] - 1
    assert got["sphericity"][i].item() == pytest.approx(cf["sphericity"], rel=1e-9)


def test_config_c3_full(F):
    """C3 in full (512^3, 2000 grains), element by element: D, LT^2 (default and fallback
    dilation), the float LT radius, and every per-label output."""
    lab, info = synth.make_config(3)
    full_check(F, lab, 1, max_label=info["max_label"], fields=True)


def test_config_c5_subset(F):
    """Three C5 images (touching cells), element by element.  Their Dmax exceeds the 1536-bin
    single-pass sort, so K5a builds every candidate list in exact D-bucket rounds."""
    lab, info = synth.make_config(5, batch=3)
    full_check(F, lab, 1, ndim=2, max_label=info["max_label"], fields=True)
    d = F.diagnostics(F.last_workspace())
    assert d["dmax"] > 1536, d


@pytest.fixture(scope="module")
def c4():
    return synth.make_config(4)


def test_config_c4_label_subset_fields(F, c4):
    """C4 at full size (1024^3) with 2000 grains kept (its 250 largest and 1750 drawn at random)
    and the others zeroed (exact: C4 grains are separated by >= 1 voxel, so the kept grains' D
    and LT^2 are unchanged), element by element against the oracle's full-grid fields.  The
    large grains' candidate lists overflow the shared list, so K5a's list staging is
    exercised."""
    lab, info = c4
    ml = info["max_label"]
    counts = np.bincount(lab.reshape(-1), minlength=ml + 1)
    order = np.argsort(counts[1:]) + 1
    rng = np.random.default_rng(45)
    keep = np.zeros(ml + 1, bool)
    keep[order[-250:]] = True
    keep[rng.choice(order[:-250], 1750, replace=False)] = True
    sub = np.where(keep[lab], lab, 0).astype(np.int32)
    full_check(F, sub, 1, max_label=ml, fields=True)
    d = F.diagnostics(F.last_workspace())
    assert d["n_staged"] > 0 and d["n_regathers"] == 0, d
    del sub


def test_config_c4_regather_path_identical(F, c4):
    """C4 at full size with the list staging disabled (test hook FASTRS_NO_LIST_STAGING): the
    overflowing candidate lists take K5a's second gather pass instead; every output is
    bit-identical to the default (staged) call, which the oracle pins element by element above."""
    lab, info = c4
    ml = info["max_label"]
    t = _dev(lab)
    a = F.sphericity_roundness(t, max_label=ml, stats=True)
    da = F.diagnostics(F.last_workspace(t.device))
    b = F.sphericity_roundness(t, max_label=ml, stats=True, flags=F.BORDER_BACKGROUND | F.NO_LIST_STAGING)
    db = F.diagnostics(F.last_workspace(t.device))
    assert da["n_staged"] > 0 and da["n_regathers"] == 0, da
    assert db["n_regathers"] > 0 and db["n_staged"] == 0, db
    for k in a:
        assert torch.equal(a[k], b[k]), k


def test_config_c4_sampled(F, c4):
    """C4 at full size in the bench's launch configuration; the oracle evaluates a seeded
    sample of labels one by one (exact by crop exactness)."""
    lab, info = c4
    ml = info["max_label"]
    t = _dev(lab)
    got = F.sphericity_roundness(t, max_label=ml, stats=True)
    rng = np.random.default_rng(44)
    mask = np.zeros(ml, np.uint8)
    mask[rng.choice(ml, 300, replace=False)] = 1
    want = oracle.sphericity_roundness(lab, max_label=ml, label_mask=mask)
    sel = mask.astype(bool)
    g = {k: v.cpu().numpy()[sel] for k, v in got.items()}
    w = {k: v[sel] for k, v in want.items()}
    compare_metrics({k: torch.from_numpy(v) for k, v in g.items()}, w)
    # whole-grid invariants
    assert int(got["volume"].sum()) == int(np.count_nonzero(lab))
    ok = got["volume"] > 0
    assert bool((got["roundness"][ok] <= 1 + 1e-12).all()) and bool((got["roundness"][ok] > 0).all())
    assert bool((got["sphericity"][ok] <= 1 + 1e-12).all())


def test_deterministic_and_host_path(F):
    lab, info = synth.make_config(2)
    t = _dev(lab)
    r1 = F.sphericity_roundness(t, max_label=51)
    r2 = F.sphericity_roundness(t, max_label=51)
    assert torch.equal(r1["sphericity"], r2["sphericity"]) and torch.equal(r1["roundness"], r2["roundness"])
    s, r = F.sphericity_roundness_host(lab, max_label=51)
    np.testing.assert_array_equal(s, r1["sphericity"].cpu().numpy())
    np.testing.assert_array_equal(r, r1["roundness"].cpu().numpy())


def test_diagnostics_counters(F):
    lab = synth.sphere(15)
    t = _dev(lab)
    F.sphericity_roundness(t, max_label=1, flags=1 | F.EXACT_PRUNE)
    d = F.diagnostics(F.last_workspace(t.device))
    assert d["status_bits"] == 0 and d["dmax"] == 226 and d["n_fg"] == 14147
    # exact lattice pruning with the 26-neighbourhood, then all |s|^2 <= 12, keeps 121
    # centres on the digital sphere r=15 (SURVEY.md §8(c) "Kept-centre counts")
    assert d["n_kept"] == 121
    lt_exact = F.local_thickness(t, flags=1 | F.EXACT_PRUNE)
    r_exact = F.sphericity_roundness(t, max_label=1, flags=1 | F.EXACT_PRUNE, stats=True)
    # the default (five stage-2 classes) keeps a superset of those balls and the same LT^2
    r_fast = F.sphericity_roundness(t, max_label=1, stats=True)
    assert F.diagnostics(F.last_workspace(t.device))["n_kept"] >= 121
    assert torch.equal(F.local_thickness(t), lt_exact)
    for k in ("volume", "n_shell", "max_lt2", "sphericity", "roundness"):
        assert torch.equal(r_fast[k], r_exact[k]), k
    F.sphericity_roundness(_dev(synth.disk(20)), max_label=1)
    d = F.diagnostics(F.last_workspace(t.device))
    assert d["n_fg"] == 1257 and d["dmax"] == 401
    assert d["n_kept"] <= 9  # 8-neighbourhood alone keeps 9; |s|^2 <= 8 keeps fewer


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_dilation_cross_check_full_size(F, cfg, c4):
    """The default exact-order cover dilation and the independent atomic sparse-table kernel
    (FASTRS_FORCE_FALLBACK) give bit-identical LT^2 on every element of the full-size
    configs (the oracle itself is checked against both on the sampled/full tests above)."""
    if cfg == 4:
        lab, info = c4
    else:
        lab, info = synth.make_config(cfg, batch=4) if cfg == 5 else synth.make_config(cfg)
    ndim = 2 if cfg == 5 else 3
    t = _dev(lab)
    a = F.local_thickness(t, ndim=ndim)
    b = F.local_thickness(t, ndim=ndim, flags=F.BORDER_BACKGROUND | F.FORCE_FALLBACK)
    assert torch.equal(a, b)
    d = F.edt_sq(t, ndim=ndim)
    assert bool((a.view(torch.int32) >= d.view(torch.int32)).all())
    del a, b, d, t
    torch.cuda.empty_cache()


def test_host_entry_point_pipelined_matches_device_call(F):
    """fastrs_sphericity_roundness_host on a volume deep enough for the chunked copy/compute
    pipeline (Z >= 512) gives results bit-identical to the device call; with a ball too big for
    one chunk (R > 128) the pipeline's halo check fails and the call recomputes: still exact."""
    lab, info = synth.make_config(3)
    ml = info["max_label"]
    want = F.sphericity_roundness(_dev(lab), max_label=ml)
    s, r = F.sphericity_roundness_host(lab, max_label=ml)
    np.testing.assert_array_equal(s, want["sphericity"].cpu().numpy())
    np.testing.assert_array_equal(r, want["roundness"].cpu().numpy())
    # small grains in the first chunks and a large ball near the end: Dmax grows from chunk to
    # chunk.  The fused per-chunk reductions use the fixed 2^-32 scale (no dependence on Dmax,
    # ADVICE r1), so they are final: bit-identical to the device call and equal to the oracle
    mixed = np.zeros((512, 96, 96), np.int32)
    k = 0
    for z in range(8, 300, 12):
        for y in range(8, 90, 12):
            k += 1
            mixed[z - 3:z + 4, y - 3:y + 4, 40:47] = np.where(synth.sphere(3, canvas=7) > 0, k, 0)
    mixed[380:461, 8:89, 8:89] = np.where(synth.sphere(40, canvas=81) > 0, k + 1, 0)
    want = F.sphericity_roundness(_dev(mixed), max_label=k + 1)
    s, r = F.sphericity_roundness_host(mixed, max_label=k + 1)
    np.testing.assert_array_equal(s, want["sphericity"].cpu().numpy())
    np.testing.assert_array_equal(r, want["roundness"].cpu().numpy())
    ref = oracle.sphericity_roundness(mixed, max_label=k + 1)
    np.testing.assert_allclose(s, ref["sphericity"], rtol=RTOL, atol=0)
    np.testing.assert_allclose(r, ref["roundness"], rtol=RTOL, atol=0)
    big = np.zeros((520, 310, 310), np.int32)
    big[5:306, 5:306, 5:306] = synth.sphere(150, canvas=301)
    big[400:440, 100:120, 100:130] = 2
    want = F.sphericity_roundness(_dev(big), max_label=2)
    s, r = F.sphericity_roundness_host(big, max_label=2)
    np.testing.assert_array_equal(s, want["sphericity"].cpu().numpy())
    np.testing.assert_array_equal(r, want["roundness"].cpu().numpy())
    assert r[0] == 1.0


def test_count_volume_subsets(F):
    """NEXT-1 (tools/count_scaling.py): subsets of the 400^3 count volume with the other labels
    zeroed; the drawn objects' metrics match the oracle (the zeroed ones stay absent)."""
    lab, info = synth.make_count_volume()
    ml = info["max_label"]
    rng = np.random.default_rng(3)
    for n in (1, 37):
        sel = np.sort(rng.choice(np.arange(1, ml + 1), n, replace=False))
        sub = np.where(np.isin(lab, sel), lab, 0).astype(np.int32)
        got = F.sphericity_roundness(_dev(sub), max_label=ml, stats=True)
        mask = np.zeros(ml, np.uint8)
        mask[sel - 1] = 1
        want = oracle.sphericity_roundness(sub, max_label=ml, label_mask=mask)
        np.testing.assert_array_equal(got["volume"].cpu().numpy()[sel - 1], want["volume"][sel - 1])
        for k in ("sphericity", "roundness", "mean_lt"):
            np.testing.assert_allclose(got[k].cpu().numpy()[sel - 1], want[k][sel - 1], rtol=RTOL, atol=0)
        assert np.isnan(got["sphericity"].cpu().numpy()[np.setdiff1d(np.arange(ml), sel - 1)]).all()


def test_touches_edge_and_filters_match_oracle(F):
    """NEXT-4 label-level filters: edge objects are flagged exactly as the oracle's
    plain definition on 2D, 3D and batched inputs, and the small-object / edge filters
     blank the same labels."""
    cases = [(synth.make_config(1)[0], 21, None), (synth.make_config(5, batch=3)[0], 500, 2),
             (synth.random_labels((2, 12, 20, 36), nlabels=6, seed=8, fill=0.8, blob=3), 6, 3),
             (synth.random_labels((33, 1, 17), nlabels=3, seed=9, fill=0.9, blob=2), 3, None)]
    for lab, ml, nd in cases:
        got = F.touches_edge(_dev(lab), ml, ndim=nd).cpu().numpy()
        want = oracle.touches_edge(lab, ml, ndim=nd)
        np.testing.assert_array_equal(got, want)
    lab, info = synth.make_config(2)
    ml = info["max_label"]
    t = _dev(lab)
    res = F.sphericity_roundness(t, max_label=ml, stats=True)
    edge = F.touches_edge(t, ml)
    F.filter_objects(res, min_volume=1000, edge=edge)
    ref = oracle.filter_objects(oracle.sphericity_roundness(lab, max_label=ml), min_volume=1000,
                                edge=oracle.touches_edge(lab, ml))
    for k in ("sphericity", "roundness"):
        g, w = res[k].cpu().numpy(), ref[k]
        np.testing.assert_array_equal(np.isnan(g), np.isnan(w))
        ok = ~np.isnan(w)
        assert ok.any()
        np.testing.assert_allclose(g[ok], w[ok], rtol=RTOL, atol=0)
