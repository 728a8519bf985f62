"""Generator scaffolding: determinism and the realised workload statistics."""
import numpy as np

import synth


def test_deterministic_c1_c2():
    for i in (1, 2):
        a, ia = synth.make_config(i)
        b, ib = synth.make_config(i)
        assert ia["sha256"] == ib["sha256"]
        np.testing.assert_array_equal(a, b)


def test_c1_c2_contents():
    lab, info = synth.make_config(1)
    assert lab.shape == (256, 256) and lab.dtype == np.int32
    assert info["max_label"] == 21 and info["n_labels_present"] == 21
    # disc r=20 at (128,128) is label 21 (closed-form check object)
    np.testing.assert_array_equal(lab[108:149, 108:149] == 21, synth.disk(20, canvas=41) == 1)
    lab, info = synth.make_config(2)
    assert lab.shape == (128, 128, 128) and info["max_label"] == 51
    assert 0.25 < info["fill"] < 0.45
    assert (lab[0] == 0).all() and (lab[-1] == 0).all()  # >= 1 element margin


def test_c5_small_batch_touching():
    lab, info = synth.make_config(5, batch=2)
    assert lab.shape == (2, 2048, 2048)
    assert 0.25 < info["fill"] < 0.5
    # touching allowed: some face-adjacent pairs of different non-zero labels exist
    a, b = lab[0, :, 1:], lab[0, :, :-1]
    assert ((a != b) & (a > 0) & (b > 0)).any()


def test_count_volume_matches_the_paper_experiment_shape():
    """The NEXT-1 stand-in volume (400^3, 15 503 objects of 27 to ~130 000 voxels):
    every object is placed, sizes span the paper's range (rasterised spheroids and rough grains
    deviate from the nominal volume by tens of percent at the extremes), fill is moderate."""
    lab, info = synth.make_count_volume()
    assert lab.shape == (400, 400, 400) and lab.dtype == np.int32
    assert info["n_labels_present"] == 15503 and info["max_label"] == 15503
    v = np.bincount(lab.ravel(), minlength=15504)[1:]
    assert v.min() >= 10 and 27 * 0.5 <= np.percentile(v, 1) and v.max() <= 2 * 130000
    assert 0.15 < info["fill"] < 0.30


def test_c5_image_shards_equal_the_batch():
    """bench.py's C5 shard of rank r (images [i0, i1) of the seeded batch) equals that slice of the
    whole batch: the draws do not depend on the shard."""
    a, _ = synth.make_config(5, batch=5)
    b, _ = synth.make_config(5, batch=5, images=(1, 4))
    np.testing.assert_array_equal(a[1:4], b)
