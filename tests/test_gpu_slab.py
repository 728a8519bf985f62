"""Z-slab path on the GPU: the four slab phases of the C ABI, driven by slab.simulate_slabs
(all ranks' slabs one after another on cuda:0 -- one GPU here; the real multi-rank exchange
code is covered over gloo in tests/test_slab.py), must give results BIT-IDENTICAL to the
single-call path fastrs_sphericity_roundness on the whole volume: every partial is an exact
integer (SURVEY.md §8(e) "Results must be bit-identical to 1 GPU")."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth
from paper_2504_05808_b200 import fastrs, slab

pytestmark = pytest.mark.gpu

KEYS = ("sphericity", "roundness", "volume", "n_shell", "max_lt2", "mean_lt", "shell_mean_lt", "axis_cb")


def _check(lab, nranks, flags=1):
    t = torch.from_numpy(np.ascontiguousarray(lab, np.int32)).cuda()
    ml = int(lab.max())
    want = fastrs.sphericity_roundness(t, max_label=ml, flags=flags, stats=True)
    got = slab.simulate_slabs(t, nranks, ml, flags=flags, stats=True)
    for k in KEYS:
        a, b = got[k].cpu().numpy(), want[k].cpu().numpy()
        np.testing.assert_array_equal(a, b, err_msg=f"{k} (nranks={nranks}, flags={flags})")
    return got["slab_info"]


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_c2_slabs_bit_identical(nranks):
    lab, _ = synth.make_config(2)
    info = _check(lab, nranks)
    assert info["H"] % 8 == 0 and info["h"] >= 1


@pytest.mark.parametrize("flags", [1, 0])
def test_touching_labels_slabs(flags):
    lab = synth.random_labels((70, 45, 50), nlabels=6, seed=11, fill=0.85, blob=5)
    if flags == 0:
        lab = np.pad(lab, 1)
    _check(lab, 3, flags)


def test_c3_eight_slabs():
    lab, _ = synth.make_config(3)
    _check(lab, 8)


def test_halo_spans_several_slabs():
    """A big sphere (r=30) across 6 slabs of 16: both halos reach two or more slabs away."""
    lab = np.zeros((96, 70, 70), np.int32)
    lab[15:76, 4:65, 4:65] = synth.sphere(30, canvas=61)
    lab[80:90, 10:60, 20:30] = 2
    info = _check(lab, 6)
    assert info["h"] > 16 and info["H"] > 16


def test_c4_four_slabs_full_size():
    """The slab phases at the bench's full size (1024^3, 20 000 grains, 4 slabs of 256)."""
    lab, _ = synth.make_config(4)
    info = _check(lab, 4)
    assert info["h"] <= 256 and info["H"] <= 256


def test_slab_phase_argument_errors():
    lab = torch.zeros((32, 16, 16), dtype=torch.int32, device="cuda")
    lab[4:20, 4:12, 4:12] = 1
    packed, _ = fastrs.slab_edt_xy(lab, None, 1)
    d, _ = fastrs.slab_edt_z(packed, 0, 32, 0, 32)
    with pytest.raises(fastrs.FastrsError) as e:  # own range not tile aligned
        fastrs.slab_reduce(lab[3:29].contiguous(), d, 3, 29, 32, 82, 1)
    assert e.value.name == "EINVAL"
    with pytest.raises(fastrs.FastrsError) as e:  # extended slab outside the grid
        fastrs.slab_edt_z(packed, 0, 32, 8, 32)
    assert e.value.name == "EINVAL"
