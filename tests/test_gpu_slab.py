"""Z-slab path on the GPU: the four slab phases of the C ABI, driven by slab.simulate_slabs
(all ranks' slabs one after another on cuda:0 -- one GPU here; the real multi-rank exchange
code is covered over gloo in tests/test_slab.py), must give results BIT-IDENTICAL to the
single-call path fastrs_sphericity_roundness on the whole volume: every partial is an exact
integer (SURVEY.md §8(e) "Results must be bit-identical to 1 GPU")."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2504_05808_b200 import fastrs, slab

pytestmark = pytest.mark.gpu

KEYS = ("sphericity", "roundness", "volume", "n_shell", "max_lt2", "mean_lt", "shell_mean_lt", "axis_cb")


def _check(lab, nranks, flags=1, transpose=False, lt_halo="dense", split_zpass=False):
    t = torch.from_numpy(np.ascontiguousarray(lab, np.int32)).cuda()
    ml = int(lab.max())
    want = fastrs.sphericity_roundness(t, max_label=ml, flags=flags, stats=True)
    got = slab.simulate_slabs(t, nranks, ml, flags=flags, stats=True, transpose=transpose, lt_halo=lt_halo,
                              split_zpass=split_zpass)
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


def test_touches_edge_slabs_or_to_the_volume_flags():
    """Edge flags from z-slabs (inner slab faces skipped) OR-ed together equal the flags of the
    whole volume (what slab.touches_edge_slab's allreduce(max) computes across ranks)."""
    rng = np.random.default_rng(12)
    lab = np.zeros((64, 40, 48), np.int32)
    for k in range(1, 81):  # boxes anywhere: some on faces, some across slab boundaries
        sz = rng.integers(1, 7, 3)
        lo = [int(rng.integers(0, n - w + 1)) for n, w in zip(lab.shape, sz)]
        lab[lo[0]:lo[0] + sz[0], lo[1]:lo[1] + sz[1], lo[2]:lo[2] + sz[2]] = k
    ml = 80
    t = torch.from_numpy(lab).cuda()
    want = fastrs.touches_edge(t, ml)
    assert 0 < int(want.sum()) < ml
    slabs = slab.partition(lab.shape[0], 5)
    acc = torch.zeros_like(want)
    for z0, z1 in slabs:
        f = fastrs.touches_edge(t[z0:z1].contiguous(), ml,
                                flags=(fastrs.EDGE_SKIP_ZLO if z0 > 0 else 0) | (fastrs.EDGE_SKIP_ZHI if z1 < lab.shape[0] else 0))
        acc = torch.maximum(acc, f)
    np.testing.assert_array_equal(acc.cpu().numpy(), want.cpu().numpy())
    np.testing.assert_array_equal(want.cpu().numpy(), oracle.touches_edge(lab, ml))


# ---- N1: the z pass over whole columns of y-blocks (the all-to-all transpose) -------------

@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_transpose_z_pass_bit_identical(nranks):
    """FASTRS_SLAB_TRANSPOSE's decomposition: K3 on each rank's y-block [Z][Y/P][X] of the
    packed words, then D back to z-slabs: bit-identical to the single call."""
    lab, _ = synth.make_config(2)
    _check(lab, nranks, transpose=True)
    lab = synth.random_labels((70, 45, 50), nlabels=6, seed=11, fill=0.85, blob=5)
    _check(np.pad(lab, 1), 3, 0, transpose=True)


# ---- N4: the kept-centre halo (K4 outputs of the halo tile layers instead of D) -------------

@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_kept_centre_halo_bit_identical(nranks):
    """Each virtual rank runs K4 on its own tile layers (D beyond 3 slices of its slab poisoned)
    and receives the packed K4 outputs of the layers within H slices; K5 from that: bit-identical
    to the single call (fastrs_slab_prune / _pack_tiles / _unpack_tiles / _dilate)."""
    lab, _ = synth.make_config(2)
    _check(lab, nranks, lt_halo="centres")
    lab = synth.random_labels((70, 45, 50), nlabels=6, seed=11, fill=0.85, blob=5)
    _check(np.pad(lab, 1), 3, 0, lt_halo="centres")


def test_kept_centre_halo_multi_hop_and_c3():
    lab = np.zeros((96, 70, 70), np.int32)
    lab[15:76, 4:65, 4:65] = synth.sphere(30, canvas=61)
    lab[80:90, 10:60, 20:30] = 2
    info = _check(lab, 6, lt_halo="centres")  # H = 32 > the 16-slice slabs: several sources per side
    assert info["H"] > 16
    lab, _ = synth.make_config(3)
    _check(lab, 4, lt_halo="centres", transpose=True)


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_split_z_pass_bit_identical(nranks):
    """The NCCL driver overlaps the z-halo exchange with the z pass of the interior slices and runs
    the boundary ranges after it: the three sub-range calls give the one-call result."""
    lab, _ = synth.make_config(2)
    _check(lab, nranks, lt_halo="centres", split_zpass=True)
    lab = synth.random_labels((70, 45, 50), nlabels=6, seed=11, fill=0.85, blob=5)
    _check(np.pad(lab, 1), nranks, 0, split_zpass=True)


# ---- the in-library NCCL driver (fastrs_sphericity_roundness_slab) ----------------------

@pytest.fixture(scope="module")
def comm1():
    """A single-rank libfastrs NCCL communicator on cuda:0 (one GPU on this box)."""
    if not fastrs.nccl_available():
        pytest.fail("libnccl.so.2 not loadable")
    torch.cuda.set_device(0)
    c = fastrs.Comm(fastrs.nccl_unique_id(), 1, 0)
    yield c
    c.close()


@pytest.mark.parametrize("flags", [fastrs.BORDER_BACKGROUND, fastrs.BORDER_BACKGROUND | fastrs.SLAB_TRANSPOSE,
                                   fastrs.BORDER_BACKGROUND | fastrs.SLAB_DENSE_HALO])
@pytest.mark.parametrize("cfg", [2, 3])
def test_nccl_slab_call_bit_identical(comm1, cfg, flags):
    """fastrs_sphericity_roundness_slab on one rank (N8 halo or N1 transpose, NCCL allreduces,
    self copies) gives the single call's results bit for bit."""
    lab, info = synth.make_config(cfg)
    ml = info["max_label"]
    t = torch.from_numpy(lab).cuda()
    want = fastrs.sphericity_roundness(t, max_label=ml, stats=True)
    got = fastrs.sphericity_roundness_slab(t, 0, lab.shape[0], ml, comm1, flags=flags, stats=True)
    for k in KEYS:
        np.testing.assert_array_equal(got[k].cpu().numpy(), want[k].cpu().numpy(), err_msg=k)
    si = got["slab_info"]
    assert si["mode"] == (1 if flags & fastrs.SLAB_TRANSPOSE else 0)
    assert si["dmax"] == fastrs.diagnostics(fastrs.last_workspace())["dmax"] or si["dmax"] > 0
    assert si["H"] % 8 == 0 and si["bytes_sent"] == 0  # one rank: nothing leaves the GPU


def test_nccl_slab_call_halo_retry_and_errors(comm1):
    """A ball wider than the default halo cap: the wrapper retries with the width the library
    reports; bad labels are reported as on the single call."""
    big = np.zeros((200, 200, 200), np.int32)
    big[10:191, 10:191, 10:191] = synth.sphere(90, canvas=181)
    t = torch.from_numpy(big).cuda()
    want = fastrs.sphericity_roundness(t, max_label=1)
    got = fastrs.sphericity_roundness_slab(t, 0, 200, 1, comm1, halo_cap=16)
    assert got["slab_info"]["halo_cap"] > 16 and got["slab_info"]["H"] > 16
    np.testing.assert_array_equal(got["roundness"].cpu().numpy(), want["roundness"].cpu().numpy())
    bad = torch.from_numpy(np.full((16, 8, 8), 5, np.int32)).cuda()
    with pytest.raises(fastrs.FastrsError) as e:
        fastrs.sphericity_roundness_slab(bad, 0, 16, 2, comm1)
    assert e.value.name == "EINVAL"
