"""Z-slab multi-GPU path, host side (-m "not gpu"): the halo-width and exchange-plan logic of
paper_2504_05808_b200/slab.py, and its real torch.distributed exchange code run over gloo with
world_size 2, 3 and 5 on the CPU, the phases replaced by the numpy stand-in of tests/_slab_numpy.py.
The assembled per-label results must equal the CPU oracle on the whole volume (integers exactly,
floats to 1e-9): a halo that is one slice too small changes them (test_halo_too_small_is_caught).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2504_05808_b200 import slab
from tests._slab_numpy import NumpyPhases


def test_partition_alignment():
    assert slab.partition(128, 4) == [(0, 32), (32, 64), (64, 96), (96, 128)]
    for Z, n in ((100, 3), (1024, 8), (24, 3), (41, 2)):
        s = slab.partition(Z, n)
        assert s[0][0] == 0 and s[-1][1] == Z and len(s) == n
        assert all(a < b for a, b in s) and all(s[i][1] == s[i + 1][0] for i in range(n - 1))
        assert all(b % 8 == 0 for _, b in s[:-1])
    with pytest.raises(ValueError):
        slab.partition(16, 4)


def test_halo_widths():
    assert slab.halo_edt(0, 64) == 0
    assert slab.halo_edt(1, 64) == 1
    for d in (2, 4, 5, 100, 101, 1515):
        h = slab.halo_edt(d, 10 ** 6)
        assert h * h >= d > (h - 1) ** 2
    assert slab.halo_edt(slab.INF, 77) == 77
    for d, r in ((1, 0), (2, 1), (226, 15), (1515, 38)):
        H = slab.halo_lt(d)
        assert H % 8 == 0 and H >= r and H - r < 8


def test_halo_plan_multi_hop():
    slabs = slab.partition(40, 5)  # 8 slices each
    plan = slab.halo_plan(slabs, 11, 40)
    # rank 2 ([16,24)) needs [5,16) from ranks 0 and 1, and [24,35) from ranks 3 and 4
    got = sorted((s, a, b) for s, d, side, a, b in plan if d == 2)
    assert got == [(0, 5, 8), (1, 8, 16), (3, 24, 32), (4, 32, 35)]
    # every rank receives exactly its clamped halo
    for d, (z0, z1) in enumerate(slabs):
        lo = sum(b - a for s, dd, side, a, b in plan if dd == d and side == "lo")
        hi = sum(b - a for s, dd, side, a, b in plan if dd == d and side == "hi")
        assert lo == z0 - max(0, z0 - 11) and hi == min(40, z1 + 11) - z1


def _volume(seed: int) -> np.ndarray:
    """Objects crossing slab boundaries: a digital sphere, a prolate spheroid along z and two
    touching random-blob labels."""
    lab = np.zeros((40, 22, 20), np.int32)
    s = synth.sphere(7)  # 19^3, radius 7
    lab[4:23, 0:19, 0:19][s > 0] = 1
    sp = synth.spheroid(8.5, 14.0)  # a wide prolate grain: D_xy > 64, so h > 8 slices
    zz, yy, xx = np.nonzero(sp)
    zz = zz + 8
    ok = (zz < 40) & (yy < 22) & (xx < 20)
    lab[zz[ok], yy[ok], xx[ok]] = 2
    blobs = synth.random_labels((12, 22, 20), nlabels=2, seed=seed, fill=0.7, blob=3)
    region = lab[27:39]
    region[(region == 0) & (blobs > 0)] = blobs[(region == 0) & (blobs > 0)] + 2
    return lab


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, lab, max_label, flags, shrink, out_dir):
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    try:
        slabs = slab.partition(lab.shape[0], world)
        z0, z1 = slabs[rank]
        phases = NumpyPhases()
        if shrink == "edt":  # deliberately too-small halos: the tests must notice
            slab.halo_edt = lambda d, Z: min(1, d)
        elif shrink == "lt":
            slab.halo_lt = lambda d, align=8: 0
        res = slab.sphericity_roundness_slab(torch.from_numpy(lab[z0:z1].copy()), slabs, max_label, flags,
                                             phases=phases, stats=True)
        if rank == 0:
            np.savez(os.path.join(out_dir, "res.npz"), **{k: v.numpy() for k, v in res.items() if k != "slab_info"},
                     h=res["slab_info"]["h"], H=res["slab_info"]["H"])
    finally:
        dist.destroy_process_group()


def _edge_worker(rank, world, port, lab, max_label, out_dir):
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    try:
        slabs = slab.partition(lab.shape[0], world)
        z0, z1 = slabs[rank]
        f = slab.touches_edge_slab(torch.from_numpy(lab[z0:z1].copy()), slabs, max_label, phases=NumpyPhases())
        if rank == 0:
            np.save(os.path.join(out_dir, "edge.npy"), f.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_touches_edge_slab_gloo_matches_oracle(world, tmp_path):
    """Edge-object flags from z-slabs (inner slab faces skipped, allreduce max) equal the oracle's
    flags on the whole volume; labels that touch only an inner slab face stay unflagged."""
    lab = _volume(seed=world)
    lab[15, 10, 10] = 9  # interior voxel on the slab boundary region
    ml = int(lab.max())
    mp.start_processes(_edge_worker, args=(world, _free_port(), lab, ml, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(os.path.join(tmp_path, "edge.npy"))
    np.testing.assert_array_equal(got, oracle.touches_edge(lab, ml))
    assert got[8] == 0


def _run(world, lab, max_label, flags, tmp_path, shrink=False):
    mp.start_processes(_worker, args=(world, _free_port(), lab, max_label, flags, shrink, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    return dict(np.load(os.path.join(tmp_path, "res.npz")))


@pytest.mark.parametrize("world,flags", [(2, 1), (5, 1), (3, 0)])
def test_slab_path_gloo_matches_oracle(world, flags, tmp_path):
    lab = _volume(seed=world)
    if flags == 0:  # without the border flag every object needs a site inside the grid
        lab = np.pad(lab, ((0, 0), (1, 1), (1, 1)))
    ml = int(lab.max())
    got = _run(world, lab, ml, flags, tmp_path)
    want = oracle.sphericity_roundness(lab, max_label=ml, flags=flags)
    np.testing.assert_array_equal(got["volume"], want["volume"])
    np.testing.assert_array_equal(got["n_shell"], want["n_shell"])
    np.testing.assert_array_equal(got["max_lt2"].astype(np.uint32), want["max_lt2"])
    ok = want["volume"] > 0
    np.testing.assert_allclose(got["sphericity"][ok], want["sphericity"][ok], rtol=1e-9)
    np.testing.assert_allclose(got["roundness"][ok], want["roundness"][ok], rtol=1e-9)
    assert got["h"] >= 1 and got["H"] % 8 == 0
    if world == 5:
        assert got["h"] > 8  # the z halo spans more than one neighbouring slab (multi-hop)


@pytest.mark.parametrize("shrink", ["edt", "lt"])
def test_halo_too_small_is_caught(shrink, tmp_path):
    """Plausible mistakes -- a one-slice z halo for the EDT, or no D halo for the dilation --
    change the assembled result, so the exact match above is a real check of the widths."""
    lab = _volume(seed=5)
    ml = int(lab.max())
    got = _run(2, lab, ml, 1, tmp_path, shrink=shrink)
    want = oracle.sphericity_roundness(lab, max_label=ml)
    ok = want["volume"] > 0
    same = np.allclose(got["sphericity"][ok], want["sphericity"][ok], rtol=1e-9) and \
        np.array_equal(got["max_lt2"].astype(np.uint32), want["max_lt2"])
    assert not same


# ---- the library's own plans (libfastrs host code used by fastrs_sphericity_roundness_slab) ----

def test_library_partition_and_halo_plan_match_python():
    """fastrs_slab_partition / fastrs_slab_halo_plan (the C++ NCCL driver's plans) equal slab.py's
    partition / halo_plan, including multi-hop halos wider than a slab."""
    from paper_2504_05808_b200 import fastrs as F
    rng = np.random.default_rng(5)
    for _ in range(200):
        P = int(rng.integers(1, 9))
        Z = int(rng.integers(8 * P, 2048))
        try:
            want = slab.partition(Z, P)
        except ValueError:
            continue
        assert F.slab_partition(Z, P) == want
        for w in (0, 1, int(rng.integers(1, 64)), int(rng.integers(1, Z + 1)), Z):
            assert F.slab_halo_plan(want, w, Z) == slab.halo_plan(want, w, Z)
