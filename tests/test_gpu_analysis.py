"""GPU parity of the analysis-protocol kernels (csrc/analysis.cu) with the oracle
(oracle/oracle_analysis.cpp): connected components bit-exact (labels and counts), Eq. 3
width/length sphericity and the S_MC perimeter / area / sphericity within 1e-9 relative (exact
integer moments / 2^-32 fixed-point sums on the GPU vs float64 sums in the oracle)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
RT = 1e-9


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2504_05808_b200 import fastrs
    fastrs.load()
    return fastrs


def _dev(a, dt=np.int32):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()


def _close(g, w):
    g = g.cpu().numpy()
    np.testing.assert_array_equal(np.isnan(g), np.isnan(w))
    ok = ~np.isnan(w)
    np.testing.assert_allclose(g[ok], w[ok], rtol=RT, atol=1e-12)


@pytest.mark.parametrize("ndim,conn", [(2, 4), (2, 8), (3, 6), (3, 18), (3, 26)])
def test_ccl_random(F, ndim, conn):
    rng = np.random.default_rng(conn + ndim)
    for _ in range(12):
        shape = tuple(int(v) for v in rng.integers(2, 70 if ndim == 2 else 24, ndim))
        m = rng.random(shape) < rng.uniform(0.2, 0.8)
        want, counts = oracle.label_components(m, conn)
        got, gc = F.label_components(_dev(m, np.uint8), conn)
        np.testing.assert_array_equal(got.cpu().numpy(), want)
        assert gc.cpu().tolist() == counts.tolist()


def test_ccl_batch_and_configs(F):
    rng = np.random.default_rng(9)
    b = rng.random((4, 37, 53)) < 0.55
    want, counts = oracle.label_components(b, 8, ndim=2)
    got, gc = F.label_components(_dev(b, np.uint8), 8, ndim=2)
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    assert gc.cpu().tolist() == counts.tolist()
    for cfg, conn in ((1, 8), (2, 26), (3, 26)):
        lab, _ = synth.make_config(cfg)
        m = lab > 0
        want, counts = oracle.label_components(m, conn)
        got, gc = F.label_components(_dev(m, np.uint8), conn)
        np.testing.assert_array_equal(got.cpu().numpy(), want)
        assert int(gc[0]) == int(counts[0])


def test_wl_parity(F):
    for lab, ml, nd in ((synth.make_config(1)[0], 21, 2), (synth.make_config(5, batch=3)[0], 500, 2),
                        (synth.random_labels((2, 33, 47), nlabels=5, seed=2, fill=0.8, blob=3), 5, 2)):
        want = oracle.sphericity_wl(lab, ml, batch=lab.shape[0] if lab.ndim == 3 else None)
        got = F.sphericity_wl(_dev(lab), ml)
        for k in ("swl", "d1", "d2"):
            _close(got[k], want[k])
    with pytest.raises(F.FastrsError):
        F.mc_measure(_dev(np.ones((4, 4))), 0)


@pytest.mark.parametrize("cfg", [1, 2, 3, 5])
def test_mc_parity(F, cfg):
    lab, info = synth.make_config(cfg, batch=2) if cfg == 5 else synth.make_config(cfg)
    ml = info["max_label"]
    nd = 2 if cfg in (1, 5) else 3
    want = oracle.mc_measure(lab, ml, ndim=nd)
    got = F.mc_measure(_dev(lab), ml, ndim=nd)
    _close(got["measure"], want["measure"])
    _close(got["sphericity_mc"], want["sphericity_mc"])


def test_mc_touching_labels_and_border(F):
    for shape in ((9, 13, 37), (21, 70), (1, 5, 6), (3, 1, 1)):
        lab = synth.random_labels(shape, nlabels=5, seed=4, fill=0.9, blob=3)
        nd = len(shape)
        want = oracle.mc_measure(lab, 5, ndim=nd)
        got = F.mc_measure(_dev(lab), 5, ndim=nd)
        _close(got["measure"], want["measure"])
        _close(got["sphericity_mc"], want["sphericity_mc"])
