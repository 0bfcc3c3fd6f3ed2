"""Dataset frames straight to the device, and the GPU eval-temporal
pipeline vs the reference's cmd_eval_temporal on the same dataset."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu


def _m():
    from paper_2301_05262_b200 import dataset
    return dataset.load_manifest(os.path.join(GOLDEN, "dataset_small"))


def _plan():
    from paper_2301_05262_b200 import network
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    return network.Plan(w, cfg, "fp32")


def test_device_batches_equal_numpy_loaders():
    from paper_2301_05262_b200 import dataset
    m = _m()
    x, cov = dataset.load_feature_batch(m, [0, 1, 2], k=1, size_index=2.0)
    for i in range(3):
        fs = dataset.load_feature_stack(m, i, 1, 2.0)
        np.testing.assert_array_equal(x[i].cpu().numpy(), fs.data)
        np.testing.assert_array_equal(cov[i].cpu().numpy(), fs.coverage)
    g, cams = dataset.load_gbuffer_batch(m)
    for i in range(3):
        gb = dataset.load_gbuffer(m, i)
        np.testing.assert_array_equal(g["position"][i].cpu().numpy(), gb.position.astype(np.float32))
        np.testing.assert_array_equal(g["coverage"][i].cpu().numpy().astype(bool), gb.coverage)
        assert np.allclose(cams[i].forward, gb.camera.forward)


def test_eval_temporal_matches_reference():
    from paper_2301_05262_b200 import dataset
    ref = load_golden("dataset_small_ref")
    m = _m()
    plan = _plan()
    vis = dataset.sequence_outputs(m, plan, 2.0).cpu().numpy()
    assert np.max(np.abs(vis - ref["vis"])) < 1e-4
    rep = dataset.eval_temporal(m, plan, 2.0, 3.0)
    assert rep.valid_pixels == int(ref["valid_pixels"])
    assert abs(rep.instability - float(ref["E"])) < 1e-4 * float(ref["E"])
