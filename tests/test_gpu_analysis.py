"""Batched multi-forward consumers on the GPU vs the reference goldens."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _phi(dtype="fp32", max_batch=32):
    from paper_2301_05262_b200 import analysis, network
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    return analysis.PlanPhi(w, cfg, dtype, max_batch=max_batch)


@pytest.mark.parametrize("max_batch", [32, 5])
def test_sensitivity_report_plan_matches_reference(max_batch):
    from paper_2301_05262_b200 import analysis
    from paper_2301_05262_b200.raster import FEATURE_CHANNELS
    g = load_golden("sensitivity")
    rep = analysis.sensitivity_report(_phi(max_batch=max_batch), list(g["stacks"]), FEATURE_CHANNELS,
                                      repeats=2, rng=np.random.default_rng(7))
    np.testing.assert_allclose(rep.absolute, g["absolute"], rtol=1e-4)
    np.testing.assert_allclose(rep.relative, g["relative"], rtol=1e-4)


def test_heldout_mse_plan_matches_reference():
    from paper_2301_05262_b200 import analysis
    g = load_golden("sensitivity")
    m = analysis.heldout_mse(_phi(max_batch=2), list(g["stacks"]), list(g["targets"]))
    assert abs(m - float(g["heldout_mse"])) <= 1e-5 * float(g["heldout_mse"])


def test_phi_call_matches_batch_and_mse():
    import torch
    from paper_2301_05262_b200 import analysis
    g = load_golden("sensitivity")
    phi = _phi()
    y1 = phi(g["stacks"][1])
    yb = phi.batch(torch.from_numpy(g["stacks"]).cuda()).cpu().numpy()
    np.testing.assert_array_equal(y1, yb[1])
    t = g["targets"][1]
    assert abs(analysis.mse(y1, t) - float(np.mean((y1.astype(np.float64) - t) ** 2))) < 1e-15
    mask = t > 0.5
    assert abs(analysis.mse(torch.from_numpy(y1).cuda(), t, mask)
               - float(np.mean(((y1.astype(np.float64) - t) ** 2)[mask]))) < 1e-15
    with pytest.raises(ValueError):
        analysis.mse(y1, t[:, :10])
