"""Blocker-search penumbra plane (configs 3/4 extension) vs oracle/blocker.py.

Parity is against our own CPU restatement (the reference has no blocker
search); the penumbra formula itself is pinned to the reference in
test_oracle_golden.py."""

import numpy as np
import pytest

from conftest import golden_camera, golden_view, load_golden

pytestmark = pytest.mark.gpu


def _frame(size_index):
    from paper_2301_05262_b200 import scenes
    spec = scenes.random_scene(12, seed=3, emitter_radius_m=size_index * 0.0625)
    return scenes.make_frame(spec, (120, 200), (512, 512))


@pytest.mark.parametrize("size_index", [0.0, 2.0, 8.0])
def test_blocker_plane_matches_oracle(size_index):
    from oracle import blocker as ob
    from oracle import features as of
    from paper_2301_05262_b200 import producer
    from paper_2301_05262_b200.raster import blocker_penumbra_batch
    fr = _frame(size_index)
    inp = producer.render_inputs([fr])
    plane = blocker_penumbra_batch(inp, [(fr.camera, fr.view, fr.scene.emitter_center, fr.size_index,
                                          fr.bias)])[0].cpu().numpy()
    h = {k: v[0].cpu().numpy() for k, v in inp.items()}
    z_f, _, _, cov = of.derive_planes(h["d"], h["normal"], h["position"], fr.camera, fr.scene.emitter_center)
    ref = ob.blocker_plane(h["d"], h["position"], z_f, cov, h["sm"], fr.view, fr.bias, fr.size_index,
                           fr.camera.focal_px)
    assert np.max(np.abs(plane - ref)) <= 1e-4 * max(1.0, float(np.abs(ref).max()))
    if size_index == 0.0:
        assert np.all(plane == 0)
    else:
        assert (plane > 0).mean() > 0.02


def test_five_channel_forward_with_blocker_plane():
    """features + blocker plane -> NetworkConfig(in_channels=5) forward
    (fp32 plan) vs the oracle forward on the same 5 planes."""
    import torch
    from oracle import network as on
    from paper_2301_05262_b200 import network, producer
    from paper_2301_05262_b200.raster import assemble_features_batch, blocker_penumbra_batch
    fr = _frame(3.0)
    inp = producer.render_inputs([fr])
    ft = (fr.camera, fr.view, fr.scene.emitter_center, fr.size_index, fr.bias)
    feats, _, _ = assemble_features_batch(inp, [ft])
    bp = blocker_penumbra_batch(inp, [ft])
    x = torch.cat([feats, bp[:, None]], dim=1)[:, :, :112, :192].contiguous()
    cfg = network.NetworkConfig(in_channels=5)
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([4, 0x11])))
    y = network.Plan(w, cfg, "fp32").forward(x)[0].cpu().numpy()
    ref = on.forward({k: v.data for k, v in w.items()}, x[0].cpu().numpy())
    assert np.max(np.abs(y - ref)) <= 1e-4


def test_blocker_frustum_error():
    from types import SimpleNamespace
    from paper_2301_05262_b200._lib import FrustumError
    from paper_2301_05262_b200.raster import blocker_penumbra_batch
    import torch
    r = load_golden("cfg1")
    v = golden_view(r)
    narrow = SimpleNamespace(**{**v.__dict__, "tan_half": v.tan_half / 20})
    inp = {k: torch.from_numpy(np.ascontiguousarray(r[k][None])).cuda() for k in ("d", "normal", "position")}
    inp["sm"] = torch.from_numpy(r["sm"][None]).cuda()
    with pytest.raises(FrustumError):
        blocker_penumbra_batch(inp, [(golden_camera(r), narrow, r["emitter_center"], 2.0, float(r["bias"]))])
