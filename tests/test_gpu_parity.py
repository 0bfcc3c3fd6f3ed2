"""CUDA path vs the oracle and the reference's golden outputs (needs a B200).

Bars (BASELINE.json north_star): texel indices bit-exact; fp32 mode
visibility <= 1e-4 max-abs; features <= 2e-6 abs (fp32 rounding of fp64 math).
"""

import numpy as np
import pytest

from conftest import golden_camera, golden_nets, golden_view, load_golden

pytestmark = pytest.mark.gpu

FEAT_TOL = 2e-6
F32_TOL = 1e-4


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _golden_inputs(r):
    return {"d": _dev(r["d"][None]), "normal": _dev(r["normal"][None]),
            "position": _dev(r["position"][None]), "sm": _dev(r["sm"][None])}


def _golden_frame(r):
    return (golden_camera(r), golden_view(r), r["emitter_center"], float(r["size_index"]),
            float(r["bias"]))


@pytest.mark.parametrize("name", ["cfg1", "variants", "canon"])
def test_features_kernel_matches_reference(name):
    from paper_2301_05262_b200.raster import assemble_features_batch
    r = load_golden(name)
    feats, idx, _ = assemble_features_batch(_golden_inputs(r), [_golden_frame(r)], want_idx=True)
    idx = idx[0].cpu().numpy()
    mism = int(np.sum(idx != r["texel_idx"]))
    assert mism == 0, f"{mism} texel indices differ"
    f = feats[0].cpu().numpy()
    assert np.max(np.abs(f - r["features"])) <= FEAT_TOL
    cov = r["d"] > 0
    assert np.all(f[:, ~cov] == 0.0)


def test_assemble_features_dropin_with_reference_style_gbuffer(cfg1):
    """The numpy-signature drop-in, fed a GBuffer that carries its own
    z_f / c_e / c_c (as the reference's render_gbuffer returns it)."""
    from oracle import features as of
    from paper_2301_05262_b200 import raster
    r = cfg1
    cam, view = golden_camera(r), golden_view(r)
    z_f, c_e, c_c, cov = of.derive_planes(r["d"], r["normal"], r["position"], cam,
                                          r["emitter_center"])
    g = raster.GBuffer(d=r["d"].astype(np.float64), normal=r["normal"].astype(np.float64),
                       position=r["position"].astype(np.float64), n_e=None, z_f=z_f, c_e=c_e,
                       c_c=c_c, coverage=cov, camera=cam)
    sm = raster.ShadowMap(depth=r["sm"], view=view, scene_diag=float(r["bias"]) / 1e-3)
    fs = raster.assemble_features(g, sm, 0.0)
    assert fs.bias == pytest.approx(float(r["bias"]))
    assert np.max(np.abs(fs.data - r["features"])) <= FEAT_TOL
    np.testing.assert_array_equal(raster.texel_indices(g, sm), r["texel_idx"])
    # with_size_index / hard_shadow_mask behave like raster.py:190-195, 281-283
    fs3 = fs.with_size_index(3.0)
    np.testing.assert_allclose(fs3.data[2][cov] - fs.data[2][cov], 3.0, atol=1e-6)
    assert raster.hard_shadow_mask(fs).sum() == int((r["features"][0] < 0).sum())


def test_frustum_error_reports_first_pixel(cfg1):
    from types import SimpleNamespace
    from oracle import features as of
    from paper_2301_05262_b200._lib import FrustumError
    from paper_2301_05262_b200.raster import assemble_features_batch
    r = cfg1
    view = golden_view(r)
    narrow = SimpleNamespace(**{**view.__dict__, "tan_half": view.tan_half / 20})
    cov = r["d"] > 0
    _, _, first = of.texel_indices(narrow, r["position"], cov)
    y, x = divmod(first, cov.shape[1])
    fr = list(_golden_frame(r))
    fr[1] = narrow
    with pytest.raises(FrustumError, match=rf"\({y}, {x}\)"):
        assemble_features_batch(_golden_inputs(r), [tuple(fr)])


@pytest.mark.parametrize("name", sorted(golden_nets()))
def test_forward_fp32_matches_reference(name):
    from paper_2301_05262_b200 import network
    c = golden_nets()[name]
    layers, base, inc, s2d, cap = (int(v) for v in c["cfg"])
    cfg = network.NetworkConfig(layers, base, inc, bool(s2d), cap)
    y = network.forward(c["w"], cfg, c["x"]).data
    assert y.shape == c["y"].shape
    assert np.max(np.abs(y - c["y"])) <= F32_TOL


def test_forward_shape_errors():
    from paper_2301_05262_b200 import network
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(0))
    with pytest.raises(ValueError, match="divisible by 16"):
        network.forward(w, cfg, np.zeros((4, 1080, 1920), np.float32))
    with pytest.raises(ValueError, match="config wants 4"):
        network.forward(w, cfg, np.zeros((5, 32, 32), np.float32))
    z = {k: np.zeros_like(v.data) for k, v in w.items()}
    np.testing.assert_array_equal(network.forward(z, cfg, np.ones((4, 32, 48), np.float32)).data,
                                  0.5)


def test_cfg1_end_to_end_fp32(cfg1):
    """Fused nsm_infer on config 1 vs the reference visibility."""
    from paper_2301_05262_b200 import network
    from paper_2301_05262_b200.infer import ShadowInference
    from types import SimpleNamespace
    r = cfg1
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    plan = network.Plan(w, cfg, "fp32")
    cam, view = golden_camera(r), golden_view(r)
    fr = SimpleNamespace(camera=cam, view=view, size_index=0.0, bias=float(r["bias"]),
                         scene=SimpleNamespace(emitter_center=r["emitter_center"]))
    run = ShadowInference(plan, [fr])
    y = run(_golden_inputs(r))[0].cpu().numpy()
    assert np.max(np.abs(y - r["visibility"])) <= F32_TOL


def test_producer_matches_reference_buffers(cfg1):
    from paper_2301_05262_b200 import producer, scenes
    fr = scenes.config_frames(1, seed=0)[0]
    inp = producer.render_inputs([fr])
    d = inp["d"][0].cpu().numpy()
    cov, gcov = d > 0, cfg1["d"] > 0
    assert np.mean(cov != gcov) < 1e-3
    both = cov & gcov
    np.testing.assert_allclose(d[both], cfg1["d"][both], rtol=1e-6)
    p = inp["position"][0].cpu().numpy()
    np.testing.assert_allclose(p[:, both], cfg1["position"][:, both], rtol=1e-5, atol=1e-6)
    n = inp["normal"][0].cpu().numpy()
    assert np.mean(np.abs(n[:, both] - cfg1["normal"][:, both]) > 1e-5) < 1e-3
    sm = inp["sm"][0].cpu().numpy()
    assert np.mean(np.isfinite(sm) != np.isfinite(cfg1["sm"])) < 1e-3
    fin = np.isfinite(sm) & np.isfinite(cfg1["sm"])
    np.testing.assert_allclose(sm[fin], cfg1["sm"][fin], rtol=1e-6)


def test_config2_1080p_fp32_vs_oracle():
    """1920x1080 (padded to 1088 for the net) through nsm_infer
    vs the numpy oracle on the identical downloaded inputs."""
    from oracle import features as of
    from oracle import network as on
    from paper_2301_05262_b200 import network, producer, scenes
    from paper_2301_05262_b200.infer import ShadowInference
    fr = scenes.config_frames(2, seed=0)[0]
    inp = producer.render_inputs([fr])
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    run = ShadowInference(network.Plan(w, cfg, "fp32"), [fr])
    y = run(inp)[0, 0].cpu().numpy()
    h = {k: v[0].cpu().numpy() for k, v in inp.items()}
    feats, cov = of.features_from_planes(h["d"], h["normal"], h["position"], h["sm"], fr.camera,
                                         fr.view, fr.scene.emitter_center, fr.size_index, fr.bias)
    xp = np.zeros((4, 1088, 1920), np.float32)
    xp[:, :1080] = feats
    ref = on.forward({k: v.data for k, v in w.items()}, xp)[0, :1080]
    assert np.max(np.abs(y - ref)) <= F32_TOL
