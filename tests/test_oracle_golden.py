"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The fixtures in tests/golden/ were produced by running the real reference
(``shadowkit``) -- see tests/golden/make_golden.py. Nothing here needs a GPU.
"""

import math

import numpy as np
import pytest

from conftest import golden_camera, golden_nets, golden_view, load_golden
from oracle import features as of
from oracle import network as on
from oracle import producer as op
from paper_2301_05262_b200 import scenes


@pytest.mark.parametrize("name", ["cfg1", "variants", "canon"])
def test_oracle_features_match_reference(name):
    r = load_golden(name)
    cam, view = golden_camera(r), golden_view(r)
    feats, cov = of.features_from_planes(r["d"], r["normal"], r["position"], r["sm"], cam, view,
                                         r["emitter_center"], float(r["size_index"]),
                                         float(r["bias"]))
    np.testing.assert_array_equal(feats, r["features"])
    ri, ci, first = of.texel_indices(view, r["position"], cov)
    assert first == -1
    idx = np.stack([ri, ci]).astype(np.int32)
    idx[:, ~cov] = -1
    np.testing.assert_array_equal(idx, r["texel_idx"])


def test_oracle_canon_fp32_inputs_close_to_fp64_reference():
    # the fp32 input format moves features by <= fp32 rounding of the planes
    r = load_golden("canon")
    assert np.max(np.abs(r["features"] - r["features_fp64_inputs"])) < 2e-5


def test_oracle_frustum_error_first_pixel():
    r = load_golden("cfg1")
    view = golden_view(r)
    view.tan_half /= 20.0                        # test_raster.py:186-200 analogue
    cov = r["d"] > 0
    z_f, c_e, c_c, cov = of.derive_planes(r["d"], r["normal"], r["position"], golden_camera(r),
                                          r["emitter_center"])
    with pytest.raises(of.FrustumError) as ei:
        of.assemble(r["d"], r["position"], z_f, c_e, c_c, cov, r["sm"], view, 0.0, 0.01)
    _, _, first = of.texel_indices(view, r["position"], cov)
    y, x = divmod(first, cov.shape[1])
    assert f"({y}, {x})" in str(ei.value)


def _weights_for(cfg_tuple, seed_words):
    from paper_2301_05262_b200.network import NetworkConfig, init_weights
    cfg = NetworkConfig(*[int(v) for v in cfg_tuple[:3]], bool(cfg_tuple[3]), int(cfg_tuple[4]))
    return cfg, init_weights(cfg, np.random.default_rng(np.random.SeedSequence(seed_words)))


def test_init_weights_bitwise_equal_reference(cfg1):
    import hashlib
    cfg, w = _weights_for((5, 16, 4, 1, 256), [0, 0x11])
    h = hashlib.sha256()
    for k in sorted(w):
        h.update(k.encode())
        h.update(np.ascontiguousarray(w[k].data, dtype="<f4").tobytes())
    assert h.hexdigest() == cfg1["weights_sha256"].item().decode()


def test_oracle_forward_cfg1_matches_reference(cfg1):
    _, w = _weights_for((5, 16, 4, 1, 256), [0, 0x11])
    y = on.forward({k: v.data for k, v in w.items()}, cfg1["features"])
    assert y.shape == (1, 256, 256)
    assert np.max(np.abs(y - cfg1["visibility"])) < 1e-6


@pytest.mark.parametrize("name", sorted(golden_nets()))
def test_oracle_forward_net_cases(name):
    c = golden_nets()[name]
    layers, base, inc, s2d, cap = (int(v) for v in c["cfg"])
    y = on.forward(c["w"], c["x"], layers=layers, base_channels=base, use_s2d=bool(s2d), cap=cap)
    assert y.shape == c["y"].shape
    assert np.max(np.abs(y - c["y"])) < 1e-6


def test_oracle_forward_fp64_close_to_fp32():
    c = golden_nets()["l5_default"]
    y64 = on.forward({k: v.astype(np.float64) for k, v in c["w"].items()},
                     c["x"].astype(np.float64))
    assert np.max(np.abs(y64 - c["y"])) < 1e-5


def test_oracle_producer_matches_reference_buffers(cfg1):
    fr = scenes.config_frames(1, seed=0)[0]
    tab = fr.scene.primitive_table()
    d, n, p = op.render_gbuffer(tab, fr.camera)
    sm = op.render_shadowmap(tab, fr.view)
    cov = d > 0
    assert np.mean(cov != (cfg1["d"] > 0)) < 1e-3
    both = cov & (cfg1["d"] > 0)
    np.testing.assert_allclose(d.astype(np.float32)[both], cfg1["d"][both], rtol=1e-6)
    np.testing.assert_allclose(p.astype(np.float32)[:, both], cfg1["position"][:, both],
                               rtol=1e-5, atol=1e-6)
    assert np.mean(np.isfinite(sm) != np.isfinite(cfg1["sm"])) < 1e-3
    fin = np.isfinite(sm) & np.isfinite(cfg1["sm"])
    np.testing.assert_allclose(sm.astype(np.float32)[fin], cfg1["sm"][fin], rtol=1e-6)


# --- SPEC known-answer tests, run on the oracle operators ---------------------

def test_spec_kats_ops():
    a, b, c, d = 1.0, 2.0, 3.0, 4.0
    x = np.array([[[a, b], [c, d]]], dtype=np.float32)
    np.testing.assert_array_equal(on.s2d(x)[:, 0, 0], [a, b, c, d])
    np.testing.assert_array_equal(on.d2s(on.s2d(x)), x)
    assert on.pool2(np.array([[[0, 1], [2, 3]]], np.float32))[0, 0, 0] == 1.5
    k = np.ones((1, 1, 3, 3), np.float32)
    y = on.conv(np.full((1, 5, 5), 2.0, np.float32), k, np.zeros(1, np.float32))
    assert y[0, 2, 2] == 18.0
    np.testing.assert_array_equal(on.up2(np.full((2, 3, 4), 0.7, np.float32)),
                                  np.full((2, 6, 8), 0.7, np.float32))


def test_spec_zero_weights_give_half():
    _, w = _weights_for((5, 16, 4, 1, 256), [1, 0x11])
    z = {k: np.zeros_like(v.data) for k, v in w.items()}
    y = on.forward(z, np.random.default_rng(0).normal(size=(4, 32, 32)).astype(np.float32))
    np.testing.assert_array_equal(y, 0.5)


def test_penumbra_formula_pinned_to_reference():
    """oracle.blocker.penumbra_widths reuses analysis.penumbra_extents
    (analysis.py:240-269): pinned on 4000 reference evaluations."""
    from oracle import blocker as ob
    g = load_golden("penumbra")
    w = ob.penumbra_widths(g["z_min"], g["z_max"], g["z_f"], g["r_e"], 1.0, 1.0)
    ref = g["x_a"] + g["x_b"]
    ref = np.where(g["r_e"] > 0, ref, 0.0)             # point lights: exact zero width
    np.testing.assert_allclose(w, ref, rtol=1e-12, atol=1e-12)


def test_blocker_plane_point_light_is_zero():
    from oracle import blocker as ob
    r = load_golden("cfg1")
    cov = r["d"] > 0
    z_f, _, _, cov = of.derive_planes(r["d"], r["normal"], r["position"], golden_camera(r),
                                      r["emitter_center"])
    p = ob.blocker_plane(r["d"], r["position"], z_f, cov, r["sm"], golden_view(r), float(r["bias"]),
                         0.0, golden_camera(r).focal_px)
    assert np.all(p == 0)
    p2 = ob.blocker_plane(r["d"], r["position"], z_f, cov, r["sm"], golden_view(r), float(r["bias"]),
                          4.0, golden_camera(r).focal_px)
    assert np.all(p2[~cov] == 0) and np.all(p2 >= 0) and (p2 > 0).mean() > 0.05


def test_oracle_temporal_matches_reference():
    """oracle.temporal vs reference motion_vectors / temporal_instability
    (raster.py:330-358, analysis.py:350-377) on the golden sequence."""
    from oracle import temporal as ot
    g = load_golden("temporal")
    t = int(g["t_frames"])
    vs, oks = [], []
    for k in range(1, t):
        v, ok = ot.motion_vectors(g[f"position{k}"], g[f"normal{k}"], g[f"d{k}"] > 0, g[f"d{k - 1}"],
                                  g[f"normal{k - 1}"], g[f"d{k - 1}"] > 0, golden_camera(g, f"cam{k - 1}"))
        assert np.max(np.abs(v - g[f"vec{k - 1}"])) < 1e-12
        np.testing.assert_array_equal(ok, g[f"valid{k - 1}"])
        vs.append(v)
        oks.append(ok)
    E, n, rej = ot.temporal_instability(list(g["frames"]), vs, oks, 3.0)
    assert n == int(g["valid_pixels"]) and rej == float(g["rejected"])
    assert abs(E - float(g["E"])) <= 1e-13 * abs(float(g["E"]))
    # static pair: identity vectors, valid == coverage (test_raster.py:219-223)
    v, ok = ot.motion_vectors(g["position0"], g["normal0"], g["d0"] > 0, g["d0"], g["normal0"],
                              g["d0"] > 0, golden_camera(g, "cam0"))
    np.testing.assert_array_equal(ok, g["static_valid"])
    assert np.max(np.abs(v - g["static_vec"])) < 1e-12


def test_sensitivity_host_logic_with_oracle_phi():
    """analysis.sensitivity_report / heldout_mse host logic (rng order,
    normalisation) with the oracle forward as phi reproduces the reference's
    report (analysis.py:100-139, training.py:179-189)."""
    from paper_2301_05262_b200 import analysis
    from paper_2301_05262_b200.raster import FEATURE_CHANNELS
    g = load_golden("sensitivity")
    _, w = _weights_for((5, 16, 4, 1, 256), [0, 0x11])
    wd = {k: v.data for k, v in w.items()}

    def phi(s):
        return on.forward(wd, s)[0]

    stacks = list(g["stacks"])
    rep = analysis.sensitivity_report(phi, stacks, FEATURE_CHANNELS, repeats=2,
                                      rng=np.random.default_rng(7))
    np.testing.assert_allclose(rep.absolute, g["absolute"], rtol=1e-5)
    np.testing.assert_allclose(rep.relative, g["relative"], rtol=1e-5)
    m = analysis.heldout_mse(phi, stacks, list(g["targets"]))
    assert abs(m - float(g["heldout_mse"])) <= 1e-6 * float(g["heldout_mse"])
    with pytest.raises(analysis.ZeroVarianceChannel):
        analysis.channel_sensitivity(phi, [np.zeros((4, 16, 16), np.float32)], 0)
    assert math.isnan(analysis.heldout_mse(phi, [], []))
