"""Frames at the edges of the fused path's input space (needs a B200).

* a camera that sees no geometry (every pixel uncovered): the reference's
  features are all zero (raster.py:266-278: uncovered pixels stay 0) and its
  visibility is ``forward`` of a zero stack; our fused 4-plane paths (fp16,
  bf16, fp32) and the 5-plane path must give the same, with no FrustumError
  (only covered pixels are projected, raster.py:251);
* that empty frame between two ordinary ones in one batch: enc0's dynamic
  tile claiming hands out its uncovered tiles like any other, and the
  ordinary frames must come out as they do alone.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MAX_ABS = 1e-2
MAX_MSE = 1e-4
RES, SM_RES = (120, 200), (512, 512)


def _weights(in_channels=4):
    from paper_2301_05262_b200 import network
    cfg = network.NetworkConfig(in_channels=in_channels)
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    # init_weights zeroes the biases, and a zero stack through a bias-free net
    # is sigmoid(0) everywhere in any precision: give them values
    rng = np.random.default_rng(7)
    for k, v in w.items():
        if k.endswith(".b"):
            v.data[...] = rng.uniform(-0.3, 0.3, v.data.shape).astype(v.data.dtype)
    return cfg, w


def _frames():
    from paper_2301_05262_b200 import scenes
    scene = scenes.random_scene(12, seed=4, emitter_radius_m=0.2)
    sky = scenes.make_frame(scene, RES, SM_RES, camera_pos=(0.0, 3.0, -6.0), target=(0.0, 12.0, 0.0))
    ground = scenes.make_frame(scene, RES, SM_RES)
    return sky, ground


def _oracle_zero_vis(w, c):
    from oracle import network as on
    hp, wp = (RES[0] + 15) // 16 * 16, (RES[1] + 15) // 16 * 16
    return on.forward({k: v.data for k, v in w.items()}, np.zeros((c, hp, wp), np.float32))[0, :RES[0], :RES[1]]


def _oracle_vis(fr, inp, i, w):
    from oracle import features as of
    from oracle import network as on
    h = {k: v[i].cpu().numpy() for k, v in inp.items()}
    feats, _ = of.features_from_planes(h["d"], h["normal"], h["position"], h["sm"], fr.camera, fr.view,
                                       fr.scene.emitter_center, fr.size_index, fr.bias)
    hp, wp = (RES[0] + 15) // 16 * 16, (RES[1] + 15) // 16 * 16
    xp = np.zeros((4, hp, wp), np.float32)
    xp[:, :RES[0], :RES[1]] = feats
    return on.forward({k: v.data for k, v in w.items()}, xp)[0, :RES[0], :RES[1]]


def _err(y, ref):
    d = np.asarray(y, np.float64) - np.asarray(ref, np.float64)
    return float(np.abs(d).max()), float(np.mean(d * d))


@pytest.mark.parametrize("dtype,planes", [("fp16", 4), ("bf16", 4), ("fp32", 4), ("fp16", 5)])
def test_frame_with_no_geometry(dtype, planes):
    from paper_2301_05262_b200 import network, producer
    from paper_2301_05262_b200.infer import ShadowInference
    sky, _ = _frames()
    inp = producer.render_inputs([sky])
    assert int((inp["d"] > 0).sum()) == 0, "the sky camera must see nothing"
    cfg, w = _weights(planes)
    run = ShadowInference(network.Plan(w, cfg, dtype), [sky], out_dtype="fp32")
    y = run(inp)[0, 0].cpu().numpy()          # __call__ checks the frustum: nothing to report
    mx, mse = _err(y, _oracle_zero_vis(w, planes))
    print(f"no geometry, {dtype} {planes}-plane: max {mx:.3g} mse {mse:.3g}")
    assert mse <= MAX_MSE
    assert mx <= (1e-4 if dtype == "fp32" else MAX_ABS if dtype == "fp16" else 3e-2)


def test_empty_frame_inside_a_batch():
    import torch
    from paper_2301_05262_b200 import network, producer
    from paper_2301_05262_b200.infer import ShadowInference
    sky, ground = _frames()
    batch = [ground, sky, ground]
    inp = producer.render_inputs(batch)
    cfg, w = _weights()
    plan = network.Plan(w, cfg, "fp16")
    y = ShadowInference(plan, batch, out_dtype="fp32")(inp)[:, 0].cpu().numpy()
    alone = ShadowInference(plan, [ground], out_dtype="fp32")({k: v[:1] for k, v in inp.items()})[0, 0]
    np.testing.assert_array_equal(y[0], alone.cpu().numpy())        # same kernels, same inputs: identical
    np.testing.assert_array_equal(y[2], y[0])
    for i, ref in ((0, _oracle_vis(ground, inp, 0, w)), (1, _oracle_zero_vis(w, 4))):
        mx, mse = _err(y[i], ref)
        assert mx <= MAX_ABS and mse <= MAX_MSE, (i, mx, mse)
    torch.cuda.synchronize()
