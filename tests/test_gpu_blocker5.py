"""The 5-plane hot path (BASELINE configs 3/4: soft shadows with the 16x16
blocker search) vs the oracle (needs a B200).

* nsm_features5 (SMEM-staged blocker search fused with the feature pass)
  vs oracle.features (planes 0-3) and oracle.blocker (plane 4; our CPU
  restatement -- the reference has no blocker search, its penumbra formula
  is pinned in test_oracle_golden.py), including the exact blocker / no
  blocker classification of every pixel;
* the fused 16-bit nsm_infer of a NetworkConfig(in_channels=5) plan vs the
  oracle forward on the oracle's 5 planes, fp16 bars (1e-2 max-abs, 1e-4
  MSE) at 1080p (config 3 frame);
* its texel indices bit-exact vs np.rint (raster.py:247-250);
* nsm_forward of a 5-plane 16-bit plan on given planes.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MAX_ABS = 1e-2
MAX_MSE = 1e-4


def _weights5(seed=0):
    from paper_2301_05262_b200 import network
    cfg = network.NetworkConfig(in_channels=5)
    return cfg, network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([seed, 0x11])))


def _oracle5(fr, inp):
    from oracle import blocker as ob
    from oracle import features as of
    h = {k: v[0].cpu().numpy() for k, v in inp.items()}
    feats, cov = of.features_from_planes(h["d"], h["normal"], h["position"], h["sm"], fr.camera, fr.view,
                                         fr.scene.emitter_center, fr.size_index, fr.bias)
    z_f, _, _, _ = of.derive_planes(h["d"], h["normal"], h["position"], fr.camera, fr.scene.emitter_center)
    bp = ob.blocker_plane(h["d"], h["position"], z_f, cov, h["sm"], fr.view, fr.bias, fr.size_index,
                          fr.camera.focal_px)
    return np.concatenate([feats, bp[None]]), cov, h


def _check_planes(got, ref, cov, what):
    d = np.abs(got[:4] - ref[:4])
    assert d.max() <= 1e-4 * max(1.0, float(np.abs(ref[:4]).max())), f"{what}: planes 0-3 off by {d.max()}"
    g4, r4 = got[4], ref[4]
    ndiff = int(((g4 > 0) != (r4 > 0)).sum())
    assert ndiff == 0, f"{what}: blocker classification differs at {ndiff} px"
    # relative, floored at 1e-3 focal lengths (~1 pixel at 1080p)
    rel = np.abs(g4 - r4) / np.maximum(1e-3, np.abs(r4))
    assert rel.max() <= 2e-3, f"{what}: penumbra plane rel err {rel.max()}"
    print(f"{what}: planes 0-3 max {d.max():.3g}, plane 4 rel {rel.max():.3g}, "
          f"{int((g4 > 0).sum())} px with blockers of {int(cov.sum())} covered")


@pytest.mark.parametrize("size_index", [0.0, 2.0, 8.0])
def test_features5_match_oracle_small(size_index):
    from paper_2301_05262_b200 import producer, scenes
    from paper_2301_05262_b200.raster import assemble_features5_batch
    fr = scenes.make_frame(scenes.random_scene(12, seed=3, emitter_radius_m=size_index * 0.0625), (120, 200),
                           (512, 512))
    inp = producer.render_inputs([fr])
    got, _, _ = assemble_features5_batch(inp, [(fr.camera, fr.view, fr.scene.emitter_center, fr.size_index,
                                                fr.bias)])
    ref, cov, _ = _oracle5(fr, inp)
    _check_planes(got[0].cpu().numpy(), ref, cov, f"120x200 size {size_index}")


@pytest.mark.parametrize("res,smres,size_index", [((97, 155), (301, 302), 2.0), ((64, 96), (2048, 2048), 8.0),
                                                  ((33, 250), (130, 514), 0.8)])
def test_features5_odd_shapes_and_unaligned_maps(res, smres, size_index):
    """Odd frame widths (scalar G-buffer loads), map rows that are not a
    multiple of 4 texels (scalar staging and window scans), a map 10x denser
    than the screen (most windows outside the staged region: the global
    16-B scan)."""
    from paper_2301_05262_b200 import producer, scenes
    from paper_2301_05262_b200.raster import assemble_features5_batch
    fr = scenes.make_frame(scenes.random_scene(10, seed=7, emitter_radius_m=size_index * 0.0625), res, smres)
    inp = producer.render_inputs([fr])
    got, idx, _ = assemble_features5_batch(inp, [(fr.camera, fr.view, fr.scene.emitter_center, fr.size_index,
                                                  fr.bias)], want_idx=True)
    ref, cov, h = _oracle5(fr, inp)
    _check_planes(got[0].cpu().numpy(), ref, cov, f"{res} map {smres} size {size_index}")
    from oracle import features as of
    ri, ci, _ = of.texel_indices(fr.view, h["position"], cov)
    idx = idx[0].cpu().numpy()
    assert int(((idx[0] != ri) & cov).sum() + ((idx[1] != ci) & cov).sum()) == 0


def test_infer5_unaligned_map_vs_oracle():
    """The fused 16-bit 5-plane path with a 1030 x 1030 map (rows not a
    multiple of 4 texels) on a 1080p config-3 camera."""
    import torch
    from oracle import network as on
    from paper_2301_05262_b200 import network, producer, scenes
    from paper_2301_05262_b200.infer import ShadowInference
    fr0 = scenes.config_frames(3, seed=4)[0]
    fr = scenes.make_frame(fr0.scene, (1080, 1920), (1030, 1030))
    inp = producer.render_inputs([fr])
    cfg, w = _weights5(seed=5)
    run = ShadowInference(network.Plan(w, cfg, "fp16"), [fr], out_dtype="fp16")
    run.launch(inp)
    run.check_frustum()
    y = run.y[0, 0].float().cpu().numpy()
    ref5, cov, h = _oracle5(fr, inp)
    xp = np.zeros((5, 1088, 1920), np.float32)
    xp[:, :1080] = ref5
    ref = on.forward({k: v.data for k, v in w.items()}, xp)[0, :1080]
    d = y.astype(np.float64) - ref
    mx, mse = float(np.abs(d).max()), float(np.mean(d * d))
    print(f"1030^2 map, 5-plane fp16: max {mx:.3g} mse {mse:.3g}")
    assert mx <= MAX_ABS and mse <= MAX_MSE


def test_features5_config3_1080p_and_texels():
    from oracle import features as of
    from paper_2301_05262_b200 import producer, scenes
    from paper_2301_05262_b200.raster import assemble_features5_batch
    fr = scenes.config_frames(3, seed=0)[0]
    inp = producer.render_inputs([fr])
    got, idx, _ = assemble_features5_batch(inp, [(fr.camera, fr.view, fr.scene.emitter_center, fr.size_index,
                                                  fr.bias)], want_idx=True)
    ref, cov, h = _oracle5(fr, inp)
    _check_planes(got[0].cpu().numpy(), ref, cov, "config 3 1080p")
    ri, ci, _ = of.texel_indices(fr.view, h["position"], cov)
    idx = idx[0].cpu().numpy()
    assert int(((idx[0] != ri) & cov).sum() + ((idx[1] != ci) & cov).sum()) == 0


@pytest.mark.parametrize("config,dtype", [(3, "fp16"), (3, "bf16"), (4, "fp16")])
def test_infer5_vs_oracle(config, dtype):
    """Fused 5-plane inference (feat5 -> enc0_s2d -> levels -> dec0 -> recon)
    vs the oracle forward(in_channels=5) on the oracle's planes."""
    import torch
    from oracle import features as of
    from oracle import network as on
    from paper_2301_05262_b200 import network, producer, scenes
    from paper_2301_05262_b200.infer import ShadowInference
    fr = scenes.config_frames(config, seed=2)[-1]
    inp = producer.render_inputs([fr])
    cfg, w = _weights5()
    run = ShadowInference(network.Plan(w, cfg, dtype), [fr], out_dtype="fp16")
    idx = torch.full((1, 2, 1080, 1920), -1, dtype=torch.int32, device="cuda")
    run.launch(inp, texel_idx=idx)
    run.check_frustum()
    y = run.y[0, 0].float().cpu().numpy()
    ref5, cov, h = _oracle5(fr, inp)
    xp = np.zeros((5, 1088, 1920), np.float32)
    xp[:, :1080] = ref5
    ref = on.forward({k: v.data for k, v in w.items()}, xp)[0, :1080]
    d = y.astype(np.float64) - ref
    mx, mse = float(np.abs(d).max()), float(np.mean(d * d))
    print(f"config {config} {dtype} 5-plane (size_index {fr.size_index:.2f}): max {mx:.3g} mse {mse:.3g}")
    assert mse <= MAX_MSE
    if dtype == "fp16":
        assert mx <= MAX_ABS
    ri, ci, _ = of.texel_indices(fr.view, h["position"], cov)
    idx = idx[0].cpu().numpy()
    assert int(((idx[0] != ri) & cov).sum() + ((idx[1] != ci) & cov).sum()) == 0


def test_forward5_16bit_on_planes():
    """nsm_forward of a 5-plane fp16 plan (pack_s2d24 -> enc0_s2d) vs the
    oracle forward on the same planes, and bitwise batch independence."""
    import torch
    from oracle import network as on
    from paper_2301_05262_b200 import network
    cfg, w = _weights5(seed=3)
    plan = network.Plan(w, cfg, "fp16")
    g = torch.Generator().manual_seed(0)
    x = torch.rand((3, 5, 96, 160), generator=g) * torch.tensor([0.5, 1.0, 4.0, 0.3, 20.0])[None, :, None, None]
    xd = x.cuda()
    yb = plan.forward(xd).cpu().numpy()
    for i in range(3):
        ref = on.forward({k: v.data for k, v in w.items()}, x[i].numpy())
        d = yb[i] - ref
        assert np.abs(d).max() <= MAX_ABS and np.mean(d * d) <= MAX_MSE
        np.testing.assert_array_equal(plan.forward(xd[i:i + 1]).cpu().numpy()[0], yb[i])


def test_fp32_plan_five_planes_infer_unsupported():
    from paper_2301_05262_b200 import network, producer, scenes
    from paper_2301_05262_b200.infer import ShadowInference
    fr = scenes.make_frame(scenes.random_scene(4, seed=1, emitter_radius_m=0.1), (64, 96), (256, 256))
    cfg, w = _weights5()
    run = ShadowInference(network.Plan(w, cfg, "fp32"), [fr])
    with pytest.raises(NotImplementedError):
        run(producer.render_inputs([fr]))


def test_host_pipeline_five_planes():
    """HostPipeline (pinned host buffers, overlapped copies) on a 5-plane
    plan returns bitwise the device-resident executor's visibility, batch
    by batch, each batch with its own scenes."""
    import torch
    from paper_2301_05262_b200 import network, producer, scenes
    from paper_2301_05262_b200.infer import HostPipeline, ShadowInference
    cfg, w = _weights5(seed=2)
    plan = network.Plan(w, cfg, "fp16")
    batches, refs, poses = [], [], []
    for b in range(3):
        frames = [scenes.make_frame(scenes.random_scene(8, seed=70 + 10 * b + s, emitter_radius_m=0.1 + 0.1 * b),
                                    (96, 160), (256, 256), camera_pos=(0.2 * b, 3.0, -6.0 + 0.2 * s))
                  for s in range(2)]
        inp = producer.render_inputs(frames)
        refs.append(ShadowInference(plan, frames, out_dtype="fp16")(inp).cpu().clone())
        batches.append({k: v.cpu().pin_memory() for k, v in inp.items()})
        poses.append(frames)
    run = ShadowInference(plan, poses[0], out_dtype="fp16")
    pipe = HostPipeline(run)
    outs = [torch.empty(run.y.shape, dtype=run.y.dtype, pin_memory=True) for _ in batches]
    for hb, ho, fr in zip(batches, outs, poses):
        pipe.submit(hb, ho, frames=fr)
    pipe.synchronize()
    for ho, ref in zip(outs, refs):
        torch.testing.assert_close(ho, ref, rtol=0, atol=0)


@pytest.mark.parametrize("hw", [(100, 164), (72, 250), (130, 96)])
def test_infer5_odd_shapes_vs_oracle(hw):
    """The fused 5-plane path on frames whose size is not a multiple of 16
    (padded level-0 grid, partial feat5 / enc0_s2d tiles, widths that are
    not a multiple of 4 -> scalar G-buffer loads) vs the oracle forward on
    the oracle's 5 planes, fp16 bars."""
    from oracle import network as on
    from paper_2301_05262_b200 import network, producer, scenes
    from paper_2301_05262_b200.infer import ShadowInference
    h, wd = hw
    fr = scenes.make_frame(scenes.random_scene(12, seed=h + wd, emitter_radius_m=0.3), (h, wd), (512, 512))
    inp = producer.render_inputs([fr])
    cfg, w = _weights5(seed=4)
    y = ShadowInference(network.Plan(w, cfg, "fp16"), [fr], out_dtype="fp32")(inp)[0, 0].cpu().numpy()
    ref5, cov, _ = _oracle5(fr, inp)
    hp, wp = (h + 15) // 16 * 16, (wd + 15) // 16 * 16
    xp = np.zeros((5, hp, wp), np.float32)
    xp[:, :h, :wd] = ref5
    ref = on.forward({k: v.data for k, v in w.items()}, xp)[0, :h, :wd]
    d = y.astype(np.float64) - ref
    mx, mse = float(np.abs(d).max()), float(np.mean(d * d))
    print(f"{hw} 5-plane fp16: max {mx:.3g} mse {mse:.3g}")
    assert mx <= MAX_ABS and mse <= MAX_MSE
