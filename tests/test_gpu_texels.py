"""Texel indices of the fused hot path, bit-exact (needs a B200).

The fused level-0 encoder (enc0) projects every covered pixel into the
shadow map with its own folded fp64 affine map (common.cuh texel_fused) and
gathers one texel.  nsm_infer_ex's parity hook returns the (row, col) it
actually gathered; north_star requires them to equal the reference's
``np.rint`` indices of ``_shadow_lookup`` (raster.py:247-250) exactly:
0 mismatches on the reference's golden frames, on 1080p and 4K frames of
the benchmark configs (vs the oracle on the identical downloaded inputs),
and on the non-TMA (LDG) producer variant.  The fused FrustumError reports
the reference's first out-of-frustum pixel (raster.py:251-255).
"""

import numpy as np
import pytest

from conftest import golden_camera, golden_view, load_golden

pytestmark = pytest.mark.gpu


def _weights():
    from paper_2301_05262_b200 import network
    cfg = network.NetworkConfig()
    return cfg, network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))


def _frame_ns(r, view=None):
    from types import SimpleNamespace
    return SimpleNamespace(camera=golden_camera(r), view=view or golden_view(r),
                           size_index=float(r["size_index"]), bias=float(r["bias"]),
                           scene=SimpleNamespace(emitter_center=r["emitter_center"]))


def _inputs(r):
    import torch
    return {k: torch.from_numpy(np.ascontiguousarray(r[k][None])).cuda()
            for k in ("d", "normal", "position", "sm")}


def _fused_texels(plan, frames, inp):
    import torch
    from paper_2301_05262_b200.infer import ShadowInference
    run = ShadowInference(plan, frames, out_dtype="fp16")
    idx = torch.full((run.n, 2, run.h, run.w), -1, dtype=torch.int32, device="cuda")
    run.launch(inp, texel_idx=idx)
    run.check_frustum()
    return idx.cpu().numpy()


def _compare(idx, ri, ci, cov, what):
    got_r, got_c = idx[0], idx[1]
    mism = int(np.sum((got_r != ri) & cov) + np.sum((got_c != ci) & cov))
    assert mism == 0, f"{what}: {mism} texel indices differ from np.rint"
    assert np.all(got_r[~cov] == -1) and np.all(got_c[~cov] == -1), f"{what}: uncovered pixel written"
    return int(cov.sum())


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("name", ["cfg1", "variants", "canon"])
def test_fused_texels_match_reference_goldens(name, dtype):
    from paper_2301_05262_b200 import network
    r = load_golden(name)
    cfg, w = _weights()
    idx = _fused_texels(network.Plan(w, cfg, dtype), [_frame_ns(r)], _inputs(r))[0]
    cov = r["d"] > 0
    n = _compare(idx, r["texel_idx"][0], r["texel_idx"][1], cov, name)
    print(f"{name} {dtype}: {n} covered pixels, 0 mismatches")


@pytest.mark.parametrize("which", ["cfg2-1080p", "cfg3-1080p", "cfg5-4k", "ldg-333w"])
def test_fused_texels_match_oracle(which):
    from oracle import features as of
    from paper_2301_05262_b200 import network, producer, scenes
    if which == "cfg2-1080p":
        fr = scenes.config_frames(2, seed=3)[0]
    elif which == "cfg3-1080p":
        fr = scenes.config_frames(3, seed=4)[0]
    elif which == "cfg5-4k":
        fr = scenes.config_frames(5, seed=0, n_frames=2)[1]
    else:        # width not a multiple of 4: no TMA tensor map, LDG producer (texel_of)
        fr = scenes.make_frame(scenes.random_scene(16, seed=7, emitter_radius_m=0.1), (250, 333), (700, 700))
    inp = producer.render_inputs([fr])
    cfg, w = _weights()
    idx = _fused_texels(network.Plan(w, cfg, "fp16"), [fr], inp)[0]
    pos = inp["position"][0].cpu().numpy()
    cov = inp["d"][0].cpu().numpy() > 0
    ri, ci, first = of.texel_indices(fr.view, pos, cov)
    assert first == -1
    n = _compare(idx, ri, ci, cov, which)
    print(f"{which}: {n} covered pixels, 0 mismatches")


@pytest.mark.parametrize("dtype", ["fp16", "fp32"])
def test_fused_frustum_error_first_pixel(cfg1, dtype):
    """FrustumError of nsm_infer names the reference's first bad pixel."""
    from types import SimpleNamespace
    from oracle import features as of
    from paper_2301_05262_b200 import network
    from paper_2301_05262_b200._lib import FrustumError
    from paper_2301_05262_b200.infer import ShadowInference
    r = cfg1
    v = golden_view(r)
    narrow = SimpleNamespace(**{**v.__dict__, "tan_half": v.tan_half / 20})
    cov = r["d"] > 0
    _, _, first = of.texel_indices(narrow, r["position"], cov)
    assert first >= 0
    y, x = divmod(first, cov.shape[1])
    cfg, w = _weights()
    run = ShadowInference(network.Plan(w, cfg, dtype), [_frame_ns(r, narrow)])
    with pytest.raises(FrustumError, match=rf"covered pixel \({y}, {x}\) projects outside"):
        run(_inputs(r))


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_fused5_frustum_error_first_pixel(cfg1, dtype):
    """The 5-plane fused pass (feat5 inside nsm_infer) and nsm_features5 also
    name the reference's first out-of-frustum pixel (raster.py:251-255)."""
    from types import SimpleNamespace
    from oracle import features as of
    from paper_2301_05262_b200 import network
    from paper_2301_05262_b200._lib import FrustumError
    from paper_2301_05262_b200.infer import ShadowInference
    from paper_2301_05262_b200.raster import assemble_features5_batch
    r = cfg1
    v = golden_view(r)
    narrow = SimpleNamespace(**{**v.__dict__, "tan_half": v.tan_half / 20})
    cov = r["d"] > 0
    _, _, first = of.texel_indices(narrow, r["position"], cov)
    y, x = divmod(first, cov.shape[1])
    cfg = network.NetworkConfig(in_channels=5)
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    fr = _frame_ns(r, narrow)
    run = ShadowInference(network.Plan(w, cfg, dtype), [fr])
    with pytest.raises(FrustumError, match=rf"covered pixel \({y}, {x}\) projects outside"):
        run(_inputs(r))
    with pytest.raises(FrustumError, match=rf"covered pixel \({y}, {x}\) projects outside"):
        assemble_features5_batch(_inputs(r), [(fr.camera, fr.view, fr.scene.emitter_center, fr.size_index,
                                                fr.bias)])


def test_per_batch_frames_and_input_validation():
    """A launch may carry its own frames (ADVICE: per-batch poses); results
    equal an executor built for those frames; bad inputs raise ValueError."""
    import torch
    from paper_2301_05262_b200 import network, producer, scenes
    from paper_2301_05262_b200.infer import ShadowInference
    cfg, w = _weights()
    plan = network.Plan(w, cfg, "fp16")
    fa = [scenes.make_frame(scenes.random_scene(8, seed=1), (96, 160), (256, 256))]
    fb = [scenes.make_frame(scenes.random_scene(8, seed=2, emitter_radius_m=0.2), (96, 160), (256, 256),
                            camera_pos=(0.5, 3.2, -5.5))]
    ia, ib = producer.render_inputs(fa), producer.render_inputs(fb)
    run = ShadowInference(plan, fa, out_dtype="fp16")
    ref_b = ShadowInference(plan, fb, out_dtype="fp16")(ib).clone()
    got_b = run(ib, frames=fb).clone()
    torch.testing.assert_close(got_b, ref_b, rtol=0, atol=0)
    with pytest.raises(ValueError):
        run.launch({**ia, "d": ia["d"].double()})
    with pytest.raises(ValueError):
        run.launch({**ia, "sm": ia["sm"][:, :128].contiguous()})
    big = [scenes.make_frame(scenes.random_scene(8, seed=1), (96, 160), (512, 512))]
    with pytest.raises(ValueError):
        run.launch(ia, frames=big)


def test_multichunk_launch_equals_single_frames():
    """11 frames in one launch (two enc0 chunks, 8 + 3, each with its own
    dynamically scheduled tiles and the shared tile counter re-zeroed
    between them) give every frame bit-for-bit what a one-frame launch gives,
    twice in a row; the texel indices of the fused pass match too."""
    import torch
    from paper_2301_05262_b200 import network, producer, scenes
    from paper_2301_05262_b200.infer import ShadowInference
    cfg, w = _weights()
    plan = network.Plan(w, cfg, "fp16")
    frames = [scenes.make_frame(scenes.random_scene(6 + i % 4, seed=40 + i, emitter_radius_m=0.05 * (i % 5)),
                                (96, 160), (256, 256), camera_pos=(0.3 * (i % 3), 3.0, -5.5 - 0.1 * i))
              for i in range(11)]
    inp = producer.render_inputs(frames)
    run = ShadowInference(plan, frames, out_dtype="fp16")
    idx = torch.full((11, 2, 96, 160), -1, dtype=torch.int32, device="cuda")
    run.launch(inp, texel_idx=idx)
    run.check_frustum()
    y1 = run.y.clone()
    run.launch(inp)
    run.check_frustum()
    torch.testing.assert_close(run.y, y1, rtol=0, atol=0)
    for i in (0, 5, 8, 10):
        one = {k: v[i:i + 1].contiguous() for k, v in inp.items()}
        r1 = ShadowInference(plan, [frames[i]], out_dtype="fp16")
        i1 = torch.full((1, 2, 96, 160), -1, dtype=torch.int32, device="cuda")
        r1.launch(one, texel_idx=i1)
        r1.check_frustum()
        torch.testing.assert_close(r1.y[0], y1[i], rtol=0, atol=0)
        torch.testing.assert_close(i1[0], idx[i], rtol=0, atol=0)
