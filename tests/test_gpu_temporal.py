"""Temporal consumers on the GPU vs the reference goldens / the oracle.

motion vectors (raster.py:330-358) and temporal instability
(analysis.py:350-377); cases follow the reference's TestMotionVectors
(tests/test_raster.py:218-258) plus the golden 4-frame sequence.
"""

import math

import numpy as np
import pytest

from conftest import golden_camera, load_golden

pytestmark = pytest.mark.gpu


def _seq():
    import torch
    g = load_golden("temporal")
    t = int(g["t_frames"])
    inp = {k: torch.from_numpy(np.stack([g[f"{k}{i}"] for i in range(t)])).cuda()
           for k in ("d", "normal", "position")}
    cams = [golden_camera(g, f"cam{i}") for i in range(t)]
    return g, t, inp, cams


def test_motion_vectors_batch_golden():
    from paper_2301_05262_b200 import temporal
    g, t, inp, cams = _seq()
    vec, valid = temporal.motion_vectors_batch(inp, cams)
    vec, valid = vec.cpu().numpy(), valid.cpu().numpy().astype(bool)
    for k in range(t - 1):
        assert np.max(np.abs(vec[k] - g[f"vec{k}"])) < 1e-9
        np.testing.assert_array_equal(valid[k], g[f"valid{k}"])


def test_temporal_instability_golden():
    import torch
    from paper_2301_05262_b200 import temporal
    g, t, inp, cams = _seq()
    vec, valid = temporal.motion_vectors_batch(inp, cams)
    rep = temporal.temporal_instability_batch(torch.from_numpy(g["frames"]).cuda(), vec, valid, 3.0)
    assert rep.valid_pixels == int(g["valid_pixels"])
    assert rep.frames_compared == t - 1
    assert abs(rep.instability - float(g["E"])) <= 1e-12 * abs(float(g["E"]))
    assert abs(rep.rejected_fraction - float(g["rejected"])) < 1e-15
    # the host-array drop-in gives the same report
    motions = [temporal.MotionField(g[f"vec{k}"], g[f"valid{k}"]) for k in range(t - 1)]
    rep2 = temporal.temporal_instability(list(g["frames"]), motions, 3.0)
    assert rep2.valid_pixels == rep.valid_pixels
    assert abs(rep2.instability - rep.instability) <= 1e-12 * rep.instability


def _gbuf(spec, cam):
    import ctypes as C
    import torch
    from paper_2301_05262_b200 import _lib
    tab = torch.from_numpy(spec.primitive_table()).cuda()
    h, w = cam.resolution
    d = torch.empty((h, w), device="cuda")
    n = torch.empty((3, h, w), device="cuda")
    p = torch.empty((3, h, w), device="cuda")
    _lib.check(_lib.lib.nsm_render_gbuffer(tab.data_ptr(), tab.shape[0], C.byref(_lib.camera_c(cam)),
                                           d.data_ptr(), n.data_ptr(), p.data_ptr(), _lib.stream_ptr()))
    from types import SimpleNamespace
    dd, nn, pp = d.cpu().numpy(), n.cpu().numpy(), p.cpu().numpy()
    return SimpleNamespace(d=dd, normal=nn, position=pp, coverage=dd > 0, camera=cam)


def _project_back(cam, d):
    """fp64 world positions on the camera rays at view depth d
    (d = t * ray.forward, raster.py:225; rays per scene.py:153-163)."""
    h, w = cam.resolution
    half_h = math.tan(cam.fov_y / 2.0)
    half_w = half_h * (w / h)
    fwd, up = np.asarray(cam.forward, np.float64), np.asarray(cam.up, np.float64)
    right = np.cross(fwd, up)
    ys, xs = np.mgrid[0:h, 0:w]
    u = ((xs + 0.5) / w * 2.0 - 1.0) * half_w
    v = (1.0 - (ys + 0.5) / h * 2.0) * half_h
    rays = fwd[:, None, None] + u * right[:, None, None] + v * up[:, None, None]
    rays /= np.linalg.norm(rays, axis=0)
    t = d.astype(np.float64) / np.tensordot(fwd, rays, axes=1)
    return np.asarray(cam.position, np.float64)[:, None, None] + rays * t


def test_static_identity():
    # test_raster.py:219-223
    from paper_2301_05262_b200 import scenes, temporal
    fr = scenes.config_frames(1, seed=3)[0]
    g = _gbuf(fr.scene, fr.camera)
    mf = temporal.motion_vectors(g, fr.camera, g)
    # the reference test uses fp64 planes (atol 1e-9); our producer writes
    # fp32 world positions, whose rounding moves the reprojection by ~1e-5 px
    np.testing.assert_allclose(mf.vectors[:, g.coverage], 0.0, atol=1e-4)
    g64 = type(g)(**{k: (v.astype(np.float64) if isinstance(v, np.ndarray) and v.dtype == np.float32 else v)
                     for k, v in vars(g).items()})
    g64.position = _project_back(fr.camera, g.d)
    mf64 = temporal.motion_vectors(g64, fr.camera, g64)
    np.testing.assert_allclose(mf64.vectors[:, g.coverage], 0.0, atol=1e-9)
    assert np.array_equal(mf64.valid, g.coverage)
    assert np.array_equal(mf.valid, g.coverage)


def test_translation_matches_analytic_shift():
    # test_raster.py:225-246: fronto-parallel plane, camera slides right
    from paper_2301_05262_b200 import scenes, temporal
    spec = scenes.SceneSpec((scenes.plane((0, 0, 4), (0, 0, -1), (4, 4)),), (0.0, 3.0, 0.0), 0.0)
    res = (40, 80)
    cam0 = scenes.CameraPose((0, 0, 0), (0, 0, 1), (0, 1, 0), math.radians(45), res)
    dx = 0.05
    cam1 = scenes.CameraPose((dx, 0, 0), (0, 0, 1), (0, 1, 0), math.radians(45), res)
    g0, g1 = _gbuf(spec, cam0), _gbuf(spec, cam1)
    mf = temporal.motion_vectors(g1, cam0, g0)
    focal = (res[0] / 2) / math.tan(math.radians(45) / 2)
    sel = mf.valid
    assert sel.mean() > 0.9
    np.testing.assert_allclose(mf.vectors[1][sel], -dx * focal / 4.0, atol=1e-5)
    np.testing.assert_allclose(mf.vectors[0][sel], 0.0, atol=1e-5)


def test_disocclusion_and_oracle_parity():
    # test_raster.py:248-258 plus oracle parity on the same GPU-rendered planes
    from oracle import temporal as ot
    from paper_2301_05262_b200 import scenes, temporal
    fr = scenes.config_frames(1, seed=4)[0]
    cam0 = fr.camera
    cam1 = scenes.CameraPose(np.asarray(cam0.position) + np.array([0.5, 0, 0]), cam0.forward, cam0.up,
                             cam0.fov_y, cam0.resolution)
    g0, g1 = _gbuf(fr.scene, cam0), _gbuf(fr.scene, cam1)
    mf = temporal.motion_vectors(g1, cam0, g0)
    assert mf.valid.sum() < g1.coverage.sum()
    vec, ok = ot.motion_vectors(g1.position, g1.normal, g1.coverage, g0.d, g0.normal, g0.coverage, cam0)
    assert np.max(np.abs(mf.vectors - vec)) < 1e-9
    assert np.mean(mf.valid != ok) == 0.0


def test_errors():
    import torch
    from paper_2301_05262_b200 import temporal
    one = torch.zeros((1, 8, 8), device="cuda")
    with pytest.raises(ValueError):
        temporal.temporal_instability_batch(one, torch.zeros((0, 2, 8, 8), dtype=torch.float64,
                                                             device="cuda"),
                                            torch.zeros((0, 8, 8), dtype=torch.uint8, device="cuda"))
    two = torch.zeros((2, 8, 8), device="cuda")
    with pytest.raises(temporal.NoValidPixels):
        temporal.temporal_instability_batch(two, torch.zeros((1, 2, 8, 8), dtype=torch.float64,
                                                             device="cuda"),
                                            torch.zeros((1, 8, 8), dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        temporal.temporal_instability([np.zeros((4, 4))], [])


def test_config4_window_instability_vs_oracle():
    """The 8-frame 1080p soft window of the bench: fused fp16 inference,
    motion vectors and instability on the device vs the oracle consumers on
    the same visibility."""
    from oracle import temporal as ot
    from paper_2301_05262_b200 import network, producer, scenes, temporal
    from paper_2301_05262_b200.infer import ShadowInference
    frames = scenes.config_frames(4, seed=0, n_frames=4)
    inp = producer.render_inputs(frames)
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    vis = ShadowInference(network.Plan(w, cfg, "fp16"), frames)(inp)[:, 0]
    vec, valid = temporal.motion_vectors_batch(inp, [f.camera for f in frames])
    rep = temporal.temporal_instability_batch(vis, vec, valid, 3.0)
    h = {k: v.cpu().numpy() for k, v in inp.items()}
    ovec, ook = [], []
    for t in range(1, len(frames)):
        v, ok = ot.motion_vectors(h["position"][t], h["normal"][t], h["d"][t] > 0, h["d"][t - 1],
                                  h["normal"][t - 1], h["d"][t - 1] > 0, frames[t - 1].camera)
        ovec.append(v)
        ook.append(ok)
    gv, gk = vec.cpu().numpy(), valid.cpu().numpy().astype(bool)
    assert max(np.max(np.abs(gv[k] - ovec[k])) for k in range(3)) < 1e-8
    assert sum(int((gk[k] != ook[k]).sum()) for k in range(3)) == 0
    E, n, rej = ot.temporal_instability(list(vis.cpu().numpy()), ovec, ook, 3.0)
    print(f"config-4 window E={rep.instability:.6g} valid={rep.valid_pixels} rejected={rej:.3f}")
    assert rep.valid_pixels == n
    assert abs(rep.instability - E) <= 1e-9 * abs(E)
