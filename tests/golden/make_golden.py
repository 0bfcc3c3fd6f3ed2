"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

It imports ``shadowkit`` (the reference package, read-only) and records its
outputs on seeded inputs built by ``paper_2301_05262_b200.scenes``. The oracle
(``oracle/``) and the CUDA path are both checked against these files; the
GPU box never needs /root/reference.

Fixtures (all ``np.savez_compressed``):

* ``cfg1.npz``   -- BASELINE config 1 (256x256, 8 objects, SM 512^2, point
  light, seed 0): reference ``render_shadowmap``/``render_gbuffer`` buffers
  (rounded to fp32, the path's input format), the reference
  ``assemble_features`` output and texel indices on those fp32 buffers, the
  reference ``network.forward`` visibility for ``init_weights(cfg,
  default_rng(SeedSequence([0, 0x11])))`` and a checksum of those weights.
* ``variants.npz`` -- non-square 96x160 camera, 300x260 map, 12 objects,
  soft light, explicit bias, size_index 3: features + indices.
* ``canon.npz``  -- the reference test-suite's canonical scene fixture
  (conftest.small_buffers: 64x128, SM 256^2, size_index 2).
* ``temporal.npz`` -- a 4-frame sequence (48x80, moving camera, light and
  one object, as config 4 at small size): reference ``motion_vectors`` per
  consecutive pair on the fp32-rounded G-buffers and reference
  ``temporal_instability`` (alpha_t 3) of seeded smooth fp32 frames.
* ``sensitivity.npz`` -- reference ``analysis.sensitivity_report`` (phi =
  reference ``network.forward``, rng default_rng(7), repeats 2) on three
  32x48 crops of the cfg1 feature stack, and ``training._eval_mse`` of the
  same stacks against seeded targets.
* ``dataset_small/`` + ``dataset_small_ref.npz`` -- a 3-frame dataset written
  by the reference's own ``dataset.generate_dataset`` (32x48, moving camera,
  1 perturbation, sizes 0/2, 4 spp) and the reference's readings of it:
  ``load_feature_stack`` (size 2), ``load_gbuffer`` planes, the
  ``cli._sequence_outputs`` visibility and the ``cmd_eval_temporal`` E.
* ``nets.npz``   -- ``network.forward`` on random planes for a spread of
  ``NetworkConfig``s (layers 2..6, in_channels 5, plain mode, channel cap,
  base 8) with random non-zero biases; weights included.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")

from shadowkit import autodiff as ad            # noqa: E402
from shadowkit import network, raster, scene as sk_scene   # noqa: E402
from shadowkit.experiments import canonical_scene   # noqa: E402

from paper_2301_05262_b200 import scenes        # noqa: E402
from oracle import features as ofeat            # noqa: E402


def to_reference_scene(spec: scenes.SceneSpec):
    objs = []
    for o in spec.objects:
        p = o.params
        if o.kind == scenes.KIND_PLANE:
            objs.append(sk_scene.Plane(p[0:3], p[3:6], tuple(p[6:8]), occluder=o.occluder))
        elif o.kind == scenes.KIND_SPHERE:
            objs.append(sk_scene.Sphere(p[0:3], p[3], occluder=o.occluder))
        else:
            objs.append(sk_scene.Box(p[0:3], p[3:6], occluder=o.occluder))
    return sk_scene.Scene(tuple(objs), sk_scene.Emitter(spec.emitter_center, 0.0))


def to_reference_camera(cam: scenes.CameraPose):
    return sk_scene.CameraPose(cam.position, cam.forward, cam.up, cam.fov_y, cam.resolution)


def view_record(view, prefix="view"):
    return {f"{prefix}_position": np.asarray(view.position), f"{prefix}_forward": np.asarray(view.forward),
            f"{prefix}_up": np.asarray(view.up), f"{prefix}_right": np.asarray(view.right),
            f"{prefix}_tan_half": np.float64(view.tan_half),
            f"{prefix}_resolution": np.asarray(view.resolution, dtype=np.int64)}


def camera_record(cam, prefix="cam"):
    return {f"{prefix}_position": np.asarray(cam.position), f"{prefix}_forward": np.asarray(cam.forward),
            f"{prefix}_up": np.asarray(cam.up), f"{prefix}_fov_y": np.float64(cam.fov_y),
            f"{prefix}_resolution": np.asarray(cam.resolution, dtype=np.int64)}


def reference_features_on_fp32(g64, sm64, cam, center, size_index, bias):
    """Reference assemble_features on the fp32-rounded buffers the GPU reads."""
    d32 = g64.d.astype(np.float32)
    n32 = g64.normal.astype(np.float32)
    p32 = g64.position.astype(np.float32)
    z_f, c_e, c_c, cov = ofeat.derive_planes(d32, n32, p32, cam, center)
    g = raster.GBuffer(d=d32.astype(np.float64), normal=n32.astype(np.float64),
                       position=p32.astype(np.float64), n_e=g64.n_e, z_f=z_f, c_e=c_e,
                       c_c=c_c, coverage=cov, camera=g64.camera)
    sm = raster.ShadowMap(depth=sm64.depth.astype(np.float32).astype(np.float64),
                          view=sm64.view, scene_diag=sm64.scene_diag)
    fs = raster.assemble_features(g, sm, size_index, bias)
    row, col, _ = sm.view.project(np.moveaxis(g.position, 0, -1))
    idx = np.stack([np.rint(row), np.rint(col)]).astype(np.int32)
    idx[:, ~cov] = -1
    return fs, idx, (d32, n32, p32), (z_f, c_e, c_c, cov)


def weights_checksum(w):
    h = hashlib.sha256()
    for k in sorted(w):
        h.update(k.encode())
        h.update(np.ascontiguousarray(w[k].data, dtype="<f4").tobytes())
    return h.hexdigest()


def make_cfg1():
    fr = scenes.config_frames(1, seed=0)[0]
    sc = to_reference_scene(fr.scene)
    cam = to_reference_camera(fr.camera)
    sm = raster.render_shadowmap(sc, sc.emitter, fr.view.resolution)
    g = raster.render_gbuffer(sc, cam, sc.emitter)
    # our frustum fit must equal the reference's exactly
    for a in ("position", "forward", "up", "right"):
        assert np.array_equal(getattr(sm.view, a), getattr(fr.view, a)), a
    assert sm.view.tan_half == fr.view.tan_half
    assert sm.scene_diag == fr.scene.diagonal
    bias = sm.default_bias
    fs, idx, (d32, n32, p32), (z_f, c_e, c_c, cov) = reference_features_on_fp32(
        g, sm, cam, sc.emitter.center, 0.0, None)
    # the derived planes recomputed from fp64 buffers match render_gbuffer
    zf64, ce64, cc64, cov64 = ofeat.derive_planes(g.d, g.normal, g.position, cam, sc.emitter.center)
    assert np.array_equal(cov64, g.coverage)
    assert np.max(np.abs(zf64 - g.z_f)) < 1e-12 and np.max(np.abs(ce64 - g.c_e)) < 1e-12
    assert np.max(np.abs(cc64 - g.c_c)) < 1e-12

    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    with ad.no_grad():
        vis = network.forward(w, cfg, fs.data).data
    rec = dict(d=d32, normal=n32, position=p32, sm=sm.depth.astype(np.float32),
               features=fs.data, texel_idx=idx, coverage=cov, bias=np.float64(bias),
               size_index=np.float64(0.0), emitter_center=np.asarray(sc.emitter.center),
               visibility=vis.astype(np.float32), weights_sha256=np.bytes_(weights_checksum(w)),
               sm64_finite=np.isfinite(sm.depth))
    rec.update(view_record(sm.view))
    rec.update(camera_record(cam))
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **rec)
    print("cfg1: covered", int(cov.sum()), "in shadow", int((fs.data[0] < 0).sum()),
          "vis range", float(vis.min()), float(vis.max()))


def make_variants():
    spec = scenes.random_scene(12, seed=7, emitter_radius_m=0.2)
    fr = scenes.make_frame(spec, (96, 160), (300, 260), camera_pos=(1.0, 2.5, -5.0),
                           target=(0.2, 0.3, 0.1), fov_deg=50.0)
    sc = to_reference_scene(spec)
    cam = to_reference_camera(fr.camera)
    sm = raster.render_shadowmap(sc, sc.emitter, (300, 260))
    g = raster.render_gbuffer(sc, cam, sc.emitter)
    fs, idx, (d32, n32, p32), _ = reference_features_on_fp32(
        g, sm, cam, sc.emitter.center, 3.0, 0.0125)
    rec = dict(d=d32, normal=n32, position=p32, sm=sm.depth.astype(np.float32),
               features=fs.data, texel_idx=idx, bias=np.float64(0.0125), size_index=np.float64(3.0),
               emitter_center=np.asarray(sc.emitter.center))
    rec.update(view_record(sm.view))
    rec.update(camera_record(cam))
    np.savez_compressed(os.path.join(HERE, "variants.npz"), **rec)
    print("variants: covered", int(g.coverage.sum()))


def make_canon():
    sc, cam = canonical_scene(resolution=(64, 128))        # conftest.py:8-11
    sm = raster.render_shadowmap(sc, sc.emitter, (256, 256))
    g = raster.render_gbuffer(sc, cam, sc.emitter)
    fs64 = raster.assemble_features(g, sm, sc.emitter.size_index)   # conftest.py:19
    fs, idx, (d32, n32, p32), _ = reference_features_on_fp32(
        g, sm, cam, sc.emitter.center, sc.emitter.size_index, None)
    rec = dict(d=d32, normal=n32, position=p32, sm=sm.depth.astype(np.float32),
               features=fs.data, features_fp64_inputs=fs64.data, texel_idx=idx,
               bias=np.float64(sm.default_bias), size_index=np.float64(sc.emitter.size_index),
               emitter_center=np.asarray(sc.emitter.center))
    rec.update(view_record(sm.view))
    rec.update(camera_record(cam))
    np.savez_compressed(os.path.join(HERE, "canon.npz"), **rec)
    print("canon: covered", int(g.coverage.sum()))


NET_CASES = [
    # name, NetworkConfig kwargs, (H, W)
    ("l5_default", {}, (32, 48)),
    ("l2", {"layers": 2}, (6, 10)),
    ("l3", {"layers": 3}, (24, 40)),
    ("l4_in5", {"layers": 4, "in_channels": 5}, (16, 40)),
    ("l6_base8", {"layers": 6, "base_channels": 8}, (64, 32)),
    ("l5_base8_cap32", {"base_channels": 8, "channel_cap": 32}, (48, 16)),
    ("l3_plain", {"layers": 3, "use_space_to_depth": False}, (16, 24)),
    ("l4_plain_in1", {"layers": 4, "use_space_to_depth": False, "in_channels": 1}, (16, 16)),
]


def make_nets():
    rec = {}
    rng = np.random.default_rng(2024)
    for name, kw, (h, w) in NET_CASES:
        cfg = network.NetworkConfig(**kw)
        wts = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([3, 0x11])))
        for k, v in wts.items():
            if k.endswith(".b"):
                v.data[:] = rng.normal(0.0, 0.1, size=v.data.shape).astype(np.float32)
        x = rng.normal(0.0, 1.0, size=(cfg.in_channels, h, w)).astype(np.float32)
        with ad.no_grad():
            y = network.forward(wts, cfg, x).data
        rec[f"{name}/x"] = x
        rec[f"{name}/y"] = y.astype(np.float32)
        rec[f"{name}/cfg"] = np.asarray([cfg.layers, cfg.base_channels, cfg.in_channels,
                                         int(cfg.use_space_to_depth), cfg.channel_cap])
        for k, v in wts.items():
            rec[f"{name}/w/{k}"] = v.data
    np.savez_compressed(os.path.join(HERE, "nets.npz"), **rec)
    print("nets:", len(NET_CASES), "cases")


def make_penumbra():
    """analysis.penumbra_extents on random valid geometry (pins the formula
    the blocker-search extension reuses)."""
    from shadowkit import analysis
    rng = np.random.default_rng(11)
    n = 4000
    z_min = rng.uniform(0.5, 5.0, n)
    z_max = z_min + rng.uniform(0.0, 1.0, n)
    z_f = z_max + rng.uniform(0.01, 4.0, n)
    r_e = rng.uniform(0.0, 0.5, n)
    xa, xb = analysis.penumbra_extents(z_min, z_max, z_f, r_e)
    np.savez_compressed(os.path.join(HERE, "penumbra.npz"), z_min=z_min, z_max=z_max, z_f=z_f,
                        r_e=r_e, x_a=xa, x_b=xb)
    print("penumbra:", n)


def make_temporal():
    from shadowkit import analysis
    rng = np.random.default_rng(np.random.SeedSequence([5, 0x7E]))
    base = scenes.random_scene(16, seed=5, emitter_radius_m=0.2)
    dirs = [scenes._unit(rng.normal(size=3)) for _ in range(3)]
    mover = 3
    t_frames, res = 4, (48, 80)
    rec, gbufs, cams = {}, [], []
    for t in range(t_frames):
        step = 0.05 * t
        objs = list(base.objects)
        p = np.asarray(objs[mover].params, dtype=np.float64)
        objs[mover] = (scenes.sphere(p[0:3] + step * dirs[1], p[3]) if objs[mover].kind == scenes.KIND_SPHERE
                       else scenes.box(p[0:3] + step * dirs[1], p[3:6] + step * dirs[1]))
        spec = scenes.SceneSpec(tuple(objs), base.emitter_center + step * dirs[0], 0.2)
        fr = scenes.make_frame(spec, res, (128, 128),
                               camera_pos=np.asarray(scenes.CAMERA_POS) + step * dirs[2])
        sc = to_reference_scene(spec)
        cam = to_reference_camera(fr.camera)
        g = raster.render_gbuffer(sc, cam, sc.emitter)
        d32, n32, p32 = (g.d.astype(np.float32), g.normal.astype(np.float32),
                         g.position.astype(np.float32))
        gbufs.append(raster.GBuffer(d=d32.astype(np.float64), normal=n32.astype(np.float64),
                                    position=p32.astype(np.float64), n_e=g.n_e, z_f=g.z_f,
                                    c_e=g.c_e, c_c=g.c_c, coverage=g.coverage, camera=cam))
        cams.append(cam)
        rec[f"d{t}"], rec[f"normal{t}"], rec[f"position{t}"] = d32, n32, p32
        rec.update(camera_record(cam, f"cam{t}"))
    motions = [raster.motion_vectors(gbufs[t], cams[t - 1], gbufs[t - 1]) for t in range(1, t_frames)]
    ys, xs = np.mgrid[0:res[0], 0:res[1]]
    frames = [(0.5 + 0.4 * np.sin(0.11 * xs + 0.07 * ys + 0.3 * t)
               + rng.normal(0.0, 0.02, size=res)).astype(np.float32) for t in range(t_frames)]
    rep = analysis.temporal_instability([f.astype(np.float64) for f in frames], motions, 3.0)
    for k, m in enumerate(motions):
        rec[f"vec{k}"], rec[f"valid{k}"] = m.vectors, m.valid
    static = raster.motion_vectors(gbufs[0], cams[0], gbufs[0])
    rec.update(frames=np.stack(frames), E=np.float64(rep.instability),
               valid_pixels=np.int64(rep.valid_pixels), rejected=np.float64(rep.rejected_fraction),
               static_vec=static.vectors, static_valid=static.valid, t_frames=np.int64(t_frames))
    np.savez_compressed(os.path.join(HERE, "temporal.npz"), **rec)
    print("temporal: valid", [int(m.valid.sum()) for m in motions], "E", rep.instability)


def make_sensitivity():
    from shadowkit import analysis, training
    feats = np.load(os.path.join(HERE, "cfg1.npz"))["features"]
    stacks = [np.ascontiguousarray(feats[:, y:y + 32, x:x + 48]) for y, x in ((96, 80), (128, 144), (160, 40))]
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))

    def phi(stack):
        with ad.no_grad():
            return network.forward(w, cfg, stack).data[0]

    rep = analysis.sensitivity_report(phi, stacks, raster.FEATURE_CHANNELS, repeats=2,
                                      rng=np.random.default_rng(7))
    trng = np.random.default_rng(8)
    targets = [trng.uniform(0, 1, size=(32, 48)).astype(np.float32) for _ in stacks]
    samples = [training.TrainingSample((s,), t, 0.0) for s, t in zip(stacks, targets)]
    m = training._eval_mse(w, cfg, samples)
    np.savez_compressed(os.path.join(HERE, "sensitivity.npz"), stacks=np.stack(stacks),
                        targets=np.stack(targets), absolute=rep.absolute, relative=rep.relative,
                        heldout_mse=np.float64(m))
    print("sensitivity:", rep.absolute, "mse", m)


SMALL_SCENE = """
[scene]
objects = [
  { type = "plane", point = [0, 0, 0], normal = [0, 1, 0], half_extent = [5, 5] },
  { type = "sphere", center = [0.3, 0.6, 0.2], radius = 0.5 },
  { type = "box", min = [-1.2, 0.0, -0.4], max = [-0.6, 0.9, 0.3] },
]
[emitter]
center = [3.0, 5.0, 2.0]
size_index = 2.0
[camera]
position = [0.0, 3.0, -6.0]
look_at = [0.0, 0.0, 0.0]
fov_deg = 60.0
resolution = [32, 48]
[perturbation]
count = 1
"""

SMALL_TRAJ = """
[[camera_keys]]
time = 0.0
position = [0.0, 3.0, -6.0]
look_at = [0.0, 0.0, 0.0]
[[camera_keys]]
time = 1.0
position = [0.3, 3.1, -5.9]
look_at = [0.0, 0.0, 0.0]
"""


def make_dataset():
    import shutil
    import tempfile
    from shadowkit import analysis, dataset
    out = os.path.join(HERE, "dataset_small")
    shutil.rmtree(out, ignore_errors=True)
    with tempfile.TemporaryDirectory() as tmp:
        sp, tp = os.path.join(tmp, "scene.toml"), os.path.join(tmp, "traj.toml")
        open(sp, "w").write(SMALL_SCENE)
        open(tp, "w").write(SMALL_TRAJ)
        st = dataset.GenerateSettings(frames=3, spp=4, msaa=1, sizes=(0.0, 2.0), shadow_res=(128, 128),
                                      perturbations=1, seed=0)
        dataset.generate_dataset(sp, tp, out, st)
    for root, _, files in os.walk(out):
        for f in files:
            if f.endswith(".png"):
                os.remove(os.path.join(root, f))
    m = dataset.load_manifest(out)
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    vis = []
    for fi in range(len(m.frames)):
        stack = dataset.load_feature_stack(m, fi, 0, 2.0)
        with ad.no_grad():
            vis.append(network.forward(w, cfg, stack.data).data[0].astype(np.float64))
    gb = [dataset.load_gbuffer(m, i) for i in range(len(vis))]
    motions = [raster.motion_vectors(gb[t], gb[t - 1].camera, gb[t - 1]) for t in range(1, len(vis))]
    rep = analysis.temporal_instability(vis, motions, 3.0)
    fs = dataset.load_feature_stack(m, 1, 1, 2.0)
    np.savez_compressed(os.path.join(HERE, "dataset_small_ref.npz"), vis=np.stack(vis).astype(np.float32),
                        E=np.float64(rep.instability), valid_pixels=np.int64(rep.valid_pixels),
                        stack_1_1_s2=fs.data, coverage_1=fs.coverage,
                        gb_position_2=gb[2].position, gb_z_f_2=gb[2].z_f,
                        target_2_s2=dataset.load_target(m, 2, 2.0))
    print("dataset: frames", len(vis), "E", rep.instability, "valid", rep.valid_pixels)


if __name__ == "__main__":
    make_dataset()
    make_sensitivity()
    make_temporal()
    make_penumbra()
    make_cfg1()
    make_variants()
    make_canon()
    make_nets()
