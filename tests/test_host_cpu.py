"""Host-side logic and the C-ABI surface, no GPU needed."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_nets

from paper_2301_05262_b200 import _lib, fileio, network, scenes
from paper_2301_05262_b200.network import NetworkConfig


def header_symbols():
    src = open(os.path.join(ROOT, "include", "nsm.h")).read()
    return sorted(set(re.findall(r"\b(nsm_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 11
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert _lib.lib.nsm_abi_version() == _lib.ABI_VERSION == 2
    # the release library ignores NSM_* switches (experiment builds only)
    assert not _lib.experiment_build()


def test_receptive_field_and_depth_kats():
    assert [network.receptive_field(l) for l in (3, 5, 7)] == [24, 96, 384]
    assert network.layers_for_penumbra(21) == 3
    assert network.layers_for_penumbra(90) == 5
    assert network.layers_for_penumbra(24) == 3
    for p in (1, 2.5, 7, 30, 97, 400):
        assert network.receptive_field(network.layers_for_penumbra(p)) >= p


def test_config_validation_and_counts():
    with pytest.raises(ValueError):
        NetworkConfig(layers=1)
    with pytest.raises(ValueError):
        NetworkConfig(base_channels=3)
    cfg = NetworkConfig()
    assert cfg.level_channels == (16, 32, 64, 128)
    assert network.param_count(cfg) == 164_500
    assert network.macs_per_pixel(cfg) == pytest.approx(3536.0)
    assert network.param_count(NetworkConfig(in_channels=5)) == 165_076
    assert sum(1 for _ in network.named_params(cfg)) == 30


def test_named_params_match_golden_weight_sets():
    for name, c in golden_nets().items():
        layers, base, inc, s2d, cap = (int(v) for v in c["cfg"])
        cfg = NetworkConfig(layers, base, inc, bool(s2d), cap)
        shapes = dict(network.named_params(cfg))
        assert set(shapes) == set(c["w"]), name
        for k, v in c["w"].items():
            assert tuple(v.shape) == shapes[k], (name, k)


def test_checkpoint_roundtrip(tmp_path):
    cfg = NetworkConfig(layers=3)
    w = network.init_weights(cfg, np.random.default_rng(0))
    network.save_network(tmp_path / "m.ckpt", w, cfg)
    w2, cfg2 = network.load_network(tmp_path / "m.ckpt")
    assert cfg2 == cfg
    for k in w:
        np.testing.assert_array_equal(w[k].data, w2[k].data)
    raw = (tmp_path / "m.ckpt").read_bytes()
    (tmp_path / "bad.ckpt").write_bytes(raw[:-3])
    with pytest.raises(fileio.FormatError):
        fileio.load_tensors(tmp_path / "bad.ckpt")
    fileio.save_tensors(tmp_path / "x.ckpt", {"l0.enc3.w": np.zeros((1, 1, 3, 3), np.float32)})
    (tmp_path / "x.ckpt.json").write_text((tmp_path / "m.ckpt.json").read_text())
    with pytest.raises(fileio.FormatError):
        network.load_network(tmp_path / "x.ckpt")


def test_floatmap_roundtrip(tmp_path):
    a = np.random.default_rng(1).normal(size=(3, 5, 7)).astype(np.float32)
    fileio.save_floatmap(tmp_path / "a.pfm", a)
    np.testing.assert_array_equal(fileio.load_floatmap(tmp_path / "a.pfm"), a)
    (tmp_path / "b.pfm").write_bytes(b"XXXX" + b"\0" * 20)
    with pytest.raises(fileio.FormatError):
        fileio.load_floatmap(tmp_path / "b.pfm")


def test_checkpoint_bytes_match_reference_format(tmp_path):
    import sys
    if not os.path.isdir("/root/reference/pkg/src"):
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, "/root/reference/pkg/src")
    ref = pytest.importorskip("shadowkit.fileio")
    named = {"a": np.arange(6, dtype=np.float32).reshape(2, 3), "b": np.ones(4, np.float32)}
    fileio.save_tensors(tmp_path / "ours.ckpt", named)
    ref.save_tensors(tmp_path / "ref.ckpt", named)
    assert (tmp_path / "ours.ckpt").read_bytes() == (tmp_path / "ref.ckpt").read_bytes()


def _plan_create_status(cfg, weights):
    names = list(weights)
    arrays = [np.ascontiguousarray(weights[k], dtype=np.float32) for k in names]
    n = len(names)
    dims = [(C.c_int32 * max(a.ndim, 1))(*a.shape) for a in arrays]
    h = C.POINTER(_lib.PlanHandle)()
    st = _lib.lib.nsm_plan_create(
        C.byref(_lib.NetConfig(*cfg)), n, (C.c_char_p * n)(*[k.encode() for k in names]),
        (C.c_void_p * n)(*[a.ctypes.data for a in arrays]),
        (C.c_int32 * n)(*[a.ndim for a in arrays]),
        (C.POINTER(C.c_int32) * n)(*[C.cast(d, C.POINTER(C.c_int32)) for d in dims]),
        _lib.NSM_F32, C.byref(h))
    return st, _lib.lib.nsm_last_error().decode()


def test_abi_validation_errors_without_gpu():
    cfg = NetworkConfig(layers=3)
    w = {k: v.data for k, v in network.init_weights(cfg, np.random.default_rng(0)).items()}
    st, msg = _plan_create_status((1, 16, 4, 1, 256), w)
    assert st == _lib.NSM_ERR_ARG and "layers" in msg
    bad = dict(w)
    bad.pop("head.b")
    st, msg = _plan_create_status((3, 16, 4, 1, 256), bad)
    assert st == _lib.NSM_ERR_FORMAT and msg == "checkpoint parameters do not match config"
    with pytest.raises(_lib.FormatError):
        _lib.check(st)
    bad = dict(w)
    bad["l0.enc3.w"] = np.zeros((16, 16, 1, 1), np.float32)
    st, msg = _plan_create_status((3, 16, 4, 1, 256), bad)
    assert st == _lib.NSM_ERR_SHAPE and "l0.enc3.w" in msg
    with pytest.raises(ValueError):
        _lib.check(st)


def test_scene_generator_deterministic_and_fit():
    a = scenes.config_frames(2, seed=3)[0]
    b = scenes.config_frames(2, seed=3)[0]
    np.testing.assert_array_equal(a.scene.primitive_table(), b.scene.primitive_table())
    assert a.camera.resolution == (1080, 1920) and a.view.resolution == (2048, 2048)
    assert len(a.scene.objects) == 33
    f4 = scenes.config_frames(4, seed=0)
    assert len(f4) == 8
    steps = [np.linalg.norm(f4[i + 1].scene.emitter_center - f4[i].scene.emitter_center)
             for i in range(7)]
    np.testing.assert_allclose(steps, 0.02)
    s = f4[0].size_index
    assert 0.8 <= s <= 8.0
    assert scenes.emitter_radius(4.0) == 0.25
    with pytest.raises(scenes.SceneError):
        scenes.emitter_radius(4.5)
