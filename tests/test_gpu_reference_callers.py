"""The drop-in claim, end to end (needs a B200): the reference's OWN callers
of the path -- ``cli.cmd_infer`` (cli.py:128-141), ``cli.cmd_eval_temporal``
via ``_sequence_outputs`` (cli.py:144-170), ``cli.cmd_sensitivity``'s phi
(cli.py:173-196) -- are run twice on the stock ``shadowkit`` package (the
copy ``oracle/make_ref.py`` stages under ``oracle/_ref``): once as shipped,
once with ``shadowkit.network.forward`` swapped for this repository's
``network.forward`` -- the two-line change INTEGRATION.md §2 shows.  The
patched run must reproduce the stock outputs within the fp32 bar (1e-4
max-abs).  The feature pass is checked the same way on objects the stock
renderer made: ``raster.render_gbuffer`` / ``render_shadowmap`` of the
reference's canonical scene (fp64 G-buffer, fp64 shadow map) into our
``raster.assemble_features``, against the stock ``assemble_features``
(raster.py:266-278) and ``np.rint`` of the stock ``EmitterView.project``
(raster.py:84-94, 247-250).

The stock package is test infrastructure (the checker), never the thing
measured; the test is skipped when the staged copy is absent.
"""

import argparse
import importlib
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF_DIR = os.path.join(ROOT, "oracle", "_ref")
DATA = os.path.join(ROOT, "tests", "golden", "dataset_small")
VIS_TOL = 1e-4


@pytest.fixture(scope="module")
def sk():
    if not os.path.isfile(os.path.join(REF_DIR, "shadowkit", "cli.py")):
        pytest.skip("oracle/_ref/shadowkit not staged (python oracle/make_ref.py)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    mods = {m: importlib.import_module("shadowkit." + m)
            for m in ("cli", "network", "raster", "scene", "fileio", "autodiff", "dataset")}
    return argparse.Namespace(**mods)


@pytest.fixture
def patched(sk, monkeypatch):
    """shadowkit.network.forward -> paper_2301_05262_b200.network.forward."""
    from paper_2301_05262_b200 import network as ours

    calls = []

    def forward(weights, cfg, x):
        calls.append(np.shape(getattr(x, "data", x)))
        return ours.forward(weights, cfg, x)

    def use():
        monkeypatch.setattr(sk.network, "forward", forward)
        return calls
    return use


def _ckpt(sk, tmp_path):
    cfg = sk.network.NetworkConfig()
    w = sk.network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    path = tmp_path / "model.ckpt"
    sk.network.save_network(path, w, cfg)
    return str(path)


def test_cmd_infer_stock_vs_dropin(sk, patched, tmp_path):
    ck = _ckpt(sk, tmp_path)
    outs = []
    for tag in ("stock", "dropin"):
        if tag == "dropin":
            calls = patched()
        args = argparse.Namespace(data=DATA, ckpt=ck, frame=1, size=2.0, out=str(tmp_path / tag))
        assert sk.cli.cmd_infer(args) == 0
        outs.append(sk.fileio.load_floatmap(tmp_path / tag / "shadow.pfm"))
    assert len(calls) == 1                       # the GPU forward really ran
    d = np.abs(outs[0].astype(np.float64) - outs[1])
    print(f"cmd_infer: stock vs drop-in max-abs {d.max():.3g}")
    assert outs[0].shape == outs[1].shape and d.max() <= VIS_TOL


def test_cmd_eval_temporal_stock_vs_dropin(sk, patched, tmp_path, capsys):
    ck = _ckpt(sk, tmp_path)
    es = []
    for tag in ("stock", "dropin"):
        if tag == "dropin":
            calls = patched()
        args = argparse.Namespace(data=DATA, ckpt=ck, size=2.0, alpha_t=3.0, out=None)
        assert sk.cli.cmd_eval_temporal(args) == 0
        line = [ln for ln in capsys.readouterr().out.splitlines() if ln.startswith("E=")][-1]
        es.append(float(line[2:]))
    assert len(calls) >= 2                       # one forward per frame of the sequence
    print(f"eval-temporal E: stock {es[0]:.9g}, drop-in {es[1]:.9g}")
    assert abs(es[0] - es[1]) <= 1e-4 * max(1.0, abs(es[0]))


def test_sensitivity_phi_stock_vs_dropin(sk, patched, tmp_path):
    """cmd_sensitivity's phi (cli.py:181-183) on the dataset's stacks."""
    weights, cfg = sk.network.load_network(_ckpt(sk, tmp_path))
    m = sk.dataset.load_manifest(DATA)
    stacks = [sk.dataset.load_feature_stack(m, fi, 0, 2.0).data for fi in range(len(m.frames))]
    with sk.autodiff.no_grad():
        ref = [sk.network.forward(weights, cfg, s).data[0] for s in stacks]
    patched()
    got = [sk.network.forward(weights, cfg, s).data[0] for s in stacks]
    d = max(float(np.abs(np.asarray(a, np.float64) - b).max()) for a, b in zip(ref, got))
    print(f"phi over {len(stacks)} stacks: max-abs {d:.3g}")
    assert d <= VIS_TOL


def test_assemble_features_on_stock_rendered_objects(sk):
    """Stock render_gbuffer / render_shadowmap objects (fp64) straight into
    our assemble_features and texel_indices."""
    from paper_2301_05262_b200 import raster as ours
    p = os.path.join(os.environ.get("TMPDIR", "/tmp"), "nsm_canonical_scene.toml")
    with open(p, "w") as f:
        f.write(sk.cli._canonical_scene_text())
    scene, camera, _ = sk.scene.load_scene(p)
    em = scene.emitter
    sm = sk.raster.render_shadowmap(scene, em, (512, 512))
    g = sk.raster.render_gbuffer(scene, camera, em)
    for size in (0.0, 2.0):
        ref = sk.raster.assemble_features(g, sm, size)
        got = ours.assemble_features(g, sm, size)
        d = np.abs(got.data.astype(np.float64) - ref.data)
        print(f"canonical scene size {size}: features max-abs {d.max():.3g}")
        assert d.max() <= 1e-5
        assert got.bias == pytest.approx(ref.bias)
        np.testing.assert_array_equal(got.coverage, ref.coverage)
    row, col, _ = sm.view.project(np.moveaxis(g.position, 0, -1))
    idx = ours.texel_indices(g, sm)
    cov = g.coverage
    assert int((idx[0][cov] != np.rint(row)[cov]).sum() + (idx[1][cov] != np.rint(col)[cov]).sum()) == 0
