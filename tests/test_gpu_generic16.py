"""Generic 16-bit path (net_gen16.cu) for every NetworkConfig the
reference accepts that the level-fused kernels do not cover (needs a B200).

Against the reference's own network.forward outputs (tests/golden/nets.npz:
layers 2-6, in_channels 1/5, plain (no space-to-depth) mode, channel caps,
base 8) at the 16-bit bars of north_star: fp16 within 1e-2 max-abs and 1e-4
MSE; bf16 within the MSE bar (its max-abs is printed: bf16 keeps 8 mantissa
bits, see test_gpu_f16.py).  Plus the fused nsm_infer entry on a generic
plan vs the oracle (features -> layers=4 net)."""

import numpy as np
import pytest

from conftest import golden_nets, golden_camera, golden_view, load_golden

pytestmark = pytest.mark.gpu

NETS = golden_nets()


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("name", sorted(NETS))
def test_generic16_forward_matches_reference(name, dtype):
    from paper_2301_05262_b200 import network
    c = NETS[name]
    layers, base, inc, s2d, cap = (int(v) for v in c["cfg"])
    cfg = network.NetworkConfig(layers, base, inc, bool(s2d), cap)
    y = network.forward(c["w"], cfg, c["x"], dtype=dtype).data
    d = np.asarray(y, np.float64) - c["y"]
    mx, mse = float(np.abs(d).max()), float(np.mean(d * d))
    print(f"{name} {cfg} {dtype}: max {mx:.3g} mse {mse:.3g}")
    assert y.shape == c["y"].shape
    assert mse <= 1e-4
    if dtype == "fp16":
        assert mx <= 1e-2


def test_generic16_infer_layers4_vs_oracle(cfg1):
    """nsm_infer on a layers=4 fp16 plan (feature pass -> generic net ->
    crop) vs the oracle on the reference golden frame."""
    from types import SimpleNamespace
    import torch
    from oracle import network as on
    from paper_2301_05262_b200 import network
    from paper_2301_05262_b200.infer import ShadowInference
    r = cfg1
    cfg = network.NetworkConfig(layers=4)
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([2, 0x11])))
    fr = SimpleNamespace(camera=golden_camera(r), view=golden_view(r), size_index=float(r["size_index"]),
                         bias=float(r["bias"]), scene=SimpleNamespace(emitter_center=r["emitter_center"]))
    inp = {k: torch.from_numpy(np.ascontiguousarray(r[k][None])).cuda() for k in ("d", "normal", "position", "sm")}
    y = ShadowInference(network.Plan(w, cfg, "fp16"), [fr])(inp)[0, 0].cpu().numpy()
    ref = on.forward({k: v.data for k, v in w.items()}, r["features"], layers=4)[0]
    d = y.astype(np.float64) - ref
    print(f"layers=4 infer fp16: max {np.abs(d).max():.3g} mse {np.mean(d * d):.3g}")
    assert np.abs(d).max() <= 1e-2 and np.mean(d * d) <= 1e-4


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_generic16_batch_independent(dtype):
    """A batch through the generic path equals its frames one by one
    (bitwise), for a layers=6 plan (not covered by the fused kernels)."""
    import torch
    from paper_2301_05262_b200 import network
    cfg = network.NetworkConfig(layers=6, base_channels=8)
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([9, 0x11])))
    plan = network.Plan(w, cfg, dtype)
    g = torch.Generator().manual_seed(1)
    x = (torch.rand((3, 4, 64, 96), generator=g) * 2).cuda()
    yb = plan.forward(x).cpu().numpy()
    for i in range(3):
        np.testing.assert_array_equal(plan.forward(x[i:i + 1]).cpu().numpy()[0], yb[i])


def test_five_plane_window_two_chunks():
    """More frames than one chunk (8) through the 5-plane fused path: the
    per-chunk feat5 / enc0_s2d launches and the frame offsets of every
    output, against single-frame runs (bitwise)."""
    import torch
    from paper_2301_05262_b200 import network, producer, scenes
    from paper_2301_05262_b200.infer import ShadowInference
    cfg = network.NetworkConfig(in_channels=5)
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    plan = network.Plan(w, cfg, "fp16")
    frames = [scenes.make_frame(scenes.random_scene(8, seed=s, emitter_radius_m=0.1 + 0.02 * s), (64, 96),
                                (256, 256)) for s in range(10)]
    inp = producer.render_inputs(frames)
    yb = ShadowInference(plan, frames, out_dtype="fp16")(inp).cpu().clone()
    for i in (0, 7, 8, 9):
        one = {k: v[i:i + 1].contiguous() for k, v in inp.items()}
        y1 = ShadowInference(plan, [frames[i]], out_dtype="fp16")(one).cpu()
        torch.testing.assert_close(y1[0], yb[i], rtol=0, atol=0)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_generic16_plan_packing_is_deterministic(dtype):
    """Generic-path plans built over and over in a process whose freed host
    memory is poisoned (glibc MALLOC_PERTURB_) give bitwise the same output,
    within the MSE bar of the reference.  (Regression: the generic packer
    once read each conv's fp32 source through a pointer into the weight blob
    it was growing -- freed memory after the first reallocation; with the
    poisoning that fails every time instead of once in ~10 runs.)"""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = f"""
import sys
sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, "tests")!r})
import numpy as np, torch
from conftest import golden_nets
from paper_2301_05262_b200 import network
c = golden_nets()["l4_plain_in1"]
layers, base, inc, s2d, cap = (int(v) for v in c["cfg"])
cfg = network.NetworkConfig(layers, base, inc, bool(s2d), cap)
x = torch.from_numpy(np.ascontiguousarray(c["x"][None])).cuda()
first = None
junk = []
for i in range(24):
    junk.append(bytearray(4096 * (i % 7 + 1)))
    y = network.Plan(c["w"], cfg, {dtype!r}).forward(x).cpu().numpy()
    first = y if first is None else first
    assert np.array_equal(y, first), i
    if i % 3 == 2:
        junk.clear()
d = np.asarray(first[0], np.float64) - c["y"]
assert float(np.mean(d * d)) <= 1e-4, float(np.mean(d * d))
print("ok")
"""
    env = dict(os.environ, MALLOC_PERTURB_="165")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
