"""fp16 / bf16 visibility error vs the fp32 oracle across weight seeds and
emitter sizes (1080p, 4-plane and 5-plane nets): how much headroom the
1e-2 max-abs bar has beyond the seeds the tests pin.
usage: python tools/seed_sweep.py [n_seeds]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle import blocker as ob, features as of, network as on
from paper_2301_05262_b200 import network, producer, scenes
from paper_2301_05262_b200.infer import ShadowInference

n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 6
for radius in (0.05, 0.5):
    fr = scenes.make_frame(scenes.random_scene(32, seed=11, emitter_radius_m=radius), (1080, 1920), (2048, 2048))
    inp = producer.render_inputs([fr])
    h = {k: v[0].cpu().numpy() for k, v in inp.items()}
    feats, cov = of.features_from_planes(h["d"], h["normal"], h["position"], h["sm"], fr.camera, fr.view,
                                         fr.scene.emitter_center, fr.size_index, fr.bias)
    z_f, _, _, _ = of.derive_planes(h["d"], h["normal"], h["position"], fr.camera, fr.scene.emitter_center)
    bp = ob.blocker_plane(h["d"], h["position"], z_f, cov, h["sm"], fr.view, fr.bias, fr.size_index,
                          fr.camera.focal_px)
    for planes in (4, 5):
        x = np.zeros((planes, 1088, 1920), np.float32)
        x[:4, :1080] = feats
        if planes == 5:
            x[4, :1080] = bp
        cfg = network.NetworkConfig(in_channels=planes)
        for seed in range(n_seeds):
            w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([seed, 0x11])))
            ref = on.forward({k: v.data for k, v in w.items()}, x)[0, :1080]
            out = []
            for dt in ("fp16", "bf16"):
                y = ShadowInference(network.Plan(w, cfg, dt), [fr], out_dtype="fp32")(inp)[0, 0].cpu().numpy()
                d = y.astype(np.float64) - ref
                out.append(f"{dt} max {np.abs(d).max():.2e} mse {np.mean(d * d):.1e}")
            print(f"size_index {fr.size_index:4.1f} planes {planes} seed {seed}: " + " | ".join(out), flush=True)
