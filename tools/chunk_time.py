"""Step time of config 4 (8 x 1080p, 4-plane fp16) through a CUDA graph, for
experiment builds (NSM_CHUNK_FRAMES etc.).  usage: python tools/chunk_time.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_05262_b200 import network, producer, scenes
from paper_2301_05262_b200.infer import ShadowInference
frames = scenes.config_frames(4, seed=0)
inp = producer.render_inputs(frames)
cfg = network.NetworkConfig()
w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
run = ShadowInference(network.Plan(w, cfg, "fp16"), frames, out_dtype="fp16")
run(inp)
run.capture(inp)
for _ in range(20):
    run.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record()
    for _ in range(20):
        run.replay()
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 20)
print(os.environ.get("NSM_CHUNK_FRAMES", "8"), "ms/step", round(best, 4), "frames/s", round(8 / best * 1e3))
