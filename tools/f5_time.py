"""Time nsm_features5 (fp16 hot-path output via nsm_infer of a 5-plane plan
is not needed: the 16-bit s2d writer is timed through ShadowInference's
per-kernel profile).  Experiment attribution: run with an experiment build
(NSM_BUILD_EXPERIMENTS=1) and NSM_F5_DBG=<mask>.  usage: python tools/f5_time.py [frames]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_05262_b200 import network, producer, scenes, _lib
from paper_2301_05262_b200.infer import ShadowInference
frames = scenes.config_frames(4, seed=0)
inp = producer.render_inputs(frames)
cfg = network.NetworkConfig(in_channels=5)
w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
run = ShadowInference(network.Plan(w, cfg, "fp16"), frames, out_dtype="fp16")
run.launch(inp)
torch.cuda.synchronize()
_lib.lib.nsm_profile_enable(1)
_lib.profile_report()
for _ in range(10):
    run.launch(inp, check=False)
torch.cuda.synchronize()
p = _lib.profile_report()
print(os.environ.get("NSM_F5_DBG", "0"), {k: round(v[1] / 10 * 1000, 1) for k, v in p.items() if k in ("feat5_blocker", "enc0_s2d")})
