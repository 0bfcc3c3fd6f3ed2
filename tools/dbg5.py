"""Debug dump of nsm_features5's per-pixel blocker search vs the oracle on a
config-3 frame.  Needs an experiment build (NSM_BUILD_EXPERIMENTS=1): the
nsm_debug_feat5 hook is not in the release library."""
import sys, numpy as np, torch, ctypes as C
sys.path.insert(0, '.')
from paper_2301_05262_b200 import producer, scenes, _lib
from paper_2301_05262_b200.raster import assemble_features5_batch
from oracle import features as of, blocker as ob
fr = scenes.config_frames(3, seed=0)[0]
inp = producer.render_inputs([fr])
dbg = torch.zeros((1, 1080, 1920, 4), dtype=torch.int32, device="cuda")
_lib.lib.nsm_debug_feat5.argtypes = [C.c_void_p]
_lib.lib.nsm_debug_feat5(dbg.data_ptr())
got, idx, _ = assemble_features5_batch(inp, [(fr.camera, fr.view, fr.scene.emitter_center, fr.size_index, fr.bias)], want_idx=True)
_lib.lib.nsm_debug_feat5(None)
g4 = got[0, 4].cpu().numpy(); D = dbg[0].cpu().numpy(); I = idx[0].cpu().numpy()
h = {k: v[0].cpu().numpy() for k, v in inp.items()}
z_f, _, _, cov = of.derive_planes(h["d"], h["normal"], h["position"], fr.camera, fr.scene.emitter_center)
r4 = ob.blocker_plane(h["d"], h["position"], z_f, cov, h["sm"], fr.view, fr.bias, fr.size_index, fr.camera.focal_px)
ri, ci, _ = of.texel_indices(fr.view, h["position"], cov)
smi = h["sm"].astype(np.float32).view(np.int32)
bad = np.argwhere((g4 > 0) != (r4 > 0))
print(len(bad))
for y, x in bad[:10]:
    r, c = ri[y, x], ci[y, x]
    W = smi[max(r-8,0):r+8, max(c-8,0):c+8].ravel()
    t = D[y, x, 2]
    bl = W[W < t]
    print(y, x, "idx", I[:, y, x], (r, c), "gpu zmin/zmax/thr/path", D[y, x], "exact zmin", W.min(), "zmax", bl.max() if len(bl) else -1)
P = D[..., 3][cov]
print("covered", cov.sum(), "not staged", (P & 1).mean(), "alone", ((P & 2) > 0).mean(), "owners", ((P & 4) > 0).mean(), "cluster1", ((P >> 3) & 1).mean())
ns = np.argwhere(cov & ((D[..., 3] & 1) == 1))
print("not staged sample", [(int(y), int(x), int(I[0, y, x]), int(I[1, y, x])) for y, x in ns[:8]])
tiles = {}
for y, x in ns:
    tiles.setdefault((y // 16, x // 64), 0)
    tiles[(y // 16, x // 64)] += 1
print("tiles", len(tiles), sorted(tiles.items(), key=lambda kv: -kv[1])[:6])
t0 = sorted(tiles.items(), key=lambda kv: -kv[1])[0][0]
m = cov[t0[0]*16:(t0[0]+1)*16, t0[1]*64:(t0[1]+1)*64]
rr = I[0, t0[0]*16:(t0[0]+1)*16, t0[1]*64:(t0[1]+1)*64][m]; cc = I[1, t0[0]*16:(t0[0]+1)*16, t0[1]*64:(t0[1]+1)*64][m]
print("tile", t0, "covered", m.sum(), "rows", rr.min(), rr.max(), "cols", cc.min(), cc.max())
