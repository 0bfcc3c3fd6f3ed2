# Per-layer bf16 vs fp16 operand-rounding error budget of the U-Net
# (torch CPU emulation, fp32 accumulate) on the cfg1 golden features at
# size_index 0 and 8.  Run: PYTHONPATH=. python tools/bf16_error_budget.py
import numpy as np, torch, torch.nn.functional as F
from paper_2301_05262_b200 import network
r=np.load('tests/golden/cfg1.npz')
cfg=network.NetworkConfig()
w=network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0,0x11])))
W={k:torch.from_numpy(v.data) for k,v in w.items()}
def q(x,dt): return x if dt is None else x.to(dt).float()
def conv(x,name,dt):
    wt=W[name+'.w']; k=wt.shape[-1]
    return F.conv2d(q(x,dt), q(wt,dt), W[name+'.b'], padding=k//2)
def up(x): return F.interpolate(x, scale_factor=2, mode='bilinear', align_corners=False)
def fwd(x, pol):
    # pol: dict layer-> dtype; activations stored rounded at level outputs with pol['store_j']
    x=F.pixel_unshuffle(x[None],2)
    skips=[]; h=x
    for j in range(3):
        h=F.relu(conv(h,f'l{j}.enc3',pol.get(f'l{j}e')))
        h=F.relu(conv(h,f'l{j}.enc1',pol.get(f'l{j}e')))
        skips.append(h); h=F.avg_pool2d(h,2)
    h=F.relu(conv(h,'l3.enc3',pol.get('l3'))); h=F.relu(conv(h,'l3.enc1',pol.get('l3')))
    for j in (2,1,0):
        h=up(h)
        if j>0: h=h+skips[j]
        h=F.relu(conv(h,f'l{j}.dec3',pol.get(f'l{j}d'))); h=F.relu(conv(h,f'l{j}.dec1',pol.get(f'l{j}d')))
    y=conv(h,'head',pol.get('head'))
    base=up(y[:,0:1]); det=y.clone(); det[:,0]=0
    return torch.sigmoid(base+F.pixel_shuffle(det,2))[0,0]
x=torch.from_numpy(r['features'].copy()); cov=torch.from_numpy(r['d']>0)
bf=torch.bfloat16; hf=torch.float16
layers=['l0e','l1e','l2e','l3','l2d','l1d','l0d','head']
for s in [0.0, 8.0]:
    xs=x.clone(); xs[2][cov]+=s
    ref=fwd(xs,{})
    allbf={l:bf for l in layers}
    print('s',s,'all bf16', (fwd(xs,allbf)-ref).abs().max().item(), 'all fp16', (fwd(xs,{l:hf for l in layers})-ref).abs().max().item())
    for l in layers:
        p=dict(allbf); p[l]=hf
        only={l:bf}
        print('  ',l,'bf16 only here:', round((fwd(xs,only)-ref).abs().max().item(),5), ' all-bf16 but fp16 here:', round((fwd(xs,p)-ref).abs().max().item(),5))
