"""GPU producers of the hot path's inputs.

``render_inputs`` ray-casts, on the device, the camera G-buffer planes
(depth, normal, world position -- raster.render_gbuffer, raster.py:217-242)
and the light-space radial shadow map (raster.render_shadowmap,
raster.py:206-214) for a list of :class:`scenes.Frame`. These are untimed
supporting kernels: the CPU reference takes ~70 s per 1080p frame here.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .scenes import Frame


def render_inputs(frames: list[Frame], device="cuda"):
    """Batched planar inputs, all frames sharing one resolution.

    Returns dict(d=(N,H,W), normal=(N,3,H,W), position=(N,3,H,W),
    sm=(N,Hs,Ws)) fp32 CUDA tensors.
    """
    import torch
    h, w = frames[0].camera.resolution
    hs, ws = frames[0].view.resolution
    for f in frames:
        if f.camera.resolution != (h, w) or f.view.resolution != (hs, ws):
            raise ValueError("all frames of a batch must share camera / map resolution")
    n = len(frames)
    dev = torch.device(device)
    d = torch.empty((n, h, w), dtype=torch.float32, device=dev)
    nrm = torch.empty((n, 3, h, w), dtype=torch.float32, device=dev)
    pos = torch.empty((n, 3, h, w), dtype=torch.float32, device=dev)
    sm = torch.empty((n, hs, ws), dtype=torch.float32, device=dev)
    st = _lib.stream_ptr()
    tables = {}
    for i, f in enumerate(frames):
        key = id(f.scene)
        if key not in tables:
            tables[key] = torch.from_numpy(f.scene.primitive_table()).to(dev)
        tab = tables[key]
        cam = _lib.camera_c(f.camera)
        view = _lib.view_c(f.view)
        _lib.check(_lib.lib.nsm_render_gbuffer(tab.data_ptr(), tab.shape[0], C.byref(cam),
                                               d[i].data_ptr(), nrm[i].data_ptr(),
                                               pos[i].data_ptr(), st))
        _lib.check(_lib.lib.nsm_render_shadowmap(tab.data_ptr(), tab.shape[0], C.byref(view),
                                                 sm[i].data_ptr(), st))
    torch.cuda.current_stream().synchronize()
    return {"d": d, "normal": nrm, "position": pos, "sm": sm}


def frame_params(frames: list[Frame], size_index=None, bias=None):
    """ctypes frame table for nsm_infer / nsm_features."""
    return _lib.frames_c([(f.camera, f.view, f.scene.emitter_center,
                           f.size_index if size_index is None else size_index,
                           f.bias if bias is None else bias) for f in frames])


def to_host(inputs) -> dict:
    return {k: v.cpu().numpy() for k, v in inputs.items()}


def stack_numpy(planes) -> np.ndarray:
    return np.ascontiguousarray(planes)
