"""Temporal consumers of the visibility: motion vectors + instability on B200.

Drop-ins for ``shadowkit.raster.motion_vectors`` (raster.py:330-358) and
``shadowkit.analysis.temporal_instability`` (analysis.py:350-377) -- the
step ``cli eval-temporal`` runs on a sequence of network outputs
(cli.py:156-171). Both run in ``libnsm.so`` (nsm_motion_vectors /
nsm_temporal_instability); the ``*_batch`` forms keep a whole window
device-resident (e.g. the 8-frame config-4 window of ``bench.py``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["MotionField", "TemporalReport", "NoValidPixels", "motion_vectors",
           "motion_vectors_batch", "temporal_instability", "temporal_instability_batch"]


class NoValidPixels(RuntimeError):
    """Every pixel of every frame pair was rejected (analysis.py:68-69)."""


@dataclass(frozen=True)
class MotionField:
    """(dy, dx) pixel offsets mapping this frame to the previous one."""

    vectors: np.ndarray     # (2, H, W) fp64
    valid: np.ndarray       # bool (H, W)


@dataclass(frozen=True)
class TemporalReport:
    instability: float
    alpha_t: float
    frames_compared: int
    valid_pixels: int
    rejected_fraction: float

    def as_text(self) -> str:
        return (f"E={self.instability:.6g} alpha_t={self.alpha_t} "
                f"pairs={self.frames_compared} valid={self.valid_pixels} "
                f"rejected={100 * self.rejected_fraction:.2f}%")


def _gbuf_batch(d, normal, position, coverage=None):
    n, h, w = d.shape
    dt = _lib.NSM_F64 if str(d.dtype).endswith("float64") else _lib.NSM_F32
    return _lib.GBufferC(dt, d.data_ptr(), normal.data_ptr(), position.data_ptr(), None, None, None,
                         coverage.data_ptr() if coverage is not None else None, h * w)


def motion_vectors_batch(inputs, cameras):
    """inputs: CUDA tensors d (T,H,W), normal/position (T,3,H,W) (fp32 or
    fp64), optional uint8 coverage (T,H,W); cameras: the T frame cameras.
    Returns (vectors (T-1,2,H,W) fp64, valid (T-1,H,W) uint8) on the device:
    pair k maps frame k+1 into frame k."""
    import torch
    d = inputs["d"]
    t, h, w = d.shape
    cov = inputs.get("coverage")
    if cov is not None:
        cov = cov.to(torch.uint8).contiguous()
    gb = _gbuf_batch(d, inputs["normal"], inputs["position"], cov)
    cams = (_lib.CameraC * max(t - 1, 1))(*[_lib.camera_c(c) for c in cameras[:t - 1]])
    vec = torch.empty((max(t - 1, 0), 2, h, w), dtype=torch.float64, device=d.device)
    valid = torch.empty((max(t - 1, 0), h, w), dtype=torch.uint8, device=d.device)
    _lib.check(_lib.lib.nsm_motion_vectors(C.byref(gb), cams, t, h, w, vec.data_ptr(),
                                           valid.data_ptr(), _lib.stream_ptr()))
    return vec, valid


def motion_vectors(g_t, camera_prev, g_prev) -> MotionField:
    """Screen-space offsets mapping frame t pixels into frame t-1."""
    import torch
    if tuple(g_t.coverage.shape) != tuple(g_prev.coverage.shape):
        raise ValueError("motion vectors need equal resolutions")
    fdt = np.float64 if np.asarray(g_t.d).dtype == np.float64 else np.float32

    def two(a, b):
        return torch.from_numpy(np.ascontiguousarray(np.stack([a, b]), dtype=fdt)).cuda()

    inputs = {"d": two(g_prev.d, g_t.d), "normal": two(g_prev.normal, g_t.normal),
              "position": two(g_prev.position, g_t.position),
              "coverage": torch.from_numpy(np.stack([g_prev.coverage, g_t.coverage]).astype(np.uint8)).cuda()}
    vec, valid = motion_vectors_batch(inputs, [camera_prev, camera_prev])
    return MotionField(vectors=vec[0].cpu().numpy(), valid=valid[0].cpu().numpy().astype(bool))


def temporal_instability_batch(vis, vectors, valid, alpha_t: float = 3.0) -> TemporalReport:
    """vis: (T,H,W) fp32 CUDA; vectors/valid as from motion_vectors_batch."""
    import torch
    t = vis.shape[0]
    if t < 2:
        raise ValueError("need at least two frames")
    if vectors.shape[0] != t - 1:
        raise ValueError("need one motion field per consecutive frame pair")
    h, w = vis.shape[1:]
    vis = vis.to(torch.float32).contiguous()
    acc = torch.empty(t - 1, dtype=torch.float64, device=vis.device)
    cnt = torch.empty(t - 1, dtype=torch.int64, device=vis.device)
    _lib.check(_lib.lib.nsm_temporal_instability(vis.data_ptr(), vectors.contiguous().data_ptr(),
                                                 valid.to(torch.uint8).contiguous().data_ptr(), t, h, w,
                                                 float(alpha_t), acc.data_ptr(), cnt.data_ptr(),
                                                 _lib.stream_ptr()))
    total, n = float(acc.sum().item()), int(cnt.sum().item())
    if n == 0:
        raise NoValidPixels("every pixel was rejected by reprojection tests")
    return TemporalReport(instability=total / n, alpha_t=float(alpha_t), frames_compared=t - 1,
                          valid_pixels=n, rejected_fraction=1.0 - n / ((t - 1) * h * w))


def temporal_instability(frames, motions, alpha_t: float = 3.0) -> TemporalReport:
    """Exponentially penalized motion-compensated frame differences."""
    import torch
    if len(frames) < 2:
        raise ValueError("need at least two frames")
    if len(motions) != len(frames) - 1:
        raise ValueError("need one motion field per consecutive frame pair")
    vis = torch.stack([torch.as_tensor(np.asarray(f, dtype=np.float32)) for f in frames]).cuda()
    vec = torch.stack([torch.as_tensor(np.asarray(m.vectors, dtype=np.float64)) for m in motions]).cuda()
    valid = torch.stack([torch.as_tensor(np.asarray(m.valid, dtype=np.uint8)) for m in motions]).cuda()
    return temporal_instability_batch(vis, vec, valid, alpha_t)
