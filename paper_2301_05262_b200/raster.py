"""Stage 1 drop-in: ``shadowkit.raster.assemble_features`` on B200.

Same signature, semantics and errors as the reference (raster.py:245-283):
the 4 feature planes ch0 = z - z_f, ch1 = z / z_f, ch2 = c_e + size_index,
ch3 = c_c / d with the biased nearest-texel shadow lookup, uncovered pixels
zeroed, ``FrustumError`` for the first covered pixel (row-major) that projects
outside the emitter frustum. The work runs in ``libnsm.so`` (nsm_features);
texel indices are computed in fp64 with round-half-even, so they are
bit-identical to the reference's ``np.rint``.

The container types mirror the reference's dataclasses field for field, so
reference ``GBuffer`` / ``ShadowMap`` objects can be passed in unchanged.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from ._lib import FrustumError
from .scenes import DEFAULT_BIAS_FACTOR, CameraPose, EmitterView

__all__ = ["FrustumError", "GBuffer", "ShadowMap", "FeatureStack", "EmitterView",
           "assemble_features", "hard_shadow_mask", "FEATURE_CHANNELS", "texel_indices"]

FEATURE_CHANNELS = ("z-z_f", "z/z_f", "c_e", "c_c/d")


@dataclass(frozen=True)
class ShadowMap:
    """Radial emitter-space depth per texel; +inf marks background."""

    depth: np.ndarray
    view: EmitterView
    scene_diag: float

    @property
    def resolution(self):
        return self.view.resolution

    @property
    def default_bias(self) -> float:
        return DEFAULT_BIAS_FACTOR * self.scene_diag


@dataclass(frozen=True)
class GBuffer:
    """Per-pixel nearest-hit attributes (raster.py:154-170)."""

    d: np.ndarray
    normal: np.ndarray
    position: np.ndarray
    n_e: np.ndarray | None
    z_f: np.ndarray
    c_e: np.ndarray
    c_c: np.ndarray
    coverage: np.ndarray
    camera: CameraPose

    @property
    def resolution(self):
        return self.coverage.shape


@dataclass(frozen=True)
class FeatureStack:
    """The 4 network input channels plus coverage; fp32 at camera resolution."""

    data: np.ndarray
    size_index: float
    coverage: np.ndarray
    bias: float

    def __post_init__(self):
        if self.data.shape[0] != 4 or self.data.ndim != 3:
            raise ValueError(f"feature stack wants (4, H, W), got {self.data.shape}")

    @property
    def resolution(self):
        return self.data.shape[1:]

    def with_size_index(self, size_index: float) -> "FeatureStack":
        """Re-target the softness dc offset on channel 2 (raster.py:190-195)."""
        data = self.data.copy()
        data[2][self.coverage] += np.float32(size_index - self.size_index)
        return replace(self, data=data, size_index=float(size_index))


def _dev(a, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def _run_features(g, sm, size_index, bias, want_idx=False):
    import torch
    d = np.asarray(g.d)
    fdt = np.float64 if d.dtype == np.float64 else np.float32
    h, w = d.shape
    keep = {k: _dev(getattr(g, k), fdt) for k in ("d", "position", "z_f", "c_e", "c_c")}
    keep["coverage"] = _dev(np.asarray(g.coverage, dtype=np.uint8), np.uint8)
    keep["normal"] = _dev(g.normal, fdt)
    smd = _dev(sm.depth, np.float32)
    gb = _lib.GBufferC(_lib.NSM_F64 if fdt == np.float64 else _lib.NSM_F32,
                       keep["d"].data_ptr(), keep["normal"].data_ptr(),
                       keep["position"].data_ptr(), keep["z_f"].data_ptr(),
                       keep["c_e"].data_ptr(), keep["c_c"].data_ptr(),
                       keep["coverage"].data_ptr(), h * w)
    frames = _lib.frames_c([(g.camera, sm.view, (0.0, 0.0, 0.0), size_index, bias)])
    out = torch.empty((1, 4, h, w), dtype=torch.float32, device="cuda")
    idx = torch.empty((1, 2, h, w), dtype=torch.int32, device="cuda") if want_idx else None
    bad = torch.empty(1, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib.nsm_features(C.byref(gb), smd.data_ptr(), 0, frames, 1, h, w,
                                     out.data_ptr(), idx.data_ptr() if want_idx else None,
                                     bad.data_ptr(), _lib.stream_ptr()))
    first = int(bad.item())
    if first != _lib.INT64_MAX:
        y, x = divmod(first, w)
        raise FrustumError(f"covered pixel ({y}, {x}) projects outside the emitter frustum")
    return out[0].cpu().numpy(), (idx[0].cpu().numpy() if want_idx else None)


def assemble_features(g, sm, size_index: float, bias: float | None = None) -> FeatureStack:
    """Derive the 4 input channels from a G-buffer and a shadow map."""
    b = sm.default_bias if bias is None else float(bias)
    data, _ = _run_features(g, sm, float(size_index), b)
    return FeatureStack(data=data, size_index=float(size_index),
                        coverage=np.asarray(g.coverage, dtype=bool), bias=b)


def texel_indices(g, sm) -> np.ndarray:
    """(2, H, W) int32 nearest (row, col) texel per pixel, -1 where uncovered
    -- the integer half of ``_shadow_lookup`` (raster.py:247-250)."""
    _, idx = _run_features(g, sm, 0.0, sm.default_bias, want_idx=True)
    return idx


def assemble_features_batch(inputs, frames, want_idx=False, check=True):
    """Torch-native batched stage 1 on device-resident planes.

    inputs: dict of fp32 CUDA tensors d (N,H,W), normal (N,3,H,W),
    position (N,3,H,W), sm (N,Hs,Ws); frames: N tuples (camera, view,
    emitter_center, size_index, bias). z_f / c_e / c_c and coverage are
    derived on the fly (raster.py:222-232). Returns (features (N,4,H,W),
    texel indices (N,2,H,W) or None, first_bad (N,) int64 device tensor).
    """
    import torch
    d = inputs["d"]
    n, h, w = d.shape
    hs, ws = inputs["sm"].shape[1:]
    gb = _lib.GBufferC(_lib.NSM_F32, d.data_ptr(), inputs["normal"].data_ptr(),
                       inputs["position"].data_ptr(), None, None, None, None, h * w)
    fr = _lib.frames_c(frames)
    out = torch.empty((n, 4, h, w), dtype=torch.float32, device=d.device)
    idx = torch.empty((n, 2, h, w), dtype=torch.int32, device=d.device) if want_idx else None
    bad = torch.empty(n, dtype=torch.int64, device=d.device)
    _lib.check(_lib.lib.nsm_features(C.byref(gb), inputs["sm"].data_ptr(), hs * ws, fr, n, h, w,
                                     out.data_ptr(), idx.data_ptr() if want_idx else None,
                                     bad.data_ptr(), _lib.stream_ptr()))
    if check:
        for i, v in enumerate(bad.cpu().tolist()):
            if v != _lib.INT64_MAX:
                y, x = divmod(int(v), w)
                raise FrustumError(f"covered pixel ({y}, {x}) projects outside the emitter frustum")
    return out, idx, bad


def blocker_penumbra_batch(inputs, frames, radius: int = 8, check=True):
    """Blocker-search penumbra-width plane (N, H, W) fp32 -- the 5th input
    plane of BASELINE configs 3/4 (a build extension: the reference has no
    blocker search; see include/nsm.h nsm_blocker_plane and oracle/blocker.py):
    the penumbra's screen width in units of the focal length, (x_a + x_b) / d.
    ``frames`` as for :func:`assemble_features_batch`; size_index sets the
    emitter radius (0.0625 m per unit, scene.py:54-58)."""
    import torch
    d = inputs["d"]
    n, h, w = d.shape
    hs, ws = inputs["sm"].shape[1:]
    gb = _lib.GBufferC(_lib.NSM_F32, d.data_ptr(), inputs["normal"].data_ptr(),
                       inputs["position"].data_ptr(), None, None, None, None, h * w)
    out = torch.empty((n, h, w), dtype=torch.float32, device=d.device)
    bad = torch.empty(n, dtype=torch.int64, device=d.device)
    _lib.check(_lib.lib.nsm_blocker_plane(C.byref(gb), inputs["sm"].data_ptr(), hs * ws,
                                          _lib.frames_c(frames), n, h, w, int(radius),
                                          out.data_ptr(), bad.data_ptr(), _lib.stream_ptr()))
    if check:
        for v in bad.cpu().tolist():
            if v != _lib.INT64_MAX:
                y, x = divmod(int(v), w)
                raise FrustumError(f"covered pixel ({y}, {x}) projects outside the emitter frustum")
    return out


def assemble_features5_batch(inputs, frames, want_idx=False, check=True):
    """The 5-plane feature pass of NetworkConfig(in_channels=5) nets (BASELINE
    configs 3/4): the 4 planes of :func:`assemble_features_batch` (fp32
    arithmetic of the fused hot path) and the 16x16 blocker-search penumbra
    plane, computed with the map windows staged in shared memory
    (nsm_features5).  Returns (features (N,5,H,W), texel indices or None,
    first_bad)."""
    import torch
    d = inputs["d"]
    n, h, w = d.shape
    hs, ws = inputs["sm"].shape[1:]
    gb = _lib.GBufferC(_lib.NSM_F32, d.data_ptr(), inputs["normal"].data_ptr(),
                       inputs["position"].data_ptr(), None, None, None, None, h * w)
    out = torch.empty((n, 5, h, w), dtype=torch.float32, device=d.device)
    idx = torch.full((n, 2, h, w), -1, dtype=torch.int32, device=d.device) if want_idx else None
    bad = torch.empty(n, dtype=torch.int64, device=d.device)
    _lib.check(_lib.lib.nsm_features5(C.byref(gb), inputs["sm"].data_ptr(), hs * ws, _lib.frames_c(frames),
                                      n, h, w, out.data_ptr(), idx.data_ptr() if want_idx else None,
                                      bad.data_ptr(), _lib.stream_ptr()))
    if check:
        for v in bad.cpu().tolist():
            if v != _lib.INT64_MAX:
                y, x = divmod(int(v), w)
                raise FrustumError(f"covered pixel ({y}, {x}) projects outside the emitter frustum")
    return out, idx, bad


def hard_shadow_mask(stack: FeatureStack) -> np.ndarray:
    """Point-light shadow test (raster.py:281-283)."""
    return (stack.data[0] < 0.0) & stack.coverage
