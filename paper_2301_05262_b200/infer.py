"""The fused hot path: G-buffer + shadow map -> visibility, batched on B200.

:class:`ShadowInference` is the torch-native entry point beside the numpy
drop-ins (``raster.assemble_features`` + ``network.forward``): one
``nsm_infer`` call per batch of frames, features never leave the chip on the
16-bit plans, optional CUDA-graph capture of the whole step.

Frames are independent (no cross-frame state at inference), so a batch is
sharded across GPUs by :mod:`paper_2301_05262_b200.shard`.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .network import NetworkConfig, Plan
from .producer import frame_params


class ShadowInference:
    """Per-device executor for batches of frames of one resolution.

    ``inputs``: dict of CUDA tensors d (N,H,W), normal (N,3,H,W),
    position (N,3,H,W), sm (N,Hs,Ws) -- fp32, contiguous.
    """

    def __init__(self, plan: Plan, frames, out_dtype: str = "fp32"):
        import torch
        self.plan = plan
        self.frames = list(frames)
        self.n = len(self.frames)
        self.h, self.w = self.frames[0].camera.resolution
        self.hs, self.ws_ = self.frames[0].view.resolution
        self.out_dtype = out_dtype
        self._fr = frame_params(self.frames)
        tdt = torch.float32 if out_dtype == "fp32" else torch.float16
        self.y = torch.empty((self.n, 1, self.h, self.w), dtype=tdt, device="cuda")
        self.first_bad = torch.empty(self.n, dtype=torch.int64, device="cuda")
        self.ws = plan.workspace(self.n, self.h, self.w)
        self._graph = None
        self._gbuf = None

    def _gb(self, inputs):
        return _lib.GBufferC(_lib.NSM_F32, inputs["d"].data_ptr(), inputs["normal"].data_ptr(),
                             inputs["position"].data_ptr(), None, None, None, None,
                             self.h * self.w)

    def launch(self, inputs, stream=None):
        """Enqueue one step on the current stream (no host sync)."""
        self._gbuf = self._gb(inputs)
        _lib.check(_lib.lib.nsm_infer(
            self.plan.handle, C.byref(self._gbuf), inputs["sm"].data_ptr(), self.hs * self.ws_,
            self._fr, self.n, self.h, self.w, self.y.data_ptr(),
            _lib.NSM_F32 if self.out_dtype == "fp32" else _lib.NSM_F16,
            self.first_bad.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
            _lib.stream_ptr(stream)))
        return self.y

    def capture(self, inputs):
        """Capture one step into a CUDA graph bound to ``inputs``' buffers."""
        import torch
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.launch(inputs)           # warm (allocs, attributes)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch(inputs)
        self._graph = g
        return g

    def replay(self):
        self._graph.replay()
        return self.y

    def check_frustum(self):
        """Raise FrustumError for the first frame with an out-of-frustum pixel."""
        bad = self.first_bad.cpu().numpy()
        for i, v in enumerate(bad):
            if v != _lib.INT64_MAX:
                y, x = divmod(int(v), self.w)
                raise _lib.FrustumError(
                    f"frame {i}: covered pixel ({y}, {x}) projects outside the emitter frustum")

    def __call__(self, inputs):
        y = self.launch(inputs)
        self.check_frustum()
        return y
