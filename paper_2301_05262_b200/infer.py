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

    def launch(self, inputs, stream=None, y=None, first_bad=None):
        """Enqueue one step on ``stream`` (default: the current stream; no
        host sync).  ``y`` / ``first_bad`` override the executor's own
        output buffers (same shapes and dtypes)."""
        y = self.y if y is None else y
        first_bad = self.first_bad if first_bad is None else first_bad
        self._gbuf = self._gb(inputs)
        _lib.check(_lib.lib.nsm_infer(
            self.plan.handle, C.byref(self._gbuf), inputs["sm"].data_ptr(), self.hs * self.ws_,
            self._fr, self.n, self.h, self.w, y.data_ptr(),
            _lib.NSM_F32 if self.out_dtype == "fp32" else _lib.NSM_F16,
            first_bad.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
            _lib.stream_ptr(stream)))
        return y

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


class HostPipeline:
    """Host-memory front end of :class:`ShadowInference`: batches of frames
    arrive in pinned host buffers and their visibility goes back to pinned
    host buffers, with the PCIe copies overlapped against the kernels.

    Three streams, two device slots: the H2D copy of batch i+1, the fused
    kernels of batch i and the D2H copy of batch i-1 run concurrently (PCIe is
    full duplex).  ``submit`` only enqueues; ``synchronize`` drains and raises
    :class:`~paper_2301_05262_b200._lib.FrustumError` like
    ``ShadowInference.__call__`` for any batch with an out-of-frustum pixel.
    """

    def __init__(self, run: ShadowInference, slots: int = 2):
        import torch
        self.run = run
        self.slots = slots
        self.h2d = torch.cuda.Stream()
        self.comp = torch.cuda.Stream()
        self.d2h = torch.cuda.Stream()
        self._dev = [None] * slots
        self.y = [torch.empty_like(run.y) for _ in range(slots)]
        self.bad = [torch.empty_like(run.first_bad) for _ in range(slots)]
        self.bad_host = [torch.empty(run.first_bad.shape, dtype=torch.int64, pin_memory=True)
                         for _ in range(slots)]
        ev = lambda: [torch.cuda.Event() for _ in range(slots)]   # noqa: E731
        self.e_in, self.e_comp, self.e_out = ev(), ev(), ev()
        self._used = [False] * slots
        self._i = 0

    def submit(self, host_inputs, host_y):
        """Enqueue one batch: ``host_inputs`` as for ShadowInference (pinned
        CPU tensors), ``host_y`` a pinned CPU tensor shaped like ``run.y``."""
        import torch
        s = self._i % self.slots
        if self._dev[s] is None:
            self._dev[s] = {k: torch.empty(v.shape, dtype=v.dtype, device="cuda")
                            for k, v in host_inputs.items()}
        dev = self._dev[s]
        if self._used[s]:
            self.h2d.wait_event(self.e_comp[s])      # slot's inputs consumed
            self.comp.wait_event(self.e_out[s])      # slot's outputs drained
        with torch.cuda.stream(self.h2d):
            for k, v in host_inputs.items():
                dev[k].copy_(v, non_blocking=True)
            self.e_in[s].record()
        self.comp.wait_event(self.e_in[s])
        self.run.launch(dev, stream=self.comp, y=self.y[s], first_bad=self.bad[s])
        self.e_comp[s].record(self.comp)
        self.d2h.wait_event(self.e_comp[s])
        with torch.cuda.stream(self.d2h):
            host_y.copy_(self.y[s], non_blocking=True)
            self.bad_host[s].copy_(self.bad[s], non_blocking=True)
            self.e_out[s].record()
        self._used[s] = True
        self._i += 1

    def synchronize(self):
        for s in range(self.slots):
            if self._used[s]:
                self.e_out[s].synchronize()
                bad = self.bad_host[s].numpy()
                for i, v in enumerate(bad):
                    if v != _lib.INT64_MAX:
                        y, x = divmod(int(v), self.run.w)
                        raise _lib.FrustumError(
                            f"frame {i}: covered pixel ({y}, {x}) projects outside the emitter frustum")
