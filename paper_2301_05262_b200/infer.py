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
    position (N,3,H,W), sm (N,Hs,Ws) -- fp32, contiguous, on the plan's
    device.  ``frames`` fixes N, (H, W) and (Hs, Ws); a launch may carry its
    own frames (cameras, emitter views, size index, bias) of the same shape.
    The executor owns its workspace, so executors sharing a plan may run on
    different streams concurrently.
    """

    def __init__(self, plan: Plan, frames, out_dtype: str = "fp32"):
        import torch
        self.plan = plan
        self.frames = list(frames)
        if not self.frames:
            raise ValueError("ShadowInference needs at least one frame")
        self.n = len(self.frames)
        self.h, self.w = self.frames[0].camera.resolution
        self.hs, self.ws_ = self.frames[0].view.resolution
        self._check_frames(self.frames)
        if out_dtype not in ("fp32", "fp16"):
            raise ValueError("out_dtype must be 'fp32' or 'fp16'")
        self.out_dtype = out_dtype
        self._fr = frame_params(self.frames)
        self.device = torch.device("cuda", plan.device)
        tdt = torch.float32 if out_dtype == "fp32" else torch.float16
        self.y = torch.empty((self.n, 1, self.h, self.w), dtype=tdt, device=self.device)
        self.first_bad = torch.empty(self.n, dtype=torch.int64, device=self.device)
        size = int(_lib.lib.nsm_workspace_size(plan.handle, self.n, self.h, self.w))
        self.ws = torch.empty(size, dtype=torch.uint8, device=self.device)
        self._graph = None
        self._gbuf = None

    def _check_frames(self, frames):
        if len(frames) != self.n:
            raise ValueError(f"executor is sized for {self.n} frames, got {len(frames)}")
        for i, f in enumerate(frames):
            if tuple(f.camera.resolution) != (self.h, self.w):
                raise ValueError(f"frame {i}: camera {tuple(f.camera.resolution)} != {(self.h, self.w)}")
            if tuple(f.view.resolution) != (self.hs, self.ws_):
                raise ValueError(f"frame {i}: shadow map {tuple(f.view.resolution)} != {(self.hs, self.ws_)}")

    def frame_table(self, frames):
        """Validated ctypes frame table for :meth:`launch` (build it once per
        batch of poses, reuse it across launches)."""
        frames = list(frames)
        self._check_frames(frames)
        return frame_params(frames)

    def check_inputs(self, inputs):
        """Raise ValueError unless ``inputs`` are fp32, contiguous, on this
        executor's device and shaped for its frames."""
        import torch
        want = {"d": (self.n, self.h, self.w), "normal": (self.n, 3, self.h, self.w),
                "position": (self.n, 3, self.h, self.w), "sm": (self.n, self.hs, self.ws_)}
        for k, shape in want.items():
            t = inputs.get(k)
            if t is None:
                raise ValueError(f"missing input plane {k!r}")
            if t.dtype != torch.float32 or not t.is_contiguous() or t.device != self.device:
                raise ValueError(f"input {k!r} must be a contiguous fp32 tensor on {self.device}")
            if tuple(t.shape) != shape:
                raise ValueError(f"input {k!r} has shape {tuple(t.shape)}, expected {shape}")

    def _gb(self, inputs):
        return _lib.GBufferC(_lib.NSM_F32, inputs["d"].data_ptr(), inputs["normal"].data_ptr(),
                             inputs["position"].data_ptr(), None, None, None, None,
                             self.h * self.w)

    def launch(self, inputs, stream=None, y=None, first_bad=None, frames=None, texel_idx=None,
               check=True):
        """Enqueue one step on ``stream`` (default: the current stream; no
        host sync).  ``y`` / ``first_bad`` override the executor's own
        output buffers (same shapes and dtypes).  ``frames``: this batch's
        frames (a list, or a table from :meth:`frame_table`); default the
        constructor's.  ``texel_idx``: optional (N, 2, H, W) int32 CUDA
        tensor receiving the fused pass's (row, col) texel of every covered
        pixel (nsm_infer_ex parity hook)."""
        import torch
        y = self.y if y is None else y
        first_bad = self.first_bad if first_bad is None else first_bad
        if check:
            self.check_inputs(inputs)
            if y.shape != self.y.shape or y.dtype != self.y.dtype or y.device != self.device:
                raise ValueError("y must match the executor's output buffer")
            if first_bad.shape != self.first_bad.shape or first_bad.dtype != torch.int64:
                raise ValueError("first_bad must be an int64 tensor of one entry per frame")
            if texel_idx is not None and (tuple(texel_idx.shape) != (self.n, 2, self.h, self.w)
                                          or texel_idx.dtype != torch.int32
                                          or texel_idx.device != self.device
                                          or not texel_idx.is_contiguous()):
                raise ValueError("texel_idx must be a contiguous (N, 2, H, W) int32 tensor")
        if frames is None:
            fr = self._fr
        elif isinstance(frames, C.Array):
            if len(frames) != self.n:
                raise ValueError(f"frame table has {len(frames)} frames, executor wants {self.n}")
            fr = frames
        else:
            fr = self.frame_table(frames)
        self._gbuf = self._gb(inputs)
        _lib.check(_lib.lib.nsm_infer_ex(
            self.plan.handle, C.byref(self._gbuf), inputs["sm"].data_ptr(), self.hs * self.ws_,
            fr, self.n, self.h, self.w, y.data_ptr(),
            _lib.NSM_F32 if self.out_dtype == "fp32" else _lib.NSM_F16,
            first_bad.data_ptr(), None if texel_idx is None else texel_idx.data_ptr(),
            self.ws.data_ptr(), self.ws.numel(), _lib.stream_ptr(stream)))
        return y

    def capture(self, inputs):
        """Capture one step into a CUDA graph bound to ``inputs``' buffers."""
        import torch
        self.check_inputs(inputs)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.launch(inputs)           # warm (allocs, attributes)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch(inputs, check=False)
        self._graph = g
        return g

    def replay(self):
        self._graph.replay()
        return self.y

    def check_frustum(self, first_bad=None, batch=None):
        """Raise FrustumError for the first frame with an out-of-frustum pixel."""
        fb = self.first_bad if first_bad is None else first_bad
        raise_first_bad(fb.cpu().numpy(), self.w, batch)

    def __call__(self, inputs, frames=None):
        y = self.launch(inputs, frames=frames)
        self.check_frustum()
        return y


def raise_first_bad(bad, w, batch=None):
    """FrustumError with the reference's message for the first frame whose
    first_bad entry is set (raster.py:251-255)."""
    for i, v in enumerate(np.asarray(bad)):
        if v != _lib.INT64_MAX:
            y, x = divmod(int(v), w)
            where = f"batch {batch} frame {i}" if batch is not None else f"frame {i}"
            raise _lib.FrustumError(
                f"{where}: covered pixel ({y}, {x}) projects outside the emitter frustum")


class HostPipeline:
    """Host-memory front end of :class:`ShadowInference`: batches of frames
    arrive in pinned host buffers and their visibility goes back to pinned
    host buffers, with the PCIe copies overlapped against the kernels.

    Three streams, ``slots`` device slots: the H2D copy of batch i+1, the
    fused kernels of batch i and the D2H copy of batch i-1 run concurrently
    (PCIe is full duplex).  Every batch may carry its own frames (poses,
    emitter views, size index, bias).  ``submit`` enqueues; before a slot is
    reused its previous batch's out-of-frustum record is checked, and
    ``synchronize`` drains and checks the rest, so a
    :class:`~paper_2301_05262_b200._lib.FrustumError` is raised for every
    offending batch (naming its submission index), never dropped.
    """

    def __init__(self, run: ShadowInference, slots: int = 2):
        import torch
        if slots < 1:
            raise ValueError("slots must be >= 1")
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
        self._batch = [None] * slots      # submission index held by each slot
        self._i = 0

    def _retire(self, s):
        """Wait for slot s's batch to drain and raise for its frustum errors."""
        b = self._batch[s]
        if b is None:
            return
        self.e_out[s].synchronize()
        self._batch[s] = None
        raise_first_bad(self.bad_host[s].numpy(), self.run.w, batch=b)

    def submit(self, host_inputs, host_y, frames=None):
        """Enqueue one batch: ``host_inputs`` as for ShadowInference (pinned
        CPU tensors), ``host_y`` a pinned CPU tensor shaped like ``run.y``,
        ``frames`` this batch's frames (list or ``run.frame_table``; default
        the executor's).  Reusing a slot first retires its previous batch:
        if that batch had an out-of-frustum pixel, FrustumError is raised
        and THIS batch is not enqueued (submit it again to continue)."""
        import torch
        s = self._i % self.slots
        self._retire(s)                 # the slot's previous batch (raises if it failed)
        table = None if frames is None else (
            frames if isinstance(frames, C.Array) else self.run.frame_table(frames))
        if self._dev[s] is None:
            self._dev[s] = {k: torch.empty(v.shape, dtype=v.dtype, device=self.run.device)
                            for k, v in host_inputs.items()}
        dev = self._dev[s]
        for k, v in host_inputs.items():
            if k not in dev or v.shape != dev[k].shape or v.dtype != dev[k].dtype:
                raise ValueError(f"host input {k!r} does not match the pipeline's slot buffers")
        if host_y.shape != self.run.y.shape or host_y.dtype != self.run.y.dtype:
            raise ValueError("host_y must match the executor's output shape and dtype")
        with torch.cuda.stream(self.h2d):
            for k, v in host_inputs.items():
                dev[k].copy_(v, non_blocking=True)
            self.e_in[s].record()
        self.comp.wait_event(self.e_in[s])
        self.run.launch(dev, stream=self.comp, y=self.y[s], first_bad=self.bad[s], frames=table)
        self.e_comp[s].record(self.comp)
        self.d2h.wait_event(self.e_comp[s])
        with torch.cuda.stream(self.d2h):
            host_y.copy_(self.y[s], non_blocking=True)
            self.bad_host[s].copy_(self.bad[s], non_blocking=True)
            self.e_out[s].record()
        self._batch[s] = self._i
        self._i += 1

    def synchronize(self):
        """Drain every slot; raise FrustumError for the earliest failed batch."""
        pending = sorted((b, s) for s, b in enumerate(self._batch) if b is not None)
        err = None
        for _, s in pending:
            try:
                self._retire(s)
            except _lib.FrustumError as e:
                err = err or e
        if err is not None:
            raise err
