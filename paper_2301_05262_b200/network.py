"""Stage 2 drop-in: the compact U-Net of ``shadowkit/network.py`` on B200.

Host-side mirror of the reference module: ``NetworkConfig`` (network.py:44-76),
``receptive_field`` / ``layers_for_penumbra`` (:79-95), the level plan
(:98-118), ``init_weights`` (:121-144, same numpy draw order so a seeded rng
gives bit-identical weights), ``param_count`` / ``net_stats`` (:147-257),
``save_network`` / ``load_network`` (:260-285) and ``forward`` (:165-209).

``forward`` keeps the reference signature (weights dict, cfg, (C, H, W) array
or Tensor) and returns an object with ``.data`` of shape (1, H, W); the work
runs in ``libnsm.so`` (nsm_forward) through a :class:`Plan`, the plan layer
that packs the weights into the kernel layout once. Batched torch-native use
goes through :meth:`Plan.forward` / :meth:`Plan.infer` directly.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import math
from dataclasses import asdict, dataclass
from pathlib import Path

import numpy as np

from . import _lib
from . import fileio
from ._lib import FormatError

__all__ = ["NetworkConfig", "Tensor", "Plan", "receptive_field", "layers_for_penumbra",
           "init_weights", "forward", "net_stats", "param_count", "save_network",
           "load_network", "named_params", "level_plan"]

_DTYPES = {"fp32": _lib.NSM_F32, "fp16": _lib.NSM_F16, "bf16": _lib.NSM_BF16}
_PRECISION = {"fp32": "fp32 (reference precision, CUDA cores)",
              "fp16": "fp16 activations and weights, fp32 accumulate",
              "bf16": "bf16 activations and weights, fp32 accumulate"}


@dataclass(frozen=True)
class NetworkConfig:
    layers: int = 5
    base_channels: int = 16
    in_channels: int = 4
    use_space_to_depth: bool = True
    channel_cap: int = 256

    def __post_init__(self):
        if self.layers < 2:
            raise ValueError("network needs layers >= 2")
        if self.base_channels < 4:
            raise ValueError("base_channels must be >= 4")
        if self.in_channels < 1:
            raise ValueError("in_channels must be >= 1")

    @property
    def level_channels(self) -> tuple:
        n = self.layers - 1 if self.use_space_to_depth else self.layers
        return tuple(min(self.base_channels * 2 ** j, self.channel_cap) for j in range(n))

    @property
    def first_in_channels(self) -> int:
        return 4 * self.in_channels if self.use_space_to_depth else self.in_channels

    @property
    def out_channels(self) -> int:
        return 4 if self.use_space_to_depth else 1

    @property
    def downsample_factor(self) -> int:
        return 2 ** (self.layers - 1)


class Tensor:
    """Result container: ``.data`` holds the numpy array (autodiff.Tensor's
    read side; the GPU path is inference-only and keeps no graph)."""

    __slots__ = ("data",)

    def __init__(self, data):
        self.data = np.asarray(data)

    @property
    def shape(self):
        return self.data.shape

    @property
    def dtype(self):
        return self.data.dtype

    def __repr__(self):
        return f"Tensor(shape={self.data.shape}, dtype={self.data.dtype})"


def receptive_field(layers: int) -> int:
    """3 * 2**l pixels (Table 1 of the paper)."""
    if layers < 1:
        raise ValueError("layers must be >= 1")
    return 3 * 2 ** layers


def layers_for_penumbra(p_w: float) -> int:
    """Smallest l >= 2 with receptive_field(l) >= p_w."""
    if p_w < 1:
        raise ValueError("penumbra width must be >= 1 pixel")
    l = max(2, math.ceil(math.log2(p_w / 3.0)))
    while receptive_field(l) < p_w:
        l += 1
    while l > 2 and receptive_field(l - 1) >= p_w:
        l -= 1
    return l


def level_plan(cfg: NetworkConfig):
    """[{enc3, enc1[, dec3, dec1]: (cin, cout)}] per level, and the head pair."""
    ch = cfg.level_channels
    plan = []
    for j, c in enumerate(ch):
        cin = cfg.first_in_channels if j == 0 else ch[j - 1]
        if j == len(ch) - 1:
            plan.append({"enc3": (cin, c), "enc1": (c, ch[j - 1] if len(ch) > 1 else ch[0])})
        else:
            plan.append({"enc3": (cin, c), "enc1": (c, c), "dec3": (c, c),
                         "dec1": (c, ch[j - 1] if j > 0 else ch[0])})
    return plan, (ch[0], cfg.out_channels)


_TAGS = (("enc3", 3), ("enc1", 1), ("dec3", 3), ("dec1", 1))


def named_params(cfg: NetworkConfig):
    """(name, shape) of every parameter, in the reference's order."""
    plan, head = level_plan(cfg)
    for j, lev in enumerate(plan):
        for tag, k in _TAGS:
            if tag in lev:
                cin, cout = lev[tag]
                yield f"l{j}.{tag}.w", (cout, cin, k, k)
                yield f"l{j}.{tag}.b", (cout,)
    yield "head.w", (head[1], head[0], 1, 1)
    yield "head.b", (head[1],)


def init_weights(cfg: NetworkConfig, rng: np.random.Generator, dtype=np.float32) -> dict:
    """He-uniform U(+-sqrt(6 / (cin k^2))) weights, zero biases; identical
    draw order to the reference, so equal rng state -> identical arrays."""
    out = {}
    for name, shape in named_params(cfg):
        if name.endswith(".w"):
            cout, cin, k, _ = shape
            bound = math.sqrt(6.0 / (cin * k * k))
            out[name] = Tensor(rng.uniform(-bound, bound, size=shape).astype(dtype))
        else:
            out[name] = Tensor(np.zeros(shape, dtype=dtype))
    return out


def param_count(cfg: NetworkConfig) -> int:
    return int(sum(np.prod(s) for _, s in named_params(cfg)))


def net_stats(cfg: NetworkConfig, resolution=(128, 256)) -> list:
    """Analytic per-level parameters, MACs per full-res pixel and temporary
    storage traffic in pixels (network.py:212-257)."""
    plan, head = level_plan(cfg)
    h, w = resolution
    full = h * w
    shift = 1 if cfg.use_space_to_depth else 0
    stats = []
    for j, lev in enumerate(plan):
        r = (h >> (j + shift)) * (w >> (j + shift))
        params = macs = 0
        io = 0.0
        for tag, k in _TAGS:
            if tag in lev:
                cin, cout = lev[tag]
                params += cin * cout * k * k + cout
                macs += cin * cout * k * k * r
                io += (cin + cout) * r
        cj = lev["enc3"][1]
        if "dec3" in lev:
            io += cj * r + cj * r / 4 + cj * r / 4 + cj * r
            if j > 0:
                io += 3 * cj * r
        if j == 0:
            params += head[0] * head[1] + head[1]
            macs += head[0] * head[1] * r
            io += (head[0] + head[1]) * r
            if cfg.use_space_to_depth:
                io += r + full + 3 * r + full
        stats.append({"level": j, "resolution": (h >> (j + shift), w >> (j + shift)),
                      "parameters": params, "flops_per_pixel": macs / full,
                      "storage_io_pixels": io})
    return stats


def macs_per_pixel(cfg: NetworkConfig) -> float:
    """Total MACs per full-resolution pixel (sum of net_stats flops_per_pixel)."""
    return float(sum(s["flops_per_pixel"] for s in net_stats(cfg, (256, 256))))


def save_network(path, weights: dict, cfg: NetworkConfig) -> None:
    fileio.save_tensors(path, {k: getattr(v, "data", v) for k, v in weights.items()})
    Path(str(path) + ".json").write_text(json.dumps(asdict(cfg), indent=2, sort_keys=True) + "\n")


def load_network(path):
    arrays = fileio.load_tensors(path)
    cfg = NetworkConfig(**json.loads(Path(str(path) + ".json").read_text()))
    if set(arrays) != {k for k, _ in named_params(cfg)}:
        raise FormatError("checkpoint parameters do not match config")
    return {k: Tensor(v) for k, v in arrays.items()}, cfg


# ---------------------------------------------------------------------------
# Plan layer
# ---------------------------------------------------------------------------

def _arr(v):
    return np.ascontiguousarray(getattr(v, "data", v), dtype=np.float32)


def _cfg_c(cfg: NetworkConfig) -> _lib.NetConfig:
    return _lib.NetConfig(cfg.layers, cfg.base_channels, cfg.in_channels,
                          int(cfg.use_space_to_depth), cfg.channel_cap)


class Plan:
    """Device-resident packed weights for one (weights, cfg, dtype).

    ``dtype``: "fp32" (reference precision), "fp16" or "bf16" (16-bit
    operands, fp32 accumulation). Immutable; safe to share across threads
    that use distinct streams/workspaces.
    """

    def __init__(self, weights: dict, cfg: NetworkConfig, dtype: str = "fp32"):
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be one of {sorted(_DTYPES)}")
        self.cfg = cfg
        self.dtype = dtype
        names = list(weights)
        arrays = [_arr(weights[k]) for k in names]
        n = len(names)
        c_names = (C.c_char_p * n)(*[k.encode() for k in names])
        c_data = (C.c_void_p * n)(*[a.ctypes.data for a in arrays])
        c_nd = (C.c_int32 * n)(*[a.ndim for a in arrays])
        dims_keep = [(C.c_int32 * max(a.ndim, 1))(*a.shape) for a in arrays]
        c_dims = (C.POINTER(C.c_int32) * n)(*[C.cast(d, C.POINTER(C.c_int32)) for d in dims_keep])
        handle = C.POINTER(_lib.PlanHandle)()
        _lib.check(_lib.lib.nsm_plan_create(C.byref(_cfg_c(cfg)), n, c_names, c_data, c_nd,
                                            c_dims, _DTYPES[dtype], C.byref(handle)))
        self._h = handle
        self._ws = {}
        self.precision = _PRECISION[dtype]
        import torch
        self.device = torch.cuda.current_device()   # nsm_plan_create allocated here

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "lib", None) is not None:   # not at interpreter teardown
            _lib.lib.nsm_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def workspace(self, n: int, h: int, w: int, device=None, stream=None):
        """Scratch for nsm_forward / nsm_infer, cached per (device, stream):
        work enqueued on different streams never shares scratch memory."""
        import torch
        dev = torch.device("cuda", self.device) if device is None else torch.device(device)
        if dev.index is not None and dev.index != self.device:
            raise ValueError(f"plan lives on cuda:{self.device}, not {dev}")
        size = int(_lib.lib.nsm_workspace_size(self._h, n, h, w))
        key = (self.device, _lib.stream_ptr(stream))
        ws = self._ws.get(key)
        if ws is None or ws.numel() < size:
            ws = torch.empty(size, dtype=torch.uint8, device=torch.device("cuda", self.device))
            self._ws[key] = ws
        return ws

    def forward(self, x, out=None):
        """x: (N, C, H, W) fp32 CUDA tensor -> (N, 1, H, W) fp32."""
        import torch
        if x.dim() == 3:
            x = x[None]
        x = x.contiguous()
        if x.dtype != torch.float32 or not x.is_cuda:
            raise ValueError("Plan.forward wants an fp32 CUDA tensor")
        if x.device.index != self.device:
            raise ValueError(f"plan lives on cuda:{self.device}, input is on {x.device}")
        n, c, h, w = x.shape
        if c != self.cfg.in_channels:
            raise ValueError(f"input has {c} channels, config wants {self.cfg.in_channels}")
        y = torch.empty((n, 1, h, w), dtype=torch.float32, device=x.device) if out is None else out
        ws = self.workspace(n, h, w, x.device)
        _lib.check(_lib.lib.nsm_forward(self._h, x.data_ptr(), n, h, w, y.data_ptr(),
                                        ws.data_ptr(), ws.numel(), _lib.stream_ptr()))
        return y


_PLAN_CACHE: dict = {}


def _fingerprint(weights) -> str:
    h = hashlib.blake2b(digest_size=16)
    for k in sorted(weights):
        a = _arr(weights[k])
        h.update(k.encode())
        h.update(a.tobytes())
    return h.hexdigest()


def plan_for(weights: dict, cfg: NetworkConfig, dtype: str = "fp32") -> Plan:
    """Cached plan keyed by the weights' content (weights may be mutated
    between calls by training code; a content change re-packs)."""
    import torch
    key = (cfg, dtype, torch.cuda.current_device(), _fingerprint(weights))
    p = _PLAN_CACHE.get(key)
    if p is None:
        if len(_PLAN_CACHE) > 16:
            _PLAN_CACHE.clear()
        p = _PLAN_CACHE[key] = Plan(weights, cfg, dtype)
    return p


def forward(weights: dict, cfg: NetworkConfig, x, dtype: str = "fp32") -> Tensor:
    """Run the network on a (in_channels, H, W) input; output is (1, H, W).

    Same contract and errors as network.forward (network.py:165-173); the
    computation runs on the GPU (nsm_forward). ``dtype`` selects the plan
    precision (default: the reference's fp32).
    """
    import torch
    a = np.asarray(getattr(x, "data", x), dtype=np.float32)
    if a.ndim != 3:
        raise ValueError(f"forward expects (channels, height, width), got {a.shape}")
    c, hh, ww = a.shape
    if c != cfg.in_channels:
        raise ValueError(f"input has {c} channels, config wants {cfg.in_channels}")
    f = cfg.downsample_factor
    if hh % f or ww % f:
        raise ValueError(f"spatial dims {hh}x{ww} must be divisible by {f}")
    plan = plan_for(weights, cfg, dtype)
    xd = torch.from_numpy(np.ascontiguousarray(a)).to(torch.device("cuda", plan.device))
    y = plan.forward(xd[None])
    return Tensor(y[0].cpu().numpy())
