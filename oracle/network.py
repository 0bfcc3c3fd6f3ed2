"""Oracle: the compact U-Net forward pass (TEST INFRASTRUCTURE ONLY).

Restates the inference semantics of ``shadowkit/autodiff.py`` and
``shadowkit/network.py`` on (C, H, W) numpy arrays:

* ``conv``      -- autodiff.conv2d, im2col + one GEMM, zero pad (k-1)/2
                   (autodiff.py:137-166)
* ``pool2``     -- autodiff.avg_pool2 (autodiff.py:241-247)
* ``up2``       -- autodiff.bilinear_upsample2 with _upsample_taps
                   (autodiff.py:258-274): half-pixel centres, edge clamped
* ``s2d``/``d2s`` -- autodiff.space_to_depth / depth_to_space
                   (autodiff.py:290-320): channel 4c + 2dy + dx
* ``sigmoid``   -- autodiff.sigmoid, the two-branch stable form (:200-203)
* ``level_plan``/``forward`` -- network._level_plan / forward
                   (network.py:98-118, 165-209)

``dtype`` follows the input (fp32 oracle by default, fp64 for tight checks).
"""

from __future__ import annotations

import numpy as np
from numpy.lib.stride_tricks import as_strided


def level_channels(layers, base_channels, use_s2d=True, cap=256):
    n = layers - 1 if use_s2d else layers
    return [min(base_channels * 2 ** j, cap) for j in range(n)]


def level_plan(layers=5, base_channels=16, in_channels=4, use_s2d=True, cap=256):
    """Per-level (cin, cout) of enc3/enc1/dec3/dec1 plus the head pair."""
    ch = level_channels(layers, base_channels, use_s2d, cap)
    first = 4 * in_channels if use_s2d else in_channels
    plan = []
    for j, c in enumerate(ch):
        cin = first if j == 0 else ch[j - 1]
        if j == len(ch) - 1:
            plan.append({"enc3": (cin, c), "enc1": (c, ch[j - 1] if len(ch) > 1 else ch[0])})
        else:
            below = ch[j - 1] if j > 0 else ch[0]
            plan.append({"enc3": (cin, c), "enc1": (c, c), "dec3": (c, c), "dec1": (c, below)})
    return plan, (ch[0], 4 if use_s2d else 1)


def conv(x, w, b):
    """Cross-correlation with zero padding; w is OIHW."""
    o, i, k, _ = w.shape
    c, h, wd = x.shape
    p = (k - 1) // 2
    xp = np.pad(x, ((0, 0), (p, p), (p, p))) if p else x
    s0, s1, s2 = xp.strides
    cols = as_strided(xp, (c, k, k, h, wd), (s0, s1, s2, s1, s2)).reshape(c * k * k, h * wd)
    y = w.reshape(o, i * k * k) @ np.ascontiguousarray(cols)
    return y.reshape(o, h, wd) + b[:, None, None]


def relu(x):
    return np.maximum(x, 0)


def pool2(x):
    c, h, w = x.shape
    return x.reshape(c, h // 2, 2, w // 2, 2).mean(axis=(2, 4))


def _taps(n, dtype):
    src = np.clip((np.arange(2 * n) + 0.5) / 2.0 - 0.5, 0.0, n - 1.0)
    lo = np.floor(src).astype(np.int64)
    return lo, np.minimum(lo + 1, n - 1), (src - lo).astype(dtype)


def up2(x):
    c, h, w = x.shape
    r0, r1, rw = _taps(h, x.dtype)
    c0, c1, cw = _taps(w, x.dtype)
    rows = x[:, r0, :] * (1 - rw)[None, :, None] + x[:, r1, :] * rw[None, :, None]
    return rows[:, :, c0] * (1 - cw)[None, None, :] + rows[:, :, c1] * cw[None, None, :]


def s2d(x):
    c, h, w = x.shape
    return np.ascontiguousarray(x.reshape(c, h // 2, 2, w // 2, 2).transpose(0, 2, 4, 1, 3)
                                .reshape(4 * c, h // 2, w // 2))


def d2s(x):
    c4, h, w = x.shape
    return np.ascontiguousarray(x.reshape(c4 // 4, 2, 2, h, w).transpose(0, 3, 1, 4, 2)
                                .reshape(c4 // 4, 2 * h, 2 * w))


def sigmoid(x):
    e = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e)).astype(x.dtype)


def forward(weights, x, layers=5, base_channels=16, use_s2d=True, cap=256):
    """(C, H, W) -> (1, H, W) visibility; ``weights`` maps reference names
    (``l{j}.{enc3,enc1,dec3,dec1}.{w,b}``, ``head.{w,b}``) to arrays."""
    x = np.asarray(x)
    dt = x.dtype
    W = {k: np.asarray(getattr(v, "data", v), dtype=dt) for k, v in weights.items()}
    c, hh, ww = x.shape
    f = 2 ** (layers - 1)
    if hh % f or ww % f:
        raise ValueError(f"spatial dims {hh}x{ww} must be divisible by {f}")
    n = len(level_channels(layers, base_channels, use_s2d, cap))
    h = s2d(x) if use_s2d else x
    skips = []
    for j in range(n - 1):
        h = relu(conv(h, W[f"l{j}.enc3.w"], W[f"l{j}.enc3.b"]))
        h = relu(conv(h, W[f"l{j}.enc1.w"], W[f"l{j}.enc1.b"]))
        skips.append(h)
        h = pool2(h)
    j = n - 1
    h = relu(conv(h, W[f"l{j}.enc3.w"], W[f"l{j}.enc3.b"]))
    h = relu(conv(h, W[f"l{j}.enc1.w"], W[f"l{j}.enc1.b"]))
    for j in range(n - 2, -1, -1):
        h = up2(h)
        if j > 0:
            h = h + skips[j]
        h = relu(conv(h, W[f"l{j}.dec3.w"], W[f"l{j}.dec3.b"]))
        h = relu(conv(h, W[f"l{j}.dec1.w"], W[f"l{j}.dec1.b"]))
    y = conv(h, W["head.w"], W["head.b"])
    if not use_s2d:
        return sigmoid(y)
    detail = y.copy()
    detail[0] = 0
    return sigmoid(up2(y[:1]) + d2s(detail))
