"""Oracle: motion vectors and temporal instability (TEST INFRASTRUCTURE ONLY).

Numpy restatement of the two temporal consumers of the path's output:

* :func:`motion_vectors` -- ``raster.motion_vectors`` (raster.py:330-358)
  with ``CameraPose.project`` (scene.py:165-183): frame t's world points
  reprojected with camera t-1; (row, col) offsets, zero on uncovered pixels;
  a pixel is valid when the rounded reprojection lands in bounds, in front of
  the camera, on covered geometry whose depth is within 1 % and whose normal
  agrees (dot >= 0.9, evaluated in the planes' precision).
* :func:`temporal_instability` -- ``analysis.temporal_instability``
  (analysis.py:350-377): mean of expm1(alpha |cur - prev[reprojected]|) over
  valid pixels of every consecutive pair.

Pinned on ``tests/golden/temporal.npz`` (reference outputs).
"""

from __future__ import annotations

import numpy as np


class NoValidPixels(RuntimeError):
    pass


def project(camera, points):
    """(row, col, depth) of world points (..., 3) -- scene.py:165-183."""
    h, w = camera.resolution
    half_h = np.tan(camera.fov_y / 2.0)
    half_w = half_h * (w / h)
    fwd = np.asarray(camera.forward, dtype=np.float64)
    up = np.asarray(camera.up, dtype=np.float64)
    right = np.cross(fwd, up)
    rel = np.asarray(points, dtype=np.float64) - np.asarray(camera.position, dtype=np.float64)
    zc = rel[..., 0] * fwd[0] + rel[..., 1] * fwd[1] + rel[..., 2] * fwd[2]
    xc = rel[..., 0] * right[0] + rel[..., 1] * right[1] + rel[..., 2] * right[2]
    yc = rel[..., 0] * up[0] + rel[..., 1] * up[1] + rel[..., 2] * up[2]
    with np.errstate(divide="ignore", invalid="ignore"):
        xn = xc / (zc * half_w)
        yn = yc / (zc * half_h)
    return (1.0 - yn) / 2.0 * h - 0.5, (xn + 1.0) / 2.0 * w - 0.5, zc


def motion_vectors(position_t, normal_t, cov_t, d_prev, normal_prev, cov_prev, camera_prev):
    """-> (vectors (2, H, W) fp64, valid (H, W) bool)."""
    h, w = cov_t.shape
    row, col, depth = project(camera_prev, np.moveaxis(np.asarray(position_t), 0, -1))
    ys, xs = np.mgrid[0:h, 0:w]
    vec = np.stack([row - ys, col - xs])
    vec[:, ~cov_t] = 0.0
    with np.errstate(invalid="ignore"):
        ri = np.where(np.isfinite(row), np.rint(row), -1).astype(np.int64)
        ci = np.where(np.isfinite(col), np.rint(col), -1).astype(np.int64)
    inb = (ri >= 0) & (ri < h) & (ci >= 0) & (ci < w) & (depth > 0)
    rs, cs = np.clip(ri, 0, h - 1), np.clip(ci, 0, w - 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.abs(np.asarray(d_prev)[rs, cs] - depth) / np.maximum(depth, 1e-12)
    nt, npv = np.asarray(normal_t), np.asarray(normal_prev)[:, rs, cs]
    nd = (nt[0] * npv[0] + nt[1] * npv[1]) + nt[2] * npv[2]
    ok = cov_t & inb & np.asarray(cov_prev)[rs, cs] & (rel <= 0.01) & (nd >= nd.dtype.type(0.9))
    return vec, ok


def temporal_instability(frames, vectors, valids, alpha_t=3.0):
    """-> (E, valid_pixels, rejected_fraction)."""
    if len(frames) < 2:
        raise ValueError("need at least two frames")
    if len(vectors) != len(frames) - 1:
        raise ValueError("need one motion field per consecutive frame pair")
    total, nvalid, npix = 0.0, 0, 0
    for t in range(1, len(frames)):
        cur = np.asarray(frames[t], dtype=np.float64)
        prev = np.asarray(frames[t - 1], dtype=np.float64)
        h, w = cur.shape
        ys, xs = np.mgrid[0:h, 0:w]
        v = vectors[t - 1]
        ri = np.clip(np.rint(ys + v[0]).astype(np.int64), 0, h - 1)
        ci = np.clip(np.rint(xs + v[1]).astype(np.int64), 0, w - 1)
        sel = np.asarray(valids[t - 1], dtype=bool)
        total += float(np.expm1(alpha_t * np.abs(cur - prev[ri, ci])[sel]).sum())
        nvalid += int(sel.sum())
        npix += cur.size
    if nvalid == 0:
        raise NoValidPixels("every pixel was rejected by reprojection tests")
    return total / nvalid, nvalid, 1.0 - nvalid / npix
