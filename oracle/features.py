"""Oracle: the screen-space feature pass (TEST INFRASTRUCTURE ONLY).

Restates ``shadowkit/raster.py``:

* :func:`derive_planes`   -- the z_f / c_e / c_c / coverage derivation of
  ``render_gbuffer`` (raster.py:222-232, 237-241), applied to G-buffer planes
  that may have been rounded to fp32 (they are upcast to fp64 first).
* :func:`texel_coords`    -- ``EmitterView.project`` (raster.py:84-94).
* :func:`shadow_lookup`   -- ``_shadow_lookup`` (raster.py:245-263).
* :func:`assemble`        -- ``assemble_features`` (raster.py:266-278).
"""

from __future__ import annotations

import numpy as np


class FrustumError(RuntimeError):
    """raster.py:60-61."""


def camera_rays(camera) -> np.ndarray:
    """Unit pixel-centre rays (H, W, 3) -- scene.py:153-163."""
    h, w = camera.resolution
    th = np.tan(camera.fov_y / 2.0)
    tw = th * (w / h)
    u = ((np.arange(w) + 0.5) / w * 2.0 - 1.0) * tw
    v = (1.0 - (np.arange(h) + 0.5) / h * 2.0) * th
    right = np.cross(camera.forward, camera.up)
    rays = (np.asarray(camera.forward)[None, None, :]
            + u[None, :, None] * right[None, None, :]
            + v[:, None, None] * np.asarray(camera.up)[None, None, :])
    return rays / np.linalg.norm(rays, axis=-1, keepdims=True)


def derive_planes(d, normal, position, camera, emitter_center):
    """(z_f, c_e, c_c, coverage) from depth/normal/position planes.

    Coverage is ``d > 0`` (render_gbuffer zeroes d on misses and every hit has
    positive view depth). Arithmetic is fp64 as in raster.py:227-232.
    """
    d = np.asarray(d, dtype=np.float64)
    n = np.moveaxis(np.asarray(normal, dtype=np.float64), 0, -1)
    p = np.moveaxis(np.asarray(position, dtype=np.float64), 0, -1)
    cov = d > 0
    rays = camera_rays(camera)
    to_e = np.asarray(emitter_center, dtype=np.float64) - p
    z_f = np.linalg.norm(to_e, axis=-1)
    with np.errstate(divide="ignore", invalid="ignore"):
        c_e = np.clip(np.sum(n * (to_e / z_f[..., None]), axis=-1), 0.0, 1.0)
    c_c = np.clip(np.sum(n * -rays, axis=-1), 0.0, 1.0)
    for a in (z_f, c_e, c_c):
        a[~cov] = 0.0
    return z_f, c_e, c_c, cov


def texel_coords(view, points):
    """(row, col, forward depth) of world points in the map (raster.py:84-94)."""
    hs, ws = view.resolution
    rel = np.asarray(points, dtype=np.float64) - np.asarray(view.position)
    zc = rel @ np.asarray(view.forward)
    with np.errstate(divide="ignore", invalid="ignore"):
        denom = zc * view.tan_half
        xn = (rel @ np.asarray(view.right)) / denom
        yn = (rel @ np.asarray(view.up)) / denom
    return (1.0 - yn) / 2.0 * hs - 0.5, (xn + 1.0) / 2.0 * ws - 0.5, zc


def texel_indices(view, position, coverage):
    """Nearest texel (round-half-even, ``np.rint``) per pixel, plus the
    row-major index of the first covered pixel outside the frustum (or -1)."""
    hs, ws = view.resolution
    row, col, zc = texel_coords(view, np.moveaxis(np.asarray(position, dtype=np.float64), 0, -1))
    ri = np.rint(row).astype(np.int64)
    ci = np.rint(col).astype(np.int64)
    bad = coverage & ((ri < 0) | (ri >= hs) | (ci < 0) | (ci >= ws) | (zc <= 0))
    first = int(np.flatnonzero(bad.ravel())[0]) if bad.any() else -1
    return ri, ci, first


def shadow_lookup(position, z_f, coverage, sm_depth, view, bias):
    """Biased occluder depth; misses clamp to z_f (raster.py:245-263)."""
    hs, ws = view.resolution
    ri, ci, first = texel_indices(view, position, coverage)
    if first >= 0:
        y, x = divmod(first, coverage.shape[1])
        raise FrustumError(f"covered pixel ({y}, {x}) projects outside the emitter frustum")
    look = np.asarray(sm_depth, dtype=np.float64)[np.clip(ri, 0, hs - 1), np.clip(ci, 0, ws - 1)]
    occ = np.where(np.isfinite(look), np.minimum(look, z_f) + bias, z_f)
    return np.where(coverage, occ, 0.0)


def assemble(d, position, z_f, c_e, c_c, coverage, sm_depth, view, size_index, bias):
    """The 4 input planes (4, H, W) fp32 (raster.py:266-278)."""
    z = shadow_lookup(position, z_f, coverage, sm_depth, view, float(bias))
    with np.errstate(divide="ignore", invalid="ignore"):
        planes = [np.where(coverage, z - z_f, 0.0),
                  np.where(coverage, z / z_f, 0.0),
                  np.where(coverage, c_e + float(size_index), 0.0),
                  np.where(coverage, c_c / np.asarray(d, dtype=np.float64), 0.0)]
    return np.stack(planes).astype(np.float32)


def features_from_planes(d, normal, position, sm_depth, camera, view, emitter_center,
                         size_index, bias):
    """End-to-end stage 1 on raw planes: derive, then assemble."""
    z_f, c_e, c_c, cov = derive_planes(d, normal, position, camera, emitter_center)
    return assemble(d, position, z_f, c_e, c_c, cov, sm_depth, view, size_index, bias), cov
