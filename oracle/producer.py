"""Oracle: ray-cast G-buffer and shadow-map passes (TEST INFRASTRUCTURE ONLY).

These produce the hot path's inputs. Restated from ``shadowkit``:

* primitive hits: Plane / Sphere / Box ``intersect`` (scene.py:218-326)
* nearest hit, first object wins ties (``Scene.intersect``, scene.py:430-441)
* ``EmitterView.texel_rays`` (raster.py:75-82), ``CameraPose.pixel_rays``
  (scene.py:153-163)
* ``render_shadowmap`` (raster.py:206-214) and the depth/normal/position part
  of ``render_gbuffer`` (raster.py:217-242)

Operates on :class:`paper_2301_05262_b200.scenes.SceneSpec` primitive
tables (kind + parameters), fp64 throughout. Small frames only.
"""

from __future__ import annotations

import numpy as np

from .features import camera_rays

KIND_PLANE, KIND_SPHERE, KIND_BOX = 0, 1, 2


def _hit_plane(row, o, d):
    p, n, u, v = row[1:4], row[4:7], row[7:10], row[10:13]
    su, sv = row[13], row[14]
    den = d @ n
    with np.errstate(divide="ignore", invalid="ignore"):
        t = ((p - o) @ n) / den
    t = np.where((np.abs(den) > 1e-12) & (t > 0.0), t, np.inf)
    hit = o + np.where(np.isfinite(t), t, 0.0)[..., None] * d
    inside = (np.abs((hit - p) @ u) <= su) & (np.abs((hit - p) @ v) <= sv)
    t = np.where(inside, t, np.inf)
    return t, np.broadcast_to(n, t.shape + (3,))


def _hit_sphere(row, o, d):
    c, r = row[1:4], row[4]
    oc = o - c
    b = np.sum(oc * d, axis=-1)
    disc = b * b - (np.sum(oc * oc, axis=-1) - r * r)
    s = np.sqrt(np.maximum(disc, 0.0))
    t = np.where(-b - s > 1e-12, -b - s, np.where(-b + s > 1e-12, -b + s, np.inf))
    t = np.where(disc >= 0.0, t, np.inf)
    return t, (o + t[..., None] * d - c) / r


def _hit_box(row, o, d):
    lo, hi = row[1:4], row[4:7]
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        a, b = (lo - o) * inv, (hi - o) * inv
    near, far = np.minimum(a, b), np.maximum(a, b)
    par = np.abs(d) < 1e-15
    ins = (o >= lo) & (o <= hi)
    near = np.where(par, np.where(ins, -np.inf, np.inf), near)
    far = np.where(par, np.where(ins, np.inf, -np.inf), far)
    tn, tf = near.max(axis=-1), far.min(axis=-1)
    t = np.where(tn > 1e-12, tn, tf)
    t = np.where((tf >= tn) & (t > 1e-12), t, np.inf)
    with np.errstate(invalid="ignore"):
        loc = (o + t[..., None] * d - (lo + hi) / 2.0) / ((hi - lo) / 2.0)
    ax = np.argmax(np.abs(loc), axis=-1)
    sgn = np.sign(np.take_along_axis(loc, ax[..., None], axis=-1))[..., 0]
    n = np.zeros(t.shape + (3,))
    np.put_along_axis(n, ax[..., None], np.where(sgn == 0.0, 1.0, sgn)[..., None], axis=-1)
    return t, n


_HIT = {KIND_PLANE: _hit_plane, KIND_SPHERE: _hit_sphere, KIND_BOX: _hit_box}


def nearest_hit(table, o, d):
    t = np.full(d.shape[:-1], np.inf)
    n = np.zeros(d.shape)
    o = np.broadcast_to(o, d.shape)
    for row in table:
        tk, nk = _HIT[int(row[0])](row, o, d)
        closer = tk < t
        t = np.where(closer, tk, t)
        n = np.where(closer[..., None], nk, n)
    return t, n


def texel_rays(view):
    hs, ws = view.resolution
    x = ((np.arange(ws) + 0.5) / ws * 2.0 - 1.0) * view.tan_half
    y = (1.0 - (np.arange(hs) + 0.5) / hs * 2.0) * view.tan_half
    r = (np.asarray(view.forward)[None, None, :] + x[None, :, None] * np.asarray(view.right)
         + y[:, None, None] * np.asarray(view.up))
    return r / np.linalg.norm(r, axis=-1, keepdims=True)


def render_shadowmap(table, view):
    t, _ = nearest_hit(table, np.asarray(view.position, dtype=np.float64), texel_rays(view))
    return t


def render_gbuffer(table, camera):
    """(d, normal(3,H,W), position(3,H,W)) with misses zeroed."""
    rays = camera_rays(camera)
    o = np.asarray(camera.position, dtype=np.float64)
    t, n = nearest_hit(table, o, rays)
    cov = np.isfinite(t)
    ts = np.where(cov, t, 0.0)
    pos = o + ts[..., None] * rays
    d = ts * (rays @ np.asarray(camera.forward))
    return d, np.moveaxis(n, -1, 0) * cov, np.moveaxis(pos, -1, 0) * cov


def _gbuf_band(args):
    table, camera, y0, y1 = args
    r = camera_rays(camera)[y0:y1]
    o = np.asarray(camera.position, dtype=np.float64)
    t, n = nearest_hit(table, o, r)
    cov = np.isfinite(t)
    ts = np.where(cov, t, 0.0)
    return (y0, (ts * (r @ np.asarray(camera.forward))).astype(np.float32),
            np.moveaxis(n * cov[..., None], -1, 0).astype(np.float32),
            np.moveaxis((o + ts[..., None] * r) * cov[..., None], -1, 0).astype(np.float32))


def _sm_band(args):
    table, view, y0, y1 = args
    return y0, nearest_hit(table, np.asarray(view.position, dtype=np.float64),
                           texel_rays(view)[y0:y1])[0].astype(np.float32)


def render_inputs_banded(table, camera, view, band=64, workers=None):
    """The hot path's fp32 input planes of one frame, rendered in row bands
    on a process pool (bounded memory at 1080p / 4K): d (H,W), normal
    (3,H,W), position (3,H,W), sm (Hs,Ws).  Used by bench.py's CPU
    reference leg, whose process must not load the CUDA library that
    renders them on the GPU."""
    import multiprocessing as mp
    import os
    h, w = camera.resolution
    hs, ws = view.resolution
    d = np.zeros((h, w), np.float32)
    nrm = np.zeros((3, h, w), np.float32)
    pos = np.zeros((3, h, w), np.float32)
    sm = np.empty((hs, ws), np.float32)
    jobs_g = [(table, camera, y, min(y + band, h)) for y in range(0, h, band)]
    jobs_s = [(table, view, y, min(y + band, hs)) for y in range(0, hs, band)]
    n = workers or max(1, len(os.sched_getaffinity(0)))
    with mp.get_context("fork").Pool(n) as pool:
        for y0, dd, nn, pp in pool.imap_unordered(_gbuf_band, jobs_g):
            d[y0:y0 + dd.shape[0]] = dd
            nrm[:, y0:y0 + dd.shape[0]] = nn
            pos[:, y0:y0 + dd.shape[0]] = pp
        for y0, ss in pool.imap_unordered(_sm_band, jobs_s):
            sm[y0:y0 + ss.shape[0]] = ss
    return {"d": d, "normal": nrm, "position": pos, "sm": sm}
