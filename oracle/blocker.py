"""Oracle: blocker-search penumbra plane (TEST INFRASTRUCTURE ONLY).

BUILD EXTENSION -- PARITY UNPINNED. The reference has no blocker search
(PCSS is out of scope); BASELINE configs 3/4 ask for a
"blocker-search penumbra estimate" plane feeding the same U-Net. This is the
definition the CUDA kernels (csrc/features.cu blocker_kernel, csrc/feat5.cu) implement, restated here in
numpy, built from reference pieces:

1. nearest texel (ri, ci) exactly as ``_shadow_lookup`` (raster.py:247-250)
2. window rows ri-R .. ri+R-1, cols ci-R .. ci+R-1 (R = 8: 16x16 texels),
   clipped to the map
3. blockers: finite texels with depth < z_f - b (the "in shadow" test of
   raster.py:259-262)
4. (z_min, z_max) over blockers -> ``analysis.penumbra_extents`` with the
   emitter radius r_e (analysis.py:240-269; its ValueError cases give 0 here,
   pre-masked as penumbra_histogram does, analysis.py:313)
5. screen width (x_a + x_b) * focal_px / d (analysis.py:319-320), divided by
   focal_px: the plane is the penumbra's screen width in units of the focal
   length, (x_a + x_b) / d -- resolution independent and O(0.1).  In pixels
   (up to ~130 at 1080p, size_index ~7) the plane drove the first layers'
   activations of a random-init in_channels=5 net to ~100, where fp16's
   absolute rounding (ulp 0.06) put the 16-bit visibility 0.10 max-abs off
   the fp32 oracle (north_star's bar: 1e-2); 0 where there are no blockers,
   uncovered pixels, or a point light.
"""

from __future__ import annotations

import math

import numpy as np

from .features import texel_indices

SIZE_TO_RADIUS = 0.5 / 2.0 / 4.0          # scene.emitter_radius slope (scene.py:54-58)


def penumbra_widths(z_min, z_max, z_f, r_e, focal_px, d):
    """Elementwise (x_a + x_b) * focal_px / d with invalid geometry -> 0."""
    z_m = (z_max + z_min) / 2.0
    r_s = (z_max - z_min) / 2.0
    hyp = np.sqrt(z_m ** 2 + r_e ** 2)
    ok = (z_min > 0) & (z_max >= z_min) & (z_f > z_max) & (z_m > 0) & (r_s <= hyp) & (r_e > 0)
    with np.errstate(all="ignore"):
        theta_d = np.arcsin(np.where(ok, r_s / hyp, 0.0))
        bq = r_e * (z_f - z_m) / z_m
        theta = np.arctan((bq + r_e) / z_f)
        ok &= (theta + theta_d) < math.pi / 2
        x_a = z_f * np.tan(theta - theta_d) - r_e
        x_b = z_f * np.tan(theta + theta_d) - r_e
        w = (x_a + x_b) * focal_px / d
    return np.where(ok, w, 0.0)


def blocker_plane(d, position, z_f, coverage, sm_depth, view, bias, size_index, focal_px, radius=8):
    """(H, W) fp32 penumbra-width plane (screen width / focal_px)."""
    hs, ws = view.resolution
    ri, ci, _ = texel_indices(view, position, coverage)
    sm = np.asarray(sm_depth, dtype=np.float64)
    thr = np.asarray(z_f, dtype=np.float64) - float(bias)
    zmin = np.full(ri.shape, np.inf)
    zmax = np.full(ri.shape, -np.inf)
    for dy in range(-radius, radius):
        for dx in range(-radius, radius):
            r, c = ri + dy, ci + dx
            inb = (r >= 0) & (r < hs) & (c >= 0) & (c < ws)
            t = sm[np.clip(r, 0, hs - 1), np.clip(c, 0, ws - 1)]
            blk = inb & np.isfinite(t) & (t < thr)
            zmin = np.where(blk, np.minimum(zmin, t), zmin)
            zmax = np.where(blk, np.maximum(zmax, t), zmax)
    have = coverage & np.isfinite(zmin)
    r_e = float(size_index) * SIZE_TO_RADIUS
    with np.errstate(all="ignore"):
        w = penumbra_widths(np.where(have, zmin, 1.0), np.where(have, zmax, 1.0),
                            np.asarray(z_f, dtype=np.float64), r_e, focal_px,
                            np.where(coverage, np.asarray(d, dtype=np.float64), 1.0))
    return np.where(have, w / float(focal_px), 0.0).astype(np.float32)
