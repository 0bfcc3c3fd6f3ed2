"""Host-side scene description for the hot path's inputs.

The hot path (feature pass + U-Net) consumes a camera G-buffer and a
light-space shadow map. This module describes the procedural scenes the
BASELINE configs name, the camera/emitter frames those buffers are rendered
in, and the emitter frustum fit; the buffers themselves are rendered on the
GPU by :mod:`paper_2301_05262_b200.producer`.

Everything here mirrors the reference's conventions so that a scene built
here can be handed to ``shadowkit`` unchanged (the golden-fixture script does
exactly that):

* ``CameraPose``     -- ``shadowkit/scene.py:102-183`` (orthonormalisation,
                        pixel-centre rays, (H, W) resolution)
* ``EmitterView``    -- ``shadowkit/raster.py:64-94``
* ``fit_emitter_view`` -- ``shadowkit/raster.py:97-134``
* primitives         -- ``shadowkit/scene.py:191-337`` (Plane, Sphere, Box)
* ``emitter_radius`` -- ``shadowkit/scene.py:54-58``
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

EMITTER_MAX_DIAMETER = 0.5      # scene.py:43
EMITTER_SIZE_MAX = 4.0          # scene.py:44
DEFAULT_SHADOW_RES = (512, 512)  # raster.py:48
DEFAULT_BIAS_FACTOR = 1e-3      # raster.py:49

# primitive kind tags shared with csrc/producer.cu
KIND_PLANE, KIND_SPHERE, KIND_BOX = 0, 1, 2


class SceneError(ValueError):
    """Invalid scene, camera or emitter description (scene.py:50-51)."""


def emitter_radius(size_index: float) -> float:
    """Radius in metres of a softness index in [0, 4] (scene.py:54-58)."""
    if not 0.0 <= size_index <= EMITTER_SIZE_MAX:
        raise SceneError(f"size_index {size_index} outside [0, {EMITTER_SIZE_MAX}]")
    return size_index * (EMITTER_MAX_DIAMETER / 2.0) / EMITTER_SIZE_MAX


def size_index_for_radius(radius: float) -> float:
    """Inverse of the radius law with no range check (the
    BASELINE soft-light radii reach size_index 8, which ``assemble_features``
    accepts even though ``Emitter`` does not)."""
    return float(radius) / ((EMITTER_MAX_DIAMETER / 2.0) / EMITTER_SIZE_MAX)


def _vec3(v) -> np.ndarray:
    a = np.asarray(v, dtype=np.float64).reshape(3).copy()
    if not np.all(np.isfinite(a)):
        raise SceneError("non-finite 3-vector")
    return a


def _unit(v: np.ndarray) -> np.ndarray:
    n = float(np.linalg.norm(v))
    if n == 0.0:
        raise SceneError("zero-length direction")
    return v / n


@dataclass(frozen=True)
class CameraPose:
    """Pinhole camera, resolution (H, W); see scene.py:102-134."""

    position: np.ndarray
    forward: np.ndarray
    up: np.ndarray
    fov_y: float
    resolution: tuple

    def __post_init__(self):
        pos = _vec3(self.position)
        f = _unit(_vec3(self.forward))
        r = np.cross(f, _vec3(self.up))
        if np.linalg.norm(r) < 1e-12:
            raise SceneError("camera up is parallel to forward")
        r = _unit(r)
        u = np.cross(r, f)
        object.__setattr__(self, "position", pos)
        object.__setattr__(self, "forward", f)
        object.__setattr__(self, "up", u)
        if not 0.0 < self.fov_y < math.pi:
            raise SceneError(f"fov_y {self.fov_y} outside (0, pi)")
        h, w = self.resolution
        if h <= 0 or w <= 0:
            raise SceneError("resolution must be positive")
        object.__setattr__(self, "resolution", (int(h), int(w)))

    @classmethod
    def look_at(cls, position, target, up=(0.0, 1.0, 0.0),
                fov_y=math.radians(45.0), resolution=(128, 256)) -> "CameraPose":
        p = _vec3(position)
        return cls(p, _vec3(target) - p, up, fov_y, resolution)

    @property
    def right(self) -> np.ndarray:
        return np.cross(self.forward, self.up)

    @property
    def focal_px(self) -> float:
        return (self.resolution[0] / 2.0) / math.tan(self.fov_y / 2.0)


@dataclass(frozen=True)
class EmitterView:
    """Square perspective frustum from the emitter centre (raster.py:64-73)."""

    position: np.ndarray
    forward: np.ndarray
    up: np.ndarray
    right: np.ndarray
    tan_half: float
    resolution: tuple


@dataclass(frozen=True)
class Primitive:
    kind: int
    params: tuple          # plane: point(3) normal(3) half(2); sphere: c(3) r; box: lo(3) hi(3)
    occluder: bool = True

    # -- geometry helpers shared by the frustum fit and the producer tables --
    def plane_tangents(self):
        """In-plane axes as scene.py:211-216 derives them."""
        n = _unit(np.asarray(self.params[3:6], dtype=np.float64))
        a = np.array([0.0, 0.0, 1.0]) if abs(n[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
        u = _unit(np.cross(n, a))
        return n, u, np.cross(n, u)

    def aabb(self):
        p = np.asarray(self.params, dtype=np.float64)
        if self.kind == KIND_PLANE:
            _, u, v = self.plane_tangents()
            su, sv = p[6], p[7]
            pts = np.array([p[0:3] + a * su * u + b * sv * v for a in (-1, 1) for b in (-1, 1)])
            return pts.min(axis=0), pts.max(axis=0)
        if self.kind == KIND_SPHERE:
            return p[0:3] - p[3], p[0:3] + p[3]
        return p[0:3], p[3:6]

    def bounding_sphere(self):
        p = np.asarray(self.params, dtype=np.float64)
        if self.kind == KIND_PLANE:
            return p[0:3], math.hypot(p[6], p[7])
        if self.kind == KIND_SPHERE:
            return p[0:3], float(p[3])
        c = (p[0:3] + p[3:6]) / 2.0
        return c, float(np.linalg.norm(p[3:6] - c))

    def contains(self, q) -> bool:
        p = np.asarray(self.params, dtype=np.float64)
        q = np.asarray(q, dtype=np.float64)
        if self.kind == KIND_SPHERE:
            return float(np.linalg.norm(q - p[0:3])) < p[3]
        if self.kind == KIND_BOX:
            return bool(np.all(q > p[0:3]) and np.all(q < p[3:6]))
        return False


def plane(point, normal, half_extent=(10.0, 10.0), occluder=False) -> Primitive:
    n = _unit(_vec3(normal))
    return Primitive(KIND_PLANE, tuple(_vec3(point)) + tuple(n) + tuple(map(float, half_extent)),
                     occluder)


def sphere(center, radius, occluder=True) -> Primitive:
    if not (np.isfinite(radius) and radius > 0):
        raise SceneError("sphere radius must be positive and finite")
    return Primitive(KIND_SPHERE, tuple(_vec3(center)) + (float(radius),), occluder)


def box(lo, hi, occluder=True) -> Primitive:
    lo, hi = _vec3(lo), _vec3(hi)
    if not np.all(hi > lo):
        raise SceneError("box needs hi > lo on every axis")
    return Primitive(KIND_BOX, tuple(lo) + tuple(hi), occluder)


@dataclass(frozen=True)
class SceneSpec:
    """Primitive list (intersection order matters: first object wins ties,
    as in scene.py:435-440) plus the emitter centre and radius."""

    objects: tuple
    emitter_center: np.ndarray
    emitter_radius: float = 0.0

    @property
    def size_index(self) -> float:
        return size_index_for_radius(self.emitter_radius)

    @property
    def bounds(self):
        los, his = zip(*(o.aabb() for o in self.objects))
        return np.min(los, axis=0), np.max(his, axis=0)

    @property
    def diagonal(self) -> float:
        lo, hi = self.bounds
        return float(np.linalg.norm(hi - lo))

    @property
    def default_bias(self) -> float:
        """raster.py:149-151."""
        return DEFAULT_BIAS_FACTOR * self.diagonal

    def occluder_depth_range(self):
        """(z_min, z_max) of occluder bounding spheres (scene.py:454-468)."""
        e = np.asarray(self.emitter_center, dtype=np.float64)
        lo, hi = np.inf, -np.inf
        for o in self.objects:
            if not o.occluder:
                continue
            c, r = o.bounding_sphere()
            d = float(np.linalg.norm(c - e))
            lo, hi = min(lo, d - r), max(hi, d + r)
        if not np.isfinite(lo):
            raise SceneError("scene has no occluder primitives")
        return max(lo, 0.0), hi

    def primitive_table(self) -> np.ndarray:
        """(n, 16) float64 rows consumed by the GPU producer.

        [kind, p0..p?, ...]: plane = point, normal, u, v, su, sv;
        sphere = centre, r; box = lo, hi.
        """
        rows = np.zeros((len(self.objects), 16), dtype=np.float64)
        for i, o in enumerate(self.objects):
            rows[i, 0] = o.kind
            p = np.asarray(o.params, dtype=np.float64)
            if o.kind == KIND_PLANE:
                n, u, v = o.plane_tangents()
                rows[i, 1:4] = p[0:3]
                rows[i, 4:7] = n
                rows[i, 7:10] = u
                rows[i, 10:13] = v
                rows[i, 13:15] = p[6:8]
            elif o.kind == KIND_SPHERE:
                rows[i, 1:5] = p[0:4]
            else:
                rows[i, 1:7] = p[0:6]
        return rows


def fit_emitter_view(scene: SceneSpec, center=None, resolution=DEFAULT_SHADOW_RES,
                     margin: float = 1.05) -> EmitterView:
    """Aim a square frustum from the emitter at the scene (raster.py:97-134)."""
    pos = _vec3(scene.emitter_center if center is None else center)
    for o in scene.objects:
        if o.contains(pos):
            raise SceneError("emitter center lies inside scene geometry")
    lo, hi = scene.bounds
    fwd = (lo + hi) / 2.0 - pos
    dist = np.linalg.norm(fwd)
    if dist < 1e-9:
        raise SceneError("emitter at the scene bounds center")
    fwd = fwd / dist
    aux = np.array([0.0, 0.0, 1.0]) if abs(fwd[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
    right = _unit(np.cross(fwd, aux))
    up = np.cross(right, fwd)
    corners = []
    for o in scene.objects:            # per-primitive boxes, not the union box
        olo, ohi = o.aabb()
        corners += [[x, y, z] for x in (olo[0], ohi[0]) for y in (olo[1], ohi[1])
                    for z in (olo[2], ohi[2])]
    rel = np.asarray(corners) - pos
    zc = rel @ fwd
    if np.any(zc <= 0):
        raise SceneError("scene bounds extend behind the emitter")
    tan_half = float(np.max(np.maximum(np.abs(rel @ right), np.abs(rel @ up)) / zc) * margin)
    if tan_half > math.tan(math.radians(80.0)):
        raise SceneError("emitter too close: frustum cannot cover the scene")
    return EmitterView(pos, fwd, up, right, tan_half, (int(resolution[0]), int(resolution[1])))


# ---------------------------------------------------------------------------
# BASELINE.json procedural scenes
# ---------------------------------------------------------------------------

LIGHT_POS = (3.0, 5.0, 2.0)
CAMERA_POS = (0.0, 3.0, -6.0)      # BASELINE leaves it open; recorded in DESIGN.md
# Fully covered variant: a camera looking steeply down at
# the ground so every pixel hits geometry, as in a typical game G-buffer.
FULL_COVER_POS = (0.0, 4.0, -0.6)
FULL_COVER_TARGET = (0.0, 0.0, 0.4)
CAMERA_FOV_DEG = 60.0
GROUND_HALF = 5.0                  # 10 m breaks the frustum fit


@dataclass(frozen=True)
class Frame:
    """One frame of a workload: scene + camera + emitter view."""

    scene: SceneSpec
    camera: CameraPose
    view: EmitterView

    @property
    def size_index(self) -> float:
        return self.scene.size_index

    @property
    def bias(self) -> float:
        return self.scene.default_bias


def random_scene(n_objects: int, seed: int, emitter_radius_m: float = 0.0,
                 light=LIGHT_POS) -> SceneSpec:
    """Ground rectangle y=0 plus ``n_objects`` boxes/spheres (50/50).

    Centres U([-2,2]x[0.2,1.5]x[-2,2]); radius / per-axis half-size U[0.1,0.5]
    (BASELINE configs[0]). Deterministic in ``seed``.
    """
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 0x5CE]))
    objs = [plane((0.0, 0.0, 0.0), (0.0, 1.0, 0.0), (GROUND_HALF, GROUND_HALF))]
    for _ in range(n_objects):
        is_box = rng.random() < 0.5
        c = rng.uniform((-2.0, 0.2, -2.0), (2.0, 1.5, 2.0))
        if is_box:
            h = rng.uniform(0.1, 0.5, size=3)
            objs.append(box(c - h, c + h))
        else:
            objs.append(sphere(c, float(rng.uniform(0.1, 0.5))))
    return SceneSpec(tuple(objs), _vec3(light), float(emitter_radius_m))


def make_frame(scene: SceneSpec, resolution, shadow_res, camera_pos=CAMERA_POS,
               target=(0.0, 0.0, 0.0), fov_deg=CAMERA_FOV_DEG) -> Frame:
    cam = CameraPose.look_at(camera_pos, target, fov_y=math.radians(fov_deg),
                             resolution=tuple(resolution))
    view = fit_emitter_view(scene, resolution=shadow_res)
    return Frame(scene, cam, view)


def full_cover(frame: Frame, offset=(0.0, 0.0, 0.0)) -> Frame:
    """The same scene and light seen by the fully covered camera."""
    off = np.asarray(offset, dtype=np.float64)
    return make_frame(frame.scene, frame.camera.resolution, frame.view.resolution,
                      camera_pos=np.asarray(FULL_COVER_POS) + off,
                      target=np.asarray(FULL_COVER_TARGET) + off)


def config_frames(config: int, seed: int = 0, n_frames: int | None = None) -> list[Frame]:
    """Frames of BASELINE.json ``configs[config - 1]`` (1-based like SURVEY §8d).

    1: 256x256, 8 objects, SM 512^2, point light.
    2: 1920x1080, 32 objects, SM 2048^2, point light.
    3: as 2 with a spherical light of radius U[0.05, 0.5].
    4: 8 consecutive frames of 3: light, one object and the camera each move
       0.02 units/frame along seeded random unit directions.
    5: 3840x2160, 64 objects, SM 4096^2, 50/50 hard/soft, one frame per scene
       (``n_frames`` scenes, default 64).
    """
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 0xC0F, config]))
    if config == 1:
        return [make_frame(random_scene(8, seed), (256, 256), (512, 512))]
    if config == 2:
        return [make_frame(random_scene(32, seed), (1080, 1920), (2048, 2048))]
    if config == 3:
        r = float(rng.uniform(0.05, 0.5))
        return [make_frame(random_scene(32, seed, r), (1080, 1920), (2048, 2048))]
    if config == 4:
        r = float(rng.uniform(0.05, 0.5))
        base = random_scene(32, seed, r)
        n = 8 if n_frames is None else int(n_frames)
        dirs = [_unit(rng.normal(size=3)) for _ in range(3)]
        mover = 1 + int(rng.integers(len(base.objects) - 1))
        frames = []
        for t in range(n):
            step = 0.02 * t
            objs = list(base.objects)
            o = objs[mover]
            p = np.asarray(o.params, dtype=np.float64)
            if o.kind == KIND_SPHERE:
                objs[mover] = sphere(p[0:3] + step * dirs[1], p[3])
            else:
                objs[mover] = box(p[0:3] + step * dirs[1], p[3:6] + step * dirs[1])
            sc = SceneSpec(tuple(objs), base.emitter_center + step * dirs[0], r)
            frames.append(make_frame(sc, (1080, 1920), (2048, 2048),
                                     camera_pos=np.asarray(CAMERA_POS) + step * dirs[2]))
        return frames
    if config == 5:
        n = 64 if n_frames is None else int(n_frames)
        frames = []
        for k in range(n):
            soft = (k % 2) == 1
            r = float(rng.uniform(0.05, 0.5)) if soft else 0.0
            frames.append(make_frame(random_scene(64, seed * 1000 + k, r),
                                     (2160, 3840), (4096, 4096)))
        return frames
    raise ValueError(f"unknown config {config}")
