"""Dataset frames straight to the device.

Reads the reference's on-disk dataset layout (dataset.py:86-245: a
``manifest.json`` plus per-frame FMAP files ``features_{k}.pfm`` (4 feature
planes + coverage) and ``gbuffer.pfm`` (d, n, p, z_f, c_e, c_c, coverage))
and lands batches of frames in HBM without intermediate numpy copies: each
file is read with ``readinto`` into one pinned staging buffer and moved by a
single asynchronous host->device copy. The numpy loaders keep the
reference's signatures (dataset.py:253-275) for drop-in use.

Consumers built on top: :func:`sequence_outputs` (cli._sequence_outputs,
cli.py:144-153) and :func:`eval_temporal` (cli.cmd_eval_temporal,
cli.py:156-171) run the whole evaluation on the GPU.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import fileio
from .raster import FeatureStack, GBuffer
from .scenes import CameraPose

__all__ = ["DatasetError", "FrameRecord", "DatasetManifest", "GBUFFER_PLANES", "load_manifest",
           "load_feature_stack", "load_gbuffer", "load_target", "read_floatmaps", "load_feature_batch",
           "load_gbuffer_batch", "sequence_outputs", "eval_temporal"]

GBUFFER_PLANES = ("d", "nx", "ny", "nz", "px", "py", "pz", "z_f", "c_e", "c_c", "coverage")


class DatasetError(RuntimeError):
    """Missing, truncated, or inconsistent dataset files (dataset.py:53-54)."""


@dataclass
class FrameRecord:
    frame_id: str
    time: float
    camera: dict
    emitter_center: list
    z_min: float
    z_max: float
    features: list
    gbuffer: str
    targets: dict


@dataclass
class DatasetManifest:
    root: Path
    scene_file: str
    scene_hash: str
    settings: dict
    frames: list
    manifest_hash: str = ""

    @property
    def resolution(self) -> tuple:
        return tuple(self.settings["resolution"])

    @property
    def sizes(self) -> tuple:
        return tuple(self.settings["sizes"])


def _pose(d: dict) -> CameraPose:
    return CameraPose(d["position"], d["forward"], d["up"], d["fov_y"], tuple(d["resolution"]))


def _header(path):
    with open(path, "rb") as fh:
        head = fh.read(16)
    if len(head) < 16 or head[:4] != fileio.FLOATMAP_MAGIC:
        raise fileio.FormatError(f"{path}: not a float map file")
    w, h, c = struct.unpack("<III", head[4:16])
    return c, h, w


def load_manifest(root) -> DatasetManifest:
    """Read and integrity-check a dataset directory (dataset.py:229-250)."""
    root = Path(root)
    try:
        payload = json.loads((root / "manifest.json").read_text())
    except FileNotFoundError as exc:
        raise DatasetError(f"{root}: no manifest.json") from exc
    frames = [FrameRecord(**f) for f in payload["frames"]]
    m = DatasetManifest(root=root, scene_file=payload["scene_file"], scene_hash=payload["scene_hash"],
                        settings=payload["settings"], frames=frames,
                        manifest_hash=payload.get("manifest_hash", ""))
    h, w = m.resolution
    for fr in frames:
        for rel in [*fr.features, fr.gbuffer, *fr.targets.values()]:
            path = root / rel
            if not path.exists():
                raise DatasetError(f"missing file {path}")
            try:
                c, fh_, fw_ = _header(path)
            except fileio.FormatError as exc:
                raise DatasetError(str(exc)) from exc
            if (fh_, fw_) != (h, w):
                raise DatasetError(f"{path}: resolution {fh_}x{fw_} does not match manifest {h}x{w}")
            if path.stat().st_size != 16 + 4 * c * fh_ * fw_:
                raise DatasetError(f"{path}: truncated")
    return m


def load_feature_stack(manifest: DatasetManifest, frame: int, k: int = 0,
                       size_index: float = 0.0) -> FeatureStack:
    """dataset.load_feature_stack (dataset.py:253-260)."""
    planes = fileio.load_floatmap(manifest.root / manifest.frames[frame].features[k])
    stack = FeatureStack(data=planes[:4], size_index=0.0, coverage=planes[4] > 0.5, bias=float("nan"))
    return stack.with_size_index(size_index) if size_index else stack


def load_gbuffer(manifest: DatasetManifest, frame: int) -> GBuffer:
    """dataset.load_gbuffer (dataset.py:263-275); n_e is not persisted."""
    rec = manifest.frames[frame]
    p = fileio.load_floatmap(manifest.root / rec.gbuffer).astype(np.float64)
    return GBuffer(d=p[0], normal=p[1:4], position=p[4:7], n_e=np.zeros_like(p[1:4]), z_f=p[7],
                   c_e=p[8], c_c=p[9], coverage=p[10] > 0.5, camera=_pose(rec.camera))


def load_target(manifest: DatasetManifest, frame: int, size_index: float) -> np.ndarray:
    """dataset.load_target (dataset.py:278-283)."""
    key = f"{float(size_index):g}"
    rec = manifest.frames[frame]
    if key not in rec.targets:
        raise DatasetError(f"frame {frame} has no target for size {key}")
    return fileio.load_floatmap(manifest.root / rec.targets[key])[0].astype(np.float64)


def read_floatmaps(paths, device="cuda"):
    """Read N same-shape FMAP files into one pinned (N, C, H, W) staging
    buffer (``readinto``, no intermediate arrays) and copy it to the device
    asynchronously. Returns the device tensor (the copy is ordered on the
    current stream)."""
    import torch
    paths = [Path(p) for p in paths]
    shape = _header(paths[0])
    stage = torch.empty((len(paths), *shape), dtype=torch.float32, pin_memory=True)
    view = memoryview(stage.numpy()).cast("B")
    per = 4 * int(np.prod(shape))
    for i, p in enumerate(paths):
        if _header(p) != shape:
            raise DatasetError(f"{p}: shape {_header(p)} differs from {shape}")
        with open(p, "rb") as fh:
            fh.seek(16)
            got = fh.readinto(view[i * per:(i + 1) * per])
            if got != per or fh.read(1):
                raise fileio.FormatError(f"{p}: truncated or trailing bytes")
    return stage.to(device, non_blocking=True)


def load_feature_batch(manifest: DatasetManifest, frames=None, k: int = 0, size_index: float = 0.0,
                       device="cuda"):
    """(features (N,4,H,W) fp32, coverage (N,H,W) bool) on the device; the
    size-index shift of FeatureStack.with_size_index applied in fp32 on
    covered pixels (raster.py:190-195)."""
    import torch
    frames = range(len(manifest.frames)) if frames is None else frames
    x = read_floatmaps([manifest.root / manifest.frames[f].features[k] for f in frames], device)
    cov = x[:, 4] > 0.5
    feats = x[:, :4]
    if size_index:
        feats[:, 2] = torch.where(cov, feats[:, 2] + np.float32(size_index), feats[:, 2])
    return feats.contiguous(), cov


def load_gbuffer_batch(manifest: DatasetManifest, frames=None, device="cuda"):
    """dict of device planes d (N,H,W), normal/position (N,3,H,W), z_f/c_e/c_c
    (N,H,W), coverage (N,H,W) uint8 -- the nsm_gbuffer layout -- plus the
    frame cameras."""
    import torch
    frames = list(range(len(manifest.frames)) if frames is None else frames)
    g = read_floatmaps([manifest.root / manifest.frames[f].gbuffer for f in frames], device)
    out = {"d": g[:, 0].contiguous(), "normal": g[:, 1:4].contiguous(), "position": g[:, 4:7].contiguous(),
           "z_f": g[:, 7].contiguous(), "c_e": g[:, 8].contiguous(), "c_c": g[:, 9].contiguous(),
           "coverage": (g[:, 10] > 0.5).to(torch.uint8)}
    return out, [_pose(manifest.frames[f].camera) for f in frames]


def sequence_outputs(manifest: DatasetManifest, plan, size_index: float = 0.0, max_batch: int = 8):
    """Network outputs of every frame's unperturbed stack, (T, H, W) fp32 on
    the device (cli._sequence_outputs, cli.py:144-153)."""
    import torch
    outs = []
    n = len(manifest.frames)
    for i in range(0, n, max_batch):
        x, _ = load_feature_batch(manifest, range(i, min(n, i + max_batch)), 0, size_index)
        outs.append(plan.forward(x)[:, 0])
    return torch.cat(outs)


def eval_temporal(manifest: DatasetManifest, plan, size_index: float = 0.0, alpha_t: float = 3.0):
    """cli.cmd_eval_temporal (cli.py:156-171) on the device: outputs,
    motion vectors from the stored G-buffers, temporal instability."""
    from . import temporal
    vis = sequence_outputs(manifest, plan, size_index)
    g, cams = load_gbuffer_batch(manifest)
    vec, valid = temporal.motion_vectors_batch(g, cams)
    return temporal.temporal_instability_batch(vis, vec, valid, alpha_t)
