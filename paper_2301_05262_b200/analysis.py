"""Batched multi-forward consumers of the network on B200.

The reference's evaluation code calls ``network.forward`` once per stack and
per perturbation -- O(10^3) forwards for a sensitivity report
(analysis.py:100-139, cli.py:173-194) and one per held-out sample for the
training score (training.py:179-189). These drop-ins keep the reference
signatures and semantics, and when ``phi`` is a :class:`PlanPhi` (a GPU
plan) they submit the stacks and all their perturbations as batches of
``nsm_forward`` calls on device-resident inputs; any other callable ``phi``
is evaluated exactly as the reference does (it is the caller's model).

Noise is drawn from the caller's ``rng`` in the reference's order (repeat
-> stack, one (H, W) normal field each), so a report equals the reference's
for the same rng seed up to the forward's arithmetic.
"""

from __future__ import annotations

import math

import numpy as np

from .network import NetworkConfig, Plan, plan_for

__all__ = ["ZeroVarianceChannel", "SensitivityReport", "PlanPhi", "channel_sensitivity",
           "sensitivity_report", "heldout_mse", "mse", "SENSITIVITY_NOISE_SCALE"]

SENSITIVITY_NOISE_SCALE = 0.1          # analysis.py:58


class ZeroVarianceChannel(ValueError):
    """Channel has no variation across the dataset (analysis.py:64-65)."""


class SensitivityReport:
    """S_i / s_i per channel (analysis.py:75-97)."""

    def __init__(self, channels, absolute, relative, frames, repeats):
        self.channels = tuple(channels)
        self.absolute = np.asarray(absolute)
        self.relative = np.asarray(relative)
        self.frames = int(frames)
        self.repeats = int(repeats)

    def as_text(self) -> str:
        lines = ["channel sensitivity (absolute, relative %):"]
        for name, s, rel in zip(self.channels, self.absolute, self.relative):
            lines.append(f"  {name:>8s}  {s:10.6f}  {100 * rel:6.2f}%")
        lines.append(f"  frames={self.frames} repeats={self.repeats}")
        return "\n".join(lines)

    def write_csv(self, path) -> None:
        import csv
        with open(path, "w", newline="") as fh:
            wr = csv.writer(fh)
            wr.writerow(["channel", "absolute", "relative"])
            for name, s, rel in zip(self.channels, self.absolute, self.relative):
                wr.writerow([name, repr(float(s)), repr(float(rel))])


class PlanPhi:
    """phi(stack) -> (H, W) image backed by a GPU plan; ``batch`` runs
    (N, C, H, W) CUDA stacks at once. ``max_batch`` bounds the frames per
    nsm_forward call (workspace)."""

    def __init__(self, weights_or_plan, cfg: NetworkConfig | None = None, dtype: str = "fp32",
                 max_batch: int = 32):
        self.plan = weights_or_plan if isinstance(weights_or_plan, Plan) else plan_for(
            weights_or_plan, cfg, dtype)
        self.max_batch = int(max_batch)

    def batch(self, x):
        import torch
        outs = [self.plan.forward(x[i:i + self.max_batch])[:, 0]
                for i in range(0, x.shape[0], self.max_batch)]
        return torch.cat(outs) if len(outs) > 1 else outs[0]

    def __call__(self, stack):
        import torch
        x = torch.from_numpy(np.ascontiguousarray(stack, dtype=np.float32)).cuda()
        return self.batch(x[None])[0].cpu().numpy()


def _sigma(stacks, channel):
    return float(np.std(np.concatenate([s[channel].ravel() for s in stacks])))


def channel_sensitivity(phi, stacks, channel: int, repeats: int = 8,
                        rng: np.random.Generator | None = None,
                        sigma: float | None = None) -> float:
    """Absolute sensitivity S_i of one channel (analysis.py:100-122)."""
    stacks = [np.asarray(s) for s in stacks]
    if rng is None:
        rng = np.random.default_rng(0)
    if sigma is None:
        sigma = _sigma(stacks, channel)
    if sigma <= 0.0 or not math.isfinite(sigma):
        raise ZeroVarianceChannel(f"channel {channel} has zero variance")
    noise = SENSITIVITY_NOISE_SCALE * sigma
    if not isinstance(phi, PlanPhi):
        base = [np.asarray(phi(s), dtype=np.float64) for s in stacks]
        total, count = 0.0, 0
        for _ in range(repeats):
            for s, b in zip(stacks, base):
                pert = s.copy()
                pert[channel] = pert[channel] + rng.normal(0.0, noise, size=s.shape[1:]).astype(s.dtype)
                delta = np.abs(np.asarray(phi(pert), dtype=np.float64) - b)
                total += float(delta.sum())
                count += delta.size
        return total / count / noise
    import torch
    shapes = {s.shape for s in stacks}
    groups = [stacks] if len(shapes) == 1 else [[s] for s in stacks]
    # device copies of the stacks and their base images, per shape group
    dev = [torch.from_numpy(np.ascontiguousarray(np.stack(g), dtype=np.float32)).cuda() for g in groups]
    base = [phi.batch(x).double() for x in dev]
    where = [(gi, k) for gi, g in enumerate(groups) for k in range(len(g))]
    total = torch.zeros((), dtype=torch.float64, device="cuda")
    count = 0
    pending = []

    def flush():
        nonlocal count
        if not pending:
            return
        gi = pending[0][0]
        x = dev[gi][[k for _, k, _ in pending]].clone()
        nz = torch.from_numpy(np.stack([z for _, _, z in pending])).cuda()
        x[:, channel] = x[:, channel] + nz          # fp32 add, as pert[channel] + noise
        y = phi.batch(x).double()
        b = base[gi][[k for _, k, _ in pending]]
        total.add_((y - b).abs().sum())
        count += y.numel()
        pending.clear()

    for _ in range(repeats):
        for gi, k in where:
            s = groups[gi][k]
            z = rng.normal(0.0, noise, size=s.shape[1:]).astype(np.float32)
            if pending and (pending[0][0] != gi or len(pending) >= phi.max_batch):
                flush()
            pending.append((gi, k, z))
    flush()
    return float(total.item()) / count / noise


def sensitivity_report(phi, stacks, channels, repeats: int = 8,
                       rng: np.random.Generator | None = None) -> SensitivityReport:
    """S_i and s_i for every channel of a stack list (analysis.py:125-139)."""
    if rng is None:
        rng = np.random.default_rng(0)
    absolute = np.array([channel_sensitivity(phi, stacks, i, repeats, rng)
                         for i in range(len(channels))])
    denom = absolute.sum()
    if denom <= 0:
        raise ZeroVarianceChannel("all channels produced zero sensitivity")
    return SensitivityReport(channels, absolute, absolute / denom, len(stacks), repeats)


def heldout_mse(phi, stacks, targets) -> float:
    """training._eval_mse (training.py:179-189) over (stack, target) pairs:
    sum of squared errors / pixel count, NaN for an empty set."""
    stacks = list(stacks)
    if not stacks:
        return math.nan
    if not isinstance(phi, PlanPhi):
        total, count = 0.0, 0
        for s, t in zip(stacks, targets):
            y = np.asarray(phi(s))
            total += float(np.sum((y - t) ** 2))
            count += y.size
        return total / count
    import torch
    total, count = 0.0, 0
    for i in range(0, len(stacks), phi.max_batch):
        chunk = stacks[i:i + phi.max_batch]
        if len({np.shape(s) for s in chunk}) != 1:
            for s, t in zip(chunk, targets[i:i + phi.max_batch]):
                total += heldout_mse(phi, [s], [t]) * np.size(t)
                count += np.size(t)
            continue
        x = torch.from_numpy(np.ascontiguousarray(np.stack(chunk), dtype=np.float32)).cuda()
        t = torch.from_numpy(np.ascontiguousarray(np.stack(targets[i:i + phi.max_batch]),
                                                  dtype=np.float32)).cuda()
        y = phi.batch(x)
        total += float(((y - t) ** 2).double().sum().item())
        count += y.numel()
    return total / count


def mse(img, ref, mask=None) -> float:
    """analysis.mse (analysis.py:380-393) for numpy arrays or CUDA tensors."""
    import torch
    a = torch.as_tensor(img).double()
    b = torch.as_tensor(ref).double().to(a.device)
    if a.shape != b.shape:
        raise ValueError(f"mse shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    d = (a - b) ** 2
    if mask is not None:
        m = torch.as_tensor(mask).to(a.device).bool()
        if m.shape != a.shape:
            raise ValueError("mask shape mismatch")
        if not bool(m.any()):
            raise ValueError("empty mask")
        return float(d[m].mean().item())
    return float(d.mean().item())
