#!/usr/bin/env python
"""Throughput benchmark of the neural-shadow-mapping hot path on B200.

Contract (one JSON line on rank 0):
    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4] [--dtype fp16]

Workload (default ``--config 4``, BASELINE.json configs[3]): a temporal
window of 8 consecutive 1920x1080 soft-shadow frames (spherical light of
radius U[0.05, 0.5], 32 objects, 2048^2 shadow map, light / one object /
camera moving 0.02 units per frame), fp16 activations with fp32
accumulation, seeded random-init weights of the reference architecture
(NetworkConfig(), 164,500 parameters). A step = the full hot path (feature
pass + U-Net -> visibility) over the 8-frame batch. Every rank processes its
own window (seed = rank): weak scaling, no collective on the data path; NCCL
only gathers the per-rank timings (max over ranks). Inputs (G-buffer and
shadow maps, ~600 MB per window) are larger than L2, so no flush is needed
between steps. Synthetic data: procedural scenes rendered on the GPU by the
repo's own producer kernels (the reference ships no dataset).

``--impl reference`` times the reference algorithm on the host CPU cores
(the numpy oracle port of shadowkit's assemble_features + forward; the
reference package itself is not present on the GPU box), one frame per step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "1080p soft-shadow frames/sec"
UNIT = "frames/s"


def metric_name(config):
    return {2: "1080p hard-shadow frames/sec", 3: METRIC, 4: METRIC,
            5: "4K hard/soft-shadow frames/sec (64-scene sweep)"}[config]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4, choices=[2, 3, 4, 5])
    ap.add_argument("--dtype", choices=["fp16", "bf16", "fp32"], default="fp16")
    ap.add_argument("--frames", type=int, default=None, help="frames per rank (default: config)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-soak", action="store_true", help="skip the 1 s clock-sampling soak")
    return ap.parse_args()


def workload_name(config):
    return {2: "cfg2-1080p-hard", 3: "cfg3-1080p-soft", 4: "cfg4-1080p-soft-window8",
            5: "cfg5-4k-sweep"}[config]


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j["hbm_gbs"], j["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


# --------------------------------------------------------------------------
# algorithmic cost models
# --------------------------------------------------------------------------

def covered_pixels(inputs):
    return int((inputs["d"] > 0).sum().item())


def kernel_models(frames, inputs, cfg, dtype):
    """Per-launch algorithmic bytes / flops of the kernels we can model."""
    n = len(frames)
    h, w = frames[0].camera.resolution
    px = n * h * w
    hp = (h + 15) // 16 * 16
    wp = (w + 15) // 16 * 16
    cov = covered_pixels(inputs)
    act = 4 if dtype == "fp32" else 2
    from paper_2301_05262_b200 import network
    st = network.net_stats(cfg, (hp, wp))
    l0 = hp // 2 * wp // 2
    models = {
        # G-buffer 28 B/px (d + normal + position fp32) + one 4-B texel per
        # covered pixel + 16 fp32 feature bytes per pixel written
        "features_kernel": {"bytes": 28 * px + 4 * cov + 16 * n * hp * wp, "flops": 0},
        # fused feature pass + L0 encoder (enc3 16->16, enc1 16->16, pool):
        # G-buffer in, texel gathers, pooled 16-ch L1 tensor out
        "enc0_fused": {"bytes": 28 * px + 4 * cov + n * (l0 // 4) * 16 * act,
                       "flops": 2 * n * l0 * (16 * 16 * 9 + 16 * 16)},
    }
    step_bytes = 28 * px + 4 * cov + px * act
    step_flops = 2.0 * n * hp * wp * sum(s["flops_per_pixel"] for s in st)
    return models, step_bytes, step_flops


def ncu_traffic(kernel, algo_bytes, frames_per_launch, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of ``kernel``,
    scaled from the committed ncu --set full capture (profiles/traffic.json,
    written by tools/ncu_summary.py traffic) to this run's frames per launch."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        t = json.load(f).get(kernel)
    if not t or t.get("workload") != workload:
        return None
    bpf = t["dram_bytes_per_frame"]
    return {"bytes": int(bpf * frames_per_launch), "algorithmic_bytes": int(algo_bytes),
            "ratio": round(bpf * frames_per_launch / algo_bytes, 3), "source": t["source"]}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def run_ours(args):
    import torch
    from paper_2301_05262_b200 import _lib, network, producer, scenes
    from paper_2301_05262_b200.infer import ShadowInference

    rank, world, local = dist_setup()
    frames = scenes.config_frames(args.config, seed=rank, n_frames=args.frames)
    if args.config in (2, 3):
        frames = frames * (args.frames or 1)
    inputs = producer.render_inputs(frames)
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    plan = network.Plan(w, cfg, args.dtype)
    out_dtype = "fp32" if args.dtype == "fp32" else "fp16"
    run = ShadowInference(plan, frames, out_dtype=out_dtype)
    run(inputs)                                  # validates frustum, warms up
    torch.cuda.synchronize()
    n = len(frames)
    h, wd = frames[0].camera.resolution

    c0 = _lib.lib.nsm_launch_count()
    if args.no_graph:
        step = lambda: run.launch(inputs)        # noqa: E731
        run.launch(inputs)
        per_step = _lib.lib.nsm_launch_count() - c0
    else:
        run.capture(inputs)
        per_step = (_lib.lib.nsm_launch_count() - c0) // 2   # warm launch + captured launch
        step = run.replay
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # keep the GPU loaded ~1 s so nvidia-smi samples clocks under load
        t_end = time.time() + (0.0 if args.no_soak else 1.0)
        while time.time() < t_end:
            for _ in range(20):
                step()
            torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        barrier(world)
    ms = e0.elapsed_time(e1) / args.steps
    ms_max = allreduce_max(ms, world)
    frames_total = n * world
    value = frames_total / (ms_max / 1e3)

    # ---- per-kernel timing (eager, traced launches on the same stream) ----
    _lib.lib.nsm_profile_enable(1)
    _lib.profile_report()
    for _ in range(args.steps):
        run.launch(inputs)
    torch.cuda.synchronize()
    prof = _lib.profile_report()
    _lib.lib.nsm_profile_enable(0)
    models, step_bytes, step_flops = kernel_models(frames, inputs, cfg, args.dtype)
    hbm, tfl, src = peaks()
    dom = max(prof, key=lambda k: prof[k][1]) if prof else None
    step_prof_ms = sum(v[1] for v in prof.values()) / max(args.steps, 1)
    roof = None
    if dom in models:
        cnt, tot = prof[dom]
        avg_ms = tot / cnt
        mb = models[dom]["bytes"] / max(1, cnt // args.steps)   # model is per step
        ach = mb / (avg_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm,
                "unit": "GB/s", "frac": round(ach / hbm, 4),
                "traffic": ncu_traffic(dom, mb, n // max(1, cnt // args.steps), workload_name(args.config)),
                "avg_launch_ms": round(avg_ms, 5), "peak_source": src,
                "share_of_step": round(tot / args.steps / step_prof_ms, 3)}
    elif dom is not None:
        cnt, tot = prof[dom]
        roof = {"bound": "hbm", "kernel": "step", "achieved":
                round(step_bytes / (ms / 1e3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(step_bytes / (ms / 1e3) / 1e9 / hbm, 4), "traffic": None,
                "peak_source": src, "dominant_kernel": dom,
                "dominant_share_of_step": round(tot / args.steps / step_prof_ms, 3)}

    # ---- end to end through the public API with host buffers ----
    # HostPipeline: pinned host inputs -> H2D (copy stream) -> fused kernels
    # -> D2H of the visibility, overlapped across consecutive batches
    e2e = None
    if not args.no_e2e:
        from paper_2301_05262_b200.infer import HostPipeline
        host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in inputs.items()}
        for k in host:
            host[k].copy_(inputs[k])
        yh = torch.empty(run.y.shape, dtype=run.y.dtype, pin_memory=True)
        h2d = sum(v.numel() * v.element_size() for v in host.values())
        d2h = yh.numel() * yh.element_size()
        pipe = HostPipeline(run)
        for _ in range(2):
            pipe.submit(host, yh)
        pipe.synchronize()
        torch.cuda.synchronize()
        k2 = max(3, min(args.steps, 10))
        barrier(world)
        e0.record(pipe.h2d)
        for _ in range(k2):
            pipe.submit(host, yh)
        e1.record(pipe.d2h)
        pipe.synchronize()
        torch.cuda.synchronize()
        barrier(world)
        ems = allreduce_max(e0.elapsed_time(e1) / k2, world)
        e2e = {"value": round(frames_total / (ems / 1e3), 3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(ems, 4), "steps": k2,
               "api": "infer.HostPipeline.submit (pinned host in/out, copies overlapped)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(frames[:1], inputs, w, reps=2)

    if rank == 0:
        mpix = value * h * wd / 1e6
        line = {
            "metric": metric_name(args.config), "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms_max, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"fp16": "f16", "bf16": "bf16", "fp32": "f32"}[args.dtype],
            "data": "synthetic (procedural scenes rendered on-GPU; random-init weights)",
            "config": {"workload": workload_name(args.config), "frames_per_rank": n,
                       "resolution": [h, wd], "net_resolution": [(h + 15) // 16 * 16, wd],
                       "shadow_map": list(frames[0].view.resolution),
                       "network": "NetworkConfig(layers=5, base=16, in=4, s2d) 164,500 params",
                       "l2": "inputs > L2 (no flush needed)",
                       "graph": not args.no_graph, "parallelism": f"frames-dp{world}"},
            "mpix_per_s": round(mpix, 2),
            "roofline": roof,
            "step_roofline": {"bytes": int(step_bytes), "flops": step_flops,
                              "gbps": round(step_bytes / (ms / 1e3) / 1e9, 1),
                              "tflops": round(step_flops / (ms / 1e3) / 1e12, 2)},
            "kernel_profile_ms_per_step": {k: round(v[1] / args.steps, 5) for k, v in
                                           sorted(prof.items(), key=lambda kv: -kv[1][1])},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(per_step * args.steps),
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# --------------------------------------------------------------------------
# CPU reference arm (the oracle port of shadowkit's algorithm)
# --------------------------------------------------------------------------

def _oracle_frame(fr, planes, weights):
    from oracle import features as of
    from oracle import network as on
    feats, _ = of.features_from_planes(planes["d"], planes["normal"], planes["position"],
                                       planes["sm"], fr.camera, fr.view, fr.scene.emitter_center,
                                       fr.size_index, fr.bias)
    h, w = feats.shape[1:]
    hp, wp = (h + 15) // 16 * 16, (w + 15) // 16 * 16
    x = np.zeros((4, hp, wp), np.float32)
    x[:, :h, :w] = feats
    return on.forward(weights, x)[:, :h, :w]


def cpu_baseline_sample(frames, inputs, weights, reps=2):
    """Time the oracle port on a bounded sample (one frame, best of reps)."""
    W = {k: v.data for k, v in weights.items()}
    planes = {k: v[0].cpu().numpy() for k, v in inputs.items()}
    best = float("inf")
    for _ in range(reps):
        t = time.perf_counter()
        _oracle_frame(frames[0], planes, W)
        best = min(best, time.perf_counter() - t)
    return {"value": round(1.0 / best, 4), "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
            "kind": "port", "sample": f"1 frame of the workload, best of {reps} "
            f"({best:.2f} s/frame; numpy+OpenBLAS threads = all cores)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    from paper_2301_05262_b200 import network, producer, scenes
    from oracle import network as _on  # noqa: F401  (fail early if absent)
    frames = scenes.config_frames(args.config, seed=0, n_frames=args.frames)
    inputs = producer.render_inputs(frames) if torch.cuda.is_available() else None
    cfg = network.NetworkConfig()
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    W = {k: v.data for k, v in w.items()}
    planes = [{k: v[i].cpu().numpy() for k, v in inputs.items()} for i in range(len(frames))]
    warm = min(args.warmup, 1)
    steps = min(args.steps, 5)
    for i in range(warm):
        _oracle_frame(frames[i % len(frames)], planes[i % len(frames)], W)
    t = time.perf_counter()
    for i in range(steps):
        _oracle_frame(frames[i % len(frames)], planes[i % len(frames)], W)
    el = time.perf_counter() - t
    value = steps / el
    h, wd = frames[0].camera.resolution
    print(json.dumps({
        "metric": metric_name(args.config), "value": round(value, 4), "unit": UNIT, "impl": "reference",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": steps, "warmup": warm,
        "ms_per_step": round(el / steps * 1e3, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (same scenes/weights as ours)",
        "config": {"workload": workload_name(args.config), "resolution": [h, wd],
                   "note": f"one frame per step; steps capped at 5 (asked {args.steps})"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT,
                         "cores": len(os.sched_getaffinity(0)), "kind": "port",
                         "sample": "one 1080p frame per step: oracle assemble_features + forward"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "mpix_per_s": round(value * h * wd / 1e6, 4),
    }))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
