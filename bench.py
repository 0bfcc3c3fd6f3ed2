#!/usr/bin/env python
"""Throughput benchmark of the neural-shadow-mapping hot path on B200.

Contract (one JSON line on rank 0):
    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4] [--dtype fp16] [--features 4|5]

Workload (default ``--config 4``, BASELINE.json configs[3]): a temporal
window of 8 consecutive 1920x1080 soft-shadow frames (spherical light of
radius U[0.05, 0.5], 32 objects, 2048^2 shadow map, light / one object /
camera moving 0.02 units per frame), fp16 activations with fp32
accumulation, seeded random-init weights of the reference architecture,
with the reference's own 4-plane feature layout (soft shadows enter through
the size-index plane).  A step = the full hot path (feature pass + U-Net ->
visibility) over the job's frames.  The same run also times, as
``variants``, the window with the 5-plane net (BASELINE's 16x16
blocker-search penumbra plane; ``--config 3`` makes that the main line) and
a fully covered camera.

Multi-GPU (north_star: "shards the frame batch and temporal window across
the GPUs"): one process per GPU.  ``--gpus N`` re-executes itself under
torchrun when WORLD_SIZE is unset.  The job's frames (config 4: the 8-frame
window; config 5: the 64 scenes) are split with ``shard.shard_bounds``
(8/4/2/1 frames per rank at N = 1/2/4/8) -- strong scaling, no collective on
the data path; NCCL gathers the per-rank step times (the job time is the
max over ranks) and, with ``--gather``, the visibility frames in frame
order.  ``--scaling weak`` gives every rank its own window instead
(labelled).  Configs 2/3 are one frame: N > 1 runs replicas.

Inputs (G-buffer + shadow maps, ~75 MB per 1080p frame) are larger than L2
across a step, so no flush is needed.  Synthetic data: procedural scenes
rendered on the GPU by the repo's producer kernels (the reference ships no
dataset).

``--impl reference`` times the reference's own CPU implementation --
``shadowkit``'s ``raster.assemble_features`` + ``network.forward`` under
``autodiff.no_grad()`` (``oracle/_ref``, staged by ``build()``; the numpy
oracle port when it is absent) -- on the host cores, with inputs rendered
on the CPU (``oracle.producer``) so that the process never loads the CUDA
library.
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

UNIT = "frames/s"


def metric_name(config):
    return {2: "1080p hard-shadow frames/sec", 3: "1080p soft-shadow frames/sec",
            4: "1080p soft-shadow frames/sec",
            5: "4K hard/soft-shadow frames/sec (64-scene sweep)"}[config]


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4, choices=[2, 3, 4, 5])
    ap.add_argument("--dtype", choices=["fp16", "bf16", "fp32"], default=None,
                    help="default: fp16 (configs 2-4), bf16 (config 5)")
    ap.add_argument("--features", type=int, choices=[4, 5], default=None,
                    help="input planes: 4 (the reference's layout: soft shadows through the size "
                         "index plane) or 5 (+ the 16x16 blocker-search penumbra plane); default: "
                         "5 for config 3 (whose text names the search), 4 otherwise")
    ap.add_argument("--frames", type=int, default=None, help="frames of the job (default: config)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: shard the job's frames over the ranks; weak: one job per rank")
    ap.add_argument("--cover", choices=["scene", "full"], default="scene",
                    help="full: the fully covered camera variant as the main workload")
    ap.add_argument("--gather", action="store_true", help="NCCL-gather the visibility to every rank")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-soak", action="store_true", help="skip the 1 s clock-sampling soak")
    ap.add_argument("--no-variants", action="store_true", help="skip the fully covered variant")
    a = ap.parse_args(argv)
    if a.dtype is None:
        a.dtype = "bf16" if a.config == 5 else "fp16"
    if a.features is None:
        a.features = 5 if a.config == 3 else 4
    return a


def workload_name(args):
    base = {2: "cfg2-1080p-hard", 3: "cfg3-1080p-soft", 4: "cfg4-1080p-soft-window8",
            5: "cfg5-4k-sweep"}[args.config]
    if args.features == 5:
        base += "-blocker"
    if args.cover == "full":
        base += "-fullcover"
    return base


# --------------------------------------------------------------------------
# job / sharding (pure host logic; tests/test_bench_shard.py drives it)
# --------------------------------------------------------------------------

def job_frames(args, seed=0):
    """All frames of one job (every rank of a strong-scaling run sees the
    same list and takes its shard)."""
    from paper_2301_05262_b200 import scenes
    if args.config in (2, 3):
        frames = scenes.config_frames(args.config, seed=seed) * (args.frames or 1)
    else:
        frames = scenes.config_frames(args.config, seed=seed, n_frames=args.frames)
    if args.cover == "full":
        frames = [full_cover_frame(f) for f in frames]
    return frames


def full_cover_frame(f):
    from paper_2301_05262_b200 import scenes
    return scenes.full_cover(f, offset=np.asarray(f.camera.position) - np.asarray(scenes.CAMERA_POS))


def rank_frames(args, rank, world):
    """(frames this rank runs, [lo, hi) of the job, job size, scaling label)."""
    from paper_2301_05262_b200 import shard
    if args.scaling == "weak":
        frames = job_frames(args, seed=shard.window_seed(rank))
        return frames, (0, len(frames)), len(frames) * world, "weak"
    frames = job_frames(args, seed=0)
    if len(frames) < world:            # one-frame configs: replicas
        return frames, (0, len(frames)), len(frames) * world, "weak"
    lo, hi = shard.shard_bounds(len(frames), rank, world)
    return frames[lo:hi], (lo, hi), len(frames), "strong"


def env_guard():
    """Refuse to time anything while experiment switches could be active."""
    bad = sorted(k for k in os.environ if k.startswith("NSM_"))
    if bad:
        sys.exit(f"bench.py: refusing to run with {bad} set (experiment switches; unset them)")


def spawn_command(args, argv, port):
    """The torchrun command line that runs this script on ``args.gpus`` ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def maybe_spawn(args):
    """--gpus N without a torchrun environment: re-exec under torchrun."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    sys.exit(subprocess.call(spawn_command(args, sys.argv[1:], port)))


# --------------------------------------------------------------------------
# distributed plumbing
# --------------------------------------------------------------------------

def dist_setup(backend=None):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if backend is None:
        backend = "nccl"
    if backend == "nccl":
        torch.cuda.set_device(local)
    # a process group whenever torchrun launched us (also at world size 1, so
    # the NCCL timing / --gather path runs on a one-GPU box too)
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        kw = {"device_id": torch.device("cuda", local)} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
    return rank, world, local


def dist_on():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def barrier(world):
    if dist_on():
        import torch.distributed as dist
        dist.barrier()


def gather_floats(vals, world, device):
    """All-gather a small float vector from every rank -> (world, len)."""
    import torch
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=device)
    if not dist_on():
        return t[None].cpu().numpy()
    import torch.distributed as dist
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return torch.stack(out).cpu().numpy()


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


def sustained_tflops():
    """Dense bf16 TFLOP/s sustained under the power cap (the denominator for
    kernels timed inside a long step); the recipe's fallback otherwise."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        if "bf16_tflops_sustained" in j:
            return j["bf16_tflops_sustained"], "measured"
    return 1400.0, "fallback"


# --------------------------------------------------------------------------
# algorithmic cost models ("roofline accounting")
# --------------------------------------------------------------------------

def covered_pixels(inputs):
    return int((inputs["d"] > 0).sum().item())


def kernel_models(frames, inputs, cfg, dtype, features):
    """Per-step algorithmic bytes / flops of the kernels we model."""
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
    if features == 5:
        # blocker pass: G-buffer in, one 4-B texel per covered pixel from
        # HBM (the 16x16 window is served by SMEM / L1), 24 16-bit s2d
        # channels per level-0 pixel out; enc0 reads them back
        models["feat5_blocker"] = {"bytes": 28 * px + 4 * cov + n * l0 * 24 * act, "flops": 0}
        models["enc0_s2d"] = {"bytes": n * l0 * 24 * act + n * (l0 // 4) * 16 * act,
                              "flops": 2 * n * l0 * (16 * 20 * 9 + 16 * 16)}
    step_bytes = 28 * px + 4 * cov + px * act
    step_flops = 2.0 * n * hp * wp * sum(s["flops_per_pixel"] for s in st)
    return models, step_bytes, step_flops


# tensor-core kernels of the 16-bit path -> (level, convolutions they run);
# dec0 = dec0_fused (polyphase tcgen05 interior) + dec0_ring (outer ring)
LEVEL_KERNELS = {
    "enc0_fused": (0, ("enc3", "enc1")), "enc0_s2d": (0, ("enc3", "enc1")),
    "lv1_enc": (1, ("enc3", "enc1")), "lv2_enc": (2, ("enc3", "enc1")), "lv3_bott": (3, ("enc3", "enc1")),
    "lv2_dec": (2, ("dec3", "dec1")), "lv1_dec": (1, ("dec3", "dec1")),
    "dec0_fused+dec0_ring": (0, ("dec3", "dec1", "head")),
}


def kernel_flops(cfg, hp, wp, n):
    """Algorithmic flops (2 x MACs) per step of each tensor-core kernel of
    the fused 16-bit path, from the reference's level plan (network.py:44-118,
    the same per-level terms as net_stats); they sum to the step's flops."""
    from paper_2301_05262_b200 import network
    plan, head = network.level_plan(cfg)
    shift = 1 if cfg.use_space_to_depth else 0
    ks = dict(network._TAGS)
    out = {}
    for name, (j, tags) in LEVEL_KERNELS.items():
        if j >= len(plan):
            continue
        r = (hp >> (j + shift)) * (wp >> (j + shift))
        macs = sum(plan[j][t][0] * plan[j][t][1] * ks[t] ** 2 for t in tags if t in plan[j])
        if "head" in tags:
            macs += head[0] * head[1]
        out[name] = 2.0 * n * macs * r
    return out


def kernel_rooflines(prof, flops, steps, tflops_peak):
    """Achieved TFLOP/s of each modelled tensor-core kernel (eager per-kernel
    profile, CUDA events on the launching stream) against the sustained bf16
    dense peak."""
    rows = {}
    for name, fl in flops.items():
        parts = name.split("+")
        if not all(p in prof for p in parts):
            continue
        ms = sum(prof[p][1] for p in parts) / steps
        t = fl / (ms / 1e3) / 1e12
        rows[name] = {"ms": round(ms, 5), "gflop": round(fl / 1e9, 2), "tflops": round(t, 1),
                      "frac": round(t / tflops_peak, 4)}
    return rows


def ncu_traffic(kernel, algo_bytes, frames_per_launch, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of ``kernel``,
    scaled from the committed ncu --set full capture (profiles/traffic.json,
    written by tools/ncu_summary.py traffic) to this run's frames per launch."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        tab = json.load(f)
    t = tab.get(kernel) if workload == "cfg4-1080p-soft-window8" else tab.get(f"{kernel}@{workload}")
    if not t or t.get("workload") != workload:
        return None
    bpf = t["dram_bytes_per_frame"]
    return {"bytes": int(bpf * frames_per_launch), "algorithmic_bytes": int(algo_bytes),
            "ratio": round(bpf * frames_per_launch / algo_bytes, 3), "source": t["source"]}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def make_plan(args):
    from paper_2301_05262_b200 import network
    cfg = network.NetworkConfig(in_channels=args.features)
    w = network.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))
    return cfg, w, network.Plan(w, cfg, args.dtype)


def time_steps(step, steps, world, soak=True, local=0):
    """Device time per step (CUDA events on the launching stream, barrier +
    synchronize on both sides), with clocks sampled under load."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t_end = time.time() + (1.0 if soak else 0.0)      # ~1 s under load for nvidia-smi
        while time.time() < t_end:
            for _ in range(20):
                step()
            torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        barrier(world)
    return e0.elapsed_time(e1) / steps, clk.summary()


def profile_kernels(launch, steps):
    """{kernel: (launches, total ms)} of ``steps`` eager launches, each
    kernel bracketed by CUDA events on its stream (nsm_profile_*).  A spin
    kernel queued first keeps the GPU busy while the host enqueues every
    launch, so the events measure device time, not host launch latency."""
    import torch
    from paper_2301_05262_b200 import _lib
    torch.cuda.synchronize()
    _lib.lib.nsm_profile_enable(1)
    _lib.profile_report()
    torch.cuda._sleep(int(2e6) * (10 + 4 * steps))      # ~1 ms per step of lead at ~2 GHz
    for _ in range(steps):
        launch()
    torch.cuda.synchronize()
    prof = _lib.profile_report()
    _lib.lib.nsm_profile_enable(0)
    return prof


def run_ours(args):
    import torch
    from paper_2301_05262_b200 import _lib, producer
    from paper_2301_05262_b200.infer import ShadowInference

    if _lib.experiment_build():
        sys.exit("bench.py: libnsm.so is an experiment build (NSM_EXPERIMENTS); rebuild the release library")
    rank, world, local = dist_setup()
    dev = torch.device("cuda", local)
    if dist_on() and rank == 0:
        nv = torch.cuda.nccl.version()
        print(f"bench.py: NCCL {'.'.join(map(str, nv)) if isinstance(nv, tuple) else nv} communicator, "
              f"{world} ranks, one GPU each", file=sys.stderr)
    frames, (lo, hi), job_n, scaling = rank_frames(args, rank, world)
    n = len(frames)
    inputs = producer.render_inputs(frames)
    cfg, w, plan = make_plan(args)
    out_dtype = "fp32" if args.dtype == "fp32" else "fp16"
    run = ShadowInference(plan, frames, out_dtype=out_dtype)
    run(inputs)                                  # validates frustum, warms up
    torch.cuda.synchronize()
    h, wd = frames[0].camera.resolution

    c0 = _lib.lib.nsm_launch_count()
    if args.no_graph:
        step = lambda: run.launch(inputs, check=False)        # noqa: E731
        run.launch(inputs)
        per_step = _lib.lib.nsm_launch_count() - c0
    else:
        run.capture(inputs)
        per_step = (_lib.lib.nsm_launch_count() - c0) // 2   # warm launch + captured launch
        step = run.replay
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ms, clocks = time_steps(step, args.steps, world, soak=not args.no_soak, local=local)
    per_rank = gather_floats([ms, n], world, dev)
    ms_max = float(per_rank[:, 0].max())
    value = job_n / (ms_max / 1e3)

    gathered = None
    if args.gather and dist_on():
        from paper_2301_05262_b200 import shard
        import torch.distributed as dist
        full = shard.gather_frames(run.y, job_n if scaling == "strong" else n * world)
        # every rank re-derives the rank-0 shard's checksum: frame order proof
        gathered = {"frames": int(full.shape[0]), "checksum": float(full.double().sum().item()),
                    "rank0_shard_equal": bool(torch.equal(full[:hi - lo], run.y) if rank == 0 else True)}
        dist.barrier()

    # ---- per-kernel timing (eager, traced launches on the same stream) ----
    prof = profile_kernels(lambda: run.launch(inputs, check=False), args.steps)
    models, step_bytes, step_flops = kernel_models(frames, inputs, cfg, args.dtype, args.features)
    hbm, tfl, src = peaks()
    tsus, tsrc = sustained_tflops()
    kflops = (kernel_flops(cfg, (h + 15) // 16 * 16, (wd + 15) // 16 * 16, n)
              if args.dtype != "fp32" else {})
    dom = max(prof, key=lambda k: prof[k][1]) if prof else None
    step_prof_ms = sum(v[1] for v in prof.values()) / max(args.steps, 1)
    # the roofline names the dominant kernel we have an algorithmic model for
    modelled = [k for k in prof if k in models]
    rk = max(modelled, key=lambda k: prof[k][1]) if modelled else None
    roof = None
    if rk is not None:
        cnt, tot = prof[rk]
        launches_per_step = max(1, cnt // args.steps)
        avg_ms = tot / cnt
        mb = models[rk]["bytes"] / launches_per_step
        ach = mb / (avg_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": rk, "achieved": round(ach, 1), "peak": hbm,
                "unit": "GB/s", "frac": round(ach / hbm, 4),
                "traffic": ncu_traffic(rk, mb, n // launches_per_step, workload_name(args)),
                "avg_launch_ms": round(avg_ms, 5), "peak_source": src,
                "algorithmic_bytes_per_launch": int(mb),
                "share_of_step": round(tot / args.steps / step_prof_ms, 3),
                "dominant_kernel": dom}

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, run, inputs, frames, job_n, world)

    # ---- variants measured in the same run: the fully covered camera (a
    # typical game G-buffer) and the same frames with the 5-plane net
    # (16x16 blocker search, BASELINE configs 3/4) or the 4-plane one ----
    variants = None
    if not args.no_variants and args.cover == "scene" and args.config in (2, 3, 4):
        variants = {}

        def timed(vframes, vplan, label, extra):
            vin = producer.render_inputs(vframes)
            vrun = ShadowInference(vplan, vframes, out_dtype=out_dtype)
            vrun(vin)
            vrun.capture(vin)
            for _ in range(3):
                vrun.replay()
            vms, _ = time_steps(vrun.replay, args.steps, world, soak=False, local=local)
            vms_max = float(gather_floats([vms], world, dev)[:, 0].max())
            vprof = profile_kernels(lambda: vrun.launch(vin, check=False), 3)
            variants[label] = {"value": round(job_n / (vms_max / 1e3), 3), "unit": UNIT,
                               "ms_per_step": round(vms_max, 5),
                               "coverage": round(covered_pixels(vin) / (len(vframes) * h * wd), 4),
                               "kernel_profile_ms_per_step": {k: round(v[1] / 3, 5) for k, v in
                                                              sorted(vprof.items(), key=lambda kv: -kv[1][1])},
                               **extra}

        timed([full_cover_frame(f) for f in frames], plan, "full_coverage",
              {"features": args.features})
        other = 5 if args.features == 4 else 4
        oargs = argparse.Namespace(**{**vars(args), "features": other})
        _, _, oplan = make_plan(oargs)
        timed(frames, oplan, "blocker_search_5plane" if other == 5 else "reference_4plane",
              {"features": other, "network": f"NetworkConfig(in_channels={other})"})
        torch.cuda.synchronize()
        variants["torch_cudnn_comparator"] = torch_comparator(args, w, frames, inputs, world, dev, local, job_n)

    # ---- bf16 precision record (config 5's dtype cannot meet the 1e-2
    # max-abs bar at large emitters, see tests/test_gpu_f16.py): the bf16
    # visibility of this rank's first frames against the fp16 plan's, which
    # the tests hold within 1e-2 / 1e-4 of the fp32 oracle ----
    precision = None
    if args.dtype == "bf16" and not args.no_variants:
        sub = frames[:2]
        sin = {k: v[:len(sub)].contiguous() for k, v in inputs.items()}
        fargs = argparse.Namespace(**{**vars(args), "dtype": "fp16"})
        _, _, fplan = make_plan(fargs)
        yb = ShadowInference(plan, sub, out_dtype="fp32")(sin).double()
        yf = ShadowInference(fplan, sub, out_dtype="fp32")(sin).double()
        d = yb - yf
        precision = {"bf16_vs_fp16_plan_max_abs": round(float(d.abs().max()), 5),
                     "bf16_vs_fp16_plan_mse": float((d * d).mean()),
                     "frames": [f"size_index {f.size_index:.2f}" for f in sub],
                     "bars": "fp16 meets 1e-2 max-abs / 1e-4 MSE vs the fp32 oracle; bf16 meets MSE only "
                             "(4K size_index 8: see tests/test_gpu_f16.py)"}
        del yb, yf, fplan

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        planes = {k: v[0].cpu().numpy() for k, v in inputs.items()}
        cpu = cpu_leg(args, [frames[0]], [planes], reps=1 if args.config == 5 else 3)

    if rank == 0:
        line = {
            "metric": metric_name(args.config), "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms_max, 5),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": {"fp16": "f16", "bf16": "bf16", "fp32": "f32"}[args.dtype],
            "data": "synthetic (procedural scenes rendered on-GPU; random-init weights)",
            "config": {"workload": workload_name(args), "job_frames": job_n,
                       "frames_per_rank": [int(v) for v in per_rank[:, 1]],
                       "resolution": [h, wd], "net_resolution": [(h + 15) // 16 * 16, wd],
                       "shadow_map": list(frames[0].view.resolution),
                       "network": f"NetworkConfig(layers=5, base=16, in={args.features}, s2d) "
                                  f"{sum(int(np.asarray(v.data).size) for v in w.values()):,} params",
                       "features": args.features,
                       "precision": plan.precision,
                       "coverage": round(covered_pixels(inputs) / (n * h * wd), 4),
                       "l2": "inputs > L2 (no flush needed)",
                       "graph": not args.no_graph,
                       "parallelism": f"frames-dp{world} ({'sharded job' if scaling == 'strong' else 'one job per rank'})"},
            "mpix_per_s": round(value * h * wd / 1e6, 2),
            "per_rank_ms": [round(float(v), 5) for v in per_rank[:, 0]],
            "roofline": roof,
            "step_roofline": {"bytes": int(step_bytes), "flops": step_flops,
                              "gbps": round(step_bytes / (ms / 1e3) / 1e9, 1),
                              "tflops": round(step_flops / (ms / 1e3) / 1e12, 2)},
            "kernel_profile_ms_per_step": {k: round(v[1] / args.steps, 5) for k, v in
                                           sorted(prof.items(), key=lambda kv: -kv[1][1])},
            "kernel_rooflines": {"peak_tflops": tsus, "peak": "bf16 dense sustained (" + tsrc + ")",
                                 "kernels": kernel_rooflines(prof, kflops, args.steps, tsus)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "variants": variants,
            "precision": precision,
            "gathered": gathered,
            "gpu_launches": int(per_step * args.steps),
            "clocks": clocks,
        }
        print(json.dumps(line))
    if dist_on():
        import torch.distributed as dist
        dist.destroy_process_group()


def torch_comparator(args, w, frames, inputs, world, dev, local, job_n):
    """The obvious library path, as a yardstick (hard part 7): the
    same network in PyTorch ops (cuDNN convolutions, channels-last, fp16,
    one CUDA graph) on feature planes computed beforehand by nsm_features --
    i.e. the U-Net alone, without the feature pass our fused path includes.
    Not the product and not a bar."""
    import torch
    import torch.nn.functional as F
    from paper_2301_05262_b200.raster import assemble_features_batch
    if args.features != 4 or args.dtype != "fp16":
        return None
    torch.backends.cudnn.benchmark = True
    h, wd = frames[0].camera.resolution
    hp = (h + 15) // 16 * 16
    feats, _, _ = assemble_features_batch(inputs, [(f.camera, f.view, f.scene.emitter_center, f.size_index,
                                                    f.bias) for f in frames])
    x = torch.zeros((len(frames), 4, hp, wd), dtype=torch.float16, device=dev)
    x[:, :, :h] = feats.half()
    x = x.contiguous(memory_format=torch.channels_last)
    W = {k: torch.from_numpy(np.asarray(v.data)).to(dev).half() for k, v in w.items()}
    W = {k: (v.contiguous(memory_format=torch.channels_last) if v.dim() == 4 else v) for k, v in W.items()}

    def conv(t, n, relu=True):
        wt = W[n + ".w"]
        y = F.conv2d(t, wt, W[n + ".b"], padding=wt.shape[-1] // 2)
        return F.relu(y) if relu else y

    def net(t):
        t = F.pixel_unshuffle(t, 2)
        skips = []
        for j in range(3):
            t = conv(conv(t, f"l{j}.enc3"), f"l{j}.enc1")
            skips.append(t)
            t = F.avg_pool2d(t, 2)
        t = conv(conv(t, "l3.enc3"), "l3.enc1")
        for j in (2, 1, 0):
            t = F.interpolate(t, scale_factor=2, mode="bilinear", align_corners=False)
            if j > 0:
                t = t + skips[j]
            t = conv(conv(t, f"l{j}.dec3"), f"l{j}.dec1")
        y = conv(t, "head", relu=False)
        base = F.interpolate(y[:, :1], scale_factor=2, mode="bilinear", align_corners=False)
        det = y.clone()
        det[:, 0] = 0
        return torch.sigmoid(base + F.pixel_shuffle(det, 2))

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            net(x)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = net(x)
    for _ in range(3):
        g.replay()
    ms, _ = time_steps(g.replay, args.steps, world, soak=False, local=local)
    ms_max = float(gather_floats([ms], world, dev)[:, 0].max())
    return {"value": round(job_n / (ms_max / 1e3), 3), "unit": UNIT, "ms_per_step": round(ms_max, 5),
            "what": "PyTorch/cuDNN fp16 U-Net only (features precomputed, CUDA graph, channels-last)",
            "output_shape": list(out.shape)}


def run_e2e(args, run, inputs, frames, job_n, world):
    """The same metric through infer.HostPipeline.submit: pinned host
    inputs -> H2D (copy stream) -> fused kernels -> D2H of the visibility,
    overlapped across consecutive batches; each batch carries its frames."""
    import torch
    from paper_2301_05262_b200.infer import HostPipeline
    host = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in inputs.items()}
    for k in host:
        host[k].copy_(inputs[k])
    yh = torch.empty(run.y.shape, dtype=run.y.dtype, pin_memory=True)
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    d2h = yh.numel() * yh.element_size()
    table = run.frame_table(frames)
    pipe = HostPipeline(run)
    for _ in range(2):
        pipe.submit(host, yh, frames=table)
    pipe.synchronize()
    torch.cuda.synchronize()
    k2 = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    e0.record(pipe.h2d)
    for _ in range(k2):
        pipe.submit(host, yh, frames=table)
    e1.record(pipe.d2h)
    pipe.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    ems = float(gather_floats([e0.elapsed_time(e1) / k2], world, run.y.device)[:, 0].max())
    return {"value": round(job_n / (ems / 1e3), 3), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d * world), "d2h_bytes_per_step": int(d2h * world),
            "ms_per_step": round(ems, 4), "steps": k2,
            "api": "infer.HostPipeline.submit (pinned host in/out, per-batch frames, copies overlapped)"}


# --------------------------------------------------------------------------
# CPU legs: the reference's own code (oracle/_ref) or the oracle port
# --------------------------------------------------------------------------

def _stock():
    """The staged reference package (oracle/_ref/shadowkit) or None."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "shadowkit")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import shadowkit
    return shadowkit


def _blas_info():
    try:
        from threadpoolctl import threadpool_info
        return [{k: d.get(k) for k in ("internal_api", "num_threads", "version")}
                for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception as e:      # noqa: BLE001
        return [f"threadpoolctl unavailable: {e}"]


def _cpu_frame_fn(args, fr, planes):
    """One frame of the reference algorithm: stage 1 + stage 2 (padded to
    1088 rows as the GPU path pads, cropped back).  Returns (callable, kind,
    what)."""
    from oracle import features as of
    from oracle import network as on
    h, w = fr.camera.resolution
    hp, wp = (h + 15) // 16 * 16, (w + 15) // 16 * 16
    sk = _stock()
    if args.features == 5:
        from oracle import blocker as ob
    if sk is not None:
        from shadowkit import autodiff as ad, network as skn, raster as skr, scene as sks
        cam = sks.CameraPose(fr.camera.position, fr.camera.forward, fr.camera.up, fr.camera.fov_y,
                             fr.camera.resolution)
        view = skr.EmitterView(np.asarray(fr.view.position), np.asarray(fr.view.forward),
                               np.asarray(fr.view.up), np.asarray(fr.view.right), float(fr.view.tan_half),
                               tuple(fr.view.resolution))
        z_f, c_e, c_c, cov = of.derive_planes(planes["d"], planes["normal"], planes["position"], fr.camera,
                                              fr.scene.emitter_center)
        g = skr.GBuffer(d=planes["d"].astype(np.float64), normal=planes["normal"].astype(np.float64),
                        position=planes["position"].astype(np.float64), n_e=None, z_f=z_f, c_e=c_e,
                        c_c=c_c, coverage=cov, camera=cam)
        sm = skr.ShadowMap(depth=planes["sm"].astype(np.float64), view=view,
                           scene_diag=float(fr.bias) / skr.DEFAULT_BIAS_FACTOR)
        cfg = skn.NetworkConfig(in_channels=args.features)
        wts = skn.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11])))

        def one():
            with ad.no_grad():
                fs = skr.assemble_features(g, sm, float(fr.size_index), float(fr.bias))
                x = np.zeros((args.features, hp, wp), np.float32)
                x[:4, :h, :w] = fs.data
                if args.features == 5:
                    x[4, :h, :w] = ob.blocker_plane(planes["d"], planes["position"], z_f, cov, planes["sm"],
                                                    fr.view, fr.bias, fr.size_index, fr.camera.focal_px)
                return skn.forward(wts, cfg, x).data[:, :h, :w]
        what = "shadowkit raster.assemble_features + network.forward (no_grad)"
        if args.features == 5:
            what += " + oracle blocker plane"
        return one, "reference", what

    from paper_2301_05262_b200 import network as pn
    cfg = pn.NetworkConfig(in_channels=args.features)
    W = {k: v.data for k, v in pn.init_weights(cfg, np.random.default_rng(np.random.SeedSequence([0, 0x11]))).items()}

    def one():
        feats, cov = of.features_from_planes(planes["d"], planes["normal"], planes["position"], planes["sm"],
                                             fr.camera, fr.view, fr.scene.emitter_center, fr.size_index, fr.bias)
        x = np.zeros((args.features, hp, wp), np.float32)
        x[:4, :h, :w] = feats
        if args.features == 5:
            z_f, _, _, _ = of.derive_planes(planes["d"], planes["normal"], planes["position"], fr.camera,
                                            fr.scene.emitter_center)
            x[4, :h, :w] = ob.blocker_plane(planes["d"], planes["position"], z_f, cov, planes["sm"], fr.view,
                                            fr.bias, fr.size_index, fr.camera.focal_px)
        return on.forward(W, x)[:, :h, :w]
    return one, "port", "oracle port of assemble_features + forward (numpy)"


def cpu_leg(args, frames, planes, reps=3):
    """Best-of-``reps`` seconds per frame of the reference algorithm on the
    host cores (BLAS capped at the process's affinity set)."""
    cores = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_limits
        limit = threadpool_limits(limits=cores)
    except Exception:          # noqa: BLE001
        limit = None
    fns = [_cpu_frame_fn(args, fr, p) for fr, p in zip(frames, planes)]
    best = float("inf")
    for r in range(reps):
        t = time.perf_counter()
        for fn, _, _ in fns:
            fn()
        best = min(best, (time.perf_counter() - t) / len(fns))
    info = _blas_info()
    if limit is not None:
        limit.restore_original_limits()
    _, kind, what = fns[0]
    return {"value": round(1.0 / best, 4), "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{len(fns)} frame(s) of the workload, best of {reps}: {what}; "
                      f"{best:.2f} s/frame", "blas": info}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import producer as op
    frames = job_frames(args, seed=0)
    sample = frames[:2] if args.config == 5 else frames[:1]       # config 5: one hard + one soft scene
    t = time.perf_counter()
    planes = [op.render_inputs_banded(f.scene.primitive_table(), f.camera, f.view) for f in sample]
    t_render = time.perf_counter() - t
    cores = len(os.sched_getaffinity(0))
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=cores):
        fns = [_cpu_frame_fn(args, fr, p) for fr, p in zip(sample, planes)]
        warm = min(args.warmup, 1)
        cap = 2 if args.config == 5 else 5
        steps = max(1, min(args.steps, cap))
        for i in range(warm):
            fns[i % len(fns)][0]()
        t = time.perf_counter()
        for i in range(steps):
            fns[i % len(fns)][0]()
        el = time.perf_counter() - t
        info = _blas_info()
    value = steps / el
    kind, what = fns[0][1], fns[0][2]
    h, wd = frames[0].camera.resolution
    print(json.dumps({
        "metric": metric_name(args.config), "value": round(value, 4), "unit": UNIT, "impl": "reference",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": steps, "warmup": warm,
        "ms_per_step": round(el / steps * 1e3, 2), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (the same seeded scenes and weights as ours; inputs ray-cast on the CPU)",
        "config": {"workload": workload_name(args), "resolution": [h, wd], "features": args.features,
                   "note": f"one frame per step (bounded sample), steps capped at {cap} (asked {args.steps}); "
                           f"inputs rendered in {t_render:.1f} s, untimed"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{len(sample)} frame(s) of the workload cycled: {what}", "blas": info},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "mpix_per_s": round(value * h * wd / 1e6, 4),
    }))


if __name__ == "__main__":
    a = parse()
    env_guard()
    if a.impl == "reference":
        run_reference(a)
    else:
        maybe_spawn(a)
        run_ours(a)
