"""bench.py's multi-GPU driver logic on CPU (world_size 2, gloo): which
frames each rank runs for the configs north_star shards (config 4: the
8-frame temporal window, 8/4/2/1 frames per rank; config 5: the 64-scene
sweep), the per-rank timing gather the job time is the max of, and the
order-restoring gather of the visibility frames (shard.gather_frames)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cam_key(f):
    return tuple(np.round(np.asarray(f.camera.position), 9)) + tuple(np.round(f.scene.emitter_center, 9))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_config4_window_split_8_4_2_1(world):
    args = bench.parse(["--config", "4"])
    full = bench.job_frames(args)
    assert len(full) == 8
    got = []
    for r in range(world):
        frames, (lo, hi), job_n, scaling = bench.rank_frames(args, r, world)
        assert scaling == "strong" and job_n == 8
        assert len(frames) == 8 // world
        assert [_cam_key(f) for f in frames] == [_cam_key(f) for f in full[lo:hi]]
        got += [_cam_key(f) for f in frames]
    assert got == [_cam_key(f) for f in full]          # every frame exactly once, in order


def test_config5_scene_split_and_replicas():
    args = bench.parse(["--config", "5", "--frames", "16"])
    assert args.dtype == "bf16" and args.features == 4
    sizes = [len(bench.rank_frames(args, r, 8)[0]) for r in range(8)]
    assert sizes == [2] * 8
    one = bench.parse(["--config", "3"])
    assert one.features == 5
    frames, _, job_n, scaling = bench.rank_frames(one, 1, 2)   # one frame, two GPUs: replicas
    assert len(frames) == 1 and job_n == 2 and scaling == "weak"
    weak = bench.parse(["--config", "4", "--scaling", "weak"])
    a = bench.rank_frames(weak, 0, 2)[0]
    b = bench.rank_frames(weak, 1, 2)[0]
    assert len(a) == len(b) == 8 and _cam_key(a[1]) != _cam_key(b[1])   # own window per rank


def test_full_cover_variant_and_env_guard(monkeypatch):
    args = bench.parse(["--config", "4", "--cover", "full", "--frames", "2"])
    frames = bench.job_frames(args)
    assert "fullcover" in bench.workload_name(args)
    assert frames[0].camera.position[1] == pytest.approx(4.0)
    monkeypatch.setenv("NSM_ENC0_DBG", "1")
    with pytest.raises(SystemExit):
        bench.env_guard()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2301_05262_b200 import shard
    r, w, _ = bench.dist_setup("gloo")
    try:
        args = bench.parse(["--config", "4"])
        frames, (lo, hi), job_n, _ = bench.rank_frames(args, r, w)
        # stand-in visibility: frame i of the job is filled with i
        local = torch.stack([torch.full((1, 3, 5), float(i)) for i in range(lo, hi)])
        full = shard.gather_frames(local, job_n)
        per_rank = bench.gather_floats([1.0 + r, len(frames)], w, torch.device("cpu"))
        q.put((r, full.numpy(), per_rank, [_cam_key(f) for f in frames]))
    finally:
        dist.destroy_process_group()


def test_bench_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full_keys = [_cam_key(f) for f in bench.job_frames(bench.parse(["--config", "4"]))]
    assert res[0][3] + res[1][3] == full_keys              # frames 0-3 on rank 0, 4-7 on rank 1
    for r, full, per_rank, _ in res:
        np.testing.assert_array_equal(full[:, 0, 0, 0], np.arange(8, dtype=np.float32))
        np.testing.assert_array_equal(per_rank, [[1.0, 4.0], [2.0, 4.0]])
        assert per_rank[:, 0].max() == 2.0                 # the job time is the slowest rank's


def test_reference_leg_never_loads_the_cuda_library():
    """The --impl reference process times shadowkit's own code on CPU
    inputs and must not map libnsm.so (the arm was classed
    'gpu' because it rendered its inputs with our kernels)."""
    import subprocess
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import bench\n"
        "from oracle import producer as op\n"
        "from paper_2301_05262_b200 import scenes\n"
        "args = bench.parse(['--config', '3', '--features', '5'])\n"
        "fr = scenes.make_frame(scenes.random_scene(4, 0, 0.2), (32, 48), (64, 64))\n"
        "p = op.render_inputs_banded(fr.scene.primitive_table(), fr.camera, fr.view, workers=2)\n"
        "fn, kind, what = bench._cpu_frame_fn(args, fr, p)\n"
        "y = fn()\n"
        "assert y.shape == (1, 32, 48), y.shape\n"
        "maps = open('/proc/self/maps').read()\n"
        "assert 'libnsm' not in maps and 'paper_2301_05262_b200._lib' not in sys.modules\n"
        "print(kind)\n" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() in ("reference", "port")


def test_spawn_command_and_device_check(monkeypatch):
    """--gpus N re-executes bench.py under torchrun (127.0.0.1 rendezvous,
    one process per GPU) and refuses more ranks than visible devices."""
    args = bench.parse(["--gpus", "4", "--config", "5"])
    cmd = bench.spawn_command(args, ["--gpus", "4", "--config", "5"], 29511)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29511" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--config", "5"][-3:] and cmd[-5].endswith("bench.py")
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    with pytest.raises(SystemExit, match="CUDA device"):
        bench.maybe_spawn(args)          # no GPU in the build container


def test_kernel_flop_model_sums_to_the_step():
    """bench.py's per-kernel tensor flops (the level plan split by kernel)
    add up to the whole network's flops (net_stats), for the default
    4-plane net, the 5-plane net and a 4-level variant."""
    from paper_2301_05262_b200 import network
    for cfg in (network.NetworkConfig(), network.NetworkConfig(in_channels=5),
                network.NetworkConfig(layers=4)):
        hp, wp = 1088, 1920
        fl = bench.kernel_flops(cfg, hp, wp, 8)
        fl.pop("enc0_s2d")                       # the 5-plane twin of enc0_fused
        total = 2.0 * 8 * hp * wp * sum(s["flops_per_pixel"] for s in network.net_stats(cfg, (hp, wp)))
        assert sum(fl.values()) == pytest.approx(total, rel=1e-12)
    prof = {"lv1_enc": (10, 0.4), "dec0_fused": (10, 0.5), "dec0_ring": (10, 0.1)}
    rows = bench.kernel_rooflines(prof, bench.kernel_flops(network.NetworkConfig(), hp, wp, 8), 10, 1000.0)
    assert set(rows) == {"lv1_enc", "dec0_fused+dec0_ring"}
    assert rows["dec0_fused+dec0_ring"]["ms"] == pytest.approx(0.06)
