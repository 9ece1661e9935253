"""Benchmark: env-steps/s (fwd+bwd) of the quadsim hot path on B200.

Headline workload (BASELINE.json configs[1], C2): full rigid-body quadrotor +
IMU noise, position task, 65,536 envs per GPU, BPTT windows of T=32 steps
(forward: fused env-step kernel; backward: analytic VJP kernel), open-loop
synthetic actions N(0, 0.3^2).  One bench "step" = one window fwd+bwd.
Secondary: depth rays/s for C3 (16,384 envs, 64x48 camera, 32 solids + ground).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: one process per GPU under torchrun; envs shard across ranks with
no communication inside the sim step (weak scaling); timing is the max over
ranks of CUDA-event time.  ``--impl reference`` times the CPU oracle port of
the same workload (numpy fp64, reference algorithm incl. its reverse pass) on
all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "env-steps/s (fwd+bwd)"
UNIT = "env-steps/s"
IMU = dict(accel_noise_std=0.1, gyro_noise_std=0.01, accel_bias_rw_std=0.01, gyro_bias_rw_std=0.001)

# Algorithmic bytes per env-step, SURVEY.md §8(d) (the fused env.step boundary,
# fp32 unpadded), full quadrotor + IMU, open-loop BPTT:
#   fwd 234 B (reads S 52, v_ema 12, raw 16, goal 12, prev effort 16, counter 4;
#       writes S 52, v_ema 12, obs 48, rewards 12, effort 16, flags 2, counter 4)
#       + IMU 72 B (bias read+write 48, readings 24)                     = 306
#   bwd 265 B - 48 B (open loop: no dL/dobs)                 = 217
FWD_BYTES = 306
BWD_BYTES = 217
# the fused-window kernels keep state/effort/counters/IMU bias on chip across
# the T steps; the payload they MUST move per env-step is smaller:
#   fwd: raw 16 + checkpoint state 52 + goal 12 + effort 16 + obs 48 + rewards 12
#        + term/trunc 2 + flags 4 + IMU 24 = 186;  bwd: 52 + 16 + 12 + 16 + 4 + 16 = 116
FWD_BYTES_FUSED = 186
BWD_BYTES_FUSED = 116


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=65536)
    ap.add_argument("--horizon", type=int, default=32)
    ap.add_argument("--model", default="full")
    ap.add_argument("--no-depth", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-imu", action="store_true", help="diagnostic: full model without the IMU")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no cpu/clock sampling)")
    ap.add_argument("--net-dtype", default="bf16", choices=["bf16", "fp32"],
                    help="C5: the policy / critic arithmetic (bf16 tensor-core kernels, or torch fp32)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c5"],
                    help="c2: headline BPTT windows; c5: SHAC training with NCCL gradient all-reduce")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (reference algorithm, numpy fp64)


def _cpu_worker(args):
    n_envs, T, model, seconds, seed = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import quadsim_oracle as O

    cfg = O.Config(task="position", dynamics=model, n_envs=n_envs, episode_len=128, dt=0.05)
    env = O.OracleTask(cfg, imu=dict(IMU, seed=seed))
    env.reset(seed)
    rng = np.random.default_rng(seed)
    A = O.MODEL_ACTION_DIM[model]
    done_steps = 0
    t0 = time.perf_counter()
    while True:
        acts = rng.normal(size=(T, n_envs, A)) * 0.3
        O.window_value_and_grad(env, acts)
        done_steps += n_envs * T
        el = time.perf_counter() - t0
        if el >= seconds:
            return done_steps, el


REF_PKG = os.path.join(ROOT, "baseline", "_ref")  # the reference package (pip --target)


def have_ref_pkg() -> bool:
    return os.path.isdir(os.path.join(REF_PKG, "quadsim"))


def _ref_worker(args):
    """The REFERENCE's own code on the C2 workload: quadsim's position task with
    the full quadrotor (FlightTask.step recorded on its Tape), the discounted
    BPTT loss and Tape.backward (q/learners.py:201-265), plus one
    ImuModel.read per step with C2's noise (q/sensors.py:508-555; the
    reference's tasks do not wire the IMU, so the window calls it after each
    step on the post-step state)."""
    n_envs, T, seconds, seed = args
    os.environ["OMP_NUM_THREADS"] = "1"
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    from quadsim import autodiff as ad
    from quadsim import dynamics as rdyn
    from quadsim import sensors as rsn
    from quadsim import tasks as rtk
    from quadsim.autodiff import Tape

    env = rtk.make_task(rtk.TaskConfig(task="position", dynamics="full", n_envs=n_envs, episode_len=128))
    env.reset(seed=seed)
    imu = rsn.ImuModel(n_envs, seed=seed, **IMU)
    g = env.params.g_vec
    dt = env.config.dt
    rng = np.random.default_rng(seed)
    done_steps = 0
    t0 = time.perf_counter()
    while True:
        raw = rng.normal(size=(T, n_envs, 4)) * 0.3
        tape = Tape()
        leaves = [tape.leaf(raw[t].copy()) for t in range(T)]
        env.detach_states()
        disc = None
        for t in range(T):
            out = env.step(leaves[t])
            term = ad.mul(ad.vmean(out.r_ctrl), 0.99 ** t)
            disc = term if disc is None else ad.add(disc, term)
            st = env.state
            imu.read(rdyn.quat_to_matrix_np(st.q.value), st.w.value, env.last_v_dot, g, dt)
            if out.done.any():
                imu.reset(out.done)
        tape.backward(ad.neg(ad.mul(disc, 1.0 / T)))
        done_steps += n_envs * T
        el = time.perf_counter() - t0
        if el >= seconds:
            return done_steps, el


def reference_continuity():
    """BASELINE.md §4 continuity points: the reference's own `quadsim bench`
    harness (q/cli.py:202-256, median of 5 after 3 warm-ups, 1 process),
    unchanged: raw full-model stepping at 8,192 envs and 64x64 depth frames."""
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    from quadsim import cli as rcli

    n = 8192
    phys = rcli.bench_physics("full", n, max(2, min(50, 40_000 // n)), 5, 3)
    depth = rcli.bench_depth(64, 1, 5, 3)  # 1 frame per trial (the harness's 10 take 80 s here)
    return {"bench_physics_full_8192_steps_per_s": phys, "bench_depth_64x64_64envs_images_per_s": depth,
            "rays_per_s": depth * 64 * 64, "harness": "quadsim.cli.bench_physics / bench_depth (q/cli.py:202-256)",
            "cores": 1}


def _cpu_depth_worker(args):
    """C3 depth on the host: the oracle's render_depth (the reference's
    algorithm: fov cull, then every kept solid per ray, fp64) over a few
    in-corridor courses of the C3 distribution, random poses and yaws."""
    n_envs, seconds, seed = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import quadsim_oracle as O

    spawn, goal = np.array([0.0, 0.0, 1.2]), np.array([8.0, 0.0, 1.5])
    scenes = [O.gen_obstacle_course(seed * 1000 + i, spawn, goal, 32 / 48.0) for i in range(n_envs)]
    prims = O.pack_primitives([sc.prims for sc in scenes])
    rng = np.random.default_rng(seed)
    rays = 0
    t0 = time.perf_counter()
    while True:
        pos = np.stack([rng.uniform(0, 8, n_envs), rng.uniform(-3, 3, n_envs), rng.uniform(0.5, 3.5, n_envs)], -1)
        O.render_depth(prims, pos, O.rotz(rng.uniform(0, 2 * np.pi, n_envs)), 64, 48, 10.0)
        rays += n_envs * 64 * 48
        el = time.perf_counter() - t0
        if el >= seconds:
            return rays, el


def cpu_baseline(seconds: float, model: str, T: int, n_sample: int = 4096, extras: bool = True):
    cores = len(os.sched_getaffinity(0))
    per = max(1, n_sample // cores)
    ctx = mp.get_context("fork")
    if have_ref_pkg() and model == "full":  # the reference package itself
        with ctx.Pool(cores) as pool:
            res = pool.map(_ref_worker, [(per, T, seconds, 1000 + i) for i in range(cores)])
        steps = sum(r[0] for r in res)
        wall = max(r[1] for r in res)
        out = {"value": steps / wall, "unit": UNIT, "cores": cores, "kind": "reference",
               "sample": f"{cores} procs x {per} envs: the reference package (quadsim, baseline/_ref) position "
                         f"task, full quadrotor, T={T} windows of FlightTask.step on its Tape + Tape.backward + "
                         f"ImuModel.read per step, fp64, for {wall:.1f}s"}
        if extras:
            out["continuity"] = reference_continuity()
        return out
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_worker, [(per, T, model, seconds, 1000 + i) for i in range(cores)])
        # depth (the metric's second half): 16 courses per process, 64x48
        dres = pool.map(_cpu_depth_worker, [(16, max(2.0, seconds / 3), 7 + i) for i in range(cores)]) \
            if extras else None
    steps = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    out = {"value": steps / wall, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"{cores} procs x {per} envs, {model}+IMU position task, T={T} windows fwd+bwd "
                     f"(numpy fp64 oracle incl. reverse pass) for {wall:.1f}s"}
    if not extras:
        return out
    # one process, same per-process sample (report both)
    one = _cpu_worker((per, T, model, max(2.0, seconds / 3), 999))
    return {"value": steps / wall, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{cores} procs x {per} envs, {model}+IMU position task, T={T} windows fwd+bwd "
                      f"(numpy fp64 oracle incl. reverse pass) for {wall:.1f}s",
            "single_process": {"value": one[0] / one[1], "unit": UNIT, "cores": 1,
                               "sample": f"1 proc x {per} envs for {one[1]:.1f}s"},
            "depth": {"value": sum(r[0] for r in dres) / max(r[1] for r in dres), "unit": "rays/s",
                      "cores": cores, "kind": "port",
                      "sample": f"{cores} procs x 16 C3 courses (32/48 density), 64x48 depth, random corridor "
                                f"poses, oracle render_depth with the reference's fov_cull (fp64)"}}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    """SM clock + throttle reasons sampled every 20 ms through NVML while the
    timed region runs (the same counters nvidia-smi reports)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.result = None
        self._stop = False

    def _loop(self):
        import pynvml as nv

        h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
        self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop:
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                self.masks.append(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        import threading

        self.sm, self.masks, self.max_mhz = [], [], None
        try:
            import pynvml as nv

            nv.nvmlInit()
            dev = os.environ.get("CUDA_VISIBLE_DEVICES")
            if dev and dev.split(",")[0].isdigit():
                self.gpu = int(dev.split(",")[self.gpu]) if self.gpu < len(dev.split(",")) else self.gpu
            self.th = threading.Thread(target=self._loop, daemon=True)
            self.th.start()
        except Exception as ex:  # pragma: no cover
            self.th = None
            self.result = {"error": str(ex)}
        return self

    def __exit__(self, *a):
        if getattr(self, "th", None) is None:
            return
        self._stop = True
        self.th.join(timeout=2)
        if self.sm:
            reasons = sorted({n for m in self.masks for n, b in self.REASONS.items() if m & b})
            self.result = {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz,
                           "reasons": reasons, "samples": len(self.sm), "source": "NVML during timed region"}


# ---------------------------------------------------------------------------


def spawn_ranks(n: int):
    """``bench.py --gpus N`` without a launcher: re-exec this command under
    torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous),
    exactly as the driver launches it."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


DIST = {"backend": None, "shared_gpu": False}


def dist_init():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank.  With fewer GPUs than ranks (a 1-GPU box running
    # --gpus 2) the ranks share GPUs over gloo: the multi-rank control flow
    # runs, but such a line's throughput is not a scaling measurement
    # ("shared_gpu": true in the JSON line).  BENCH_DIST_BACKEND overrides.
    ndev = max(1, torch.cuda.device_count())
    DIST["shared_gpu"] = world > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("BENCH_DIST_BACKEND", "gloo" if DIST["shared_gpu"] else "nccl")
        DIST["backend"] = backend
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def time_graph(fn, iters: int) -> float:
    import torch

    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def fov_kept_counts(sc, pos, cs, cam):
    """Per-env counts of the solids the reference's own fov_cull keeps
    (q/sensors.py:338-374: bounding sphere vs the 4 frustum planes + behind
    plane, and the range ball), for the culled flops/ray figure SURVEY §8d
    asks to headline.  Yaw-only camera at pos (no offset)."""
    import torch

    th, tv = float(np.tan(cam.fov_h / 2)), float(np.tan(cam.fov_v / 2))
    nrm = torch.tensor([[th, -1.0, 0.0], [th, 1.0, 0.0], [tv, 0.0, -1.0], [tv, 0.0, 1.0], [1.0, 0.0, 0.0]],
                       dtype=torch.float64, device=pos.device)
    nrm = nrm / nrm.norm(dim=-1, keepdim=True)
    p = pos[:, :3].double()
    c, s_ = cs[:, 0].double(), cs[:, 1].double()

    def keep(cen, rad, valid):
        rel = cen.double() - p[:, None, :]
        loc = torch.stack([c[:, None] * rel[..., 0] + s_[:, None] * rel[..., 1],
                           -s_[:, None] * rel[..., 0] + c[:, None] * rel[..., 1], rel[..., 2]], -1)
        sd = loc @ nrm.T
        inside = (sd >= -rad.double()[..., None] - 1e-9).all(-1)
        rng = loc.norm(dim=-1) - rad.double() <= cam.max_range + 1e-9
        return (inside & rng & valid).sum(1)

    cnt = sc.counts
    ar = lambda m: torch.arange(m, device=pos.device)[None, :]
    ks = keep(sc.spheres[..., :3], sc.spheres[..., 3], ar(sc.spheres.shape[1]) < cnt[:, 0:1])
    kb = keep(sc.boxes[..., :3], sc.boxes[..., 4:7].norm(dim=-1), ar(sc.boxes.shape[1]) < cnt[:, 1:2])
    kc = keep(sc.cylinders[..., :3], torch.sqrt(sc.cylinders[..., 3] ** 2 + sc.cylinders[..., 4] ** 2),
              ar(sc.cylinders.shape[1]) < cnt[:, 2:3])
    return ks, kb, kc


def bench_depth(dev, rank, world=1, frames=20):
    """C3: 16,384 envs, 64x48 depth, 32 solids (10 sph, 9 box, 13 cyl) + ground."""
    import torch

    from paper_2509_10247_b200 import sensors as sn
    from paper_2509_10247_b200 import world as wd

    E = 16384
    spawn, goal = np.array([0.0, 0.0, 1.2]), np.array([8.0, 0.0, 1.5])
    sc = wd.gen_obstacle_courses(3 + rank, E, spawn, goal, density=32 / 48.0, device=dev,
                                 env_offset=rank * E, check=False)
    g = torch.Generator(device="cpu").manual_seed(7 + rank)
    along = torch.rand(E, generator=g) * 8.0
    lat = (torch.rand(E, generator=g) - 0.5) * 6.0
    z = 0.5 + torch.rand(E, generator=g) * 3.0
    yaw = torch.rand(E, generator=g) * 2 * np.pi
    pos = torch.zeros(E, 4)
    pos[:, 0], pos[:, 1], pos[:, 2] = along, lat, z
    pos = pos.to(dev)
    cs = torch.stack([torch.cos(yaw), torch.sin(yaw)], -1).to(dev).contiguous()
    cam = sn.CameraIntrinsics(width=64, height=48, max_range=10.0)
    R = cam.n_rays

    def frame():
        sn.cast_rays(sc, pos, 4, cs, cam, 0, True)

    def timed(tiled, sensor, kind):
        sn.TILED = tiled

        def f():
            sn.cast_rays(sc, pos, 4, cs, sensor, kind, True)

        for _ in range(3):
            f()
        out = time_graph(f, frames)
        sn.TILED = True
        return out

    ms = max_over_ranks(timed(True, cam, 0), world)
    ms_untiled = max_over_ranks(timed(False, cam, 0), world)
    # spawn-facing-goal poses (SURVEY §8d's other C3 pose set): near the spawn,
    # looking down the corridor through the course, yaw jitter 0.1 rad
    pos_rand, cs_rand = pos, cs
    g2 = torch.Generator(device="cpu").manual_seed(17 + rank)
    pos_sf = torch.zeros(E, 4)
    pos_sf[:, 0] = torch.rand(E, generator=g2)
    pos_sf[:, 1] = (torch.rand(E, generator=g2) - 0.5) * 2.0
    pos_sf[:, 2] = 0.8 + torch.rand(E, generator=g2) * 0.8
    yaw_sf = torch.atan2(float(goal[1]) - pos_sf[:, 1], float(goal[0]) - pos_sf[:, 0]) + 0.1 * torch.randn(E, generator=g2)
    pos, cs = pos_sf.to(dev), torch.stack([torch.cos(yaw_sf), torch.sin(yaw_sf)], -1).to(dev).contiguous()
    ms_sf = max_over_ranks(timed(True, cam, 0), world)
    ks2, kb2, kc2 = fov_kept_counts(sc, pos, cs, cam)
    pos, cs = pos_rand, cs_rand
    lidar = sn.LidarPattern(n_azimuth=360, n_elevation=16, max_range=20.0)
    ms_lidar = max_over_ranks(timed(True, lidar, 1), world)
    E *= world  # rays of all ranks in the max-over-ranks frame time
    cnt = sc.counts.double().cpu().numpy()
    # un-culled algorithmic flops per ray: 14 + 10 ns + 6 nb + 31 nc (+1 ground)
    flops_frame = float(np.sum(14 + 10 * cnt[:, 0] + 6 * cnt[:, 1] + 31 * cnt[:, 2] + cnt[:, 3])) * R * world
    ks, kb, kc = fov_kept_counts(sc, pos, cs, cam)
    flops_culled = float((14 + 10 * ks + 6 * kb + 31 * kc).sum().item() + cnt[:, 3].sum()) * R * world
    flops_sf = float((14 + 10 * ks2 + 6 * kb2 + 31 * kc2).sum().item() + cnt[:, 3].sum()) * R * world
    return {"rays_per_s": E * R / (ms * 1e-3), "ms_per_frame": ms, "n_envs": E, "rays_per_env": R,
            "mean_solids": float(cnt[:, :3].sum(1).mean()),
            "tflops_uncull_equiv": flops_frame / (ms * 1e-3) / 1e12,
            "flops_per_ray": {"uncull": flops_frame / (E * R), "fov_culled": flops_culled / (E * R)},
            "tflops_culled_equiv": flops_culled / (ms * 1e-3) / 1e12,
            "kernel": "k_raycast_tiled<0> (per-warp cone culling, 64-ray tiles, 2 rays per lane)",
            "spawn_facing": {"ms_per_frame": ms_sf, "rays_per_s": E * R / (ms_sf * 1e-3),
                             "flops_per_ray_fov_culled": flops_sf / (E * R),
                             "tflops_culled_equiv": flops_sf / (ms_sf * 1e-3) / 1e12},
            "untiled": {"rays_per_s": E * R / (ms_untiled * 1e-3), "ms_per_frame": ms_untiled,
                        "tflops_uncull_equiv": flops_frame / (ms_untiled * 1e-3) / 1e12},
            "lidar_360x16": {"rays_per_s": E * lidar.n_rays / (ms_lidar * 1e-3), "ms_per_frame": ms_lidar}}


def bench_c3_env(dev, steps=20):
    """C3 as a closed-loop env: the avoidance task (32-solid courses, SDF
    penalty, collisions) with the 64x48 depth camera rendered every step,
    16,384 envs, through the public ``FlightTask.step`` (fused step kernel +
    tiled ray caster per step), forward only as a policy rollout sees it."""
    import torch

    import paper_2509_10247_b200 as qs

    E = 16384
    cfg = qs.TaskConfig(task="avoidance", dynamics="pm_continuous", n_envs=E, sensor="depth", depth_width=64,
                        depth_height=48, density=32 / 48.0, episode_len=128)
    env = qs.make_task(cfg, device=dev, strict=False)
    env.reset(seed=2)
    g = torch.Generator(device="cpu").manual_seed(21)
    acts = (torch.randn(steps, E, env.action_dim, generator=g) * 0.3).to(dev)
    with torch.no_grad():
        for t in range(3):
            env.step(acts[t])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(steps):
            out = env.step(acts[t])
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    assert out.obs.visual is not None and tuple(out.obs.visual.shape) == (E, 48, 64)
    return {"ms_per_env_step": ms, "env_steps_per_s": E / (ms * 1e-3), "rays_per_s": E * 3072 / (ms * 1e-3),
            "n_envs": E, "api": "FlightTask.step (no grad): fused step kernel + depth render per step"}


def bench_scene_gen(dev):
    """Obstacle-course generation (resets / re-randomisation):
    16,384 courses of the C3 distribution per launch, each with its
    feasibility BFS on the 0.25 m occupancy grid, outdoor and indoor (the
    reference: 52 / 31 scenes/s).  Timed on the device."""
    import torch

    from paper_2509_10247_b200 import world as wd

    E = 16384
    out = {}
    for style in ("outdoor", "indoor"):
        def gen(seed=[100]):
            seed[0] += 1
            return wd.gen_obstacle_courses(seed[0], E, [0.0, 0.0, 1.2], [8.0, 0.0, 1.5], 32 / 48.0, style=style,
                                           device=dev, check=False)

        gen()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            gen()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        out[style] = {"ms_per_batch": ms, "scenes_per_s": E / (ms * 1e-3), "n_envs": E}
    return out


def measure_fp32_peak(dev):
    """FFMA and FFMA2 throughput on this GPU (qs_probe_fp32): the measured FP32
    denominator BASELINE.md §3 asks for.  Full occupancy (8 x 256 threads per
    SM), 8 independent chains per thread, best of 5 launches."""
    import torch

    from paper_2509_10247_b200 import _lib as L

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, iters = sms * 8, 4096
    out = torch.zeros(blocks, device=dev)
    res = {}
    for mode, name in ((0, "ffma"), (1, "ffma2")):
        best = None
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            L.check(L.lib().qs_probe_fp32(mode, blocks, iters, L.ptr(out), L.stream_handle(dev)), "probe")
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        flops = blocks * 256 * iters * 16 * 8 * 2 * (2 if mode else 1)
        res[name + "_tflops"] = flops / (best * 1e-3) / 1e12
    return res


def bench_c4(dev):
    """C4 (BASELINE configs[3]) at 16,384 envs: indoor courses (5-box shell with
    a ceiling at 3 m), one LiDAR 360x16 sweep plus one 64x48 depth frame per
    env; and the multi-agent sim: a 4-agent line formation (4,096 envs x 4
    rows, formation penalty + all-agent success), T=32 BPTT windows fwd+bwd.
    Multi-agent *racing* is not in the reference (q/tasks.py:859-860)."""
    import torch

    import paper_2509_10247_b200 as qs
    from paper_2509_10247_b200 import sensors as sn
    from paper_2509_10247_b200 import world as wd
    from paper_2509_10247_b200.window import BpttWindow

    E = 16384
    sc = wd.gen_obstacle_courses(11, E, [0.0, 0.0, 1.2], [8.0, 0.0, 1.5], density=32 / 48.0, style="indoor",
                                 device=dev, check=False)
    g = torch.Generator(device="cpu").manual_seed(13)
    pos = torch.zeros(E, 4)
    pos[:, 0] = torch.rand(E, generator=g) * 8.0
    pos[:, 1] = (torch.rand(E, generator=g) - 0.5) * 6.0
    pos[:, 2] = 0.5 + torch.rand(E, generator=g) * 2.0
    yaw = torch.rand(E, generator=g) * 2 * np.pi
    pos = pos.to(dev)
    cs = torch.stack([torch.cos(yaw), torch.sin(yaw)], -1).to(dev).contiguous()
    cam = sn.CameraIntrinsics(width=64, height=48, max_range=10.0)
    lidar = sn.LidarPattern(n_azimuth=360, n_elevation=16, max_range=20.0)

    def frame():
        sn.cast_rays(sc, pos, 4, cs, lidar, 1, True)
        sn.cast_rays(sc, pos, 4, cs, cam, 0, True)

    for _ in range(3):
        frame()
    ms = time_graph(frame, 20)
    rays = E * (lidar.n_rays + cam.n_rays)
    # the formation runs the position task: with obstacles, a 4-agent line can
    # fail to fit next to an obstacle the course generator keeps clear of the
    # spawn point only, and the reference then raises GenerationError
    # (q/world.py:409-448) -- at 4,096 courses some always do
    cfg = qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=4096, n_agents=4, formation="line",
                        formation_side=1.0, episode_len=128)
    env = qs.make_task(cfg, device=dev, strict=False)
    env.reset(seed=1)
    win = BpttWindow(env, 32)
    win.actions.copy_(torch.randn(32, env.N, env.action_dim, generator=g).to(dev) * 0.3)
    win.capture()
    for _ in range(3):
        win.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        win.run()
    e1.record()
    torch.cuda.synchronize()
    ms_win = e0.elapsed_time(e1) / 10
    n_rows = env.N
    del win, env
    # closed loop through the env API: the racing task (gates, full quadrotor)
    # at 16,384 envs, one LiDAR 360x16 sweep / one 64x48 depth frame per step
    racing = {}
    for sensor in ("lidar", "depth"):
        kw = dict(lidar=lidar) if sensor == "lidar" else dict(depth_width=64, depth_height=48)
        renv = qs.make_task(qs.TaskConfig(task="racing", dynamics="full", n_envs=E, sensor=sensor, **kw),
                            device=dev, strict=False)
        renv.reset(seed=3)
        act = torch.zeros(E, renv.action_dim, device=dev)
        for _ in range(3):
            renv.step(act)
        ms_step = time_graph(lambda: renv.step(act), 20)
        racing[sensor] = {"ms_per_step": ms_step, "env_steps_per_s": E / (ms_step * 1e-3),
                          "rays_per_env": renv.obs_spec()["visual"].get("rays") if sensor == "lidar" else 64 * 48}
        del renv
    return {"indoor_lidar_plus_depth": {"ms_per_frame": ms, "rays_per_s": rays / (ms * 1e-3), "n_envs": E,
                                        "rays_per_env": lidar.n_rays + cam.n_rays},
            "racing_env_step": {"task": "racing (5 gates), full quadrotor, FlightTask.step + sensor render",
                                "n_envs": E, **{k: v for k, v in racing.items()}},
            "multi_agent_formation_window": {"task": "position", "envs": 4096, "agents": 4,
                                             "formation": "line, side 1 m", "horizon": 32,
                                             "ms_per_window": ms_win,
                                             "row_steps_per_s": n_rows * 32 / (ms_win * 1e-3)}}


def bench_c1(dev):
    """C1: pm_continuous / pm_discrete position task, 1,024 envs.
    The 0.4 MB working set makes it latency-bound, so it reports microseconds:
    (i) one `env.step` forward through the public API, (ii) the T=32 open-loop
    BPTT window L = -(1/32) sum_t 0.99^t mean(r_ctrl_t) fwd+bwd as one graph
    replay, (iii) the same loss through `env.step` + torch.autograd."""
    import torch

    import paper_2509_10247_b200 as qs
    from paper_2509_10247_b200.window import BpttWindow

    out = {}
    raw = np.random.default_rng(0).normal(size=(32, 1024, 3)) * 0.3
    for model in ("pm_continuous", "pm_discrete"):
        cfg = qs.TaskConfig(task="position", dynamics=model, n_envs=1024, episode_len=10 ** 6)
        env = qs.make_task(cfg, device=dev, strict=False)
        env.reset(seed=1)
        acts = torch.as_tensor(raw, dtype=torch.float32, device=dev)
        for t in range(8):
            env.step(acts[t])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(200):
            env.step(acts[t % 32])
        e1.record()
        torch.cuda.synchronize()
        step_us = e0.elapsed_time(e1) / 200 * 1e3
        env.reset(seed=1)
        win = BpttWindow(env, 32)
        win.actions.copy_(acts)
        win.capture()
        for _ in range(5):
            win.run()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(100):
            win.run()
        e1.record()
        torch.cuda.synchronize()
        win_us = e0.elapsed_time(e1) / 100 * 1e3
        env.reset(seed=1)

        def autograd_window():
            a_ = acts.clone().requires_grad_(True)
            env.detach_states()
            tot = 0.0
            for t in range(32):
                tot = tot + env.step(a_[t]).r_ctrl.mean() * 0.99 ** t
            (-tot / 32).backward()
            return a_.grad

        autograd_window()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            autograd_window()
        e1.record()
        torch.cuda.synchronize()
        ag_us = e0.elapsed_time(e1) / 5 * 1e3
        # (iv) the same user loop (env.step + torch.autograd.grad) captured in a
        # CUDA graph by the caller; the env's functional state is carried
        # through static buffers, as ShortHorizonTrainer(cuda_graph=True) does
        a_static = acts.clone().requires_grad_(True)
        carry = [env._S.detach().clone(), env._goal.clone(), env._peff.clone()]

        def graph_window():
            env._S, env._goal, env._peff = carry
            tot = 0.0
            for t in range(32):
                tot = tot + env.step(a_static[t]).r_ctrl.mean() * 0.99 ** t
            (g,) = torch.autograd.grad(-tot / 32, a_static)
            carry[0].copy_(env._S.detach())
            carry[1].copy_(env._goal)
            carry[2].copy_(env._peff)
            return g

        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(3):
                graph_window()
        torch.cuda.current_stream(dev).wait_stream(side)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            graph_window()
        env._S, env._goal, env._peff = carry
        agg_us = time_graph(gr.replay, 50) * 1e3
        out[model] = {"env_step_fwd_us": step_us, "bptt_window_fwd_bwd_us": win_us,
                      "bptt_window_autograd_graph_us": agg_us,
                      "bptt_window_autograd_us": ag_us}
    return out


def run_ours(a):
    import torch

    world, rank, local = dist_init()
    dev = torch.device("cuda", local if world > 1 else 0)
    import paper_2509_10247_b200 as qs
    from paper_2509_10247_b200.window import BpttWindow

    N, T = a.envs, a.horizon
    cfg = qs.TaskConfig(task="position", dynamics=a.model, n_envs=N, episode_len=128,
                        imu=qs.ImuSpec(**IMU) if a.model == "full" and not a.no_imu else None)
    env = qs.make_task(cfg, device=dev, strict=False, env_offset=rank * N)
    env.reset(seed=1)
    win = BpttWindow(env, T)
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    actions = (torch.randn(T, N, env.action_dim, generator=g) * 0.3).to(dev)
    win.actions.copy_(actions)
    win.capture()
    if a.profile:
        for _ in range(max(1, a.warmup)):
            win.run()
        torch.cuda.synchronize()
        print(json.dumps({"profile_run": True, "loss": float(win.loss64 if win.fused else win.loss)}))
        return
    for _ in range(a.warmup):
        win.run()
    torch.cuda.synchronize()
    # the NVML sampler ticks every 20 ms and one window is ~0.3 ms: keep the
    # same workload running (untimed soak, >= 0.4 s) under the sampler right
    # up to the timed region so its clock record describes the loaded GPU
    with ClockSampler(torch.cuda.current_device()) as clk:
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 0.4:
            for _ in range(20):
                win.run()
            torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            win.run()
        e1.record()
        torch.cuda.synchronize()
        barrier(world)
        ms = e0.elapsed_time(e1) / a.steps
    ms = max_over_ranks(ms, world)
    value = world * N * T / (ms * 1e-3)
    loss = float(win.loss64 if win.fused else win.loss)
    assert np.isfinite(loss)

    # per-kernel durations: one graph holding only the window-forward launch,
    # one holding only the window-backward launch (same buffers as above)
    from paper_2509_10247_b200 import _lib as L

    lib = L.lib()

    def fwd_only():
        L.check(lib.qs_task_window_fwd(env._cfg, env._scene.struct(), win._window_io(), L.stream_handle(dev)), "fwd")

    def bwd_only():
        L.check(lib.qs_task_window_bwd(env._cfg, env._scene.struct(), win._window_io(), L.stream_handle(dev)), "bwd")

    graphs = {}
    for name, fn in (("fwd", fwd_only), ("bwd", bwd_only)):
        fn()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        graphs[name] = gr
    reps = max(5, a.steps // 2)
    ms_fwd = time_graph(graphs["fwd"].replay, reps)
    ms_bwd = time_graph(graphs["bwd"].replay, reps)
    peak = 6553.3
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    gbs_fwd = FWD_BYTES * N * T / (ms_fwd * 1e-3) / 1e9
    gbs_bwd = BWD_BYTES * N * T / (ms_bwd * 1e-3) / 1e9
    dom = "fwd" if ms_fwd >= ms_bwd else "bwd"
    achieved = gbs_fwd if dom == "fwd" else gbs_bwd
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(f"window_{dom}")
    except Exception:
        pass
    # the per-step kernels behind FlightTask.step (closed-loop path), same workload
    win_ps = BpttWindow(env, T, fused=False)
    win_ps.actions.copy_(actions)
    win_ps.capture()
    ms_per_step_path = time_graph(lambda: win_ps.run(), reps)
    del win_ps

    # e2e through the public window API: pinned host actions in, loss out
    host = actions.cpu().pin_memory()
    torch.cuda.synchronize()
    # a stream of 50 windows (~40 ms): long enough that filling and draining
    # the copy pipeline (one upload, one download) is ~2% of it
    e2e_iters = max(3, min(max(a.steps, 50), 100))
    # serial: copy, window, read the loss -- one after the other
    t0 = time.perf_counter()
    for _ in range(e2e_iters):
        loss_t, _ = win.run(host)
        float(loss_t.item())
    serial_s = max_over_ranks((time.perf_counter() - t0) / e2e_iters, world)
    # streamed: the next window's H2D overlaps this window's kernels, and each
    # window's product -- dL/d(actions), (T,N,A) fp32 -- is downloaded to
    # pinned host memory on a third stream (full-duplex PCIe), with its loss
    grads_host = [torch.empty_like(host).pin_memory() for _ in range(2)]
    win.run_pipelined([host] * 2, grad_out=grads_host)  # warm-up: captures the second buffer's graph
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    win.run_pipelined([host] * e2e_iters, grad_out=[grads_host[k % 2] for k in range(e2e_iters)])
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_iters, world)
    assert bool(torch.isfinite(grads_host[0]).all())
    e2e = {"value": world * N * T / e2e_s, "unit": UNIT, "h2d_bytes_per_step": host.numel() * 4,
           "d2h_bytes_per_step": grads_host[0].numel() * 4 + 8,
           "api": "paper_2509_10247_b200.window.BpttWindow.run_pipelined(pinned host action batches, "
                  "grad_out=pinned host gradient buffers)",
           "timed": f"host wall clock around a stream of {e2e_iters} windows (H2D actions, fwd+bwd, D2H "
                    "dL/d(actions) and loss), max over ranks",
           "serial_value": world * N * T / serial_s,
           "serial_api": "BpttWindow.run(host actions) + loss.item() per window (gradient left on the device)"}

    # eager public API (env.step + torch.autograd) for reference, 1 window
    eager = None
    if rank == 0:
        env2 = qs.make_task(cfg, device=dev, strict=False, env_offset=rank * N)
        env2.reset(seed=1)

        def eager_window():
            acts = host.to(dev, non_blocking=True).requires_grad_(True)
            env2.detach_states()
            tot = 0.0
            # unbind: one stack in the backward, not the full-size zero tensor
            # select's backward builds per step for acts[t]
            for t, a_t in enumerate(acts.unbind(0)):
                tot = tot + env2.step(a_t).r_ctrl.mean() * 0.99 ** t
            loss_e = -tot / T
            loss_e.backward()
            return float(loss_e.item())

        for _ in range(2):
            eager_window()  # warm-up (allocator, autograd)
        torch.cuda.synchronize()
        times = []
        for _ in range(5):
            t0 = time.perf_counter()
            eager_window()
            times.append(time.perf_counter() - t0)
        times.sort()
        eager = {"value": N * T / times[len(times) // 2], "unit": UNIT,
                 "api": "FlightTask.step + torch.autograd backward, per window (host sync per window)",
                 "timed": "median of 5 windows (host-bound: Python step loop + autograd)",
                 "window_ms": [round(1e3 * t, 3) for t in times]}
        del env2

    depth = None
    if not a.no_depth:
        depth = bench_depth(dev, rank, world)
        probe = measure_fp32_peak(dev)
        fp32_peak = probe["ffma_tflops"]
        depth["fp32_peak_tflops"] = fp32_peak
        depth["fp32_peak_source"] = ("measured here: FFMA probe (qs_probe_fp32), full occupancy; nominal "
                                     "148 SM x 128 x 2 x 1.965 GHz = 74.4")
        depth["ffma2_tflops_measured"] = probe["ffma2_tflops"]
        depth["frac_uncull_equiv"] = depth["tflops_uncull_equiv"] / (fp32_peak * world)
        depth["frac_culled_equiv"] = depth["tflops_culled_equiv"] / (fp32_peak * world)
        depth["spawn_facing"]["frac_culled_equiv"] = depth["spawn_facing"]["tflops_culled_equiv"] / (fp32_peak * world)
        depth["frac_note"] = ("flops are the reference algorithm's (SURVEY §8d: per ray, every solid its fov_cull "
                              "keeps); the per-tile cone/sector cull tests far fewer solids per ray, so a "
                              "fraction above 1 means less arithmetic than that algorithm, not more than peak")

    c1 = bench_c1(dev) if rank == 0 and not a.no_depth else None
    c4 = bench_c4(dev) if rank == 0 and not a.no_depth else None
    c3_env = bench_c3_env(dev) if rank == 0 and not a.no_depth else None
    scene_gen = bench_scene_gen(dev) if rank == 0 and not a.no_depth else None

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline(a.cpu_seconds, a.model, T)
        cpu["host"] = cpu_model()

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (in-kernel Philox resets, actions N(0,0.3^2))",
        "config": {"workload": f"C2: {a.model} quadrotor + IMU, position task, {N} envs/GPU, BPTT window T={T} "
                               f"fwd+bwd (open-loop actions)", "envs_per_gpu": N, "horizon": T,
                   "parallelism": f"env-sharded x{world}, no collective in the sim step",
                   "l2": "window footprint ~%d MB > 126 MB L2 (no flush needed)" % int(
                       (win.S.numel() + win.obs.numel() + win.goal.numel() * 2 + win.actions.numel() * 2) * 4 / 1e6)},
        "roofline": {"bound": "hbm", "kernel": f"k_window_{dom} (qs_task_window_{dom})", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_env_step": {"fwd": FWD_BYTES, "bwd": BWD_BYTES},
                     "units_per_launch": N * T, "ms_per_launch": {"fwd": ms_fwd, "bwd": ms_bwd},
                     "gbs": {"fwd": gbs_fwd, "bwd": gbs_bwd}, "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)",
                     "bytes_source": "SURVEY.md §8(d) per env-step boundary bytes (full+IMU; open-loop bwd)",
                     "fused_payload": {
                         "bytes_per_env_step": {"fwd": FWD_BYTES_FUSED, "bwd": BWD_BYTES_FUSED},
                         "gbs": {"fwd": FWD_BYTES_FUSED * N * T / (ms_fwd * 1e-3) / 1e9,
                                 "bwd": BWD_BYTES_FUSED * N * T / (ms_bwd * 1e-3) / 1e9},
                         "note": "bytes the fused-window kernels must move; they are issue-bound (profiles/README.md)"},
                     # the bytes the forward really moves (ncu dram read+write of one launch,
                     # profiles/traffic.json) over this run's launch time
                     "dram_measured": ({"gbs": traffic / (ms_fwd * 1e-3) / 1e9,
                                        "frac_of_peak": traffic / (ms_fwd * 1e-3) / 1e9 / peak,
                                        "source": "ncu dram__bytes_read+write of k_window_fwd (profiles/traffic.json)"}
                                       if traffic else None)},
        "per_step_kernels": {"ms_per_window": ms_per_step_path,
                             "env_steps_per_s": world * N * T / (ms_per_step_path * 1e-3),
                             "note": "same window through the per-step kernels behind FlightTask.step"},
        "dist": {"backend": DIST["backend"], "shared_gpu": DIST["shared_gpu"],
                 "note": "ranks share GPUs (control flow only, not a scaling number)" if DIST["shared_gpu"]
                 else "one GPU per rank"},
        "e2e": e2e, "e2e_eager": eager,
        "gpu_launches": a.steps * win.launches_per_window,
        "clocks": getattr(clk, "result", None),
        "cpu_baseline": cpu,
        "depth": depth,
        "c1_latency": c1,
        "c4": c4,
        "c3_env": c3_env,
        "scene_gen": scene_gen,
        "loss": loss,
    }
    print(json.dumps(line))


def run_reference(a):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    per_step_seconds = max(2.0, min(10.0, 60.0 / max(1, a.steps + a.warmup)))
    for _ in range(a.warmup):
        cpu_baseline(min(2.0, per_step_seconds), a.model, a.horizon, n_sample=1024, extras=False)
    vals = []
    last = None
    for _ in range(a.steps):
        last = cpu_baseline(per_step_seconds, a.model, a.horizon, extras=False)
        vals.append(last["value"])
    v = statistics.median(vals)
    ms = a.envs * a.horizon / v * 1e3
    last["value"] = v
    last["host"] = cpu_model()
    if last.get("kind") == "reference":
        last["continuity"] = reference_continuity()
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": {
            "workload": f"C2: {a.model} quadrotor + IMU, position task, BPTT window T={a.horizon} fwd+bwd; "
                        + ("the reference package (baseline/_ref)" if last.get("kind") == "reference"
                           else "CPU oracle port") + " on a bounded env sample"},
        "cpu_baseline": last, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def run_c5(a):
    """C5: SHAC-style differentiable training, pm_continuous position task,
    131,072 envs per GPU, horizon 16, GRU-64 + MLP-128^2 policy, privileged
    critic; policy/critic gradients averaged by NCCL all-reduce across ranks.
    Whole updates replay from one CUDA graph per rank (with NCCL the
    all-reduces are captured inside it).  Reports training env-steps/s
    (CUDA-event time, max over ranks) and the all-reduce device time
    separately (the same collectives timed standalone with CUDA events)."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_init()
    dev = torch.device("cuda", local if world > 1 else 0)
    import paper_2509_10247_b200 as qs
    from paper_2509_10247_b200.train import LearnerOptions, ShortHorizonTrainer

    N = 131072 if a.envs == 65536 else a.envs
    cfg = qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=N, episode_len=128)
    env = qs.make_task(cfg, device=dev, strict=False, env_offset=rank * N)
    env.reset(seed=1)
    graph = world == 1 or DIST["backend"] == "nccl"
    tr = ShortHorizonTrainer(env, LearnerOptions(algo="shac", horizon=16, seed=0, cuda_graph=graph,
                                                 net_dtype=a.net_dtype))
    for _ in range(max(a.warmup, 4 if graph else 1)):
        tr.update()
    torch.cuda.synchronize()
    tr.allreduce_ms()
    with ClockSampler(torch.cuda.current_device()) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            out = tr.update()
        e1.record()
        torch.cuda.synchronize()
        barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1) / a.steps, world)
    ar_inline = max_over_ranks(tr.allreduce_ms() / a.steps, world)
    # the update's collectives timed standalone: one policy all-reduce and
    # critic_iters critic all-reduces per update, NCCL on the current stream
    ar = {"policy_floats": sum(p.numel() for p in tr.policy.parameters()),
          "critic_floats": sum(p.numel() for p in tr.value.parameters())}
    if world > 1:
        for key in ("policy_floats", "critic_floats"):
            buf = torch.zeros(ar[key], device=dev if DIST["backend"] == "nccl" else "cpu")
            for _ in range(5):
                dist.all_reduce(buf)
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            for _ in range(50):
                dist.all_reduce(buf)
            f1.record()
            torch.cuda.synchronize()
            ar[key.replace("floats", "allreduce_ms")] = max_over_ranks(f0.elapsed_time(f1) / 50, world)
        ar["per_update_ms"] = ar["policy_allreduce_ms"] + tr.opts.critic_iters * ar["critic_allreduce_ms"]
    if rank == 0:
        print(json.dumps({
            "metric": "env-steps/s (SHAC train: policy + sim fwd+bwd + critic)", "value": world * N * 16 / (ms * 1e-3),
            "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak",
            "dtype": "f32 sim, " + ("bf16 policy/critic matmuls" if a.net_dtype == "bf16" else "fp32 policy/critic"),
            "data": "synthetic (in-kernel Philox resets)",
            "config": {"workload": f"C5: SHAC, pm_continuous position, {N} envs/GPU x {world}, horizon 16",
                       "parallelism": f"env-sharded x{world}; NCCL all-reduce of policy+critic grads",
                       "cuda_graph": graph},
            "dist": {"backend": DIST["backend"], "shared_gpu": DIST["shared_gpu"]},
            "allreduce": ar, "allreduce_ms_per_update_eager": ar_inline if not graph else None,
            "clocks": getattr(clk, "result", None), "last": out}))


if __name__ == "__main__":
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c5":
        run_c5(args)
    else:
        run_ours(args)
