"""Small end-to-end workload touching every kernel family once at small, odd
sizes (partial CTAs, 16-40 envs) -- scene generation,
Philox spawn, per-step fwd + VJP, fused windows (TMA action ring, cp.async
checkpoint ring), tiled and untiled ray casting incl. the recast depth VJP,
SDF, IMU.  Meant for compute-sanitizer (memcheck / racecheck / synccheck);
that tool is closed on this build's GPU pool, so the workload runs as a GPU
test (tests/test_gpu_extras.py) and every result it produces is checked
elsewhere against the oracle.
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402
from paper_2509_10247_b200 import sensors as sn  # noqa: E402
from paper_2509_10247_b200.window import BpttWindow  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    # fused windows (full + IMU: TMA ring; bwd: cp.async ring) and the per-step path
    cfg = qs.TaskConfig(task="position", dynamics="full", n_envs=300, episode_len=6,
                        imu=qs.ImuSpec(0.1, 0.01, 0.01, 0.001))
    env = qs.make_task(cfg, device=dev, strict=False)
    env.reset(seed=1)
    for fused in (True, False):
        win = BpttWindow(env, 8, fused=fused)
        win.actions.copy_(torch.randn(8, env.N, env.action_dim, device=dev) * 0.3)
        win.run()
    a = torch.zeros(env.N, env.action_dim, device=dev, requires_grad=True)
    env.step(a).r_ctrl.sum().backward()
    # avoidance with depth (scene gen, SDF, tiled render) and differentiable depth
    cfg = qs.TaskConfig(task="avoidance", dynamics="pm_continuous", n_envs=40, sensor="depth", depth_width=64,
                        depth_height=48, density=0.5, differentiable_depth=True, regen_scene_on_reset=False)
    env = qs.make_task(cfg, device=dev, strict=False)
    env.reset(seed=2)
    a = torch.zeros(env.N, env.action_dim, device=dev, requires_grad=True)
    out = env.step(a)
    (out.r_ctrl.sum() + out.obs.visual.sum() * 1e-3).backward()
    # LiDAR, indoor (extended culling), every tile width, untiled + stored-VJP path
    sc = qs.world.gen_obstacle_courses(5, 16, [0.0, 0.0, 1.2], [8.0, 0.0, 1.5], 0.6, style="indoor", device=dev,
                                       check=False)
    pos = torch.zeros(16, 4, device=dev)
    pos[:, 0] = torch.linspace(0, 8, 16)
    pos[:, 2] = 1.2
    cs = torch.stack([torch.cos(torch.arange(16.0)), torch.sin(torch.arange(16.0))], -1).to(dev).contiguous()
    for sensor, k in ((sn.LidarPattern(n_azimuth=360, n_elevation=16), 1),
                      (sn.CameraIntrinsics(width=64, height=48, max_range=10.0), 0)):
        for w in (32, 64, 128):
            sn.TILE_WIDTH = w
            sn.cast_rays(sc, pos, 4, cs, sensor, k, True, want_hit=True)
        sn.TILE_WIDTH = 0
        for tiled in (True, False):
            sn.TILED = tiled
            p = pos[:, :3].clone().requires_grad_(True)
            sn.render_depth_differentiable(sc, p, cs, sensor, k).sum().backward()
        sn.TILED = True
    torch.cuda.synchronize()
    env.check_errors()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
