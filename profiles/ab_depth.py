"""Ray-caster A/B timing: C3 depth (random corridor poses and spawn-facing-goal
poses), LiDAR 360x16, and the C4 indoor LiDAR + depth frame; checks the tiled
kernel against the untiled one on every workload (hit masks exact, depth
within 1e-4 m).

    python profiles/ab_depth.py            # prints one JSON line
"""

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_10247_b200 import sensors as sn  # noqa: E402
from paper_2509_10247_b200 import world as wd  # noqa: E402


def poses(E, spawn_facing, seed=7):
    g = torch.Generator(device="cpu").manual_seed(seed)
    pos = torch.zeros(E, 4)
    if spawn_facing:
        pos[:, 0] = torch.rand(E, generator=g) * 1.0
        pos[:, 1] = (torch.rand(E, generator=g) - 0.5) * 2.0
        pos[:, 2] = 0.8 + torch.rand(E, generator=g) * 0.8
        goal = torch.tensor([8.0, 0.0, 1.5])
        yaw = torch.atan2(goal[1] - pos[:, 1], goal[0] - pos[:, 0]) + 0.1 * torch.randn(E, generator=g)
    else:
        pos[:, 0] = torch.rand(E, generator=g) * 8.0
        pos[:, 1] = (torch.rand(E, generator=g) - 0.5) * 6.0
        pos[:, 2] = 0.5 + torch.rand(E, generator=g) * 3.0
        yaw = torch.rand(E, generator=g) * 2 * np.pi
    return pos, torch.stack([torch.cos(yaw), torch.sin(yaw)], -1).contiguous()


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def run(sc, pos, cs, sensor, kind):
    out = {}
    sn.TILED = True
    d_t, h_t, _ = sn.cast_rays(sc, pos, 4, cs, sensor, kind, True, want_hit=True)
    d_t, h_t = d_t.clone(), h_t.clone()
    out["ms"] = timed(lambda: sn.cast_rays(sc, pos, 4, cs, sensor, kind, True))
    sn.TILED = False
    d_u, h_u, _ = sn.cast_rays(sc, pos, 4, cs, sensor, kind, True, want_hit=True)
    sn.TILED = True
    out["max_abs_diff_vs_untiled"] = float((d_t - d_u).abs().max())
    out["hit_mismatch"] = int((h_t != h_u).sum())
    out["rays_per_s"] = pos.shape[0] * sensor.n_rays / (out["ms"] * 1e-3)
    return out


def main():
    dev = torch.device("cuda", 0)
    E = 16384
    res = {}
    cam = sn.CameraIntrinsics(width=64, height=48, max_range=10.0)
    lidar = sn.LidarPattern(n_azimuth=360, n_elevation=16, max_range=20.0)
    sc = wd.gen_obstacle_courses(3, E, np.array([0.0, 0.0, 1.2]), np.array([8.0, 0.0, 1.5]), density=32 / 48.0,
                                 device=dev, check=False)
    for name, sf in (("c3_random", False), ("c3_spawn_facing", True)):
        pos, cs = poses(E, sf)
        res[name] = run(sc, pos.to(dev), cs.to(dev), cam, 0)
    pos, cs = poses(E, False)
    res["lidar"] = run(sc, pos.to(dev), cs.to(dev), lidar, 1)
    # differentiable depth (forward + VJP): tiled recast vs untiled stored dt/do
    pos_d, cs_d = pos.to(dev), cs.to(dev)
    gdep = torch.randn(E, cam.n_rays, device=dev)
    for name, tiled in (("diff_depth_tiled_recast", True), ("diff_depth_untiled_stored", False)):
        sn.TILED = tiled

        def fb():
            p = pos_d[:, :3].clone().requires_grad_(True)
            d = sn.render_depth_differentiable(sc, p, cs_d, cam, 0)
            d.backward(gdep)

        res[name] = {"ms_fwd_bwd": timed(fb, 10)}
        sn.TILED = True
    sci = wd.gen_obstacle_courses(11, E, [0.0, 0.0, 1.2], [8.0, 0.0, 1.5], density=32 / 48.0, style="indoor",
                                  device=dev, check=False)
    pos, cs = poses(E, False, seed=9)
    pos[:, 2] = pos[:, 2].clamp(0.3, 2.7)
    res["indoor_lidar"] = run(sci, pos.to(dev), cs.to(dev), lidar, 1)
    res["indoor_depth"] = run(sci, pos.to(dev), cs.to(dev), cam, 0)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
