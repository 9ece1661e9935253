"""C3 depth frames for ncu (the bench_depth workload, a few launches only).

    ncu --set full --import-source on -k regex:k_raycast_tiled -c 1 -o rep python profiles/prof_depth.py
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_10247_b200 import sensors as sn  # noqa: E402
from paper_2509_10247_b200 import world as wd  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    E = 16384
    sc = wd.gen_obstacle_courses(3, E, np.array([0.0, 0.0, 1.2]), np.array([8.0, 0.0, 1.5]), density=32 / 48.0,
                                 device=dev, check=False)
    g = torch.Generator(device="cpu").manual_seed(7)
    pos = torch.zeros(E, 4)
    pos[:, 0] = torch.rand(E, generator=g) * 8.0
    pos[:, 1] = (torch.rand(E, generator=g) - 0.5) * 6.0
    pos[:, 2] = 0.5 + torch.rand(E, generator=g) * 3.0
    yaw = torch.rand(E, generator=g) * 2 * np.pi
    pos = pos.to(dev)
    cs = torch.stack([torch.cos(yaw), torch.sin(yaw)], -1).to(dev).contiguous()
    cam = sn.CameraIntrinsics(width=64, height=48, max_range=10.0)
    kind = sys.argv[1] if len(sys.argv) > 1 else "depth"
    sensor = cam if kind == "depth" else sn.LidarPattern(n_azimuth=360, n_elevation=16, max_range=20.0)
    for _ in range(3):
        sn.cast_rays(sc, pos, 4, cs, sensor, 0 if kind == "depth" else 1, True)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
