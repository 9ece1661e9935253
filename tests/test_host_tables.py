"""Host-side geometry the tiled ray caster's exactness rests on (CPU): every
ray of a tile lies inside the tile's bounding cone, inside its azimuth sector,
and inside its vertical direction range; the tiles cover every ray once."""

import numpy as np
import pytest
import torch


@pytest.mark.parametrize("width", [32, 64, 128])
@pytest.mark.parametrize("kind", ["camera", "lidar", "lidar_full"])
def test_tile_tables_bound_their_rays(kind, width):
    from paper_2509_10247_b200 import sensors as sn

    sensor = {"camera": sn.CameraIntrinsics(width=64, height=48, max_range=10.0),
              "lidar": sn.LidarPattern(n_azimuth=360, n_elevation=16, max_range=20.0),
              "lidar_full": sn.LidarPattern(n_azimuth=90, n_elevation=4, max_range=20.0)}[kind]
    sn._TILE_CACHE.clear()
    rays, cones, tdirs = sn._tile_table(sensor, torch.device("cpu"), width)
    rays, cones, tdirs = rays.numpy(), cones.double().numpy(), tdirs.numpy()
    d = sensor.pixel_dirs() if kind == "camera" else sensor.ray_dirs()
    assert rays.shape[1] == width and tdirs.shape == (rays.shape[0], width, 4)
    # the kernel's tile-ordered direction table repeats the ray table's fp32 values
    dir32 = sn._dir_table(sensor, torch.device("cpu")).numpy()
    ok = rays >= 0
    assert np.array_equal(tdirs[ok][:, :3], dir32[rays[ok], :3])
    assert np.array_equal(np.ascontiguousarray(tdirs[..., 3]).view(np.int32), rays)  # int32 bits
    got = np.sort(rays[rays >= 0])
    assert np.array_equal(got, np.arange(len(d)))  # a partition of the rays
    for t in range(len(rays)):
        v = d[rays[t][rays[t] >= 0]]
        ax, cth = cones[t, :3], cones[t, 3]
        assert np.all(v @ ax >= cth - 1e-6)  # bounding cone
        assert abs(cones[t, 3] ** 2 + cones[t, 4] ** 2 - 1) < 1e-5
        if cones[t, 7] > -1.5:  # azimuth sector (half-width <= pi/2)
            h = v[:, :2]
            hn = np.linalg.norm(h, axis=1)
            h = h[hn > 1e-12] / hn[hn > 1e-12, None]
            assert np.all(h @ cones[t, 5:7] >= cones[t, 7] - 1e-6)
            assert cones[t, 7] >= -1e-9 and abs(cones[t, 7] ** 2 + cones[t, 8] ** 2 - 1) < 1e-5
        assert v[:, 2].min() >= cones[t, 9] - 1e-7 and v[:, 2].max() <= cones[t, 10] + 1e-7
