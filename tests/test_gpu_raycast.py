"""Ray casting at benchmark scale: tiled (per-warp cone culling) == untiled ==
oracle, for depth and LiDAR over in-kernel generated C3/C4-style scenes."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _scene_and_poses(qs, E, seed, style="outdoor", density=32 / 48.0):
    sc = qs.world.gen_obstacle_courses(seed, E, [0.0, 0.0, 1.2], [8.0, 0.0, 1.5], density, style=style,
                                       device="cuda", check=False)
    g = torch.Generator().manual_seed(seed)
    pos = torch.zeros(E, 4)
    pos[:, 0] = torch.rand(E, generator=g) * 8.0
    pos[:, 1] = (torch.rand(E, generator=g) - 0.5) * 6.0
    pos[:, 2] = 0.5 + torch.rand(E, generator=g) * 2.0
    yaw = torch.rand(E, generator=g) * 2 * np.pi
    cs = torch.stack([torch.cos(yaw), torch.sin(yaw)], -1).contiguous()
    return sc, pos.cuda(), cs.cuda(), yaw.numpy()


@pytest.mark.parametrize("kind", ["depth", "lidar"])
def test_tiled_equals_untiled_bitwise(kind):
    import paper_2509_10247_b200 as qs
    sn = qs.sensors

    sc, pos, cs, _ = _scene_and_poses(qs, 2048, 5, style="indoor" if kind == "lidar" else "outdoor")
    sensor = sn.CameraIntrinsics(width=64, height=48, max_range=10.0) if kind == "depth" else \
        sn.LidarPattern(n_azimuth=360, n_elevation=16, max_range=20.0)
    k = 0 if kind == "depth" else 1
    sn.TILED = True
    a, ha, _ = sn.cast_rays(sc, pos, 4, cs, sensor, k, True, want_hit=True)
    a0, _, _ = sn.cast_rays(sc, pos, 4, cs, sensor, k, False)  # tile culling only
    sn.TILED = False
    b, hb, _ = sn.cast_rays(sc, pos, 4, cs, sensor, k, True, want_hit=True)
    c, _, _ = sn.cast_rays(sc, pos, 4, cs, sensor, k, False)  # no culling at all
    sn.TILED = True
    # culling never changes an image (q/sensors.py:338-374): bitwise within a kernel
    assert torch.equal(a, a0)
    assert torch.equal(b, c)
    # the two kernels share one arithmetic core per primitive: identical images
    assert torch.equal(a, b)
    assert torch.equal(ha, hb)


@pytest.mark.parametrize("width", [32, 64, 128])
@pytest.mark.parametrize("kind,style", [("depth", "outdoor"), ("depth", "indoor"), ("lidar", "outdoor"),
                                        ("lidar", "indoor")])
def test_tile_widths_bitwise(kind, style, width):
    """Every tile width (1, 2 or 4 rays per lane; 2 and 4 run the packed
    FFMA2 ray-pair tests) and both culling modes (indoor scenes take the
    extended per-tile culling) give the untiled kernel's image bit for bit."""
    import paper_2509_10247_b200 as qs
    sn = qs.sensors

    sc, pos, cs, _ = _scene_and_poses(qs, 1024, 11, style=style)
    sensor = sn.CameraIntrinsics(width=64, height=48, max_range=10.0) if kind == "depth" else \
        sn.LidarPattern(n_azimuth=360, n_elevation=16, max_range=20.0)
    k = 0 if kind == "depth" else 1
    old = sn.TILE_WIDTH
    try:
        sn.TILE_WIDTH = width
        sn.TILED = True
        a, ha, _ = sn.cast_rays(sc, pos, 4, cs, sensor, k, True, want_hit=True)
        sn.TILED = False
        b, hb, _ = sn.cast_rays(sc, pos, 4, cs, sensor, k, True, want_hit=True)
    finally:
        sn.TILED = True
        sn.TILE_WIDTH = old
    assert torch.equal(a, b)
    assert torch.equal(ha, hb)
    assert float(ha.float().mean()) > 0.05  # the scenes are actually hit


def test_tiled_degenerate_rays_and_origins():
    """Axis-parallel rays (0 * inf slab terms, vertical rays against cylinder
    sides, horizontal rays against caps) and origins exactly on surface planes:
    the tiled kernel's bit-order min and the untiled kernel agree, and the
    reference's t >= 0 convention holds (a surface at distance 0 is a hit)."""
    import paper_2509_10247_b200 as qs
    sn = qs.sensors
    W = qs.world

    class AxisRays(sn.LidarPattern):  # +-x, +-y, +-z and two oblique rays
        def ray_dirs(self):
            return np.array([[1.0, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1],
                             [0.6, 0, 0.8], [0, 0.6, -0.8]])

    prims = sn.PrimitiveSet(spheres=[[4.0, 0.0, 1.0, 0.5]], boxes=[[2.5, 0.0, 1.0, 0.5, 1.0, 1.0]],
                            cylinders=[[0.0, 3.0, 1.0, 0.5, 1.0]], ground_z=0.0)
    z3 = np.zeros(3)
    scn = W.Scene(prims=prims, bounds_lo=z3 - 10, bounds_hi=z3 + 10, spawn=z3, goal=z3)
    E = 8
    sc = W.scenes_to_device([scn] * E, device="cuda")
    pos = torch.zeros(E, 4)
    # x-axis aligned origins: on the box's x face plane, inside the box, on the
    # ground plane, on the cylinder's top cap plane, and generic
    pos[:, :3] = torch.tensor([[2.0, 0.0, 1.0], [2.5, 0.0, 1.0], [0.0, 0.0, 0.0], [0.0, 3.0, 2.0],
                               [0.0, 3.0, 1.0], [-1.0, 0.0, 1.0], [0.0, 0.0, 1.0], [3.0, 0.0, 2.0]])
    cs = torch.tensor([[1.0, 0.0]] * 4 + [[0.0, 1.0]] * 4).contiguous()
    rays = AxisRays(n_azimuth=8, n_elevation=1, max_range=20.0)
    for sensor, k in ((rays, 1), (sn.CameraIntrinsics(width=16, height=8, max_range=10.0), 0)):
        for width in (32, 64):
            sn.TILE_WIDTH = width
            sn.TILED = True
            a, ha, _ = sn.cast_rays(sc, pos.cuda(), 4, cs.cuda(), sensor, k, True, want_hit=True)
            sn.TILED = False
            b, hb, _ = sn.cast_rays(sc, pos.cuda(), 4, cs.cuda(), sensor, k, True, want_hit=True)
            sn.TILED = True
            sn.TILE_WIDTH = 0
            assert torch.equal(a.abs(), b.abs()), (a, b)  # -0 vs +0 only
            assert torch.equal(ha, hb)
            assert bool(torch.isfinite(a).all())
            if k == 1:  # origin on the box's x-min face looking +x, on the ground looking down,
                # on the cylinder's top cap looking down: surfaces at t = 0 are hits
                assert float(a[0, 0]) == 0.0 and float(a[2, 5]) == 0.0 and float(a[3, 5]) == 0.0
                assert float(a[1, 0]) == 0.5  # inside the box: the exit face


def test_depth_matches_oracle_on_generated_scenes():
    import paper_2509_10247_b200 as qs
    from oracle import quadsim_oracle as O

    sn = qs.sensors
    E = 256
    sc, pos, cs, yaw = _scene_and_poses(qs, E, 9)
    cam = sn.CameraIntrinsics(width=64, height=48, max_range=10.0)
    d, hit, _ = sn.cast_rays(sc, pos, 4, cs, cam, 0, True, want_hit=True)
    scenes = qs.world.device_scene_to_scenes(sc)
    prims = O.pack_primitives([{"spheres": s.prims.spheres, "boxes": s.prims.boxes,
                                "cylinders": s.prims.cylinders, "ground_z": s.prims.ground_z} for s in scenes])
    # the oracle sees the fp32 scene and poses the kernel saw
    ref = O.render_depth(prims, pos[:, :3].double().cpu().numpy(), O.rotz(np.arctan2(cs[:, 1].cpu().numpy(),
                         cs[:, 0].cpu().numpy())), 64, 48, 10.0).reshape(E, -1)
    err = np.abs(d.cpu().numpy() - ref)
    # north-star bar: 1e-4 m; allow a handful of grazing rays (reported)
    bad = err > 1e-4
    assert bad.mean() < 1e-4, (bad.sum(), err.max())
    mask_ref = ref < 10.0
    flips = (hit.cpu().numpy().astype(bool) != mask_ref)
    assert flips.mean() < 1e-4, flips.sum()


@pytest.mark.parametrize("kind,style", [("depth", "outdoor"), ("depth", "indoor"), ("lidar", "outdoor")])
def test_depth_vjp_recast_equals_stored(kind, style):
    """The tiled recast VJP (no dt/do in HBM) gives the untiled kernel's
    stored-dt/do gradient: same hit surfaces, fp32 summation order only."""
    import paper_2509_10247_b200 as qs
    sn = qs.sensors

    sc, pos, cs, _ = _scene_and_poses(qs, 512, 13, style=style)
    sensor = sn.CameraIntrinsics(width=64, height=48, max_range=10.0) if kind == "depth" else \
        sn.LidarPattern(n_azimuth=360, n_elevation=16, max_range=20.0)
    k = 0 if kind == "depth" else 1
    g = torch.randn(512, sensor.n_rays, generator=torch.Generator().manual_seed(3)).cuda()
    grads = []
    for tiled in (True, False):
        sn.TILED = tiled
        p = pos[:, :3].clone().requires_grad_(True)
        d = sn.render_depth_differentiable(sc, p, cs, sensor, k)
        (d * g).sum().backward()
        grads.append(p.grad.clone())
        sn.TILED = True
    a, b = grads
    assert float(b.abs().max()) > 0
    err = (a - b).abs() / (b.abs() + 1e-3 * float(b.abs().max()))
    assert float(err.max()) < 1e-4, float(err.max())
