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


# ---------------------------------------------------------------------------
# exactness against the fp64 oracle at the C3 / C4 shapes.  The north star asks
# for depth within 1e-4 m and EXACT hit/miss masks.  fp32 can only promise that
# for rays whose fp64 answer is itself stable under fp32-sized input noise, so
# every deviating ray is listed with its fp64 margin and must lie inside the
# documented epsilon-band: moving the ray's origin by
# PROBE_DELTA = 5 um along any axis changes the fp64 reference's own hit/miss
# or depth by more than the 1e-4 m bar (grazing tangents, edges and corners,
# t within 5 um of max_range).  Any deviation outside that band fails.

PROBE_DELTA = 5e-6


def _oracle_chunk(args):
    from oracle import quadsim_oracle as O

    prims, pos, R, kind, shape, max_range = args
    if kind == "depth":
        return O.render_depth(prims, pos, R, shape[0], shape[1], max_range).reshape(len(pos), -1)
    return O.render_lidar(prims, pos, R, shape[0], shape[1], max_range)


def _oracle_frames(prims, pos, R, kind, shape, max_range, chunk=32):
    import multiprocessing as mp
    import os

    from oracle import quadsim_oracle as O

    E = len(pos)
    jobs = [(O.prims_take(prims, slice(s, s + chunk)), pos[s:s + chunk], R[s:s + chunk], kind, shape, max_range)
            for s in range(0, E, chunk)]
    n = max(1, min(len(jobs), len(os.sched_getaffinity(0))))
    with mp.get_context("fork").Pool(n) as pool:
        return np.concatenate(pool.map(_oracle_chunk, jobs))


def _probe_margin(prims, env, origin, dirs, max_range):
    """fp64 depth of each listed ray and its largest change when the origin
    moves by +-PROBE_DELTA along x, y, z (uncull: the reference's cull is a
    conservative superset filter and never changes a ray)."""
    from oracle import quadsim_oracle as O

    pe = O.prims_take(prims, env)
    base = O.raycast(pe, origin, dirs[:, None, :], max_range)[:, 0]
    dev = np.zeros_like(base)
    flip = np.zeros(base.shape, bool)
    for ax in range(3):
        for sgn in (-1.0, 1.0):
            o2 = origin.copy()
            o2[:, ax] += sgn * PROBE_DELTA
            t = O.raycast(pe, o2, dirs[:, None, :], max_range)[:, 0]
            dev = np.maximum(dev, np.abs(t - base))
            flip |= (t < max_range) != (base < max_range)
    return base, dev, flip


def _check_against_oracle(qs, E, seed, kind, style):
    from oracle import quadsim_oracle as O

    sn = qs.sensors
    sc, pos, cs, _ = _scene_and_poses(qs, E, seed, style=style)
    if kind == "depth":
        sensor = sn.CameraIntrinsics(width=64, height=48, max_range=10.0)
        shape, k = (64, 48), 0
        body_dirs = O.pixel_dirs(64, 48)
    else:
        sensor = sn.LidarPattern(n_azimuth=360, n_elevation=16, max_range=20.0)
        shape, k = (360, 16), 1
        body_dirs = O.lidar_dirs(360, 16)
    d, hit, _ = sn.cast_rays(sc, pos, 4, cs, sensor, k, True, want_hit=True)
    d, hit = d.double().cpu().numpy(), hit.cpu().numpy().astype(bool)
    scenes = qs.world.device_scene_to_scenes(sc)
    prims = O.pack_primitives([{"spheres": s.prims.spheres, "boxes": s.prims.boxes,
                                "cylinders": s.prims.cylinders, "ground_z": s.prims.ground_z} for s in scenes])
    # the oracle sees the fp32 scene and poses the kernel saw
    p64 = pos[:, :3].double().cpu().numpy()
    csn = cs.double().cpu().numpy()
    R = O.rotz(np.arctan2(csn[:, 1], csn[:, 0]))
    mr = sensor.max_range
    ref = _oracle_frames(prims, p64, R, kind, shape, mr)
    err = np.abs(d - ref)
    bad_depth = err > 1e-4
    flips = hit != (ref < mr)
    dev_mask = bad_depth | flips
    env_i, ray_i = np.nonzero(dev_mask)
    dirs = np.einsum("bij,rj->bri", R, body_dirs)
    ok = True
    lines = []
    if len(env_i):
        base, dev, pflip = _probe_margin(prims, env_i, p64[env_i], dirs[env_i, ray_i], mr)
        assert np.allclose(base, ref[env_i, ray_i], rtol=0, atol=1e-12)
        in_band = (dev > 1e-4) | pflip
        for j in range(len(env_i)):
            lines.append(f"  env {env_i[j]} ray {ray_i[j]}: gpu {d[env_i[j], ray_i[j]]:.6f} ref {base[j]:.6f} "
                         f"flip {bool(flips[env_i[j], ray_i[j]])} fp64 probe dev {dev[j]:.3e} "
                         f"probe flip {bool(pflip[j])} {'in band' if in_band[j] else 'OUT OF BAND'}")
        ok = bool(in_band.all())
    print(f"\n{kind}/{style} {E} envs x {d.shape[1]} rays: max err {err[~dev_mask].max() if (~dev_mask).any() else 0:.2e} "
          f"on {int((~dev_mask).sum())} rays; {int(bad_depth.sum())} depth and {int(flips.sum())} hit-mask "
          f"deviations, all listed:")
    print("\n".join(lines))
    assert ok, "deviation outside the documented epsilon-band"
    assert dev_mask.mean() < 1e-4
    return err


@pytest.mark.parametrize("kind,style,E", [("depth", "outdoor", 1024), ("depth", "indoor", 512),
                                          ("lidar", "indoor", 256)])
def test_render_matches_oracle_exact_masks(kind, style, E):
    """C3 (64x48 depth, 32 solids + ground) and C4 (LiDAR 360x16, indoor shell
    with ceiling) against the fp64 oracle: depth within 1e-4 m and hit masks
    equal on every ray outside the epsilon-band; the band's rays listed."""
    import paper_2509_10247_b200 as qs

    _check_against_oracle(qs, E, 9, kind, style)


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
