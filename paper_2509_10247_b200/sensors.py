"""Ray-cast depth/LiDAR sensing, signed distance, IMU and point-mass attitude.

Mirrors ``q/sensors.py`` (reference ``/root/reference/pkg/src/quadsim``): same
names, argument meaning and errors, but every batched computation runs in the
sm_100a kernels of ``libquadsim_b200.so`` on torch CUDA tensors (fp32).
Host-side pieces are limited to container types, ray-direction tables computed
once per sensor (fp64, as the reference does) and the DAIM dump format.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from paper_2509_10247_b200 import _lib as L

FAR = 1e9  # q/sensors.py:25


class SensorContractError(ValueError):
    pass


# ---------------------------------------------------------------------------
# obstacle containers (q/sensors.py:32-124)


@dataclass
class PrimitiveSet:
    """One scene's obstacles (host container, q/sensors.py:32-69)."""

    spheres: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))
    boxes: np.ndarray = field(default_factory=lambda: np.zeros((0, 6)))
    cylinders: np.ndarray = field(default_factory=lambda: np.zeros((0, 5)))
    ground_z: float | None = None

    def __post_init__(self):
        self.spheres = np.asarray(self.spheres, dtype=np.float64).reshape(-1, 4)
        self.boxes = np.asarray(self.boxes, dtype=np.float64).reshape(-1, 6)
        self.cylinders = np.asarray(self.cylinders, dtype=np.float64).reshape(-1, 5)

    @property
    def n_solids(self) -> int:
        return len(self.spheres) + len(self.boxes) + len(self.cylinders)


@dataclass
class BatchedPrimitives:
    """Padded per-env primitive arrays (q/sensors.py:72-97); numpy or torch."""

    spheres: object  # (B, Sm, 4)
    sph_valid: object  # (B, Sm) bool
    boxes: object  # (B, Bm, 6)
    box_valid: object
    cylinders: object  # (B, Cm, 5)
    cyl_valid: object
    ground_z: object  # (B,), nan = no ground

    @property
    def batch(self) -> int:
        return self.spheres.shape[0]

    def masked(self, keep_sph, keep_box, keep_cyl) -> "BatchedPrimitives":
        return BatchedPrimitives(self.spheres, self.sph_valid & keep_sph, self.boxes,
                                 self.box_valid & keep_box, self.cylinders, self.cyl_valid & keep_cyl,
                                 self.ground_z)


def pack_primitives(sets) -> BatchedPrimitives:
    """q/sensors.py:100-124 (host packing of PrimitiveSet lists)."""
    B = len(sets)
    Sm = max([len(s.spheres) for s in sets] + [1])
    Bm = max([len(s.boxes) for s in sets] + [1])
    Cm = max([len(s.cylinders) for s in sets] + [1])
    sph = np.zeros((B, Sm, 4)); sv = np.zeros((B, Sm), bool)
    box = np.zeros((B, Bm, 6)); bv = np.zeros((B, Bm), bool)
    cyl = np.zeros((B, Cm, 5)); cv = np.zeros((B, Cm), bool)
    gz = np.full(B, np.nan)
    for i, s in enumerate(sets):
        sph[i, :len(s.spheres)] = s.spheres; sv[i, :len(s.spheres)] = True
        box[i, :len(s.boxes)] = s.boxes; bv[i, :len(s.boxes)] = True
        cyl[i, :len(s.cylinders)] = s.cylinders; cv[i, :len(s.cylinders)] = True
        if s.ground_z is not None:
            gz[i] = s.ground_z
    return BatchedPrimitives(sph, sv, box, bv, cyl, cv, gz)


def _t(x, device, dtype=torch.float32):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype)
    a = np.asarray(x)
    if not a.flags.writeable:  # read-only views (e.g. broadcast) cannot back a tensor
        a = a.copy()
    return torch.as_tensor(a, dtype=dtype, device=device)


def _valid_first(data, valid):
    """Stable-compact valid lanes to the front (device gather); returns data, counts."""
    order = torch.sort((~valid).to(torch.int8), dim=1, stable=True).indices
    idx = order.unsqueeze(-1).expand(-1, -1, data.shape[-1])
    return torch.gather(data, 1, idx), valid.sum(dim=1).to(torch.int32)


class DeviceScene:
    """Per-env obstacle/bounds/gate tensors in the kernel layout.

    spheres (E,Sm,4); boxes (E,Bm,8) = c,_,h,_; cylinders (E,Cm,8) = c,r,hh,...;
    counts (E,4) = n_sph, n_box, n_cyl, has_ground; ground_z (E,);
    bounds (E,2,4); spawn_goal (E,2,4); gates (E,G,8) = c,inner,n,frame.
    """

    def __init__(self, n_envs, device, Sm=1, Bm=1, Cm=1, n_gates=0):
        f = dict(device=device, dtype=torch.float32)
        self.device = device
        self.n_envs = n_envs
        self.spheres = torch.zeros(n_envs, max(Sm, 1), 4, **f)
        self.boxes = torch.zeros(n_envs, max(Bm, 1), 8, **f)
        self.cylinders = torch.zeros(n_envs, max(Cm, 1), 8, **f)
        self.counts = torch.zeros(n_envs, 4, dtype=torch.int32, device=device)
        self.ground_z = torch.zeros(n_envs, **f)
        self.bounds = torch.zeros(n_envs, 2, 4, **f)
        self.spawn_goal = torch.zeros(n_envs, 2, 4, **f)
        self.gates = torch.zeros(n_envs, max(n_gates, 1), 8, **f)
        self._struct = None
        # scenes with large boxes (indoor shells) take the tiled ray caster's
        # extended per-tile culling (qs_ray_cfg.cull bit 1)
        self.ext_cull = False

    @classmethod
    def from_batched(cls, bp: BatchedPrimitives, device, n_gates=0) -> "DeviceScene":
        E = bp.batch
        sph = _t(bp.spheres, device).reshape(E, -1, 4)
        box = _t(bp.boxes, device).reshape(E, -1, 6)
        cyl = _t(bp.cylinders, device).reshape(E, -1, 5)
        sc = cls(E, device, sph.shape[1], box.shape[1], cyl.shape[1], n_gates)
        sv = _t(bp.sph_valid, device, torch.bool).reshape(E, -1)
        bv = _t(bp.box_valid, device, torch.bool).reshape(E, -1)
        cv = _t(bp.cyl_valid, device, torch.bool).reshape(E, -1)
        s, ns = _valid_first(sph, sv)
        b, nb = _valid_first(box, bv)
        c, nc = _valid_first(cyl, cv)
        sc.spheres.copy_(s)
        sc.boxes[..., 0:3] = b[..., 0:3]
        sc.boxes[..., 4:7] = b[..., 3:6]
        sc.cylinders[..., 0:5] = c
        gz = _t(bp.ground_z, device, torch.float64 if not isinstance(bp.ground_z, torch.Tensor) else None).reshape(E)
        has_g = torch.isfinite(gz)
        sc.ground_z.copy_(torch.where(has_g, gz, torch.zeros_like(gz)).float())
        sc.counts.copy_(torch.stack([ns, nb, nc, has_g.to(torch.int32)], dim=-1))
        return sc

    def clone(self) -> "DeviceScene":
        """Deep copy (copy-on-write regeneration: autograd nodes recorded
        against this scene keep seeing it unchanged)."""
        sc = DeviceScene.__new__(DeviceScene)
        sc.device, sc.n_envs, sc.ext_cull, sc._struct = self.device, self.n_envs, self.ext_cull, None
        for k in ("spheres", "boxes", "cylinders", "counts", "ground_z", "bounds", "spawn_goal", "gates"):
            setattr(sc, k, getattr(self, k).clone())
        return sc

    def set_rows(self, e_slice, other: "DeviceScene"):
        for k in ("spheres", "boxes", "cylinders", "counts", "ground_z", "bounds", "spawn_goal", "gates"):
            getattr(self, k)[e_slice] = getattr(other, k)

    def tensors(self) -> list:
        """The scene as the op layer takes it (quadsim::task_step's ``scene``)."""
        return [self.bounds, self.spawn_goal, self.spheres, self.boxes, self.cylinders, self.counts,
                self.ground_z, self.gates]

    def struct(self) -> L.QsScene:
        s = L.QsScene()
        s.bounds = self.bounds.data_ptr()
        s.spawn_goal = self.spawn_goal.data_ptr()
        s.spheres = self.spheres.data_ptr()
        s.boxes = self.boxes.data_ptr()
        s.cylinders = self.cylinders.data_ptr()
        s.counts = self.counts.data_ptr()
        s.ground_z = self.ground_z.data_ptr()
        s.gates = self.gates.data_ptr()
        s.Sm, s.Bm, s.Cm = self.spheres.shape[1], self.boxes.shape[1], self.cylinders.shape[1]
        return s

    def to_batched(self) -> BatchedPrimitives:
        """Back to the reference's padded form (torch tensors on device)."""
        ns, nb, nc, hg = (self.counts[:, k] for k in range(4))
        ar = lambda m: torch.arange(m, device=self.device)[None]  # noqa: E731
        box = torch.cat([self.boxes[..., 0:3], self.boxes[..., 4:7]], dim=-1)
        return BatchedPrimitives(
            self.spheres, ar(self.spheres.shape[1]) < ns[:, None], box, ar(box.shape[1]) < nb[:, None],
            self.cylinders[..., 0:5], ar(self.cylinders.shape[1]) < nc[:, None],
            torch.where(hg.bool(), self.ground_z, torch.full_like(self.ground_z, float("nan"))))


def as_device_scene(prims, device) -> DeviceScene:
    if isinstance(prims, DeviceScene):
        return prims
    if isinstance(prims, PrimitiveSet):
        prims = pack_primitives([prims])
    return DeviceScene.from_batched(prims, device)


# ---------------------------------------------------------------------------
# camera / LiDAR models (q/sensors.py:276-335)


@dataclass
class CameraIntrinsics:
    width: int = 64
    height: int = 64
    fov_h: float = float(np.deg2rad(90.0))
    fov_v: float = float(np.deg2rad(75.0))
    max_range: float = 10.0
    offset: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        if not (0 < self.fov_h < np.pi and 0 < self.fov_v < np.pi):
            raise SensorContractError("FOV must lie in (0, pi)")
        if self.width * self.height < 1 or self.max_range <= 0:
            raise SensorContractError("need width*height >= 1 and max_range > 0")
        self.offset = np.asarray(self.offset, dtype=np.float64)

    @property
    def n_rays(self) -> int:
        return self.width * self.height

    def pixel_dirs(self) -> np.ndarray:
        """(H*W, 3) unit body-frame directions, fp64 (q/sensors.py:292-302)."""
        th = np.tan(self.fov_h / 2)
        tv = np.tan(self.fov_v / 2)
        cols = (np.arange(self.width) + 0.5) / self.width
        rows = (np.arange(self.height) + 0.5) / self.height
        y = th * (1.0 - 2.0 * cols)
        z = tv * (1.0 - 2.0 * rows)
        zz, yy = np.meshgrid(z, y, indexing="ij")
        d = np.stack([np.ones_like(yy), yy, zz], axis=-1).reshape(-1, 3)
        return d / np.linalg.norm(d, axis=-1, keepdims=True)


@dataclass
class LidarPattern:
    n_azimuth: int = 16
    n_elevation: int = 4
    azimuth_extent: float = 2 * np.pi
    elevation_extent: float = float(np.deg2rad(30.0))
    max_range: float = 20.0
    offset: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        if not (0 < self.azimuth_extent <= 2 * np.pi and 0 < self.elevation_extent < np.pi):
            raise SensorContractError("angular extents out of range")
        self.offset = np.asarray(self.offset, dtype=np.float64)

    @property
    def n_rays(self) -> int:
        return self.n_azimuth * self.n_elevation

    def ray_dirs(self) -> np.ndarray:
        """(A*E, 3) body-frame directions, azimuth-major (q/sensors.py:323-335)."""
        az = np.linspace(0.0, self.azimuth_extent, self.n_azimuth, endpoint=False)
        el = (np.linspace(-0.5, 0.5, self.n_elevation) * self.elevation_extent
              if self.n_elevation > 1 else np.zeros(1))
        aa, ee = np.meshgrid(az, el, indexing="ij")
        return np.stack([np.cos(ee) * np.cos(aa), np.cos(ee) * np.sin(aa), np.sin(ee)],
                        axis=-1).reshape(-1, 3)


_DIR_CACHE: dict = {}


def _dir_table(sensor, device) -> torch.Tensor:
    key = (type(sensor).__name__, repr(sensor), str(device))
    t = _DIR_CACHE.get(key)
    if t is None:
        d = sensor.pixel_dirs() if isinstance(sensor, CameraIntrinsics) else sensor.ray_dirs()
        t = torch.zeros(d.shape[0], 4, dtype=torch.float32, device=device)
        t[:, :3] = torch.as_tensor(d, dtype=torch.float32, device=device)
        _DIR_CACHE[key] = t
    return t


_TILE_CACHE: dict = {}


def _tile_table(sensor, device, width=None):
    """Group the sensor's rays into angularly compact tiles of ``width`` (32, 64
    or 128) with a bounding cone each (fp64 host geometry, once per sensor):
    8 x (width/8) pixel blocks for a camera, consecutive azimuth-major runs for
    a LiDAR."""
    if width is None:
        width = TILE_WIDTH or (64 if isinstance(sensor, CameraIntrinsics) else 128)
    key = (type(sensor).__name__, repr(sensor), str(device), width)
    hit = _TILE_CACHE.get(key)
    if hit is not None:
        return hit
    if isinstance(sensor, CameraIntrinsics):
        d = sensor.pixel_dirs()
        W, H = sensor.width, sensor.height
        bw, bh = (8, width // 8) if width <= 64 else (16, width // 16)
        tiles = []
        for ty in range(0, H, bh):
            for tx in range(0, W, bw):
                tiles.append([r * W + c for r in range(ty, min(H, ty + bh)) for c in range(tx, min(W, tx + bw))])
    else:
        d = sensor.ray_dirs()
        tiles = [list(range(s, min(len(d), s + width))) for s in range(0, len(d), width)]
    # lane j of the kernel's warp owns slots j, j + 32, ...: order each full
    # tile so that a lane's rays are consecutive in the image (horizontally
    # adjacent pixels / consecutive LiDAR rays), so it stores them with one
    # vector store.  The tile's ray SET (and so its cone) is unchanged.
    rpl = width // 32
    if rpl > 1 and LANE_CONSECUTIVE:
        tiles = [[t[(p % 32) * rpl + p // 32] for p in range(width)] if len(t) == width else t for t in tiles]
    rays = np.full((len(tiles), width), -1, dtype=np.int32)
    # axis xyz, cos/sin(half-angle) | sector centre xy, cos/sin(sector half-width) | pad
    cones = np.zeros((len(tiles), 12))
    for k, t in enumerate(tiles):
        rays[k, :len(t)] = t
        v = d[t]
        ax = v.sum(0)
        n = np.linalg.norm(ax)
        ax = ax / n if n > 1e-12 else np.array([1.0, 0.0, 0.0])
        c = float(np.min(v @ ax)) if n > 1e-12 else -1.0
        th = min(np.pi, np.arccos(np.clip(c, -1.0, 1.0)) + 1e-6)  # widen for round-off
        cones[k, :3] = ax
        cones[k, 3] = np.cos(th)
        cones[k, 4] = np.sin(th)
        # azimuth sector of the tile's rays (a yaw-only camera keeps it a
        # sector in the world frame); exactly vertical rays have no azimuth and
        # can only hit footprints containing the origin, which are always kept
        hxy = v[:, :2]
        hn = np.linalg.norm(hxy, axis=1)
        hxy = hxy[hn > 1e-12] / hn[hn > 1e-12, None]
        cen = hxy.sum(0) if len(hxy) else np.array([1.0, 0.0])
        cn = np.linalg.norm(cen)
        w = np.pi
        if cn > 1e-9:
            cen = cen / cn
            w = float(np.arccos(np.clip(np.min(hxy @ cen), -1.0, 1.0))) + 1e-6 if len(hxy) else 0.0
        cones[k, 5:7] = cen
        if w <= np.pi / 2:  # the tangent-sector test needs half-width + footprint angle <= pi
            cones[k, 7] = np.cos(w)
            cones[k, 8] = np.sin(w)
        else:
            cones[k, 7] = -2.0
        cones[k, 9] = float(v[:, 2].min())  # vertical range of the tile's directions
        cones[k, 10] = float(v[:, 2].max())
    # tile-ordered direction table for the kernel: (dir xyz as the fp32 values
    # of the sensor's ray table, ray index as int32 bits; -1 = empty slot)
    dirs32 = d.astype(np.float32)
    td = np.zeros((len(tiles), width, 4), dtype=np.float32)
    ok = rays >= 0
    td[ok, :3] = dirs32[rays[ok]]
    td[..., 3] = rays.view(np.float32)  # the int32 ray index bit for bit (-1: empty slot)
    out = (torch.as_tensor(rays, device=device), torch.as_tensor(cones, dtype=torch.float32, device=device),
           torch.as_tensor(td, device=device))
    _TILE_CACHE[key] = out
    return out


def _ray_cfg(sensor, kind, cull, n_agents=1) -> L.QsRayCfg:
    rc = L.QsRayCfg()
    rc.kind = kind
    rc.cull = 1 if cull else 0
    rc.n_agents = n_agents
    if sensor is None:
        return rc
    rc.n_rays = sensor.n_rays
    rc.max_range = float(sensor.max_range)
    if isinstance(sensor, CameraIntrinsics):
        rc.tan_h = float(np.tan(sensor.fov_h / 2))
        rc.tan_v = float(np.tan(sensor.fov_v / 2))
    for i in range(3):
        rc.offset[i] = float(sensor.offset[i])
    return rc


def _yaw_cs_from_R(R: torch.Tensor):
    """(cos, sin) of a yaw-only attitude, or None when R is not yaw-only."""
    R = R.to(torch.float32)
    if not (torch.all(R[:, 2, 2] == 1.0) and torch.all(R[:, 2, :2] == 0) and torch.all(R[:, :2, 2] == 0)):
        return None
    return torch.stack([R[:, 0, 0], R[:, 1, 0]], dim=-1).contiguous()


def _pos4(p: torch.Tensor) -> torch.Tensor:
    out = torch.zeros(p.shape[0], 4, dtype=torch.float32, device=p.device)
    out[:, :3] = p
    return out


def cast_rays(scene: DeviceScene, pos: torch.Tensor, pos_stride: int, cam_cs, sensor, kind: int,
              cull: bool = True, n_agents: int = 1, want_hit=False, want_grad=False):
    """Launch the ray-cast kernel.  pos: (N, pos_stride) fp32 device rows."""
    N = pos.shape[0] if pos.dim() == 2 else pos.numel() // pos_stride
    rc = _ray_cfg(sensor, kind, cull, n_agents)
    if getattr(scene, "ext_cull", False):
        rc.cull |= 2
    dev = scene.device
    out = torch.empty(N, rc.n_rays, dtype=torch.float32, device=dev)
    hit = torch.empty(N, rc.n_rays, dtype=torch.uint8, device=dev) if want_hit else None
    dT = torch.empty(N, rc.n_rays, 4, dtype=torch.float32, device=dev) if want_grad else None
    dirs = _dir_table(sensor, dev)
    if not want_grad and kind in (0, 1) and TILED:
        tr, tc, td = _tile_table(sensor, dev)
        L.check(L.lib().qs_raycast_tiled(rc, scene.struct(), N, L.ptr(pos), pos_stride, L.ptr(cam_cs),
                                         L.ptr(td), L.ptr(tc), tr.shape[0], tr.shape[1], L.ptr(out),
                                         L.ptr(hit), L.stream_handle(dev)), "qs_raycast_tiled")
        return out, hit, dT
    L.check(L.lib().qs_raycast(rc, scene.struct(), N, L.ptr(pos), pos_stride, L.ptr(cam_cs),
                               L.ptr(dirs), None, L.ptr(out), L.ptr(hit), L.ptr(dT),
                               L.stream_handle(dev)), "qs_raycast")
    return out, hit, dT


TILED = True  # per-warp cone culling (k_raycast_tiled); False selects the untiled kernel
# rays per tile of the tiled kernel (32 x rays per lane): 0 = per sensor (8x8
# pixel blocks for cameras, 8 azimuths x 16 elevations for LiDARs, the fastest
# measured, profiles/README.md); QS_TILE_WIDTH overrides it for A/B runs
TILE_WIDTH = int(os.environ.get("QS_TILE_WIDTH", "0"))
# give each lane consecutive rays within a tile (vector stores); 0 for A/B runs
LANE_CONSECUTIVE = os.environ.get("QS_TILE_LANE_ORDER", "1") != "0"


def raycast(prims, origins, dirs, max_range: float, chunk_elems: int = 0, device=None):
    """Nearest-hit distance (B,R) for unit rays, clamped (q/sensors.py:245-269)."""
    dev = L.require_cuda(device if device is not None else L.tensor_device(origins))
    sc = as_device_scene(prims, dev)
    o = _pos4(_t(origins, dev).reshape(-1, 3))
    d = _t(dirs, dev)
    B, R = d.shape[:2]
    dw = torch.zeros(B, R, 4, dtype=torch.float32, device=dev)
    dw[..., :3] = d
    rc = L.QsRayCfg()
    rc.kind, rc.n_rays, rc.cull, rc.max_range, rc.n_agents = 2, R, 0, float(max_range), 1
    out = torch.empty(B, R, dtype=torch.float32, device=dev)
    L.check(L.lib().qs_raycast(rc, sc.struct(), B, L.ptr(o), 4, None, None, L.ptr(dw), L.ptr(out),
                               None, None, L.stream_handle(dev)), "qs_raycast")
    return out


def _render(prims, body_pos, body_R, sensor, kind, cull, device):
    dev = L.require_cuda(device if device is not None else L.tensor_device(body_pos))
    sc = as_device_scene(prims, dev)
    pos = _pos4(_t(body_pos, dev).reshape(-1, 3))
    R = _t(body_R, dev)
    cs = _yaw_cs_from_R(R)
    if cs is not None:
        out, _, _ = cast_rays(sc, pos, 4, cs, sensor, kind, cull)
        return out
    # general attitude: rotate the body table per row, no culling (cull never
    # changes the image, q/sensors.py:338-374)
    d_body = _dir_table(sensor, dev)[:, :3]
    dirs = torch.einsum("bij,rj->bri", R, d_body)
    origin = pos[:, :3] + torch.einsum("bij,j->bi", R, _t(sensor.offset, dev))
    return raycast(sc, origin, dirs, sensor.max_range, device=dev)


def render_depth(prims, body_pos, body_R, intrinsics: CameraIntrinsics, cull: bool = True, device=None):
    """Depth images (B,H,W), Euclidean ray distance (q/sensors.py:377-389)."""
    B = body_pos.shape[0]
    out = _render(prims, body_pos, body_R, intrinsics, 0, cull, device)
    return out.reshape(B, intrinsics.height, intrinsics.width)


def render_lidar(prims, body_pos, body_R, pattern: LidarPattern, device=None):
    """Range array (B, A*E) (q/sensors.py:392-410)."""
    return _render(prims, body_pos, body_R, pattern, 1, True, device)


def fov_cull(prims, cam_pos, cam_R, intrinsics: CameraIntrinsics):
    """Conservative frustum keep-masks (q/sensors.py:338-374), on device."""
    dev = L.require_cuda(L.tensor_device(cam_pos))
    th = np.tan(intrinsics.fov_h / 2)
    tv = np.tan(intrinsics.fov_v / 2)
    n = np.array([[th, -1.0, 0.0], [th, 1.0, 0.0], [tv, 0.0, -1.0], [tv, 0.0, 1.0], [1.0, 0.0, 0.0]])
    n = torch.as_tensor(n / np.linalg.norm(n, axis=-1, keepdims=True), dtype=torch.float32, device=dev)
    cp = _t(cam_pos, dev)
    R = _t(cam_R, dev)

    def keep(c, rad):
        local = torch.einsum("bji,bpj->bpi", R, c - cp[:, None, :])
        sd = torch.einsum("kp,bnp->bnk", n, local)
        inside = torch.all(sd >= -rad[..., None] - 1e-6, dim=-1)
        return inside & (torch.linalg.norm(local, dim=-1) - rad <= intrinsics.max_range + 1e-6)

    s = _t(prims.spheres, dev)
    b = _t(prims.boxes, dev)
    c = _t(prims.cylinders, dev)
    return (keep(s[..., :3], s[..., 3]), keep(b[..., :3], torch.linalg.norm(b[..., 3:6], dim=-1)),
            keep(c[..., :3], torch.sqrt(c[..., 3] ** 2 + c[..., 4] ** 2)))


class _RenderDepthFn(torch.autograd.Function):
    """Opt-in differentiable depth: d depth / d body position via the analytic
    d t / d o = -n / (n . d) of the hit surface (new capability; no reference).

    Cameras and LiDARs take the tiled ray caster both ways: the forward renders
    with no per-ray gradient output, and the backward recasts the same tiles to
    find each ray's hit surface (``qs_raycast_tiled_vjp``), so no (N, R, 4)
    dt/do tensor goes through HBM.  Generic rays (kind 2) keep the untiled
    kernel's stored dt/do + ``qs_raycast_vjp``."""

    @staticmethod
    def forward(ctx, pos3, scene, cam_cs, sensor, kind, n_agents):
        pos = _pos4(pos3.detach())
        recast = kind in (0, 1) and TILED
        out, _, dT = cast_rays(scene, pos, 4, cam_cs, sensor, kind, True, n_agents, want_grad=not recast)
        ctx.recast, ctx.scene, ctx.sensor, ctx.kind, ctx.n_agents = recast, scene, sensor, kind, n_agents
        ctx.save_for_backward(pos, cam_cs if cam_cs is not None else pos.new_zeros(0), dT if dT is not None
                              else pos.new_zeros(0))
        ctx.has_cs = cam_cs is not None
        return out

    @staticmethod
    def backward(ctx, g):
        pos, cs, dT = ctx.saved_tensors
        N, R = g.shape
        gp = torch.zeros(N, 4, dtype=torch.float32, device=g.device)
        if ctx.recast:
            rc = _ray_cfg(ctx.sensor, ctx.kind, True, ctx.n_agents)
            if getattr(ctx.scene, "ext_cull", False):
                rc.cull |= 2
            tr, tc, td = _tile_table(ctx.sensor, g.device)
            L.check(L.lib().qs_raycast_tiled_vjp(rc, ctx.scene.struct(), N, L.ptr(pos), 4,
                                                 L.ptr(cs) if ctx.has_cs else None, L.ptr(td), L.ptr(tc),
                                                 tr.shape[0], tr.shape[1], L.ptr(g.contiguous()), L.ptr(gp), 4,
                                                 L.stream_handle(g.device)), "qs_raycast_tiled_vjp")
        else:
            L.check(L.lib().qs_raycast_vjp(N, R, L.ptr(g.contiguous()), L.ptr(dT), L.ptr(gp), 4,
                                           L.stream_handle(g.device)), "qs_raycast_vjp")
        return gp[:, :3], None, None, None, None, None


def render_depth_differentiable(scene: DeviceScene, pos3: torch.Tensor, cam_cs: torch.Tensor,
                                sensor, kind=0, n_agents=1):
    return _RenderDepthFn.apply(pos3, scene, cam_cs, sensor, kind, n_agents)


# ---------------------------------------------------------------------------
# signed distance (q/sensors.py:417-501)


def _sdf_launch(sc: DeviceScene, p: torch.Tensor, n_agents: int, grad: bool):
    N = p.shape[0]
    pts = _pos4(p)
    out = torch.empty(N, dtype=torch.float32, device=p.device)
    g = torch.empty(N, 4, dtype=torch.float32, device=p.device) if grad else None
    L.check(L.lib().qs_sdf(sc.struct(), N, n_agents, L.ptr(pts), L.ptr(out), L.ptr(g),
                           L.stream_handle(p.device)), "qs_sdf")
    return out, g


def sdf_np(points, prims, n_agents: int = 1, device=None):
    """Signed distance (B,) to the nearest surface; FAR when the scene is empty."""
    dev = L.require_cuda(device if device is not None else L.tensor_device(points))
    sc = as_device_scene(prims, dev)
    out, _ = _sdf_launch(sc, _t(points, dev).reshape(-1, 3), n_agents, False)
    return out


class _SdfFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, p, sc, n_agents):
        out, g = _sdf_launch(sc, p.detach().float(), n_agents, True)
        ctx.save_for_backward(g)
        return out

    @staticmethod
    def backward(ctx, go):
        (g,) = ctx.saved_tensors
        return go[:, None] * g[:, :3], None, None


def sdf_var(p: torch.Tensor, prims, n_agents: int = 1):
    """Differentiable twin: gradient routes to the first argmin primitive."""
    sc = as_device_scene(prims, p.device)
    return _SdfFn.apply(p, sc, n_agents)


# ---------------------------------------------------------------------------
# IMU (q/sensors.py:508-555)


class ImuModel:
    """Accelerometer + gyro with white noise and random-walk bias.

    Noise is drawn in-kernel from Philox keyed by (seed, row, read index);
    ``read(..., noise=(4,B,3))`` injects host draws instead (same order as the
    reference: bias_a, bias_g, noise_a, noise_g).
    """

    def __init__(self, batch: int, accel_noise_std=0.0, gyro_noise_std=0.0, accel_bias_rw_std=0.0,
                 gyro_bias_rw_std=0.0, seed: int = 0, device=None):
        if min(accel_noise_std, gyro_noise_std, accel_bias_rw_std, gyro_bias_rw_std) < 0:
            raise SensorContractError("noise/drift stds must be >= 0")
        self.device = L.require_cuda(device)
        self.batch = batch
        self.accel_noise_std, self.gyro_noise_std = float(accel_noise_std), float(gyro_noise_std)
        self.accel_bias_rw_std, self.gyro_bias_rw_std = float(accel_bias_rw_std), float(gyro_bias_rw_std)
        self.seed = int(seed)
        self._tick = 0
        self._bias = torch.zeros(batch, 8, dtype=torch.float32, device=self.device)

    @property
    def accel_bias(self):
        return self._bias[:, 0:3]

    @property
    def gyro_bias(self):
        return self._bias[:, 4:7]

    def reset(self, env_mask=None):
        if env_mask is None:
            self._bias.zero_()
        else:
            m = _t(env_mask, self.device, torch.bool)
            self._bias[m] = 0.0

    def read(self, body_R, w_body, v_dot, g_vec, dt: float, noise=None):
        dev = self.device
        B = self.batch
        R = _t(body_R, dev).reshape(B, 9).contiguous()
        w = _pos4(_t(w_body, dev).reshape(B, 3)) if w_body is not None else None
        vd = _pos4(_t(v_dot, dev).reshape(B, 3))
        g = [float(x) for x in np.asarray(g_vec, dtype=np.float64).reshape(3)]
        nz = _t(noise, dev).reshape(4, B, 3).contiguous() if noise is not None else None
        out = torch.empty(B, 6, dtype=torch.float32, device=dev)
        gbuf = (L.f32 * 3)(*g)
        L.check(L.lib().qs_imu_read(B, L.ptr(R), L.ptr(w), L.ptr(vd), C_addr(gbuf), float(dt),
                                    self.accel_noise_std, self.gyro_noise_std, self.accel_bias_rw_std,
                                    self.gyro_bias_rw_std, self.seed, self._tick, L.ptr(nz),
                                    L.ptr(self._bias), L.ptr(out), L.stream_handle(dev)), "qs_imu_read")
        self._tick += 1
        return out[:, 0:3], out[:, 3:6]


def C_addr(buf):
    import ctypes

    return ctypes.addressof(buf)


# ---------------------------------------------------------------------------
# point-mass attitude (q/sensors.py:562-611)


def ema_update(v_ema, v, alpha: float):
    if not (0.0 < alpha <= 1.0):
        raise SensorContractError("ema alpha must lie in (0, 1]")
    return (1.0 - alpha) * v_ema + alpha * v


def reconstruct_attitude(a_thrust, v_ema, device=None):
    """(B,3,3) attitude with columns (x_b, y_b, z_b) (q/sensors.py:569-606)."""
    dev = L.require_cuda(device if device is not None else L.tensor_device(a_thrust))
    a = _pos4(_t(a_thrust, dev).reshape(-1, 3))
    ve = _pos4(_t(v_ema, dev).reshape(-1, 3))
    B = a.shape[0]
    R = torch.empty(B, 9, dtype=torch.float32, device=dev)
    L.check(L.lib().qs_reconstruct_attitude(B, L.ptr(a), L.ptr(ve), L.ptr(R), L.stream_handle(dev)),
            "qs_reconstruct_attitude")
    return R.reshape(B, 3, 3)


def yaw_of(R):
    """Yaw of body x about world z (q/sensors.py:609-611)."""
    if isinstance(R, torch.Tensor):
        return torch.atan2(R[..., 1, 0], R[..., 0, 0])
    return np.arctan2(R[..., 1, 0], R[..., 0, 0])


# ---------------------------------------------------------------------------
# DAIM dump format (q/sensors.py:614-642)

DUMP_MAGIC = b"DAIM"


def write_depth_dump(path, image, frame_index: int = 0) -> None:
    if isinstance(image, torch.Tensor):
        image = image.detach().cpu().numpy()
    img = np.asarray(image, dtype="<f4")
    if img.ndim == 1:
        img = img[None, :]
    h, w = img.shape
    with open(path, "wb") as f:
        f.write(DUMP_MAGIC)
        f.write(struct.pack("<III", w, h, frame_index))
        f.write(img.tobytes(order="C"))


def read_depth_dump(path):
    with open(path, "rb") as f:
        head = f.read(16)
        if len(head) != 16 or head[:4] != DUMP_MAGIC:
            raise SensorContractError(f"not a depth dump: {path}")
        w, h, idx = struct.unpack("<III", head[4:])
        data = np.frombuffer(f.read(), dtype="<f4")
    if data.size != w * h:
        raise SensorContractError(f"truncated depth dump: {path}")
    return data.reshape(h, w), idx


def ray_primitive(origin, direction, prim):
    """q/sensors.py:219-242: smallest t >= 0 of one unit ray against one
    primitive ("sphere", (4,)) | ("box", (6,)) | ("cylinder", (5,)) | ("ground", z),
    or None -- through the same ray-cast kernel as every sensor."""
    direction = np.asarray(direction, dtype=np.float64)
    if abs(np.linalg.norm(direction) - 1.0) > 1e-9:
        raise SensorContractError("ray direction must be unit-norm")
    kind, data = prim
    if kind not in ("sphere", "box", "cylinder", "ground"):
        raise SensorContractError(f"unknown primitive kind '{kind}'")
    ps = PrimitiveSet(spheres=data if kind == "sphere" else np.zeros((0, 4)),
                      boxes=data if kind == "box" else np.zeros((0, 6)),
                      cylinders=data if kind == "cylinder" else np.zeros((0, 5)),
                      ground_z=float(data) if kind == "ground" else None)
    big = 1e30
    t = raycast(pack_primitives([ps]), np.asarray(origin, dtype=np.float64)[None, :],
                direction[None, None, :], big, device=L.require_cuda(None))
    v = float(t.reshape(-1)[0])
    return None if v >= big else v
