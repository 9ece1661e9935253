"""fp64 numpy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line it restates; ``q/`` is
``/root/reference/pkg/src/quadsim/``.  The restatement is value-level (no
autodiff tape): gradients come from central differences in fp64
(``fd_grad_actions``), the reference's own oracle technique
(``pkg/tests/oracles.py:15-30``).  Parity of this module with the reference is
pinned by ``tests/golden`` fixtures produced by the reference itself.

Nothing in the product package imports this module.
"""

from __future__ import annotations

import copy
import math
from dataclasses import dataclass, field

import numpy as np

GRAVITY = np.array([0.0, 0.0, -9.81])
FAR = 1e9  # q/sensors.py:25
TERM_NONE, TERM_SUCCESS, TERM_COLLISION, TERM_BOUNDS = 0, 1, 2, 3  # q/tasks.py:25-28

SPHERE_R = (0.3, 1.0)  # q/world.py:21-24
BOX_HALF = (0.2, 1.0)
CYL_R = (0.2, 0.6)
CYL_HH = (0.5, 2.0)
GRID_RES = 0.25


class OracleGenerationError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# dynamics (q/dynamics.py)


@dataclass
class Params:
    """q/dynamics.py:42-82 (QuadParams).  drag_coeff / lag_decay scalar or (B,)."""

    dt: float = 0.01
    inertia: np.ndarray = field(default_factory=lambda: np.diag([2.3e-3, 2.3e-3, 4.0e-3]))
    drag_matrix_diag: np.ndarray = field(default_factory=lambda: np.zeros(3))
    drag_coeff: object = 0.3
    latency: object = 4.0
    g_vec: np.ndarray = field(default_factory=lambda: GRAVITY.copy())
    rate_gains: np.ndarray = field(default_factory=lambda: np.array([20.0, 20.0, 8.0]))

    @property
    def inertia_inv(self):
        return np.linalg.inv(np.asarray(self.inertia, dtype=np.float64))

    @property
    def lag_decay(self):
        return np.exp(-np.asarray(self.latency, dtype=np.float64) * self.dt)


MODEL_ACTION_DIM = {"full": 4, "simplified": 4, "pm_continuous": 3, "pm_discrete": 3}
STATE_FIELDS = {
    "full": ("p", "v", "q", "w"),
    "simplified": ("p", "v", "R"),
    "pm_continuous": ("p", "v", "a_lat"),
    "pm_discrete": ("p", "v", "u_prev"),
}


def action_box(model: str, g_vec=GRAVITY):
    """q/dynamics.py:342-346 (full), :398-402 (pm_cont), :424-425 (pm_disc)."""
    gz = -g_vec[2]
    if model in ("full", "simplified"):  # :342-346, :373-376
        return np.array([0.0, -6.0, -6.0, -3.0]), np.array([2.0 * gz, 6.0, 6.0, 3.0])
    if model == "pm_continuous":
        return np.array([-6.0, -6.0, gz - 6.0]), np.array([6.0, 6.0, gz + 6.0])
    if model == "pm_discrete":
        return np.full(3, -6.0), np.full(3, 6.0)
    raise ValueError(model)


def init_state(model: str, p, v, g_vec=GRAVITY):
    """q/dynamics.py:324-330, 386-390, 412-416."""
    B = p.shape[0]
    st = {"p": np.array(p, dtype=np.float64), "v": np.array(v, dtype=np.float64)}
    if model == "full":
        q = np.zeros((B, 4))
        q[:, 0] = 1.0
        st["q"] = q
        st["w"] = np.zeros((B, 3))
    elif model == "simplified":  # q/dynamics.py:356-360
        st["R"] = np.broadcast_to(np.eye(3), (B, 3, 3)).copy()
    elif model == "pm_continuous":
        st["a_lat"] = np.broadcast_to(-g_vec, (B, 3)).copy()
    else:
        st["u_prev"] = np.zeros((B, 3))
    return st


def squash(raw, lo, hi):
    """q/dynamics.py:277-284: center + half * tanh(raw)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    return (lo + hi) * 0.5 + (hi - lo) * 0.5 * np.tanh(raw)


def _cross(a, b):
    return np.cross(a, b)


def quat_rotate(q, v):
    """q/autodiff.py:737-750: v + 2 (w (u x v) + u x (u x v))."""
    u = q[..., 1:]
    w = q[..., :1]
    v = np.broadcast_to(v, u.shape)
    uv = _cross(u, v)
    uuv = _cross(u, uv)
    return v + (uv * w + uuv) * 2.0


def quat_mul(q, r):
    """q/autodiff.py:689-701 (Hamilton product, scalar first)."""
    qw, qx, qy, qz = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    rw, rx, ry, rz = r[..., 0], r[..., 1], r[..., 2], r[..., 3]
    return np.stack([
        qw * rw - qx * rx - qy * ry - qz * rz,
        qw * rx + qx * rw + qy * rz - qz * ry,
        qw * ry - qx * rz + qy * rw + qz * rx,
        qw * rz + qx * ry - qy * rx + qz * rw,
    ], axis=-1)


def quat_to_matrix(q):
    """q/dynamics.py:448-460."""
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    R = np.empty(q.shape[:-1] + (3, 3))
    R[..., 0, 0] = 1 - 2 * (y * y + z * z)
    R[..., 0, 1] = 2 * (x * y - w * z)
    R[..., 0, 2] = 2 * (x * z + w * y)
    R[..., 1, 0] = 2 * (x * y + w * z)
    R[..., 1, 1] = 1 - 2 * (x * x + z * z)
    R[..., 1, 2] = 2 * (y * z - w * x)
    R[..., 2, 0] = 2 * (x * z - w * y)
    R[..., 2, 1] = 2 * (y * z + w * x)
    R[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def _bcast(x, B):
    x = np.asarray(x, dtype=np.float64)
    return x if x.ndim == 0 else x.reshape(B, 1)


def step_pm_continuous(st, u, prm: Params):
    """q/dynamics.py:237-258."""
    B = u.shape[0]
    decay = _bcast(prm.lag_decay, B)
    d = _bcast(prm.drag_coeff, B)
    a_next = u + (st["a_lat"] - u) * decay
    v_dot = a_next + prm.g_vec - d * st["v"]
    return {"p": st["p"] + st["v"] * prm.dt, "v": st["v"] + v_dot * prm.dt, "a_lat": a_next}


def step_pm_discrete(st, u, prm: Params):
    """q/dynamics.py:261-274."""
    dt = prm.dt
    return {
        "p": st["p"] + (st["v"] * dt + u * (0.5 * dt * dt)),
        "v": st["v"] + (st["u_prev"] + u) * (0.5 * dt),
        "u_prev": u.copy(),
    }


def step_full(st, act, prm: Params):
    """q/dynamics.py:140-186 (rate_loop :140-152, step :155-186)."""
    p, v, q, w = st["p"], st["v"], st["q"], st["w"]
    c = act[:, 0:1]
    w_cmd = act[:, 1:4]
    J = np.asarray(prm.inertia)
    Jinv = prm.inertia_inv
    z_b = quat_rotate(q, np.array([0.0, 0.0, 1.0]))
    qc = np.concatenate([q[:, :1], -q[:, 1:]], axis=-1)
    v_body = quat_rotate(qc, v)
    drag = quat_rotate(q, prm.drag_matrix_diag * v_body)
    v_dot = (prm.g_vec + z_b * c) - drag
    err = prm.rate_gains * (w_cmd - w)
    Jw = w @ J.T
    gyro = np.cross(w, Jw)
    tau = err @ J.T + gyro
    w_dot = (tau - gyro) @ Jinv.T
    q_dot = quat_mul(q, np.concatenate([np.zeros((q.shape[0], 1)), w], axis=-1)) * 0.5
    dt = prm.dt
    qn = q + q_dot * dt
    qn = qn / np.sqrt(np.sum(qn * qn, axis=-1, keepdims=True))
    return {"p": p + v * dt, "v": v + v_dot * dt, "q": qn, "w": w + w_dot * dt}


def step_simplified(st, act, prm: Params):
    """q/dynamics.py:189-234 (Gram-Schmidt columns :189-198)."""
    p, v, R = st["p"], st["v"], st["R"]
    c = act[:, 0:1]
    wx, wy, wz = act[:, 1], act[:, 2], act[:, 3]
    zero = np.zeros_like(wx)
    skew = np.stack([np.stack([zero, -wz, wy], -1), np.stack([wz, zero, -wx], -1),
                     np.stack([-wy, wx, zero], -1)], -2)
    R_dot = R @ skew
    M = R + R_dot * prm.dt
    x, y = M[..., 0], M[..., 1]
    xn = x / np.linalg.norm(x, axis=-1, keepdims=True)
    y_orth = y - xn * np.sum(y * xn, -1, keepdims=True)
    yn = y_orth / np.linalg.norm(y_orth, axis=-1, keepdims=True)
    zn = np.cross(xn, yn)
    v_dot = R[..., 2] * c + prm.g_vec
    return {"p": p + v * prm.dt, "v": v + v_dot * prm.dt, "R": np.stack([xn, yn, zn], -1)}


def model_step(model: str, st, act, prm: Params):
    if model == "full":
        return step_full(st, act, prm)
    if model == "simplified":
        return step_simplified(st, act, prm)
    if model == "pm_continuous":
        return step_pm_continuous(st, act, prm)
    return step_pm_discrete(st, act, prm)


def thrust_accel(model: str, st, g_vec=GRAVITY):
    """q/dynamics.py:406 (pm_cont), :430 (pm_disc)."""
    if model == "pm_continuous":
        return st["a_lat"]
    return st["u_prev"] - g_vec


# ---------------------------------------------------------------------------
# attitude (q/sensors.py:562-611, q/tasks.py:129-137)


def ema_update(v_ema, v, alpha):
    """q/sensors.py:562-566."""
    return (1.0 - alpha) * v_ema + alpha * v


def reconstruct_attitude(a_thrust, v_ema):
    """q/sensors.py:569-606."""
    B = a_thrust.shape[0]
    tn = np.linalg.norm(a_thrust, axis=-1)
    z_b = np.where((tn > 1e-6)[:, None], a_thrust / np.maximum(tn, 1e-12)[:, None],
                   np.array([0.0, 0.0, 1.0]))
    horiz = v_ema.copy()
    horiz[:, 2] = 0.0
    hn = np.linalg.norm(horiz, axis=-1)
    x_ref = np.where((hn > 1e-3)[:, None], horiz / np.maximum(hn, 1e-12)[:, None],
                     np.array([1.0, 0.0, 0.0]))
    zz = z_b[:, 2]
    upright = np.abs(zz) > 0.1
    xz = -(x_ref[:, 0] * z_b[:, 0] + x_ref[:, 1] * z_b[:, 1]) / np.where(upright, zz, 1.0)
    x_solve = np.stack([x_ref[:, 0], x_ref[:, 1], xz], axis=-1)
    x_gs = x_ref - np.sum(x_ref * z_b, axis=-1, keepdims=True) * z_b
    x_raw = np.where(upright[:, None], x_solve, x_gs)
    xn = np.linalg.norm(x_raw, axis=-1)
    fb = np.cross(np.broadcast_to([0.0, 1.0, 0.0], (B, 3)), z_b)
    fn = np.linalg.norm(fb, axis=-1)
    fb = fb / np.maximum(fn, 1e-12)[:, None]
    x_b = np.where((xn > 1e-9)[:, None], x_raw / np.maximum(xn, 1e-12)[:, None], fb)
    y_b = np.cross(z_b, x_b)
    return np.stack([x_b, y_b, z_b], axis=-1)


def yaw_of(R):
    """q/sensors.py:609-611."""
    return np.arctan2(R[..., 1, 0], R[..., 0, 0])


def rotz(yaw):
    """q/tasks.py:129-137."""
    c, s = np.cos(yaw), np.sin(yaw)
    R = np.zeros(np.shape(yaw) + (3, 3))
    R[..., 0, 0] = c
    R[..., 0, 1] = -s
    R[..., 1, 0] = s
    R[..., 1, 1] = c
    R[..., 2, 2] = 1.0
    return R


def matvec(R, v):
    return np.sum(R * v[..., None, :], axis=-1)


def attitude(model: str, st, v_ema, g_vec=GRAVITY):
    """q/tasks.py:400-410."""
    if model == "full":
        return quat_to_matrix(st["q"])
    if model == "simplified":
        return st["R"]
    return reconstruct_attitude(thrust_accel(model, st, g_vec), v_ema)


# ---------------------------------------------------------------------------
# primitives, ray casting, sdf (q/sensors.py:32-501)


def pack_primitives(sets):
    """q/sensors.py:100-124.  ``sets``: dicts with spheres/boxes/cylinders/ground_z."""
    B = len(sets)
    sp = [np.asarray(s.get("spheres", np.zeros((0, 4))), dtype=np.float64).reshape(-1, 4) for s in sets]
    bx = [np.asarray(s.get("boxes", np.zeros((0, 6))), dtype=np.float64).reshape(-1, 6) for s in sets]
    cy = [np.asarray(s.get("cylinders", np.zeros((0, 5))), dtype=np.float64).reshape(-1, 5) for s in sets]
    Sm = max([len(a) for a in sp] + [1])
    Bm = max([len(a) for a in bx] + [1])
    Cm = max([len(a) for a in cy] + [1])
    out = {
        "spheres": np.zeros((B, Sm, 4)), "sph_valid": np.zeros((B, Sm), bool),
        "boxes": np.zeros((B, Bm, 6)), "box_valid": np.zeros((B, Bm), bool),
        "cylinders": np.zeros((B, Cm, 5)), "cyl_valid": np.zeros((B, Cm), bool),
        "ground_z": np.full(B, np.nan),
    }
    for i, s in enumerate(sets):
        out["spheres"][i, :len(sp[i])] = sp[i]
        out["sph_valid"][i, :len(sp[i])] = True
        out["boxes"][i, :len(bx[i])] = bx[i]
        out["box_valid"][i, :len(bx[i])] = True
        out["cylinders"][i, :len(cy[i])] = cy[i]
        out["cyl_valid"][i, :len(cy[i])] = True
        if s.get("ground_z") is not None:
            out["ground_z"][i] = s["ground_z"]
    return out


def prims_take(prims, idx):
    return {k: v[idx] for k, v in prims.items()}


def _ray_spheres(o, d, spheres, valid):
    """q/sensors.py:131-143."""
    oc = o[:, None, :] - spheres[..., :3]
    b = np.einsum("brk,bsk->brs", d, oc)
    c = np.sum(oc * oc, axis=-1) - spheres[..., 3] ** 2
    disc = b * b - c[:, None, :]
    with np.errstate(invalid="ignore"):
        sq = np.sqrt(np.maximum(disc, 0.0))
        t1 = -b - sq
        t2 = -b + sq
    t = np.where(t1 >= 0.0, t1, np.where(t2 >= 0.0, t2, np.inf))
    return np.where((disc >= 0.0) & valid[:, None, :], t, np.inf)


def _ray_boxes(o, d, boxes, valid):
    """q/sensors.py:146-164."""
    lo = boxes[..., :3] - boxes[..., 3:6]
    hi = boxes[..., :3] + boxes[..., 3:6]
    od = o[:, None, None, :]
    dd = d[:, :, None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        t1 = (lo[:, None] - od) / dd
        t2 = (hi[:, None] - od) / dd
        tn = np.minimum(t1, t2)
        tf = np.maximum(t1, t2)
    tn = np.nan_to_num(tn, nan=np.inf)
    tf = np.nan_to_num(tf, nan=-np.inf)
    t_near = np.max(tn, axis=-1)
    t_far = np.min(tf, axis=-1)
    hit = (t_near <= t_far) & (t_far >= 0.0) & valid[:, None, :]
    t = np.where(t_near >= 0.0, t_near, t_far)
    return np.where(hit, t, np.inf)


def _ray_cylinders(o, d, cyls, valid):
    """q/sensors.py:167-206."""
    cx, cy, cz, r, hh = (cyls[..., i] for i in range(5))
    ox = o[:, 0:1, None] - cx[:, None, :]
    oy = o[:, 1:2, None] - cy[:, None, :]
    oz = o[:, 2:3, None] - cz[:, None, :]
    dx = d[..., 0][:, :, None]
    dy = d[..., 1][:, :, None]
    dz = d[..., 2][:, :, None]
    a = dx * dx + dy * dy
    b = ox * dx + oy * dy
    c = ox * ox + oy * oy - (r * r)[:, None, :]
    disc = b * b - a * c
    with np.errstate(divide="ignore", invalid="ignore"):
        sq = np.sqrt(np.maximum(disc, 0.0))
        ts1 = (-b - sq) / a
        ts2 = (-b + sq) / a

        def side_ok(t):
            z = oz + t * dz
            return (disc >= 0.0) & (a > 1e-300) & (t >= 0.0) & (np.abs(z) <= hh[:, None, :])

        t_side = np.where(side_ok(ts1), ts1, np.where(side_ok(ts2), ts2, np.inf))
        t_top = (hh[:, None, :] - oz) / dz
        t_bot = (-hh[:, None, :] - oz) / dz

        def cap_ok(t):
            x = ox + t * dx
            y = oy + t * dy
            inside = x * x + y * y <= (r * r)[:, None, :]
            return (t >= 0.0) & np.isfinite(t) & inside

        t_top = np.where(cap_ok(t_top), t_top, np.inf)
        t_bot = np.where(cap_ok(t_bot), t_bot, np.inf)
    t = np.minimum(t_side, np.minimum(t_top, t_bot))
    return np.where(valid[:, None, :], t, np.inf)


def _ray_ground(o, d, ground_z):
    """q/sensors.py:209-216."""
    oz = o[:, 2][:, None]
    dz = d[..., 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        t = (ground_z[:, None] - oz) / dz
    ok = np.isfinite(t) & (t >= 0.0)
    return np.where(ok, t, np.inf)


def raycast(prims, origins, dirs, max_range, chunk_elems=4_000_000):
    """q/sensors.py:245-269.  Returns (B,R) clamped to max_range."""
    B, R = dirs.shape[:2]
    P = prims["spheres"].shape[1] + prims["boxes"].shape[1] + prims["cylinders"].shape[1]
    rows = max(1, min(B, chunk_elems // max(1, R * max(P, 1))))
    out = np.empty((B, R))
    for s in range(0, B, rows):
        sl = slice(s, min(B, s + rows))
        o, d = origins[sl], dirs[sl]
        t = np.full((o.shape[0], R), np.inf)
        if prims["sph_valid"][sl].any():
            t = np.minimum(t, _ray_spheres(o, d, prims["spheres"][sl], prims["sph_valid"][sl]).min(axis=-1))
        if prims["box_valid"][sl].any():
            t = np.minimum(t, _ray_boxes(o, d, prims["boxes"][sl], prims["box_valid"][sl]).min(axis=-1))
        if prims["cyl_valid"][sl].any():
            t = np.minimum(t, _ray_cylinders(o, d, prims["cylinders"][sl], prims["cyl_valid"][sl]).min(axis=-1))
        t = np.minimum(t, _ray_ground(o, d, prims["ground_z"][sl]))
        out[sl] = np.minimum(t, max_range)
    return out


def pixel_dirs(width, height, fov_h=np.deg2rad(90.0), fov_v=np.deg2rad(75.0)):
    """q/sensors.py:292-302."""
    th = np.tan(fov_h / 2)
    tv = np.tan(fov_v / 2)
    cols = (np.arange(width) + 0.5) / width
    rows = (np.arange(height) + 0.5) / height
    y = th * (1.0 - 2.0 * cols)
    z = tv * (1.0 - 2.0 * rows)
    zz, yy = np.meshgrid(z, y, indexing="ij")
    d = np.stack([np.ones_like(yy), yy, zz], axis=-1).reshape(-1, 3)
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def lidar_dirs(n_az, n_el, az_ext=2 * np.pi, el_ext=np.deg2rad(30.0)):
    """q/sensors.py:323-335."""
    az = np.linspace(0.0, az_ext, n_az, endpoint=False)
    el = np.linspace(-0.5, 0.5, n_el) * el_ext if n_el > 1 else np.zeros(1)
    aa, ee = np.meshgrid(az, el, indexing="ij")
    return np.stack([np.cos(ee) * np.cos(aa), np.cos(ee) * np.sin(aa), np.sin(ee)],
                    axis=-1).reshape(-1, 3)


def _bounding_radii(prims):
    return (prims["spheres"][..., 3],
            np.linalg.norm(prims["boxes"][..., 3:6], axis=-1),
            np.sqrt(prims["cylinders"][..., 3] ** 2 + prims["cylinders"][..., 4] ** 2))


def fov_cull(prims, cam_pos, cam_R, max_range, fov_h=np.deg2rad(90.0), fov_v=np.deg2rad(75.0)):
    """q/sensors.py:338-374."""
    th = np.tan(fov_h / 2)
    tv = np.tan(fov_v / 2)
    normals = np.array([[th, -1.0, 0.0], [th, 1.0, 0.0], [tv, 0.0, -1.0], [tv, 0.0, 1.0],
                        [1.0, 0.0, 0.0]])
    normals /= np.linalg.norm(normals, axis=-1, keepdims=True)

    def keep(cen, rad):
        rel = cen - cam_pos[:, None, :]
        local = np.einsum("bji,bpj->bpi", cam_R, rel)
        sd = np.einsum("kp,bnp->bnk", normals, local)
        inside = np.all(sd >= -rad[..., None] - 1e-9, axis=-1)
        rng_ok = np.linalg.norm(local, axis=-1) - rad <= max_range + 1e-9
        return inside & rng_ok

    rs, rb, rc = _bounding_radii(prims)
    return (keep(prims["spheres"][..., :3], rs), keep(prims["boxes"][..., :3], rb),
            keep(prims["cylinders"][..., :3], rc))


def _masked(prims, ks, kb, kc):
    out = dict(prims)
    out["sph_valid"] = prims["sph_valid"] & ks
    out["box_valid"] = prims["box_valid"] & kb
    out["cyl_valid"] = prims["cyl_valid"] & kc
    return out


def render_depth(prims, body_pos, body_R, width, height, max_range, cull=True,
                 offset=np.zeros(3)):
    """q/sensors.py:377-389."""
    B = body_pos.shape[0]
    cam_pos = body_pos + np.einsum("bij,j->bi", body_R, offset)
    dirs = np.einsum("bij,rj->bri", body_R, pixel_dirs(width, height))
    use = prims
    if cull:
        use = _masked(prims, *fov_cull(prims, cam_pos, body_R, max_range))
    return raycast(use, cam_pos, dirs, max_range).reshape(B, height, width)


def render_lidar(prims, body_pos, body_R, n_az, n_el, max_range, az_ext=2 * np.pi,
                 el_ext=np.deg2rad(30.0), offset=np.zeros(3)):
    """q/sensors.py:392-410."""
    origin = body_pos + np.einsum("bij,j->bi", body_R, offset)
    dirs = np.einsum("bij,rj->bri", body_R, lidar_dirs(n_az, n_el, az_ext, el_ext))
    rs, rb, rc = _bounding_radii(prims)

    def ball(cen, rad):
        return np.linalg.norm(cen - origin[:, None, :], axis=-1) - rad <= max_range + 1e-9

    use = _masked(prims, ball(prims["spheres"][..., :3], rs), ball(prims["boxes"][..., :3], rb),
                  ball(prims["cylinders"][..., :3], rc))
    return raycast(use, origin, dirs, max_range)


def sdf(points, prims):
    """q/sensors.py:417-445 (sdf_np)."""
    B = points.shape[0]
    best = np.full(B, FAR)
    if prims["sph_valid"].any():
        d = np.linalg.norm(points[:, None, :] - prims["spheres"][..., :3], axis=-1) - prims["spheres"][..., 3]
        best = np.minimum(best, np.where(prims["sph_valid"], d, FAR).min(axis=-1))
    if prims["box_valid"].any():
        q = np.abs(points[:, None, :] - prims["boxes"][..., :3]) - prims["boxes"][..., 3:6]
        d = np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(q.max(axis=-1), 0.0)
        best = np.minimum(best, np.where(prims["box_valid"], d, FAR).min(axis=-1))
    if prims["cyl_valid"].any():
        dxy = np.linalg.norm(points[:, None, :2] - prims["cylinders"][..., :2], axis=-1) - prims["cylinders"][..., 3]
        dz = np.abs(points[:, None, 2] - prims["cylinders"][..., 2]) - prims["cylinders"][..., 4]
        d = np.sqrt(np.maximum(dxy, 0.0) ** 2 + np.maximum(dz, 0.0) ** 2) + np.minimum(np.maximum(dxy, dz), 0.0)
        best = np.minimum(best, np.where(prims["cyl_valid"], d, FAR).min(axis=-1))
    has_g = np.isfinite(prims["ground_z"])
    best = np.minimum(best, np.where(has_g, points[:, 2] - np.where(has_g, prims["ground_z"], -FAR), FAR))
    return best


def sdf_single_scene(points, prims1):
    """q/world.py:182-196 (sdf_np_all): many points against one packed scene."""
    n = points.shape[0]
    rep = {k: np.broadcast_to(v, (n,) + v.shape[1:]) for k, v in prims1.items()}
    return sdf(points, rep)


# ---------------------------------------------------------------------------
# IMU (q/sensors.py:508-555)


class Imu:
    """ImuModel restated; ``normals`` optionally injected (same draw order)."""

    def __init__(self, batch, accel_noise_std=0.0, gyro_noise_std=0.0, accel_bias_rw_std=0.0,
                 gyro_bias_rw_std=0.0, seed=0):
        self.batch = batch
        self.sa, self.sg, self.ra, self.rg = accel_noise_std, gyro_noise_std, accel_bias_rw_std, gyro_bias_rw_std
        self.accel_bias = np.zeros((batch, 3))
        self.gyro_bias = np.zeros((batch, 3))
        self._rng = np.random.default_rng(seed)

    def reset(self, mask=None):
        if mask is None:
            self.accel_bias[:] = 0.0
            self.gyro_bias[:] = 0.0
        else:
            self.accel_bias[mask] = 0.0
            self.gyro_bias[mask] = 0.0

    def draw(self):
        """The four normal blocks in the reference's draw order (:544-554)."""
        B = self.batch
        n_ba = self._rng.standard_normal((B, 3))
        n_bg = self._rng.standard_normal((B, 3))
        n_a = self._rng.standard_normal((B, 3)) if self.sa else np.zeros((B, 3))
        n_g = self._rng.standard_normal((B, 3)) if self.sg else np.zeros((B, 3))
        return n_ba, n_bg, n_a, n_g

    def read(self, body_R, w_body, v_dot, g_vec, dt, normals=None):
        n_ba, n_bg, n_a, n_g = self.draw() if normals is None else normals
        sq = np.sqrt(dt)
        self.accel_bias += self.ra * sq * n_ba
        self.gyro_bias += self.rg * sq * n_bg
        accel = np.einsum("bji,bj->bi", body_R, v_dot - g_vec) + self.accel_bias
        if self.sa:
            accel = accel + self.sa * n_a
        if w_body is None:
            w_body = np.zeros((self.batch, 3))
        gyro = w_body + self.gyro_bias
        if self.sg:
            gyro = gyro + self.sg * n_g
        return accel, gyro


# ---------------------------------------------------------------------------
# world generation and resets (q/world.py)


@dataclass
class RandomizationSpec:
    """q/world.py:114-127."""

    drag_coeff: tuple = (0.1, 0.5)
    latency: tuple = (2.0, 8.0)
    action_scale: tuple = (1.0, 1.0)
    per_episode: bool = True


def randomize_params(spec: RandomizationSpec, seed, episode, n):
    """q/world.py:130-137."""
    rng = np.random.default_rng([seed & 0x7FFFFFFF, episode])
    return {
        "drag_coeff": rng.uniform(*spec.drag_coeff, size=n),
        "latency": rng.uniform(*spec.latency, size=n),
        "action_scale": rng.uniform(*spec.action_scale, size=n),
    }


def formation_offsets(kind, n_agents, side=2.0):
    """q/world.py:386-406."""
    if n_agents == 1:
        return np.zeros((1, 3))
    if kind == "line":
        out = np.zeros((n_agents, 3))
        out[:, 1] = (np.arange(n_agents) - (n_agents - 1) / 2) * side
        return out
    if kind == "square":
        rows = int(np.ceil(np.sqrt(n_agents)))
        out = np.array([[(i % rows) * side, (i // rows) * side, 0.0] for i in range(n_agents)])
        return out - out.mean(axis=0)
    if kind == "circle":
        ang = 2 * np.pi * np.arange(n_agents) / n_agents
        r = side / (2 * np.sin(np.pi / n_agents))
        return np.stack([r * np.cos(ang), r * np.sin(ang), np.zeros(n_agents)], axis=-1)
    raise OracleGenerationError(kind)


@dataclass
class Scene:
    """q/world.py:61-70."""

    prims: dict
    bounds_lo: np.ndarray
    bounds_hi: np.ndarray
    spawn: np.ndarray
    goal: np.ndarray
    gates: list = field(default_factory=list)  # (center, normal, inner, frame)
    seed: int = 0
    style: str = "outdoor"


def grid_path_exists(scene: Scene, r_quad=0.15, res=GRID_RES):
    """q/world.py:144-179 (6-connected BFS over the inflated occupancy grid)."""
    lo = scene.bounds_lo + 1e-9
    hi = scene.bounds_hi - 1e-9
    dims = np.maximum(2, np.ceil((hi - lo) / res).astype(int))
    axes = [lo[i] + (np.arange(dims[i]) + 0.5) * (hi[i] - lo[i]) / dims[i] for i in range(3)]
    xx, yy, zz = np.meshgrid(*axes, indexing="ij")
    pts = np.stack([xx, yy, zz], axis=-1).reshape(-1, 3)
    sd = sdf_single_scene(pts, pack_primitives([scene.prims]))
    free = (sd > r_quad + 0.05).reshape(tuple(dims))

    def cell_of(p):
        idx = ((p - lo) / (hi - lo) * dims).astype(int)
        return tuple(np.clip(idx, 0, dims - 1))

    start, target = cell_of(scene.spawn), cell_of(scene.goal)
    if not free[start] or not free[target]:
        return False
    visited = np.zeros_like(free)
    visited[start] = True
    while True:
        grown = visited.copy()
        grown[1:, :, :] |= visited[:-1, :, :]
        grown[:-1, :, :] |= visited[1:, :, :]
        grown[:, 1:, :] |= visited[:, :-1, :]
        grown[:, :-1, :] |= visited[:, 1:, :]
        grown[:, :, 1:] |= visited[:, :, :-1]
        grown[:, :, :-1] |= visited[:, :, 1:]
        grown &= free
        if grown[target]:
            return True
        if np.array_equal(grown, visited):
            return False
        visited = grown


def _dist_rows(ends, spheres, boxes, cyls):
    def ds(rows):
        d = np.linalg.norm(ends[:, None, :] - rows[None, :, :3], axis=-1)
        return (d - rows[None, :, 3]).min(axis=0)

    def db(rows):
        q = np.abs(ends[:, None, :] - rows[None, :, :3]) - rows[None, :, 3:6]
        return (np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(q.max(-1), 0.0)).min(axis=0)

    def dc(rows):
        dxy = np.linalg.norm(ends[:, None, :2] - rows[None, :, :2], axis=-1) - rows[None, :, 3]
        dz = np.abs(ends[:, None, 2] - rows[None, :, 2]) - rows[None, :, 4]
        out = np.sqrt(np.maximum(dxy, 0) ** 2 + np.maximum(dz, 0) ** 2)
        out += np.minimum(np.maximum(dxy, dz), 0.0)
        return out.min(axis=0)

    return ds, db, dc


def obstacle_course_frame(spawn, goal, style="outdoor", corridor_halfwidth=3.0):
    """Corridor frame + bounds (q/world.py:224-249)."""
    span = goal - spawn
    dist = float(np.linalg.norm(span))
    fwd = span / dist
    fwd_h = np.array([fwd[0], fwd[1], 0.0])
    fwd_h = fwd_h / max(np.linalg.norm(fwd_h), 1e-9)
    left = np.array([-fwd_h[1], fwd_h[0], 0.0])
    height = 3.0 if style == "indoor" else 4.0
    pad = 1.5
    corners = np.array([spawn + fwd_h * a + left * b
                        for a in (-pad, dist + pad)
                        for b in (-corridor_halfwidth - pad, corridor_halfwidth + pad)])
    lo = np.array([corners[:, 0].min(), corners[:, 1].min(), 0.0])
    hi = np.array([corners[:, 0].max(), corners[:, 1].max(), height])
    return dist, fwd_h, left, height, lo, hi


def shell_boxes(lo, hi, height):
    """Indoor shell: ceiling + 4 walls (q/world.py:284-296)."""
    cx, cy = (lo[:2] + hi[:2]) / 2
    sx, sy = (hi[:2] - lo[:2]) / 2
    wt = 0.1
    return np.array([
        [cx, cy, height + wt, sx + 1, sy + 1, wt],
        [lo[0] - wt, cy, height / 2, wt, sy + 1, height],
        [hi[0] + wt, cy, height / 2, wt, sy + 1, height],
        [cx, lo[1] - wt, height / 2, sx + 1, wt, height],
        [cx, hi[1] + wt, height / 2, sx + 1, wt, height],
    ])


def gen_obstacle_course(seed, spawn, goal, density, style="outdoor", r_quad=0.15, clearance=0.5,
                        corridor_halfwidth=3.0, max_attempts=100):
    """q/world.py:207-340."""
    spawn = np.asarray(spawn, dtype=np.float64)
    goal = np.asarray(goal, dtype=np.float64)
    dist, fwd_h, left, height, lo, hi = obstacle_course_frame(spawn, goal, style, corridor_halfwidth)
    if dist <= 2.0:
        raise OracleGenerationError("spawn and goal too close")
    n_total = int(round(density * dist * 2 * corridor_halfwidth))
    for attempt in range(max_attempts):
        rng = np.random.default_rng([seed & 0x7FFFFFFF, attempt])
        n_cyl = int(round(0.4 * n_total))
        n_sph = int(round(0.3 * n_total))
        n_box = n_total - n_cyl - n_sph

        def corridor_point(n):
            along = rng.uniform(0.0, dist, size=n)
            lat = rng.uniform(-corridor_halfwidth, corridor_halfwidth, size=n)
            z = rng.uniform(0.3, height - 0.3, size=n)
            pts = spawn[None] + along[:, None] * fwd_h[None] + lat[:, None] * left[None]
            pts[:, 2] = z
            return pts

        spheres = np.zeros((0, 4))
        if n_sph:
            c = corridor_point(n_sph)
            spheres = np.column_stack([c, rng.uniform(*SPHERE_R, size=n_sph)])
        boxes = np.zeros((0, 6))
        if n_box:
            c = corridor_point(n_box)
            boxes = np.column_stack([c, rng.uniform(*BOX_HALF, size=(n_box, 3))])
        cylinders = np.zeros((0, 5))
        if n_cyl:
            c = corridor_point(n_cyl)
            r = rng.uniform(*CYL_R, size=n_cyl)
            hh = rng.uniform(*CYL_HH, size=n_cyl)
            c[:, 2] = hh
            cylinders = np.column_stack([c, r, hh])
        shell = shell_boxes(lo, hi, height) if style == "indoor" else np.zeros((0, 6))
        all_boxes = np.vstack([boxes, shell]) if len(shell) else boxes
        keep_min = r_quad + clearance
        ends = np.stack([spawn, goal])
        ds, db, dc = _dist_rows(ends, spheres, boxes, cylinders)
        if len(spheres):
            spheres = spheres[ds(spheres) > keep_min]
        if len(all_boxes):
            keep = np.ones(len(all_boxes), dtype=bool)
            keep[:len(boxes)] = db(all_boxes[:len(boxes)]) > keep_min
            all_boxes = all_boxes[keep]
        if len(cylinders):
            cylinders = cylinders[dc(cylinders) > keep_min]
        prims = {"spheres": spheres, "boxes": all_boxes, "cylinders": cylinders, "ground_z": 0.0}
        scene = Scene(prims=prims, bounds_lo=lo, bounds_hi=hi, spawn=spawn.copy(), goal=goal.copy(),
                      seed=seed, style=style)
        if grid_path_exists(scene, r_quad=r_quad):
            return scene
    raise OracleGenerationError(f"no feasible scene (seed={seed})")


def gen_race_track(seed, n_gates, spread=10.0):
    """q/world.py:347-379."""
    rng = np.random.default_rng(seed & 0x7FFFFFFF)
    spawn = np.array([0.0, 0.0, 1.5])
    heading = 0.0
    pos = spawn.copy()
    gates = []
    for k in range(n_gates):
        spacing = rng.uniform(4.0, spread)
        heading += rng.uniform(-np.pi / 6, np.pi / 6) if k else 0.0
        d = np.array([np.cos(heading), np.sin(heading), 0.0])
        pos = pos + d * spacing
        center = pos.copy()
        center[2] = rng.uniform(1.0, 2.5)
        gates.append((center, d.copy(), 0.8, 0.3))
    pts = np.array([g[0] for g in gates] + [spawn])
    lo = pts.min(axis=0) - 5.0
    hi = pts.max(axis=0) + 5.0
    lo[2] = 0.0
    hi[2] = max(hi[2], 4.0)
    return Scene(prims={"ground_z": 0.0}, bounds_lo=lo, bounds_hi=hi, spawn=spawn,
                 goal=gates[-1][0].copy(), gates=gates, seed=seed, style="racing")


def sample_reset(scene: Scene, n_agents, formation, rng, d_min=0.6, r_quad=0.15, clearance=0.3,
                 max_attempts=100):
    """q/world.py:409-448."""
    packed = pack_primitives([scene.prims])
    for _ in range(max_attempts):
        spawns = scene.spawn[None] + formation + rng.normal(scale=0.15, size=(n_agents, 3))
        spawns[:, 2] = np.clip(spawns[:, 2], scene.bounds_lo[2] + 0.3, scene.bounds_hi[2] - 0.3)
        if n_agents > 1:
            dd = np.linalg.norm(spawns[:, None] - spawns[None], axis=-1)
            dd[np.arange(n_agents), np.arange(n_agents)] = np.inf
            if dd.min() < d_min:
                continue
        if sdf_single_scene(spawns, packed).min() <= r_quad + clearance:
            continue
        inside = np.all(spawns > scene.bounds_lo + 0.2, axis=-1) & np.all(spawns < scene.bounds_hi - 0.2, axis=-1)
        if not inside.all():
            continue
        return spawns, scene.goal[None] + formation
    raise OracleGenerationError("could not place agents")


# ---------------------------------------------------------------------------
# the task environment (q/tasks.py)


@dataclass
class Weights:
    """q/tasks.py:37-64."""

    w_p: float = 1.0
    w_v: float = 0.5
    w_a: float = 0.01
    w_s: float = 0.05
    w_t: float = 2.0
    w_o: float = 2.0
    w_f: float = 0.5
    w_g: float = 1.0
    near_radius: float = 1.0
    near_width: float = 0.25
    track_gain: float = 1.2
    v_max: float = 3.0
    sdf_sharpness: float = 0.25
    gate_pass_bonus: float = 5.0
    gate_crash_penalty: float = 5.0
    goal_bonus: float = 10.0


@dataclass
class Config:
    """q/tasks.py:67-106 (TaskConfig), plus optional IMU for config C2."""

    task: str = "position"
    dynamics: str = "pm_continuous"
    n_envs: int = 64
    n_agents: int = 1
    episode_len: int = 128
    dt: float = 0.05
    goal_dist: float = 8.0
    success_radius: float = 0.5
    hover_speed: float = 0.5
    collision_radius: float = 0.15
    d_min: float = 0.6
    d_safe: float = 0.5
    sensor: str = "none"
    sensor_stride: int = 1
    depth_width: int = 16
    depth_height: int = 9
    depth_max_range: float = 10.0
    lidar: tuple = (16, 4, 2 * np.pi, np.deg2rad(30.0), 20.0)  # n_az, n_el, az_ext, el_ext, range
    density: float = 0.1
    style: str = "outdoor"
    n_gates: int = 5
    gate_spread: float = 10.0
    formation: str = "line"
    formation_side: float = 2.0
    yaw_ema_alpha: float = 0.1
    obs_clip: float = 10.0
    weights: Weights = field(default_factory=Weights)
    rl_weights: Weights = field(default_factory=lambda: Weights(w_p=0.2))
    randomization: RandomizationSpec | None = None


def _stable_sigmoid(x):
    """q/autodiff.py:446-456."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ev = np.exp(x[~pos])
    out[~pos] = ev / (1.0 + ev)
    return out


class OracleTask:
    """FlightTask + PositionTask/AvoidanceTask/RacingTask restated (q/tasks.py:198-972).

    State is plain numpy; ``step(raw)`` returns a dict of fp64 arrays.
    ``scene_provider(seed, e)`` may override per-env scene generation (used to
    feed fixture scenes).  ``reset_log`` records every spawn draw (env ids,
    episode counter, p/v/goal/v_ema, DR draws) so GPU tests can inject them.
    """

    def __init__(self, cfg: Config, scene_provider=None, imu=None):
        self.cfg = cfg
        self.model = cfg.dynamics
        self.base = Params(dt=cfg.dt)
        self.n_envs, self.n_agents = cfg.n_envs, cfg.n_agents
        self.N = cfg.n_envs * cfg.n_agents
        self.A = MODEL_ACTION_DIM[self.model]
        self.template = formation_offsets(cfg.formation, cfg.n_agents, cfg.formation_side)
        self.scene_provider = scene_provider
        self.imu_cfg = imu  # dict(accel_noise_std=..., seed=...) or None
        self.reset_log = []

    # -- lifecycle (q/tasks.py:327-391)
    def reset(self, seed):
        self.seed = int(seed)
        self.episode_counter = 0
        self.steps_total = 0
        self.frame_cache = None
        self.finished = self.successes = self.collisions = 0
        self.finished_return = 0.0
        self._build_scenes()
        self._apply_randomization()
        self.state = None
        self._spawn_all(np.ones(self.n_envs, bool))
        self.steps = np.zeros(self.n_envs, np.int64)
        self.ep_return = np.zeros(self.n_envs)
        if self.imu_cfg is not None:
            kw = dict(self.imu_cfg)
            self.imu = Imu(self.N, **kw)
        return {"proprio": self.observe_proprio(), "visual": self.render()}

    def _build_scenes(self):
        cfg = self.cfg
        if cfg.task == "position":  # q/tasks.py:661-674
            ext = cfg.goal_dist
            lo = np.array([-2.0, -ext - 2.0, 0.0])
            hi = np.array([ext + 2.0, ext + 2.0, 4.0])
            self.scene = Scene(prims={"ground_z": 0.0}, bounds_lo=lo, bounds_hi=hi,
                               spawn=np.array([0.0, 0.0, 1.2]), goal=np.array([ext * 0.75, 0.0, 1.5]))
            self.scenes = [self.scene] * self.n_envs
        elif cfg.task == "avoidance":  # q/tasks.py:769-787
            spawn = np.array([0.0, 0.0, 1.2])
            goal = np.array([cfg.goal_dist, 0.0, 1.5])
            self.scenes = []
            for e in range(self.n_envs):
                s = (self.scene_provider(self.seed, e) if self.scene_provider else
                     gen_obstacle_course((self.seed * 100_003 + e) & 0x7FFFFFFF, spawn, goal,
                                         cfg.density, cfg.style, cfg.collision_radius))
                self.scenes.append(s)
        else:  # racing q/tasks.py:850-871
            self.scenes = [self.scene_provider(self.seed, e) if self.scene_provider else
                           gen_race_track((self.seed * 99_991 + e) & 0x7FFFFFFF, cfg.n_gates, cfg.gate_spread)
                           for e in range(self.n_envs)]
            self.gate_c = np.stack([[g[0] for g in s.gates] for s in self.scenes])
            self.gate_n = np.stack([[g[1] for g in s.gates] for s in self.scenes])
            self.gate_in = np.stack([[g[2] for g in s.gates] for s in self.scenes])
            self.gate_fw = np.stack([[g[3] for g in s.gates] for s in self.scenes])
        per_env = pack_primitives([s.prims for s in self.scenes])
        self.prims = {k: np.repeat(v, self.n_agents, axis=0) for k, v in per_env.items()}
        lo = np.stack([s.bounds_lo for s in self.scenes])
        hi = np.stack([s.bounds_hi for s in self.scenes])
        self.bounds_lo = np.repeat(lo + 1e-6, self.n_agents, axis=0)
        self.bounds_hi = np.repeat(hi - 1e-6, self.n_agents, axis=0)

    def _apply_randomization(self):
        """q/tasks.py:352-375."""
        spec = self.cfg.randomization
        lo, hi = action_box(self.model)
        self.params = self.base
        if spec is None:
            self.act_lo = np.broadcast_to(lo, (self.N, self.A)).copy()
            self.act_hi = np.broadcast_to(hi, (self.N, self.A)).copy()
            return
        dr = randomize_params(spec, self.seed, self.episode_counter, self.N)
        self.dr_drag, self.dr_lat, self.dr_scale = dr["drag_coeff"], dr["latency"], dr["action_scale"]
        self._install_randomization()

    def _install_randomization(self):
        lo, hi = action_box(self.model)
        self.params = Params(dt=self.cfg.dt, drag_coeff=self.dr_drag.copy(), latency=self.dr_lat.copy())
        c, h = (lo + hi) / 2, (hi - lo) / 2
        s = self.dr_scale[:, None]
        self.act_lo = c[None] - h[None] * s
        self.act_hi = c[None] + h[None] * s

    def _redraw_randomization(self, env_mask):
        """q/tasks.py:377-387."""
        spec = self.cfg.randomization
        if spec is None or not spec.per_episode:
            return
        rows = np.repeat(env_mask, self.n_agents)
        dr = randomize_params(spec, self.seed, self.episode_counter, self.N)
        self.dr_drag[rows] = dr["drag_coeff"][rows]
        self.dr_lat[rows] = dr["latency"][rows]
        self.dr_scale[rows] = dr["action_scale"][rows]
        self._install_randomization()

    def _spawn_all(self, env_mask):
        """q/tasks.py:687-721 (position), :789-815 (avoidance), :873-902 (racing)."""
        cfg, na = self.cfg, self.n_agents
        if self.state is None:
            self.goals = np.zeros((self.N, 3))
            self.v_ema = np.zeros((self.N, 3))
            self.state = init_state(self.model, np.zeros((self.N, 3)), np.zeros((self.N, 3)))
            self.prev_effort = np.zeros((self.N, self.A))
            if cfg.task == "racing":
                self.next_gate = np.zeros(self.n_envs, np.int64)
        p_new = self.state["p"].copy()
        v_new = self.state["v"].copy()
        ids = np.flatnonzero(env_mask)
        for e in ids:
            rows = slice(e * na, (e + 1) * na)
            if cfg.task == "position":
                rng = np.random.default_rng([self.seed & 0x7FFFFFFF, 0xA0, e, self.episode_counter])
                spawn, goal = self._sample_pair(rng)
                p_new[rows] = spawn[None] + self.template + rng.normal(scale=0.1, size=(na, 3))
                v_new[rows] = rng.normal(scale=0.3, size=(na, 3))
                self.goals[rows] = goal[None] + self.template
                head = goal - spawn
            elif cfg.task == "avoidance":
                sc = self.scenes[e]
                rng = np.random.default_rng([self.seed & 0x7FFFFFFF, 0xA1, e, self.episode_counter])
                spawns, goals = sample_reset(sc, na, self.template, rng, d_min=cfg.d_min,
                                             r_quad=cfg.collision_radius)
                p_new[rows] = spawns
                v_new[rows] = rng.normal(scale=0.2, size=(na, 3))
                self.goals[rows] = goals + rng.normal(scale=0.2, size=3)[None]
                head = sc.goal - sc.spawn
            else:
                sc = self.scenes[e]
                rng = np.random.default_rng([self.seed & 0x7FFFFFFF, 0xA2, e, self.episode_counter])
                p_new[e] = sc.spawn + rng.normal(scale=0.2, size=3)
                v_new[e] = rng.normal(scale=0.2, size=3)
                self.next_gate[e] = 0
                self.goals[e] = self.gate_c[e, 0]
                head = self.gate_c[e, 0] - sc.spawn
            head = np.array(head, dtype=np.float64)
            head[2] = 0.0
            head /= max(np.linalg.norm(head), 1e-9)
            self.v_ema[rows] = head[None]
        rows_mask = np.repeat(env_mask, na)
        self.reset_log.append({
            "env_ids": ids.copy(), "episode_counter": self.episode_counter,
            "p": p_new[rows_mask].copy(), "v": v_new[rows_mask].copy(),
            "goal": self.goals[rows_mask].copy(), "v_ema": self.v_ema[rows_mask].copy(),
        })
        self.episode_counter += 1
        fresh = init_state(self.model, p_new, v_new)
        for k in self.state:
            m = rows_mask.reshape((-1,) + (1,) * (fresh[k].ndim - 1))
            self.state[k] = np.where(m, fresh[k], self.state[k])
        self.prev_effort[rows_mask] = 0.0

    def _sample_pair(self, rng):
        """q/tasks.py:676-685."""
        lo, hi = self.scene.bounds_lo, self.scene.bounds_hi
        for _ in range(100):
            spawn = rng.uniform(lo + 0.8, hi - 0.8)
            goal = rng.uniform(lo + 0.8, hi - 0.8)
            d = np.linalg.norm(goal - spawn)
            if 2.5 <= d <= self.cfg.goal_dist:
                return spawn, goal
        raise OracleGenerationError("could not sample spawn/goal pair")

    # -- frames and observations (q/tasks.py:400-463)
    def attitude(self):
        return attitude(self.model, self.state, self.v_ema, self.params.g_vec)

    def yaw(self):
        return yaw_of(self.attitude())

    def observe_proprio(self):
        """q/tasks.py:415-442 (+ racing extras :904-915)."""
        yaw = self.yaw()
        unrot = rotz(-yaw)
        clip = self.cfg.obs_clip
        st = self.state
        parts = [np.clip(matvec(unrot, self.goals - st["p"]), -clip, clip), matvec(unrot, st["v"])]
        if self.model == "pm_continuous":
            parts.append(matvec(unrot, st["a_lat"]))
        elif self.model == "pm_discrete":
            parts.append(matvec(unrot, st["u_prev"]))
        elif self.model == "simplified":
            parts.append(matvec(unrot, st["R"][..., 2]))
        else:
            parts.append(matvec(unrot, quat_rotate(st["q"], np.array([0.0, 0.0, 1.0]))))
            parts.append(st["w"])
        if self.cfg.task == "racing":
            e = np.arange(self.n_envs)
            idx = self.next_gate
            nxt = np.minimum(idx + 1, self.cfg.n_gates - 1)
            parts.append(np.clip(matvec(unrot, self.gate_c[e, idx] - st["p"]), -clip, clip))
            parts.append(np.einsum("bij,bj->bi", unrot, self.gate_n[e, idx]))
            parts.append(np.clip(matvec(unrot, self.gate_c[e, nxt] - st["p"]), -clip, clip))
        return np.concatenate(parts, axis=-1)

    def render(self, force=False):
        """q/tasks.py:447-463."""
        cfg = self.cfg
        if cfg.sensor == "none":
            return None
        if cfg.sensor_stride > 1 and self.frame_cache is not None and not force:
            if self.steps_total % cfg.sensor_stride != 0:
                return self.frame_cache
        Rc = rotz(self.yaw())
        pos = self.state["p"]
        if cfg.sensor == "depth":
            frame = render_depth(self.prims, pos, Rc, cfg.depth_width, cfg.depth_height, cfg.depth_max_range)
        else:
            n_az, n_el, az_ext, el_ext, rng_max = cfg.lidar
            frame = render_lidar(self.prims, pos, Rc, n_az, n_el, rng_max, az_ext, el_ext)
        self.frame_cache = frame
        return frame

    # -- stepping (q/tasks.py:549-600)
    def step(self, raw, imu_normals=None):
        cfg = self.cfg
        raw = np.asarray(raw, dtype=np.float64)
        assert raw.shape == (self.N, self.A)
        finite = np.isfinite(raw).all(axis=-1)
        if not finite.all():
            raise ValueError(f"non-finite action for env row {int(np.argmin(finite))}")
        squashed = squash(raw, self.act_lo, self.act_hi)
        # the reference tape treats the yaw frame and prev_effort as constants
        # (q/tasks.py:416-418, :569-570); FD gradients replay them frozen
        fz = None
        if getattr(self, "freeze", None) is not None:
            fz = self.freeze[self.freeze_t]
            self.freeze_t += 1
        elif getattr(self, "record", None) is not None:
            self.record.append({"yaw": self.yaw() if self.model.startswith("pm") else None,
                                "prev_effort": self.prev_effort.copy()})
        if self.model.startswith("pm"):
            cmd = matvec(rotz(self.yaw() if fz is None else fz["yaw"]), squashed)
        else:
            cmd = squashed
        prev = self.state
        for k, v in prev.items():
            if not np.all(np.isfinite(v)):
                raise ValueError(f"non-finite state field '{k}'")
        st2 = model_step(self.model, prev, cmd, self.params)
        v_dot = (st2["v"] - prev["v"]) / cfg.dt
        self.v_ema = ema_update(self.v_ema, st2["v"], cfg.yaw_ema_alpha)
        effort = squashed - (self.act_lo + self.act_hi) / 2 * np.ones((self.N, 1))
        d_effort = effort - (self.prev_effort if fz is None else fz["prev_effort"])
        self.prev_effort = effort.copy()
        r_ctrl, r_goal, r_rl, term, aux = self._rewards(prev, st2, effort, d_effort)
        imu_out = None
        if self.imu_cfg is not None:
            if self.model == "full":
                Rb, wb = quat_to_matrix(st2["q"]), st2["w"]
            elif self.model == "simplified":
                Rb, wb = st2["R"], None
            else:
                Rb = reconstruct_attitude(thrust_accel(self.model, st2), self.v_ema)
                wb = None
            imu_out = self.imu.read(Rb, wb, v_dot, self.params.g_vec, cfg.dt, normals=imu_normals)
        self.steps += 1
        self.steps_total += 1
        term_env = term.reshape(self.n_envs, self.n_agents)[:, 0]
        trunc_env = (self.steps >= cfg.episode_len) & (term_env == TERM_NONE)
        truncated = np.repeat(trunc_env, self.n_agents)
        self.ep_return += r_rl.reshape(self.n_envs, self.n_agents)[:, 0]
        done_env = (term_env != TERM_NONE) | trunc_env
        self.state = st2
        self.last_v_dot = v_dot
        state2_pre = {k: v.copy() for k, v in st2.items()}
        if done_env.any():
            self.finished += int(done_env.sum())
            self.successes += int((term_env[done_env] == TERM_SUCCESS).sum())
            self.collisions += int((term_env[done_env] == TERM_COLLISION).sum())
            self.finished_return += float(self.ep_return[done_env].sum())
            self._spawn_all(done_env)
            self._redraw_randomization(done_env)
            self.steps[done_env] = 0
            self.ep_return[done_env] = 0.0
            if self.imu_cfg is not None:
                self.imu.reset(np.repeat(done_env, self.n_agents))
        out = {
            "proprio": self.observe_proprio(), "visual": self.render(),
            "r_ctrl": r_ctrl, "r_goal": r_goal, "r_rl": r_rl, "terminated": term,
            "truncated": truncated, "done": np.repeat(done_env, self.n_agents),
            "state2": state2_pre, "v_dot": v_dot,
        }
        out.update(aux)
        if imu_out is not None:
            out["imu_accel"], out["imu_gyro"] = imu_out
        return out

    # -- rewards (q/tasks.py:144-192, 625-650, 723-763, 817-844, 925-972)
    def _base_reward(self, st2, effort, d_effort):
        w = self.cfg.weights
        off = self.goals - st2["p"]
        dist = np.linalg.norm(off, axis=-1)
        speed = np.linalg.norm(st2["v"], axis=-1)
        near = _stable_sigmoid((w.near_radius - dist) * (1.0 / w.near_width))
        sd = np.minimum(dist * w.track_gain, w.v_max)
        v_des = off * (sd / np.maximum(dist, 1e-9))[:, None]
        track = np.linalg.norm(st2["v"] - v_des, axis=-1)
        r = -(dist * w.w_p + speed * near * w.w_v + np.linalg.norm(effort, axis=-1) * w.w_a
              + np.linalg.norm(d_effort, axis=-1) * w.w_s + track * w.w_t)
        return r, dist, speed

    def _rl_scalar(self, st2, effort, d_effort, r_goal, extra=0.0):
        """q/tasks.py:744-763."""
        w = self.cfg.rl_weights
        off = self.goals - st2["p"]
        dist = np.linalg.norm(off, axis=-1)
        speed = np.linalg.norm(st2["v"], axis=-1)
        near = 1.0 / (1.0 + np.exp(-(w.near_radius - dist) / w.near_width))
        eff = np.linalg.norm(effort, axis=-1)
        deff = np.linalg.norm(d_effort, axis=-1)
        sd = np.minimum(dist * w.track_gain, w.v_max)
        v_des = off * (sd / np.maximum(dist, 1e-9))[:, None]
        track = np.linalg.norm(st2["v"] - v_des, axis=-1)
        dist_c = np.minimum(dist, self.cfg.obs_clip)
        r = -(w.w_p * dist_c + w.w_v * speed * near + w.w_a * eff + w.w_s * deff + w.w_t * track)
        return r + w.goal_bonus * r_goal + extra

    def _formation(self, p):
        """q/tasks.py:173-192."""
        na = self.n_agents
        p3 = p.reshape(self.n_envs, na, 3)
        pen = np.zeros(self.n_envs)
        coll = np.zeros(self.n_envs, bool)
        for i in range(na):
            for j in range(i + 1, na):
                dij = np.linalg.norm(p3[:, i] - p3[:, j], axis=-1)
                ref = float(np.linalg.norm(self.template[i] - self.template[j]))
                pen = pen + (dij - ref) ** 2
                coll |= dij < self.cfg.d_min
        return np.repeat(pen * self.cfg.weights.w_f, na), coll

    def _terminate(self, success, bounds, collision):
        term = np.zeros(self.N, np.int8)
        term[success] = TERM_SUCCESS
        term[bounds] = TERM_BOUNDS
        term[collision] = TERM_COLLISION
        r_goal = np.zeros(self.N)
        r_goal[term == TERM_SUCCESS] = 1.0
        r_goal[(term == TERM_BOUNDS) | (term == TERM_COLLISION)] = -1.0
        return term, r_goal

    def _success_bounds(self, dist, speed, p):
        na, ne = self.n_agents, self.n_envs
        at_goal = (dist < self.cfg.success_radius) & (speed < self.cfg.hover_speed)
        success = np.repeat(at_goal.reshape(ne, na).all(axis=-1), na)
        out = np.any(p < self.bounds_lo, axis=-1) | np.any(p > self.bounds_hi, axis=-1)
        bounds = np.repeat(out.reshape(ne, na).any(axis=-1), na)
        return success, bounds

    def _rewards(self, prev, st2, effort, d_effort):
        cfg = self.cfg
        na, ne = self.n_agents, self.n_envs
        aux = {}
        if cfg.task == "racing":
            return self._racing_rewards(prev, st2, effort)
        r, dist, speed = self._base_reward(st2, effort, d_effort)
        coll_env = np.zeros(ne, bool)
        extra = 0.0
        if cfg.task == "avoidance":
            sd = sdf(st2["p"], self.prims)
            w = cfg.weights
            r = r - w.w_o * np.logaddexp(0.0, (cfg.d_safe - sd) * (1.0 / w.sdf_sharpness))
            coll_env = (sd <= cfg.collision_radius).reshape(ne, na).any(axis=-1)
            wr = cfg.rl_weights
            extra = -(wr.w_o * np.logaddexp(0.0, (cfg.d_safe - sd) / wr.sdf_sharpness))
            aux["sdf"] = sd
        if na > 1:
            pen, inter = self._formation(st2["p"])
            r = r - pen
            coll_env |= inter
        success, bounds = self._success_bounds(dist, speed, st2["p"])
        term, r_goal = self._terminate(success, bounds, np.repeat(coll_env, na))
        r_rl = self._rl_scalar(st2, effort, d_effort, r_goal, extra=extra)
        return r, r_goal, r_rl, term, aux

    def _racing_rewards(self, prev, st2, effort):
        """q/tasks.py:925-972."""
        cfg = self.cfg
        w = cfg.rl_weights
        e = np.arange(self.n_envs)
        idx = self.next_gate
        c = self.gate_c[e, idx]
        n = self.gate_n[e, idx]
        p0, p1 = prev["p"], st2["p"]
        r_rl = w.w_g * (np.linalg.norm(p0 - c, axis=-1) - np.linalg.norm(p1 - c, axis=-1))
        s0 = np.sum((p0 - c) * n, axis=-1)
        s1 = np.sum((p1 - c) * n, axis=-1)
        crossing = (s0 < 0.0) & (s1 >= 0.0)
        term = np.zeros(self.N, np.int8)
        r_goal = np.zeros(self.N)
        if crossing.any():
            frac = -s0 / np.maximum(s1 - s0, 1e-12)
            x = p0 + frac[:, None] * (p1 - p0)
            rv = (x - c) - np.sum((x - c) * n, axis=-1, keepdims=True) * n
            radial = np.linalg.norm(rv, axis=-1)
            inner = self.gate_in[e, idx]
            outer = inner + self.gate_fw[e, idx]
            passed = crossing & (radial < inner)
            crashed = crossing & (radial >= inner) & (radial < outer)
            r_rl[passed] += w.gate_pass_bonus
            r_rl[crashed] -= w.gate_crash_penalty
            term[crashed] = TERM_COLLISION
            r_goal[crashed] = -1.0
            finished = passed & (idx == cfg.n_gates - 1)
            term[finished] = TERM_SUCCESS
            r_goal[finished] = 1.0
            adv = passed & ~finished
            self.next_gate[adv] = idx[adv] + 1
            self.goals[adv] = self.gate_c[e[adv], self.next_gate[adv]]
        out = np.any(p1 < self.bounds_lo, axis=-1) | np.any(p1 > self.bounds_hi, axis=-1)
        newly = out & (term == TERM_NONE)
        term[newly] = TERM_BOUNDS
        r_goal[newly] = -1.0
        r_rl[newly] -= w.goal_bonus
        return np.zeros(self.N), r_goal, r_rl, term, {}

    # -- helpers for tests
    def snapshot(self):
        return copy.deepcopy(self.__dict__)

    def restore(self, snap):
        self.__dict__.update(copy.deepcopy(snap))


def window_loss(env: OracleTask, actions, gamma=0.99):
    """L = -(1/T) sum_t gamma^t mean(r_ctrl_t)  (q/learners.py:214-223, :254)."""
    T = actions.shape[0]
    tot = 0.0
    for t in range(T):
        out = env.step(actions[t])
        tot += gamma ** t * out["r_ctrl"].mean()
    return -tot / T


def fd_grad_actions(env: OracleTask, actions, gamma=0.99, h_scale=1e-6):
    """dL/d(raw actions) by central differences, batched across envs.

    Envs are independent, so perturbing component (t,k) of every
    env at once yields each env's partial derivative from the env-wise loss
    contributions.  Uses h = h_scale*(1+|x|) like pkg/tests/oracles.py:15-30.
    """
    T, N, A = actions.shape
    snap = env.snapshot()
    env.record = []
    for t in range(T):
        env.step(actions[t])
    frozen = env.record
    env.record = None

    def per_env_loss(acts):
        env.restore(snap)
        env.freeze, env.freeze_t = frozen, 0
        tot = np.zeros(N)
        for t in range(T):
            out = env.step(acts[t])
            tot += gamma ** t * out["r_ctrl"] / N
        env.freeze = None
        return -tot / T

    na = env.n_agents
    g = np.zeros_like(actions)
    for t in range(T):
        for k in range(A):
            for a in range(na):  # agents of one env are coupled: perturb one at a time
                rows = np.arange(a, N, na)
                h = h_scale * (1.0 + np.abs(actions[t, rows, k]))
                ap = actions.copy()
                ap[t, rows, k] += h
                am = actions.copy()
                am[t, rows, k] -= h
                lp = per_env_loss(ap).reshape(env.n_envs, na).sum(-1)
                lm = per_env_loss(am).reshape(env.n_envs, na).sum(-1)
                g[t, rows, k] = (lp - lm) / (2.0 * h)
    env.restore(snap)
    return g


# ---------------------------------------------------------------------------
# reverse pass (restates the reference tape's backward for the position task,
# q/autodiff.py:201-237 over the ops recorded by q/tasks.py:549-637).  Used as
# the CPU baseline of the fwd+bwd benchmark and pinned to the golden tape
# gradients in tests/test_oracle_golden.py.


def _qconj(q):
    return np.concatenate([q[:, :1], -q[:, 1:]], axis=-1)


def _qrot_vjp_q(q, v, g):
    u, w = q[:, 1:], q[:, :1]
    v = np.broadcast_to(v, u.shape)
    gw = 2.0 * np.sum(g * np.cross(u, v), axis=-1, keepdims=True)
    gu = (2.0 * w * np.cross(v, g) + 2.0 * np.sum(u * v, -1, keepdims=True) * g
          + 2.0 * np.sum(g * u, -1, keepdims=True) * v - 4.0 * np.sum(g * v, -1, keepdims=True) * u)
    return np.concatenate([gw, gu], axis=-1)


def _norm_vjp(a, n, g):
    safe = np.maximum(n, np.finfo(np.float64).tiny)
    return (g / safe)[:, None] * a


def step_full_vjp(st, act, prm: Params, gs):
    """VJP of step_full (q/dynamics.py:155-186)."""
    p, v, q, w = st["p"], st["v"], st["q"], st["w"]
    c = act[:, 0:1]
    dt = prm.dt
    zero = np.zeros((q.shape[0], 1))
    r = np.concatenate([zero, w], axis=-1)
    qd = quat_mul(q, r) * 0.5
    qn = q + qd * dt
    nn = np.sqrt(np.sum(qn * qn, -1, keepdims=True))
    qo = qn / nn
    gq_ = gs["q"]
    gqn = (gq_ - qo * np.sum(qo * gq_, -1, keepdims=True)) / nn
    gqd = gqn * dt * 0.5
    gq = gqn + quat_mul(gqd, _qconj(r))
    gw_q = quat_mul(_qconj(q), gqd)[:, 1:]
    gwdot = gs["w"] * dt
    K = prm.rate_gains
    g_wc = K * gwdot
    gw = gs["w"] - K * gwdot + gw_q
    gvdot = gs["v"] * dt
    gp = gs["p"].copy()
    gv = gs["v"] + gs["p"] * dt
    zb = quat_rotate(q, np.array([0.0, 0.0, 1.0]))
    g_c = np.sum(gvdot * zb, -1, keepdims=True)
    gq = gq + _qrot_vjp_q(q, np.array([0.0, 0.0, 1.0]), gvdot * c)
    D = prm.drag_matrix_diag
    if np.any(D != 0):
        qc = _qconj(q)
        vb = quat_rotate(qc, v)
        dv = D * vb
        gdrag = -gvdot
        gq = gq + _qrot_vjp_q(q, dv, gdrag)
        gdv = quat_rotate(qc, gdrag)
        gvb = D * gdv
        gv = gv + quat_rotate(q, gvb)
        g2 = _qrot_vjp_q(qc, v, gvb)
        gq = gq + np.concatenate([g2[:, :1], -g2[:, 1:]], -1)
    return {"p": gp, "v": gv, "q": gq, "w": gw}, np.concatenate([g_c, g_wc], -1)


def model_step_vjp(model, st, act, prm: Params, gs):
    if model == "full":
        return step_full_vjp(st, act, prm, gs)
    dt = prm.dt
    B = act.shape[0]
    if model == "pm_continuous":
        decay = _bcast(prm.lag_decay, B)
        d = _bcast(prm.drag_coeff, B)
        ga = gs["a_lat"] + gs["v"] * dt
        return ({"p": gs["p"].copy(), "v": gs["v"] - gs["v"] * (d * dt) + gs["p"] * dt, "a_lat": ga * decay},
                ga - ga * decay)
    gu = gs["p"] * (0.5 * dt * dt) + gs["v"] * (0.5 * dt) + gs["u_prev"]
    return ({"p": gs["p"].copy(), "v": gs["v"] + gs["p"] * dt, "u_prev": gs["v"] * (0.5 * dt)}, gu)


def reward_ctrl_vjp(w: Weights, off, v, eff, deff, g):
    """VJP of reward_position + velocity_field_error (q/tasks.py:144-165, 625-637)."""
    dist = np.linalg.norm(off, axis=-1)
    speed = np.linalg.norm(v, axis=-1)
    x = (w.near_radius - dist) * (1.0 / w.near_width)
    near = _stable_sigmoid(x)
    m = np.maximum(dist, 1e-9)
    sd = np.minimum(dist * w.track_gain, w.v_max)
    k = sd / m
    vdes = off * k[:, None]
    ev = v - vdes
    track = np.linalg.norm(ev, axis=-1)
    gp = -g
    g_dist = gp * w.w_p
    g_speed = gp * w.w_v * near
    g_near = gp * w.w_v * speed
    g_dist = g_dist + g_near * near * (1 - near) * (-1.0 / w.near_width)
    gev = _norm_vjp(ev, track, gp * w.w_t)
    g_v = gev + _norm_vjp(v, speed, g_speed)
    g_vdes = -gev
    g_off = g_vdes * k[:, None]
    g_k = np.sum(g_vdes * off, -1)
    g_sd = g_k / m
    g_m = -g_k * sd / (m * m)
    g_dist = g_dist + np.where(dist * w.track_gain <= w.v_max, g_sd * w.track_gain, 0.0)
    g_dist = g_dist + np.where(dist >= 1e-9, g_m, 0.0)
    g_off = g_off + _norm_vjp(off, dist, g_dist)
    en = np.linalg.norm(eff, axis=-1)
    dn = np.linalg.norm(deff, axis=-1)
    g_eff = _norm_vjp(eff, en, gp * w.w_a) + _norm_vjp(deff, dn, gp * w.w_s)
    return g_off, g_v, g_eff


def window_value_and_grad(env: OracleTask, actions, gamma=0.99, before_step=None):
    """Position-task BPTT window: L and dL/d(raw actions) by the reverse pass.

    Forward runs env.step (resets included); the backward replays the
    recorded checkpoints in reverse with the tape's semantics: yaw frame and
    prev_effort constant, gradient cut at resets (q/tasks.py:712-721).
    ``before_step(env, t)`` (tests) may overwrite the carried state before
    step t is recorded (teacher forcing): the reverse pass then evaluates the
    chain rule along the forced trajectory.
    """
    cfg = env.cfg
    assert cfg.task == "position" and env.n_agents == 1
    T, N, A = actions.shape
    recs = []
    loss = 0.0
    for t in range(T):
        if before_step is not None:
            before_step(env, t)
        st = {k: v.copy() for k, v in env.state.items()}
        yaw = env.yaw() if env.model.startswith("pm") else None
        lo, hi = env.act_lo.copy(), env.act_hi.copy()
        prm = copy.copy(env.params)
        goals, peff = env.goals.copy(), env.prev_effort.copy()
        out = env.step(actions[t])
        loss += gamma ** t * out["r_ctrl"].mean()
        recs.append((st, yaw, lo, hi, prm, goals, peff, out["state2"], out["done"]))
    loss = -loss / T
    g_act = np.zeros_like(actions)
    gS_next = None
    for t in reversed(range(T)):
        st, yaw, lo, hi, prm, goals, peff, st2, done = recs[t]
        raw = actions[t]
        th = np.tanh(raw)
        half = (hi - lo) * 0.5
        center = (lo + hi) * 0.5
        sq = center + half * th
        eff = sq - center
        deff = eff - peff
        cmd = matvec(rotz(yaw), sq) if yaw is not None else sq
        gs2 = {k: np.zeros_like(v) for k, v in st2.items()}
        if gS_next is not None:
            keep = (~done)[:, None]
            for k in gs2:
                gs2[k] = np.where(keep, gS_next[k], 0.0)
        g_r = np.full(N, -(gamma ** t) / (T * N))
        g_off, g_v, g_eff = reward_ctrl_vjp(cfg.weights, goals - st2["p"], st2["v"], eff, deff, g_r)
        gs2["p"] = gs2["p"] - g_off
        gs2["v"] = gs2["v"] + g_v
        gS, g_cmd = model_step_vjp(env.model, st, cmd, prm, gs2)
        g_sq = matvec(np.swapaxes(rotz(yaw), -1, -2), g_cmd) if yaw is not None else g_cmd
        g_sq = g_sq + g_eff
        g_act[t] = g_sq * half * (1.0 - th * th)
        gS_next = gS
    return loss, g_act
