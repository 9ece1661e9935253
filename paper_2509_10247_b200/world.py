"""Scenes, resets and procedural generation (mirrors ``q/world.py``).

``gen_obstacle_courses`` generates a whole batch of feasible obstacle courses
in-kernel (``qs_gen_obstacle_course``: Philox sampling + grid-BFS
feasibility, one CTA per env); ``gen_race_tracks`` does the same for race
tracks (``qs_gen_race_track``, one thread per env).  ``randomize_params`` is
the reference's host draw used by
reference-compatible reset providers; per-episode randomisation inside the
rollout is drawn in-kernel (``qs_task_step_fwd``).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np
import torch

from paper_2509_10247_b200 import _lib as L
from paper_2509_10247_b200.sensors import DeviceScene, PrimitiveSet, pack_primitives  # noqa: F401

SCENE_FORMAT_VERSION = 1
SPHERE_R = (0.3, 1.0)  # q/world.py:21-24
BOX_HALF = (0.2, 1.0)
CYL_R = (0.2, 0.6)
CYL_HH = (0.5, 2.0)
GRID_RES = 0.25


class GenerationError(RuntimeError):
    def __init__(self, message, seed=None):
        super().__init__(f"{message} (seed={seed})")
        self.seed = seed


@dataclass
class Gate:
    center: np.ndarray
    normal: np.ndarray
    inner_radius: float = 0.8
    frame_width: float = 0.3
    order: int = 0

    def to_json(self):
        return {"center": list(map(float, self.center)), "normal": list(map(float, self.normal)),
                "inner_radius": float(self.inner_radius), "frame_width": float(self.frame_width),
                "order": int(self.order)}

    @classmethod
    def from_json(cls, d):
        return cls(center=np.array(d["center"]), normal=np.array(d["normal"]),
                   inner_radius=d["inner_radius"], frame_width=d["frame_width"], order=d["order"])


@dataclass
class Scene:
    """q/world.py:61-111 (Scene JSON v1 included)."""

    prims: PrimitiveSet
    bounds_lo: np.ndarray
    bounds_hi: np.ndarray
    spawn: np.ndarray
    goal: np.ndarray
    gates: list = field(default_factory=list)
    seed: int = 0
    style: str = "outdoor"

    def to_json(self) -> str:
        return json.dumps({
            "version": SCENE_FORMAT_VERSION, "seed": int(self.seed), "style": self.style,
            "bounds_lo": list(map(float, self.bounds_lo)), "bounds_hi": list(map(float, self.bounds_hi)),
            "spawn": list(map(float, self.spawn)), "goal": list(map(float, self.goal)),
            "spheres": self.prims.spheres.tolist(), "boxes": self.prims.boxes.tolist(),
            "cylinders": self.prims.cylinders.tolist(), "ground_z": self.prims.ground_z,
            "gates": [g.to_json() for g in self.gates],
        })

    @classmethod
    def from_json(cls, text: str) -> "Scene":
        d = json.loads(text)
        if d.get("version") != SCENE_FORMAT_VERSION:
            raise GenerationError(f"unsupported scene format version {d.get('version')}")
        prims = PrimitiveSet(spheres=np.array(d["spheres"]).reshape(-1, 4),
                             boxes=np.array(d["boxes"]).reshape(-1, 6),
                             cylinders=np.array(d["cylinders"]).reshape(-1, 5), ground_z=d["ground_z"])
        return cls(prims=prims, bounds_lo=np.array(d["bounds_lo"]), bounds_hi=np.array(d["bounds_hi"]),
                   spawn=np.array(d["spawn"]), goal=np.array(d["goal"]),
                   gates=[Gate.from_json(g) for g in d["gates"]], seed=d["seed"], style=d["style"])


@dataclass
class RandomizationSpec:
    """q/world.py:114-127."""

    drag_coeff: tuple = (0.1, 0.5)
    latency: tuple = (2.0, 8.0)
    action_scale: tuple = (1.0, 1.0)
    per_episode: bool = True

    def __post_init__(self):
        for name in ("drag_coeff", "latency", "action_scale"):
            lo, hi = getattr(self, name)
            if not (0 <= lo <= hi):
                raise GenerationError(f"invalid randomization range for {name}")


def randomize_params(spec: RandomizationSpec, seed: int, episode: int, n: int = 1):
    """Reference-compatible host draw (q/world.py:130-137), used by reset providers."""
    rng = np.random.default_rng([seed & 0x7FFFFFFF, episode])
    return {"drag_coeff": rng.uniform(*spec.drag_coeff, size=n),
            "latency": rng.uniform(*spec.latency, size=n),
            "action_scale": rng.uniform(*spec.action_scale, size=n)}


def formation_offsets(kind: str, n_agents: int, side: float = 2.0) -> np.ndarray:
    """Formation templates (q/world.py:386-406)."""
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
    raise GenerationError(f"unknown formation '{kind}'")


def course_counts(spawn, goal, density, corridor_halfwidth=3.0):
    dist = float(np.linalg.norm(np.asarray(goal, float) - np.asarray(spawn, float)))
    n_total = int(round(density * dist * 2 * corridor_halfwidth))
    n_cyl = int(round(0.4 * n_total))
    n_sph = int(round(0.3 * n_total))
    return n_sph, n_total - n_cyl - n_sph, n_cyl


def gen_obstacle_courses(seed: int, n_envs: int, spawn, goal, density: float, style: str = "outdoor",
                         r_quad: float = 0.15, clearance: float = 0.5, corridor_halfwidth: float = 3.0,
                         max_attempts: int = 100, device=None, env_offset: int = 0,
                         check: bool = True, out: DeviceScene | None = None, env_mask=None, episode=None,
                         episode_stride: int = 1, err=None) -> DeviceScene:
    """Batch of feasible obstacle courses generated on the GPU (q/world.py:207-340).

    With ``out``/``env_mask``/``episode`` (device tensors) it regenerates, in
    place and without a host sync, only the masked envs' courses keyed by their
    episode index: obstacle re-randomisation on reset."""
    dev = L.require_cuda(device if out is None else out.device)
    spawn = np.asarray(spawn, dtype=np.float64)
    goal = np.asarray(goal, dtype=np.float64)
    if np.linalg.norm(goal - spawn) <= 2.0:
        raise GenerationError("spawn and goal must be more than 2 m apart", seed)
    if density < 0:
        raise GenerationError("density must be >= 0", seed)
    ns, nb, nc = course_counts(spawn, goal, density, corridor_halfwidth)
    nb_tot = nb + (5 if style == "indoor" else 0)
    sc = out if out is not None else DeviceScene(n_envs, dev, max(ns, 1), max(nb_tot, 1), max(nc, 1))
    sc.ext_cull = style == "indoor"  # the 5-box shell spans the whole course
    cfg = L.QsGenCfg()
    cfg.env_mask, cfg.episode, cfg.episode_stride = L.ptr(env_mask), L.ptr(episode), int(episode_stride)
    for i in range(3):
        cfg.spawn[i], cfg.goal[i] = float(spawn[i]), float(goal[i])
    cfg.density, cfg.r_quad, cfg.clearance = float(density), float(r_quad), float(clearance)
    cfg.corridor_halfwidth = float(corridor_halfwidth)
    cfg.indoor = 1 if style == "indoor" else 0
    cfg.max_attempts = int(max_attempts)
    cfg.Sm, cfg.Bm, cfg.Cm = sc.spheres.shape[1], sc.boxes.shape[1], sc.cylinders.shape[1]
    cfg.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    cfg.env_offset = int(env_offset)
    if err is None:
        err = torch.tensor([0, 2**31 - 1], dtype=torch.int32, device=dev)
    L.check(L.lib().qs_gen_obstacle_course(
        cfg, n_envs, L.ptr(sc.bounds), L.ptr(sc.spawn_goal), L.ptr(sc.spheres), L.ptr(sc.boxes),
        L.ptr(sc.cylinders), L.ptr(sc.counts), L.ptr(sc.ground_z), L.ptr(err),
        L.stream_handle(dev)), "qs_gen_obstacle_course")
    if check:
        e = err.tolist()
        if e[0] == L.QS_ERR_GENERATION:
            raise GenerationError(f"no feasible scene after {max_attempts} attempts (env {e[1]})", seed)
    return sc


def gen_obstacle_course(seed: int, spawn, goal, density: float, style: str = "outdoor",
                        r_quad: float = 0.15, clearance: float = 0.5, corridor_halfwidth: float = 3.0,
                        max_attempts: int = 100, device=None) -> Scene:
    """Single-scene convenience wrapper returning a host ``Scene``."""
    sc = gen_obstacle_courses(seed, 1, spawn, goal, density, style, r_quad, clearance,
                              corridor_halfwidth, max_attempts, device)
    return device_scene_to_scenes(sc, style=style, seed=seed)[0]


def device_scene_to_scenes(sc: DeviceScene, style="outdoor", seed=0) -> list:
    cnt = sc.counts.cpu().numpy()
    sph = sc.spheres.double().cpu().numpy()
    box = sc.boxes.double().cpu().numpy()
    cyl = sc.cylinders.double().cpu().numpy()
    bd = sc.bounds.double().cpu().numpy()
    sg = sc.spawn_goal.double().cpu().numpy()
    gz = sc.ground_z.double().cpu().numpy()
    gt = sc.gates.double().cpu().numpy() if style == "racing" else None
    out = []
    for e in range(sc.n_envs):
        ns, nb, nc, hg = cnt[e]
        prims = PrimitiveSet(spheres=sph[e, :ns], boxes=np.concatenate([box[e, :nb, 0:3], box[e, :nb, 4:7]], -1),
                             cylinders=cyl[e, :nc, 0:5], ground_z=float(gz[e]) if hg else None)
        gates = [] if gt is None else [Gate(center=g[0:3], normal=g[4:7], inner_radius=float(g[3]),
                                            frame_width=float(g[7]), order=k) for k, g in enumerate(gt[e])]
        out.append(Scene(prims=prims, bounds_lo=bd[e, 0, :3], bounds_hi=bd[e, 1, :3], spawn=sg[e, 0, :3],
                         goal=sg[e, 1, :3], gates=gates, seed=seed, style=style))
    return out


def gen_race_tracks(seed: int, n_envs: int, n_gates: int, spread: float = 10.0, device=None, env_offset: int = 0,
                    out: DeviceScene | None = None, env_mask=None, episode=None,
                    episode_stride: int = 1) -> DeviceScene:
    """Batch of race tracks generated on the GPU (q/world.py:347-379), one
    thread per env, Philox keyed by (seed, global env id, episode): gates
    chained along an open loop (spacing U(4, spread), heading turns
    U(-pi/6, pi/6) after the first gate, heights U(1, 2.5)), goal at the last
    gate, bounds the track's extent +-5 m with floor 0 and ceiling >= 4.

    The reference draws each env's track with its own PCG64 stream on the host
    (seeded ``(seed*99991 + e) & 0x7FFFFFFF``); those exact tracks can be
    injected through ``FlightTask(scene_source=...)``.  With ``out`` /
    ``env_mask`` / ``episode`` only the masked envs are regenerated, in place
    and without a host sync (re-randomisation on reset)."""
    if n_gates < 1:
        raise GenerationError("need at least one gate", seed)
    if n_gates > L.MAX_GATES:
        raise GenerationError(f"n_gates must be <= {L.MAX_GATES}", seed)
    if spread < 4.0:
        raise GenerationError("spread must be >= 4 m", seed)
    dev = L.require_cuda(device if out is None else out.device)
    sc = out if out is not None else DeviceScene(n_envs, dev, n_gates=n_gates)
    if sc.gates.shape[1] != n_gates:
        raise GenerationError("scene gate table does not match n_gates", seed)
    cfg = L.QsTrackCfg()
    cfg.n_gates, cfg.spread = int(n_gates), float(spread)
    cfg.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    cfg.env_offset = int(env_offset)
    cfg.env_mask, cfg.episode, cfg.episode_stride = L.ptr(env_mask), L.ptr(episode), int(episode_stride)
    L.check(L.lib().qs_gen_race_track(cfg, n_envs, L.ptr(sc.bounds), L.ptr(sc.spawn_goal), L.ptr(sc.gates),
                                      L.ptr(sc.counts), L.ptr(sc.ground_z), L.stream_handle(dev)),
            "qs_gen_race_track")
    return sc


def gen_race_track(seed: int, n_gates: int, spread: float = 10.0, device=None) -> Scene:
    """Single-track convenience wrapper (q/world.py:347 name) returning a host
    ``Scene`` with its gates, generated by the device kernel."""
    sc = gen_race_tracks(seed, 1, n_gates, spread, device)
    return device_scene_to_scenes(sc, style="racing", seed=seed)[0]


def scenes_to_device(scenes: list, device, n_gates: int = 0) -> DeviceScene:
    """Upload host ``Scene`` objects (obstacles, bounds, spawn/goal, gates)."""
    from paper_2509_10247_b200.sensors import pack_primitives

    sc = DeviceScene.from_batched(pack_primitives([s.prims for s in scenes]), device, n_gates=n_gates)
    sc.ext_cull = any(len(s.prims.boxes) and float(np.hypot(s.prims.boxes[:, 3], s.prims.boxes[:, 4]).max()) > 2.0
                      for s in scenes)
    E = len(scenes)
    bd = np.zeros((E, 2, 4))
    sg = np.zeros((E, 2, 4))
    for e, s in enumerate(scenes):
        bd[e, 0, :3], bd[e, 1, :3] = s.bounds_lo, s.bounds_hi
        sg[e, 0, :3], sg[e, 1, :3] = s.spawn, s.goal
    sc.bounds.copy_(torch.as_tensor(bd, dtype=torch.float32))
    sc.spawn_goal.copy_(torch.as_tensor(sg, dtype=torch.float32))
    if n_gates:
        gt = np.zeros((E, n_gates, 8))
        for e, s in enumerate(scenes):
            for k, g in enumerate(s.gates[:n_gates]):
                gt[e, k, 0:3], gt[e, k, 3] = g.center, g.inner_radius
                gt[e, k, 4:7], gt[e, k, 7] = g.normal, g.frame_width
        sc.gates.copy_(torch.as_tensor(gt, dtype=torch.float32))
    return sc


def sdf_np_all(points, prims):
    """q/world.py:182-196: signed distance of many points to ONE packed scene
    (every point is a row of that scene's single env)."""
    from paper_2509_10247_b200 import sensors as sn

    pts = np.atleast_2d(np.asarray(points, dtype=np.float64)) if not isinstance(points, torch.Tensor) else points
    n = pts.shape[0]
    if getattr(prims, "batch", 1) != 1:
        raise GenerationError("sdf_np_all expects a single-scene pack")
    return sn.sdf_np(pts, prims, n_agents=n)


def scene_sdf(scene: "Scene", points):
    """q/world.py:199-200."""
    return sdf_np_all(points, pack_primitives([scene.prims]))
