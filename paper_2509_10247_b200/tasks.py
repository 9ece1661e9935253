"""The flight tasks behind one batched, dual-reward stepping interface.

Mirrors ``q/tasks.py`` (TaskConfig, make_task, FlightTask.reset/step/observe/
detach_states, StepOutput, the TERM_* codes and contract errors) on torch CUDA
tensors.  ``FlightTask.step`` is ONE fused sm_100a kernel per env
(``qs_task_step_fwd``: squash -> yaw frame -> dynamics -> EMA -> rewards ->
termination -> auto-reset -> observation [-> IMU]) behind the torch custom op
``quadsim::task_step`` (``csrc/qs_torch_ops.cpp``), whose C++ autograd node
runs the analytic VJP kernel (``qs_task_step_bwd``) as its backward.  It saves
only the step's checkpoint (state, raw action, goal, previous effort, per-row
params, a 4-byte flag record).

Batch layout is env-major: row = env * n_agents + agent.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from paper_2509_10247_b200 import _lib as L
from paper_2509_10247_b200 import dynamics as dyn
from paper_2509_10247_b200 import sensors as sn
from paper_2509_10247_b200 import world as wd

TERM_NONE = 0
TERM_SUCCESS = 1
TERM_COLLISION = 2
TERM_BOUNDS = 3

TASK_NAMES = ("position", "avoidance", "racing")
_INT_MAX = 2**31 - 1


class TaskContractError(ValueError):
    pass


@dataclass
class RewardWeights:
    """q/tasks.py:37-54."""

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


def default_rl_weights() -> RewardWeights:
    """q/tasks.py:57-64."""
    return RewardWeights(w_p=0.2)


@dataclass
class ImuSpec:
    """IMU attached to every row (q/sensors.py:508-530 parameters)."""

    accel_noise_std: float = 0.0
    gyro_noise_std: float = 0.0
    accel_bias_rw_std: float = 0.0
    gyro_bias_rw_std: float = 0.0


@dataclass
class TaskConfig:
    """q/tasks.py:67-106, plus two opt-in extensions: ``imu`` (config C2) and
    ``differentiable_depth`` (analytic depth VJP; off keeps reference gradients)."""

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
    lidar: sn.LidarPattern | None = None
    density: float = 0.1
    style: str = "outdoor"
    n_gates: int = 5
    gate_spread: float = 10.0
    formation: str = "line"
    formation_side: float = 2.0
    yaw_ema_alpha: float = 0.1
    obs_clip: float = 10.0
    weights: RewardWeights = field(default_factory=RewardWeights)
    rl_weights: RewardWeights = field(default_factory=default_rl_weights)
    randomization: wd.RandomizationSpec | None = None
    regen_scene_on_reset: bool = False
    imu: ImuSpec | None = None
    differentiable_depth: bool = False

    def __post_init__(self):
        if self.task not in TASK_NAMES:
            raise TaskContractError(f"unknown task '{self.task}'")
        if self.n_envs < 1 or self.n_agents < 1 or self.episode_len < 1:
            raise TaskContractError("n_envs, n_agents, episode_len must be >= 1")
        if min(self.success_radius, self.collision_radius, self.dt) <= 0:
            raise TaskContractError("radii and dt must be positive")
        if self.n_agents > L.MAX_AGENTS:
            raise TaskContractError(f"n_agents must be <= {L.MAX_AGENTS}")


@dataclass
class Obs:
    proprio: torch.Tensor  # (N, P), autograd-connected
    visual: torch.Tensor | None = None  # (N, H, W) or (N, R)
    imu: tuple | None = None  # (accel (N,3), gyro (N,3)) when config.imu is set


@dataclass
class StepOutput:
    obs: Obs
    r_ctrl: torch.Tensor  # (N,) differentiable
    r_goal: torch.Tensor  # (N,) in {+1, -1, 0}
    r_rl: torch.Tensor  # (N,)
    terminated: torch.Tensor  # (N,) int8 TERM_*
    truncated: torch.Tensor  # (N,) bool

    @property
    def done(self) -> torch.Tensor:
        return (self.terminated != TERM_NONE) | self.truncated


def rotz_np(yaw: np.ndarray) -> np.ndarray:
    """q/tasks.py:129-137."""
    c, s = np.cos(yaw), np.sin(yaw)
    R = np.zeros(np.shape(yaw) + (3, 3))
    R[..., 0, 0], R[..., 0, 1], R[..., 1, 0], R[..., 1, 1], R[..., 2, 2] = c, -s, s, c, 1.0
    return R


def rotz(yaw: torch.Tensor) -> torch.Tensor:
    c, s = torch.cos(yaw), torch.sin(yaw)
    z, o = torch.zeros_like(c), torch.ones_like(c)
    return torch.stack([c, -s, z, s, c, z, z, z, o], -1).reshape(yaw.shape + (3, 3))


# ---------------------------------------------------------------------------
# module-level reward primitives (q/tasks.py:144-192), torch versions for API
# parity; the env step itself evaluates them inside the fused kernel.


def reward_position(dist, speed_gated, effort, d_effort, track_err, w: RewardWeights):
    pen = dist * w.w_p
    pen = pen + speed_gated * w.w_v
    pen = pen + effort * w.w_a
    pen = pen + d_effort * w.w_s
    pen = pen + track_err * w.w_t
    return -pen


def velocity_field_error(offset, v, w: RewardWeights):
    n = torch.linalg.norm(offset, dim=-1)
    speed_des = torch.clamp(n * w.track_gain, max=w.v_max)
    v_des = offset * (speed_des / torch.clamp(n, min=1e-9))[..., None]
    return torch.linalg.norm(v - v_des, dim=-1)


def obstacle_penalty(sdf, w: RewardWeights, d_safe: float):
    return torch.nn.functional.softplus((d_safe - sdf) / w.sdf_sharpness) * w.w_o


def formation_terms(p, template, d_min: float, w_f: float):
    n_agents = template.shape[0]
    if n_agents < 2:
        raise TaskContractError("formation terms need n_agents >= 2")
    pen = None
    coll = torch.zeros(p.shape[0], dtype=torch.bool, device=p.device)
    for i in range(n_agents):
        for j in range(i + 1, n_agents):
            dij = torch.linalg.norm(p[:, i] - p[:, j], dim=-1)
            ref = float(np.linalg.norm(template[i] - template[j]))
            t = (dij - ref) ** 2
            pen = t if pen is None else pen + t
            coll |= dij < d_min
    return pen * w_f, coll


# ---------------------------------------------------------------------------


def _fill_weights(dst: L.QsWeights, w: RewardWeights):
    for name, _ in L.QsWeights._fields_:
        setattr(dst, name, float(getattr(w, name)))


class FlightTask:
    """Batched environment (q/tasks.py:198-655) on one CUDA device.

    Extra keyword arguments (all optional):
      device        -- CUDA device (default: current)
      strict        -- validate actions/state synchronously and raise the
                       reference's contract errors before stepping (True);
                       False leaves validation to the kernel's device error
                       word (``check_errors()``) so steps never sync
      env_offset    -- global id of local env 0 (sharded multi-GPU runs)
      reset_source  -- reference-compatible injection: callable
                       (env_ids, episode_counter, initial) -> dict of spawn
                       draws; resets are then applied from host tables
                       (one host sync per step) instead of in-kernel Philox
      scene_source  -- callable(seed, n_envs) -> list of world.Scene (or a
                       DeviceScene) overriding in-kernel scene generation
    """

    def __init__(self, config: TaskConfig, params: dyn.QuadParams | None = None, device=None,
                 strict: bool = True, env_offset: int = 0, reset_source=None, scene_source=None):
        self.config = config
        self.device = L.require_cuda(device)
        base = params or dyn.QuadParams(dt=config.dt)
        if base.dt != config.dt:
            from dataclasses import replace

            base = replace(base, dt=config.dt)
        self.base_params = base
        self.model = dyn.make_model(config.dynamics, base, device=self.device)
        self.n_envs = config.n_envs
        self.n_agents = config.n_agents
        self.N = config.n_envs * config.n_agents
        self.action_dim = self.model.action_dim
        self.strict = strict
        self.env_offset = int(env_offset)
        self.reset_source = reset_source
        self.scene_source = scene_source
        self._template = wd.formation_offsets(config.formation, config.n_agents, config.formation_side)
        self.camera = sn.CameraIntrinsics(width=config.depth_width, height=config.depth_height,
                                          max_range=config.depth_max_range) if config.sensor == "depth" else None
        self.lidar = (config.lidar or sn.LidarPattern()) if config.sensor == "lidar" else None
        self.imu_noise_source = None  # test hook: callable(step_index) -> (4,N,3)
        self._episode_counter = 0
        self._regen = False
        self._S = None

    # -- spec of the policy-visible observation (q/tasks.py:225-297)

    def obs_spec(self) -> dict:
        fields = [{"name": "goal_offset", "size": 3, "frame": "yaw-local", "units": "m"},
                  {"name": "velocity", "size": 3, "frame": "yaw-local", "units": "m/s"}]
        fields += self._extra_proprio_spec()
        visual = None
        if self.camera is not None:
            visual = {"kind": "depth", "height": self.camera.height, "width": self.camera.width,
                      "max_range": self.camera.max_range, "units": "m"}
        elif self.lidar is not None:
            visual = {"kind": "lidar", "rays": self.lidar.n_rays, "max_range": self.lidar.max_range,
                      "units": "m"}
        return {"task": self.config.task, "dynamics": self.config.dynamics, "action_dim": self.action_dim,
                "proprio": fields, "proprio_dim": sum(f["size"] for f in fields), "visual": visual}

    def _extra_proprio_spec(self):
        name = self.config.dynamics
        if name == "pm_continuous":
            out = [{"name": "latent_accel", "size": 3, "frame": "yaw-local", "units": "m/s^2"}]
        elif name == "pm_discrete":
            out = [{"name": "prev_accel_cmd", "size": 3, "frame": "yaw-local", "units": "m/s^2"}]
        elif name == "simplified":
            out = [{"name": "body_z_axis", "size": 3, "frame": "yaw-local", "units": "1"}]
        else:
            out = [{"name": "body_z_axis", "size": 3, "frame": "yaw-local", "units": "1"},
                   {"name": "body_rates", "size": 3, "frame": "body", "units": "rad/s"}]
        if self.config.task == "racing":
            out += [{"name": "next_gate_offset", "size": 3, "frame": "yaw-local", "units": "m"},
                    {"name": "next_gate_normal", "size": 3, "frame": "yaw-local", "units": "1"},
                    {"name": "second_gate_offset", "size": 3, "frame": "yaw-local", "units": "m"}]
        return out

    @property
    def proprio_dim(self) -> int:
        return L.lib().qs_proprio_dim(L.MODEL_IDS[self.config.dynamics], L.TASK_IDS[self.config.task])

    _FIELD_SCALE = {"goal_offset": 0.2, "velocity": 1.0 / 3.0, "latent_accel": 0.1, "prev_accel_cmd": 0.1,
                    "body_z_axis": 1.0, "body_rates": 1.0 / 3.0, "next_gate_offset": 0.2,
                    "next_gate_normal": 1.0, "second_gate_offset": 0.2}

    def proprio_scale(self) -> tuple:
        out = []
        for f in self.obs_spec()["proprio"]:
            out += [self._FIELD_SCALE[f["name"]]] * f["size"]
        return tuple(out)

    # -- statistics (q/tasks.py:301-323); read lazily from the device

    def reset_stats(self):
        if getattr(self, "_stats", None) is not None:
            self._stats.zero_()

    def _stat(self, i):
        return float(self._stats[i].item()) if getattr(self, "_stats", None) is not None else 0.0

    @property
    def finished_episodes(self) -> int:
        return int(self._stat(0))

    @property
    def successful_episodes(self) -> int:
        return int(self._stat(1))

    @property
    def collision_episodes(self) -> int:
        return int(self._stat(2))

    @property
    def finished_return(self) -> float:
        return self._stat(3)

    @property
    def success_rate(self) -> float:
        f = self.finished_episodes
        return self.successful_episodes / f if f else 0.0

    @property
    def collision_rate(self) -> float:
        f = self.finished_episodes
        return self.collision_episodes / f if f else 0.0

    @property
    def mean_episode_return(self) -> float:
        f = self.finished_episodes
        return self.finished_return / f if f else 0.0

    # -- configuration struct

    def _build_cfg(self) -> L.QsTaskCfg:
        c = self.config
        cfg = L.QsTaskCfg()
        lo, hi = self.model.action_box()
        dyn.fill_dyn_cfg(cfg, c.dynamics, self.base_params, (lo, hi))
        cfg.task = L.TASK_IDS[c.task]
        cfg.n_envs, cfg.n_agents = self.n_envs, self.n_agents
        cfg.episode_len, cfg.action_dim = c.episode_len, self.action_dim
        cfg.proprio_dim = self.proprio_dim
        cfg.n_gates = c.n_gates if c.task == "racing" else 0
        cfg.env_offset = self.env_offset
        cfg.seed = (int(getattr(self, "seed", 0)) * 0x9E3779B97F4A7C15 + 0x1234567) & 0xFFFFFFFFFFFFFFFF
        cfg.success_radius, cfg.hover_speed = c.success_radius, c.hover_speed
        cfg.collision_radius, cfg.d_min, cfg.d_safe = c.collision_radius, c.d_min, c.d_safe
        cfg.yaw_ema_alpha, cfg.obs_clip, cfg.goal_dist = c.yaw_ema_alpha, c.obs_clip, c.goal_dist
        for a in range(self.n_agents):
            for k in range(3):
                cfg.formation[a][k] = float(self._template[a, k])
            for b in range(self.n_agents):
                cfg.form_ref[a][b] = float(np.linalg.norm(self._template[a] - self._template[b]))
        _fill_weights(cfg.w, c.weights)
        _fill_weights(cfg.w_rl, c.rl_weights)
        spec = c.randomization
        cfg.dr_enabled = 1 if spec is not None else 0
        if spec is not None:
            cfg.dr_per_episode = 1 if spec.per_episode else 0
            for i in range(2):
                cfg.dr_drag[i], cfg.dr_latency[i] = spec.drag_coeff[i], spec.latency[i]
                cfg.dr_scale[i] = spec.action_scale[i]
        if c.imu is not None:
            cfg.imu_enabled = 1
            cfg.imu_accel_std, cfg.imu_gyro_std = c.imu.accel_noise_std, c.imu.gyro_noise_std
            cfg.imu_accel_rw, cfg.imu_gyro_rw = c.imu.accel_bias_rw_std, c.imu.gyro_bias_rw_std
        # deferred resets: host-injected draws, or a scene regeneration that must
        # precede the spawn draw (spawn/goal come from the regenerated course)
        cfg.reset_mode = 1 if (self.reset_source is not None or self._regen) else 0
        cfg.want_cam = 1 if c.sensor != "none" else 0
        return cfg

    # -- scenes (q/tasks.py:661-674, 769-787, 850-871)

    def _build_scenes(self):
        c = self.config
        dev = self.device
        E = self.n_envs
        if self.scene_source is not None and c.task != "position":
            src = self.scene_source(self.seed, E)
            if isinstance(src, sn.DeviceScene):
                self._scene = src
                self.scenes = None
            else:
                self.scenes = list(src)
                self._scene = wd.scenes_to_device(self.scenes, dev, n_gates=c.n_gates if c.task == "racing" else 0)
        elif c.task == "position":
            ext = c.goal_dist
            lo = np.array([-2.0, -ext - 2.0, 0.0])
            hi = np.array([ext + 2.0, ext + 2.0, 4.0])
            self.scene = wd.Scene(prims=sn.PrimitiveSet(ground_z=0.0), bounds_lo=lo, bounds_hi=hi,
                                  spawn=np.array([0.0, 0.0, 1.2]), goal=np.array([ext * 0.75, 0.0, 1.5]),
                                  seed=self.seed)
            sc = sn.DeviceScene(E, dev)
            sc.counts[:, 3] = 1
            sc.bounds[:, 0, :3] = torch.as_tensor(lo, dtype=torch.float32)
            sc.bounds[:, 1, :3] = torch.as_tensor(hi, dtype=torch.float32)
            sc.spawn_goal[:, 0, :3] = torch.as_tensor(self.scene.spawn, dtype=torch.float32)
            sc.spawn_goal[:, 1, :3] = torch.as_tensor(self.scene.goal, dtype=torch.float32)
            self._scene = sc
            self.scenes = None
        elif c.task == "avoidance":
            self._gen_args = dict(spawn=[0.0, 0.0, 1.2], goal=[c.goal_dist, 0.0, 1.5], density=c.density,
                                  style=c.style, r_quad=c.collision_radius, env_offset=self.env_offset)
            self._scene = wd.gen_obstacle_courses(self.seed, E, device=dev, check=self.strict, **self._gen_args)
            self.scenes = None
        else:  # racing: device-generated tracks (q/world.py:347-379; reference tracks via scene_source)
            if c.n_gates > L.MAX_GATES:
                raise TaskContractError(f"n_gates must be <= {L.MAX_GATES}")
            self._track_args = dict(n_gates=c.n_gates, spread=c.gate_spread, env_offset=self.env_offset)
            self._scene = wd.gen_race_tracks(self.seed, E, device=dev, **self._track_args)
            self.scenes = None
        if c.task == "racing" and self.n_agents != 1:
            raise TaskContractError("racing is single-agent")
        if c.task == "racing" and c.n_gates > L.MAX_GATES:
            raise TaskContractError(f"n_gates must be <= {L.MAX_GATES}")

    # -- lifecycle

    def _alloc_persistent(self):
        dev, N, E = self.device, self.N, self.n_envs
        f = dict(device=dev, dtype=torch.float32)
        self._meta = torch.zeros(E, 4, dtype=torch.int32, device=dev)
        self._ep_ret = torch.zeros(E, **f)
        self._stats = torch.zeros(4, dtype=torch.float64, device=dev)
        # {code, first row} of kernel-reported errors; [2]: qs_task_validate's
        # code << 27 | row key (strict steps)
        self._err = torch.tensor([0, _INT_MAX, _INT_MAX], dtype=torch.int32, device=dev)
        self._empty = torch.empty(0, dtype=torch.float32, device=dev)
        self._imu_bias = torch.zeros(N, 8, **f) if self.config.imu is not None else None

    def _new_io(self):
        io = L.QsStepIo()
        io.meta, io.ep_return = L.ptr(self._meta), L.ptr(self._ep_ret)
        io.imu_bias = L.ptr(self._imu_bias)
        io.stats, io.err = L.ptr(self._stats), L.ptr(self._err)
        return io

    def reset(self, seed: int) -> StepOutput:
        self.seed = int(seed)
        self._episode_counter = 0
        self._steps_total = 0
        self._frame_cache = None
        c = self.config
        if c.regen_scene_on_reset and (c.task == "position" or self.scene_source is not None):
            raise TaskContractError("regen_scene_on_reset needs the avoidance or racing task with generated "
                                    "scenes (no scene_source)")
        self._regen = bool(c.regen_scene_on_reset)
        self._build_scenes()
        self._alloc_persistent()
        self._cfg = self._build_cfg()
        self._cfg_blob = torch.frombuffer(bytearray(bytes(self._cfg)), dtype=torch.uint8)  # quadsim::task_step
        self._ops = L.fast_ops()
        dev, N = self.device, self.N
        NP = L.lib().qs_state_planes(L.MODEL_IDS[self.config.dynamics])
        f = dict(device=dev, dtype=torch.float32)
        S = torch.zeros(NP, N, 4, **f)
        goal = torch.zeros(N, 4, **f)
        peff = torch.zeros(N, 4, **f)
        dr = torch.zeros(N, 4, **f) if self.config.randomization is not None else None
        io = self._new_io()
        io.S_out, io.goal_out, io.peff_out, io.dr_out = L.ptr(S), L.ptr(goal), L.ptr(peff), L.ptr(dr)
        if self.reset_source is not None:
            tab, keep = self._reset_table(np.arange(self.n_envs), initial=True)
            L.check(L.lib().qs_task_spawn(self._cfg, self._scene.struct(), io, None, tab,
                                          L.stream_handle(dev)), "qs_task_spawn")
            del keep
        else:
            L.check(L.lib().qs_task_spawn(self._cfg, self._scene.struct(), io, None, None,
                                          L.stream_handle(dev)), "qs_task_spawn")
        self._episode_counter += 1
        self._S, self._goal, self._peff, self._dr = S, goal, peff, dr
        self._raise_errors()
        obs = self.observe()
        zero = torch.zeros(N, **f)
        return StepOutput(obs=obs, r_ctrl=zero, r_goal=zero.clone(), r_rl=zero.clone(),
                          terminated=torch.zeros(N, dtype=torch.int8, device=dev),
                          truncated=torch.zeros(N, dtype=torch.bool, device=dev))

    def _reset_table(self, env_ids, initial=False):
        """Host-injected spawn draws (reference-compatible resets)."""
        d = self.reset_source(np.asarray(env_ids), self._episode_counter, initial)
        na, N, dev = self.n_agents, self.N, self.device
        rows = (np.asarray(env_ids)[:, None] * na + np.arange(na)[None]).reshape(-1)
        mask = np.zeros(self.n_envs, np.uint8)
        mask[np.asarray(env_ids)] = 1

        def full(key, width=4):
            a = np.zeros((N, width))
            v = np.asarray(d[key], dtype=np.float64).reshape(len(rows), -1)
            a[rows, :v.shape[1]] = v
            return torch.as_tensor(a, dtype=torch.float32, device=dev)

        keep = {"mask": torch.as_tensor(mask, device=dev), "p": full("p"), "v": full("v"),
                "goal": full("goal"), "v_ema": full("v_ema")}
        tab = L.QsResetTable()
        tab.env_mask, tab.p, tab.v = L.ptr(keep["mask"]), L.ptr(keep["p"]), L.ptr(keep["v"])
        tab.goal, tab.v_ema = L.ptr(keep["goal"]), L.ptr(keep["v_ema"])
        if "dr" in d and self.config.randomization is not None:
            dr = np.zeros((N, 4))
            v = np.asarray(d["dr"], dtype=np.float64).reshape(len(rows), 3)
            dr[rows, 0] = v[:, 0]
            dr[rows, 1] = np.exp(-v[:, 1] * self.config.dt)
            dr[rows, 2] = v[:, 2]
            dr[rows, 3] = v[:, 1]
            keep["dr"] = torch.as_tensor(dr, dtype=torch.float32, device=dev)
            tab.dr = L.ptr(keep["dr"])
        if "next_gate" in d:
            ng = np.zeros(self.n_envs, np.int32)
            ng[np.asarray(env_ids)] = np.asarray(d["next_gate"])
            keep["ng"] = torch.as_tensor(ng, device=dev)
            tab.next_gate = L.ptr(keep["ng"])
        return tab, keep

    def detach_states(self):
        """Cut the gradient at a training-window boundary (q/tasks.py:393-396)."""
        self._S = self._S.detach()

    # -- state views

    @property
    def state(self) -> dyn.QuadState:
        return dyn.unpack_state(self.config.dynamics, self._S)

    @state.setter
    def state(self, st: dyn.QuadState):
        ve = dyn.v_ema_of(self._S).detach()
        fields = {k: (v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v)))
                  .to(device=self.device, dtype=torch.float32) for k, v in st.fields().items()}
        self._S = dyn.pack_state(self.config.dynamics, dyn.QuadState(**fields), ve)

    @property
    def goals(self) -> torch.Tensor:
        return self._goal[:, 0:3]

    @goals.setter
    def goals(self, g):
        new = torch.zeros_like(self._goal)
        new[:, 0:3] = torch.as_tensor(np.asarray(g) if not isinstance(g, torch.Tensor) else g,
                                      dtype=torch.float32, device=self.device)
        self._goal = new

    @property
    def v_ema(self) -> torch.Tensor:
        return dyn.v_ema_of(self._S).detach()

    @v_ema.setter
    def v_ema(self, ve):
        ve = torch.as_tensor(np.asarray(ve) if not isinstance(ve, torch.Tensor) else ve,
                             dtype=torch.float32, device=self.device)
        S = self._S.clone()
        S[0, :, 3], S[1, :, 3], S[dyn.vema_plane(S), :, 3] = ve[:, 0], ve[:, 1], ve[:, 2]
        self._S = S

    @property
    def steps_in_episode(self) -> torch.Tensor:
        return self._meta[:, 0]

    @property
    def next_gate(self) -> torch.Tensor:
        return self._meta[:, 3]

    # racing gate arrays (q/tasks.py:864-867), views of the device gate table
    # (E, G, 8) = centre xyz, inner radius, normal xyz, frame width
    def _gate_table(self) -> torch.Tensor:
        if self.config.task != "racing" or self._scene.gates is None:
            raise AttributeError("gate arrays exist only for the racing task")
        return self._scene.gates

    @property
    def gate_centers(self) -> torch.Tensor:
        return self._gate_table()[..., 0:3]

    @property
    def gate_normals(self) -> torch.Tensor:
        return self._gate_table()[..., 4:7]

    @property
    def gate_inner(self) -> torch.Tensor:
        return self._gate_table()[..., 3]

    @property
    def gate_frame(self) -> torch.Tensor:
        return self._gate_table()[..., 7]

    @property
    def params(self) -> dyn.QuadParams:
        if self._dr is None:
            return self.base_params
        d = self._dr.double().cpu().numpy()
        return self.base_params.with_randomized(drag_coeff=d[:, 0], latency=d[:, 3])

    @property
    def action_lo(self):
        lo, hi = self.model.action_box()
        if self._dr is None:
            return lo
        s = self._dr[:, 2].double().cpu().numpy()[:, None]
        return (lo + hi) / 2 - (hi - lo) / 2 * s

    @property
    def action_hi(self):
        lo, hi = self.model.action_box()
        if self._dr is None:
            return hi
        s = self._dr[:, 2].double().cpu().numpy()[:, None]
        return (lo + hi) / 2 + (hi - lo) / 2 * s

    @property
    def prims(self) -> sn.BatchedPrimitives:
        bp = self._scene.to_batched()
        if self.n_agents == 1:
            return bp
        r = lambda a: torch.repeat_interleave(a, self.n_agents, dim=0)  # noqa: E731
        return sn.BatchedPrimitives(r(bp.spheres), r(bp.sph_valid), r(bp.boxes), r(bp.box_valid),
                                    r(bp.cylinders), r(bp.cyl_valid), r(bp.ground_z))

    @property
    def bounds_lo_per_row(self) -> torch.Tensor:
        return torch.repeat_interleave(self._scene.bounds[:, 0, :3] + 1e-6, self.n_agents, dim=0)

    @property
    def bounds_hi_per_row(self) -> torch.Tensor:
        return torch.repeat_interleave(self._scene.bounds[:, 1, :3] - 1e-6, self.n_agents, dim=0)

    @bounds_lo_per_row.setter
    def bounds_lo_per_row(self, lo):
        lo = torch.as_tensor(np.asarray(lo) if not isinstance(lo, torch.Tensor) else lo, dtype=torch.float32,
                             device=self.device).reshape(self.N, 3)
        self._scene.bounds[:, 0, :3] = lo[::self.n_agents] - 1e-6

    @bounds_hi_per_row.setter
    def bounds_hi_per_row(self, hi):
        hi = torch.as_tensor(np.asarray(hi) if not isinstance(hi, torch.Tensor) else hi, dtype=torch.float32,
                             device=self.device).reshape(self.N, 3)
        self._scene.bounds[:, 1, :3] = hi[::self.n_agents] + 1e-6

    # -- observation (q/tasks.py:415-463)

    def observe(self) -> Obs:
        dev = self.device
        obs = torch.empty(self.N, self.proprio_dim, dtype=torch.float32, device=dev)
        cam = torch.empty(self.N, 2, dtype=torch.float32, device=dev)
        io = self._new_io()
        io.S_out, io.goal_out, io.obs, io.cam = L.ptr(self._S), L.ptr(self._goal), L.ptr(obs), L.ptr(cam)
        L.check(L.lib().qs_task_observe(self._cfg, self._scene.struct(), io, L.stream_handle(dev)),
                "qs_task_observe")
        proprio = obs
        if self._S.requires_grad:
            # reconstruct the observation as a differentiable function of the
            # state: obs_k = obs_k(S) is linear in S with the kernel's frame,
            # so route it through one fused step-free VJP via autograd
            proprio = _ObserveFn.apply(self._S, obs, self)
        return Obs(proprio=proprio, visual=self._render(self._S.detach(), cam, force=True))

    def _render(self, S, cam, force=False):
        c = self.config
        sensor = self.camera if self.camera is not None else self.lidar
        if sensor is None:
            return None
        if not force and c.sensor_stride > 1 and self._frame_cache is not None:
            if self._steps_total % c.sensor_stride != 0:
                return self._frame_cache
        kind = 0 if self.camera is not None else 1
        if c.differentiable_depth and self.camera is not None:
            frame = sn.render_depth_differentiable(self._scene, S[0, :, 0:3], cam, sensor, kind,
                                                   self.n_agents)
        else:
            frame, _, _ = sn.cast_rays(self._scene, S[0].detach() if S.requires_grad else S[0], 4, cam,
                                       sensor, kind, True, self.n_agents)
        if self.camera is not None:
            frame = frame.reshape(self.N, self.camera.height, self.camera.width)
        self._frame_cache = frame
        return frame

    # -- stepping (q/tasks.py:549-600)

    def _check_inputs(self, raw: torch.Tensor):
        if tuple(raw.shape) != (self.N, self.action_dim):
            raise TaskContractError(f"action shape {tuple(raw.shape)} != {(self.N, self.action_dim)}")

    def check_errors(self):
        """Raise the contract error recorded by the kernels (syncs)."""
        self._raise_errors()

    def _raise_errors(self):
        code, row, key = self._err.tolist()  # the one host read of a strict step
        if key != _INT_MAX:  # qs_task_validate: the step was rejected before anything changed
            code, row = key >> 27, key & ((1 << 27) - 1)
            self._err[2] = _INT_MAX
            if code == L.QS_ERR_NONFINITE_ACTION:
                raise TaskContractError(f"non-finite action for env row {row}")
            raise dyn.ContractError(f"non-finite state (row {row})")
        if code == 0:
            return
        self._err.copy_(torch.tensor([0, _INT_MAX, _INT_MAX], dtype=torch.int32))
        if code == L.QS_ERR_NONFINITE_ACTION:
            raise TaskContractError(f"non-finite action for env row {row}")
        if code == L.QS_ERR_NONFINITE_STATE:
            raise dyn.ContractError(f"non-finite state (row {row})")
        if code == L.QS_ERR_GENERATION:
            raise wd.GenerationError(f"could not sample a reset (row {row})", self.seed)
        raise L.QuadsimLibraryError(f"device error code {code} at row {row}")

    def _deferred_resets(self, out, cow_scene: bool):
        """reset_mode 1 (injected reset draws, or scene regeneration that must
        precede the spawn): the step kernel left the done rows un-reset; spawn
        them now and re-observe (q/tasks.py:583-594)."""
        S_out, obs, flags, goal_out, peff_out, dr_out, cam, imu_out = (out[0], out[1], out[7], out[8], out[9],
                                                                        out[10], out[11], out[12])
        io = self._new_io()
        io.S_out, io.goal_out, io.peff_out = L.ptr(S_out), L.ptr(goal_out), L.ptr(peff_out)
        io.dr_out = L.ptr(dr_out) if dr_out.numel() else None
        io.obs, io.flags = L.ptr(obs), L.ptr(flags)
        io.cam = L.ptr(cam) if cam.numel() else None
        stream = L.stream_handle(self.device)
        if self.reset_source is not None:  # host-injected draws (syncs on the done mask)
            done_env = (flags.view(self.n_envs, self.n_agents)[:, 0] & 1).cpu().numpy().astype(bool)
            if done_env.any():
                ids = np.flatnonzero(done_env)
                tab, keep = self._reset_table(ids)
                self._regen_scenes(keep["mask"], cow_scene)
                L.check(L.lib().qs_task_spawn(self._cfg, self._scene.struct(), io, tab.env_mask, tab, stream),
                        "qs_task_spawn")
                self._episode_counter += 1
                del keep
        else:  # device-only: done mask -> new course -> Philox spawn, no host sync
            mask = (flags.view(self.n_envs, self.n_agents)[:, 0] & 1).to(torch.uint8)
            self._regen_scenes(mask, cow_scene)
            L.check(L.lib().qs_task_spawn(self._cfg, self._scene.struct(), io, L.ptr(mask), None, stream),
                    "qs_task_spawn")
        L.check(L.lib().qs_task_observe(self._cfg, self._scene.struct(), io, stream), "qs_task_observe")
        self._frame_cache = None

    def _regen_scenes(self, mask, cow: bool = False):
        """Re-randomise the obstacle course of every env in ``mask`` (uint8, device),
        keyed by (seed, env, episode) — ``meta[:, 1]`` already holds the new
        episode index.  The reference declares ``regen_scene_on_reset`` without
        wiring it (q/tasks.py:98); the course distribution is q/world.py:207-340.

        ``cow``: the current scene is referenced by recorded autograd nodes,
        whose backward re-evaluates the SDF at the primitive the forward chose;
        regenerate into a copy so those nodes keep their course."""
        if not self._regen:
            return
        if cow:
            self._scene = self._scene.clone()
        if self.config.task == "racing":
            wd.gen_race_tracks(self.seed, self.n_envs, out=self._scene, env_mask=mask, episode=self._meta[:, 1],
                               episode_stride=4, **self._track_args)
            return
        wd.gen_obstacle_courses(self.seed, self.n_envs, check=False, out=self._scene, env_mask=mask,
                                episode=self._meta[:, 1], episode_stride=4, err=self._err, **self._gen_args)

    def step(self, raw_action) -> StepOutput:
        raw = raw_action
        if not (type(raw) is torch.Tensor and raw.dtype is torch.float32 and raw.device == self.device):
            raw = raw if isinstance(raw, torch.Tensor) else torch.as_tensor(np.asarray(raw))
            raw = raw.to(device=self.device, dtype=torch.float32)
        self._check_inputs(raw)
        if not raw.is_contiguous():
            raw = raw.contiguous()
        noise = None
        if self._imu_bias is not None and self.imu_noise_source is not None:
            noise = torch.as_tensor(np.asarray(self.imu_noise_source(self._steps_total)), dtype=torch.float32,
                                    device=self.device).reshape(4, self.N, 3).contiguous()
        E = self._empty
        bufs = [self._goal, self._peff, self._dr if self._dr is not None else E, self._meta, self._ep_ret,
                self._imu_bias if self._imu_bias is not None else E, self._stats, self._err]
        # one dispatcher call: the fused step kernel (quadsim::task_step); with
        # strict=True a validation kernel runs first and guards the step
        out = self._ops.task_step(self._cfg_blob, self._scene.tensors(), self._S, raw, bufs, noise,
                                  self.config.sensor != "none", self.strict, self._cfg.proprio_dim)
        if self.strict:  # raise-before-mutate: a rejected step changed nothing
            self._raise_errors()
        if self._cfg.reset_mode == 1:
            self._deferred_resets(out, cow_scene=bool(self._S.requires_grad or raw.requires_grad))
        S_out, obs, r_ctrl, r_goal, r_rl, term, trunc, flags, goal_out, peff_out, dr_out, cam, imu_out = out
        self._S, self._goal, self._peff = S_out, goal_out, peff_out
        if self._dr is not None:
            self._dr = dr_out
        self._steps_total += 1
        self._last_flags = flags
        visual = self._render(S_out, cam) if self.config.sensor != "none" else None
        imu = (imu_out[:, 0:3], imu_out[:, 3:6]) if self._imu_bias is not None else None
        return StepOutput(obs=Obs(proprio=obs, visual=visual, imu=imu), r_ctrl=r_ctrl, r_goal=r_goal,
                          r_rl=r_rl, terminated=term, truncated=trunc)

    def state_records(self):
        return {k: v.detach().cpu().tolist() for k, v in self.state.fields().items()}

    # -- critic features (q/tasks.py:292-297, 465-545)

    def privileged_dim(self) -> int:
        return 14

    def privileged_scale(self) -> tuple:
        return (0.2,) * 3 + (1 / 3.0,) * 3 + (0.1,) * 3 + (0.2,) + (1.0,) * 3 + (0.2,)

    def _thrust(self, st: dyn.QuadState) -> torch.Tensor:
        """q/tasks.py:479-498."""
        name = self.config.dynamics
        if name == "pm_continuous":
            return st.a_lat
        if name == "pm_discrete":
            g = getattr(self, "_g_dev", None)
            if g is None:  # cached: no host->device copy per call (CUDA-graph capture)
                g = self._g_dev = torch.as_tensor(self.base_params.g_vec, dtype=torch.float32, device=self.device)
            return st.u_prev - g
        if name == "simplified":
            return st.R[:, :, 2] * 9.81
        w, x, y, z = st.q.unbind(-1)
        zb = torch.stack([2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)], -1)
        return zb * 9.81

    def privileged_var(self) -> torch.Tensor:
        """(N,14) critic features, differentiable through the state (q/tasks.py:500-523):
        yaw-local goal offset, velocity, thrust; sdf clamped to +-5; yaw-local
        clearance direction (constant); goal distance.  The clearance direction
        is the sdf kernel's analytic gradient of the nearest primitive, which is
        what the reference's 6-probe central difference (h=1e-4, :465-477)
        approximates; in fp32 that difference quotient would be noise-limited."""
        st = self.state
        cam = _cam_of(self)
        c, s = cam[:, 0:1], cam[:, 1:2]

        def unrot(v):
            return torch.cat([c * v[:, 0:1] + s * v[:, 1:2], -s * v[:, 0:1] + c * v[:, 1:2], v[:, 2:3]], -1)

        off = self.goals - st.p
        sd = sn.sdf_var(st.p, self._scene, self.n_agents)
        _, grad = sn._sdf_launch(self._scene, st.p.detach(), self.n_agents, True)
        return torch.cat([unrot(off), unrot(st.v), unrot(self._thrust(st)), torch.clamp(sd, -5.0, 5.0)[:, None],
                          unrot(grad[:, 0:3]), torch.linalg.norm(off, dim=-1, keepdim=True)], -1)

    def privileged_state(self) -> torch.Tensor:
        """No-grad twin of privileged_var (q/tasks.py:525-545), one kernel
        (qs_task_privileged) on the current state."""
        out = torch.empty(self.N, 14, dtype=torch.float32, device=self.device)
        io = self._new_io()
        io.S_out, io.goal_out = L.ptr(self._S.detach()), L.ptr(self._goal)
        L.check(L.lib().qs_task_privileged(self._cfg, self._scene.struct(), io, L.ptr(out),
                                           L.stream_handle(self.device)), "qs_task_privileged")
        return out


class _ObserveFn(torch.autograd.Function):
    """observe() on a grad-carrying state: value from qs_task_observe, VJP from
    qs_task_step_bwd's observation path is not reusable here, so the (linear,
    fixed-frame) observation Jacobian is applied with torch ops."""

    @staticmethod
    def forward(ctx, S, obs, env):
        ctx.env = env
        ctx.save_for_backward(S, obs)
        return obs.clone()

    @staticmethod
    def backward(ctx, g):
        S, obs = ctx.saved_tensors
        env = ctx.env
        model = env.config.dynamics
        with torch.enable_grad():
            Sd = S.detach().requires_grad_(True)
            st = dyn.unpack_state(model, Sd)
            # frame (yaw) is a constant: recover cos/sin from the kernel's own
            # observation of the velocity (v_loc = Rz(-yaw) v)
            cam = _cam_of(env)
            c, s = cam[:, 0:1], cam[:, 1:2]

            def unrot(x):
                return torch.cat([c * x[:, 0:1] + s * x[:, 1:2], -s * x[:, 0:1] + c * x[:, 1:2], x[:, 2:3]], -1)

            clip = env.config.obs_clip
            off = unrot(env.goals - st.p)
            inside = ((off >= -clip) & (off <= clip)).float()
            parts = [off * inside, unrot(st.v)]
            if model == "full":
                w, x, y, z = st.q.unbind(-1)
                zb = torch.stack([2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)], -1)
                parts += [unrot(zb), st.w]
            elif model == "simplified":
                parts.append(unrot(st.R[:, :, 2]))
            else:
                parts.append(unrot(st.a_lat if model == "pm_continuous" else st.u_prev))
            lin = torch.cat(parts, -1)
            P = lin.shape[1]
            (gS,) = torch.autograd.grad(lin, Sd, g[:, :P])
        return gS, None, None


def _cam_of(env):
    cam = torch.empty(env.N, 2, dtype=torch.float32, device=env.device)
    obs = torch.empty(env.N, env.proprio_dim, dtype=torch.float32, device=env.device)
    io = env._new_io()
    io.S_out, io.goal_out, io.obs, io.cam = L.ptr(env._S.detach()), L.ptr(env._goal), L.ptr(obs), L.ptr(cam)
    L.check(L.lib().qs_task_observe(env._cfg, env._scene.struct(), io, L.stream_handle(env.device)),
            "qs_task_observe")
    return cam


class PositionTask(FlightTask):
    """Reach and hover at a target (q/tasks.py:658-763)."""


class AvoidanceTask(FlightTask):
    """Position control through generated obstacle fields (q/tasks.py:766-844)."""


class RacingTask(FlightTask):
    """Traverse gates in order (q/tasks.py:847-972)."""


def make_task(config: TaskConfig, params: dyn.QuadParams | None = None, **kw) -> FlightTask:
    """q/tasks.py:1004-1008."""
    cls = {"position": PositionTask, "avoidance": AvoidanceTask, "racing": RacingTask}[config.task]
    return cls(config, params, **kw)
