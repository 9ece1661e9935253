"""Differentiable quadrotor dynamics on sm_100a (mirrors ``q/dynamics.py``).

Conventions are the reference's: z-up world, g = (0, 0, -9.81), thrust as
mass-normalised acceleration, quaternions (w, x, y, z).  ``DynamicsModel.step``
runs the hand-written forward kernel (``qs_dyn_step_fwd``) and its autograd
backward is the analytic VJP kernel (``qs_dyn_step_bwd``); states are torch
CUDA fp32 tensors.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np
import torch

from paper_2509_10247_b200 import _lib as L

GRAVITY = np.array([0.0, 0.0, -9.81])
MODEL_NAMES = ("full", "simplified", "pm_continuous", "pm_discrete")


class ContractError(ValueError):
    """A dynamics precondition was violated (bad shape, non-finite state)."""


@dataclass
class QuadParams:
    """q/dynamics.py:42-82.  drag_coeff / latency may be scalars or (B,) arrays."""

    mass: float = 1.0
    inertia: np.ndarray = field(default_factory=lambda: np.diag([2.3e-3, 2.3e-3, 4.0e-3]))
    drag_matrix_diag: np.ndarray = field(default_factory=lambda: np.zeros(3))
    drag_coeff: object = 0.3
    latency: object = 4.0
    g_vec: np.ndarray = field(default_factory=lambda: GRAVITY.copy())
    rate_gains: np.ndarray = field(default_factory=lambda: np.array([20.0, 20.0, 8.0]))
    dt: float = 0.01

    def __post_init__(self):
        self.inertia = np.asarray(self.inertia, dtype=np.float64)
        J = self.inertia
        if J.shape != (3, 3) or not np.allclose(J, J.T):
            raise ContractError("inertia must be a symmetric 3x3 matrix")
        if np.any(np.linalg.eigvalsh(J) <= 0):
            raise ContractError("inertia must be positive definite")
        if self.dt <= 0:
            raise ContractError("dt must be positive")
        self.drag_matrix_diag = np.asarray(self.drag_matrix_diag, dtype=np.float64)
        if np.any(self.drag_matrix_diag < 0) or np.any(np.asarray(self.drag_coeff) < 0):
            raise ContractError("drag terms must be non-negative")
        if np.any(np.asarray(self.latency) < 0):
            raise ContractError("latency must be non-negative")
        self.g_vec = np.asarray(self.g_vec, dtype=np.float64)
        self.rate_gains = np.asarray(self.rate_gains, dtype=np.float64)

    @property
    def inertia_inv(self):
        return np.linalg.inv(self.inertia)

    @property
    def lag_decay(self):
        return np.exp(-np.asarray(self.latency, dtype=np.float64) * self.dt)

    def with_randomized(self, drag_coeff=None, latency=None) -> "QuadParams":
        return replace(self, drag_coeff=self.drag_coeff if drag_coeff is None else drag_coeff,
                       latency=self.latency if latency is None else latency)


FIELDS = {
    "full": ("p", "v", "q", "w"),
    "simplified": ("p", "v", "R"),
    "pm_continuous": ("p", "v", "a_lat"),
    "pm_discrete": ("p", "v", "u_prev"),
}


@dataclass
class QuadState:
    """Batched state (q/dynamics.py:85-117); fields are (B,k) tensors."""

    p: torch.Tensor
    v: torch.Tensor
    q: torch.Tensor | None = None
    R: torch.Tensor | None = None
    w: torch.Tensor | None = None
    a_lat: torch.Tensor | None = None
    u_prev: torch.Tensor | None = None

    @property
    def batch(self) -> int:
        return self.p.shape[0]

    def fields(self):
        out = {"p": self.p, "v": self.v}
        for name in ("q", "R", "w", "a_lat", "u_prev"):
            v = getattr(self, name)
            if v is not None:
                out[name] = v
        return out

    def detached(self) -> "QuadState":
        return QuadState(**{k: v.detach() for k, v in self.fields().items()})

    def values(self):
        return {k: v.detach() for k, v in self.fields().items()}


def model_of_state(st: QuadState) -> str:
    if st.q is not None:
        return "full"
    if st.R is not None:
        return "simplified"
    if st.a_lat is not None:
        return "pm_continuous"
    return "pm_discrete"


def pack_state(model: str, st: QuadState, v_ema: torch.Tensor | None = None) -> torch.Tensor:
    """QuadState -> (NP,B,4) planes; v_ema rides in the pad lanes."""
    B = st.p.shape[0]
    dev = st.p.device
    ve = v_ema if v_ema is not None else torch.zeros(B, 3, dtype=torch.float32, device=dev)
    ve = ve.to(torch.float32)
    f = lambda x: x.to(torch.float32)  # noqa: E731
    planes = [torch.cat([f(st.p), ve[:, 0:1]], -1), torch.cat([f(st.v), ve[:, 1:2]], -1)]
    if model == "full":
        planes += [f(st.q), torch.cat([f(st.w), ve[:, 2:3]], -1)]
    elif model == "simplified":
        R = f(st.R)
        z = torch.zeros(B, 1, dtype=torch.float32, device=dev)
        planes += [torch.cat([R[:, :, 0], ve[:, 2:3]], -1), torch.cat([R[:, :, 1], z], -1),
                   torch.cat([R[:, :, 2], z], -1)]
    else:
        x = st.a_lat if model == "pm_continuous" else st.u_prev
        planes.append(torch.cat([f(x), ve[:, 2:3]], -1))
    return torch.stack(planes, 0).contiguous()


def unpack_state(model: str, S: torch.Tensor) -> QuadState:
    """(NP,B,4) planes -> QuadState of views (autograd flows through them)."""
    if model == "full":
        return QuadState(p=S[0, :, 0:3], v=S[1, :, 0:3], q=S[2], w=S[3, :, 0:3])
    if model == "simplified":
        return QuadState(p=S[0, :, 0:3], v=S[1, :, 0:3], R=torch.stack([S[2, :, 0:3], S[3, :, 0:3], S[4, :, 0:3]], -1))
    x = S[2, :, 0:3]
    if model == "pm_continuous":
        return QuadState(p=S[0, :, 0:3], v=S[1, :, 0:3], a_lat=x)
    return QuadState(p=S[0, :, 0:3], v=S[1, :, 0:3], u_prev=x)


def vema_plane(S: torch.Tensor) -> int:
    """Plane whose pad lane holds v_ema.z: the last plane, except for the
    simplified model whose R columns 1 and 2 have no spare lane meaning."""
    return 2 if S.shape[0] == 5 else S.shape[0] - 1


def v_ema_of(S: torch.Tensor) -> torch.Tensor:
    return torch.stack([S[0, :, 3], S[1, :, 3], S[vema_plane(S), :, 3]], -1)


def fill_dyn_cfg(cfg: L.QsTaskCfg, model: str, params: QuadParams, action_box=None):
    cfg.model = L.MODEL_IDS[model]
    cfg.dt = float(params.dt)
    for i in range(3):
        cfg.g[i] = float(params.g_vec[i])
        cfg.drag_diag[i] = float(params.drag_matrix_diag[i])
        cfg.rate_gains[i] = float(params.rate_gains[i])
    dc = np.asarray(params.drag_coeff, dtype=np.float64)
    ld = np.asarray(params.lag_decay, dtype=np.float64)
    cfg.drag_coeff = float(dc) if dc.ndim == 0 else 0.0
    cfg.lag_decay = float(ld) if ld.ndim == 0 else 0.0
    if action_box is not None:
        lo, hi = action_box
        for i in range(len(lo)):
            cfg.act_lo[i], cfg.act_hi[i] = float(lo[i]), float(hi[i])
            # the kernels' fp32 (lo+hi)*0.5 and (hi-lo)*0.5, precomputed once
            l32, h32 = np.float32(lo[i]), np.float32(hi[i])
            cfg.act_center[i] = float((l32 + h32) * np.float32(0.5))
            cfg.act_half[i] = float((h32 - l32) * np.float32(0.5))
    cfg.imu_sqrt_dt = float(np.sqrt(np.float32(params.dt)))
    return cfg


def per_row_params(params: QuadParams, B: int, device) -> torch.Tensor | None:
    """(B,4) drag, lag_decay, action scale (1), latency when params are per env."""
    dc = np.asarray(params.drag_coeff, dtype=np.float64)
    lat = np.asarray(params.latency, dtype=np.float64)
    if dc.ndim == 0 and lat.ndim == 0:
        return None
    out = np.zeros((B, 4))
    out[:, 0] = np.broadcast_to(dc, (B,))
    out[:, 1] = np.broadcast_to(np.exp(-lat * params.dt), (B,))
    out[:, 2] = 1.0
    out[:, 3] = np.broadcast_to(lat, (B,))
    return torch.as_tensor(out, dtype=torch.float32, device=device)


class _DynStepFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, S, act, model, cfg, dr, err):
        ctx.set_materialize_grads(False)
        B = S.shape[1]
        S = S.contiguous()
        act = act.contiguous()
        So = torch.empty_like(S)
        L.check(L.lib().qs_dyn_step_fwd(L.MODEL_IDS[model], B, L.ptr(S), L.ptr(act), L.ptr(dr), cfg,
                                        L.ptr(So), L.ptr(err), L.stream_handle(S.device)),
                "qs_dyn_step_fwd")
        ctx.save_for_backward(S, act)
        ctx.model, ctx.cfg, ctx.dr = model, cfg, dr
        return So

    @staticmethod
    def backward(ctx, gSo):
        S, act = ctx.saved_tensors
        if gSo is None:
            return None, None, None, None, None, None
        B = S.shape[1]
        gS = torch.empty_like(S)
        ga = torch.empty_like(act)
        L.check(L.lib().qs_dyn_step_bwd(L.MODEL_IDS[ctx.model], B, L.ptr(S), L.ptr(act), L.ptr(ctx.dr),
                                        ctx.cfg, L.ptr(gSo.contiguous()), L.ptr(gS), L.ptr(ga),
                                        L.stream_handle(S.device)), "qs_dyn_step_bwd")
        return gS, ga, None, None, None, None


def _check_state_finite(st: QuadState):
    """q/dynamics.py:130-133 (synchronous, like the reference)."""
    for name, v in st.fields().items():
        if not bool(torch.isfinite(v).all()):
            raise ContractError(f"non-finite state field '{name}'")


class DynamicsModel:
    """Uniform interface (q/dynamics.py:291-320)."""

    name = ""
    action_dim = 0

    def __init__(self, params: QuadParams, device=None):
        self.params = params
        self.device = L.require_cuda(device)

    def _t(self, x):
        if isinstance(x, torch.Tensor):
            return x.to(device=self.device, dtype=torch.float32)
        return torch.as_tensor(np.asarray(x), dtype=torch.float32, device=self.device)

    def step(self, state: QuadState, action, check: bool = True) -> QuadState:
        """Advance one step; ``action`` is a squashed (B, action_dim) command."""
        if check:
            _check_state_finite(state)
        act = self._t(action) if not isinstance(action, torch.Tensor) else action.float()
        B = state.batch
        cfg = fill_dyn_cfg(L.QsTaskCfg(), self.name, self.params)
        dr = per_row_params(self.params, B, self.device)
        err = torch.zeros(2, dtype=torch.int32, device=self.device)
        S = pack_state(self.name, state)
        So = _DynStepFn.apply(S, act, self.name, cfg, dr, err)
        return unpack_state(self.name, So)

    def init_state(self, p, v) -> QuadState:
        raise NotImplementedError

    def hover_action(self, batch: int) -> torch.Tensor:
        raise NotImplementedError

    def action_box(self):
        raise NotImplementedError

    def thrust_accel(self, state: QuadState):
        raise NotImplementedError


class FullQuadrotor(DynamicsModel):
    name = "full"
    action_dim = 4

    def init_state(self, p, v):
        p, v = self._t(p), self._t(v)
        B = p.shape[0]
        q = torch.zeros(B, 4, dtype=torch.float32, device=self.device)
        q[:, 0] = 1.0
        return QuadState(p=p, v=v, q=q, w=torch.zeros(B, 3, dtype=torch.float32, device=self.device))

    def hover_action(self, batch):
        a = torch.zeros(batch, 4, dtype=torch.float32, device=self.device)
        a[:, 0] = float(-self.params.g_vec[2])
        return a

    def action_box(self):
        gz = -self.params.g_vec[2]
        return np.array([0.0, -6.0, -6.0, -3.0]), np.array([2.0 * gz, 6.0, 6.0, 3.0])

    def attitude(self, state):
        return quat_to_matrix(state.q)


class SimplifiedQuadrotor(DynamicsModel):
    """q/dynamics.py:352-379: v' = v + (R e_z c + g) dt, R' = GS(R + R[w]x dt)."""

    name = "simplified"
    action_dim = 4

    def init_state(self, p, v):
        p, v = self._t(p), self._t(v)
        R = torch.eye(3, dtype=torch.float32, device=self.device).expand(p.shape[0], 3, 3).contiguous()
        return QuadState(p=p, v=v, R=R)

    def hover_action(self, batch):
        a = torch.zeros(batch, 4, dtype=torch.float32, device=self.device)
        a[:, 0] = float(-self.params.g_vec[2])
        return a

    def action_box(self):
        gz = -self.params.g_vec[2]
        return np.array([0.0, -6.0, -6.0, -3.0]), np.array([2.0 * gz, 6.0, 6.0, 3.0])

    def attitude(self, state):
        return state.R


class PointMassContinuous(DynamicsModel):
    name = "pm_continuous"
    action_dim = 3

    def init_state(self, p, v):
        p, v = self._t(p), self._t(v)
        a0 = self._t(-self.params.g_vec).expand(p.shape[0], 3).contiguous()
        return QuadState(p=p, v=v, a_lat=a0)

    def hover_action(self, batch):
        return self._t(-self.params.g_vec).expand(batch, 3).contiguous()

    def action_box(self):
        gz = -self.params.g_vec[2]
        return np.array([-6.0, -6.0, gz - 6.0]), np.array([6.0, 6.0, gz + 6.0])

    def thrust_accel(self, state):
        return state.a_lat


class PointMassDiscrete(DynamicsModel):
    name = "pm_discrete"
    action_dim = 3

    def init_state(self, p, v):
        p, v = self._t(p), self._t(v)
        return QuadState(p=p, v=v, u_prev=torch.zeros(p.shape[0], 3, dtype=torch.float32, device=self.device))

    def hover_action(self, batch):
        return torch.zeros(batch, 3, dtype=torch.float32, device=self.device)

    def action_box(self):
        return np.full(3, -6.0), np.full(3, 6.0)

    def thrust_accel(self, state):
        return state.u_prev - self._t(self.params.g_vec)


_MODELS = {c.name: c for c in (FullQuadrotor, SimplifiedQuadrotor, PointMassContinuous, PointMassDiscrete)}


def make_model(name: str, params: QuadParams | None = None, device=None) -> DynamicsModel:
    """q/dynamics.py:437-441."""
    try:
        cls = _MODELS[name]
    except KeyError:
        raise ContractError(f"unknown dynamics model '{name}'; choose from {tuple(_MODELS)}")
    return cls(params or QuadParams(), device=device)


def rate_loop(w: torch.Tensor, w_cmd: torch.Tensor, params: QuadParams) -> torch.Tensor:
    """Body-rate P controller with gyroscopic feedforward (q/dynamics.py:140-152):
    tau = J (K (w_cmd - w)) + w x (J w).  The step kernels use the algebraically
    equal w_dot = K (w_cmd - w); this is the torque for API parity."""
    J = torch.as_tensor(params.inertia, dtype=w.dtype, device=w.device)
    K = torch.as_tensor(params.rate_gains, dtype=w.dtype, device=w.device)
    return (K * (w_cmd - w)) @ J.T + torch.cross(w, w @ J.T, dim=-1)


def action_squash(raw: torch.Tensor, lo, hi) -> torch.Tensor:
    """tanh squash into [lo, hi] (q/dynamics.py:277-284)."""
    lo = torch.as_tensor(np.asarray(lo), dtype=torch.float32, device=raw.device)
    hi = torch.as_tensor(np.asarray(hi), dtype=torch.float32, device=raw.device)
    return (lo + hi) * 0.5 + (hi - lo) * 0.5 * torch.tanh(raw)


def quat_to_matrix(q: torch.Tensor) -> torch.Tensor:
    """q/dynamics.py:448-460."""
    w, x, y, z = q.unbind(-1)
    return torch.stack([
        1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
        2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
        2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y),
    ], -1).reshape(q.shape[:-1] + (3, 3))


@dataclass
class RolloutGrad:
    grad: torch.Tensor
    detached: bool


def rollout_grad(model: DynamicsModel, state0: QuadState, raw_actions, t1: int, t2: int,
                 weights: dict | None = None, squash: bool = False) -> RolloutGrad:
    """d(w . s_t2) / d(a_t1) through a rollout of the kernel steps (q/dynamics.py:481-520)."""
    raw = model._t(raw_actions)
    T = raw.shape[0]
    if not (0 <= t1 < t2 <= T):
        raise ContractError(f"need 0 <= t1 < t2 <= T, got t1={t1}, t2={t2}, T={T}")
    leaves = [raw[t].clone().requires_grad_(True) for t in range(T)]
    lo, hi = model.action_box()
    st = state0
    for t in range(t2):
        act = action_squash(leaves[t], lo, hi) if squash else leaves[t]
        st = model.step(st, act, check=False)
    root = None
    for name, var in st.fields().items():
        if weights is not None:
            if name not in weights:
                continue
            w = model._t(weights[name]).expand_as(var)
        else:
            w = torch.ones_like(var)
        term = (var * w).sum()
        root = term if root is None else root + term
    (g,) = torch.autograd.grad(root, [leaves[t1]], allow_unused=True)
    if g is None:
        return RolloutGrad(torch.zeros_like(leaves[t1]), True)
    return RolloutGrad(g, False)


# ---------------------------------------------------------------------------
# the reference's functional step API (q/dynamics.py:155-274): thin wrappers
# over the same kernels as DynamicsModel.step; commands are already squashed


def _functional_step(name, state, act, params):
    dev = act.device if isinstance(act, torch.Tensor) else None
    return make_model(name, params, device=dev).step(state, act)


def step_full(state: QuadState, thrust, w_cmd, params: QuadParams) -> QuadState:
    """q/dynamics.py:155-186: collective thrust (B,) and body-rate command (B,3)."""
    th = torch.as_tensor(thrust, dtype=torch.float32).reshape(-1, 1)
    w = torch.as_tensor(w_cmd, dtype=torch.float32).reshape(-1, 3)
    return _functional_step("full", state, torch.cat([th.to(w.device), w], -1), params)


def step_simplified(state: QuadState, thrust, w, params: QuadParams) -> QuadState:
    """q/dynamics.py:203-234."""
    th = torch.as_tensor(thrust, dtype=torch.float32).reshape(-1, 1)
    w = torch.as_tensor(w, dtype=torch.float32).reshape(-1, 3)
    return _functional_step("simplified", state, torch.cat([th.to(w.device), w], -1), params)


def step_pm_continuous(state: QuadState, u, params: QuadParams) -> QuadState:
    """q/dynamics.py:237-258 (u: world-frame commanded acceleration (B,3))."""
    return _functional_step("pm_continuous", state, u, params)


def step_pm_discrete(state: QuadState, u, params: QuadParams) -> QuadState:
    """q/dynamics.py:261-274."""
    return _functional_step("pm_discrete", state, u, params)


def quat_to_matrix_np(q: np.ndarray) -> np.ndarray:
    """q/dynamics.py:448-460: (w, x, y, z) unit quaternions (B,4) -> (B,3,3) (host helper)."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)
