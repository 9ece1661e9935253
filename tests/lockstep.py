"""Lockstep harness: the GPU env and the fp64 CPU oracle stepped side by side
(TEST INFRASTRUCTURE ONLY).

* ``OracleLockstep`` drives ``oracle.OracleTask`` and ``tasks.FlightTask`` with
  the same raw actions and the same IMU normals; the GPU env's resets are the
  oracle's own PCG64 draws (the reference's spawn sampling, q/tasks.py:687-721,
  restated by the oracle and pinned by the golden fixtures), injected through
  ``reset_source``.  With ``teacher_force=True`` every step starts both sides
  from the SAME fp32-representable carried state (the oracle's, rounded), so
  each step's outputs are single-step results and are held to the north
  star's 1e-5 without any compounding allowance.
* ``InjectedOracle`` is an ``OracleTask`` whose resets take their spawn rows
  from a table (the GPU's own in-kernel Philox resets), for comparing paths
  whose resets cannot be injected (the fused BPTT window).
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import quadsim_oracle as O

import paper_2509_10247_b200 as qs
from paper_2509_10247_b200 import dynamics as dyn

STATE_KEYS = O.STATE_FIELDS


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def rel_err(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(x - ref) / np.maximum(np.abs(ref), 1.0)))


def gpu_state(env) -> dict:
    return {k: v.detach().double().cpu().numpy() for k, v in env.state.fields().items()}


def set_gpu_carry(env, state: dict, goals, v_ema, prev_effort=None, imu_bias=None, steps=None):
    """Overwrite the GPU env's carried state (functional state planes, goals,
    v_ema, previous effort, IMU bias, episode step counters)."""
    dev = env.device
    t = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float32, device=dev)  # noqa: E731
    env.state = dyn.QuadState(**{k: t(v) for k, v in state.items()})
    env.v_ema = t(v_ema)
    env.goals = t(goals)
    if prev_effort is not None:
        pe = torch.zeros_like(env._peff)
        pe[:, :prev_effort.shape[1]] = t(prev_effort)
        env._peff = pe
    if imu_bias is not None:
        ba, bg = imu_bias
        b = torch.zeros_like(env._imu_bias)
        b[:, 0:3] = t(ba)
        b[:, 4:7] = t(bg)
        env._imu_bias.copy_(b)
    if steps is not None:
        env._meta[:, 0] = torch.as_tensor(np.asarray(steps), dtype=torch.int32, device=dev)


class OracleLockstep:
    """GPU FlightTask and OracleTask over the same inputs.

    ``kw`` are TaskConfig keywords shared by both (position/avoidance tasks
    without scene injection).  ``imu``: dict of the four IMU stds or None.
    """

    def __init__(self, kw: dict, seed: int, imu: dict | None = None, noise_seed: int = 5, device="cuda"):
        self.kw = dict(kw)
        self.imu = imu
        ocfg = O.Config(**kw)
        self.oracle = O.OracleTask(ocfg, imu=None if imu is None else dict(imu, seed=0))
        self.oracle.reset(seed)
        cfg = qs.TaskConfig(**kw, imu=None if imu is None else qs.ImuSpec(**imu))
        self._noise = None
        self.env = qs.make_task(cfg, device=device, reset_source=self._reset_src)
        self.env.imu_noise_source = (lambda step: self._noise) if imu is not None else None
        self.out0 = self.env.reset(seed)
        self.rng = np.random.default_rng(noise_seed)
        self.N = self.env.N
        self.model = kw.get("dynamics", "pm_continuous")

    def _reset_src(self, env_ids, counter, initial):
        log = self.oracle.reset_log[0 if initial else -1]
        assert np.array_equal(np.asarray(env_ids), log["env_ids"]), (env_ids, log["env_ids"])
        return {"p": log["p"], "v": log["v"], "goal": log["goal"], "v_ema": log["v_ema"]}

    def force_carry(self):
        """Round the oracle's carried state to fp32 and load it on both sides."""
        o = self.oracle
        for k in o.state:
            o.state[k] = f32(o.state[k])
        o.goals = f32(o.goals)
        o.v_ema = f32(o.v_ema)
        o.prev_effort = f32(o.prev_effort)
        bias = None
        if self.imu is not None:
            o.imu.accel_bias = f32(o.imu.accel_bias)
            o.imu.gyro_bias = f32(o.imu.gyro_bias)
            bias = (o.imu.accel_bias, o.imu.gyro_bias)
        set_gpu_carry(self.env, o.state, o.goals, o.v_ema, o.prev_effort, bias, o.steps)

    def step(self, raw, teacher_force=False):
        """One step on both sides; returns (gpu record, oracle record)."""
        if teacher_force:
            self.force_carry()
        normals = None
        if self.imu is not None:
            normals = tuple(self.rng.standard_normal((self.N, 3)) for _ in range(4))
            self._noise = np.stack(normals)
        ref = self.oracle.step(raw, imu_normals=normals)
        out = self.env.step(torch.as_tensor(raw, dtype=torch.float32, device=self.env.device))
        rec = {"proprio": out.obs.proprio.detach().double().cpu().numpy(),
               "r_ctrl": out.r_ctrl.detach().double().cpu().numpy(),
               "r_goal": out.r_goal.double().cpu().numpy(), "r_rl": out.r_rl.double().cpu().numpy(),
               "term": out.terminated.cpu().numpy(), "trunc": out.truncated.cpu().numpy(),
               "state": gpu_state(self.env), "goals": self.env.goals.double().cpu().numpy(),
               "v_ema": self.env.v_ema.double().cpu().numpy(),
               "steps": self.env.steps_in_episode.cpu().numpy()}
        if out.obs.imu is not None:
            rec["imu_accel"] = out.obs.imu[0].double().cpu().numpy()
            rec["imu_gyro"] = out.obs.imu[1].double().cpu().numpy()
        if out.obs.visual is not None:
            rec["visual"] = out.obs.visual.double().cpu().numpy()
        ref = dict(ref)
        ref["state"] = self.oracle.state
        ref["goals"] = self.oracle.goals
        ref["v_ema"] = self.oracle.v_ema
        ref["steps"] = self.oracle.steps
        return rec, ref


def compare_step(rec, ref, model, tol, depth_tol=1e-4):
    """Exact: termination codes, truncation, r_goal, episode step counters
    (reset indices).  Within ``tol`` (relative, floored at 1): state, goals,
    v_ema, observation, r_ctrl, r_rl, IMU.  Returns the per-quantity errors."""
    assert np.array_equal(rec["term"], ref["terminated"]), np.flatnonzero(rec["term"] != ref["terminated"])
    assert np.array_equal(rec["trunc"], ref["truncated"])
    assert np.array_equal(rec["r_goal"], ref["r_goal"])
    assert np.array_equal(rec["steps"], ref["steps"])
    errs = {"proprio": rel_err(rec["proprio"], ref["proprio"]), "r_ctrl": rel_err(rec["r_ctrl"], ref["r_ctrl"]),
            "r_rl": rel_err(rec["r_rl"], ref["r_rl"]), "goals": rel_err(rec["goals"], ref["goals"]),
            "v_ema": rel_err(rec["v_ema"], ref["v_ema"])}
    for k in STATE_KEYS[model]:
        errs["s_" + k] = rel_err(rec["state"][k], ref["state"][k])
    if "imu_accel" in rec:
        errs["imu_accel"] = rel_err(rec["imu_accel"], ref["imu_accel"])
        errs["imu_gyro"] = rel_err(rec["imu_gyro"], ref["imu_gyro"])
    for k, v in errs.items():
        assert v <= tol, (k, v, errs)
    if "visual" in rec:
        errs["visual"] = float(np.abs(rec["visual"].reshape(ref["visual"].shape) - ref["visual"]).max())
        assert errs["visual"] <= depth_tol, errs
    return errs


class InjectedOracle(O.OracleTask):
    """OracleTask whose resets land on rows given by ``self.inject`` (a dict
    of per-row arrays p, v, goal, v_ema), e.g. the GPU's in-kernel Philox
    resets.  Everything else -- which envs reset, counters, prev-effort and
    IMU-bias zeroing, the gradient cut -- is the oracle's own logic
    (q/tasks.py:583-611, 712-721)."""

    inject = None

    def _spawn_all(self, env_mask):
        if self.inject is None or self.state is None:
            return super()._spawn_all(env_mask)
        na = self.n_agents
        rows = np.repeat(env_mask, na)
        p_new = self.state["p"].copy()
        v_new = self.state["v"].copy()
        p_new[rows] = self.inject["p"][rows]
        v_new[rows] = self.inject["v"][rows]
        self.goals[rows] = self.inject["goal"][rows]
        self.v_ema[rows] = self.inject["v_ema"][rows]
        self.episode_counter += 1
        fresh = O.init_state(self.model, p_new, v_new)
        for k in self.state:
            m = rows.reshape((-1,) + (1,) * (fresh[k].ndim - 1))
            self.state[k] = np.where(m, fresh[k], self.state[k])
        self.prev_effort[rows] = 0.0


def window_slot(win, t):
    """The fused window's carried-state checkpoint of slot t as numpy
    (state fields, goals, v_ema, prev effort)."""
    model = win.env.config.dynamics
    S = win.S[t]
    st = {k: v.detach().double().cpu().numpy() for k, v in dyn.unpack_state(model, S).fields().items()}
    ve = dyn.v_ema_of(S).double().cpu().numpy()
    goal = win.goal[t][:, 0:3].double().cpu().numpy()
    peff = win.peff[t][:, :win.env.action_dim].double().cpu().numpy()
    return st, goal, ve, peff
