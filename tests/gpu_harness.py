"""Build GPU envs that replay a golden fixture exactly (test infrastructure).

Resets are injected from the fixture through the env's ``reset_source`` hook
and scenes through ``scene_source``, so the GPU run sees the reference's own
PCG64 draws; everything else is computed by the kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from golden_utils import TASK_CASES, load, scene_from_json

import paper_2509_10247_b200 as qs
from paper_2509_10247_b200 import sensors as sn
from paper_2509_10247_b200 import tasks as tk
from paper_2509_10247_b200 import world as wd

# tolerances stated by the north star (BASELINE.json)
STATE_TOL = 1e-5  # |x - ref| <= tol * max(|ref|, 1)   (fp32 vs fp64 oracle)
DEPTH_TOL = 1e-4  # metres
GRAD_TOL = 1e-4  # max-normalised


def state_err(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(x - ref) / np.maximum(np.abs(ref), 1.0))) if ref.size else 0.0


def grad_err(g, ref):
    g = np.asarray(g, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    s = np.abs(ref).max()
    return float(np.abs(g - ref).max() / s) if s > 0 else float(np.abs(g).max())


def task_config(name) -> tk.TaskConfig:
    spec = TASK_CASES[name]
    kw = dict(spec["cfg"])
    if "randomization" in spec:
        kw["randomization"] = wd.RandomizationSpec(**spec["randomization"])
    if "lidar" in spec:
        n_az, n_el = spec["lidar"]
        kw["lidar"] = sn.LidarPattern(n_azimuth=n_az, n_elevation=n_el)
    return tk.TaskConfig(**kw)


def _to_pkg_scene(s):
    prims = sn.PrimitiveSet(spheres=s.prims.get("spheres", np.zeros((0, 4))),
                            boxes=s.prims.get("boxes", np.zeros((0, 6))),
                            cylinders=s.prims.get("cylinders", np.zeros((0, 5))),
                            ground_z=s.prims.get("ground_z"))
    gates = [wd.Gate(center=c, normal=n, inner_radius=i, frame_width=f) for (c, n, i, f) in s.gates]
    return wd.Scene(prims=prims, bounds_lo=s.bounds_lo, bounds_hi=s.bounds_hi, spawn=s.spawn, goal=s.goal,
                    gates=gates)


class FixtureReplay:
    """reset_source that hands back the fixture's post-reset rows."""

    def __init__(self, z, n_agents, dr=False):
        self.z = z
        self.na = n_agents
        self.dr = dr
        self.t = 0  # index of the fixture state the next reset lands in

    def __call__(self, env_ids, counter, initial):
        z, na = self.z, self.na
        i = 0 if initial else self.t
        rows = (np.asarray(env_ids)[:, None] * na + np.arange(na)[None]).reshape(-1)
        d = {"p": z[f"s{i}_p"][rows], "v": z[f"s{i}_v"][rows], "goal": z[f"goals{i}"][rows],
             "v_ema": z[f"v_ema{i}"][rows]}
        if self.dr:
            d["dr"] = z[f"dr{i}"][rows]
        return d


def build_env(name, device="cuda"):
    z = load(f"task_{name}")
    cfg = task_config(name)
    scene_source = None
    if "scenes_json" in z:
        scenes = [_to_pkg_scene(scene_from_json(s)) for s in z["scenes_json"]]
        scene_source = lambda seed, n: scenes  # noqa: E731
    rep = FixtureReplay(z, cfg.n_agents, dr=cfg.randomization is not None)
    env = tk.make_task(cfg, device=device, reset_source=rep, scene_source=scene_source)
    out0 = env.reset(int(z["seed"]))
    if "teleport_p" in z:
        env.state = env.model.init_state(z["teleport_p"], z["teleport_v"])
        out0 = tk.StepOutput(obs=env.observe(), r_ctrl=out0.r_ctrl, r_goal=out0.r_goal, r_rl=out0.r_rl,
                             terminated=out0.terminated, truncated=out0.truncated)
    return env, z, rep, out0


def replay(name, device="cuda", with_grad=True):
    """Run the fixture's actions through the GPU env; returns per-step records."""
    env, z, rep, out0 = build_env(name, device)
    T = int(z["T"])
    raw = torch.as_tensor(z["raw"], dtype=torch.float32, device=device)
    leaves = [raw[t].clone().requires_grad_(with_grad) for t in range(T)]
    env.detach_states()
    recs = []
    loss = 0.0
    for t in range(T):
        rep.t = t + 1
        out = env.step(leaves[t])
        loss = loss + out.r_ctrl.mean() * (0.99 ** t)
        rec = {"proprio": out.obs.proprio.detach().cpu().numpy(), "r_ctrl": out.r_ctrl.detach().cpu().numpy(),
               "r_goal": out.r_goal.cpu().numpy(), "r_rl": out.r_rl.cpu().numpy(),
               "term": out.terminated.cpu().numpy(), "trunc": out.truncated.cpu().numpy(),
               "state": {k: v.detach().cpu().numpy() for k, v in env.state.fields().items()},
               "goals": env.goals.cpu().numpy(), "v_ema": env.v_ema.cpu().numpy(),
               "steps": env.steps_in_episode.cpu().numpy()}
        if out.obs.visual is not None:
            rec["visual"] = out.obs.visual.detach().cpu().numpy()
        recs.append(rec)
    loss = -loss / T
    grad = None
    if with_grad:
        grads = torch.autograd.grad(loss, leaves, allow_unused=True)
        grad = np.stack([g.cpu().numpy() if g is not None else np.zeros(leaves[0].shape) for g in grads])
    return env, z, recs, float(loss.detach()), grad, out0
