"""Generate golden fixtures by running the REAL reference (dev container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (``/root/reference/pkg/src/quadsim``) is pure Python/numpy and
importable here but does not exist on the GPU box, so its outputs are committed
as small ``.npz`` fixtures next to this script.  Every fixture is fp64.
Re-running this script reproduces the committed files bit for bit (all inputs
are seeded).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from quadsim import autodiff as ad  # noqa: E402
from quadsim import dynamics as dyn  # noqa: E402
from quadsim import sensors as sn  # noqa: E402
from quadsim import tasks as tk  # noqa: E402
from quadsim import world as wd  # noqa: E402
from quadsim.autodiff import Tape, Var  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)/1024:.1f} KiB)")


# ---------------------------------------------------------------------------
# dynamics: 3 models, random states/actions, T steps + rollout_grad


def gen_dynamics():
    out = {}
    rng = np.random.default_rng(100)
    B, T = 16, 8
    for name in ("full", "pm_continuous", "pm_discrete", "simplified"):
        for variant in ("default", "drag"):
            if variant == "drag" and name in ("pm_discrete", "simplified"):
                continue
            kw = {}
            if variant == "drag":
                if name == "full":
                    kw["drag_matrix_diag"] = np.array([0.3, 0.25, 0.5])
                else:
                    kw["drag_coeff"] = rng.uniform(0.1, 0.5, size=B)
                    kw["latency"] = rng.uniform(2.0, 8.0, size=B)
            params = dyn.QuadParams(dt=0.02, **kw)
            model = dyn.make_model(name, params)
            st = model.init_state(rng.normal(size=(B, 3)), rng.normal(size=(B, 3)) * 0.5)
            if name == "full":
                q = rng.normal(size=(B, 4))
                q /= np.linalg.norm(q, axis=-1, keepdims=True)
                st = dyn.QuadState(p=st.p, v=st.v, q=Var(q), w=Var(rng.normal(size=(B, 3))))
            elif name == "pm_continuous":
                st = dyn.QuadState(p=st.p, v=st.v, a_lat=Var(rng.normal(size=(B, 3)) * 3))
            elif name == "simplified":
                q = rng.normal(size=(B, 4))
                q /= np.linalg.norm(q, axis=-1, keepdims=True)
                st = dyn.QuadState(p=st.p, v=st.v, R=Var(dyn.quat_to_matrix_np(q)))
            else:
                st = dyn.QuadState(p=st.p, v=st.v, u_prev=Var(rng.normal(size=(B, 3))))
            raw = rng.normal(size=(T, B, model.action_dim)) * 0.7
            key = f"{name}_{variant}"
            for k, v in st.values().items():
                out[f"{key}/s0_{k}"] = v
            out[f"{key}/raw"] = raw
            if variant == "drag":
                if name == "full":
                    out[f"{key}/drag_diag"] = params.drag_matrix_diag
                else:
                    out[f"{key}/drag_coeff"] = np.asarray(params.drag_coeff)
                    out[f"{key}/latency"] = np.asarray(params.latency)
            lo, hi = model.action_box()
            s = st
            for t in range(T):
                s = model.step(s, dyn.action_squash(Var(raw[t]), lo, hi))
                for k, v in s.values().items():
                    out[f"{key}/s{t+1}_{k}"] = v
            # tape gradient through the squashed rollout (dynamics-level BPTT)
            for (t1, t2) in ((0, T), (3, T), (T - 1, T)):
                g = dyn.rollout_grad(model, st, raw, t1, t2, squash=True)
                out[f"{key}/rgrad_{t1}_{t2}"] = g.grad
    save("dynamics", **out)


# ---------------------------------------------------------------------------
# task trajectories with tape gradients


TASK_CASES = {
    # C1 shape (scaled down for the fixture): pm position, 32-step window
    "pos_pmc": dict(cfg=dict(task="position", dynamics="pm_continuous", n_envs=64, episode_len=10),
                    T=32, scale=0.3, seed=1),
    "pos_pmd": dict(cfg=dict(task="position", dynamics="pm_discrete", n_envs=64, episode_len=10),
                    T=32, scale=0.3, seed=1),
    "pos_full": dict(cfg=dict(task="position", dynamics="full", n_envs=32, episode_len=7),
                     T=16, scale=0.3, seed=2),
    "pos_pmc_dr": dict(cfg=dict(task="position", dynamics="pm_continuous", n_envs=16, episode_len=6,
                                randomization=wd.RandomizationSpec(action_scale=(0.7, 1.0))),
                       T=16, scale=0.5, seed=3),
    "pos_form": dict(cfg=dict(task="position", dynamics="pm_continuous", n_envs=8, n_agents=3,
                              episode_len=9, formation="line"),
                     T=12, scale=0.4, seed=4),
    "avoid_depth": dict(cfg=dict(task="avoidance", dynamics="pm_continuous", n_envs=6, episode_len=8,
                                 sensor="depth", density=0.12),
                        T=12, scale=0.6, seed=5),
    "avoid_lidar_indoor": dict(cfg=dict(task="avoidance", dynamics="full", n_envs=4, episode_len=6,
                                        sensor="lidar", style="indoor", density=0.12,
                                        lidar=sn.LidarPattern(n_azimuth=24, n_elevation=3)),
                               T=8, scale=0.4, seed=6),
    "avoid_form": dict(cfg=dict(task="avoidance", dynamics="pm_discrete", n_envs=4, n_agents=2,
                                episode_len=7, density=0.1, formation="line", formation_side=1.5),
                       T=8, scale=0.5, seed=7),
    "racing": dict(cfg=dict(task="racing", dynamics="pm_continuous", n_envs=8, episode_len=30,
                            n_gates=3, gate_spread=6.0),
                   T=14, scale=0.2, seed=8, teleport="gates"),
    # success / bounds events: some envs start hovering on their goal, some
    # leave the arena (q/tasks.py:639-650, 734-737)
    "pos_events": dict(cfg=dict(task="position", dynamics="pm_continuous", n_envs=24, episode_len=20),
                       T=10, scale=0.1, seed=9, teleport="goal_bounds"),
    "pos_full_events": dict(cfg=dict(task="position", dynamics="full", n_envs=16, episode_len=20),
                            T=8, scale=0.1, seed=10, teleport="goal_bounds"),
    # collisions: quads launched at their nearest obstacle (q/tasks.py:823)
    "avoid_collide": dict(cfg=dict(task="avoidance", dynamics="pm_continuous", n_envs=6, episode_len=20,
                                   density=0.2),
                          T=10, scale=0.1, seed=11, teleport="obstacle"),
    # simplified quadrotor, with resets and success/bounds events
    "pos_simp": dict(cfg=dict(task="position", dynamics="simplified", n_envs=24, episode_len=7),
                     T=16, scale=0.3, seed=12, teleport="goal_bounds"),
}


def _state_arrays(env):
    return {k: v.copy() for k, v in env.state.values().items()}


def _redraw_without_aliasing(self, env_mask):
    """q/tasks.py:377-387 with copy-before-write.

    The stock method writes the new draws into ``_dr_drag`` in place; that
    array is aliased by ``params.drag_coeff`` and so by every earlier step's
    tape closure (q/dynamics.py:252, q/tasks.py:366-368), which makes the tape
    gradient of pre-reset steps use the post-reset drag.  This variant only
    breaks the alias; the forward values are unchanged.
    """
    self._dr_drag = self._dr_drag.copy()
    self._dr_latency = self._dr_latency.copy()
    self._dr_scale = self._dr_scale.copy()
    _STOCK_REDRAW(self, env_mask)


_STOCK_REDRAW = tk.FlightTask._redraw_randomization


def gen_task(name, spec):
    rec = _gen_task(name, spec)
    if spec["cfg"].get("randomization") is not None:
        tk.FlightTask._redraw_randomization = _redraw_without_aliasing
        try:
            fixed = _gen_task(name, spec)
        finally:
            tk.FlightTask._redraw_randomization = _STOCK_REDRAW
        for k in rec:
            if k not in ("grad", "loss"):
                assert np.array_equal(rec[k], fixed[k]), k
        rec["grad_unaliased"] = fixed["grad"]
    save(f"task_{name}", **rec)


def _gen_task(name, spec):
    cfg = tk.TaskConfig(**spec["cfg"])
    env = tk.make_task(cfg)
    out0 = env.reset(seed=spec["seed"])
    rec = {}
    rec["seed"] = np.array(spec["seed"])
    rec["T"] = np.array(spec["T"])
    if cfg.task in ("avoidance", "racing"):
        per_env = [s.to_json() for s in env.scenes]
        rec["scenes_json"] = np.array(per_env)
    if spec.get("teleport") == "goal_bounds":
        p = env.state.p.value.copy()
        v = env.state.v.value.copy()
        k = env.N // 3
        p[:k] = env.goals[:k] + 0.05
        v[:k] = 0.02
        hi = env.bounds_hi_per_row[k:2 * k]
        p[k:2 * k] = hi - 0.05
        v[k:2 * k] = 3.0
        st = env.model.init_state(p, v)
        env.state = st
        rec["teleport_p"], rec["teleport_v"] = p, v
        out0 = tk.StepOutput(obs=env.observe(), r_ctrl=out0.r_ctrl, r_goal=out0.r_goal,
                             r_rl=out0.r_rl, terminated=out0.terminated, truncated=out0.truncated)
    if spec.get("teleport") == "obstacle":
        p = env.state.p.value.copy()
        v = env.state.v.value.copy()
        for e in range(env.N):
            sp = env.prims.spheres[e][env.prims.sph_valid[e]]
            if len(sp):
                c, r = sp[0, :3], sp[0, 3]
                p[e] = c - np.array([r + 0.45, 0.0, 0.0])
                v[e] = np.array([3.0, 0.0, 0.0])
        st = env.model.init_state(p, v)
        env.state = st
        rec["teleport_p"], rec["teleport_v"] = p, v
        out0 = tk.StepOutput(obs=env.observe(), r_ctrl=out0.r_ctrl, r_goal=out0.r_goal,
                             r_rl=out0.r_rl, terminated=out0.terminated, truncated=out0.truncated)
    if spec.get("teleport") == "gates":
        # put each quad just before its first gate, flying through it:
        # lateral offsets span pass / crash / miss (q/tasks.py:937-961)
        c0 = env.gate_centers[:, 0]
        n0 = env.gate_normals[:, 0]
        lat = np.stack([-n0[:, 1], n0[:, 0], np.zeros(env.N)], axis=-1)
        offs = np.array([0.0, 0.3, 0.7, 0.85, 0.95, 1.05, 1.3, 0.5])[: env.N]
        p = c0 - n0 * 0.4 + lat * offs[:, None]
        v = n0 * 4.0
        st = env.model.init_state(p, v)
        env.state = st
        rec["teleport_p"] = p
        rec["teleport_v"] = v
        out0 = tk.StepOutput(obs=env.observe(), r_ctrl=out0.r_ctrl, r_goal=out0.r_goal,
                             r_rl=out0.r_rl, terminated=out0.terminated, truncated=out0.truncated)
    for k, v in _state_arrays(env).items():
        rec[f"s0_{k}"] = v
    rec["goals0"] = env.goals.copy()
    rec["v_ema0"] = env.v_ema.copy()
    rec["proprio0"] = out0.obs.proprio.value.copy()
    if out0.obs.visual is not None:
        rec["visual0"] = out0.obs.visual.copy()
    if cfg.randomization is not None:
        rec["dr0"] = np.stack([env._dr_drag, env._dr_latency, env._dr_scale], axis=-1).copy()
    if cfg.task == "racing":
        rec["next_gate0"] = env.next_gate.copy()
    rng = np.random.default_rng(1000 + spec["seed"])
    T = spec["T"]
    raw = rng.normal(size=(T, env.N, env.action_dim)) * spec["scale"]
    rec["raw"] = raw
    tape = Tape()
    leaves = [tape.leaf(raw[t].copy()) for t in range(T)]
    env.detach_states()
    disc = None
    for t in range(T):
        out = env.step(leaves[t])
        term = ad.mul(ad.vmean(out.r_ctrl), 0.99 ** t)
        disc = term if disc is None else ad.add(disc, term)
        rec[f"proprio{t+1}"] = out.obs.proprio.value.copy()
        if out.obs.visual is not None:
            rec[f"visual{t+1}"] = np.asarray(out.obs.visual).copy()
        rec[f"r_ctrl{t+1}"] = out.r_ctrl.value.copy()
        rec[f"r_goal{t+1}"] = out.r_goal.copy()
        rec[f"r_rl{t+1}"] = out.r_rl.copy()
        rec[f"term{t+1}"] = out.terminated.copy()
        rec[f"trunc{t+1}"] = out.truncated.copy()
        for k, v in _state_arrays(env).items():
            rec[f"s{t+1}_{k}"] = v
        rec[f"goals{t+1}"] = env.goals.copy()
        rec[f"v_ema{t+1}"] = env.v_ema.copy()
        rec[f"steps{t+1}"] = env.steps_in_episode.copy()
        if cfg.randomization is not None:
            rec[f"dr{t+1}"] = np.stack([env._dr_drag, env._dr_latency, env._dr_scale], axis=-1).copy()
        if cfg.task == "racing":
            rec[f"next_gate{t+1}"] = env.next_gate.copy()
    loss = ad.neg(ad.mul(disc, 1.0 / T))
    grads = tape.backward(loss)
    rec["loss"] = np.array(loss.value)
    rec["grad"] = np.stack([grads[l] for l in leaves])
    rec["stats"] = np.array([env.finished_episodes, env.successful_episodes, env.collision_episodes,
                             env.finished_return])
    return rec


# ---------------------------------------------------------------------------
# ray casting, culling, sdf


def _random_scene(rng, n=8, extent=8.0, ground_p=0.5):
    """Same distribution as pkg/tests/test_sensors.py:22-41."""
    spheres = np.column_stack([rng.uniform(-extent, extent, size=(n, 2)), rng.uniform(0.0, 4.0, size=n),
                               rng.uniform(0.3, 1.0, size=n)])
    boxes = np.column_stack([rng.uniform(-extent, extent, size=(n, 2)), rng.uniform(0.0, 4.0, size=n),
                             rng.uniform(0.2, 1.0, size=(n, 3))])
    cyls = np.column_stack([rng.uniform(-extent, extent, size=(n, 2)), rng.uniform(0.0, 4.0, size=n),
                            rng.uniform(0.2, 0.6, size=n), rng.uniform(0.5, 2.0, size=n)])
    ground = -1.0 if rng.uniform() < ground_p else None
    return sn.PrimitiveSet(spheres=spheres, boxes=boxes, cylinders=cyls, ground_z=ground)


def gen_sensors():
    rng = np.random.default_rng(200)
    B = 12
    sets = []
    for i in range(B):
        s = _random_scene(rng, n=int(rng.integers(1, 9)))
        # ragged: drop some types entirely in a few envs
        if i % 5 == 1:
            s = sn.PrimitiveSet(spheres=s.spheres, ground_z=s.ground_z)
        if i % 5 == 3:
            s = sn.PrimitiveSet(boxes=s.boxes, cylinders=s.cylinders, ground_z=0.0)
        sets.append(s)
    sets.append(sn.PrimitiveSet())  # empty scene, no ground
    B = len(sets)
    prims = sn.pack_primitives(sets)
    pos = np.column_stack([rng.uniform(-4, 4, size=(B, 2)), rng.uniform(0.2, 3.0, size=B)])
    yaw = rng.uniform(0, 2 * np.pi, size=B)
    R = tk.rotz_np(yaw)
    rec = {"pos": pos, "yaw": yaw}
    for k in ("spheres", "sph_valid", "boxes", "box_valid", "cylinders", "cyl_valid", "ground_z"):
        rec[f"prims_{k}"] = getattr(prims, k)
    cam = sn.CameraIntrinsics(width=32, height=24, max_range=10.0)
    rec["depth_cull"] = sn.render_depth(prims, pos, R, cam, cull=True)
    rec["depth_nocull"] = sn.render_depth(prims, pos, R, cam, cull=False)
    cam9 = sn.CameraIntrinsics(width=16, height=9, max_range=7.0)  # has dz==0 rows
    rec["depth_16x9"] = sn.render_depth(prims, pos, R, cam9)
    lid = sn.LidarPattern(n_azimuth=36, n_elevation=5, max_range=15.0)
    rec["lidar"] = sn.render_lidar(prims, pos, R, lid)
    # arbitrary (non-camera) unit rays incl. exact axis directions
    d = rng.normal(size=(B, 64, 3))
    d[:, :6] = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]])
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    rec["ray_dirs"] = d
    rec["ray_t"] = sn.raycast(prims, pos, d, 12.0)
    ks, kb, kc = sn.fov_cull(prims, pos, R, cam)
    rec["cull_s"], rec["cull_b"], rec["cull_c"] = ks, kb, kc
    # sdf at random points + on-surface-ish points
    pts = np.column_stack([rng.uniform(-8, 8, size=(B, 2)), rng.uniform(-0.5, 4.0, size=B)])
    rec["sdf_pts"] = pts
    rec["sdf"] = sn.sdf_np(pts, prims)
    tape = Tape()
    pv = tape.leaf(pts.copy())
    sv = sn.sdf_var(pv, prims)
    rec["sdf_var"] = sv.value
    rec["sdf_grad"] = tape.backward(ad.vsum(sv))[pv]
    # known answers (pkg/tests/test_sensors.py:50-71)
    rec["ka_sphere"] = np.array(sn.ray_primitive([0, 0, 0], [1, 0, 0], ("sphere", [5, 0, 0, 1])))
    rec["ka_box"] = np.array(sn.ray_primitive([0, 0, 0], [1, 0, 0], ("box", [2.5, 0, 0, 0.5, 1, 1])))
    rec["ka_cyl_side"] = np.array(sn.ray_primitive([0, 0, 0], [1, 0, 0], ("cylinder", [4, 0, 0, 1, 2])))
    rec["ka_cyl_cap"] = np.array(sn.ray_primitive([4, 0, 10], [0, 0, -1], ("cylinder", [4, 0, 0, 1, 2])))
    rec["ka_ground"] = np.array(sn.ray_primitive([0, 0, 2], [0, 0, -1], ("ground", -1.0)))
    # attitude reconstruction
    a = rng.normal(size=(64, 3)) * 4 + np.array([0, 0, 9.81])
    a[:4] = [[0, 0, 0], [1, 0, 0], [0, 0, 9.81], [0, 1e-7, 0]]
    ve = rng.normal(size=(64, 3))
    ve[4:8] = [[0, 0, 1], [1e-4, 0, 0], [0, 0, 0], [0, -1, 0]]
    rec["att_a"], rec["att_v"] = a, ve
    rec["att_R"] = sn.reconstruct_attitude(a, ve)
    save("sensors", **rec)


def gen_imu():
    rec = {}
    g = np.array([0.0, 0.0, -9.81])
    rng = np.random.default_rng(300)
    B, T = 8, 6
    imu = sn.ImuModel(batch=B, accel_noise_std=0.1, gyro_noise_std=0.01, accel_bias_rw_std=0.01,
                      gyro_bias_rw_std=0.001, seed=17)
    q = rng.normal(size=(B, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    R = dyn.quat_to_matrix_np(q)
    for t in range(T):
        w = rng.normal(size=(B, 3))
        vdot = rng.normal(size=(B, 3))
        a, gy = imu.read(R, w, vdot, g, 0.05)
        rec[f"w{t}"], rec[f"vdot{t}"], rec[f"accel{t}"], rec[f"gyro{t}"] = w, vdot, a, gy
        rec[f"ba{t}"], rec[f"bg{t}"] = imu.accel_bias.copy(), imu.gyro_bias.copy()
    rec["R"] = R
    save("imu", **rec)


def gen_world():
    rec = {}
    spawn = np.array([0.0, 0.0, 1.2])
    goal = np.array([8.0, 0.0, 1.5])
    for i, (seed, style, dens) in enumerate([(11, "outdoor", 0.1), (12, "indoor", 0.1), (13, "outdoor", 0.25)]):
        s = wd.gen_obstacle_course(seed, spawn, goal, dens, style=style)
        rec[f"scene{i}"] = np.array(s.to_json())
        rec[f"scene{i}_feasible"] = np.array(wd.grid_path_exists(s))
    t = wd.gen_race_track(21, 5, 10.0)
    rec["race"] = np.array(t.to_json())
    for kind in ("line", "square", "circle"):
        rec[f"form_{kind}"] = wd.formation_offsets(kind, 5, 2.0)
    spec = wd.RandomizationSpec()
    dr = wd.randomize_params(spec, 5, 3, n=10)
    rec["dr"] = np.stack([dr["drag_coeff"], dr["latency"], dr["action_scale"]], axis=-1)
    save("world", **rec)


def gen_learners():
    """TD-lambda targets (q/learners.py:78-113), the critic side of configs C5."""
    from quadsim import learners as ln

    rng = np.random.default_rng(400)
    T, N = 16, 32
    r = rng.normal(size=(T, N))
    values = rng.normal(size=(T, N))
    boot = rng.normal(size=N)
    done = rng.uniform(size=(T, N)) < 0.1
    rec = {"r": r, "values": values, "boot": boot, "done": done}
    rec["td"] = ln.td_lambda_targets(r, values, boot, done, 0.99, 0.95)
    rec["td_k4"] = ln.td_lambda_targets(r, values, boot, done, 0.99, 0.95, k=4)
    save("learners", **rec)


def gen_nets_ppo():
    """Networks (q/nets.py:85-274) through the weight container (:316-377), and
    the PPO pieces (q/learners.py:116-131, 345-385): GAE with cuts, advantage
    normalisation, running return-std reward scaling, tanh-squashed log-prob."""
    from quadsim import learners as ln
    from quadsim import nets

    rec = {}
    cdir = os.path.join(OUT, "nets_container")
    rng = np.random.default_rng([5 & 0x7FFFFFFF, 0x11])  # the learners' init stream
    arch_d = nets.PolicyArch(proprio_dim=9, action_dim=3,
                             visual={"kind": "depth", "height": 12, "width": 16, "max_range": 10.0},
                             recurrent=True, hidden=16, mlp=(32, 32), conv_feat=8,
                             input_scale=tuple(np.linspace(0.2, 1.0, 9)))
    pol_d = nets.PolicyNet(arch_d, rng)
    val = nets.ValueNet(13, rng, hidden=(32, 32), input_scale=tuple(np.linspace(0.5, 1.5, 13)))
    for k, v in pol_d.ps.arrays.items():
        rec["init_depth/" + k] = v.copy()
    for k, v in val.ps.arrays.items():
        rec["init_value/" + k] = v.copy()
    rng2 = np.random.default_rng(77)
    for ps in (pol_d.ps, val.ps):  # trained-looking weights (biases nonzero), then f32
        for k in ps.arrays:
            ps.arrays[k] = ps.arrays[k] + 0.1 * rng2.normal(size=ps.arrays[k].shape)
        ps.round_to_f32()
    arch_l = nets.PolicyArch(proprio_dim=12, action_dim=4, visual={"kind": "lidar", "rays": 24, "max_range": 20.0},
                             recurrent=False, hidden=16, mlp=(32, 32), conv_feat=8)
    pol_l = nets.PolicyNet(arch_l, np.random.default_rng(9))
    for k in pol_l.ps.arrays:
        pol_l.ps.arrays[k] = pol_l.ps.arrays[k] + 0.1 * rng2.normal(size=pol_l.ps.arrays[k].shape)
    pol_l.ps.round_to_f32()
    nets.save_container(cdir, {"policy": pol_d.ps, "value": val.ps, "policy_lidar": pol_l.ps},
                        {"note": "tests/golden/make_golden.py gen_nets_ppo"})
    B = 5
    pro = rng2.normal(size=(B, 9))
    img = rng2.uniform(0.0, 12.0, size=(B, 12, 16))
    h0 = rng2.normal(size=(B, 16)) * 0.5
    mu, ls, h1 = pol_d.forward(pol_d.ps.bind(None), Var(pro), img, Var(h0))
    rec.update({"d_pro": pro, "d_img": img, "d_h0": h0, "d_mu": mu.value, "d_ls": ls.value, "d_h1": h1.value})
    pro_l = rng2.normal(size=(B, 12))
    scan = rng2.uniform(0.0, 25.0, size=(B, 24))
    mu, ls, _ = pol_l.forward(pol_l.ps.bind(None), Var(pro_l), scan, None)
    rec.update({"l_pro": pro_l, "l_scan": scan, "l_mu": mu.value, "l_ls": ls.value})
    priv = rng2.normal(size=(B, 13))
    rec.update({"v_in": priv, "v_out": val.forward(val.ps.bind(None), priv).value})
    # PPO pieces
    T, N = 12, 16
    r = rng2.normal(size=(T, N))
    values = rng2.normal(size=(T, N))
    boot = rng2.normal(size=N)
    done = rng2.uniform(size=(T, N)) < 0.15
    adv, rets = ln.gae_advantages(r, values, boot, done, 0.99, 0.95)
    rec.update({"g_r": r, "g_values": values, "g_boot": boot, "g_done": done, "g_adv": adv, "g_rets": rets,
                "g_norm": ln.normalize(adv)})

    class _Stub:  # just the running return-std state of a PPO learner
        pass

    st = _Stub()
    st.opts = ln.LearnerOptions(algo="ppo", gamma=0.99)
    st._ret_trace, st._ret_count, st._ret_mean, st._ret_m2 = np.zeros(N), 1e-4, 0.0, 1.0
    for u in range(3):
        rw = rng2.normal(size=(T, N)) * (1.0 + u)
        dn = rng2.uniform(size=(T, N)) < 0.1
        rec[f"s_r{u}"], rec[f"s_done{u}"] = rw, dn
        rec[f"s_scaled{u}"] = ln.PPO._scale_rewards(st, rw, dn)
    mu = rng2.normal(size=(N, 3))
    logs = rng2.normal(size=(N, 3)) * 0.3 - 1.0
    a = mu + np.exp(logs) * rng2.normal(size=(N, 3))
    half = np.abs(rng2.normal(size=(N, 3))) + 1.0
    rec.update({"lp_mu": mu, "lp_logs": logs, "lp_a": a, "lp_half": half,
                "lp": ln.PPO._log_prob(st, Var(mu), Var(logs), Var(a), half).value})
    save("nets_ppo", **rec)
    # run artefacts (q/io.py): a trajectory dump and a metrics CSV of the same data
    from quadsim import io as qio

    N, S = 3, 2
    tw = qio.TrajectoryWriter(os.path.join(OUT, "trajectory.jsonl"), env_limit=2)
    io_rec = {}
    for step in range(S):
        states = {"p": rng2.normal(size=(N, 3)), "v": rng2.normal(size=(N, 3))}
        acts = rng2.normal(size=(N, 3))
        rc, rg = rng2.normal(size=N), np.array([0.0, 1.0, -1.0])
        term, trunc = np.array([0, 1, 2], dtype=np.int8), np.array([False, True, False])
        tw.write_step(step, states, acts, rc, rg, term, trunc)
        io_rec.update({f"t{step}_p": states["p"], f"t{step}_v": states["v"], f"t{step}_a": acts,
                       f"t{step}_rc": rc, f"t{step}_rg": rg, f"t{step}_term": term, f"t{step}_trunc": trunc})
    tw.close()
    mw = qio.MetricsWriter(os.path.join(OUT, "metrics.csv"))
    for u in range(3):
        mw.write({"update": u, "loss": float(rng2.normal()), "steps_per_sec": float(rng2.uniform() * 1e6)})
        io_rec[f"m{u}"] = np.array([u])
    mw.close()
    save("io_inputs", **io_rec)


# ---------------------------------------------------------------------------
# C1 at its exact shape: pm position task, 1,024 envs, reset(seed=1),
# raw = default_rng(0).normal(size=(32,1024,3))*0.3, episode_len 1e6,
# L = -(1/32) sum_t 0.99^t mean(r_ctrl_t) and dL/d(raw) through the tape.
# Per-step rewards and the gradient are stored as float32 (the GPU bars are
# 1e-5 / 1e-4, far above fp32 storage round-off), loss and states as fp64.


def gen_c1():
    raw = np.random.default_rng(0).normal(size=(32, 1024, 3)) * 0.3
    for name, short in (("pm_continuous", "pmc"), ("pm_discrete", "pmd")):
        cfg = tk.TaskConfig(task="position", dynamics=name, n_envs=1024, episode_len=10 ** 6)
        env = tk.make_task(cfg)
        env.reset(seed=1)
        rec = {}
        for k, v in _state_arrays(env).items():
            rec[f"s0_{k}"] = v
        rec["goals0"] = env.goals.copy()
        tape = Tape()
        leaves = [tape.leaf(raw[t].copy()) for t in range(32)]
        env.detach_states()
        disc = None
        r_ctrl, r_rl, term = [], [], []
        for t in range(32):
            out = env.step(leaves[t])
            term_ = ad.mul(ad.vmean(out.r_ctrl), 0.99 ** t)
            disc = term_ if disc is None else ad.add(disc, term_)
            r_ctrl.append(out.r_ctrl.value.copy())
            r_rl.append(out.r_rl.copy())
            term.append(out.terminated.copy())
            if t == 15:
                for k, v in _state_arrays(env).items():
                    rec[f"s16_{k}"] = v
        loss = ad.neg(ad.mul(disc, 1.0 / 32))
        grads = tape.backward(loss)
        for k, v in _state_arrays(env).items():
            rec[f"s32_{k}"] = v
        rec["goals32"] = env.goals.copy()
        rec["loss"] = np.array(loss.value)
        rec["grad"] = np.stack([grads[l] for l in leaves]).astype(np.float32)
        rec["r_ctrl"] = np.stack(r_ctrl).astype(np.float32)
        rec["r_rl"] = np.stack(r_rl).astype(np.float32)
        rec["term"] = np.stack(term)
        rec["stats"] = np.array([env.finished_episodes, env.successful_episodes, env.collision_episodes,
                                 env.finished_return])
        save(f"c1_{short}", **rec)


# ---------------------------------------------------------------------------
# wire / disk formats written by the reference: Scene JSON v1
# (q/world.py:72-111) for an outdoor course, an indoor course and a race
# track, and DAIM depth / LiDAR dumps (q/sensors.py:614-642)


def gen_formats():
    import json

    scenes = [wd.gen_obstacle_course(41, np.array([0.0, 0.0, 1.2]), np.array([8.0, 0.0, 1.5]), 0.12),
              wd.gen_obstacle_course(42, np.array([0.0, 0.0, 1.2]), np.array([8.0, 0.0, 1.5]), 0.1, style="indoor"),
              wd.gen_race_track(43, 5, 10.0)]
    with open(os.path.join(OUT, "scenes_v1.json"), "w") as f:
        json.dump([s.to_json() for s in scenes], f)
    prims = sn.pack_primitives([scenes[0].prims])
    R = np.eye(3)[None]
    depth = sn.render_depth(prims, np.array([[0.5, 0.2, 1.2]]), R, sn.CameraIntrinsics(width=64, height=48))
    sn.write_depth_dump(os.path.join(OUT, "depth_64x48.daim"), depth[0], frame_index=7)
    lidar = sn.render_lidar(prims, np.array([[0.5, 0.2, 1.2]]), R, sn.LidarPattern(n_azimuth=36, n_elevation=4))
    sn.write_depth_dump(os.path.join(OUT, "lidar_36x4.daim"), lidar[0], frame_index=3)
    np.savez_compressed(os.path.join(OUT, "formats.npz"), depth=depth[0], lidar=lidar[0])
    print("wrote scenes_v1.json, depth_64x48.daim, lidar_36x4.daim, formats.npz")


if __name__ == "__main__":
    which = sys.argv[1:] or ["dynamics", "sensors", "imu", "world", "tasks", "learners", "nets_ppo", "c1", "formats"]
    if "nets_ppo" in which:
        gen_nets_ppo()
    if "c1" in which:
        gen_c1()
    if "formats" in which:
        gen_formats()
    if "learners" in which:
        gen_learners()
    if "dynamics" in which:
        gen_dynamics()
    if "sensors" in which:
        gen_sensors()
    if "imu" in which:
        gen_imu()
    if "world" in which:
        gen_world()
    if "tasks" in which:
        for name, spec in TASK_CASES.items():
            gen_task(name, spec)
