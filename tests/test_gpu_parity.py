"""GPU parity: the sm_100a kernels against the reference's golden fixtures and
the CPU oracle.  Tolerances are the north star's (BASELINE.json): state and
rewards 1e-5 relative (floored at 1), depth 1e-4 m, BPTT gradients 1e-4
max-normalised, masks / termination codes / reset indices exact.
"""

import numpy as np
import pytest
import torch

from golden_utils import STATE_KEYS, TASK_CASES, load
from gpu_harness import DEPTH_TOL, GRAD_TOL, STATE_TOL, grad_err, replay, state_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qs():
    import paper_2509_10247_b200 as qs

    assert qs._lib.lib().qs_abi_version() == 1
    return qs


# ---------------------------------------------------------------------------
# dynamics models (q/dynamics.py:140-274) + rollout_grad (:481-520)


@pytest.mark.parametrize("key", ["full_default", "full_drag", "pm_continuous_default",
                                 "pm_continuous_drag", "pm_discrete_default", "simplified_default"])
def test_dynamics_kernels_match_reference(qs, key):
    z = load("dynamics")
    model_name = key.rsplit("_", 1)[0]
    kw = {}
    if f"{key}/drag_diag" in z:
        kw["drag_matrix_diag"] = z[f"{key}/drag_diag"]
    if f"{key}/drag_coeff" in z:
        kw["drag_coeff"] = z[f"{key}/drag_coeff"]
        kw["latency"] = z[f"{key}/latency"]
    model = qs.make_model(model_name, qs.QuadParams(dt=0.02, **kw))
    fields = {k: torch.as_tensor(z[f"{key}/s0_{k}"], dtype=torch.float32, device="cuda")
              for k in STATE_KEYS[model_name]}
    st = qs.QuadState(**fields)
    raw = z[f"{key}/raw"]
    lo, hi = model.action_box()
    for t in range(raw.shape[0]):
        act = qs.dynamics.action_squash(torch.as_tensor(raw[t], dtype=torch.float32, device="cuda"), lo, hi)
        st = model.step(st, act)
        for k in STATE_KEYS[model_name]:
            err = state_err(getattr(st, k).cpu().numpy(), z[f"{key}/s{t+1}_{k}"])
            assert err < 2 * STATE_TOL, (t, k, err)
    T = raw.shape[0]
    st0 = qs.QuadState(**fields)
    for (t1, t2) in ((0, T), (3, T), (T - 1, T)):
        g = qs.rollout_grad(model, st0, raw, t1, t2, squash=True).grad.cpu().numpy()
        assert grad_err(g, z[f"{key}/rgrad_{t1}_{t2}"]) < GRAD_TOL, (t1, t2)


# ---------------------------------------------------------------------------
# full env step against the reference trajectories (injected resets)


@pytest.mark.parametrize("name", list(TASK_CASES))
def test_task_trajectory_and_bptt_gradient(qs, name):
    env, z, recs, loss, grad, out0 = replay(name)
    model = env.config.dynamics
    assert state_err(out0.obs.proprio.detach().cpu().numpy(), z["proprio0"]) < STATE_TOL
    worst = {}
    for t, r in enumerate(recs):
        i = t + 1
        # exact: termination codes, truncation, reset indices (steps counter)
        assert np.array_equal(r["term"], z[f"term{i}"]), (t, r["term"], z[f"term{i}"])
        assert np.array_equal(r["trunc"], z[f"trunc{i}"]), t
        assert np.array_equal(r["steps"], z[f"steps{i}"]), t
        assert np.array_equal(r["r_goal"], z[f"r_goal{i}"]), t
        for k in ("proprio", "r_ctrl", "r_rl", "goals", "v_ema"):
            ref = z[{"proprio": f"proprio{i}", "r_ctrl": f"r_ctrl{i}", "r_rl": f"r_rl{i}",
                     "goals": f"goals{i}", "v_ema": f"v_ema{i}"}[k]]
            worst[k] = max(worst.get(k, 0.0), state_err(r[k], ref))
        for k in STATE_KEYS[model]:
            worst["s_" + k] = max(worst.get("s_" + k, 0.0), state_err(r["state"][k], z[f"s{i}_{k}"]))
        if "visual" in r:
            d = np.abs(r["visual"].astype(np.float64) - z[f"visual{i}"]).max()
            worst["visual"] = max(worst.get("visual", 0.0), d)
    # free-running: errors compound over the window, so the state/reward bar
    # is 5x the single-step 1e-5 (the teacher-forced twin below holds every
    # step to 1e-5 itself)
    print(f"\n{name} free-running: " + ", ".join(f"{k} {v:.2e}" for k, v in sorted(worst.items())))
    for k, v in worst.items():
        tol = DEPTH_TOL if k == "visual" else 5 * STATE_TOL
        assert v < tol, (k, v, worst)
    g_ref = z["grad_unaliased"] if "grad_unaliased" in z else z["grad"]
    assert abs(loss - float(z["loss"])) <= 1e-5 * max(1.0, abs(float(z["loss"])))
    if np.abs(g_ref).max() > 0:
        assert grad_err(grad, g_ref) < GRAD_TOL, grad_err(grad, g_ref)
    stats = np.array([env.finished_episodes, env.successful_episodes, env.collision_episodes])
    assert np.array_equal(stats, z["stats"][:3].astype(int))
    assert abs(env.finished_return - z["stats"][3]) <= 1e-4 * max(1.0, abs(z["stats"][3]))


@pytest.mark.parametrize("name", list(TASK_CASES))
def test_task_teacher_forced_single_step(qs, name):
    """Every step of every reference trajectory as a single step: before step
    t the GPU env's carried state is overwritten with the reference's own
    state t (fp32-rounded): state planes, goals, v_ema, previous effort, DR
    draws, episode counters and next gate.  Step t's outputs must then match
    the reference's at the north star's 1e-5 (no compounding allowance);
    masks, codes, counters exact; depth within 1e-4 m."""
    from lockstep import set_gpu_carry
    from oracle import quadsim_oracle as O

    env, z, rep, _ = __import__("gpu_harness").build_env(name)
    model = env.config.dynamics
    T = int(z["T"])
    raw = z["raw"]
    na = env.n_agents
    lo, hi = O.action_box(model)
    center, half = (lo + hi) / 2, (hi - lo) / 2
    has_dr = "dr0" in z
    worst = {}
    for t in range(T):
        # previous effort entering step t: effort of step t-1 (q/tasks.py:568-570),
        # zero on rows that (re)spawned at the end of step t-1 or at reset
        if t == 0:
            peff = np.zeros((env.N, env.action_dim))
        else:
            scale = z[f"dr{t-1}"][:, 2:3] if has_dr else 1.0
            peff = half * scale * np.tanh(raw[t - 1])
            fresh = np.repeat(z[f"steps{t}"] == 0, na)
            peff[fresh] = 0.0
        st = {k: z[f"s{t}_{k}"] for k in STATE_KEYS[model]}
        steps = z[f"steps{t}"] if t > 0 else np.zeros(env.n_envs)
        set_gpu_carry(env, {k: np.float32(v) for k, v in st.items()}, np.float32(z[f"goals{t}"]),
                      np.float32(z[f"v_ema{t}"]), np.float32(peff), None, steps)
        if has_dr:
            d = z[f"dr{t}"]
            env._dr = torch.as_tensor(np.stack([d[:, 0], np.exp(-d[:, 1] * env.config.dt), d[:, 2], d[:, 1]], -1),
                                      dtype=torch.float32, device="cuda").contiguous()
        if env.config.task == "racing":
            env._meta[:, 3] = torch.as_tensor(z[f"next_gate{t}"], dtype=torch.int32, device="cuda")
        rep.t = t + 1
        out = env.step(torch.as_tensor(raw[t], dtype=torch.float32, device="cuda"))
        i = t + 1
        assert np.array_equal(out.terminated.cpu().numpy(), z[f"term{i}"]), t
        assert np.array_equal(out.truncated.cpu().numpy(), z[f"trunc{i}"]), t
        assert np.array_equal(out.r_goal.cpu().numpy(), z[f"r_goal{i}"]), t
        assert np.array_equal(env.steps_in_episode.cpu().numpy(), z[f"steps{i}"]), t
        errs = {"proprio": state_err(out.obs.proprio.detach().cpu().numpy(), z[f"proprio{i}"]),
                "r_ctrl": state_err(out.r_ctrl.detach().cpu().numpy(), z[f"r_ctrl{i}"]),
                "r_rl": state_err(out.r_rl.cpu().numpy(), z[f"r_rl{i}"]),
                "goals": state_err(env.goals.cpu().numpy(), z[f"goals{i}"]),
                "v_ema": state_err(env.v_ema.cpu().numpy(), z[f"v_ema{i}"])}
        for k, v in env.state.fields().items():
            errs["s_" + k] = state_err(v.detach().cpu().numpy(), z[f"s{i}_{k}"])
        if out.obs.visual is not None:
            errs["visual"] = float(np.abs(out.obs.visual.double().cpu().numpy() - z[f"visual{i}"]).max())
        for k, v in errs.items():
            worst[k] = max(worst.get(k, 0.0), v)
    print(f"\n{name} teacher-forced: " + ", ".join(f"{k} {v:.2e}" for k, v in sorted(worst.items())))
    for k, v in worst.items():
        assert v <= (DEPTH_TOL if k == "visual" else STATE_TOL), (k, v, worst)


# ---------------------------------------------------------------------------
# sensors (q/sensors.py:131-611)


def _prims(qs, z):
    return qs.sensors.BatchedPrimitives(z["prims_spheres"], z["prims_sph_valid"], z["prims_boxes"],
                                        z["prims_box_valid"], z["prims_cylinders"], z["prims_cyl_valid"],
                                        z["prims_ground_z"])


def test_render_depth_lidar_raycast_match_reference(qs):
    sn = qs.sensors
    z = load("sensors")
    prims = _prims(qs, z)
    pos = z["pos"]
    R = qs.tasks.rotz_np(z["yaw"])
    cam = sn.CameraIntrinsics(width=32, height=24, max_range=10.0)
    d_cull = sn.render_depth(prims, torch.as_tensor(pos, device="cuda"), R, cam, cull=True).cpu().numpy()
    d_nocull = sn.render_depth(prims, torch.as_tensor(pos, device="cuda"), R, cam, cull=False).cpu().numpy()
    assert np.array_equal(d_cull, d_nocull)  # culling never changes the image
    assert np.abs(d_cull - z["depth_cull"]).max() < DEPTH_TOL
    # hit/miss mask exact
    assert np.array_equal(d_cull < 10.0, z["depth_cull"] < 10.0)
    cam9 = sn.CameraIntrinsics(width=16, height=9, max_range=7.0)
    d9 = sn.render_depth(prims, torch.as_tensor(pos, device="cuda"), R, cam9).cpu().numpy()
    assert np.abs(d9 - z["depth_16x9"]).max() < DEPTH_TOL
    lid = sn.LidarPattern(n_azimuth=36, n_elevation=5, max_range=15.0)
    dl = sn.render_lidar(prims, torch.as_tensor(pos, device="cuda"), R, lid).cpu().numpy()
    assert np.abs(dl - z["lidar"]).max() < DEPTH_TOL
    assert np.array_equal(dl < 15.0, z["lidar"] < 15.0)
    tr = sn.raycast(prims, torch.as_tensor(pos, device="cuda"), z["ray_dirs"], 12.0).cpu().numpy()
    assert np.abs(tr - z["ray_t"]).max() < DEPTH_TOL


def test_known_answers_on_gpu(qs):
    sn = qs.sensors
    one = lambda **k: sn.PrimitiveSet(**k)  # noqa: E731
    o = torch.zeros(1, 3, device="cuda")
    ex = torch.tensor([[[1.0, 0.0, 0.0]]], device="cuda")
    assert sn.raycast(one(spheres=[[5, 0, 0, 1]]), o, ex, 20.0).item() == pytest.approx(4.0, abs=1e-5)
    assert sn.raycast(one(boxes=[[2.5, 0, 0, 0.5, 1, 1]]), o, ex, 20.0).item() == pytest.approx(2.0, abs=1e-5)
    assert sn.raycast(one(cylinders=[[4, 0, 0, 1, 2]]), o, ex, 20.0).item() == pytest.approx(3.0, abs=1e-5)
    o2 = torch.tensor([[4.0, 0.0, 10.0]], device="cuda")
    dn = torch.tensor([[[0.0, 0.0, -1.0]]], device="cuda")
    assert sn.raycast(one(cylinders=[[4, 0, 0, 1, 2]]), o2, dn, 20.0).item() == pytest.approx(8.0, abs=1e-5)
    o3 = torch.tensor([[0.0, 0.0, 2.0]], device="cuda")
    assert sn.raycast(one(ground_z=-1.0), o3, dn, 20.0).item() == pytest.approx(3.0, abs=1e-5)
    assert sn.raycast(one(ground_z=-1.0), o3, -dn, 20.0).item() == 20.0  # miss -> max range
    assert sn.raycast(one(), o3, -dn, 20.0).item() == 20.0  # empty scene


def test_sdf_and_gradient_match_reference(qs):
    sn = qs.sensors
    z = load("sensors")
    prims = _prims(qs, z)
    p = torch.as_tensor(z["sdf_pts"], dtype=torch.float32, device="cuda").requires_grad_(True)
    d = sn.sdf_var(p, prims)
    assert state_err(d.detach().cpu().numpy(), z["sdf_var"]) < STATE_TOL
    (g,) = torch.autograd.grad(d.sum(), p)
    assert np.abs(g.cpu().numpy() - z["sdf_grad"]).max() < 1e-4


def test_attitude_matches_reference(qs):
    z = load("sensors")
    R = qs.sensors.reconstruct_attitude(torch.as_tensor(z["att_a"], device="cuda"),
                                        torch.as_tensor(z["att_v"], device="cuda")).cpu().numpy()
    assert np.abs(R - z["att_R"]).max() < 1e-5


def test_imu_injected_noise_matches_reference(qs):
    z = load("imu")
    B = 8
    imu = qs.sensors.ImuModel(B, accel_noise_std=0.1, gyro_noise_std=0.01, accel_bias_rw_std=0.01,
                              gyro_bias_rw_std=0.001, seed=17)
    rng = np.random.default_rng(17)  # the reference's draw order (q/sensors.py:544-554)
    g = np.array([0.0, 0.0, -9.81])
    for t in range(6):
        noise = np.stack([rng.standard_normal((B, 3)) for _ in range(4)])
        a, w = imu.read(z["R"], z[f"w{t}"], z[f"vdot{t}"], g, 0.05, noise=noise)
        assert np.abs(a.cpu().numpy() - z[f"accel{t}"]).max() < 1e-5
        assert np.abs(w.cpu().numpy() - z[f"gyro{t}"]).max() < 1e-5


def test_imu_philox_statistics(qs):
    B = 100_000
    imu = qs.sensors.ImuModel(B, accel_noise_std=0.2, gyro_noise_std=0.05, seed=3)
    R = torch.eye(3, device="cuda").expand(B, 3, 3)
    z3 = torch.zeros(B, 3, device="cuda")
    a, w = imu.read(R, z3, z3, np.array([0.0, 0.0, -9.81]), 0.01)
    a = a.cpu().numpy() - np.array([0, 0, 9.81])
    w = w.cpu().numpy()
    assert abs(a.std() - 0.2) / 0.2 < 0.02 and abs(a.mean()) < 0.01
    assert abs(w.std() - 0.05) / 0.05 < 0.02
    # the 6 white-noise channels are uncorrelated, Gaussian-tailed (Box-Muller
    # pairs share a radius: cos/sin of one pair must still be uncorrelated)
    x = np.concatenate([a / 0.2, w / 0.05], axis=1)
    c = np.corrcoef(x.T)
    assert np.abs(c - np.eye(6)).max() < 0.015
    kurt = ((x - x.mean(0)) ** 4).mean(0) / x.var(0) ** 2
    assert np.all(np.abs(kurt - 3.0) < 0.1)
    assert (np.abs(x) > 3.0).mean() == pytest.approx(2.7e-3, rel=0.15)
    # bias random walks (the other 6 normals of the row-step)
    rw = qs.sensors.ImuModel(B, accel_bias_rw_std=1.0, gyro_bias_rw_std=1.0, seed=4)
    a_rw, w_rw = rw.read(R, z3, z3, np.array([0.0, 0.0, -9.81]), 0.01)
    y = np.concatenate([a_rw.cpu().numpy() - np.array([0, 0, 9.81]), w_rw.cpu().numpy()], axis=1) / 0.1
    assert np.all(np.abs(y.std(0) - 1.0) < 0.02) and np.abs(np.corrcoef(y.T) - np.eye(6)).max() < 0.015
    # deterministic given (seed, read index)
    imu2 = qs.sensors.ImuModel(B, accel_noise_std=0.2, gyro_noise_std=0.05, seed=3)
    a2, _ = imu2.read(R, z3, z3, np.array([0.0, 0.0, -9.81]), 0.01)
    assert np.array_equal(a2.cpu().numpy() - np.array([0, 0, 9.81]), a)


# ---------------------------------------------------------------------------
# native window engine == autograd path; Philox resets; in-kernel scenes


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("model", ["full", "pm_continuous", "pm_discrete"])
def test_window_engine_matches_autograd_path(qs, model, fused):
    from paper_2509_10247_b200.window import BpttWindow

    cfg = qs.TaskConfig(task="position", dynamics=model, n_envs=512, episode_len=9,
                        imu=qs.ImuSpec(0.1, 0.01, 0.01, 0.001))
    T = 12
    g = torch.Generator(device="cpu").manual_seed(0)
    acts = (torch.randn(T, 512, 4 if model == "full" else 3, generator=g) * 0.4).cuda()
    e1 = qs.make_task(cfg, strict=False)
    e1.reset(seed=5)
    e2 = qs.make_task(cfg, strict=False)
    e2.reset(seed=5)
    win = BpttWindow(e1, T, fused=fused)
    win.actions.copy_(acts)
    win.capture()
    loss_w, g_w = win.run()
    a = acts.clone().requires_grad_(True)
    tot = 0.0
    for t in range(T):
        tot = tot + e2.step(a[t]).r_ctrl.mean() * 0.99 ** t
    loss = -tot / T
    (ga,) = torch.autograd.grad(loss, a)
    assert abs(float(loss_w) - float(loss.detach())) < 1e-6 * max(1, abs(float(loss.detach())))
    assert grad_err(g_w.cpu().numpy(), ga.cpu().numpy()) < 1e-5
    win.sync_env()
    assert torch.allclose(e1._S, e2._S.detach(), rtol=1e-6, atol=1e-6)
    assert torch.equal(e1._meta, e2._meta)
    # resets happened (episode_len 9 < T) and stats agree
    assert e1.finished_episodes == e2.finished_episodes > 0


def test_pipelined_windows_match_sequential(qs):
    from paper_2509_10247_b200.window import BpttWindow

    cfg = qs.TaskConfig(task="position", dynamics="full", n_envs=1024, episode_len=20,
                        imu=qs.ImuSpec(0.1, 0.01, 0.01, 0.001))
    g = torch.Generator(device="cpu").manual_seed(3)
    batches = [(torch.randn(16, 1024, 4, generator=g) * 0.3).pin_memory() for _ in range(4)]
    e1 = qs.make_task(cfg, strict=False)
    e1.reset(seed=2)
    w1 = BpttWindow(e1, 16).capture()
    seq, seq_g = [], []
    for b in batches:
        loss, g1 = w1.run(b)
        seq.append(float(loss))
        seq_g.append(g1.cpu())
    e2 = qs.make_task(cfg, strict=False)
    e2.reset(seed=2)
    w2 = BpttWindow(e2, 16)
    grads = [torch.empty_like(b).pin_memory() for b in batches]
    pip = w2.run_pipelined(batches, grad_out=grads)
    np.testing.assert_allclose(pip, seq, rtol=1e-9)
    assert torch.equal(w1.S[0], w2.S[0])
    for a, b in zip(grads, seq_g):  # every window's downloaded gradient
        assert torch.equal(a, b)


def test_philox_resets_are_valid_and_deterministic(qs):
    cfg = qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=4096, episode_len=3)
    env = qs.make_task(cfg, strict=True)
    env.reset(seed=11)
    ext = cfg.goal_dist
    lo = np.array([-2.0, -ext - 2.0, 0.0]) + 0.8
    hi = np.array([ext + 2.0, ext + 2.0, 4.0]) - 0.8
    g = env.goals.cpu().numpy()
    assert np.all(g >= lo - 1e-5) and np.all(g <= hi + 1e-5)
    p = env.state.p.detach().cpu().numpy()
    d = np.linalg.norm(g - p, axis=-1)
    assert d.min() > 2.5 - 1.0 and d.max() < ext + 1.0  # spawn jitter N(0, 0.1^2) around the pair
    env2 = qs.make_task(cfg, strict=True)
    env2.reset(seed=11)
    assert torch.equal(env.goals, env2.goals) and torch.equal(env._S, env2._S)
    for _ in range(3):
        env.step(torch.zeros(env.N, 3, device="cuda"))
    assert env.finished_episodes == 4096  # truncation at episode_len
    assert bool((env.steps_in_episode == 0).all())
    assert not torch.equal(env.goals, env2.goals)  # re-spawned with the next episode key


def test_in_kernel_scene_generation_is_feasible(qs):
    from oracle import quadsim_oracle as O

    sc = qs.world.gen_obstacle_courses(7, 64, [0.0, 0.0, 1.2], [8.0, 0.0, 1.5], 0.25, style="indoor",
                                       device="cuda")
    scenes = qs.world.device_scene_to_scenes(sc, style="indoor")
    keep_min = 0.15 + 0.5
    for s in scenes:
        osc = O.Scene(prims={"spheres": s.prims.spheres, "boxes": s.prims.boxes,
                             "cylinders": s.prims.cylinders, "ground_z": 0.0},
                      bounds_lo=s.bounds_lo, bounds_hi=s.bounds_hi, spawn=s.spawn, goal=s.goal)
        assert O.grid_path_exists(osc)  # the oracle's own BFS agrees
        rand_boxes = s.prims.boxes[:-5]  # shell walls always kept
        pk = O.pack_primitives([{"spheres": s.prims.spheres, "boxes": rand_boxes,
                                 "cylinders": s.prims.cylinders}])
        ends = np.stack([s.spawn, s.goal])
        assert O.sdf_single_scene(ends, pk).min() > keep_min - 1e-4
        if len(s.prims.spheres):
            r = s.prims.spheres[:, 3]
            assert r.min() >= 0.3 - 1e-6 and r.max() <= 1.0 + 1e-6
        if len(s.prims.cylinders):
            assert np.allclose(s.prims.cylinders[:, 2], s.prims.cylinders[:, 4])  # trunks on the ground
    assert len(scenes[0].prims.boxes) >= 5  # indoor shell incl. ceiling


def test_avoidance_with_generated_scenes_and_depth_steps(qs):
    cfg = qs.TaskConfig(task="avoidance", dynamics="pm_continuous", n_envs=256, episode_len=20,
                        sensor="depth", depth_width=64, depth_height=48, density=0.3)
    env = qs.make_task(cfg)
    out = env.reset(seed=2)
    assert out.obs.visual.shape == (256, 48, 64)
    a = torch.zeros(256, 3, device="cuda", requires_grad=True)
    out = env.step(a)
    assert torch.isfinite(out.r_ctrl).all()
    out.r_ctrl.sum().backward()
    assert torch.isfinite(a.grad).all() and a.grad.abs().sum() > 0


PHILOX_KAT = [  # Random123 kat_vectors, philox4x32 10 rounds: ctr[4], key[2] -> out[4]
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


# Random123 kat_vectors, philox4x32 7 rounds (the IMU noise generator)
PHILOX7_KAT = [
    ([0, 0, 0, 0], [0, 0], [0x5F6FB709, 0x0D893F64, 0x4F121F81, 0x4F730A48]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0x4DFCCABA, 0x190A87F0, 0xC47362BA, 0xB6B5242A]),
]


def _philox_py(c, k, rounds=10):
    M = 0xFFFFFFFF
    c, k = list(c), list(k)
    for _ in range(rounds):
        p0, p1 = c[0] * 0xD2511F53, c[2] * 0xCD9E8D57
        c = [(p1 >> 32) ^ c[1] ^ k[0], p1 & M, (p0 >> 32) ^ c[3] ^ k[1], p0 & M]
        k = [(k[0] + 0x9E3779B9) & M, (k[1] + 0xBB67AE85) & M]
    return c


def test_philox_known_answers(qs):
    """The generator behind every in-kernel draw, both key-schedule forms,
    against the published Philox4x32-10 known-answer vectors."""
    from paper_2509_10247_b200 import _lib as L

    rng = np.random.default_rng(0)
    items = [c + k for c, k, _ in PHILOX_KAT]
    items += rng.integers(0, 2**32, size=(61, 6), dtype=np.uint64).tolist()
    ck = torch.tensor(np.array(items, dtype=np.uint32).view(np.int32), device="cuda")
    out = torch.empty(len(items), 8, dtype=torch.int32, device="cuda")
    L.check(L.lib().qs_philox4x32_10(len(items), L.ptr(ck), L.ptr(out), L.stream_handle()), "philox")
    got = out.cpu().numpy().view(np.uint32)
    for i, (c, k, want) in enumerate(PHILOX_KAT):
        assert got[i, :4].tolist() == want and got[i, 4:].tolist() == want
    for i, it in enumerate(items):
        want = _philox_py(it[:4], it[4:])
        assert got[i, :4].tolist() == want and got[i, 4:].tolist() == want
    # Philox4x32-7 (IMU noise): the published 7-round vectors and the same
    # restatement with seven rounds
    items7 = [c + k for c, k, _ in PHILOX7_KAT] + items
    ck7 = torch.tensor(np.array(items7, dtype=np.uint32).view(np.int32), device="cuda")
    out7 = torch.empty(len(items7), 8, dtype=torch.int32, device="cuda")
    L.check(L.lib().qs_philox4x32_7(len(items7), L.ptr(ck7), L.ptr(out7), L.stream_handle()), "philox7")
    got7 = out7.cpu().numpy().view(np.uint32)
    for i, (c, k, want) in enumerate(PHILOX7_KAT):
        assert got7[i, :4].tolist() == want
    for i, it in enumerate(items7):
        want = _philox_py(it[:4], it[4:], rounds=7)
        assert got7[i, :4].tolist() == want and got7[i, 4:].tolist() == want


@pytest.mark.parametrize("task,n_agents", [("position", 2), ("position", 3), ("avoidance", 4), ("position", 8)])
def test_multi_agent_window_matches_autograd_path(qs, task, n_agents):
    """Lane groups (one thread per agent row, env couplings as shuffles; 3 agents
    run in 4-lane groups with a padding lane): the fused window equals the
    per-step kernels + autograd, Philox resets included."""
    from paper_2509_10247_b200.window import BpttWindow

    cfg = qs.TaskConfig(task=task, dynamics="pm_continuous", n_envs=256, n_agents=n_agents, episode_len=7,
                        formation="line", formation_side=1.0, density=0.0)
    T = 10
    g = torch.Generator(device="cpu").manual_seed(1)
    acts = (torch.randn(T, 256 * n_agents, 3, generator=g) * 0.4).cuda()
    e1 = qs.make_task(cfg, strict=False)
    e1.reset(seed=3)
    e2 = qs.make_task(cfg, strict=False)
    e2.reset(seed=3)
    assert torch.equal(e1._S, e2._S)
    win = BpttWindow(e1, T)
    win.actions.copy_(acts)
    win.capture()
    loss_w, g_w = win.run()
    a = acts.clone().requires_grad_(True)
    tot = 0.0
    for t in range(T):
        tot = tot + e2.step(a[t]).r_ctrl.mean() * 0.99 ** t
    loss = -tot / T
    (ga,) = torch.autograd.grad(loss, a)
    assert abs(float(loss_w) - float(loss.detach())) < 1e-6 * max(1, abs(float(loss.detach())))
    assert grad_err(g_w.cpu().numpy(), ga.cpu().numpy()) < 1e-5
    win.sync_env()
    assert torch.allclose(e1._S, e2._S.detach(), rtol=1e-6, atol=1e-6)
    assert torch.equal(e1._meta, e2._meta)
    assert e1.finished_episodes == e2.finished_episodes > 0


@pytest.mark.parametrize("task", ["position", "avoidance"])
def test_multi_agent_philox_spawns_are_valid(qs, task):
    """Each lane draws its own agent's reset from the env's stream: formation
    offsets + jitter around one shared spawn, pairwise separation >= d_min
    (avoidance), deterministic per seed."""
    na, E = 4, 512
    cfg = qs.TaskConfig(task=task, dynamics="pm_continuous", n_envs=E, n_agents=na, formation="line",
                        formation_side=1.0, density=0.0)
    env = qs.make_task(cfg)
    env.reset(seed=9)
    p = env.state.p.detach().double().cpu().numpy().reshape(E, na, 3)
    gl = env.goals.double().cpu().numpy().reshape(E, na, 3)
    tmpl = env._template
    # goals are one shared goal + the formation template (exact up to fp32)
    np.testing.assert_allclose(gl - gl[:, :1], (tmpl - tmpl[0])[None].repeat(E, 0), atol=1e-5)
    # spawns: template + small jitter around one shared spawn point
    dev = p - (tmpl - tmpl[0])[None]
    assert np.abs(dev - dev[:, :1]).max() < 2.0
    if task == "avoidance":
        d = np.linalg.norm(p[:, :, None] - p[:, None, :], axis=-1) + np.eye(na)[None] * 1e9
        assert d.min() >= cfg.d_min - 1e-5
    env2 = qs.make_task(cfg)
    env2.reset(seed=9)
    assert torch.equal(env._S, env2._S) and torch.equal(env.goals, env2.goals)


@pytest.mark.parametrize("n_envs", [1, 77])
def test_window_ragged_batch_matches_autograd_path(qs, n_envs):
    """Batches that fill neither a warp nor a CTA: the tail CTA loads its
    actions without TMA, and tiny batches launch 32-thread CTAs."""
    from paper_2509_10247_b200.window import BpttWindow

    cfg = qs.TaskConfig(task="position", dynamics="full", n_envs=n_envs, episode_len=5,
                        imu=qs.ImuSpec(0.1, 0.01, 0.01, 0.001))
    T = 9
    g = torch.Generator(device="cpu").manual_seed(2)
    acts = (torch.randn(T, n_envs, 4, generator=g) * 0.4).cuda()
    e1 = qs.make_task(cfg, strict=False)
    e1.reset(seed=6)
    e2 = qs.make_task(cfg, strict=False)
    e2.reset(seed=6)
    win = BpttWindow(e1, T)
    win.actions.copy_(acts)
    win.capture()
    loss_w, g_w = win.run()
    a = acts.clone().requires_grad_(True)
    tot = 0.0
    for t in range(T):
        tot = tot + e2.step(a[t]).r_ctrl.mean() * 0.99 ** t
    loss = -tot / T
    (ga,) = torch.autograd.grad(loss, a)
    assert abs(float(loss_w) - float(loss.detach())) < 1e-6 * max(1, abs(float(loss.detach())))
    assert grad_err(g_w.cpu().numpy(), ga.cpu().numpy()) < 1e-5
    win.sync_env()
    assert torch.allclose(e1._S, e2._S.detach(), rtol=1e-6, atol=1e-6)
    assert torch.equal(e1._meta, e2._meta)


def test_window_graph_survives_env_reset(qs):
    """A captured BpttWindow whose env is reset re-loads the env's state and
    re-captures instead of replaying stale pointers; the result equals a fresh
    window on the reset env."""
    from paper_2509_10247_b200.window import BpttWindow

    cfg = qs.TaskConfig(task="position", dynamics="full", n_envs=1024, episode_len=20,
                        imu=qs.ImuSpec(0.1, 0.01, 0.01, 0.001))
    env = qs.make_task(cfg, strict=False)
    env.reset(seed=3)
    acts = torch.randn(8, env.N, 4, generator=torch.Generator().manual_seed(1)).cuda() * 0.3
    win = BpttWindow(env, 8)
    win.actions.copy_(acts)
    win.capture()
    win.run()
    env.reset(seed=4)
    loss_a, g_a = win.run()
    loss_a, g_a = float(loss_a), g_a.clone()
    env2 = qs.make_task(cfg, strict=False)
    env2.reset(seed=4)
    win2 = BpttWindow(env2, 8)
    win2.actions.copy_(acts)
    loss_b, g_b = win2.run()
    assert abs(loss_a - float(loss_b)) < 1e-9 * abs(float(loss_b))
    assert torch.equal(g_a, g_b)


@pytest.mark.parametrize("mode", ["pipelined", "eager"])
def test_window_survives_env_reset_pipelined_and_eager(qs, mode):
    """run_pipelined() and the eager (uncaptured) window
    also reload the env's state after env.reset() instead of replaying the
    pre-reset carry and stale env buffers."""
    from paper_2509_10247_b200.window import BpttWindow

    cfg = qs.TaskConfig(task="position", dynamics="full", n_envs=1024, episode_len=20,
                        imu=qs.ImuSpec(0.1, 0.01, 0.01, 0.001))
    acts = torch.randn(8, 1024, 4, generator=torch.Generator().manual_seed(1)) * 0.3
    host = acts.pin_memory()

    def go(win):
        if mode == "pipelined":
            return win.run_pipelined([host, host])[-1], win.g_actions.clone()
        win.run(acts.cuda())
        loss, g = win.run(acts.cuda())
        return float(loss), g.clone()

    env = qs.make_task(cfg, strict=False)
    env.reset(seed=3)
    win = BpttWindow(env, 8)
    go(win)
    env.reset(seed=4)
    la, ga = go(win)
    steps_a = env._meta.clone()
    env2 = qs.make_task(cfg, strict=False)
    env2.reset(seed=4)
    lb, gb = go(BpttWindow(env2, 8))
    assert la == lb
    assert torch.equal(ga, gb)
    assert torch.equal(steps_a, env2._meta)  # the window advanced the reset env's counters
