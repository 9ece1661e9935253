"""The reference's own known-answer and property tests, re-run against the
sm_100a kernels (pkg/tests/test_dynamics.py, test_sensors.py, test_tasks.py).
Tolerances are the fp64 reference's, relaxed to fp32 round-off where noted."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qs():
    import paper_2509_10247_b200 as qs

    return qs


def P(qs, **kw):
    return qs.QuadParams(**kw)


def np_(x):
    return x.detach().double().cpu().numpy()


# ---------------------------------------------------------------------------
# dynamics (pkg/tests/test_dynamics.py)


def test_hover_fixed_points(qs):  # :33-64
    cases = [("full", dict(drag_matrix_diag=np.array([0.3, 0.3, 0.1])), 4),
             ("simplified", {}, 2), ("pm_continuous", dict(drag_coeff=0.7), 3), ("pm_discrete", {}, 2)]
    for name, kw, B in cases:
        m = qs.make_model(name, P(qs, **kw))
        p0 = np.ones((B, 3)) if name == "pm_continuous" else np.zeros((B, 3))
        s = m.init_state(p0, np.zeros((B, 3)))
        s2 = m.step(s, m.hover_action(B))
        for k, v in s.fields().items():
            np.testing.assert_allclose(np_(s2.fields()[k]), np_(v), atol=1e-6, err_msg=f"{name}.{k}")


def test_full_free_fall(qs):  # :67-73
    prm = P(qs)
    m = qs.make_model("full", prm)
    s2 = m.step(m.init_state(np.zeros((1, 3)), np.zeros((1, 3))), torch.zeros(1, 4, device="cuda"))
    assert float(s2.v[0, 2]) == pytest.approx(-9.81 * prm.dt, abs=1e-7)


def test_simplified_yaw_rotation_small_dt(qs):  # :76-91
    prm = P(qs, dt=1e-4)
    m = qs.make_model("simplified", prm)
    s = m.init_state(np.zeros((1, 3)), np.zeros((1, 3)))
    wz = 2.0
    s2 = m.step(s, torch.tensor([[9.81, 0.0, 0.0, wz]], device="cuda"))
    ang = wz * prm.dt
    R_expect = np.array([[math.cos(ang), -math.sin(ang), 0.0], [math.sin(ang), math.cos(ang), 0.0], [0, 0, 1.0]])
    np.testing.assert_allclose(np_(s2.R)[0], R_expect, atol=1e-6)


def test_pm_continuous_large_lambda_limit(qs):  # :94-100
    m = qs.make_model("pm_continuous", P(qs, latency=1e3))
    u = torch.tensor([[1.0, -2.0, 12.0]], device="cuda")
    s2 = m.step(m.init_state(np.zeros((1, 3)), np.zeros((1, 3))), u)
    np.testing.assert_allclose(np_(s2.a_lat), np_(u), rtol=1e-3)


def test_pm_discrete_ballistic_and_constant_action(qs):  # :103-129
    m = qs.make_model("pm_discrete", P(qs, dt=0.1))
    s = qs.QuadState(p=torch.zeros(1, 3, device="cuda"), v=torch.tensor([[1.0, 0.0, 0.0]], device="cuda"),
                     u_prev=torch.zeros(1, 3, device="cuda"))
    s2 = m.step(s, torch.zeros(1, 3, device="cuda"))
    np.testing.assert_allclose(np_(s2.p), [[0.1, 0.0, 0.0]], atol=1e-7)
    dt = 0.05
    m = qs.make_model("pm_discrete", P(qs, dt=dt))
    u = np.array([[0.3, -0.2, 0.5]])
    s = qs.QuadState(p=torch.zeros(1, 3, device="cuda"), v=torch.zeros(1, 3, device="cuda"),
                     u_prev=torch.as_tensor(u, dtype=torch.float32, device="cuda"))
    p, v = np.zeros(3), np.zeros(3)
    for _ in range(10):
        s = m.step(s, torch.as_tensor(u, dtype=torch.float32, device="cuda"))
        p = p + v * dt + 0.5 * u[0] * dt * dt
        v = v + u[0] * dt
    np.testing.assert_allclose(np_(s.p)[0], p, atol=1e-6)
    np.testing.assert_allclose(np_(s.v)[0], v, atol=1e-6)


def test_rate_loop_identities(qs):  # :136-161
    prm = P(qs)
    w = torch.tensor([[0.4, -0.2, 0.9]], dtype=torch.float64)
    J = torch.as_tensor(prm.inertia)
    tau = qs.dynamics.rate_loop(w, w, prm)
    np.testing.assert_allclose(tau.numpy(), torch.cross(w, w @ J.T, dim=-1).numpy(), rtol=1e-12)
    z = torch.zeros(2, 3, dtype=torch.float64)
    assert torch.equal(qs.dynamics.rate_loop(z, z, prm), torch.zeros(2, 3, dtype=torch.float64))


def test_non_finite_state_rejected(qs):  # :204-214
    m = qs.make_model("full", P(qs))
    s = m.init_state(np.zeros((2, 3)), np.zeros((2, 3)))
    s.p[1, 0] = float("nan")
    with pytest.raises(qs.dynamics.ContractError):
        m.step(s, m.hover_action(2))


def test_step_determinism(qs):  # :192-201
    for name in ("full", "simplified", "pm_continuous", "pm_discrete"):
        m = qs.make_model(name, P(qs))
        g = torch.Generator().manual_seed(0)
        s = m.init_state(torch.randn(64, 3, generator=g), torch.randn(64, 3, generator=g))
        a = torch.randn(64, m.action_dim, generator=g).cuda()
        x, y = m.step(s, a), m.step(s, a)
        for k in x.fields():
            assert torch.equal(x.fields()[k], y.fields()[k])


def test_pm_discrete_one_step_jacobians(qs):  # :269-287
    dt = 0.1
    m = qs.make_model("pm_discrete", P(qs, dt=dt))
    B = 3
    s = m.init_state(np.zeros((B, 3)), np.zeros((B, 3)))
    raw = np.zeros((1, B, 3))
    g_p = qs.rollout_grad(m, s, raw, 0, 1, weights={"p": np.ones((B, 3))}).grad
    np.testing.assert_allclose(np_(g_p), np.full((B, 3), 0.5 * dt * dt), atol=1e-7)
    g_v = qs.rollout_grad(m, s, raw, 0, 1, weights={"v": np.ones((B, 3))}).grad
    np.testing.assert_allclose(np_(g_v), np.full((B, 3), 0.5 * dt), atol=1e-7)


def test_squash_center_asymptote_and_box(qs):  # :314-336
    lo, hi = np.full(3, -6.0), np.full(3, 6.0)
    sq = qs.dynamics.action_squash
    assert torch.equal(sq(torch.zeros(1, 3, device="cuda"), lo, hi), torch.zeros(1, 3, device="cuda"))
    np.testing.assert_allclose(np_(sq(torch.full((1, 3), 50.0, device="cuda"), lo, hi)), 6.0, atol=1e-6)
    np.testing.assert_allclose(np_(sq(torch.ones(1, 3, device="cuda"), lo, hi)), 4.569564935734589, rtol=1e-6)
    lo4, hi4 = np.array([0.0, -6.0, -6.0, -3.0]), np.array([19.62, 6.0, 6.0, 3.0])
    raw = torch.as_tensor(np.random.default_rng(3).normal(size=(64, 4)) * 2, dtype=torch.float32, device="cuda")
    out = np_(sq(raw, lo4, hi4))
    assert np.all(out > lo4) and np.all(out < hi4)


def test_energy_drift_is_second_order(qs):  # :343-360
    prm = P(qs, dt=0.01)
    m = qs.make_model("full", prm)
    s = m.init_state(np.zeros((1, 3)), np.array([[2.0, 0.0, 3.0]]))
    act = torch.zeros(1, 4, device="cuda")

    def energy(st):
        v = np_(st.v)[0]
        return 0.5 * v @ v + 9.81 * np_(st.p)[0, 2]

    drift = []
    for _ in range(50):
        e0 = energy(s)
        s = m.step(s, act)
        drift.append(abs(energy(s) - e0))
    bound = 0.5 * 9.81 ** 2 * prm.dt ** 2
    assert max(drift) <= bound * 1.001 + 2e-5  # + fp32 round-off of the energies


@torch.no_grad()
def test_attitude_normalization_long_run(qs):  # :363-383
    prm = P(qs, dt=0.01)
    fm, sm = qs.make_model("full", prm), qs.make_model("simplified", prm)
    sf = fm.init_state(np.zeros((2, 3)), np.zeros((2, 3)))
    ss = sm.init_state(np.zeros((2, 3)), np.zeros((2, 3)))
    act = np.random.default_rng(13).normal(size=(2, 4))
    act[:, 0] = 9.81
    act = torch.as_tensor(act, dtype=torch.float32, device="cuda")
    for _ in range(20_000):
        sf = fm.step(sf, act, check=False)
        ss = sm.step(ss, act, check=False)
    np.testing.assert_allclose(np.linalg.norm(np_(sf.q), axis=-1), 1.0, atol=1e-5)
    R = np_(ss.R)
    np.testing.assert_allclose(np.einsum("bji,bjk->bik", R, R), np.broadcast_to(np.eye(3), (2, 3, 3)), atol=1e-5)


# ---------------------------------------------------------------------------
# sensors (pkg/tests/test_sensors.py)


def test_sphere_hit_residual(qs):  # :79-88
    sn = qs.sensors
    rng = np.random.default_rng(0)
    for _ in range(10):
        c = rng.uniform(-5, 5, 3)
        r = rng.uniform(0.3, 2.0)
        o = c + rng.normal(size=3) * 8
        d = c - o + rng.normal(size=3) * 0.1 * r
        d /= np.linalg.norm(d)
        t = float(sn.raycast(sn.PrimitiveSet(spheres=[[*c, r]]), torch.as_tensor(o[None]).cuda(),
                             torch.as_tensor(d[None, None]).cuda(), 100.0))
        if t < 100.0:
            assert abs(np.linalg.norm(o + t * d - c) - r) < 1e-4


def test_empty_scene_wall_and_order_independence(qs):  # :154-185
    sn = qs.sensors
    cam = sn.CameraIntrinsics(width=16, height=9, max_range=10.0)
    pos = torch.tensor([[0.0, 0.0, 1.0]], device="cuda")
    R = np.eye(3)[None]
    img = sn.render_depth(sn.PrimitiveSet(), pos, R, cam)
    assert torch.all(img == 10.0)
    wall = sn.PrimitiveSet(boxes=[[4.0, 0.0, 0.0, 0.5, 50.0, 50.0]])  # face at x=3.5
    img = np_(sn.render_depth(wall, pos, R, cam))[0]
    dirs = cam.pixel_dirs().reshape(9, 16, 3)
    np.testing.assert_allclose(img, np.minimum(3.5 / dirs[..., 0], 10.0), atol=1e-5)
    rng = np.random.default_rng(5)
    sph = np.column_stack([rng.uniform(1, 8, (6, 1)), rng.uniform(-3, 3, (6, 2)), rng.uniform(0.3, 1, (6, 1))])
    box = np.column_stack([rng.uniform(1, 8, (6, 1)), rng.uniform(-3, 3, (6, 2)), rng.uniform(0.2, 1, (6, 3))])
    a = sn.render_depth(sn.PrimitiveSet(spheres=sph, boxes=box, ground_z=0.0), pos, R, cam)
    b = sn.render_depth(sn.PrimitiveSet(spheres=sph[::-1], boxes=box[::-1], ground_z=0.0), pos, R, cam)
    assert torch.equal(a, b)


def test_lidar_pattern_layout(qs):  # :188-208
    sn = qs.sensors
    pat = sn.LidarPattern(n_azimuth=8, n_elevation=3, max_range=20.0)
    d = pat.ray_dirs()
    np.testing.assert_allclose(np.linalg.norm(d, axis=-1), 1.0, atol=1e-12)
    # azimuth-major: index a * n_el + e
    np.testing.assert_allclose(d[0 * 3 + 1], [1.0, 0.0, 0.0], atol=1e-12)
    ranges = np_(sn.render_lidar(sn.PrimitiveSet(ground_z=0.0), torch.tensor([[0.0, 0.0, 2.0]], device="cuda"),
                                 np.eye(3)[None], pat))[0]
    el = np.linspace(-0.5, 0.5, 3) * np.deg2rad(30.0)
    expect = np.where(np.sin(el) < 0, np.minimum(2.0 / -np.sin(np.minimum(el, -1e-300)), 20.0), 20.0)
    np.testing.assert_allclose(ranges.reshape(8, 3), np.broadcast_to(expect, (8, 3)), atol=1e-4)


def test_attitude_identity_and_yaw(qs):  # :351-383
    sn = qs.sensors
    R = np_(sn.reconstruct_attitude(torch.tensor([[0.0, 0.0, 9.81]]).cuda(), torch.tensor([[1.0, 0.0, 0.0]]).cuda()))
    np.testing.assert_allclose(R[0], np.eye(3), atol=1e-6)
    R = np_(sn.reconstruct_attitude(torch.tensor([[0.0, 0.0, 9.81]]).cuda(), torch.tensor([[0.0, 2.0, 0.0]]).cuda()))
    assert float(sn.yaw_of(R)[0]) == pytest.approx(np.pi / 2, abs=1e-6)
    rng = np.random.default_rng(1)
    R = np_(sn.reconstruct_attitude(torch.as_tensor(rng.normal(size=(64, 3)) * 5).cuda(),
                                    torch.as_tensor(rng.normal(size=(64, 3))).cuda()))
    np.testing.assert_allclose(np.einsum("bji,bjk->bik", R, R), np.broadcast_to(np.eye(3), (64, 3, 3)), atol=1e-5)


def test_imu_hover_and_freefall(qs):  # :305-313
    sn = qs.sensors
    g = np.array([0.0, 0.0, -9.81])
    imu = sn.ImuModel(batch=2)
    I = np.broadcast_to(np.eye(3), (2, 3, 3)).copy()
    a, w = imu.read(I, np.zeros((2, 3)), np.zeros((2, 3)), g, 0.01)
    np.testing.assert_allclose(np_(a), np.broadcast_to([0, 0, 9.81], (2, 3)), atol=1e-6)
    assert torch.equal(w, torch.zeros(2, 3, device="cuda"))
    a, _ = imu.read(I, None, np.broadcast_to(g, (2, 3)), g, 0.01)
    np.testing.assert_allclose(np_(a), 0.0, atol=1e-6)


# ---------------------------------------------------------------------------
# tasks (pkg/tests/test_tasks.py)


def cfg_position(qs, **kw):
    base = dict(task="position", dynamics="pm_continuous", n_envs=4, episode_len=16, goal_dist=6.0)
    base.update(kw)
    return qs.TaskConfig(**base)


def test_reset_determinism_and_initial_goal_vector(qs):  # :30-50
    a = qs.make_task(cfg_position(qs)).reset(seed=3)
    b = qs.make_task(cfg_position(qs)).reset(seed=3)
    assert torch.equal(a.obs.proprio, b.obs.proprio)
    c = qs.make_task(cfg_position(qs)).reset(seed=4)
    assert not torch.equal(a.obs.proprio, c.obs.proprio)
    env = qs.make_task(cfg_position(qs))
    out = env.reset(seed=5)
    yaw = np_(qs.sensors.yaw_of(qs.sensors.reconstruct_attitude(env.state.a_lat, env.v_ema)))
    expect = np.einsum("bij,bj->bi", qs.tasks.rotz_np(-yaw), np_(env.goals) - np_(env.state.p))
    np.testing.assert_allclose(np_(out.obs.proprio)[:, :3], expect, atol=1e-5)


def test_truncation_and_autoreset_detach(qs):  # :65-85
    env = qs.make_task(cfg_position(qs, n_envs=2, episode_len=3))
    env.reset(seed=2)
    acts = [torch.zeros(env.N, 3, device="cuda", requires_grad=True) for _ in range(3)]
    outs = [env.step(a) for a in acts]
    assert bool(outs[-1].truncated.all())
    assert torch.equal(env.steps_in_episode, torch.zeros(2, dtype=torch.int32, device="cuda"))
    g = torch.autograd.grad(outs[-1].obs.proprio.sum(), acts, allow_unused=True, retain_graph=True)
    assert all(x is None or float(x.abs().sum()) == 0.0 for x in g)
    (g0,) = torch.autograd.grad(outs[1].r_ctrl.sum(), [acts[0]])
    assert float(g0.abs().sum()) > 0


def test_success_and_bounds_termination(qs):  # :88-114
    env = qs.make_task(cfg_position(qs, n_envs=2, episode_len=64))
    env.reset(seed=3)
    env.state = env.model.init_state(env.goals.clone(), torch.zeros(2, 3, device="cuda"))
    out = env.step(torch.zeros(2, 3, device="cuda"))
    assert bool((out.terminated == qs.tasks.TERM_SUCCESS).all())
    assert torch.equal(out.r_goal, torch.ones(2, device="cuda"))
    assert env.finished_episodes == 2 and env.successful_episodes == 2
    env = qs.make_task(cfg_position(qs, n_envs=1, episode_len=64))
    env.reset(seed=4)
    p = env.bounds_hi_per_row.clone() + 5.0
    env.state = env.model.init_state(p, torch.zeros(1, 3, device="cuda"))
    out = env.step(torch.zeros(1, 3, device="cuda"))
    assert int(out.terminated[0]) == qs.tasks.TERM_BOUNDS and float(out.r_goal[0]) == -1.0


def test_non_finite_action_names_row(qs):  # :117-123
    env = qs.make_task(cfg_position(qs, n_envs=2))
    env.reset(seed=0)
    bad = torch.zeros(env.N, env.action_dim, device="cuda")
    bad[1, 0] = float("nan")
    with pytest.raises(qs.TaskContractError, match="row 1"):
        env.step(bad)
    # non-strict envs report the same contract violation lazily
    env2 = qs.make_task(cfg_position(qs, n_envs=2), strict=False)
    env2.reset(seed=0)
    env2.step(bad)
    with pytest.raises(qs.TaskContractError, match="row 1"):
        env2.check_errors()


def test_at_goal_reward_zero(qs):  # :126-143
    w = qs.tasks.RewardWeights()
    z = torch.zeros(1)
    assert float(qs.tasks.reward_position(z, z, z, z, z, w)[0]) == 0.0
    err = qs.tasks.velocity_field_error(torch.zeros(2, 3), torch.zeros(2, 3), w)
    assert torch.all(err == 0)


def test_yaw_invariance_observations_and_rewards(qs):  # :288-335
    rng = np.random.default_rng(17)
    for trial in range(5):
        envs = [qs.make_task(cfg_position(qs, n_envs=10, episode_len=10 ** 6)) for _ in range(2)]
        for e in envs:
            e.reset(seed=100 + trial)
        p = rng.normal(size=(10, 3)) * 2 + [2, 0, 2]
        v = rng.normal(size=(10, 3))
        a = rng.normal(size=(10, 3)) + [0, 0, 9.81]
        goals = np_(envs[0].goals)
        for e in envs:
            e.state = qs.QuadState(p=torch.as_tensor(p, dtype=torch.float32).cuda(),
                                   v=torch.as_tensor(v, dtype=torch.float32).cuda(),
                                   a_lat=torch.as_tensor(a, dtype=torch.float32).cuda())
            e.v_ema = v.copy()
            e.goals = goals
            e.bounds_lo_per_row = np.full((10, 3), -1e6)
            e.bounds_hi_per_row = np.full((10, 3), 1e6)
        psi = rng.uniform(0, 2 * np.pi)
        c, s = np.cos(psi), np.sin(psi)
        Rz = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])
        e2 = envs[1]
        e2.goals = goals @ Rz.T
        e2.state = qs.QuadState(p=torch.as_tensor(p @ Rz.T, dtype=torch.float32).cuda(),
                                v=torch.as_tensor(v @ Rz.T, dtype=torch.float32).cuda(),
                                a_lat=torch.as_tensor(a @ Rz.T, dtype=torch.float32).cuda())
        e2.v_ema = v @ Rz.T
        o1, o2 = envs[0].observe(), envs[1].observe()
        np.testing.assert_allclose(np_(o1.proprio), np_(o2.proprio), atol=2e-5)
        act = torch.as_tensor(rng.normal(size=(10, 3)) * 0.5, dtype=torch.float32).cuda()
        s1, s2 = envs[0].step(act), envs[1].step(act)
        np.testing.assert_allclose(np_(s1.r_ctrl), np_(s2.r_ctrl), atol=2e-5)
        assert torch.equal(s1.r_goal, s2.r_goal)
        np.testing.assert_allclose(np_(s1.obs.proprio), np_(s2.obs.proprio), atol=2e-5)


def test_dual_reward_contract_and_detach(qs):  # :565-589
    env = qs.make_task(cfg_position(qs))
    env.reset(seed=61)
    a = (torch.randn(4, 3, generator=torch.Generator().manual_seed(0)) * 0.1).cuda().requires_grad_(True)
    out = env.step(a)
    (g,) = torch.autograd.grad(out.r_ctrl.sum(), a)
    assert float(g.abs().sum()) > 0
    assert not out.r_goal.requires_grad and not out.r_rl.requires_grad
    assert set(np.unique(np_(out.r_goal))).issubset({-1.0, 0.0, 1.0})
    env.reset(seed=62)
    a0 = torch.zeros(4, 3, device="cuda", requires_grad=True)
    env.step(a0)
    env.detach_states()
    a1 = torch.zeros(4, 3, device="cuda", requires_grad=True)
    out = env.step(a1)
    g0, g1 = torch.autograd.grad(out.r_ctrl.sum(), [a0, a1], allow_unused=True)
    assert g0 is None or float(g0.abs().sum()) == 0.0
    assert float(g1.abs().sum()) > 0


# ---------------------------------------------------------------------------
# racing (pkg/tests/test_tasks.py:402-480): gate arrays + pass / crash through env.step


def race_cfg(qs, **kw):
    base = dict(task="racing", dynamics="pm_continuous", n_envs=1, episode_len=256, n_gates=3, gate_spread=6.0)
    base.update(kw)
    return qs.TaskConfig(**base)


def _through_gate(qs, env, offset):
    """Place the drone 0.5 m before gate 0 (+ offset) moving 1 m per step along
    its normal (pm_continuous integrates p with the pre-step velocity)."""
    c = env.gate_centers[0, 0].double()
    n = env.gate_normals[0, 0].double()
    p = (c - 0.5 * n + offset)[None].float()
    v = (n / env.config.dt)[None].float()
    env.state = env.model.init_state(p, v)
    return env.step(torch.zeros(1, 3, device="cuda"))


def test_racing_gate_arrays_and_initial_goal(qs):  # :864-867, 887-891
    env = qs.make_task(race_cfg(qs))
    env.reset(seed=31)
    g = qs.world.device_scene_to_scenes(env._scene, style="racing")[0].gates
    assert env.gate_centers.shape == (1, 3, 3)
    np.testing.assert_allclose(np_(env.gate_centers[0]), np.stack([x.center for x in g]), atol=1e-6)
    np.testing.assert_allclose(np_(env.gate_normals[0]), np.stack([x.normal for x in g]), atol=1e-6)
    np.testing.assert_allclose(np_(env.gate_inner[0]), [x.inner_radius for x in g], atol=1e-6)
    np.testing.assert_allclose(np_(env.gate_frame[0]), [x.frame_width for x in g], atol=1e-6)
    assert torch.equal(env.goals[0], env.gate_centers[0, 0])
    assert int(env.next_gate[0]) == 0


def test_racing_gate_pass_and_crash(qs):  # :427-458
    env = qs.make_task(race_cfg(qs))
    env.reset(seed=32)
    out = _through_gate(qs, env, torch.zeros(3, dtype=torch.float64, device="cuda"))
    assert int(out.terminated[0]) == 0  # a clean pass through a non-final gate
    assert int(env.next_gate[0]) == 1
    assert torch.equal(env.goals[0], env.gate_centers[0, 1])
    env.reset(seed=32)
    n = env.gate_normals[0, 0].double()
    up = torch.tensor([0.0, 0.0, 1.0], dtype=torch.float64, device="cuda")
    radial = up - torch.dot(up, n) * n
    radial = radial / radial.norm()
    r_hit = float(env.gate_inner[0, 0]) + 0.5 * float(env.gate_frame[0, 0])
    out = _through_gate(qs, env, radial * r_hit)
    assert int(out.terminated[0]) == qs.tasks.TERM_COLLISION
    assert float(out.r_goal[0]) == -1.0
