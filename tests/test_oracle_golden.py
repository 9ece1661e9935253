"""Pin the CPU oracle to the reference's own outputs (golden fixtures).

These run without a GPU.  Every fixture in tests/golden was produced by the
real reference (tests/golden/make_golden.py); the oracle restatement must
reproduce it to fp64 round-off before any GPU parity claim is trusted.
"""

import numpy as np
import pytest

from golden_utils import (TASK_CASES, fixture_state, load, oracle_config, scene_from_json,
                          STATE_KEYS)
from oracle import quadsim_oracle as O

RTOL = 1e-10


def close(a, b, tol=1e-10):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    np.testing.assert_allclose(a, b, rtol=tol, atol=tol)


# ---------------------------------------------------------------------------
# dynamics


@pytest.mark.parametrize("key", ["full_default", "full_drag", "pm_continuous_default",
                                 "pm_continuous_drag", "pm_discrete_default", "simplified_default"])
def test_dynamics_rollout_matches_reference(key):
    z = load("dynamics")
    model = key.rsplit("_", 1)[0]
    prm = O.Params(dt=0.02)
    if f"{key}/drag_diag" in z:
        prm.drag_matrix_diag = z[f"{key}/drag_diag"]
    if f"{key}/drag_coeff" in z:
        prm.drag_coeff = z[f"{key}/drag_coeff"]
        prm.latency = z[f"{key}/latency"]
    st = {k: z[f"{key}/s0_{k}"] for k in STATE_KEYS[model]}
    raw = z[f"{key}/raw"]
    lo, hi = O.action_box(model)
    for t in range(raw.shape[0]):
        st = O.model_step(model, st, O.squash(raw[t], lo, hi), prm)
        for k in STATE_KEYS[model]:
            close(st[k], z[f"{key}/s{t+1}_{k}"], 1e-12)


# ---------------------------------------------------------------------------
# sensors


def _fixture_prims(z):
    return {k: z[f"prims_{k}"] for k in ("spheres", "sph_valid", "boxes", "box_valid", "cylinders",
                                         "cyl_valid", "ground_z")}


def test_raycast_render_cull_sdf_match_reference():
    z = load("sensors")
    prims = _fixture_prims(z)
    pos, yaw = z["pos"], z["yaw"]
    R = O.rotz(yaw)
    close(O.render_depth(prims, pos, R, 32, 24, 10.0, cull=True), z["depth_cull"], 1e-12)
    close(O.render_depth(prims, pos, R, 32, 24, 10.0, cull=False), z["depth_nocull"], 1e-12)
    # culling never changes the image (pkg/tests/test_sensors.py:136-151)
    assert np.array_equal(z["depth_cull"], z["depth_nocull"])
    close(O.render_depth(prims, pos, R, 16, 9, 7.0), z["depth_16x9"], 1e-12)
    close(O.render_lidar(prims, pos, R, 36, 5, 15.0), z["lidar"], 1e-12)
    close(O.raycast(prims, pos, z["ray_dirs"], 12.0), z["ray_t"], 1e-12)
    ks, kb, kc = O.fov_cull(prims, pos, R, 10.0)
    assert np.array_equal(ks, z["cull_s"]) and np.array_equal(kb, z["cull_b"])
    assert np.array_equal(kc, z["cull_c"])
    close(O.sdf(z["sdf_pts"], prims), z["sdf"], 1e-12)
    close(O.reconstruct_attitude(z["att_a"], z["att_v"]), z["att_R"], 1e-12)


def test_known_answers():
    z = load("sensors")
    assert float(z["ka_sphere"]) == pytest.approx(4.0, abs=1e-12)
    assert float(z["ka_box"]) == pytest.approx(2.0, abs=1e-12)
    assert float(z["ka_cyl_side"]) == pytest.approx(3.0, abs=1e-12)
    assert float(z["ka_cyl_cap"]) == pytest.approx(8.0, abs=1e-12)
    assert float(z["ka_ground"]) == pytest.approx(3.0, abs=1e-12)


def test_imu_matches_reference():
    z = load("imu")
    g = np.array([0.0, 0.0, -9.81])
    imu = O.Imu(8, accel_noise_std=0.1, gyro_noise_std=0.01, accel_bias_rw_std=0.01,
                gyro_bias_rw_std=0.001, seed=17)
    for t in range(6):
        a, w = imu.read(z["R"], z[f"w{t}"], z[f"vdot{t}"], g, 0.05)
        close(a, z[f"accel{t}"], 1e-12)
        close(w, z[f"gyro{t}"], 1e-12)


def test_world_generation_matches_reference():
    z = load("world")
    spawn = np.array([0.0, 0.0, 1.2])
    goal = np.array([8.0, 0.0, 1.5])
    for i, (seed, style, dens) in enumerate([(11, "outdoor", 0.1), (12, "indoor", 0.1), (13, "outdoor", 0.25)]):
        ref = scene_from_json(z[f"scene{i}"])
        s = O.gen_obstacle_course(seed, spawn, goal, dens, style=style)
        for k in ("spheres", "boxes", "cylinders"):
            close(s.prims[k], ref.prims[k], 1e-12)
        close(s.bounds_lo, ref.bounds_lo, 1e-12)
        close(s.bounds_hi, ref.bounds_hi, 1e-12)
        assert O.grid_path_exists(s) == bool(z[f"scene{i}_feasible"])
    ref = scene_from_json(z["race"])
    t = O.gen_race_track(21, 5, 10.0)
    for (c, n, _, _), (cr, nr, _, _) in zip(t.gates, ref.gates):
        close(c, cr, 1e-12)
        close(n, nr, 1e-12)
    for kind in ("line", "square", "circle"):
        close(O.formation_offsets(kind, 5, 2.0), z[f"form_{kind}"], 1e-12)
    dr = O.randomize_params(O.RandomizationSpec(), 5, 3, 10)
    close(np.stack([dr["drag_coeff"], dr["latency"], dr["action_scale"]], -1), z["dr"], 1e-15)


# ---------------------------------------------------------------------------
# task trajectories


def build_oracle_task(name):
    z = load(f"task_{name}")
    cfg = oracle_config(name)
    provider = None
    if "scenes_json" in z:
        scenes = [scene_from_json(s) for s in z["scenes_json"]]
        provider = lambda seed, e: scenes[e]  # noqa: E731
    env = O.OracleTask(cfg, scene_provider=provider)
    env.reset(int(z["seed"]))
    if "teleport_p" in z:
        st = O.init_state(cfg.dynamics, z["teleport_p"], z["teleport_v"])
        env.state = st
    return env, z


@pytest.mark.parametrize("name", list(TASK_CASES))
def test_task_trajectory_matches_reference(name):
    env, z = build_oracle_task(name)
    cfg = env.cfg
    for k, v in fixture_state(z, 0, cfg.dynamics).items():
        close(env.state[k], v)
    close(env.goals, z["goals0"])
    close(env.observe_proprio(), z["proprio0"])
    if "visual0" in z:
        close(env.render(force=True), z["visual0"])
    raw = z["raw"]
    for t in range(int(z["T"])):
        out = env.step(raw[t])
        i = t + 1
        close(out["proprio"], z[f"proprio{i}"])
        close(out["r_ctrl"], z[f"r_ctrl{i}"])
        close(out["r_goal"], z[f"r_goal{i}"])
        close(out["r_rl"], z[f"r_rl{i}"])
        assert np.array_equal(out["terminated"], z[f"term{i}"])
        assert np.array_equal(out["truncated"], z[f"trunc{i}"])
        for k, v in fixture_state(z, i, cfg.dynamics).items():
            close(env.state[k], v)
        close(env.goals, z[f"goals{i}"])
        close(env.v_ema, z[f"v_ema{i}"])
        assert np.array_equal(env.steps, z[f"steps{i}"])
        if f"visual{i}" in z:
            close(out["visual"], z[f"visual{i}"])
        if f"dr{i}" in z:
            close(np.stack([env.dr_drag, env.dr_lat, env.dr_scale], -1), z[f"dr{i}"])
    close(np.array([env.finished, env.successes, env.collisions, env.finished_return]), z["stats"])


@pytest.mark.parametrize("name", ["pos_full", "pos_form", "avoid_form", "pos_pmc_dr", "avoid_collide",
                                  "pos_events", "pos_simp"])
def test_oracle_fd_gradient_matches_reference_tape(name):
    """Central-difference BPTT gradient of the oracle == the reference's tape gradient."""
    env, z = build_oracle_task(name)
    raw = z["raw"]
    T = int(z["T"])
    g_ref = z["grad"]
    if "grad_unaliased" in z:
        # reference tape defect under per-episode DR (see make_golden.py:
        # _redraw_without_aliasing); the forward is identical either way
        g_ref = z["grad_unaliased"]
    g = O.fd_grad_actions(env, raw[:T])
    scale = np.abs(g_ref).max()
    assert np.abs(g - g_ref).max() / scale < 1e-6


@pytest.mark.parametrize("name", ["pos_pmc", "pos_pmd"])
def test_oracle_fd_gradient_long_window(name):
    env, z = build_oracle_task(name)
    g = O.fd_grad_actions(env, z["raw"])
    g_ref = z["grad"]
    assert np.abs(g - g_ref).max() / np.abs(g_ref).max() < 1e-6


@pytest.mark.parametrize("name", ["pos_pmc", "pos_pmd", "pos_full", "pos_pmc_dr", "pos_events",
                                  "pos_full_events"])
def test_oracle_reverse_pass_matches_reference_tape(name):
    env, z = build_oracle_task(name)
    loss, g = O.window_value_and_grad(env, z["raw"])
    g_ref = z["grad_unaliased"] if "grad_unaliased" in z else z["grad"]
    assert abs(loss - float(z["loss"])) < 1e-12
    assert np.abs(g - g_ref).max() / np.abs(g_ref).max() < 1e-10


# ---------------------------------------------------------------------------
# C1 at its exact shape (1,024 envs x 32 steps, reset(seed=1), default_rng(0)
# actions): the oracle's forward, resets and reverse pass against the
# reference's own run (tests/golden/make_golden.py:gen_c1)


@pytest.mark.parametrize("short,model", [("pmc", "pm_continuous"), ("pmd", "pm_discrete")])
def test_c1_exact_shape_oracle_matches_reference(short, model):
    z = load(f"c1_{short}")
    env = O.OracleTask(O.Config(task="position", dynamics=model, n_envs=1024, episode_len=10 ** 6))
    env.reset(1)
    for k in STATE_KEYS[model]:
        close(env.state[k], z[f"s0_{k}"], 1e-12)
    raw = np.random.default_rng(0).normal(size=(32, 1024, 3)) * 0.3
    snap = env.snapshot()
    r_ctrl, term = [], []
    for t in range(32):
        out = env.step(raw[t])
        r_ctrl.append(out["r_ctrl"])
        term.append(out["terminated"])
        if t == 15:
            for k in STATE_KEYS[model]:
                close(env.state[k], z[f"s16_{k}"], 1e-10)
    for k in STATE_KEYS[model]:
        close(env.state[k], z[f"s32_{k}"], 1e-10)
    assert np.array_equal(np.stack(term), z["term"])
    np.testing.assert_allclose(np.stack(r_ctrl), z["r_ctrl"], rtol=1e-6, atol=1e-6)  # f32 storage
    env.restore(snap)
    loss, g = O.window_value_and_grad(env, raw)
    assert abs(loss - float(z["loss"])) < 1e-10
    assert np.abs(g - z["grad"]).max() / np.abs(z["grad"]).max() < 1e-6  # f32 storage
