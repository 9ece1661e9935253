"""Opt-in depth VJP against fp64 central differences, in-kernel domain
randomisation statistics, and the differentiable-depth env path."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_depth_vjp_matches_central_differences():
    """d depth / d position: analytic -n/(n.d) vs the oracle's fp64 central
    difference (h = 1e-6 (1+|x|), pkg/tests/oracles.py:15-30), away from
    silhouettes (rays whose FD stencil changes the hit primitive are excluded)."""
    import paper_2509_10247_b200 as qs
    from oracle import quadsim_oracle as O

    sn = qs.sensors
    rng = np.random.default_rng(0)
    E = 16
    sets = []
    for _ in range(E):
        sph = np.column_stack([rng.uniform(2, 7, 3), rng.uniform(-3, 3, 3), rng.uniform(0.5, 2.5, 3),
                               rng.uniform(0.4, 1.0, 3)])
        box = np.column_stack([rng.uniform(2, 7, 2), rng.uniform(-3, 3, 2), rng.uniform(0.5, 2.5, 2),
                               rng.uniform(0.3, 0.8, (2, 3))])
        cyl = np.column_stack([rng.uniform(2, 7, 2), rng.uniform(-3, 3, 2), rng.uniform(0.8, 1.5, 2),
                               rng.uniform(0.2, 0.5, 2), rng.uniform(0.8, 1.5, 2)])
        sets.append(sn.PrimitiveSet(spheres=sph, boxes=box, cylinders=cyl, ground_z=0.0))
    bp = sn.pack_primitives(sets)
    sc = sn.DeviceScene.from_batched(bp, "cuda")
    pos = np.column_stack([np.zeros(E), rng.uniform(-0.5, 0.5, E), rng.uniform(1.0, 2.0, E)])
    cam = sn.CameraIntrinsics(width=16, height=12, max_range=10.0)
    cs = torch.tensor([[1.0, 0.0]] * E, device="cuda")
    p4 = torch.zeros(E, 4, device="cuda")
    p4[:, :3] = torch.as_tensor(pos)
    depth, _, dT = sn.cast_rays(sc, p4, 4, cs, cam, 0, True, want_grad=True)
    dT = dT[..., :3].cpu().numpy()
    prims = O.pack_primitives([{"spheres": s.spheres, "boxes": s.boxes, "cylinders": s.cylinders,
                                "ground_z": 0.0} for s in sets])
    dirs = np.broadcast_to(cam.pixel_dirs(), (E, cam.n_rays, 3))
    base = O.raycast(prims, pos, dirs, 10.0)
    ok_total, bad = 0, 0
    for k in range(3):
        h = 1e-6 * (1 + np.abs(pos[:, k]))
        pp, pm = pos.copy(), pos.copy()
        pp[:, k] += h
        pm[:, k] -= h
        fp = O.raycast(prims, pp, dirs, 10.0)
        fm = O.raycast(prims, pm, dirs, 10.0)
        fd = (fp - fm) / (2 * h[:, None])
        smooth = (np.abs(fp - base) < 1e-3) & (np.abs(fm - base) < 1e-3) & (base < 10.0)
        err = np.abs(dT[..., k] - fd)[smooth]
        ok_total += smooth.sum()
        bad += int((err > 1e-3 * (1 + np.abs(fd[smooth]))).sum())
    assert ok_total > 1000
    assert bad / ok_total < 2e-3, (bad, ok_total)


def test_differentiable_depth_env_backprop():
    import paper_2509_10247_b200 as qs

    cfg = qs.TaskConfig(task="avoidance", dynamics="pm_continuous", n_envs=64, sensor="depth", depth_width=16,
                        depth_height=12, density=0.3, differentiable_depth=True)
    env = qs.make_task(cfg)
    env.reset(seed=1)
    a = torch.zeros(64, 3, device="cuda", requires_grad=True)
    env.step(a)  # explicit Euler: p_{t+1} = p_t + v_t dt, so a_t reaches depth at t+2
    out = env.step(torch.zeros(64, 3, device="cuda"))
    assert out.obs.visual.requires_grad
    (g,) = torch.autograd.grad(out.obs.visual.sum(), a)
    assert torch.isfinite(g).all() and g.abs().sum() > 0


def test_in_kernel_domain_randomisation_statistics():
    import paper_2509_10247_b200 as qs

    spec = qs.world.RandomizationSpec(drag_coeff=(0.1, 0.5), latency=(2.0, 8.0), action_scale=(0.5, 1.0))
    cfg = qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=20000, episode_len=2,
                        randomization=spec)
    env = qs.make_task(cfg)
    env.reset(seed=7)
    dr = env._dr.double().cpu().numpy()
    for col, (lo, hi) in ((0, spec.drag_coeff), (3, spec.latency), (2, spec.action_scale)):
        x = dr[:, col]
        assert x.min() >= lo - 1e-6 and x.max() <= hi + 1e-6
        assert abs(x.mean() - (lo + hi) / 2) < 0.01 * (hi - lo) + 1e-6
        assert abs(x.std() - (hi - lo) / np.sqrt(12)) < 0.02 * (hi - lo)
    np.testing.assert_allclose(dr[:, 1], np.exp(-dr[:, 3] * cfg.dt), rtol=1e-5)
    before = dr.copy()
    for _ in range(2):  # episode_len 2: every env resets and redraws (per_episode)
        env.step(torch.zeros(env.N, 3, device="cuda"))
    after = env._dr.double().cpu().numpy()
    assert (np.abs(after - before).max(axis=1) > 0).mean() > 0.99


def test_obstacle_rerandomisation_on_reset():
    """regen_scene_on_reset (declared, unwired at q/tasks.py:98): a done env gets
    a fresh course keyed by (seed, env, episode) on the device, then a Philox
    spawn on that course; envs that did not finish keep theirs."""
    import paper_2509_10247_b200 as qs
    from oracle import quadsim_oracle as O

    E = 96
    cfg = qs.TaskConfig(task="avoidance", dynamics="pm_continuous", n_envs=E, episode_len=3, density=0.3,
                        regen_scene_on_reset=True)
    env = qs.make_task(cfg)
    env.reset(seed=5)
    sc = env._scene
    snap = lambda: [t.clone() for t in (sc.spheres, sc.boxes, sc.cylinders, sc.counts)]
    before = snap()
    ever_done = np.zeros(E, bool)
    for step in range(3):
        prev = snap()
        out = env.step(torch.zeros(E, 3, device="cuda"))
        done = (env._last_flags.cpu().numpy() & 1).astype(bool)
        now = snap()
        changed = np.zeros(E, bool)
        for a, b in zip(prev, now):
            changed |= (a != b).reshape(E, -1).any(1).cpu().numpy()
        assert not changed[~done].any(), step  # untouched unless reset
        assert changed[done].all(), step
        ever_done |= done
        p = env.state.p.detach().cpu().numpy()
        spawn = sc.spawn_goal[:, 0, :3].cpu().numpy()
        if done.any():
            assert np.linalg.norm(p[done] - spawn[done], axis=-1).max() < 1.0  # spawned on the new course
        assert torch.isfinite(out.obs.proprio).all()
    assert ever_done.all()  # episode_len 3 truncates everything
    after = snap()
    moved = torch.zeros(E, dtype=torch.bool, device="cuda")
    for a, b in zip(before, after):
        moved |= (a != b).reshape(E, -1).any(1)
    assert moved.all()
    # deterministic: regenerating every env at its current episode reproduces the live scenes
    ref = qs.world.gen_obstacle_courses(5, E, [0.0, 0.0, 1.2], [cfg.goal_dist, 0.0, 1.5], cfg.density,
                                        cfg.style, r_quad=cfg.collision_radius, device="cuda",
                                        episode=env._meta[:, 1], episode_stride=4)
    for a, b in zip((ref.spheres, ref.boxes, ref.cylinders, ref.counts), after):
        assert torch.equal(a, b)
    env.check_errors()
    for s in qs.world.device_scene_to_scenes(sc, style=cfg.style):
        osc = O.Scene(prims={"spheres": s.prims.spheres, "boxes": s.prims.boxes,
                             "cylinders": s.prims.cylinders, "ground_z": 0.0},
                      bounds_lo=s.bounds_lo, bounds_hi=s.bounds_hi, spawn=s.spawn, goal=s.goal)
        assert O.grid_path_exists(osc)


def test_every_kernel_family_at_small_odd_sizes():
    """profiles/sanitize_workload.py: partial CTAs and tiny batches through the
    windows (TMA / cp.async rings), per-step path, scene gen, tiled/untiled
    ray casting at every tile width and both depth VJPs; no device error."""
    import importlib.util
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "sanitize_workload.py")
    spec = importlib.util.spec_from_file_location("sanitize_workload", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.main()


def test_regen_scene_gradient_uses_pre_regeneration_course():
    """with regen_scene_on_reset, a step whose env resets
    regenerates that env's course inside the step; the step's backward must
    still evaluate the obstacle penalty's SDF against the course the forward
    used.  Episodes of 4 steps: the loss over steps 0..3 must have the same
    gradient whether courses are regenerated at step 3 (and again at step 7,
    run but not in the loss) or never."""
    import paper_2509_10247_b200 as qs

    grads = []
    for regen, T in ((False, 4), (True, 4), (True, 8)):
        cfg = qs.TaskConfig(task="avoidance", dynamics="pm_continuous", n_envs=64, episode_len=4, density=0.25,
                            regen_scene_on_reset=regen)
        env = qs.make_task(cfg, strict=False)
        env.reset(seed=5)
        g = torch.Generator().manual_seed(9)
        acts = (torch.randn(T, env.N, 3, generator=g) * 0.4).cuda().requires_grad_(True)
        env.detach_states()
        loss = 0.0
        for t in range(T):
            out = env.step(acts[t])
            if t < 4:
                loss = loss + out.r_ctrl.mean() * 0.99 ** t
        (gr,) = torch.autograd.grad(-loss / 4, acts)
        grads.append(gr[:4].cpu())
        assert float(out.r_ctrl.abs().sum()) > 0
    assert float(grads[0].abs().max()) > 0
    assert torch.equal(grads[0], grads[1])
    assert torch.equal(grads[0], grads[2])


@pytest.mark.parametrize("case", ["full_imu_window", "pm_dr_window", "avoid_regen_steps"])
def test_sharding_invariance(case):
    """Multi-GPU readiness: N envs in one env equal two
    env_offset shards of N/2 bit for bit -- Philox spawns, DR draws, IMU noise
    and (regenerated) obstacle courses are keyed by global env id, so results
    do not depend on how envs are split over ranks."""
    import paper_2509_10247_b200 as qs
    from paper_2509_10247_b200.window import BpttWindow

    if case == "avoid_regen_steps":
        N, T = 512, 12
        kw = dict(task="avoidance", dynamics="pm_continuous", episode_len=4, density=0.2,
                  regen_scene_on_reset=True)
    elif case == "pm_dr_window":
        N, T = 2048, 16
        kw = dict(task="position", dynamics="pm_continuous", episode_len=5,
                  randomization=qs.world.RandomizationSpec(action_scale=(0.7, 1.0)))
    else:
        N, T = 2048, 16
        kw = dict(task="position", dynamics="full", episode_len=5, imu=qs.ImuSpec(0.1, 0.01, 0.01, 0.001))
    g = torch.Generator().manual_seed(4)
    A = 4 if kw["dynamics"] == "full" else 3
    acts = (torch.randn(T, N, A, generator=g) * 0.5).cuda()

    def run(n, off):
        env = qs.make_task(qs.TaskConfig(n_envs=n, **kw), strict=False, env_offset=off)
        env.reset(seed=7)
        a = acts[:, off:off + n]
        if case == "avoid_regen_steps":
            sph0 = env._scene.spheres.clone()
            recs = []
            with torch.no_grad():
                for t in range(T):
                    out = env.step(a[t])
                    recs.append((env._S.clone(), out.r_rl.clone(), out.terminated.clone(), out.obs.proprio.clone()))
            sc = env._scene
            assert not torch.equal(sph0, sc.spheres)  # the courses were regenerated at the resets
            return recs, (sc.spheres.clone(), sc.boxes.clone(), sc.cylinders.clone(), sc.counts.clone())
        win = BpttWindow(env, T)
        win.actions.copy_(a)
        _, ga = win.run()
        out = [win.S[1:].clone(), win.r.clone(), win.term.clone(), ga.clone()]
        if win.imu is not None:
            out.append(win.imu.clone())
        if win.dr is not None:
            out.append(win.dr[1:].clone())
        return out, None

    full, sc_full = run(N, 0)
    h0, sc0 = run(N // 2, 0)
    h1, sc1 = run(N // 2, N // 2)
    if case == "avoid_regen_steps":
        for (Sf, rf, tf, of), (S0, r0, t0, o0), (S1, r1, t1, o1) in zip(full, h0, h1):
            assert torch.equal(Sf, torch.cat([S0, S1], 1))
            assert torch.equal(rf, torch.cat([r0, r1])) and torch.equal(tf, torch.cat([t0, t1]))
            assert torch.equal(of, torch.cat([o0, o1]))
        for a, b, c in zip(sc_full, sc0, sc1):
            k = min(a.shape[1], b.shape[1]) if a.dim() > 2 else None
            assert torch.equal(a[:N // 2, :k] if k else a[:N // 2], b[:, :k] if k else b)
            assert torch.equal(a[N // 2:, :k] if k else a[N // 2:], c[:, :k] if k else c)
        return
    # dL/d(actions) carries the loss's 1/(T N) factor: the halves' gradients
    # are exactly twice the full batch's (a power-of-two scale commutes with
    # every rounding of the linear VJP chain)
    full[3] = full[3] * 2
    # window buffers: rows are the last axis before the per-row payload
    for f, a, b in zip(full, h0, h1):
        if f.dim() == 4:  # S (T, NP, N, 4)
            assert torch.equal(f, torch.cat([a, b], 2))
        elif f.shape[1] == 3 and f.dim() == 3:  # r (T, 3, N)
            assert torch.equal(f, torch.cat([a, b], 2))
        else:  # (T, N, ...)
            assert torch.equal(f, torch.cat([a, b], 1))


def test_device_race_tracks_follow_reference_distribution():
    """qs_gen_race_track (q/world.py:347-379 on the GPU, Philox): the track
    geometry the reference generates -- consecutive gate spacing in [4, spread]
    along the running heading, heading turns within +-pi/6 after the first
    gate, heights U(1, 2.5), normals = travel direction, spawn (0,0,1.5), goal
    at the last gate, bounds = extent +-5 m with floor 0 and ceiling >= 4 --
    with the reference's first moments; deterministic and keyed by global env
    id; 16,384 tracks per launch."""
    import paper_2509_10247_b200 as qs
    from oracle import quadsim_oracle as O

    E, G, spread = 16384, 5, 10.0
    sc = qs.world.gen_race_tracks(3, E, G, spread)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        qs.world.gen_race_tracks(4, E, G, spread, out=sc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"\n16,384 race tracks: {ms * 1e3:.1f} us per batch")
    assert ms < 10.0
    sc = qs.world.gen_race_tracks(3, E, G, spread)
    gt = sc.gates.double().cpu().numpy()
    c, n = gt[..., 0:3], gt[..., 4:7]
    prev = np.concatenate([np.tile([[[0.0, 0.0, 1.5]]], (E, 1, 1)), c[:, :-1]], 1)
    step = c[..., :2] - prev[..., :2]
    spacing = np.linalg.norm(step, axis=-1)
    assert spacing.min() >= 4.0 - 1e-4 and spacing.max() <= spread + 1e-4
    np.testing.assert_allclose(step / spacing[..., None], n[..., :2], atol=1e-4)  # normal = travel direction
    assert np.abs(n[..., 2]).max() == 0.0 and np.allclose(n[:, 0], [1.0, 0.0, 0.0], atol=1e-6)
    head = np.arctan2(n[..., 1], n[..., 0])
    turn = np.angle(np.exp(1j * np.diff(head, axis=1)))
    assert np.abs(turn).max() <= np.pi / 6 + 1e-5
    assert c[..., 2].min() >= 1.0 and c[..., 2].max() <= 2.5
    assert np.all(gt[..., 3] == np.float32(0.8)) and np.all(gt[..., 7] == np.float32(0.3))
    # first moments against the reference generator (the oracle restates it)
    ref = [O.gen_race_track(s, G, spread) for s in range(2000)]
    rc = np.stack([[g[0] for g in t.gates] for t in ref])
    rprev = np.concatenate([np.tile([[[0.0, 0.0, 1.5]]], (2000, 1, 1)), rc[:, :-1]], 1)
    rsp = np.linalg.norm(rc[..., :2] - rprev[..., :2], axis=-1)
    assert abs(spacing.mean() - rsp.mean()) < 0.1 and abs(spacing.std() - rsp.std()) < 0.1
    assert abs(c[..., 2].mean() - rc[..., 2].mean()) < 0.03
    bd = sc.bounds.double().cpu().numpy()
    sg = sc.spawn_goal.double().cpu().numpy()
    pts = np.concatenate([c, np.tile([[[0.0, 0.0, 1.5]]], (E, 1, 1))], 1)
    np.testing.assert_allclose(bd[:, 0, :2], pts[..., :2].min(1) - 5.0, atol=1e-4)
    np.testing.assert_allclose(bd[:, 1, :2], pts[..., :2].max(1) + 5.0, atol=1e-4)
    assert np.all(bd[:, 0, 2] == 0.0) and np.all(bd[:, 1, 2] >= 4.0)
    np.testing.assert_allclose(sg[:, 1, :3], c[:, -1], atol=0)
    assert np.all(sg[:, 0, :3] == [0.0, 0.0, 1.5])
    # deterministic, and keyed by global env id (sharding-invariant)
    again = qs.world.gen_race_tracks(3, E, G, spread)
    half = qs.world.gen_race_tracks(3, E // 2, G, spread, env_offset=E // 2)
    assert torch.equal(again.gates, sc.gates) and torch.equal(half.gates, sc.gates[E // 2:])


def test_racing_env_regenerates_tracks_on_reset():
    """regen_scene_on_reset for racing: a done env gets a new device-generated
    track keyed by its new episode; envs that did not reset keep theirs."""
    import paper_2509_10247_b200 as qs

    cfg = qs.TaskConfig(task="racing", dynamics="pm_continuous", n_envs=256, episode_len=3, n_gates=4,
                        regen_scene_on_reset=True)
    env = qs.make_task(cfg, strict=False)
    env.reset(seed=12)
    g0 = env.gate_centers.clone()
    with torch.no_grad():
        for _ in range(3):
            out = env.step(torch.zeros(256, 3, device="cuda"))
    done = out.done.cpu().numpy()
    assert done.all()  # truncation at episode_len
    g1 = env.gate_centers
    changed = (g1 != g0).flatten(1).any(1).cpu().numpy()
    assert changed.all()
    assert torch.equal(env.goals, g1[:, 0])  # respawned toward the new first gate
