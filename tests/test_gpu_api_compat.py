"""The reference's convenience API on the kernels: single-ray known answers
(pkg/tests/test_sensors.py:49-75, fp32 tolerance), functional dynamics steps,
scene SDF, learner names and greedy evaluation."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_ray_primitive_known_answers():
    from paper_2509_10247_b200 import sensors as sn

    assert sn.ray_primitive([0, 0, 0], [1, 0, 0], ("sphere", [5, 0, 0, 1])) == pytest.approx(4.0, abs=1e-5)
    assert sn.ray_primitive([0, 0, 0], [1, 0, 0], ("box", [2.5, 0, 0, 0.5, 1, 1])) == pytest.approx(2.0, abs=1e-5)
    assert sn.ray_primitive([0, 0, 0], [1, 0, 0], ("cylinder", [4, 0, 0, 1, 2])) == pytest.approx(3.0, abs=1e-5)
    assert sn.ray_primitive([4, 0, 10], [0, 0, -1], ("cylinder", [4, 0, 0, 1, 2])) == pytest.approx(8.0, abs=1e-5)
    assert sn.ray_primitive([0, 0, 2], [0, 0, -1], ("ground", -1.0)) == pytest.approx(3.0, abs=1e-5)
    assert sn.ray_primitive([0, 0, 2], [0, 0, 1], ("ground", -1.0)) is None
    with pytest.raises(sn.SensorContractError):
        sn.ray_primitive([0, 0, 0], [2, 0, 0], ("sphere", [5, 0, 0, 1]))


@pytest.mark.parametrize("name", ["full", "simplified", "pm_continuous", "pm_discrete"])
def test_functional_steps_equal_model_step(name):
    from paper_2509_10247_b200 import dynamics as dyn

    params = dyn.QuadParams()
    m = dyn.make_model(name, params)
    B = 64
    g = torch.Generator().manual_seed(3)
    st = m.init_state(torch.randn(B, 3, generator=g).cuda(), torch.randn(B, 3, generator=g).cuda() * 0.5)
    act = (torch.rand(B, m.action_dim, generator=g).cuda() * 2 - 1) * 2.0
    ref = m.step(st, act)
    if name in ("full", "simplified"):
        got = getattr(dyn, "step_" + name)(st, act[:, 0], act[:, 1:], params)
    else:
        got = getattr(dyn, "step_" + name)(st, act, params)
    for k, v in ref.fields().items():
        torch.testing.assert_close(got.fields()[k], v)


def test_scene_sdf_matches_oracle():
    from oracle import quadsim_oracle as O
    from paper_2509_10247_b200 import world as wd

    scn = wd.gen_obstacle_course(4, [0.0, 0.0, 1.2], [8.0, 0.0, 1.5], 0.6)
    pts = np.random.default_rng(2).uniform([-1, -4, 0], [9, 4, 3], size=(500, 3))
    got = wd.scene_sdf(scn, pts).cpu().numpy()
    prims = O.pack_primitives([{"spheres": scn.prims.spheres, "boxes": scn.prims.boxes,
                                "cylinders": scn.prims.cylinders, "ground_z": scn.prims.ground_z}])
    ref = O.sdf(pts, O.prims_take(prims, np.zeros(len(pts), dtype=int)))
    np.testing.assert_allclose(got, ref, atol=2e-5)


def test_learner_names_and_evaluate():
    import paper_2509_10247_b200 as qs
    from paper_2509_10247_b200 import train

    assert train.ALGOS == ("bptt", "shac", "sha2c", "ppo")
    env = qs.make_task(qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=256, episode_len=20),
                       strict=False)
    env.reset(seed=1)
    lr = train.SHAC(env, train.LearnerOptions(horizon=4, critic_iters=1))
    assert lr.opts.algo == "shac" and type(lr).__name__ == "SHAC"
    lr.update()
    res = train.evaluate(env, lr.policy, n_episodes=300, seed=5)
    assert res["episodes"] >= 300 and 0.0 <= res["success_rate"] <= 1.0
    lo, hi = res["success_ci95"]
    assert 0.0 <= lo <= res["success_rate"] <= hi <= 1.0
    assert train.wilson_interval(0, 0) == (0.0, 1.0)


def test_strict_step_raises_before_mutating():
    """strict=True: qs_task_validate + the guarded step kernel, one host read of
    the error word: a rejected step leaves every env buffer untouched (the
    reference raises before stepping, q/tasks.py:551-558); the lowest bad
    action row wins over any bad state row (action check first)."""
    import numpy as np

    import paper_2509_10247_b200 as qs

    env = qs.make_task(qs.TaskConfig(task="position", dynamics="full", n_envs=64, episode_len=3,
                                     imu=qs.ImuSpec(0.1, 0.01, 0.01, 0.001)))
    env.reset(seed=1)
    for _ in range(2):
        env.step(torch.zeros(64, 4, device="cuda"))
    snap = [t.clone() for t in (env._S, env._goal, env._peff, env._meta, env._ep_ret, env._imu_bias, env._stats)]
    bad = torch.zeros(64, 4, device="cuda")
    bad[9, 2] = float("inf")
    bad[40, 0] = float("nan")
    with pytest.raises(qs.TaskContractError, match="row 9$"):
        env.step(bad)
    for a, b in zip(snap, (env._S, env._goal, env._peff, env._meta, env._ep_ret, env._imu_bias, env._stats)):
        assert torch.equal(a, b)
    # non-finite state (q/dynamics.py:130-133), reported when the actions are fine
    p = env.state.p.clone()
    p[5, 1] = float("nan")
    p[7, 0] = float("inf")
    env.state = qs.QuadState(p=p, v=env.state.v, q=env.state.q, w=env.state.w)
    with pytest.raises(qs.dynamics.ContractError, match="row 5"):
        env.step(torch.zeros(64, 4, device="cuda"))
    with pytest.raises(qs.TaskContractError, match="row 9$"):  # actions first
        env.step(bad)
    # a clean env keeps stepping after a rejected step
    env.reset(seed=1)
    out = env.step(torch.zeros(64, 4, device="cuda"))
    assert np.isfinite(out.r_ctrl.cpu().numpy()).all()


def test_task_step_is_a_registered_torch_op():
    """quadsim::task_step is a dispatcher op with CUDA, Meta and Autograd
    kernels: FakeTensor tracing sees its output shapes; eager calls carry
    the C++ autograd node whose backward is the analytic VJP."""
    from torch._subclasses.fake_tensor import FakeTensorMode

    import paper_2509_10247_b200 as qs
    from paper_2509_10247_b200 import _lib as L

    ops = L.ops()
    assert hasattr(ops, "task_step") and hasattr(L.fast_ops(), "task_step")
    env = qs.make_task(qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=32), strict=False)
    env.reset(seed=2)
    raw = torch.zeros(32, 3, device="cuda", requires_grad=True)
    out = env.step(raw)
    assert out.r_ctrl.grad_fn is not None and "TaskStepFn" in out.r_ctrl.grad_fn.name()
    (g,) = torch.autograd.grad(out.r_ctrl.sum(), raw)
    assert g.shape == (32, 3) and bool(torch.isfinite(g).all())
    E = env._empty
    with FakeTensorMode(allow_non_fake_inputs=True) as fm:
        S = fm.from_tensor(env._S)
        r = fm.from_tensor(torch.zeros(32, 3, device="cuda"))
        bufs = [env._goal, env._peff, E, env._meta, env._ep_ret, E, env._stats, env._err]
        res = ops.task_step(env._cfg_blob, env._scene.tensors(), S, r, bufs, None, False, False, env._cfg.proprio_dim)
    assert [tuple(t.shape) for t in res[:3]] == [tuple(env._S.shape), (32, 9), (32,)]
