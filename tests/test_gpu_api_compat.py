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
