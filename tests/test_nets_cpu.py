"""Learner networks and PPO pieces on CPU against the reference's own outputs
(tests/golden/nets_ppo.npz and the weight container in
tests/golden/nets_container/, written by make_golden.py gen_nets_ppo from
q/nets.py and q/learners.py)."""

import os
import shutil

import numpy as np
import pytest
import torch

from golden_utils import GOLDEN, load

CDIR = os.path.join(GOLDEN, "nets_container")


def _depth_arch(nets):
    return nets.PolicyArch(proprio_dim=9, action_dim=3,
                           visual={"kind": "depth", "height": 12, "width": 16, "max_range": 10.0},
                           recurrent=True, hidden=16, mlp=(32, 32), conv_feat=8,
                           input_scale=tuple(np.linspace(0.2, 1.0, 9)))


def _lidar_arch(nets):
    return nets.PolicyArch(proprio_dim=12, action_dim=4, visual={"kind": "lidar", "rays": 24, "max_range": 20.0},
                           recurrent=False, hidden=16, mlp=(32, 32), conv_feat=8)


def test_initial_weights_equal_the_reference_stream():
    """Same seed -> the reference's initial arrays (q/learners.py:145-169)."""
    from paper_2509_10247_b200 import nets

    z = load("nets_ppo")
    rng = np.random.default_rng([5 & 0x7FFFFFFF, 0x11])
    pol = nets.PolicyNet(_depth_arch(nets), rng)
    val = nets.ValueNet(13, rng, hidden=(32, 32), input_scale=tuple(np.linspace(0.5, 1.5, 13)))
    for prefix, mod in (("init_depth/", pol), ("init_value/", val)):
        names = [k[len(prefix):] for k in z.files if k.startswith(prefix)]
        got = nets.ref_params(mod)
        assert sorted(names) == sorted(got)
        for n in names:
            np.testing.assert_array_equal(got[n][0].detach().numpy(), z[prefix + n].astype(np.float32))


def test_container_forward_matches_reference():
    """Weights read from a reference-written container reproduce the reference
    forward (policy with conv encoder + GRU, LiDAR policy, critic) in fp64."""
    from paper_2509_10247_b200 import nets

    z = load("nets_ppo")
    sets, manifest = nets.read_container(CDIR)
    assert manifest["format_version"] == 1
    pol = nets.PolicyNet(_depth_arch(nets)).double()
    nets.load_into(pol, sets["policy"])
    mu, ls, h1 = pol(torch.as_tensor(z["d_pro"]), torch.as_tensor(z["d_img"]), torch.as_tensor(z["d_h0"]))
    np.testing.assert_allclose(mu.detach().numpy(), z["d_mu"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(ls.detach().numpy(), z["d_ls"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(h1.detach().numpy(), z["d_h1"], rtol=1e-10, atol=1e-12)
    pl = nets.PolicyNet(_lidar_arch(nets)).double()
    nets.load_into(pl, sets["policy_lidar"])
    mu, ls, h = pl(torch.as_tensor(z["l_pro"]), torch.as_tensor(z["l_scan"]))
    assert h is None
    np.testing.assert_allclose(mu.detach().numpy(), z["l_mu"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(ls.detach().numpy(), z["l_ls"], rtol=1e-10, atol=1e-12)
    val = nets.ValueNet(13, hidden=(32, 32), input_scale=tuple(np.linspace(0.5, 1.5, 13))).double()
    nets.load_into(val, sets["value"])
    np.testing.assert_allclose(val(torch.as_tensor(z["v_in"])).detach().numpy(), z["v_out"], rtol=1e-10,
                               atol=1e-12)


def test_container_round_trip_is_byte_identical(tmp_path):
    """load -> save writes the reference's blob byte for byte, with the same
    layer table (names, shapes, activation tags, offsets)."""
    from paper_2509_10247_b200 import nets
    import json

    sets, manifest = nets.read_container(CDIR)
    pol = nets.PolicyNet(_depth_arch(nets))
    val = nets.ValueNet(13, hidden=(32, 32))
    pl = nets.PolicyNet(_lidar_arch(nets))
    nets.load_into(pol, sets["policy"])
    nets.load_into(val, sets["value"])
    nets.load_into(pl, sets["policy_lidar"])
    out = str(tmp_path / "c")
    nets.save_container(out, {"policy": pol, "value": val, "policy_lidar": pl}, {"note": manifest["note"]})
    with open(os.path.join(CDIR, "weights.bin"), "rb") as f, open(os.path.join(out, "weights.bin"), "rb") as g:
        assert f.read() == g.read()
    m2 = json.load(open(os.path.join(out, "manifest.json")))
    assert m2["layers"] == manifest["layers"] and m2["total_floats"] == manifest["total_floats"]


def test_container_integrity_errors(tmp_path):
    from paper_2509_10247_b200 import nets

    bad = tmp_path / "bad"
    shutil.copytree(CDIR, bad)
    with open(bad / "weights.bin", "r+b") as f:
        f.truncate(100)
    with pytest.raises(nets.IntegrityError, match="manifest expects"):
        nets.read_container(str(bad))
    (bad / "manifest.json").write_text('{"format_version": 2}')
    with pytest.raises(nets.IntegrityError, match="unsupported container version"):
        nets.read_container(str(bad))
    sets, _ = nets.read_container(CDIR)
    with pytest.raises(nets.IntegrityError, match="mismatch"):
        nets.load_into(nets.PolicyNet(_lidar_arch(nets)), sets["policy"])


def test_ppo_pieces_match_reference():
    """GAE with cuts, advantage normalisation, running return-std scaling over
    three windows (stateful), tanh-squashed log-prob."""
    from paper_2509_10247_b200 import train

    z = load("nets_ppo")
    t = lambda k: torch.as_tensor(z[k])  # noqa: E731
    adv, rets = train.gae_advantages(t("g_r"), t("g_values"), t("g_boot"), t("g_done"), 0.99, 0.95)
    np.testing.assert_allclose(adv.numpy(), z["g_adv"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(rets.numpy(), z["g_rets"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(train.normalize(adv).numpy(), z["g_norm"], rtol=1e-12, atol=1e-12)
    sc = train.ReturnScaler(z["g_r"].shape[1], 0.99, torch.device("cpu"))
    for u in range(3):
        got = sc(t(f"s_r{u}"), t(f"s_done{u}"))
        np.testing.assert_allclose(got.numpy(), z[f"s_scaled{u}"], rtol=1e-12, atol=1e-12)
    lp = train.ppo_log_prob(t("lp_mu"), t("lp_logs"), t("lp_a"), t("lp_half"))
    np.testing.assert_allclose(lp.numpy(), z["lp"], rtol=1e-12, atol=1e-12)
    # and the reference test's direct formula (pkg/tests/test_learners.py:208-221)
    mu, logs, a, half = (z[k] for k in ("lp_mu", "lp_logs", "lp_a", "lp_half"))
    zz = (a - mu) / np.exp(logs)
    base = -0.5 * np.sum(zz ** 2, -1) - np.sum(logs, -1) - 1.5 * np.log(2 * np.pi)
    corr = np.sum(np.log(half) + np.log1p(-np.tanh(a) ** 2), -1)
    np.testing.assert_allclose(lp.numpy(), base - corr, rtol=1e-9)


def test_c5_policy_has_the_reference_parameter_count():
    """GRU-64 + tanh MLP 128^2 (+ linear 128) + heads on the pm proprio: the
    56,518 parameters SURVEY §8d counts for the reference; critic 18,561."""
    from paper_2509_10247_b200 import nets

    rng = np.random.default_rng([0, 0x11])
    pol = nets.PolicyNet(nets.PolicyArch(proprio_dim=9, action_dim=3), rng)
    assert pol.n_params() == 56518
    # privileged state: 14 features (q/tasks.py:465-545)
    val = nets.ValueNet(14, rng)
    assert val.n_params() == 18561


def test_quat_to_matrix_np_matches_oracle():
    from oracle import quadsim_oracle as O
    from paper_2509_10247_b200 import dynamics as dyn

    q = np.random.default_rng(1).normal(size=(16, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    np.testing.assert_allclose(dyn.quat_to_matrix_np(q), O.quat_to_matrix(q), rtol=1e-14, atol=1e-14)
