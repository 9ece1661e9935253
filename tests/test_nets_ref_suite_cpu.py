"""The reference's own network / optimiser / container tests
(pkg/tests/test_nets.py), re-run against the torch modules (fp64, CPU)."""

import math

import numpy as np
import pytest
import torch


def small_policy(recurrent=True, visual=None, seed=0):
    from paper_2509_10247_b200 import nets

    arch = nets.PolicyArch(proprio_dim=5, action_dim=3, visual=visual, recurrent=recurrent, hidden=8,
                           mlp=(16, 16), conv_feat=6)
    return nets.PolicyNet(arch, np.random.default_rng(seed)).double()


def central_diff(f, x, h_scale=1e-6):  # pkg/tests/oracles.py:15-30
    g = np.zeros_like(x)
    for i in range(x.size):
        h = h_scale * (1.0 + abs(x[i]))
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        g[i] = (f(xp) - f(xm)) / (2 * h)
    return g


def test_zero_weights_give_bias_outputs():  # :19-28
    from paper_2509_10247_b200 import nets

    pol = small_policy(recurrent=False)
    with torch.no_grad():
        for _, (p, _t) in nets.ref_params(pol).items():
            p.zero_()
        pol.mu.b.copy_(torch.tensor([0.3, -0.2, 0.1]))
        pol.sig.b.fill_(-0.7)
    mu, logs, _ = pol(torch.zeros(4, 5, dtype=torch.float64))
    np.testing.assert_allclose(mu.detach().numpy(), np.broadcast_to([0.3, -0.2, 0.1], (4, 3)))
    np.testing.assert_allclose(np.exp(logs.detach().numpy()), np.full((4, 3), np.exp(-0.7)))


def test_policy_forward_deterministic():  # :31-38
    pol = small_policy()
    x = torch.as_tensor(np.random.default_rng(1).normal(size=(3, 5)))
    h = pol.initial_hidden(3).double()
    np.testing.assert_array_equal(pol(x, None, h)[0].detach().numpy(), pol(x, None, h)[0].detach().numpy())


def test_policy_gradcheck_every_weight():  # :41-72
    from paper_2509_10247_b200 import nets

    pol = small_policy(recurrent=True)
    rng = np.random.default_rng(3)
    x = torch.as_tensor(rng.normal(size=(2, 5)))
    h0 = torch.as_tensor(rng.normal(size=(2, 8)) * 0.3)

    def out():
        mu, logs, h = pol(x, None, h0)
        return mu.sum() + logs.sum() + 0.5 * h.sum()

    pol.zero_grad()
    out().backward()
    for name, (p, _t) in nets.ref_params(pol).items():
        base = p.detach().clone()

        def f(w, p=p, base=base):
            with torch.no_grad():
                p.copy_(torch.as_tensor(w).reshape(base.shape))
                v = float(out())
                p.copy_(base)
            return v

        g_fd = central_diff(f, base.numpy().ravel().copy(), 1e-5)
        np.testing.assert_allclose(p.grad.numpy().ravel(), g_fd, rtol=1e-4, atol=1e-6, err_msg=name)


def test_conv_encoder_shapes_and_gradflow():  # :75-85
    visual = {"kind": "depth", "height": 9, "width": 16, "max_range": 10.0}
    pol = small_policy(recurrent=False, visual=visual)
    img = torch.as_tensor(np.random.default_rng(5).uniform(0, 10, size=(4, 9, 16)))
    mu, _, _ = pol(torch.zeros(4, 5, dtype=torch.float64), img)
    assert tuple(mu.shape) == (4, 3)
    mu.sum().backward()
    assert float(pol.enc.k1.grad.abs().sum()) > 0 and float(pol.enc.out.W.grad.abs().sum()) > 0


def test_conv_encoder_rejects_tiny_images():  # :88-90
    from paper_2509_10247_b200 import nets

    with pytest.raises(ValueError, match="too small"):
        nets.ConvEncoder(4, 4, 8, np.random.default_rng(0))


def test_hidden_reset_makes_output_independent_of_history():  # :93-103
    pol = small_policy(recurrent=True)
    x = torch.as_tensor(np.random.default_rng(7).normal(size=(2, 5)))
    h_a = torch.as_tensor(np.random.default_rng(8).normal(size=(2, 8)))
    done = torch.tensor([True, True])
    h_a = torch.where(done[:, None], torch.zeros_like(h_a), h_a)
    np.testing.assert_array_equal(pol(x, None, h_a)[0].detach().numpy(),
                                  pol(x, None, torch.zeros(2, 8, dtype=torch.float64))[0].detach().numpy())


def test_gru_gradcheck():  # :106-126
    from paper_2509_10247_b200 import nets

    cell = nets.GRUCell(4, 6, np.random.default_rng(11)).double()
    rng = np.random.default_rng(12)
    x0 = rng.normal(size=(2, 4))
    h0 = torch.as_tensor(rng.normal(size=(2, 6)) * 0.5)
    xv = torch.as_tensor(x0).requires_grad_(True)
    torch.tanh(cell(xv, h0)).sum().backward()
    f = lambda xf: float(torch.tanh(cell(torch.as_tensor(xf.reshape(2, 4)), h0)).sum().detach())  # noqa: E731
    np.testing.assert_allclose(xv.grad.numpy(), central_diff(f, x0.ravel()).reshape(2, 4), rtol=1e-6, atol=1e-8)


def _adam(params, lr):
    return torch.optim.Adam(params, lr=lr)


def test_adam_zero_grad_and_zero_lr_noop():  # :132-143
    w = torch.nn.Parameter(torch.tensor([1.0, -2.0], dtype=torch.float64))
    opt = _adam([w], 1e-2)
    w.grad = torch.zeros(2, dtype=torch.float64)
    opt.step()
    np.testing.assert_array_equal(w.detach().numpy(), [1.0, -2.0])
    w2 = torch.nn.Parameter(torch.tensor([1.0, -2.0], dtype=torch.float64))
    opt2 = _adam([w2], 0.0)
    w2.grad = torch.tensor([0.5, 0.5], dtype=torch.float64)
    opt2.step()
    np.testing.assert_array_equal(w2.detach().numpy(), [1.0, -2.0])


def test_adam_matches_hand_computed_sequence():  # :146-154 (oracles.adam_ref)
    grads = [0.3, -0.1, 0.25]
    x = torch.nn.Parameter(torch.tensor([1.5], dtype=torch.float64))
    opt = _adam([x], 0.01)
    for g in grads:
        x.grad = torch.tensor([g], dtype=torch.float64)
        opt.step()
    m = v = 0.0
    e = 1.5
    for t, g in enumerate(grads, start=1):
        m = 0.9 * m + 0.1 * g
        v = 0.999 * v + 0.001 * g * g
        e -= 0.01 * (m / (1 - 0.9 ** t)) / (math.sqrt(v / (1 - 0.999 ** t)) + 1e-8)
    assert float(x.detach()) == pytest.approx(e, rel=1e-14)


def test_adam_grad_clip():  # :157-169
    from paper_2509_10247_b200.train import clip_grads_

    x = torch.nn.Parameter(torch.zeros(1, dtype=torch.float64))
    opt = _adam([x], 0.1)
    x.grad = torch.tensor([100.0], dtype=torch.float64)
    gnorm = clip_grads_([x], 1.0)
    opt.step()
    assert float(gnorm) == pytest.approx(100.0)
    x2 = torch.nn.Parameter(torch.zeros(1, dtype=torch.float64))
    opt2 = _adam([x2], 0.1)
    x2.grad = torch.tensor([1.0], dtype=torch.float64)
    opt2.step()
    np.testing.assert_allclose(x.detach().numpy(), x2.detach().numpy(), rtol=1e-12)


def test_container_forward_bit_exact_after_round_trip(tmp_path):  # :175-205
    from paper_2509_10247_b200 import nets

    pol = small_policy(seed=3)
    meta = {"observation_spec": {"proprio_dim": 5}, "architecture": {"hidden": 8}}
    nets.save_container(str(tmp_path / "c1"), {"policy": pol}, meta)
    sets, manifest = nets.read_container(str(tmp_path / "c1"))
    assert manifest["observation_spec"] == {"proprio_dim": 5}
    p1 = small_policy(seed=99)
    nets.load_into(p1, sets["policy"])
    nets.save_container(str(tmp_path / "c2"), {"policy": p1}, {})
    sets2, _ = nets.read_container(str(tmp_path / "c2"))
    p2 = small_policy(seed=98)
    nets.load_into(p2, sets2["policy"])
    x = torch.as_tensor(np.random.default_rng(0).normal(size=(10, 5)))
    h = torch.zeros(10, 8, dtype=torch.float64)
    np.testing.assert_array_equal(p1(x, None, h)[0].detach().numpy(), p2(x, None, h)[0].detach().numpy())
    for k in sets["policy"]:
        np.testing.assert_array_equal(sets["policy"][k], sets2["policy"][k])


def test_container_bad_manifest(tmp_path):  # :218-222
    from paper_2509_10247_b200 import nets

    (tmp_path / "ckpt").mkdir()
    (tmp_path / "ckpt" / "manifest.json").write_text("{not json")
    with pytest.raises(nets.IntegrityError):
        nets.read_container(str(tmp_path / "ckpt"))
