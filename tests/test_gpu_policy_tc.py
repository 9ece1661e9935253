"""The policy trunk + Gaussian heads on tcgen05 (qs_policy_trunk_fwd/_bwd,
q/nets.py:198-256) against torch autograd in fp32 on the same weights: the
forward y, dL/dh and every parameter gradient to bf16-operand accuracy."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ptrs(*ts):
    from paper_2509_10247_b200 import _lib as L

    return [L.ptr(t) for t in ts]


@pytest.mark.parametrize("n_out,N", [(6, 128 * 148 + 77), (8, 1000)])
def test_policy_trunk_fwd_bwd_match_autograd(n_out, N):
    from paper_2509_10247_b200 import _lib as L

    g = torch.Generator().manual_seed(n_out)
    r = lambda *s, sc=1.0: (torch.randn(*s, generator=g) * sc).cuda()  # noqa: E731
    W0, b0 = r(64, 128, sc=0.15), r(128, sc=0.1)
    W1, b1 = r(128, 128, sc=0.1), r(128, sc=0.1)
    W2, b2 = r(128, 128, sc=0.1), r(128, sc=0.1)
    Wh, bh = r(128, n_out, sc=0.1), r(n_out, sc=0.1)
    h = r(N, 64, sc=0.8)
    dy = r(N, n_out)
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    y = torch.empty(N, n_out, device="cuda")
    L.check(L.lib().qs_policy_trunk_fwd(N, n_out, *_ptrs(h, W0, b0, W1, b1, W2, b2, Wh, bh, y), n_sm,
                                        L.stream_handle()), "fwd")
    params = [W0, b0, W1, b1, W2, b2, Wh, bh]
    grads = [torch.full_like(p, 7.0) for p in params]  # overwritten, not accumulated
    dh = torch.empty_like(h)
    work = torch.empty(L.lib().qs_policy_work_floats(0, n_sm), device="cuda")
    L.check(L.lib().qs_policy_trunk_bwd(N, n_out, None, *_ptrs(h, dy), 0,
                                        *_ptrs(W0, b0, W1, b1, W2, b2, Wh, dh, grads[0], grads[1], grads[2], grads[3],
                                               grads[4], grads[5], grads[6], grads[7], work), work.numel(), n_sm,
                                        L.stream_handle()), "bwd")
    leaves = [p.clone().requires_grad_(True) for p in params]
    hl = h.clone().requires_grad_(True)
    w0, c0, w1, c1, w2, c2, wh, ch = leaves
    z = torch.tanh(torch.tanh(torch.tanh(hl @ w0 + c0) @ w1 + c1) @ w2 + c2)
    y_ref = z @ wh + ch
    (y_ref * dy).sum().backward()

    def rel(a, b):
        return float((a - b).abs().max()) / (float(b.abs().max()) + 1e-12)

    assert rel(y, y_ref.detach()) < 2e-2, rel(y, y_ref.detach())
    assert rel(dh, hl.grad) < 3e-2, rel(dh, hl.grad)
    for name, a, b in zip(["W0", "b0", "W1", "b1", "W2", "b2", "Wh", "bh"], grads, [p.grad for p in leaves]):
        assert rel(a, b) < 3e-2, (name, rel(a, b))


def test_policynet_autocast_uses_trunk_kernels_and_matches_torch_path():
    """PolicyNet under bf16 autocast routes the trunk + heads through
    _TrunkFn; its outputs and parameter gradients agree with the torch bf16
    path (QS_POLICY_TRUNK=torch) of the same module."""
    import numpy as np

    from paper_2509_10247_b200 import nets

    arch = nets.PolicyArch(proprio_dim=10, action_dim=3, recurrent=True, hidden=64, mlp=(128, 128),
                           input_scale=tuple(np.linspace(0.3, 1.5, 10)))
    pol = nets.PolicyNet(arch, np.random.default_rng(3)).cuda()
    x = torch.randn(3000, 10, device="cuda")
    h0 = torch.randn(3000, 64, device="cuda") * 0.5
    reset = torch.rand(3000, device="cuda") < 0.2

    def run(fused):
        old = nets.FUSED_TRUNK
        nets.FUSED_TRUNK = fused
        try:
            pol.zero_grad(set_to_none=True)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                mu, ls, h = pol(x, h=h0, h_reset=reset)
            (mu.square().sum() + (ls * 0.3).sum() + h.square().sum()).backward()
            return mu.detach(), ls.detach(), {k: p.grad.clone() for k, p in pol.named_parameters()}
        finally:
            nets.FUSED_TRUNK = old

    mu_f, ls_f, g_f = run(True)
    mu_t, ls_t, g_t = run(False)
    assert float((mu_f - mu_t).abs().max()) < 2e-2 * float(mu_t.abs().max()) + 1e-4
    assert float((ls_f - ls_t).abs().max()) < 2e-2 * float(ls_t.abs().max()) + 1e-4
    for k in g_t:
        d = float((g_f[k] - g_t[k]).abs().max())
        assert d < 5e-2 * float(g_t[k].abs().max()) + 1e-6, (k, d)


@pytest.mark.parametrize("n_in,N", [(10, 128 * 148 + 77), (16, 3000), (3, 500)])
def test_policy_gru_fwd_bwd_match_autograd(n_in, N):
    """qs_policy_gru_fwd (GRU cell + trunk + heads) and qs_policy_gru_bwd
    (the cell's backward) against fp32 autograd of the reference equations."""
    from paper_2509_10247_b200 import _lib as L

    g = torch.Generator().manual_seed(100 + n_in)
    r = lambda *s, sc=1.0: (torch.randn(*s, generator=g) * sc).cuda()  # noqa: E731
    Wi, bi, Wg, bg = r(n_in, 192, sc=0.3), r(192, sc=0.1), r(64, 192, sc=0.15), r(192, sc=0.1)
    W0, b0, W1, b1 = r(64, 128, sc=0.15), r(128, sc=0.1), r(128, 128, sc=0.1), r(128, sc=0.1)
    W2, b2, Wh, bh = r(128, 128, sc=0.1), r(128, sc=0.1), r(128, 6, sc=0.1), r(6, sc=0.1)
    x, h = r(N, n_in), r(N, 64, sc=0.6)
    gh = r(N, 64, sc=0.5)
    reset = (torch.rand(N, generator=g) < 0.1).cuda()  # rows whose carried h restarts at 0
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    h_out, y = torch.empty(N, 64, device="cuda"), torch.empty(N, 6, device="cuda")
    L.check(L.lib().qs_policy_gru_fwd(N, n_in, 6, None, *_ptrs(x, None, h, reset, Wi, bi, Wg, bg, W0, b0, W1, b1, W2,
                                                                b2, Wh, bh, h_out, y), 0, n_sm, L.stream_handle()),
            "gru fwd")
    # the same from the pre-converted bf16 weight image (bulk-copied by every CTA): same bits
    img = torch.empty(L.lib().qs_policy_image_bytes() // 2, dtype=torch.bfloat16, device="cuda")
    L.check(L.lib().qs_policy_pack_image(n_in, 6, *_ptrs(Wi, Wg, W0, W1, W2, Wh), 0, L.ptr(img), L.stream_handle()),
            "image")
    h_out2, y2 = torch.empty_like(h_out), torch.empty_like(y)
    L.check(L.lib().qs_policy_gru_fwd(N, n_in, 6, *_ptrs(img, x, None, h, reset, Wi, bi, Wg, bg, W0, b0, W1, b1, W2,
                                                          b2, Wh, bh, h_out2, y2), 0, n_sm, L.stream_handle()),
            "gru fwd img")
    assert torch.equal(h_out, h_out2) and torch.equal(y, y2)
    dx, dh = torch.empty_like(x), torch.empty_like(h)
    gr = [torch.full_like(t, 7.0) for t in (Wi, bi, Wg, bg)]  # overwritten, not accumulated
    work = torch.empty(L.lib().qs_policy_work_floats(1, n_sm), device="cuda")
    L.check(L.lib().qs_policy_gru_bwd(N, n_in, None, *_ptrs(x, None, h, reset, gh, None, Wi, bi, Wg, bg, dx, dh, *gr,
                                                            work),
                                      work.numel(), n_sm, L.stream_handle()), "gru bwd")
    # reproducible: a second pass (from the weight image) gives the same bits
    gr2 = [torch.zeros_like(t) for t in (Wi, bi, Wg, bg)]
    L.check(L.lib().qs_policy_gru_bwd(N, n_in, *_ptrs(img, x, None, h, reset, gh, None, Wi, bi, Wg, bg, dx, dh, *gr2,
                                                      work),
                                      work.numel(), n_sm, L.stream_handle()), "gru bwd")
    assert all(torch.equal(a, b) for a, b in zip(gr, gr2))
    leaves = [t.clone().requires_grad_(True) for t in (x, h, Wi, bi, Wg, bg)]
    xl, hl, wi, ci, wg, cg = leaves
    hm = torch.where(reset[:, None], torch.zeros_like(hl), hl)
    gi, gg = xl @ wi + ci, hm @ wg + cg
    rr = torch.sigmoid(gi[:, :64] + gg[:, :64])
    zz = torch.sigmoid(gi[:, 64:128] + gg[:, 64:128])
    nn = torch.tanh(gi[:, 128:] + rr * gg[:, 128:])
    h_ref = nn + zz * (hm - nn)
    z = torch.tanh(torch.tanh(torch.tanh(h_ref @ W0 + b0) @ W1 + b1) @ W2 + b2)
    y_ref = z @ Wh + bh
    (h_ref * gh).sum().backward()

    def rel(a, b):
        return float((a - b).abs().max()) / (float(b.abs().max()) + 1e-12)

    assert rel(h_out, h_ref.detach()) < 1e-2, rel(h_out, h_ref.detach())
    assert rel(y, y_ref.detach()) < 2e-2, rel(y, y_ref.detach())
    for name, a, b in zip(["dx", "dh", "Wi", "bi", "Wg", "bg"], [dx, dh, *gr], [t.grad for t in leaves]):
        assert rel(a, b) < 3e-2, (name, rel(a, b))


def test_policynet_recurrent_rollout_gradients_match_torch_path():
    """Four recurrent steps with the hidden state carried (reset mask mid-way,
    parameters packed once as the trainer does): the fused kernels' rollout
    loss and every parameter gradient against the torch bf16 path."""
    import numpy as np

    from paper_2509_10247_b200 import nets

    arch = nets.PolicyArch(proprio_dim=9, action_dim=3, recurrent=True, hidden=64, mlp=(128, 128),
                           input_scale=tuple(np.linspace(0.2, 2.0, 9)))
    pol = nets.PolicyNet(arch, np.random.default_rng(11)).cuda()
    g = torch.Generator(device="cuda").manual_seed(5)
    xs = [torch.randn(2048, 9, device="cuda", generator=g) for _ in range(4)]
    resets = [None, torch.rand(2048, device="cuda", generator=g) < 0.3, None,
              torch.rand(2048, device="cuda", generator=g) < 0.3]

    def rollout(fused):
        old = nets.FUSED_TRUNK
        nets.FUSED_TRUNK = fused
        try:
            pol.zero_grad(set_to_none=True)
            packed = pol.pack_weights() if fused else None
            h, loss = None, 0.0
            with torch.autocast("cuda", dtype=torch.bfloat16):
                for x, rs in zip(xs, resets):
                    mu, ls, h = pol(x, h=h, h_reset=rs, packed=packed)
                    loss = loss + (mu - 0.1).square().mean() + 0.2 * ls.mean() + 0.05 * h.square().mean()
            loss.backward()
            return float(loss.detach()), {k: p.grad.clone() for k, p in pol.named_parameters()}
        finally:
            nets.FUSED_TRUNK = old

    lf, gf = rollout(True)
    lt, gt = rollout(False)
    assert abs(lf - lt) < 2e-2 * abs(lt) + 1e-4, (lf, lt)
    for k in gt:
        d = float((gf[k] - gt[k]).abs().max())
        assert d < 6e-2 * float(gt[k].abs().max()) + 1e-6, (k, d, float(gt[k].abs().max()))
