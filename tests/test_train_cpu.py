"""Trainer host logic on CPU: TD-lambda against the reference's values and the
multi-rank gradient all-reduce over gloo (world_size 2)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_utils import load


def test_td_lambda_matches_reference():
    from paper_2509_10247_b200.train import td_lambda_targets

    z = load("learners")
    G = td_lambda_targets(torch.as_tensor(z["r"]), torch.as_tensor(z["values"]), torch.as_tensor(z["boot"]),
                          torch.as_tensor(z["done"]), 0.99, 0.95)
    np.testing.assert_allclose(G.numpy(), z["td"], rtol=1e-12, atol=1e-12)


def test_shard_envs_partitions_global_ids():
    from paper_2509_10247_b200.train import shard_envs

    for n, w in ((1048576, 8), (100, 3), (5, 8)):
        spans = [shard_envs(n, r, w) for r in range(w)]
        ids = np.concatenate([np.arange(a, b) for a, b in spans])
        assert np.array_equal(ids, np.arange(n))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_10247_b200.train import allreduce_mean_

    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(5, 7), torch.nn.Tanh(), torch.nn.Linear(7, 3))
    x = torch.randn(16, 5, generator=torch.Generator().manual_seed(100 + rank))  # rank-local data
    net(x).pow(2).mean().backward()
    local = [p.grad.clone() for p in net.parameters()]
    allreduce_mean_(list(net.parameters()))
    q.put((rank, [g.numpy() for g in local], [p.grad.numpy() for p in net.parameters()]))
    dist.barrier()
    dist.destroy_process_group()


def test_gradient_allreduce_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (loc, red)) for r, loc, red in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mean = [(a + b) / 2 for a, b in zip(res[0][0], res[1][0])]
    for r in (0, 1):
        for got, want in zip(res[r][1], mean):
            np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-7)
    # the two ranks had different local gradients and now agree exactly
    assert not np.allclose(res[0][0][0], res[1][0][0])
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)


def _scaler_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_10247_b200.train import ReturnScaler

    z = load("nets_ppo")
    N = z["s_r0"].shape[1]
    lo, hi = rank * N // world, (rank + 1) * N // world  # this rank's env shard
    sc = ReturnScaler(hi - lo, 0.99, torch.device("cpu"))
    outs = [sc(torch.as_tensor(z[f"s_r{u}"][:, lo:hi]), torch.as_tensor(z[f"s_done{u}"][:, lo:hi])).numpy()
            for u in range(3)]
    q.put((rank, lo, hi, outs))
    dist.barrier()
    dist.destroy_process_group()


def test_return_scaler_sharded_two_ranks_gloo():
    """PPO reward scaling over env shards on 2 ranks equals the reference's
    single-process scaling of the whole batch (moments merged by all-reduce)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() + 7) % 1000
    procs = [ctx.Process(target=_scaler_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    z = load("nets_ppo")
    for rank, lo, hi, outs in res:
        for u in range(3):
            np.testing.assert_allclose(outs[u], z[f"s_scaled{u}"][:, lo:hi], rtol=1e-10, atol=1e-12)


def test_td_lambda_k_steps_matches_reference():
    """SHA2C's k-step critic window (q/learners.py:95-113): the reference's own
    k=4 output (golden), its k=2 hand mixture (pkg/tests/test_learners.py:79-92)
    and the recorded-rollout N=2, T=4, k=4 case (:62-76)."""
    from paper_2509_10247_b200.train import LearnerOptions, td_lambda_targets

    z = load("learners")
    G = td_lambda_targets(torch.as_tensor(z["r"]), torch.as_tensor(z["values"]), torch.as_tensor(z["boot"]),
                          torch.as_tensor(z["done"]), 0.99, 0.95, 4)
    np.testing.assert_allclose(G.numpy(), z["td_k4"], rtol=1e-12, atol=1e-12)
    rng = np.random.default_rng(3)
    T, N = 6, 3
    r, values, boot = rng.normal(size=(T, N)), rng.normal(size=(T, N)), rng.normal(size=N)
    done = np.zeros((T, N), dtype=bool)
    lam, gamma = 0.9, 0.98
    got = td_lambda_targets(torch.as_tensor(r), torch.as_tensor(values), torch.as_tensor(boot),
                            torch.as_tensor(done), gamma, lam, 2).numpy()
    for t in range(T - 2):
        g1 = r[t] + gamma * values[t + 1]
        g2 = r[t] + gamma * r[t + 1] + gamma ** 2 * values[t + 2]
        np.testing.assert_allclose(got[t], (1 - lam) * g1 + lam * g2, rtol=1e-12)
    # k >= T is the full recursive mixture
    full = td_lambda_targets(torch.as_tensor(r), torch.as_tensor(values), torch.as_tensor(boot),
                             torch.as_tensor(done), gamma, lam)
    k6 = td_lambda_targets(torch.as_tensor(r), torch.as_tensor(values), torch.as_tensor(boot),
                           torch.as_tensor(done), gamma, lam, 6)
    assert torch.equal(full, k6)
    assert LearnerOptions().algo == "sha2c" and LearnerOptions(k_steps=4).k_steps == 4


def test_policy_pack_layout():
    """The fused policy step's flat parameter layout (nets._pack_offsets): the
    parameters of PolicyNet._fused_params back to back (the two heads as the
    planar blocks [W_mu | W_sigma], [b_mu | b_sigma] the kernels read), every
    matrix the kernels stage with 16-byte loads on a 4-float boundary, and
    pack_weights differentiable back to each parameter."""
    from paper_2509_10247_b200 import nets

    for n_in in (3, 9, 10, 16):
        arch = nets.PolicyArch(proprio_dim=n_in, action_dim=3, recurrent=True, hidden=64, mlp=(128, 128))
        pol = nets.PolicyNet(arch, np.random.default_rng(0))
        offs = nets._pack_offsets(n_in, 3)
        params = pol._fused_params()
        total = sum(p.numel() for p in params)
        o = 0
        for k, (off, n) in offs.items():
            assert off == o
            o += n
            if k in ("Wi", "Wg", "W0", "W1", "W2", "Wh"):
                assert off % 4 == 0, k
        assert o == total
        assert offs["Wh"][1] == pol.mu.W.numel() + pol.sig.W.numel() and offs["bh"][1] == 6
        wp = pol.pack_weights()
        assert wp.numel() == total and not hasattr(wp, "_qs_image")  # CPU: no kernel image
        # the planar head block: W_mu (128, 3) row-major, then W_sigma
        assert torch.equal(wp[offs["Wh"][0]:offs["Wh"][0] + 384].view(128, 3), pol.mu.W.detach())
        (wp * torch.arange(total, dtype=wp.dtype)).sum().backward()
        po = 0
        for p in params:
            assert torch.equal(p.grad.reshape(-1), torch.arange(po, po + p.numel(), dtype=wp.dtype))
            po += p.numel()
    # shapes the fused step does not cover: no pack
    arch = nets.PolicyArch(proprio_dim=9, action_dim=3, recurrent=True, hidden=32, mlp=(64, 64))
    assert nets.PolicyNet(arch, np.random.default_rng(0)).pack_weights() is None
