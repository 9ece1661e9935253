"""Short-horizon differentiable policy training on the B200 env (config C5).

This is the caller side of the hot path: BPTT / SHAC / SHA2C windows
(q/learners.py:201-324) driving ``FlightTask.step`` through torch autograd.
Each env step is one fused forward kernel; its backward is the analytic VJP
kernel.  The policy and critic are plain torch modules, so their matmuls run
on tensor cores through cuBLAS; they are library code, not the hot path.

Multi-GPU: one process per GPU.  Envs shard by ``env_offset``, so every rank
simulates distinct global envs and the sim step never communicates.  After
each backward, the flattened policy gradient (and each critic iteration's
gradient) is averaged with ONE NCCL all-reduce (``torch.distributed``,
backend "nccl").  The same code runs with "gloo" on CPU tensors in the tests.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import torch
import torch.distributed as dist

LOG_SIGMA_MIN = -5.0  # q/nets.py:22


@dataclass
class LearnerOptions:
    """q/learners.py:34-58 (actor/critic subset)."""

    algo: str = "shac"  # bptt | shac | sha2c
    horizon: int = 16
    gamma: float = 0.99
    td_lambda: float = 0.95
    actor_lr: float = 2e-3
    critic_lr: float = 2e-3
    critic_iters: int = 8
    grad_clip: float = 5.0
    explore: bool = True
    recurrent: bool = True
    hidden: int = 64
    mlp: tuple = (128, 128)
    log_sigma_init: float = -1.2
    log_sigma_max: float = 2.0
    seed: int = 0
    # matmul precision of the policy/critic on CUDA: "bf16" runs them on the
    # tensor cores under torch.autocast (fp32 master weights, fp32 sim
    # gradients); "fp32" keeps the reference's all-fp32 arithmetic (SIMT GEMMs)
    net_dtype: str = "bf16"


class PolicyNet(torch.nn.Module):
    """GRU-64 + tanh MLP trunk + (mu, log_sigma) heads (q/nets.py:183-256)."""

    def __init__(self, proprio_dim, action_dim, input_scale=None, recurrent=True, hidden=64, mlp=(128, 128),
                 log_sigma_init=-1.2, log_sigma_max=2.0):
        super().__init__()
        scale = torch.ones(proprio_dim) if input_scale is None else torch.as_tensor(input_scale, dtype=torch.float32)
        self.register_buffer("input_scale", scale)
        self.gru = torch.nn.GRUCell(proprio_dim, hidden) if recurrent else None
        sizes = [hidden if recurrent else proprio_dim] + list(mlp)
        self.trunk = torch.nn.ModuleList(torch.nn.Linear(a, b) for a, b in zip(sizes[:-1], sizes[1:]))
        self.mu = torch.nn.Linear(mlp[-1], action_dim)
        self.sig = torch.nn.Linear(mlp[-1], action_dim)
        for head in (self.mu, self.sig):
            torch.nn.init.normal_(head.weight, std=0.01 * (2.0 / (mlp[-1] + action_dim)) ** 0.5)
            torch.nn.init.zeros_(head.bias)
        torch.nn.init.constant_(self.sig.bias, log_sigma_init)
        self.hidden = hidden
        self.log_sigma_max = log_sigma_max

    def initial_hidden(self, batch, device):
        return torch.zeros(batch, self.hidden, device=device) if self.gru is not None else None

    def forward(self, proprio, h=None):
        x = proprio * self.input_scale
        if self.gru is not None:
            h = self.gru(x, h).float()
            x = h
        for layer in self.trunk:
            x = torch.tanh(layer(x))
        mu, ls = self.mu(x).float(), self.sig(x).float()
        return mu, torch.clamp(ls, LOG_SIGMA_MIN, self.log_sigma_max), h


class ValueNet(torch.nn.Module):
    """Privileged-state MLP critic (q/nets.py:259-274)."""

    def __init__(self, n_in, hidden=(128, 128), input_scale=None):
        super().__init__()
        scale = torch.ones(n_in) if input_scale is None else torch.as_tensor(input_scale, dtype=torch.float32)
        self.register_buffer("input_scale", scale)
        sizes = [n_in] + list(hidden) + [1]
        self.layers = torch.nn.ModuleList(torch.nn.Linear(a, b) for a, b in zip(sizes[:-1], sizes[1:]))

    def forward(self, x):
        x = x * self.input_scale
        for i, layer in enumerate(self.layers):
            x = layer(x)
            if i < len(self.layers) - 1:
                x = torch.tanh(x)
        return x[..., 0].float()


def td_lambda_targets(r, values, bootstrap, done, gamma, lam):
    """TD(lambda) targets with termination cuts (q/learners.py:78-94), (T,N)."""
    T = r.shape[0]
    cont = 1.0 - done.to(r.dtype)
    G = torch.empty_like(r)
    nxt = bootstrap
    for t in reversed(range(T)):
        v_next = values[t + 1] if t + 1 < T else bootstrap
        G[t] = r[t] + gamma * cont[t] * ((1.0 - lam) * v_next + lam * nxt)
        nxt = G[t]
    return G


def allreduce_mean_(params, group=None):
    """Average .grad of ``params`` over ranks with one flattened all-reduce."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return
    grads = [p.grad for p in params if p.grad is not None]
    if not grads:
        return
    flat = torch.cat([g.reshape(-1) for g in grads])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    flat /= dist.get_world_size(group)
    off = 0
    for g in grads:
        n = g.numel()
        g.copy_(flat[off:off + n].view_as(g))
        off += n


def shard_envs(n_total: int, rank: int, world: int):
    """Contiguous global env range of ``rank`` (sharding is by global env id)."""
    per = (n_total + world - 1) // world
    lo = min(n_total, rank * per)
    return lo, min(n_total, lo + per)


class ShortHorizonTrainer:
    """BPTT (q/learners.py:251-265), SHAC (:274-303) and SHA2C (:315-324)."""

    def __init__(self, env, opts: LearnerOptions = LearnerOptions(), group=None):
        self.env, self.opts, self.group = env, opts, group
        dev = env.device
        g = torch.Generator(device="cpu").manual_seed(opts.seed)
        torch.manual_seed(opts.seed)  # identical initial weights on every rank
        self.policy = PolicyNet(env.proprio_dim, env.action_dim, env.proprio_scale(), opts.recurrent, opts.hidden,
                                opts.mlp, opts.log_sigma_init, opts.log_sigma_max).to(dev)
        self.actor_opt = torch.optim.Adam(self.policy.parameters(), lr=opts.actor_lr)
        self.needs_critic = opts.algo in ("shac", "sha2c")
        if self.needs_critic:
            self.value = ValueNet(env.privileged_dim(), opts.mlp, env.privileged_scale()).to(dev)
            self.critic_opt = torch.optim.Adam(self.value.parameters(), lr=opts.critic_lr)
        self.hidden = self.policy.initial_hidden(env.N, dev)
        self.update_count = 0
        self._gen = torch.Generator(device=dev)
        self._gen.manual_seed(opts.seed * 1_000_003 + env.env_offset)
        self.timing = {"sim_fwd_bwd_s": 0.0, "allreduce_s": 0.0}
        if opts.net_dtype not in ("bf16", "fp32"):
            raise ValueError("net_dtype must be 'bf16' or 'fp32'")
        self._amp = opts.net_dtype == "bf16" and dev.type == "cuda"

    def _nets(self):
        """autocast scope for policy/critic evaluations (no-op for fp32 / CPU)."""
        return torch.autocast("cuda", dtype=torch.bfloat16, enabled=self._amp)

    def collect_window(self, record_privileged: bool):
        """q/learners.py:201-230."""
        env, opts = self.env, self.opts
        T = opts.horizon
        env.detach_states()
        obs = env.observe()
        h = self.hidden.detach() if self.hidden is not None else None
        disc = 0.0
        r_ctrl, r_goal, dones, priv = [], [], [], []
        for t in range(T):
            if record_privileged:
                priv.append(env.privileged_state())
            with self._nets():
                mu, log_sigma, h = self.policy(obs.proprio, h)
            a = mu
            if opts.explore:
                eps = torch.randn(mu.shape, generator=self._gen, device=mu.device)
                a = mu + torch.exp(log_sigma) * eps
            out = env.step(a)
            if h is not None:
                h = torch.where(out.done[:, None], torch.zeros_like(h), h)
            disc = disc + out.r_ctrl.mean() * (opts.gamma ** t)
            r_ctrl.append(out.r_ctrl.detach())
            r_goal.append(out.r_goal)
            dones.append(out.done)
            obs = out.obs
        if h is not None:
            self.hidden = h.detach()
        return disc, torch.stack(r_ctrl), torch.stack(r_goal), torch.stack(dones), (
            torch.stack(priv) if record_privileged else None)

    def update(self) -> dict:
        opts = self.opts
        t0 = time.perf_counter()
        disc, r_ctrl, r_goal, dones, priv = self.collect_window(self.needs_critic)
        body = disc
        if self.needs_critic:
            for p in self.value.parameters():
                p.requires_grad_(False)
            with self._nets():
                v_term = self.value(self.env.privileged_var())  # grad flows through the state
            for p in self.value.parameters():
                p.requires_grad_(True)
            body = body + v_term.mean() * (opts.gamma ** opts.horizon)
        loss = -body / opts.horizon
        if not bool(torch.isfinite(loss)):
            raise FloatingPointError("non-finite actor loss; check reward terms")
        self.actor_opt.zero_grad(set_to_none=True)
        loss.backward()
        torch.cuda.synchronize(self.env.device) if self.env.device.type == "cuda" else None
        t1 = time.perf_counter()
        allreduce_mean_(list(self.policy.parameters()), self.group)
        t2 = time.perf_counter()
        gnorm = torch.nn.utils.clip_grad_norm_(self.policy.parameters(), opts.grad_clip)
        self.actor_opt.step()
        out = {"loss": float(loss.detach()), "grad_norm": float(gnorm)}
        if self.needs_critic:
            out["critic_loss"] = self._critic_update(r_ctrl if opts.algo == "shac" else r_goal, dones, priv)
        self.update_count += 1
        self.timing["sim_fwd_bwd_s"] += t1 - t0
        self.timing["allreduce_s"] += t2 - t1
        out["steps_per_sec"] = opts.horizon * self.env.N / (time.perf_counter() - t0)
        return out

    def _critic_update(self, r, dones, priv):
        """TD-lambda targets + full-batch MSE fit (q/learners.py:232-245, 286-292)."""
        opts = self.opts
        with torch.no_grad():
            T, N, K = priv.shape
            with self._nets():
                values = self.value(priv.reshape(T * N, K)).reshape(T, N)
                boot = self.value(self.env.privileged_state())
            targets = td_lambda_targets(r, values, boot, dones, opts.gamma, opts.td_lambda)
        X = priv.reshape(-1, priv.shape[-1])
        y = targets.reshape(-1)
        loss_val = 0.0
        for _ in range(opts.critic_iters):
            self.critic_opt.zero_grad(set_to_none=True)
            with self._nets():
                pred = self.value(X)
            loss = ((pred - y) ** 2).mean()
            loss.backward()
            allreduce_mean_(list(self.value.parameters()), self.group)
            torch.nn.utils.clip_grad_norm_(self.value.parameters(), opts.grad_clip)
            self.critic_opt.step()
            loss_val = float(loss.detach())
        return loss_val
