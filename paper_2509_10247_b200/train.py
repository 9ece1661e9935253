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

import numpy as np
import torch
import torch.distributed as dist

from paper_2509_10247_b200.nets import (LOG_SIGMA_MIN, PolicyArch, PolicyNet, ValueNet, value_fit_grad,  # noqa: F401
                                        value_forward)


@dataclass
class LearnerOptions:
    """q/learners.py:34-58 (actor/critic subset)."""

    algo: str = "sha2c"  # bptt | shac | sha2c (the reference's default, q/learners.py:31)
    horizon: int = 16
    gamma: float = 0.99
    td_lambda: float = 0.95
    k_steps: int | None = None  # critic k-step return window; None -> horizon (q/learners.py:38)
    actor_lr: float = 2e-3
    critic_lr: float = 2e-3
    critic_iters: int = 8
    grad_clip: float = 5.0
    explore: bool = True
    recurrent: bool = True
    hidden: int = 64
    mlp: tuple = (128, 128)
    conv_feat: int = 32
    log_sigma_init: float = -1.2
    log_sigma_max: float = 2.0
    # PPO specifics (q/learners.py:52-59)
    ppo_horizon: int = 32
    clip_eps: float = 0.2
    ppo_epochs: int = 4
    ppo_minibatch: int = 512
    entropy_coef: float = 1e-3
    value_coef: float = 0.5
    reward_norm: bool = True
    seed: int = 0
    # matmul precision of the policy/critic on CUDA: "bf16" runs them on the
    # tensor cores under torch.autocast (fp32 master weights, fp32 sim
    # gradients); "fp32" keeps the reference's all-fp32 arithmetic (SIMT GEMMs)
    net_dtype: str = "bf16"
    # bf16 critic fit through the fused forward+backward kernel (nets.value_fit_grad)
    fused_critic: bool = True
    # replay each whole update (rollout, BPTT backward, actor step, critic fit)
    # from one CUDA graph (ShortHorizonTrainer; single-rank, no-sensor envs).
    # The env's kernel configuration is frozen into the graph at capture; an
    # env.reset() (new buffers) triggers a re-capture, other changes need one
    cuda_graph: bool = False


def td_lambda_targets(r, values, bootstrap, done, gamma, lam, k=None):
    """TD(lambda) targets with termination cuts (q/learners.py:78-113), (T,N).

    ``k`` limits the return window (SHA2C's k-step critic target,
    q/learners.py:95-113): G_t mixes the n-step returns n = 1..min(k, T-t)
    with weights (1-lam) lam^(n-1), the last one taking the remaining
    lam^(steps-1).  The n loop runs over all t at once (k vector steps)."""
    T = r.shape[0]
    if ((k is None or k >= T) and r.is_cuda and r.dim() == 2 and r.dtype == torch.float32 and
            values.dtype == torch.float32 and bootstrap.dtype == torch.float32 and done.dtype == torch.bool and
            not (torch.is_grad_enabled() and (r.requires_grad or values.requires_grad or bootstrap.requires_grad))):
        # one CUDA kernel (qs_td_lambda): a thread per env walks the window
        # backwards with the same rounding as the loop below
        from paper_2509_10247_b200 import _lib as L

        r_, v_, b_ = r.contiguous(), values.contiguous(), bootstrap.contiguous()
        d_ = done.contiguous().view(torch.uint8)
        G = torch.empty_like(r_)
        L.check(L.lib().qs_td_lambda(T, r_.shape[1], L.ptr(r_), L.ptr(v_), L.ptr(b_), L.ptr(d_), float(gamma),
                                     float(lam), 1.0 - float(lam), L.ptr(G), L.stream_handle(r_.device)),
                "qs_td_lambda")
        return G
    cont = 1.0 - done.to(r.dtype)
    if k is None or k >= T:
        G = torch.empty_like(r)
        nxt = bootstrap
        for t in reversed(range(T)):
            v_next = values[t + 1] if t + 1 < T else bootstrap
            G[t] = r[t] + gamma * cont[t] * ((1.0 - lam) * v_next + lam * nxt)
            nxt = G[t]
        return G
    dev = r.device
    v_ext = torch.cat([values, bootstrap[None]], 0)  # V(s_t), t = 0..T
    ts = torch.arange(T, device=dev)
    steps = torch.clamp(T - ts, max=k)  # (T,)
    running = torch.zeros_like(r)
    alive = torch.ones_like(r)
    mix = torch.zeros_like(r)
    disc = 1.0
    for n in range(1, k + 1):
        idx = torch.clamp(ts + n - 1, max=T - 1)  # r/cont index t+n-1 (clamped where n > steps: weight 0)
        r_n, c_n = r[idx], cont[idx]
        running = running + disc * alive * r_n
        g_n = running + gamma * disc * alive * c_n * v_ext[torch.clamp(ts + n, max=T)]
        full_w = torch.full((T,), (1.0 - lam) * lam ** (n - 1), dtype=r.dtype, device=dev)
        last_w = torch.full((T,), lam ** (n - 1), dtype=r.dtype, device=dev)
        w = torch.where(n < steps, full_w, torch.where(n == steps, last_w, torch.zeros_like(last_w)))
        mix = mix + w[:, None] * g_n
        alive = alive * c_n
        disc *= gamma
    return mix


def gae_advantages(r, values, bootstrap, done, gamma, lam):
    """Standard GAE with cuts at done (q/learners.py:116-127): (adv, targets)."""
    T = r.shape[0]
    cont = 1.0 - done.to(r.dtype)
    adv = torch.empty_like(r)
    acc = torch.zeros_like(bootstrap)
    for t in reversed(range(T)):
        v_next = values[t + 1] if t + 1 < T else bootstrap
        delta = r[t] + gamma * cont[t] * v_next - values[t]
        acc = delta + gamma * lam * cont[t] * acc
        adv[t] = acc
    return adv, adv + values


def normalize(adv, eps: float = 1e-8):
    """q/learners.py:130-131 (population std, as numpy's)."""
    return (adv - adv.mean()) / (adv.std(unbiased=False) + eps)


class ReturnScaler:
    """PPO reward scaling by a running estimate of the discounted-return std
    (q/learners.py:345-366): per step, the return trace of every env is merged
    into running moments (parallel Welford), traces reset at done; the window's
    rewards are divided by the std after the window.  The moments live on the
    device; ``group`` merges every rank's batch (the global batch of the
    sharded envs), which with one rank is exactly the reference's update."""

    def __init__(self, n_envs, gamma, device, group=None):
        self.gamma = gamma
        self.trace = torch.zeros(n_envs, dtype=torch.float64, device=device)
        # count, mean, m2 -- the reference's initial state
        self.mom = torch.tensor([1e-4, 0.0, 1.0], dtype=torch.float64, device=device)
        self.group = group

    def __call__(self, rewards, dones):
        T = rewards.shape[0]
        distributed = dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1
        for t in range(T):
            self.trace = rewards[t].double() + self.gamma * self.trace
            b = self.trace
            n_b = torch.tensor(float(b.numel()), dtype=torch.float64, device=b.device)
            s1, s2 = b.sum(), (b * b).sum()
            if distributed:
                st = torch.stack([n_b, s1, s2])
                dist.all_reduce(st, group=self.group)
                n_b, s1, s2 = st[0], st[1], st[2]
            mean_b = s1 / n_b
            var_b = torch.clamp(s2 / n_b - mean_b * mean_b, min=0.0) if distributed else b.var(unbiased=False)
            cnt, mean, m2 = self.mom[0], self.mom[1], self.mom[2]
            delta = mean_b - mean
            tot = cnt + n_b
            self.mom = torch.stack([tot, mean + delta * n_b / tot, m2 + var_b * n_b + delta * delta * cnt * n_b / tot])
            self.trace = torch.where(dones[t], torch.zeros_like(self.trace), self.trace)
        std = torch.sqrt(self.mom[2] / self.mom[0])
        return (rewards.double() / torch.clamp(std, min=1e-8)).to(rewards.dtype)


def ppo_log_prob(mu, log_sigma, a_raw, half):
    """Gaussian log-density of the raw action with the tanh-squash correction
    (q/learners.py:368-385): log|da/draw| = log(half) + 2 (log 2 - x - softplus(-2x))."""
    z = (a_raw - mu) / torch.exp(log_sigma)
    A = mu.shape[-1]
    base = -(0.5 * (z * z).sum(-1) + log_sigma.sum(-1) + 0.5 * np.log(2 * np.pi) * A)
    corr = 2.0 * (np.log(2.0) - a_raw - torch.nn.functional.softplus(-2.0 * a_raw)) + torch.log(half)
    return base - corr.sum(-1)


def clip_grads_(params, clip: float):
    """Global-norm clip with the reference Adam's rule (q/nets.py:293-298):
    scale by clip / (norm + 1e-12) when norm > clip.  Returns the pre-clip
    norm as a device tensor (no host sync)."""
    grads = [p.grad for p in params if p.grad is not None]
    if not grads:
        return torch.zeros(())
    norm = torch.linalg.vector_norm(torch.stack(torch._foreach_norm(grads)).double())
    scale = torch.where(norm > clip, clip / (norm + 1e-12), torch.ones_like(norm))
    torch._foreach_mul_(grads, scale.to(grads[0].dtype))
    return norm


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


def make_nets(env, opts, critic: bool):
    """Policy (and critic) with the reference's architecture, parameter names
    and initial weights for ``opts.seed`` (q/learners.py:141-169)."""
    rng = np.random.default_rng([opts.seed & 0x7FFFFFFF, 0x11])
    spec = env.obs_spec()
    recurrent = opts.recurrent and opts.algo != "ppo"  # recurrent PPO is out of the reference's scope (:335-337)
    policy = PolicyNet(PolicyArch(proprio_dim=spec["proprio_dim"], action_dim=spec["action_dim"],
                                  visual=spec["visual"], recurrent=recurrent, hidden=opts.hidden,
                                  mlp=tuple(opts.mlp), conv_feat=opts.conv_feat,
                                  log_sigma_init=opts.log_sigma_init, log_sigma_max=opts.log_sigma_max,
                                  input_scale=env.proprio_scale()), rng)
    value = ValueNet(env.privileged_dim(), rng, hidden=tuple(opts.mlp),
                     input_scale=env.privileged_scale()) if critic else None
    return policy, value


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
        # the reference's init stream and order (q/learners.py:141-169): the
        # same seed gives the reference's initial weights, on every rank
        self.policy, self.value = make_nets(env, opts, critic=opts.algo in ("shac", "sha2c", "ppo"))
        self.policy.to(dev)
        graph = opts.cuda_graph and dev.type == "cuda"
        # fused Adam: one kernel per step for all parameters (device-side step
        # counter, so it captures into the update's CUDA graph)
        fused = dev.type == "cuda"
        self.actor_opt = torch.optim.Adam(self.policy.parameters(), lr=opts.actor_lr, capturable=graph,
                                          fused=fused)
        self.needs_critic = self.value is not None
        if self.needs_critic:
            self.value.to(dev)
            self.critic_opt = torch.optim.Adam(self.value.parameters(), lr=opts.critic_lr, capturable=graph,
                                               fused=fused)
        self.hidden = self.policy.initial_hidden(env.N, dev)
        self.update_count = 0
        self._gen = torch.Generator(device=dev)
        self._gen.manual_seed(opts.seed * 1_000_003 + env.env_offset)
        self.timing = {"sim_fwd_bwd_s": 0.0, "allreduce_s": 0.0}
        if opts.net_dtype not in ("bf16", "fp32"):
            raise ValueError("net_dtype must be 'bf16' or 'fp32'")
        self._amp = opts.net_dtype == "bf16" and dev.type == "cuda"
        self._graph = None
        self._graph_mode = graph
        self._warm = 0
        self._capturing = False
        self._ar_events = []

    def _distributed(self) -> bool:
        return dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1

    def allreduce_ms(self) -> float:
        """Device time (CUDA events, ms) of the policy-gradient all-reduces of
        the eager updates since the last call (syncs).  Captured updates run
        the collective inside the graph; bench.py times it standalone."""
        if not self._ar_events:
            return 0.0
        self._ar_events[-1][1].synchronize()
        ms = sum(a.elapsed_time(b) for a, b in self._ar_events)
        self._ar_events = []
        return ms

    def _nets(self):
        """autocast scope for policy/critic evaluations (no-op for fp32 / CPU);
        the cast cache is off under graph capture (torch's requirement)."""
        return torch.autocast("cuda", dtype=torch.bfloat16, enabled=self._amp, cache_enabled=not self._graph_mode)

    def collect_window(self, record_privileged: bool):
        """q/learners.py:201-230."""
        env, opts = self.env, self.opts
        T = opts.horizon
        env.detach_states()
        obs = env.observe()
        h = self.hidden.detach() if self.hidden is not None else None
        disc = 0.0
        r_ctrl, r_goal, dones, priv = [], [], [], []
        reset = None  # rows whose episode ended last step: their hidden state restarts at 0
        # the fused policy step's parameters packed once for the window (bf16 mode)
        packed = self.policy.pack_weights() if self._amp else None
        for t in range(T):
            if record_privileged:
                priv.append(env.privileged_state())
            with self._nets():
                mu, log_sigma, h = self.policy(obs.proprio, obs.visual, h, h_reset=reset, packed=packed)
            a = mu
            if opts.explore:
                eps = torch.randn(mu.shape, generator=self._gen, device=mu.device)
                a = mu + torch.exp(log_sigma) * eps
            out = env.step(a)
            reset = out.done if h is not None else None
            disc = disc + out.r_ctrl.mean() * (opts.gamma ** t)
            r_ctrl.append(out.r_ctrl.detach())
            r_goal.append(out.r_goal)
            dones.append(out.done)
            obs = out.obs
        if h is not None:
            self.hidden = torch.where(reset[:, None], torch.zeros_like(h), h).detach()
        return disc, torch.stack(r_ctrl), torch.stack(r_goal), torch.stack(dones), (
            torch.stack(priv) if record_privileged else None)

    def _update_tensors(self):
        """One update with every result left on the device (no host sync):
        (actor loss, pre-clip grad norm, critic loss or None)."""
        opts = self.opts
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
        self.actor_opt.zero_grad(set_to_none=not self._graph_mode)
        loss.backward()
        timed = self._distributed() and not self._capturing
        if timed:  # device time of the collective: events on the stream that waits for it
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        allreduce_mean_(list(self.policy.parameters()), self.group)
        if timed:
            e1.record()
            self._ar_events.append((e0, e1))
        gnorm = clip_grads_(list(self.policy.parameters()), opts.grad_clip)
        self.actor_opt.step()
        closs = None
        if self.needs_critic:
            closs = self._critic_update(r_ctrl if opts.algo == "shac" else r_goal, dones, priv)
        return loss.detach(), gnorm, closs

    def update(self) -> dict:
        opts = self.opts
        t0 = time.perf_counter()
        if self._graph is not None and any(a is not b for a, b in zip(self._env_bufs, self._env_buffers())):
            self._graph = None  # env.reset() re-allocated the buffers the graph points at
        if self._graph_mode and self._graph is None and self._warm >= 3:
            self._capture()  # records only: this call's update is the first replay
        if self._graph is not None:
            self._sync_carry()
            self._graph.replay()
            loss, gnorm, closs = self._graph_out
        elif self._graph_mode:  # the eager warm-up updates torch asks for, on a side stream
            side = torch.cuda.Stream(self.env.device)
            side.wait_stream(torch.cuda.current_stream(self.env.device))
            with torch.cuda.stream(side):
                loss, gnorm, closs = self._update_tensors()
            torch.cuda.current_stream(self.env.device).wait_stream(side)
            self._warm += 1
        else:
            loss, gnorm, closs = self._update_tensors()
        out = {"loss": float(loss), "grad_norm": float(gnorm)}  # the update's one host sync
        if not np.isfinite(out["loss"]):
            raise FloatingPointError("non-finite actor loss; check reward terms")
        if closs is not None:
            out["critic_loss"] = float(closs)
        self.update_count += 1
        self.timing["sim_fwd_bwd_s"] += time.perf_counter() - t0
        out["steps_per_sec"] = opts.horizon * self.env.N / (time.perf_counter() - t0)
        return out

    def _env_buffers(self):
        """The env objects a captured update holds pointers to (reset() replaces them)."""
        e = self.env
        return (e._meta, e._ep_ret, e._stats, e._err, e._imu_bias, e._scene, e._cfg)

    def _sync_carry(self):
        """The env was reset or stepped outside the graph since the last replay
        (e.g. by evaluate()): load its current state into the graph's carry
        buffers and rebind."""
        env, c = self.env, self._carry
        if env._S is c["S"] and (c["hidden"] is None or self.hidden is c["hidden"]):
            return
        c["S"].copy_(env._S.detach())
        c["goal"].copy_(env._goal)
        c["peff"].copy_(env._peff)
        if c["dr"] is not None:
            c["dr"].copy_(env._dr)
        if c["hidden"] is not None and self.hidden is not c["hidden"]:
            c["hidden"].copy_(self.hidden)
        env._S, env._goal, env._peff = c["S"], c["goal"], c["peff"]
        if c["dr"] is not None:
            env._dr = c["dr"]
        if c["hidden"] is not None:
            self.hidden = c["hidden"]

    def _capture(self):
        """Record one whole update into a CUDA graph (torch's whole-network
        capture: forward, autograd backward and capturable Adam).  The env's
        functional state (S, goal, effort, randomisation) and the GRU hidden
        state are carried through static buffers that the graph reads at its
        start and rewrites at its end; counters, statistics and the error word
        already live in device buffers updated in place.  update() runs three
        eager updates on a side stream before capturing (lazy optimiser /
        autograd state); capturing executes nothing."""
        env = self.env
        if self._distributed() and dist.get_backend(self.group) != "nccl":
            raise RuntimeError("cuda_graph with several ranks needs the NCCL backend (the all-reduce is "
                               "captured into the graph; gloo collectives run on the host)")
        if env.strict or env.config.sensor != "none" or env.reset_source is not None or env._regen:
            raise RuntimeError("cuda_graph needs strict=False, no sensor, in-kernel resets and no scene regen")
        carry = {"S": env._S.detach().clone(), "goal": env._goal.clone(), "peff": env._peff.clone(),
                 "dr": env._dr.clone() if env._dr is not None else None,
                 "hidden": self.hidden.clone() if self.hidden is not None else None}

        def bind():
            env._S, env._goal, env._peff = carry["S"], carry["goal"], carry["peff"]
            if carry["dr"] is not None:
                env._dr = carry["dr"]
            if carry["hidden"] is not None:
                self.hidden = carry["hidden"]

        def carry_back():
            carry["S"].copy_(env._S.detach())
            carry["goal"].copy_(env._goal)
            carry["peff"].copy_(env._peff)
            if carry["dr"] is not None:
                carry["dr"].copy_(env._dr)
            if carry["hidden"] is not None:
                carry["hidden"].copy_(self.hidden)

        g = torch.cuda.CUDAGraph()
        g.register_generator_state(self._gen)
        bind()
        self._capturing = True
        try:
            with torch.cuda.graph(g):
                out = self._update_tensors()
                carry_back()
        finally:
            self._capturing = False
        bind()
        self._graph, self._graph_out = g, out
        self._carry = carry
        self._env_bufs = self._env_buffers()

    def _critic_update(self, r, dones, priv):
        """TD-lambda targets + full-batch MSE fit (q/learners.py:232-245, 286-292)."""
        opts = self.opts
        with torch.no_grad():
            T, N, K = priv.shape
            if self._amp and K <= 14 and tuple(opts.mlp) == (128, 128) and opts.fused_critic:
                # the critic's values for the targets on the tcgen05 path (one kernel each)
                values = value_forward(self.value, priv.reshape(T * N, K)).reshape(T, N)
                boot = value_forward(self.value, self.env.privileged_state())
            else:
                with self._nets():
                    values = self.value(priv.reshape(T * N, K)).reshape(T, N)
                    boot = self.value(self.env.privileged_state())
            targets = td_lambda_targets(r, values, boot, dones, opts.gamma, opts.td_lambda, opts.k_steps)
        X = priv.reshape(-1, priv.shape[-1])
        y = targets.reshape(-1)
        fused = opts.fused_critic and self._amp and X.shape[1] <= 16 and tuple(opts.mlp) == (128, 128)
        for _ in range(opts.critic_iters):
            self.critic_opt.zero_grad(set_to_none=not self._graph_mode)
            if fused:  # one kernel: forward + backward of the whole batch, grads into .grad
                loss = value_fit_grad(self.value, X, y)
            else:
                with self._nets():
                    pred = self.value(X)
                loss = ((pred - y) ** 2).mean()
                loss.backward()
            allreduce_mean_(list(self.value.parameters()), self.group)
            clip_grads_(list(self.value.parameters()), opts.grad_clip)
            self.critic_opt.step()
        return loss.detach()  # the last iteration's loss (device scalar)


class PPOTrainer:
    """Clipped surrogate + GAE on the RL reward scalar (q/learners.py:327-487).

    Rollouts run the forward-only env step (no autograd graph: one fused
    kernel per step); the policy is the reference's non-recurrent MLP (with its
    conv / LiDAR encoder when the task has a visual observation).  Rewards are
    scaled by the running discounted-return std; advantages are GAE with cuts
    at done, normalised over the window.  Each epoch visits the window's rows
    in a fresh permutation, in minibatches; the actor and critic each take one
    Adam step per minibatch (global-norm clip ``grad_clip``), their gradients
    averaged across ranks first (NCCL; gloo in the CPU tests).  Deviation: the
    exploration noise and the permutations come from torch's Philox
    generators, not numpy's (values are not pinned by the reference's tests,
    only their statistics and determinism)."""

    def __init__(self, env, opts: LearnerOptions, group=None):
        self.env, self.opts, self.group = env, opts, group
        dev = env.device
        self.policy, self.value = make_nets(env, opts, critic=True)
        self.policy.to(dev)
        self.value.to(dev)
        self.actor_opt = torch.optim.Adam(self.policy.parameters(), lr=opts.actor_lr)
        self.critic_opt = torch.optim.Adam(self.value.parameters(), lr=opts.critic_lr)
        self.scaler = ReturnScaler(env.N, opts.gamma, dev, group)
        self.update_count = 0
        self._gen = torch.Generator(device=dev)
        self._gen.manual_seed(opts.seed * 1_000_003 + env.env_offset + 0xB)
        self._amp = opts.net_dtype == "bf16" and dev.type == "cuda"

    def _nets(self):
        return torch.autocast("cuda", dtype=torch.bfloat16, enabled=self._amp)

    def _half(self):
        env = self.env
        half = (torch.as_tensor(env.action_hi, dtype=torch.float32, device=env.device) -
                torch.as_tensor(env.action_lo, dtype=torch.float32, device=env.device)) / 2.0
        return half.expand(env.N, env.action_dim) if half.dim() == 1 else half

    def collect(self):
        env, opts = self.env, self.opts
        T = opts.ppo_horizon
        half = self._half()
        env.detach_states()
        obs = env.observe()
        pro, vis, acts, logps, vals, rews, dones, priv = [], [], [], [], [], [], [], []
        with torch.no_grad():
            for t in range(T):
                p = env.privileged_state()
                with self._nets():
                    mu, log_sigma, _ = self.policy(obs.proprio, obs.visual, None)
                    v = self.value(p)
                eps = torch.randn(mu.shape, generator=self._gen, device=mu.device)
                a = mu + torch.exp(log_sigma) * eps
                logps.append(ppo_log_prob(mu, log_sigma, a, half))
                pro.append(obs.proprio.detach())
                if obs.visual is not None:
                    vis.append(obs.visual)
                priv.append(p)
                vals.append(v.float())
                out = env.step(a)
                acts.append(a)
                rews.append(out.r_rl.float())
                dones.append(out.done)
                obs = out.obs
            with self._nets():
                boot = self.value(env.privileged_state()).float()
        st = lambda xs: torch.stack(xs) if xs else None  # noqa: E731
        return st(pro), st(vis), st(acts), st(logps), st(vals), st(rews), st(dones), st(priv), boot, half

    def update(self) -> dict:
        env, opts = self.env, self.opts
        t0 = time.perf_counter()
        pro, vis, acts, logps, vals, rews, dones, priv, boot, half = self.collect()
        T, N = rews.shape
        scaled = self.scaler(rews, dones) if opts.reward_norm else rews
        adv, rets = gae_advantages(scaled, vals, boot, dones, opts.gamma, opts.td_lambda)
        adv_n = normalize(adv)
        n_rows = T * N
        flat = lambda x: x.reshape(n_rows, *x.shape[2:]) if x is not None else None  # noqa: E731
        pro_f, vis_f, a_f, old_f, adv_f, ret_f, priv_f = (flat(pro), flat(vis), flat(acts), logps.reshape(-1),
                                                           adv_n.reshape(-1), rets.reshape(-1), flat(priv))
        half_f = half.repeat(T, 1)
        mb = min(opts.ppo_minibatch, n_rows)
        pi_loss = v_loss = ent = torch.zeros((), device=env.device)
        pgen = torch.Generator(device=env.device)
        for epoch in range(opts.ppo_epochs):
            pgen.manual_seed(((opts.seed & 0xFFFFFFFF) << 20) ^ (self.update_count << 8) ^ epoch)
            order = torch.randperm(n_rows, generator=pgen, device=env.device)
            for s0 in range(0, n_rows, mb):
                rows = order[s0:s0 + mb]
                with self._nets():
                    mu, log_sigma, _ = self.policy(pro_f[rows], vis_f[rows] if vis_f is not None else None, None)
                logp = ppo_log_prob(mu, log_sigma, a_f[rows], half_f[rows])
                ratio = torch.exp(logp - old_f[rows])
                r_clip = torch.clamp(ratio, 1.0 - opts.clip_eps, 1.0 + opts.clip_eps)
                adv_rows = adv_f[rows]
                surr = torch.minimum(ratio * adv_rows, r_clip * adv_rows).mean()
                entropy = (log_sigma.sum(-1) + 0.5 * mu.shape[-1] * np.log(2 * np.pi * np.e)).mean()
                actor_loss = -(surr + opts.entropy_coef * entropy)
                self.actor_opt.zero_grad(set_to_none=True)
                actor_loss.backward()
                allreduce_mean_(list(self.policy.parameters()), self.group)
                clip_grads_(list(self.policy.parameters()), opts.grad_clip)
                self.actor_opt.step()
                with self._nets():
                    pred = self.value(priv_f[rows]).float()
                value_loss = ((pred - ret_f[rows]) ** 2).mean()
                self.critic_opt.zero_grad(set_to_none=True)
                (value_loss * opts.value_coef).backward()
                allreduce_mean_(list(self.value.parameters()), self.group)
                clip_grads_(list(self.value.parameters()), opts.grad_clip)
                self.critic_opt.step()
                pi_loss, v_loss, ent = actor_loss.detach(), value_loss.detach(), entropy.detach()
        self.update_count += 1
        return {"loss": float(pi_loss), "critic_loss": float(v_loss), "entropy": float(ent),
                "reward_mean": float(rews.mean()), "steps_per_sec": T * N / (time.perf_counter() - t0)}


def make_learner(env, opts: LearnerOptions, group=None):
    """q/learners.py:66-71."""
    if opts.algo in ("bptt", "shac", "sha2c"):
        return ShortHorizonTrainer(env, opts, group)
    if opts.algo == "ppo":
        return PPOTrainer(env, opts, group)
    raise ValueError(f"unknown algorithm '{opts.algo}'; choose from ('bptt', 'shac', 'sha2c', 'ppo')")


# ---------------------------------------------------------------------------
# the reference's learner names (q/learners.py:63-71, 248-324, 494-527)

ALGOS = ("bptt", "shac", "sha2c", "ppo")


def _preset(algo):
    class _Learner(ShortHorizonTrainer):
        def __init__(self, env, opts: LearnerOptions = LearnerOptions(), group=None):
            from dataclasses import replace

            super().__init__(env, replace(opts, algo=algo), group)

    _Learner.__name__ = _Learner.__qualname__ = algo.upper()
    return _Learner


BPTT, SHAC, SHA2C = _preset("bptt"), _preset("shac"), _preset("sha2c")
PPO = PPOTrainer


def wilson_interval(successes: int, n: int, z: float = 1.96):
    """q/learners.py:494-501."""
    if n == 0:
        return (0.0, 1.0)
    p = successes / n
    denom = 1 + z * z / n
    center = (p + z * z / (2 * n)) / denom
    spread = z * np.sqrt(p * (1 - p) / n + z * z / (4 * n * n)) / denom
    return (max(0.0, center - spread), min(1.0, center + spread))


@torch.no_grad()
def evaluate(env, policy, n_episodes: int, seed: int, max_steps: int | None = None) -> dict:
    """Greedy (mean-action) rollouts until n_episodes finish (q/learners.py:504-527)."""
    out = env.reset(seed)
    env.reset_stats()
    hidden = policy.initial_hidden(env.N, env.device)
    obs = out.obs
    cap = max_steps or (env.config.episode_len * (n_episodes // env.n_envs + 2) * 2)
    steps = 0
    while env.finished_episodes < n_episodes and steps < cap:
        mu, _s, h2 = policy(obs.proprio, obs.visual, hidden)
        res = env.step(mu)
        if hidden is not None:
            hidden = torch.where(res.done[:, None], torch.zeros_like(h2), h2.float())
        obs = res.obs
        steps += 1
    lo, hi = wilson_interval(env.successful_episodes, env.finished_episodes)
    return {"episodes": env.finished_episodes, "success_rate": env.success_rate,
            "collision_rate": env.collision_rate, "mean_episode_reward": env.mean_episode_return,
            "success_ci95": (lo, hi), "steps": steps}
