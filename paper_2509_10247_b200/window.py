"""Native BPTT window engine: T fused env steps forward, T analytic VJP steps
backward, no autograd bookkeeping, optionally replayed from one CUDA graph.

This is ``collect_window`` + ``Tape.backward`` of the reference BPTT learner
(q/learners.py:201-230, 251-265) for an open-loop action sequence: the loss is
L = -(1/T) sum_t gamma^t mean(r_ctrl_t) and the engine returns dL/d(raw
actions).  It drives exactly the same kernels as ``FlightTask.step`` and its
autograd node (``qs_task_step_fwd`` / ``qs_task_step_bwd``), with every
per-step checkpoint preallocated so a whole window is graph-capturable.
"""

from __future__ import annotations

import torch

from paper_2509_10247_b200 import _lib as L
from paper_2509_10247_b200.tasks import FlightTask


class BpttWindow:
    def __init__(self, env: FlightTask, horizon: int, gamma: float = 0.99, want_obs: bool = True,
                 fused: bool = True, imu_noise: torch.Tensor | None = None):
        """``imu_noise``: optional (T, 4, N, 3) normals injected into the IMU
        (bias walk accel, bias walk gyro, white accel, white gyro -- the
        reference's draw order, q/sensors.py:544-554) instead of the in-kernel
        Philox draws; for exact parity checks."""
        if env.reset_source is not None:
            raise ValueError("BpttWindow needs in-kernel (Philox) resets; reset_source forces host syncs")
        if env._cfg.reset_mode != 0:
            raise ValueError("BpttWindow resets inline; regen_scene_on_reset needs the per-step env.step path")
        self.env, self.T, self.gamma = env, horizon, gamma
        dev, N, T = env.device, env.N, horizon
        f = dict(device=dev, dtype=torch.float32)
        NP = env._S.shape[0]
        A, P = env.action_dim, env.proprio_dim
        self.S = torch.zeros(T + 1, NP, N, 4, **f)
        self.goal = torch.zeros(T + 1, N, 4, **f)
        self.peff = torch.zeros(T + 1, N, 4, **f)
        self.dr = torch.zeros(T + 1, N, 4, **f) if env._dr is not None else None
        self.flags = torch.zeros(T, N, dtype=torch.int32, device=dev)
        self.obs = torch.zeros(T, N, P, **f) if want_obs else torch.zeros(1, N, P, **f)
        self.r = torch.zeros(T, 3, N, **f)  # r_ctrl, r_goal, r_rl
        self.term = torch.zeros(T, N, dtype=torch.int8, device=dev)
        self.trunc = torch.zeros(T, N, dtype=torch.bool, device=dev)
        self.imu = torch.zeros(T, N, 6, **f) if env._imu_bias is not None else None
        self.actions = torch.zeros(T, N, A, **f)
        self.imu_noise = None
        if imu_noise is not None:
            if self.imu is None:
                raise ValueError("imu_noise needs an env built with TaskConfig.imu")
            self.imu_noise = torch.as_tensor(imu_noise, dtype=torch.float32, device=dev).reshape(T, 4, N, 3)
            self.imu_noise = self.imu_noise.contiguous()
        self.g_actions = torch.zeros(T, N, A, **f)
        self.gS = torch.zeros(2, NP, N, 4, **f)
        # dL/dr_ctrl_t = -gamma^t / (T N)
        w = torch.tensor([-(gamma ** t) / (T * N) for t in range(T)], **f)
        self.g_r = w[:, None].expand(T, N).contiguous()
        self.w_loss = w[:, None] * 1.0
        self.loss = torch.zeros((), **f)
        self.loss64 = torch.zeros((), dtype=torch.float64, device=dev)
        self.want_obs = want_obs
        self.fused = fused
        self.graph = None
        self.launches_per_window = 2 if fused else 2 * T
        self._load_env_state()
        self._bound = self._env_buffers()

    def _load_env_state(self):
        e = self.env
        self.S[0].copy_(e._S.detach())
        self.goal[0].copy_(e._goal)
        self.peff[0].copy_(e._peff)
        if self.dr is not None:
            self.dr[0].copy_(e._dr)

    def _store_env_state(self):
        e = self.env
        e._S = self.S[self.T].clone()
        e._goal = self.goal[self.T].clone()
        e._peff = self.peff[self.T].clone()
        if self.dr is not None:
            e._dr = self.dr[self.T].clone()

    def _window_io(self) -> L.QsWindowIo:
        e = self.env
        w = L.QsWindowIo()
        w.T = self.T
        w.S, w.goal, w.peff = L.ptr(self.S), L.ptr(self.goal), L.ptr(self.peff)
        w.dr = L.ptr(self.dr)
        w.actions = L.ptr(self.actions)
        w.meta, w.ep_return, w.imu_bias = L.ptr(e._meta), L.ptr(e._ep_ret), L.ptr(e._imu_bias)
        w.imu_out = L.ptr(self.imu)
        w.imu_noise = L.ptr(self.imu_noise)
        w.obs = L.ptr(self.obs) if self.want_obs else None
        w.r, w.terminated, w.truncated, w.flags = L.ptr(self.r), L.ptr(self.term), L.ptr(self.trunc), L.ptr(self.flags)
        w.stats, w.err = L.ptr(e._stats), L.ptr(e._err)
        w.g_rctrl = None
        w.g_rctrl_scale = -1.0 / (self.T * e.N)
        w.gamma = self.gamma
        w.g_actions = L.ptr(self.g_actions)
        w.loss = L.ptr(self.loss64)  # accumulated by the forward kernel
        w.carry = 1  # the backward moves slot T into slot 0 for the next window
        return w

    def _run(self):
        e = self.env
        lib = L.lib()
        cfg, sc = e._cfg, e._scene.struct()
        stream = L.stream_handle(e.device)
        T = self.T
        if self.fused:
            w = self._window_io()
            L.check(lib.qs_task_window_fwd(cfg, sc, w, stream), "qs_task_window_fwd")
            L.check(lib.qs_task_window_bwd(cfg, sc, w, stream), "qs_task_window_bwd")
            return
        for t in range(T):
            io = e._new_io()
            io.S_in, io.S_out, io.raw = L.ptr(self.S[t]), L.ptr(self.S[t + 1]), L.ptr(self.actions[t])
            io.goal_in, io.goal_out = L.ptr(self.goal[t]), L.ptr(self.goal[t + 1])
            io.peff_in, io.peff_out = L.ptr(self.peff[t]), L.ptr(self.peff[t + 1])
            if self.dr is not None:
                io.dr_in, io.dr_out = L.ptr(self.dr[t]), L.ptr(self.dr[t + 1])
            if self.imu is not None:
                io.imu_out = L.ptr(self.imu[t])
                io.imu_noise = L.ptr(self.imu_noise[t]) if self.imu_noise is not None else None
            io.obs = L.ptr(self.obs[t if self.want_obs else 0])
            io.r_ctrl, io.r_goal, io.r_rl = L.ptr(self.r[t, 0]), L.ptr(self.r[t, 1]), L.ptr(self.r[t, 2])
            io.terminated, io.truncated, io.flags = L.ptr(self.term[t]), L.ptr(self.trunc[t]), L.ptr(self.flags[t])
            lib.qs_task_step_fwd(cfg, sc, io, stream)
        for t in reversed(range(T)):
            g = L.QsStepGrad()
            g.S_in, g.raw, g.goal_in, g.peff_in = L.ptr(self.S[t]), L.ptr(self.actions[t]), L.ptr(self.goal[t]), L.ptr(self.peff[t])
            g.dr_in = L.ptr(self.dr[t]) if self.dr is not None else None
            g.flags = L.ptr(self.flags[t])
            g.g_S_out = L.ptr(self.gS[(t + 1) % 2]) if t < T - 1 else None
            g.g_rctrl = L.ptr(self.g_r[t])
            g.g_S_in, g.g_raw = L.ptr(self.gS[t % 2]), L.ptr(self.g_actions[t])
            lib.qs_task_step_bwd(cfg, sc, g, stream)
        self._finish()

    def _finish(self):
        T = self.T
        torch.sum(self.r[:, 0] * self.w_loss, dim=(0, 1), out=self.loss)
        # carry the final state into slot 0 for the next window
        self.S[0].copy_(self.S[T])
        self.goal[0].copy_(self.goal[T])
        self.peff[0].copy_(self.peff[T])
        if self.dr is not None:
            self.dr[0].copy_(self.dr[T])

    def capture(self):
        """Record one window into a CUDA graph (replayed by ``run``)."""
        s = torch.cuda.Stream(self.env.device)
        s.wait_stream(torch.cuda.current_stream(self.env.device))
        e = self.env
        live = [x for x in (self.S[0], self.goal[0], self.peff[0], e._meta, e._ep_ret, e._stats, e._imu_bias,
                            self.dr[0] if self.dr is not None else None) if x is not None]
        snap = [x.clone() for x in live]
        with torch.cuda.stream(s):
            self._run()  # warm-up outside capture (lazy init)
        torch.cuda.current_stream(self.env.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._run()
        # capture launches nothing; warm-up did: restore the pre-warm-up state
        for dst, src in zip(live, snap):
            dst.copy_(src)
        self.graph = g
        self._bound = self._env_buffers()
        return self

    def _env_buffers(self):
        """The env objects a window (captured or eager) points at; env.reset()
        replaces them."""
        e = self.env
        return (e._meta, e._ep_ret, e._stats, e._err, e._imu_bias, e._scene, e._cfg)

    def _stale(self) -> bool:
        return any(a is not b for a, b in zip(self._bound, self._env_buffers()))

    def _refresh(self):
        """After env.reset(): reload the carried state from the env (graph,
        pipeline and eager paths alike) and re-capture what was captured."""
        if not self._stale():
            return
        self._load_env_state()
        had_graph, had_pipe = self.graph is not None, getattr(self, "_pipe", None) is not None
        if had_pipe:
            self.actions = self._pipe["bufs"][0]
        self.graph = None
        self._pipe = None
        self._bound = self._env_buffers()
        if had_graph and not had_pipe:
            self.capture()

    def run(self, actions: torch.Tensor | None = None):
        """One window (fwd + bwd).  Returns (loss tensor, dL/d actions (T,N,A))."""
        self._refresh()
        if actions is not None:
            self.actions.copy_(actions, non_blocking=True)
        if self.graph is not None:
            self.graph.replay()
        else:
            self._run()
        return (self.loss64 if self.fused else self.loss), self.g_actions

    def sync_env(self):
        """Write the window's final state back into the env object."""
        self._store_env_state()

    # -- host-fed streaming: the next window's action upload overlaps this
    #    window's kernels (double-buffered device actions, one graph each)

    def _ensure_pipeline(self):
        if getattr(self, "_pipe", None) is not None:
            return
        dev = self.env.device
        # two device action buffers and two gradient buffers, one graph each:
        # window k reads actions[k%2] and writes dL/d actions into grads[k%2]
        bufs = [self.actions, torch.zeros_like(self.actions)]
        gbufs = [self.g_actions, torch.zeros_like(self.g_actions)]
        graphs = []
        keep, gkeep = self.actions, self.g_actions
        for b, gb in zip(bufs, gbufs):
            self.actions, self.g_actions = b, gb
            self.graph = None
            self.capture()
            graphs.append(self.graph)
        self.actions, self.g_actions = keep, gkeep
        self.graph = graphs[0]
        self._pipe = {"bufs": bufs, "gbufs": gbufs, "graphs": graphs, "copy": torch.cuda.Stream(dev),
                      "d2h": torch.cuda.Stream(dev)}

    def run_pipelined(self, host_batches, grad_out=None):
        """Run one window per pinned host action batch (T,N,A); returns the
        host losses.  H2D of batch k+1 runs on a copy stream while window k
        computes; each window's loss is read back with an async D2H copy.

        ``grad_out``: optional list (one per batch) of pinned host (T,N,A)
        tensors receiving each window's dL/d(actions) -- the product of a
        BPTT window (q/learners.py:251-265).  The gradient download of window
        k runs on a third stream, overlapped with window k+1's compute and
        upload (PCIe is full duplex); all copies have landed on return."""
        self._refresh()
        self._ensure_pipeline()
        P = self._pipe
        comp = torch.cuda.current_stream(self.env.device)
        cp, d2h = P["copy"], P["d2h"]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        computed = [torch.cuda.Event(), torch.cuda.Event()]
        drained = [torch.cuda.Event(), torch.cuda.Event()]
        for e in free + drained:
            e.record(comp)
        losses = torch.zeros(len(host_batches), dtype=torch.float64).pin_memory()
        # each window's loss is parked on the device by a kernel on the compute
        # stream and read back once at the end: a per-window 8-byte D2H on the
        # compute stream would queue behind the 33.5 MB gradient downloads
        loss_dev = torch.zeros(len(host_batches), dtype=torch.float64, device=self.env.device)

        def upload(k):
            b = k % 2
            with torch.cuda.stream(cp):
                cp.wait_event(free[b])
                P["bufs"][b].copy_(host_batches[k], non_blocking=True)
                ready[b].record(cp)

        if host_batches:
            upload(0)
        for k in range(len(host_batches)):
            b = k % 2
            if k + 1 < len(host_batches):
                upload(k + 1)
            comp.wait_event(ready[b])
            comp.wait_event(drained[b])  # window k-2's gradient has left grads[b]
            P["graphs"][b].replay()
            free[b].record(comp)
            loss_dev[k:k + 1].add_(self.loss64)
            if grad_out is not None:
                computed[b].record(comp)
                with torch.cuda.stream(d2h):
                    d2h.wait_event(computed[b])
                    grad_out[k].copy_(P["gbufs"][b], non_blocking=True)
                    drained[b].record(d2h)
        losses.copy_(loss_dev, non_blocking=True)
        comp.synchronize()
        if grad_out is not None:
            d2h.synchronize()
        return losses.tolist()
