"""Policy / value networks of the learners, as torch modules (q/nets.py).

The caller side of the simulation core: the only dense
contractions of the reference, so on the GPU they are plain torch layers whose
matmuls and convolutions run on the tensor cores through cuBLAS/cuDNN (library
code, not the hot path).  What is mirrored exactly:

- architecture and parameter names of ``q/nets.py:85-274`` -- ``Linear`` (x W +
  b, W stored (n_in, n_out)), the tanh ``MLP`` with a linear last layer, the
  GRU cell (gate order r, z, n), the two-conv ``ConvEncoder`` (3x3 stride 2,
  im2col channel-major patches, position-major flatten), the LiDAR linear
  encoder, the Gaussian policy heads with log_sigma clamped to [-5, max];
- initialisation: built with a numpy Generator, every array is drawn from it
  in the reference's order with the same Xavier scales, so a learner seeded
  like the reference starts from the reference's weights;
- the weight container (``q/nets.py:316-377``): ``manifest.json`` +
  little-endian float32 ``weights.bin``, readable by the reference and vice
  versa, with the same integrity errors.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np
import torch

CONTAINER_VERSION = 1  # q/nets.py:21
LOG_SIGMA_MIN = -5.0
LOG_SIGMA_MAX = 2.0


class IntegrityError(RuntimeError):
    """q/nets.py:26-27."""


def _xavier(rng, n_in, n_out, scale=1.0):  # q/nets.py:64-66
    s = scale * np.sqrt(2.0 / (n_in + n_out))
    return rng.normal(scale=s, size=(n_in, n_out))


class _LinearFn(torch.autograd.Function):
    """x W + b whose bias gradient is a (1 x M) @ (M x n) GEMM.  torch's own
    addmm backward reduces the bias gradient with a generic column-reduction
    kernel that runs at ~0.2 TB/s on the learners' tall (131,072 x 128) bf16
    gradients -- a quarter of a C5 update's GPU time (profiles/README.md)."""

    @staticmethod
    def forward(ctx, x, W, b):
        ctx.save_for_backward(x, W)
        return torch.addmm(b, x, W)

    @staticmethod
    def backward(ctx, g):
        x, W = ctx.saved_tensors
        g = g.contiguous()
        gx = g @ W.t() if ctx.needs_input_grad[0] else None
        gW = x.t() @ g if ctx.needs_input_grad[1] else None
        gb = None
        if ctx.needs_input_grad[2]:
            gb = (torch.ones(1, g.shape[0], dtype=g.dtype, device=g.device) @ g)[0]
        return gx, gW, gb


def _linear(x, W, b):
    if torch.is_autocast_enabled(x.device.type) and x.is_cuda:
        dt = torch.get_autocast_dtype("cuda")
        with torch.autocast("cuda", enabled=False):
            return _LinearFn.apply(x.to(dt), W.to(dt), b.to(dt))
    return _LinearFn.apply(x, W.to(x.dtype), b.to(x.dtype))


class Linear(torch.nn.Module):
    """y = x W + b with W (n_in, n_out) (q/nets.py:73-82); ``tag`` is the
    container's activation tag."""

    def __init__(self, n_in, n_out, rng=None, scale=1.0, tag="linear"):
        super().__init__()
        w = _xavier(rng, n_in, n_out, scale) if rng is not None else np.zeros((n_in, n_out))
        self.W = torch.nn.Parameter(torch.as_tensor(w, dtype=torch.float32))
        self.b = torch.nn.Parameter(torch.zeros(n_out))
        self.tag = tag

    def forward(self, x):
        return _linear(x, self.W, self.b) if x.dim() == 2 else x @ self.W + self.b


class MLP(torch.nn.Module):
    """tanh MLP, linear last layer; layers l0, l1, ... (q/nets.py:85-104)."""

    def __init__(self, n_in, hidden, n_out, rng=None, out_scale=1.0):
        super().__init__()
        sizes = [n_in] + list(hidden) + [n_out]
        self.layers = torch.nn.ModuleList()
        for i in range(len(sizes) - 1):
            last = i == len(sizes) - 2
            self.layers.append(Linear(sizes[i], sizes[i + 1], rng, out_scale if last else 1.0,
                                      "linear" if last else "tanh"))

    def forward(self, x):
        for i, layer in enumerate(self.layers):
            x = layer(x)
            if i < len(self.layers) - 1:
                x = torch.tanh(x)
        return x


class GRUCell(torch.nn.Module):
    """Standard GRU equations with the reference's layout (q/nets.py:107-132):
    Wi (n_in, 3H), Wh (H, 3H), gates (r, z, n)."""

    def __init__(self, n_in, n_hidden, rng=None):
        super().__init__()
        H = n_hidden
        wi = _xavier(rng, n_in, 3 * H) if rng is not None else np.zeros((n_in, 3 * H))
        wh = _xavier(rng, H, 3 * H) if rng is not None else np.zeros((H, 3 * H))
        self.Wi = torch.nn.Parameter(torch.as_tensor(wi, dtype=torch.float32))
        self.Wh = torch.nn.Parameter(torch.as_tensor(wh, dtype=torch.float32))
        self.bi = torch.nn.Parameter(torch.zeros(3 * H))
        self.bh = torch.nn.Parameter(torch.zeros(3 * H))
        self.n_hidden = H

    def forward(self, x, h):
        if x.is_cuda:
            # gate GEMMs through _linear (input padded to a multiple of 16
            # features: cuBLAS picks slow legacy kernels for K = 9), then torch's
            # fused gate kernel, which has the same (r, z, n) equations
            pad = (-x.shape[1]) % 16
            xp = torch.nn.functional.pad(x, (0, pad)) if pad else x
            Wi = torch.nn.functional.pad(self.Wi, (0, 0, 0, pad)) if pad else self.Wi
            gi = _linear(xp, Wi, self.bi)
            gh = _linear(h.to(gi.dtype) if gi.dtype != h.dtype else h, self.Wh, self.bh)
            return torch.ops.aten._thnn_fused_gru_cell(gi, gh, h.to(gi.dtype))[0]
        if x.dtype == torch.float32:
            return torch._VF.gru_cell(x, h, self.Wi.t(), self.Wh.t(), self.bi, self.bh)
        H = self.n_hidden
        gi = x @ self.Wi + self.bi
        gh = h @ self.Wh + self.bh
        r = torch.sigmoid(gi[:, :H] + gh[:, :H])
        z = torch.sigmoid(gi[:, H:2 * H] + gh[:, H:2 * H])
        n = torch.tanh(gi[:, 2 * H:] + r * gh[:, 2 * H:])
        return (1.0 - z) * n + z * h


class ConvEncoder(torch.nn.Module):
    """Two 3x3 stride-2 tanh convs (1 -> c1 -> c2), position-major flatten,
    tanh linear (q/nets.py:135-180).  k1 (9, c1), k2 (9 c1, c2) in the
    reference's im2col layout (row = c_in * 9 + 3 di + dj)."""

    def __init__(self, height, width, n_out, rng=None, c1=8, c2=16):
        super().__init__()
        self.c1, self.c2 = c1, c2
        self.h1, self.w1 = (height - 3) // 2 + 1, (width - 3) // 2 + 1
        self.h2, self.w2 = (self.h1 - 3) // 2 + 1, (self.w1 - 3) // 2 + 1
        if self.h2 < 1 or self.w2 < 1:
            raise ValueError(f"image {height}x{width} too small for the 2-conv encoder")
        z = lambda *s: np.zeros(s)  # noqa: E731
        self.k1 = torch.nn.Parameter(torch.as_tensor(_xavier(rng, 9, c1) if rng is not None else z(9, c1),
                                                     dtype=torch.float32))
        self.b1 = torch.nn.Parameter(torch.zeros(c1))
        self.k2 = torch.nn.Parameter(torch.as_tensor(_xavier(rng, 9 * c1, c2) if rng is not None
                                                     else z(9 * c1, c2), dtype=torch.float32))
        self.b2 = torch.nn.Parameter(torch.zeros(c2))
        self.flat = c2 * self.h2 * self.w2
        self.out = Linear(self.flat, n_out, rng, tag="tanh")

    @staticmethod
    def _kernel(k, c_in):  # (c_in * 9, c_out) -> (c_out, c_in, 3, 3)
        return k.t().reshape(k.shape[1], c_in, 3, 3)

    def forward(self, img):
        B = img.shape[0]
        x = img.reshape(B, 1, img.shape[-2], img.shape[-1])
        k1, k2 = self._kernel(self.k1, 1).to(x.dtype), self._kernel(self.k2, self.c1).to(x.dtype)
        y = torch.tanh(torch.nn.functional.conv2d(x, k1, self.b1.to(x.dtype), stride=2))
        y = torch.tanh(torch.nn.functional.conv2d(y, k2, self.b2.to(x.dtype), stride=2))
        feat = y.permute(0, 2, 3, 1).reshape(B, self.flat)  # position-major, as the im2col rows
        return torch.tanh(self.out(feat))


# the GRU cell, trunk and heads of the reference policy shape on the tcgen05
# kernels (qs_policy_gru_fwd/_bwd, qs_policy_trunk_fwd/_bwd) under bf16
# autocast; QS_POLICY_TRUNK=torch keeps torch's GEMMs
FUSED_TRUNK = os.environ.get("QS_POLICY_TRUNK", "tc") != "torch"


def _work(which, n_sm, dev):
    """Scratch for a policy gradient kernel's per-CTA partials (0 trunk, 1 GRU)."""
    from paper_2509_10247_b200 import _lib as L

    return torch.empty(L.lib().qs_policy_work_floats(which, n_sm), dtype=torch.float32, device=dev)


class _TrunkFn(torch.autograd.Function):
    """y = tanh(tanh(tanh(h W0 + b0) W1 + b1) W2 + b2) Wh + bh (q/nets.py:241-256)
    as two tcgen05 kernels: the forward, and a backward that recomputes the
    forward per 128-row tile and returns dL/dh with every parameter gradient
    (bf16 operands, fp32 accumulation -- torch's bf16 autocast arithmetic)."""

    @staticmethod
    def forward(ctx, h, W0, b0, W1, b1, W2, b2, Wh, bh):
        from paper_2509_10247_b200 import _lib as L

        h = h.contiguous()
        ws = [t.detach().float().contiguous() for t in (W0, b0, W1, b1, W2, b2, Wh, bh)]
        N, n_out = h.shape[0], ws[6].shape[1]
        y = torch.empty(N, n_out, dtype=torch.float32, device=h.device)
        n_sm = torch.cuda.get_device_properties(h.device).multi_processor_count
        L.check(L.lib().qs_policy_trunk_fwd(N, n_out, L.ptr(h), *[L.ptr(t) for t in ws], L.ptr(y), n_sm,
                                            L.stream_handle(h.device)), "qs_policy_trunk_fwd")
        ctx.save_for_backward(h, *ws[:7])
        ctx.n_sm = n_sm
        return y

    @staticmethod
    def backward(ctx, gy):
        from paper_2509_10247_b200 import _lib as L

        h, W0, b0, W1, b1, W2, b2, Wh = ctx.saved_tensors
        gy = gy.contiguous().float()
        N, n_out = gy.shape
        dh = torch.empty_like(h)
        grads = [torch.empty_like(t) for t in (W0, b0, W1, b1, W2, b2, Wh)]
        gbh = torch.empty(n_out, dtype=torch.float32, device=h.device)
        work = _work(0, ctx.n_sm, h.device)
        L.check(L.lib().qs_policy_trunk_bwd(N, n_out, None, L.ptr(h), L.ptr(gy), *[L.ptr(t) for t in
                                                                              (W0, b0, W1, b1, W2, b2, Wh)],
                                            L.ptr(dh), *[L.ptr(t) for t in grads], L.ptr(gbh), L.ptr(work),
                                            work.numel(), ctx.n_sm,
                                            L.stream_handle(h.device)), "qs_policy_trunk_bwd")
        return (dh, *grads, gbh)


class _PolicyStepFn(torch.autograd.Function):
    """(h', y) = (GRU(x * scale, h masked by reset), trunk + heads of h')
    (q/nets.py:107-132, 241-256) in one tcgen05 kernel (qs_policy_gru_fwd);
    the backward is the trunk's (qs_policy_trunk_bwd, dL/dy -> dL/dh') then the
    GRU cell's (qs_policy_gru_bwd, dL/dh' from the trunk plus the carried one).
    The parameters enter as ONE flat tensor (``PolicyNet.pack_weights``, layout
    ``_pack_offsets``): a rollout packs them once, and the 16 steps' gradients
    accumulate into one buffer instead of 14 per step.  The kernels run in
    planar mode: y is (2, N, A) -- mu, then log-sigma, each contiguous -- and
    the heads [W_mu | W_sigma], [b_mu | b_sigma] are read and their gradients
    written as the flat buffer's own slices (no concatenation or split)."""

    @staticmethod
    def forward(ctx, x, scale, h, reset, wp, n_in, A):
        from paper_2509_10247_b200 import _lib as L

        ctx.set_materialize_grads(False)
        x, h = x.contiguous(), h.contiguous()
        rs = reset.contiguous().view(torch.uint8) if reset is not None else None
        img = getattr(wp, "_qs_image", None)  # bf16 weight image built with the pack (once per rollout)
        wp = wp.detach()
        offs = _pack_offsets(n_in, A)
        if wp.numel() != sum(n for _, n in offs.values()):
            raise ValueError("packed policy weights do not match this policy's shapes")
        v = {k: wp[o:o + n] for k, (o, n) in offs.items()}
        N = x.shape[0]
        if img is None:
            img = _policy_image(v, n_in, A)
        h_out = torch.empty(N, h.shape[1], dtype=torch.float32, device=x.device)
        y = torch.empty(2, N, A, dtype=torch.float32, device=x.device)
        n_sm = torch.cuda.get_device_properties(x.device).multi_processor_count
        L.check(L.lib().qs_policy_gru_fwd(N, n_in, 2 * A, L.ptr(img), L.ptr(x), L.ptr(scale), L.ptr(h), L.ptr(rs),
                                          *[L.ptr(v[k]) for k in ("Wi", "bi", "Wg", "bg", "W0", "b0", "W1", "b1", "W2",
                                                                  "b2", "Wh", "bh")],
                                          L.ptr(h_out), L.ptr(y), 1, n_sm, L.stream_handle(x.device)),
                "qs_policy_gru_fwd")
        ctx.save_for_backward(x, scale, h, rs, h_out, wp, img)
        ctx.n_sm, ctx.A, ctx.n_in = n_sm, A, n_in
        return h_out, y

    @staticmethod
    def backward(ctx, g_h, g_y):
        from paper_2509_10247_b200 import _lib as L

        x, scale, h, rs, h_out, wp, img = ctx.saved_tensors
        N, A, n_in = x.shape[0], ctx.A, ctx.n_in
        dev, st = x.device, L.stream_handle(x.device)
        offs = _pack_offsets(n_in, A)
        v = {k: wp[o:o + n] for k, (o, n) in offs.items()}
        gw = torch.empty_like(wp)  # every slice is written by the two kernels
        gv = {k: gw[o:o + n] for k, (o, n) in offs.items()}
        g_y = torch.zeros(2, N, A, device=dev) if g_y is None else g_y.contiguous().float()
        g_h = None if g_h is None else g_h.contiguous().float()
        dh_t = torch.empty_like(h_out)
        work = _work(0, ctx.n_sm, dev)
        L.check(L.lib().qs_policy_trunk_bwd(N, 2 * A, L.ptr(img), L.ptr(h_out), L.ptr(g_y), 1,
                                            *[L.ptr(v[k]) for k in ("W0", "b0", "W1", "b1", "W2", "b2", "Wh")],
                                            L.ptr(dh_t),
                                            *[L.ptr(gv[k]) for k in ("W0", "b0", "W1", "b1", "W2", "b2", "Wh", "bh")],
                                            L.ptr(work), work.numel(), ctx.n_sm, st), "qs_policy_trunk_bwd")
        dx, dh = torch.empty_like(x), torch.empty_like(h)
        work = _work(1, ctx.n_sm, dev)
        L.check(L.lib().qs_policy_gru_bwd(N, n_in, L.ptr(img), L.ptr(x), L.ptr(scale), L.ptr(h), L.ptr(rs),
                                          L.ptr(dh_t), L.ptr(g_h), *[L.ptr(v[k]) for k in ("Wi", "bi", "Wg", "bg")],
                                          L.ptr(dx), L.ptr(dh), *[L.ptr(gv[k]) for k in ("Wi", "bi", "Wg", "bg")],
                                          L.ptr(work), work.numel(), ctx.n_sm, st), "qs_policy_gru_bwd")
        return dx, None, dh, None, gw, None, None


def _policy_image(v, n_in, A):
    """The kernels' bf16 weight image (qs_policy_pack_image) of the packed slices v."""
    from paper_2509_10247_b200 import _lib as L

    dev = v["W0"].device
    img = torch.empty(L.lib().qs_policy_image_bytes() // 2, dtype=torch.bfloat16, device=dev)
    L.check(L.lib().qs_policy_pack_image(n_in, 2 * A, L.ptr(v["Wi"]), L.ptr(v["Wg"]), L.ptr(v["W0"]),
                                         L.ptr(v["W1"]), L.ptr(v["W2"]), L.ptr(v["Wh"]), 1, L.ptr(img),
                                         L.stream_handle(dev)), "qs_policy_pack_image")
    return img


def _pack_offsets(n_in, A, H=64, W=128):
    """Flat layout of the fused policy-step parameters: the order of
    ``PolicyNet._fused_params``, with the two heads as the planar blocks the
    kernels read -- Wh = [W_mu | W_sigma] as (2, 128, A), bh = [b_mu | b_sigma].
    Every matrix starts on a 16-byte boundary (16-byte staging loads)."""
    sizes = [("Wi", n_in * 3 * H), ("bi", 3 * H), ("Wg", H * 3 * H), ("bg", 3 * H), ("W0", H * W), ("b0", W),
             ("W1", W * W), ("b1", W), ("W2", W * W), ("b2", W), ("Wh", 2 * W * A), ("bh", 2 * A)]
    out, o = {}, 0
    for k, n in sizes:
        out[k] = (o, n)
        o += n
    return out


@dataclass
class PolicyArch:
    """q/nets.py:183-195."""

    proprio_dim: int
    action_dim: int
    visual: dict | None = None  # {"kind": "depth", "height", "width", "max_range"} | {"kind": "lidar", "rays", ...}
    recurrent: bool = True
    hidden: int = 64
    mlp: tuple = (128, 128)
    conv_feat: int = 32
    log_sigma_init: float = -1.2
    log_sigma_max: float = LOG_SIGMA_MAX
    input_scale: tuple | None = None


class PolicyNet(torch.nn.Module):
    """Optionally recurrent, optionally convolutional Gaussian policy
    (q/nets.py:198-256): forward -> (mu, log_sigma, next_hidden)."""

    def __init__(self, arch: PolicyArch, rng=None):
        super().__init__()
        self.arch = arch
        # fp64 like the reference's conditioning; cast to the input's dtype per call
        scale = torch.ones(arch.proprio_dim, dtype=torch.float64) if arch.input_scale is None else \
            torch.as_tensor(arch.input_scale, dtype=torch.float64)
        self.register_buffer("input_scale", scale)
        feat = arch.proprio_dim
        self.enc = None
        if arch.visual is not None:
            if arch.visual["kind"] == "depth":
                self.enc = ConvEncoder(arch.visual["height"], arch.visual["width"], arch.conv_feat, rng)
            else:  # lidar ranges enter as a flat vector
                self.enc = Linear(arch.visual["rays"], arch.conv_feat, rng, tag="tanh")
            feat += arch.conv_feat
        self.gru = GRUCell(feat, arch.hidden, rng) if arch.recurrent else None
        self.trunk = MLP(arch.hidden if arch.recurrent else feat, arch.mlp, arch.mlp[-1], rng)
        self.mu = Linear(arch.mlp[-1], arch.action_dim, rng, scale=0.01)
        self.sig = Linear(arch.mlp[-1], arch.action_dim, rng, scale=0.01)
        with torch.no_grad():
            self.sig.b.fill_(arch.log_sigma_init)
        self.hidden = arch.hidden

    def _fused_params(self):
        """The parameters of the fused policy step, in ``_pack_offsets`` order."""
        g, L = self.gru, self.trunk.layers
        return [g.Wi, g.bi, g.Wh, g.bh, L[0].W, L[0].b, L[1].W, L[1].b, L[2].W, L[2].b, self.mu.W,
                self.sig.W, self.mu.b, self.sig.b]

    def _scale_f32(self):
        """The input scale as fp32 on the module's device (cached; the buffer is fp64)."""
        sc = self.input_scale
        key = (sc.device, sc.data_ptr(), sc._version)
        if getattr(self, "_scale_key", None) != key:
            self._scale_cache = sc.to(torch.float32).contiguous()
            self._scale_key = key
        return self._scale_cache

    def pack_weights(self):
        """One flat, differentiable copy of the fused step's parameters; pass
        it to every step of a rollout (``forward(..., packed=...)``) so their
        gradients accumulate in one buffer.  None when the fused step does
        not apply to this architecture."""
        if self.gru is None or self.hidden != 64 or tuple(self.arch.mlp) != (128, 128) or \
                2 * self.arch.action_dim > 8:
            return None
        wp = torch.cat([p.reshape(-1) for p in self._fused_params()])
        if wp.is_cuda:  # the kernels' bf16 weight image, built once with the pack
            with torch.no_grad():
                n_in = self.gru.Wi.shape[0]
                v = {k: wp[o:o + n] for k, (o, n) in _pack_offsets(n_in, self.arch.action_dim).items()}
                wp._qs_image = _policy_image(v, n_in, self.arch.action_dim)
        return wp

    def initial_hidden(self, batch, device=None):
        return torch.zeros(batch, self.hidden, device=device) if self.gru is not None else None

    def forward(self, proprio, visual=None, h=None, h_reset=None, packed=None):
        """h_reset (bool (N,), optional): rows whose carried hidden state
        restarts at zero before this step (the trainer's episode resets,
        q/learners.py:215-217), folded into the fused kernel when it runs.
        packed: ``pack_weights()`` of this module, reused across a rollout."""
        A = self.arch.action_dim
        layers = self.trunk.layers
        trunk_ok = (FUSED_TRUNK and proprio.is_cuda and proprio.dim() == 2 and proprio.dtype == torch.float32 and
                    torch.is_autocast_enabled() and len(layers) == 3 and
                    tuple(l.W.shape for l in layers) == ((64, 128), (128, 128), (128, 128)) and 2 * A <= 8)
        if (trunk_ok and self.enc is None and self.gru is not None and self.hidden == 64 and
                proprio.shape[1] <= 16):
            # bf16 policy mode: input scale, GRU cell, trunk and both heads in one
            # tcgen05 kernel; mu and log-sigma come out as two contiguous planes
            if h is None:
                h = torch.zeros(proprio.shape[0], self.hidden, device=proprio.device)
            wp = packed if packed is not None else self.pack_weights()
            h, y = _PolicyStepFn.apply(proprio, self._scale_f32(), h.float(), h_reset, wp, proprio.shape[1], A)
            mu, ls = y.unbind(0)
            return mu, torch.clamp(ls, LOG_SIGMA_MIN, self.arch.log_sigma_max), h
        x = proprio * self.input_scale.to(proprio.dtype)
        if self.enc is not None:
            if visual is None:
                raise ValueError("policy expects a visual observation")
            img = visual.to(x.dtype) * (1.0 / float(self.arch.visual.get("max_range", 1.0)))
            f = self.enc(img) if self.arch.visual["kind"] == "depth" else torch.tanh(self.enc(img))
            x = torch.cat([x, f.to(x.dtype)], -1)
        trunk_ok = trunk_ok and x.dtype == torch.float32
        if self.gru is not None:
            if h is None:
                h = torch.zeros(x.shape[0], self.hidden, device=x.device, dtype=x.dtype)
            elif h_reset is not None:
                h = torch.where(h_reset[:, None], torch.zeros_like(h), h)
            h = self.gru(x, h.to(x.dtype)).float() if x.dtype != torch.float64 else self.gru(x, h)
            x = h.to(x.dtype)
        if trunk_ok and x.shape[1] == 64:
            # bf16 policy mode: trunk and both heads in two tcgen05 kernels
            y = _TrunkFn.apply(x, layers[0].W, layers[0].b, layers[1].W, layers[1].b, layers[2].W, layers[2].b,
                               torch.cat([self.mu.W, self.sig.W], 1), torch.cat([self.mu.b, self.sig.b]))
            return y[:, :A], torch.clamp(y[:, A:2 * A], LOG_SIGMA_MIN, self.arch.log_sigma_max), h
        z = torch.tanh(self.trunk(x))
        if z.is_cuda and z.dim() == 2:
            # both heads as ONE GEMM, widened to a multiple of 8 outputs (the
            # narrow N = A GEMMs, and their weight-gradient GEMMs with N = A,
            # fall to slow unaligned kernels)
            pad = (-2 * A) % 8
            W = torch.nn.functional.pad(torch.cat([self.mu.W, self.sig.W], 1), (0, pad))
            b = torch.nn.functional.pad(torch.cat([self.mu.b, self.sig.b]), (0, pad))
            y = _linear(z, W, b)
            mu, ls = y[:, :A], y[:, A:2 * A]
        else:
            mu, ls = self.mu(z), self.sig(z)
        out_t = torch.float64 if z.dtype == torch.float64 else torch.float32
        return mu.to(out_t), torch.clamp(ls.to(out_t), LOG_SIGMA_MIN, self.arch.log_sigma_max), h

    def n_params(self) -> int:
        return sum(p.numel() for p in self.parameters())


class ValueNet(torch.nn.Module):
    """Privileged-state MLP critic (q/nets.py:259-274): (B, K) -> (B,);
    parameters value.l0, value.l1, ..."""

    def __init__(self, n_in, rng=None, hidden=(128, 128), input_scale=None):
        super().__init__()
        scale = torch.ones(n_in, dtype=torch.float64) if input_scale is None else \
            torch.as_tensor(input_scale, dtype=torch.float64)
        self.register_buffer("input_scale", scale)
        self.value = MLP(n_in, hidden, 1, rng)

    def forward(self, x):
        x = x * self.input_scale.to(x.dtype)
        y = self.value(x)[..., 0]
        return y if y.dtype == torch.float64 else y.float()

    def n_params(self) -> int:
        return sum(p.numel() for p in self.parameters())


def value_fit_grad(value: "ValueNet", x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """Full-batch gradient of L = mean((value(x) - y)^2) written into the
    ``.grad`` of every ValueNet parameter by ONE fused kernel (forward and
    backward on the tensor cores, activations never leave shared memory;
    ``qs_mlp3_fit_grad``).  Returns L (a device scalar, no host sync).  For the
    reference critic shape: two tanh layers of width 128, at most 16 inputs,
    fp32 CUDA tensors x (M, K), y (M,)."""
    from paper_2509_10247_b200 import _lib as L

    layers = value.value.layers
    if len(layers) != 3 or layers[0].W.shape[1] != 128 or layers[1].W.shape != (128, 128) or \
            layers[2].W.shape != (128, 1) or x.shape[1] > 16:
        raise ValueError("value_fit_grad: needs the (128, 128) critic with <= 16 inputs")
    dev = x.device
    x = x.contiguous().float()
    y = y.contiguous().float()
    M, K = x.shape
    params = [layers[0].W, layers[0].b, layers[1].W, layers[1].b, layers[2].W, layers[2].b]
    flat = torch.zeros(sum(p.numel() for p in params) + 1, dtype=torch.float32, device=dev)
    grads, off = [], 0
    for p in params:
        grads.append(flat[off:off + p.numel()].view_as(p))
        off += p.numel()
    loss = flat[off:]
    scale = value.input_scale.to(device=dev, dtype=torch.float32).contiguous()
    w = [p.detach().float().contiguous() for p in params]
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    # tcgen05 kernel (TMEM accumulators) for <= 14 inputs -- the privileged
    # state's 14; the mma.sync kernel otherwise (QS_CRITIC_KERNEL=mma forces it)
    tc = K <= 14 and os.environ.get("QS_CRITIC_KERNEL", "tc") != "mma"
    args = [M, K, L.ptr(x), L.ptr(scale), L.ptr(y), L.ptr(w[0]), L.ptr(w[1]), L.ptr(w[2]), L.ptr(w[3]),
            L.ptr(w[4]), L.ptr(w[5]), L.ptr(grads[0]), L.ptr(grads[1]), L.ptr(grads[2]), L.ptr(grads[3]),
            L.ptr(grads[4]), L.ptr(grads[5]), L.ptr(loss)]
    if tc:  # per-CTA partials summed in a fixed order: reproducible gradients
        n_work = L.lib().qs_mlp3_work_floats(n_sm)
        work = torch.empty(n_work, dtype=torch.float32, device=dev)
        L.check(L.lib().qs_mlp3_fit_grad_tc(*args, L.ptr(work), n_work, n_sm, L.stream_handle(dev)),
                "qs_mlp3_fit_grad_tc")
    else:
        L.check(L.lib().qs_mlp3_fit_grad(*args, n_sm, L.stream_handle(dev)), "qs_mlp3_fit_grad")
    for p, gr in zip(params, grads):
        p.grad = gr
    return loss[0]


def value_forward(value: "ValueNet", x: torch.Tensor) -> torch.Tensor:
    """value(x) for the reference critic shape (two tanh layers of width 128,
    <= 14 inputs) by one tcgen05 kernel (``qs_mlp3_forward_tc``; bf16 operands,
    fp32 accumulation in TMEM, as torch's bf16 autocast computes it), no
    autograd: the TD-lambda targets' values and bootstrap (q/learners.py:286-292)."""
    from paper_2509_10247_b200 import _lib as L

    layers = value.value.layers
    if len(layers) != 3 or layers[0].W.shape[1] != 128 or layers[1].W.shape != (128, 128) or \
            layers[2].W.shape != (128, 1) or x.shape[1] > 14:
        raise ValueError("value_forward: needs the (128, 128) critic with <= 14 inputs")
    dev = x.device
    x = x.contiguous().float()
    M, K = x.shape
    w = [p.detach().float().contiguous() for p in (layers[0].W, layers[0].b, layers[1].W, layers[1].b,
                                                   layers[2].W, layers[2].b)]
    scale = value.input_scale.to(device=dev, dtype=torch.float32).contiguous()
    out = torch.empty(M, dtype=torch.float32, device=dev)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    L.check(L.lib().qs_mlp3_forward_tc(M, K, L.ptr(x), L.ptr(scale), L.ptr(w[0]), L.ptr(w[1]), L.ptr(w[2]),
                                       L.ptr(w[3]), L.ptr(w[4]), L.ptr(w[5]), L.ptr(out), n_sm,
                                       L.stream_handle(dev)), "qs_mlp3_forward_tc")
    return out


# ---------------------------------------------------------------------------
# the reference's parameter names <-> module parameters


def ref_params(module: torch.nn.Module) -> dict:
    """Ordered {reference name: (parameter, activation tag)}, in the order the
    reference's ParamSet holds them (its construction order)."""
    out = {}
    if isinstance(module, PolicyNet):
        if module.enc is not None:
            if isinstance(module.enc, ConvEncoder):
                e = module.enc
                out.update({"enc.k1": (e.k1, "conv"), "enc.b1": (e.b1, "conv"), "enc.k2": (e.k2, "conv"),
                            "enc.b2": (e.b2, "conv"), "enc.out.W": (e.out.W, "tanh"),
                            "enc.out.b": (e.out.b, "tanh")})
            else:
                out.update({"enc.lidar.W": (module.enc.W, "tanh"), "enc.lidar.b": (module.enc.b, "tanh")})
        if module.gru is not None:
            g = module.gru
            out.update({"gru.Wi": (g.Wi, "gru"), "gru.Wh": (g.Wh, "gru"), "gru.bi": (g.bi, "gru"),
                        "gru.bh": (g.bh, "gru")})
        for i, layer in enumerate(module.trunk.layers):
            out[f"trunk.l{i}.W"] = (layer.W, layer.tag)
            out[f"trunk.l{i}.b"] = (layer.b, layer.tag)
        out.update({"mu.W": (module.mu.W, "linear"), "mu.b": (module.mu.b, "linear"),
                    "sig.W": (module.sig.W, "linear"), "sig.b": (module.sig.b, "linear")})
    elif isinstance(module, ValueNet):
        for i, layer in enumerate(module.value.layers):
            out[f"value.l{i}.W"] = (layer.W, layer.tag)
            out[f"value.l{i}.b"] = (layer.b, layer.tag)
    else:
        raise TypeError("ref_params expects a PolicyNet or ValueNet")
    return out


def save_container(dirpath: str, modules: dict, meta: dict) -> None:
    """manifest.json + weights.bin, little-endian float32 (q/nets.py:316-345);
    ``modules`` maps set names ("policy", "value") to PolicyNet / ValueNet."""
    os.makedirs(dirpath, exist_ok=True)
    layers, blobs, offset = [], [], 0
    for set_name, mod in modules.items():
        for name, (p, tag) in ref_params(mod).items():
            a32 = p.detach().double().cpu().numpy().astype("<f4")
            layers.append({"set": set_name, "name": name, "shape": list(a32.shape), "activation": tag,
                           "offset": offset})
            blobs.append(a32.tobytes(order="C"))
            offset += a32.size
    manifest = {"format_version": CONTAINER_VERSION, "total_floats": offset, "layers": layers, **meta}
    with open(os.path.join(dirpath, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=2)
    with open(os.path.join(dirpath, "weights.bin"), "wb") as f:
        f.write(b"".join(blobs))


def read_container(dirpath: str):
    """(arrays {set: {name: float64 ndarray}}, manifest) with the reference's
    integrity checks (q/nets.py:348-377)."""
    try:
        with open(os.path.join(dirpath, "manifest.json")) as f:
            manifest = json.load(f)
    except (OSError, json.JSONDecodeError) as e:
        raise IntegrityError(f"unreadable manifest: {e}")
    if manifest.get("format_version") != CONTAINER_VERSION:
        raise IntegrityError(f"unsupported container version {manifest.get('format_version')}")
    try:
        blob = np.fromfile(os.path.join(dirpath, "weights.bin"), dtype="<f4")
    except OSError as e:
        raise IntegrityError(f"unreadable weight blob: {e}")
    if blob.size != manifest["total_floats"]:
        raise IntegrityError(f"weight blob holds {blob.size} floats, manifest expects {manifest['total_floats']}")
    sets: dict = {}
    for layer in manifest["layers"]:
        n = int(np.prod(layer["shape"])) if layer["shape"] else 1
        vals = blob[layer["offset"]:layer["offset"] + n]
        if vals.size != n:
            raise IntegrityError(f"layer '{layer['name']}' truncated")
        sets.setdefault(layer["set"], {})[layer["name"]] = vals.astype(np.float64).reshape(layer["shape"])
    return sets, manifest


load_container = read_container  # q/nets.py:348 name; arrays in place of ParamSets


def load_into(module: torch.nn.Module, arrays: dict) -> None:
    """Copy one container set into a PolicyNet / ValueNet (names and shapes
    must match the module's architecture)."""
    want = ref_params(module)
    missing = set(want) - set(arrays)
    extra = set(arrays) - set(want)
    if missing or extra:
        raise IntegrityError(f"container/architecture mismatch: missing {sorted(missing)}, extra {sorted(extra)}")
    with torch.no_grad():
        for name, (p, _tag) in want.items():
            a = torch.as_tensor(arrays[name])
            if tuple(a.shape) != tuple(p.shape):
                raise IntegrityError(f"layer '{name}': shape {tuple(a.shape)} != {tuple(p.shape)}")
            p.copy_(a.to(p.dtype))
