"""Time of the policy-step kernels against the row count (1..8+ tiles per
SM): the intercept is the per-CTA prologue (weight staging), the slope the
per-tile cost."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_10247_b200 import _lib as L  # noqa: E402


def ev_time(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


g = torch.Generator().manual_seed(0)
r = lambda *s, sc=0.1: (torch.randn(*s, generator=g) * sc).cuda()  # noqa: E731
n_in, A = 10, 3
Wi, bi, Wg, bg = r(n_in, 192), r(192), r(64, 192), r(192)
W0, b0, W1, b1, W2, b2, Wh, bh = r(64, 128), r(128), r(128, 128), r(128), r(128, 128), r(128), r(128, 6), r(6)
n_sm = torch.cuda.get_device_properties(0).multi_processor_count
P = lambda *ts: [L.ptr(t) for t in ts]  # noqa: E731
st = L.stream_handle()
for tiles_per_sm in (1, 2, 4, 7, 14, 28):
    N = 128 * n_sm * tiles_per_sm
    x, h = r(N, n_in), r(N, 64)
    ho, y = torch.empty(N, 64, device="cuda"), torch.empty(N, 6, device="cuda")
    dy, dh = r(N, 6), torch.empty(N, 64, device="cuda")
    gr = [torch.empty_like(t) for t in (W0, b0, W1, b1, W2, b2, Wh, bh)]
    gg = [torch.empty_like(t) for t in (Wi, bi, Wg, bg)]
    w0 = torch.empty(L.lib().qs_policy_work_floats(0, n_sm), device="cuda")
    w1 = torch.empty(L.lib().qs_policy_work_floats(1, n_sm), device="cuda")
    dx = torch.empty_like(x)
    img = torch.empty(L.lib().qs_policy_image_bytes() // 2, dtype=torch.bfloat16, device="cuda")
    L.lib().qs_policy_pack_image(n_in, 6, *P(Wi, Wg, W0, W1, W2, Wh), 0, L.ptr(img), st)
    fwd = ev_time(lambda: L.lib().qs_policy_gru_fwd(N, n_in, 6, L.ptr(img), L.ptr(x), None, L.ptr(h), None, *P(Wi, bi, Wg, bg, W0, b0, W1, b1, W2,
                                                                                  b2, Wh, bh, ho, y), 0, n_sm, st))
    tb = ev_time(lambda: L.lib().qs_policy_trunk_bwd(N, 6, L.ptr(img), *P(ho, dy), 0, *P(W0, b0, W1, b1, W2, b2, Wh, dh, *gr, w0),
                                                     w0.numel(), n_sm, st))
    gb = ev_time(lambda: L.lib().qs_policy_gru_bwd(N, n_in, L.ptr(img), L.ptr(x), None, L.ptr(h), None, *P(dh), None, *P(Wi, bi, Wg, bg, dx, dh,
                                                                                            *gg, w1), w1.numel(), n_sm,
                                                   st))
    print(f"tiles/SM {tiles_per_sm:3d}  N {N:8d}  fwd {fwd:7.1f} us  trunk_bwd {tb:7.1f} us  gru_bwd {gb:7.1f} us")
