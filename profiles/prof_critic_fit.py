"""Critic fit pieces at C5 size (2,097,152 rows x 14): the fused gradient
kernel vs torch autograd (bf16 autocast), and the value forward used for the
TD-lambda targets."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_10247_b200 import nets  # noqa: E402


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


M = 16 * 131072
val = nets.ValueNet(14, np.random.default_rng(0)).cuda()
X = torch.randn(M, 14, device="cuda")
y = torch.randn(M, device="cuda")


def fused():
    nets.value_fit_grad(val, X, y)


def torch_ag():
    for p in val.parameters():
        p.grad = None
    with torch.autocast("cuda", dtype=torch.bfloat16):
        pred = val(X)
    ((pred - y) ** 2).mean().backward()


def fwd():
    with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
        val(X)


def fwd_tc():
    nets.value_forward(val, X)


res = {"fused_grad_ms": timed(fused), "torch_autocast_grad_ms": timed(torch_ag), "torch_fwd_ms": timed(fwd),
       "tcgen05_fwd_ms": timed(fwd_tc)}
flops = M * 2 * (16 * 128 + 3 * 128 * 128 + 16 * 128)
res["fused_tflops"] = flops / (res["fused_grad_ms"] * 1e-3) / 1e12
print(res)
