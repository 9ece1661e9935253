"""One C5-size call of each learner-side tcgen05 kernel (policy GRU + trunk
forward, trunk backward, GRU backward, critic fit), for ncu:
    ncu --set full -k regex:"k_policy|k_gru|k_mlp3" python profiles/prof_policy_kernels.py
Prints CUDA-event times per call when run without ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_10247_b200 import nets  # noqa: E402

N = 131072
arch = nets.PolicyArch(proprio_dim=10, action_dim=3, recurrent=True, hidden=64, mlp=(128, 128))
pol = nets.PolicyNet(arch, np.random.default_rng(0)).cuda()
val = nets.ValueNet(14, np.random.default_rng(1)).cuda()
x = torch.randn(N, 10, device="cuda")
h0 = torch.randn(N, 64, device="cuda") * 0.5
X = torch.randn(16 * N, 14, device="cuda")
y = torch.randn(16 * N, device="cuda")


def policy_step():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        mu, ls, h = pol(x, h=h0)
    (mu.sum() + ls.sum() + h.sum()).backward()


def critic():
    nets.value_fit_grad(val, X, y)


def timed(fn, n=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


if os.environ.get("PROF_ONCE"):
    policy_step()
    critic()
    torch.cuda.synchronize()
else:
    print({"policy_step_fwd_bwd_ms": timed(policy_step), "critic_fit_ms": timed(critic)})
