"""C1 drop-in path: 32 x FlightTask.step + autograd backward at 1,024 envs;
host time split (forward loop / backward) and cProfile of the backward."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402

env = qs.make_task(qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=1024, episode_len=10 ** 6),
                   device="cuda", strict=False)
env.reset(seed=1)
acts = torch.randn(32, 1024, 3, device="cuda") * 0.3


def window():
    a = acts.clone().requires_grad_(True)
    env.detach_states()
    tot = 0.0
    t0 = time.perf_counter()
    for t in range(32):
        tot = tot + env.step(a[t]).r_ctrl.mean() * 0.99 ** t
    loss = -tot / 32
    t1 = time.perf_counter()
    loss.backward()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


for _ in range(5):
    window()
f = b = 0.0
for _ in range(20):
    x, y = window()
    f += x / 20
    b += y / 20
print(f"forward loop {f*1e3:.2f} ms, backward {b*1e3:.2f} ms")
pr = cProfile.Profile()
a = acts.clone().requires_grad_(True)
env.detach_states()
tot = 0.0
for t in range(32):
    tot = tot + env.step(a[t]).r_ctrl.mean() * 0.99 ** t
loss = -tot / 32
pr.enable()
loss.backward()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
