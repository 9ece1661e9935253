"""Host cost of one FlightTask.step (C1 shape) under cProfile."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402

cfg = qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=1024, episode_len=10 ** 6)
env = qs.make_task(cfg, device="cuda", strict=False)
env.reset(seed=1)
a = torch.zeros(1024, 3, device="cuda")
for _ in range(50):
    env.step(a)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500):
    env.step(a)
torch.cuda.synchronize()
print("us/step", (time.perf_counter() - t0) / 500 * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    env.step(a)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
