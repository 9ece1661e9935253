"""torch profiler table of one C5 rollout window (collect_window)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402
from paper_2509_10247_b200.train import LearnerOptions, ShortHorizonTrainer  # noqa: E402

env = qs.make_task(qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=131072, episode_len=128),
                   device="cuda", strict=False)
env.reset(seed=1)
tr = ShortHorizonTrainer(env, LearnerOptions(algo="shac", horizon=16, seed=0))
for _ in range(3):
    tr.update()
torch.cuda.synchronize()
import torch.profiler as P  # noqa: E402

with P.profile(activities=[P.ProfilerActivity.CPU, P.ProfilerActivity.CUDA]) as prof:
    out = tr.collect_window(True)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=22))
