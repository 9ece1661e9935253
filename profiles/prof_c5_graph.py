"""Kernel launch list of one C5 update replayed from its CUDA graph (run under
ncu --metrics gpu__time_duration.sum): which kernels the 46 ms are made of."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402
from paper_2509_10247_b200.train import LearnerOptions, ShortHorizonTrainer  # noqa: E402

env = qs.make_task(qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=131072, episode_len=128),
                   device="cuda", strict=False)
env.reset(seed=1)
tr = ShortHorizonTrainer(env, LearnerOptions(algo="shac", horizon=16, seed=0, cuda_graph=True))
for _ in range(5):
    tr.update()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profiled_update")
tr.update()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok")
