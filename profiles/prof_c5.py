"""Per-kernel device time of one C5 SHAC update (131,072 envs, horizon 16),
eager (no CUDA graph) under torch.profiler: which kernels the update spends
its time in.  Run on the GPU box; prints a table sorted by device time."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402
from paper_2509_10247_b200.train import LearnerOptions, ShortHorizonTrainer  # noqa: E402

N = 131072
cfg = qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=N, episode_len=128)
env = qs.make_task(cfg, device="cuda", strict=False)
env.reset(seed=1)
tr = ShortHorizonTrainer(env, LearnerOptions(algo="shac", horizon=16, seed=0, cuda_graph=False))
for _ in range(4):
    tr.update()
torch.cuda.synchronize()
n = 3
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(n):
        tr.update()
    torch.cuda.synchronize()
tot = 0.0
rows = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name[:90]
        t, c = rows.get(k, (0.0, 0))
        rows[k] = (t + e.device_time / n, c + 1)
        tot += e.device_time / n
print(f"total device us per update: {tot:.1f}")
for k, (t, c) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{t:9.1f} us {100 * t / tot:5.1f}%  x{c // n:4d}  {k}")

# the same, attributed to the torch operators that launched them
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof2:
    for _ in range(n):
        tr.update()
    torch.cuda.synchronize()
print(prof2.key_averages().table(sort_by="self_cuda_time_total", row_limit=30, max_name_column_width=60))
