import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_2509_10247_b200 as qs
from paper_2509_10247_b200.train import LearnerOptions, ShortHorizonTrainer
dev = torch.device('cuda', 0)
cfg = qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=131072, episode_len=128)
env = qs.make_task(cfg, device=dev, strict=False)
env.reset(seed=1)
tr = ShortHorizonTrainer(env, LearnerOptions(algo="shac", horizon=16, seed=0))
for _ in range(3): tr.update()
torch.cuda.synchronize()
t0=time.perf_counter()
for _ in range(3): tr.update()
torch.cuda.synchronize(); print('per update ms', (time.perf_counter()-t0)/3*1e3)
# split timing
import torch.profiler as P
with P.profile(activities=[P.ProfilerActivity.CPU, P.ProfilerActivity.CUDA]) as prof:
    tr.update(); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
