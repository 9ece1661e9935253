"""C5 update split into phases (rollout+BPTT backward, actor step, critic fit),
each bracketed by cuda synchronize; prints ms per phase."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402
from paper_2509_10247_b200.train import LearnerOptions, ShortHorizonTrainer  # noqa: E402

dev = torch.device("cuda", 0)
env = qs.make_task(qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=131072, episode_len=128),
                   device=dev, strict=False)
env.reset(seed=1)
tr = ShortHorizonTrainer(env, LearnerOptions(algo="shac", horizon=16, seed=0))
for _ in range(3):
    tr.update()
ph = {"collect": 0.0, "backward": 0.0, "actor_step": 0.0, "critic": 0.0, "total": 0.0}
K = 5
for _ in range(K):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    disc, r_ctrl, r_goal, dones, priv = tr.collect_window(True)
    with tr._nets():
        v_term = tr.value(env.privileged_var())
    loss = -(disc + v_term.mean() * 0.99 ** 16) / 16
    torch.cuda.synchronize(); t1 = time.perf_counter()
    tr.actor_opt.zero_grad(set_to_none=True)
    loss.backward()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    torch.nn.utils.clip_grad_norm_(tr.policy.parameters(), 5.0)
    tr.actor_opt.step()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    tr._critic_update(r_ctrl, dones, priv)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    for k, v in zip(ph, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
        ph[k] += v * 1e3 / K
print({k: round(v, 2) for k, v in ph.items()})
