"""C3 closed-loop env step with and without obstacle re-randomisation on reset."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402

for regen in (False, True):
    E = 16384
    cfg = qs.TaskConfig(task="avoidance", dynamics="pm_continuous", n_envs=E, sensor="depth", depth_width=64,
                        depth_height=48, density=32 / 48.0, episode_len=32, regen_scene_on_reset=regen)
    env = qs.make_task(cfg, strict=False)
    env.reset(seed=2)
    acts = torch.randn(40, E, 3, device="cuda") * 0.3
    with torch.no_grad():
        for t in range(5):
            env.step(acts[t])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(40):
            env.step(acts[t])
        e1.record()
        torch.cuda.synchronize()
    print("regen", regen, "ms/step", e0.elapsed_time(e1) / 40)
