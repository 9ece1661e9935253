"""Multi-agent avoidance windows (C4 sim side) for timing / ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402
from paper_2509_10247_b200.window import BpttWindow  # noqa: E402


def run(density, n_agents=4, envs=4096, task="avoidance", reps=5):
    cfg = qs.TaskConfig(task=task, dynamics="pm_continuous", n_envs=envs, n_agents=n_agents, formation="line",
                        formation_side=1.0, episode_len=128, density=density)
    env = qs.make_task(cfg, device="cuda", strict=False)
    for seed in range(1, 20):
        try:
            env.reset(seed=seed)
            break
        except qs.world.GenerationError:
            continue
    win = BpttWindow(env, 32)
    g = torch.Generator().manual_seed(0)
    win.actions.copy_(torch.randn(32, env.N, env.action_dim, generator=g).cuda() * 0.3)
    win.capture()
    for _ in range(2):
        win.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        win.run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(task, "density", density, "agents", n_agents, "ms/window", round(ms, 3), "row-steps/s",
          f"{env.N * 32 / ms * 1e3:.3e}", "finished", env.finished_episodes, "err", env._err.tolist())


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(float(sys.argv[1]), reps=1)
    else:
        run(0.1)
        run(0.0)
        run(0.1, n_agents=1, envs=16384)
        run(0.0, n_agents=4, task="position")
