"""A/B timing of the C2 window kernels between library builds.

    QS_LIB_PATH=<lib.so> python profiles/ab_window.py [label]

Full quadrotor + IMU, 65,536 envs, T=32, after 200 windows (steady-state
resets): per-launch fwd / bwd (CUDA events over graph replays) and the whole
window.  Run it for each build in one gpurun call, alternating."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_10247_b200 as qs  # noqa: E402
from paper_2509_10247_b200 import _lib as L  # noqa: E402
from paper_2509_10247_b200.window import BpttWindow  # noqa: E402


def timed(fn, n=50, graph=True):
    run = fn
    if graph:
        g = torch.cuda.CUDAGraph()
        fn()
        with torch.cuda.graph(g):
            fn()
        run = g.replay
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


env = qs.make_task(qs.TaskConfig(task="position", dynamics=os.environ.get("AB_MODEL", "full"), n_envs=65536,
                                 episode_len=128, imu=qs.ImuSpec(0.1, 0.01, 0.01, 0.001)), strict=False)
env.reset(seed=1)
win = BpttWindow(env, 32)
A = env.action_dim
win.actions.copy_(torch.randn(32, 65536, A, generator=torch.Generator().manual_seed(3)).cuda() * 0.3)
win.capture()
for _ in range(200):
    win.run()
lib = L.lib()
fwd = timed(lambda: L.check(lib.qs_task_window_fwd(env._cfg, env._scene.struct(), win._window_io(),
                                                   L.stream_handle()), "fwd"))
bwd = timed(lambda: L.check(lib.qs_task_window_bwd(env._cfg, env._scene.struct(), win._window_io(),
                                                   L.stream_handle()), "bwd"))
whole = timed(win.run, graph=False)
print(f"{sys.argv[1] if len(sys.argv) > 1 else L.LIB_PATH}: fwd {fwd:.1f} us  bwd {bwd:.1f} us  "
      f"window {whole:.1f} us", flush=True)
