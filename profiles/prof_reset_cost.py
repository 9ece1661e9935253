import sys, torch, json
sys.path.insert(0,'/root/repo')
import paper_2509_10247_b200 as qs
from paper_2509_10247_b200.window import BpttWindow
from paper_2509_10247_b200 import _lib as L
import bench
for scale, elen in ((0.3, 128), (0.0, 10**6), (0.05, 10**6)):
    cfg = qs.TaskConfig(task="position", dynamics="full", n_envs=65536, episode_len=elen, imu=qs.ImuSpec(**bench.IMU))
    env = qs.make_task(cfg, device="cuda", strict=False); env.reset(seed=1)
    win = BpttWindow(env, 32)
    g = torch.Generator().manual_seed(1234)
    win.actions.copy_((torch.randn(32, 65536, 4, generator=g) * scale).cuda())
    win.capture()
    for _ in range(5): win.run()
    torch.cuda.synchronize()
    f0 = env.finished_episodes
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): win.run()
    e1.record(); torch.cuda.synchronize()
    print(scale, elen, 'ms/window', e0.elapsed_time(e1)/20, 'resets/window', (env.finished_episodes - f0)/20)
