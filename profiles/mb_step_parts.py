"""Host cost of the pieces of one FlightTask.step at C1 (pm_continuous, 1,024 envs)."""
import time, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2509_10247_b200 as qs
from paper_2509_10247_b200 import tasks as T
env = qs.make_task(qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=1024, episode_len=10**6), strict=False)
env.reset(seed=1)
a = torch.zeros(1024, 3, device="cuda")
def t(f, n=3000):
    for _ in range(100): f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e6
print("env.step", t(lambda: env.step(a)))
E = env._empty
def bufs():
    return [env._goal, env._peff, env._dr if env._dr is not None else E, env._meta, env._ep_ret,
            env._imu_bias if env._imu_bias is not None else E, env._stats, env._err]
print("bufs list", t(bufs))
print("scene.tensors", t(lambda: env._scene.tensors()))
print("check_inputs", t(lambda: env._check_inputs(a)))
print("type checks", t(lambda: (type(a) is torch.Tensor and a.dtype is torch.float32 and a.device == env.device)))
b = bufs(); sc = env._scene.tensors()
print("op", t(lambda: env._ops.task_step(env._cfg_blob, sc, env._S, a, b, None, False, False, env._cfg.proprio_dim)))
out = env._ops.task_step(env._cfg_blob, sc, env._S, a, b, None, False, False, env._cfg.proprio_dim)
print("StepOutput", t(lambda: T.StepOutput(obs=T.Obs(proprio=out[1], visual=None, imu=None), r_ctrl=out[2], r_goal=out[3], r_rl=out[4], terminated=out[5], truncated=out[6])))
print("unpack 13", t(lambda: tuple(out)))
