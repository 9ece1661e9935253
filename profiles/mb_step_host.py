import time, torch, sys
sys.path.insert(0,'.')
import paper_2509_10247_b200 as qs
from paper_2509_10247_b200 import _lib as L
env = qs.make_task(qs.TaskConfig(task="position", dynamics="pm_continuous", n_envs=1024, episode_len=10**6), strict=False)
env.reset(seed=1)
a = torch.zeros(1024, 3, device="cuda")
def t(f, n=2000):
    for _ in range(50): f()
    torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/n*1e6
print("env.step", t(lambda: env.step(a)))
E=env._empty
bufs=[env._goal, env._peff, E, env._meta, env._ep_ret, E, env._stats, env._err]
sc=env._scene.tensors()
ops=L.ops()
print("op call", t(lambda: ops.task_step(env._cfg_blob, sc, env._S, a, bufs, None, False, False, env._cfg.proprio_dim)))
op=ops.task_step.default
fast=L.fast_ops().task_step
print("fast pybind call", t(lambda: fast(env._cfg_blob, sc, env._S, a, bufs, None, False, False, env._cfg.proprio_dim)))
print("op overload call", t(lambda: op(env._cfg_blob, sc, env._S, a, bufs, None, False, False, env._cfg.proprio_dim)))
with torch.no_grad():
    print("op call no_grad", t(lambda: op(env._cfg_blob, sc, env._S, a, bufs, None, False, False, env._cfg.proprio_dim)))
# raw ctypes launch with a prebuilt io
io = env._new_io()
outs = op(env._cfg_blob, sc, env._S, a, bufs, None, False, False, env._cfg.proprio_dim)
io.S_in, io.S_out, io.raw = L.ptr(env._S), L.ptr(outs[0]), L.ptr(a)
io.goal_in, io.goal_out, io.peff_in, io.peff_out = L.ptr(env._goal), L.ptr(outs[8]), L.ptr(env._peff), L.ptr(outs[9])
io.obs, io.r_ctrl, io.r_goal, io.r_rl = L.ptr(outs[1]), L.ptr(outs[2]), L.ptr(outs[3]), L.ptr(outs[4])
io.terminated, io.truncated, io.flags = L.ptr(outs[5]), L.ptr(outs[6]), L.ptr(outs[7])
st = env._scene.struct(); lib=L.lib(); h=L.stream_handle()
print("ctypes launch only", t(lambda: lib.qs_task_step_fwd(env._cfg, st, io, h)))
print("13 torch.empty", t(lambda: [torch.empty(1024, device='cuda') for _ in range(13)]))
print("torch.add", t(lambda: torch.add(a, a)))
