"""ctypes binding of the C ABI in ``include/quadsim_b200.h``.

There is no fallback: if ``libquadsim_b200.so`` is missing or CUDA is not
available the calls raise.  Structures mirror the header field for field.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# QS_LIB_PATH: load another build of the same library (A/B measurements)
LIB_PATH = os.environ.get("QS_LIB_PATH") or os.path.join(_PKG, "libquadsim_b200.so")

QS_OK = 0
QS_ERR_NONFINITE_ACTION = 1
QS_ERR_NONFINITE_STATE = 2
QS_ERR_GENERATION = 3
QS_ERR_BAD_ARGUMENT = 4
QS_ERR_LAUNCH = 5

MODEL_IDS = {"full": 0, "pm_continuous": 1, "pm_discrete": 2, "simplified": 3}
TASK_IDS = {"position": 0, "avoidance": 1, "racing": 2}
MAX_AGENTS = 8
MAX_GATES = 16

f32, i32, i64, u64, vp = C.c_float, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p


class QsWeights(C.Structure):
    _fields_ = [(n, f32) for n in (
        "w_p", "w_v", "w_a", "w_s", "w_t", "w_o", "w_f", "w_g", "near_radius", "near_width",
        "track_gain", "v_max", "sdf_sharpness", "gate_pass_bonus", "gate_crash_penalty", "goal_bonus")]


class QsTaskCfg(C.Structure):
    _fields_ = [
        ("model", i32), ("task", i32), ("n_envs", i32), ("n_agents", i32),
        ("episode_len", i32), ("action_dim", i32), ("proprio_dim", i32), ("n_gates", i32),
        ("env_offset", i64), ("seed", u64),
        ("dt", f32), ("success_radius", f32), ("hover_speed", f32), ("collision_radius", f32),
        ("d_min", f32), ("d_safe", f32), ("yaw_ema_alpha", f32), ("obs_clip", f32), ("goal_dist", f32),
        ("g", f32 * 3), ("drag_diag", f32 * 3), ("rate_gains", f32 * 3),
        ("drag_coeff", f32), ("lag_decay", f32),
        ("act_lo", f32 * 4), ("act_hi", f32 * 4),
        ("formation", (f32 * 3) * MAX_AGENTS), ("form_ref", (f32 * MAX_AGENTS) * MAX_AGENTS),
        ("w", QsWeights), ("w_rl", QsWeights),
        ("dr_enabled", i32), ("dr_per_episode", i32),
        ("dr_drag", f32 * 2), ("dr_latency", f32 * 2), ("dr_scale", f32 * 2),
        ("imu_enabled", i32), ("imu_accel_std", f32), ("imu_gyro_std", f32), ("imu_accel_rw", f32),
        ("imu_gyro_rw", f32),
        ("reset_mode", i32), ("want_cam", i32),
        ("act_center", f32 * 4), ("act_half", f32 * 4), ("imu_sqrt_dt", f32),
        ("rng_round_keys", C.c_uint32 * 20), ("guard", i32),
    ]


class QsScene(C.Structure):
    _fields_ = [("bounds", vp), ("spawn_goal", vp), ("spheres", vp), ("boxes", vp),
                ("cylinders", vp), ("counts", vp), ("ground_z", vp), ("gates", vp),
                ("Sm", i32), ("Bm", i32), ("Cm", i32)]


class QsStepIo(C.Structure):
    _fields_ = [(n, vp) for n in (
        "S_in", "S_out", "raw", "goal_in", "goal_out", "peff_in", "peff_out", "dr_in", "dr_out",
        "meta", "ep_return", "imu_bias", "imu_noise", "imu_out", "obs", "r_ctrl", "r_goal", "r_rl",
        "terminated", "truncated", "flags", "cam", "stats", "err")]


class QsStepGrad(C.Structure):
    _fields_ = [(n, vp) for n in (
        "S_in", "raw", "goal_in", "peff_in", "dr_in", "flags", "g_S_out", "g_obs", "g_rctrl",
        "g_S_in", "g_raw")]


class QsWindowIo(C.Structure):
    _fields_ = [("T", i32)] + [(n, vp) for n in (
        "S", "goal", "peff", "dr", "actions", "meta", "ep_return", "imu_bias", "imu_noise", "imu_out",
        "obs", "r", "terminated", "truncated", "flags", "stats", "err", "g_rctrl")] + [
        ("g_rctrl_scale", f32), ("gamma", f32)] + [(n, vp) for n in ("g_S_final", "g_actions", "g_S0", "loss")] + [
        ("carry", i32)]


class QsResetTable(C.Structure):
    _fields_ = [(n, vp) for n in ("env_mask", "p", "v", "goal", "v_ema", "dr", "next_gate")]


class QsRayCfg(C.Structure):
    _fields_ = [("kind", i32), ("n_rays", i32), ("cull", i32), ("max_range", f32), ("tan_h", f32),
                ("tan_v", f32), ("offset", f32 * 3), ("n_agents", i32)]


class QsGenCfg(C.Structure):
    _fields_ = [("spawn", f32 * 3), ("goal", f32 * 3), ("density", f32), ("r_quad", f32),
                ("clearance", f32), ("corridor_halfwidth", f32), ("indoor", i32),
                ("max_attempts", i32), ("Sm", i32), ("Bm", i32), ("Cm", i32), ("seed", u64),
                ("env_offset", i64), ("env_mask", vp), ("episode", vp), ("episode_stride", i32)]


class QsTrackCfg(C.Structure):
    _fields_ = [("n_gates", i32), ("spread", f32), ("seed", u64), ("env_offset", i64), ("env_mask", vp),
                ("episode", vp), ("episode_stride", i32)]


P = C.POINTER
_SIGS = {
    "qs_abi_version": ([], i32),
    "qs_proprio_dim": ([i32, i32], i32),
    "qs_state_planes": ([i32], i32),
    "qs_task_step_fwd": ([P(QsTaskCfg), P(QsScene), P(QsStepIo), vp], i32),
    "qs_task_validate": ([P(QsTaskCfg), P(QsStepIo), vp], i32),
    "qs_task_step_bwd": ([P(QsTaskCfg), P(QsScene), P(QsStepGrad), vp], i32),
    "qs_task_spawn": ([P(QsTaskCfg), P(QsScene), P(QsStepIo), vp, P(QsResetTable), vp], i32),
    "qs_task_observe": ([P(QsTaskCfg), P(QsScene), P(QsStepIo), vp], i32),
    "qs_task_window_fwd": ([P(QsTaskCfg), P(QsScene), P(QsWindowIo), vp], i32),
    "qs_task_window_bwd": ([P(QsTaskCfg), P(QsScene), P(QsWindowIo), vp], i32),
    "qs_task_privileged": ([P(QsTaskCfg), P(QsScene), P(QsStepIo), vp, vp], i32),
    "qs_mlp3_fit_grad": ([i64, i32] + [vp] * 16 + [i32, vp], i32),
    "qs_mlp3_fit_grad_tc": ([i64, i32] + [vp] * 17 + [i64, i32, vp], i32),
    "qs_mlp3_work_floats": ([i32], i64),
    "qs_td_lambda": ([i32, i64] + [vp] * 4 + [f32, f32, f32, vp, vp], i32),
    "qs_mlp3_forward_tc": ([i64, i32] + [vp] * 9 + [i32, vp], i32),
    "qs_policy_trunk_fwd": ([i64, i32] + [vp] * 10 + [i32, vp], i32),
    "qs_policy_trunk_bwd": ([i64, i32, vp, vp, vp, i32] + [vp] * 17 + [i64, i32, vp], i32),
    "qs_policy_gru_fwd": ([i64, i32, i32] + [vp] * 19 + [i32, i32, vp], i32),
    "qs_policy_gru_bwd": ([i64, i32] + [vp] * 18 + [i64, i32, vp], i32),
    "qs_policy_pack_image": ([i32, i32] + [vp] * 6 + [i32, vp, vp], i32),
    "qs_policy_image_bytes": ([], i64),
    "qs_policy_work_floats": ([i32, i32], i64),
    "qs_raycast": ([P(QsRayCfg), P(QsScene), i32, vp, i32, vp, vp, vp, vp, vp, vp, vp], i32),
    "qs_raycast_vjp": ([i32, i32, vp, vp, vp, i32, vp], i32),
    "qs_raycast_tiled": ([P(QsRayCfg), P(QsScene), i32, vp, i32, vp, vp, vp, i32, i32, vp, vp, vp], i32),
    "qs_raycast_tiled_vjp": ([P(QsRayCfg), P(QsScene), i32, vp, i32, vp, vp, vp, i32, i32, vp, vp, i32, vp], i32),
    "qs_sdf": ([P(QsScene), i32, i32, vp, vp, vp, vp], i32),
    "qs_imu_read": ([i32, vp, vp, vp, vp, f32, f32, f32, f32, f32, u64, i64, vp, vp, vp, vp], i32),
    "qs_dyn_step_fwd": ([i32, i32, vp, vp, vp, P(QsTaskCfg), vp, vp, vp], i32),
    "qs_dyn_step_bwd": ([i32, i32, vp, vp, vp, P(QsTaskCfg), vp, vp, vp, vp], i32),
    "qs_reconstruct_attitude": ([i32, vp, vp, vp, vp], i32),
    "qs_philox4x32_10": ([i32, vp, vp, vp], i32),
    "qs_philox4x32_7": ([i32, vp, vp, vp], i32),
    "qs_probe_fp32": ([i32, i32, i32, vp, vp], i32),
    "qs_probe_umma": ([i32, vp, vp, vp, vp], i32),
    "qs_gen_obstacle_course": ([P(QsGenCfg), i32, vp, vp, vp, vp, vp, vp, vp, vp, vp], i32),
    "qs_gen_race_track": ([P(QsTrackCfg), i32, vp, vp, vp, vp, vp, vp], i32),
}

_lib = None
_ops = None
OPS_PATH = os.path.join(_PKG, "_qs_torch_ops.so")


class QuadsimLibraryError(RuntimeError):
    pass


def ops():
    """``torch.ops.quadsim``: the torch custom-op layer over the C ABI
    (``csrc/qs_torch_ops.cpp``; raises when it is missing: no fallback)."""
    global _ops
    if _ops is None:
        lib()
        if not os.path.exists(OPS_PATH):
            raise QuadsimLibraryError(
                f"{OPS_PATH} is missing; build it with `python -m paper_2509_10247_b200.build`")
        torch.ops.load_library(OPS_PATH)
        _register_fakes()
        _ops = torch.ops.quadsim
    return _ops


def _register_fakes():
    """Shape (fake) implementation of quadsim::task_step for FakeTensor /
    torch.compile tracing: the outputs' shapes follow from S_in, the
    action-free flags and proprio_dim (the cfg bytes stay on the host)."""

    @torch.library.register_fake("quadsim::task_step")
    def _task_step_fake(cfg, scene, S_in, raw, bufs, imu_noise, want_cam, strict, proprio_dim):
        N = S_in.shape[1]
        f = dict(dtype=torch.float32, device=S_in.device)
        has_dr, has_imu = bufs[2].numel() > 0, bufs[5].numel() > 0
        return [torch.empty_like(S_in), S_in.new_empty((N, proprio_dim)), S_in.new_empty(N), S_in.new_empty(N),
                S_in.new_empty(N), torch.empty(N, dtype=torch.int8, device=S_in.device),
                torch.empty(N, dtype=torch.bool, device=S_in.device),
                torch.empty(N, dtype=torch.int32, device=S_in.device), torch.empty(N, 4, **f),
                torch.empty(N, 4, **f), torch.empty(N if has_dr else 0, 4, **f),
                torch.empty(N if want_cam else 0, 2, **f), torch.empty(N if has_imu else 0, 6, **f)]


_fast = None


def fast_ops():
    """The op library's direct Python entry points (same kernels and C++
    autograd node as torch.ops.quadsim, without the generic boxing)."""
    global _fast
    if _fast is None:
        ops()
        import importlib

        _fast = importlib.import_module("paper_2509_10247_b200._qs_torch_ops")
    return _fast


def lib():
    """The loaded CUDA library (raises when it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise QuadsimLibraryError(
                f"{LIB_PATH} is missing; build it with `python -m paper_2509_10247_b200.build`")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(device=None):
    """The raw cudaStream_t of the current stream on ``device`` (fast path: no
    Stream object is built on every kernel launch).  Kernels launch on the
    calling thread's current device, so a call for another device makes that
    device current first (FlightTask(device="cuda:1") without set_device)."""
    cur = torch.cuda.current_device()
    if device is None:
        idx = cur
    elif isinstance(device, int):
        idx = device
    else:
        idx = device.index if isinstance(device, torch.device) and device.index is not None else cur
    if idx != cur:
        torch.cuda.set_device(idx)
    return torch._C._cuda_getCurrentRawStream(idx)


def check(status: int, what: str):
    if status != QS_OK:
        raise QuadsimLibraryError(f"{what} failed with status {status}")


def tensor_device(x):
    """The device of a torch tensor, None otherwise (numpy >= 2 arrays carry a
    ``.device`` of their own, "cpu", which must not pick the device)."""
    return x.device if isinstance(x, torch.Tensor) else None


def require_cuda(device) -> torch.device:
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device()) \
        if torch.cuda.is_available() else None
    if dev is None or dev.type != "cuda" or not torch.cuda.is_available():
        raise QuadsimLibraryError("quadsim_b200 runs only on a CUDA device (B200, sm_100a); "
                                  "no CPU fallback exists")
    return dev
