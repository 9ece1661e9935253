"""B200-native quadsim: the DiffAero data-parallel simulation core on sm_100a.

Python API mirroring the reference package ``quadsim`` (``q/`` =
``/root/reference/pkg/src/quadsim``) for the hot path: dynamics models and
rollouts, ray-cast sensing, IMU, resets and the three flight tasks.  All
batched math runs in hand-written CUDA kernels (``libquadsim_b200.so``,
C ABI in ``include/quadsim_b200.h``); there is no CPU fallback.
"""

from paper_2509_10247_b200 import _lib  # noqa: F401
from paper_2509_10247_b200 import dynamics, sensors, tasks, world  # noqa: F401
from paper_2509_10247_b200.dynamics import QuadParams, QuadState, make_model, rollout_grad  # noqa: F401
from paper_2509_10247_b200.tasks import (StepOutput, TaskConfig, TaskContractError, make_task,  # noqa: F401
                                         ImuSpec)

__all__ = ["dynamics", "sensors", "tasks", "world", "make_model", "make_task", "TaskConfig",
           "QuadParams", "QuadState", "StepOutput", "TaskContractError", "rollout_grad", "ImuSpec"]
