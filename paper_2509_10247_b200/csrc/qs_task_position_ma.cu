// Position task, multi-agent formation (q/tasks.py:173-192, 723-742) instantiations.
#include "qs_task_impl.cuh"
namespace qs {
QS_DEFINE_TASK_DISPATCH(QS_TASK_POSITION, QS_MAX_AGENTS)
}
