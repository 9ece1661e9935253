// Avoidance task, multi-agent (q/tasks.py:817-844) instantiations.
#include "qs_task_impl.cuh"
namespace qs {
QS_DEFINE_TASK_DISPATCH(QS_TASK_AVOIDANCE, QS_MAX_AGENTS)
}
