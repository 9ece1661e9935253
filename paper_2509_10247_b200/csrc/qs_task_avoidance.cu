// Avoidance task, single agent (q/tasks.py:766-844) instantiations.
#include "qs_task_impl.cuh"
namespace qs {
QS_DEFINE_TASK_DISPATCH(QS_TASK_AVOIDANCE, 1)
}
