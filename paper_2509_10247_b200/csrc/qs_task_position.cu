// Position task, single agent (q/tasks.py:658-763) instantiations.
#include "qs_task_impl.cuh"
namespace qs {
QS_DEFINE_TASK_DISPATCH(QS_TASK_POSITION, 1)
}
