// Position task instantiations (q/tasks.py:658-763).
#include "qs_task_impl.cuh"
namespace qs {
QS_DEFINE_TASK_DISPATCH(QS_TASK_POSITION, true)
}
