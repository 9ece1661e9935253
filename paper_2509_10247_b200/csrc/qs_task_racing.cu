// Racing task, single agent only (q/tasks.py:847-972, :859-860) instantiations.
#include "qs_task_impl.cuh"
namespace qs {
QS_DEFINE_TASK_DISPATCH(QS_TASK_RACING, 1)
}
