// Racing task instantiations (q/tasks.py:847-972); single agent only (:859-860).
#include "qs_task_impl.cuh"
namespace qs {
QS_DEFINE_TASK_DISPATCH(QS_TASK_RACING, false)
}
