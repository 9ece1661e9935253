// C ABI for the fused task step (include/quadsim_b200.h).
#include "qs_dynamics.cuh"

namespace qs {
template <int T, int NA>
int task_dispatch_na(int op, const qs_task_cfg* cfg, const qs_scene* sc, const void* p,
                     const uint8_t* mask, const qs_reset_table* tab, cudaStream_t s);

template <int T>
int task_dispatch(int op, const qs_task_cfg* cfg, const qs_scene* sc, const void* p,
                  const uint8_t* mask, const qs_reset_table* tab, cudaStream_t s) {
  if (cfg->n_agents > 1) {
    if (T == QS_TASK_RACING) return QS_ERR_BAD_ARGUMENT;  // racing is single-agent (q/tasks.py:859)
    return task_dispatch_na<T == QS_TASK_RACING ? QS_TASK_POSITION : T, QS_MAX_AGENTS>(op, cfg, sc, p, mask,
                                                                                       tab, s);
  }
  return task_dispatch_na<T, 1>(op, cfg, sc, p, mask, tab, s);
}
}

namespace {
int task_call(int op, const qs_task_cfg* cfg, const qs_scene* sc, const void* p,
              const uint8_t* mask, const qs_reset_table* tab, void* stream) {
  if (!cfg || !sc || !p) return QS_ERR_BAD_ARGUMENT;
  if (cfg->n_agents < 1 || cfg->n_agents > QS_MAX_AGENTS) return QS_ERR_BAD_ARGUMENT;
  if (cfg->n_envs <= 0) return QS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  qs_task_cfg c = *cfg;  // private copy carrying the derived Philox round keys
  philox_round_keys(c.seed, c.rng_round_keys);
  cfg = &c;
  switch (cfg->task) {
    case QS_TASK_POSITION: return qs::task_dispatch<QS_TASK_POSITION>(op, cfg, sc, p, mask, tab, s);
    case QS_TASK_AVOIDANCE: return qs::task_dispatch<QS_TASK_AVOIDANCE>(op, cfg, sc, p, mask, tab, s);
    case QS_TASK_RACING: return qs::task_dispatch<QS_TASK_RACING>(op, cfg, sc, p, mask, tab, s);
  }
  return QS_ERR_BAD_ARGUMENT;
}
}  // namespace

extern "C" {

int qs_abi_version(void) { return QS_ABI_VERSION; }

int qs_proprio_dim(int32_t model, int32_t task) {
  int base = model == QS_MODEL_FULL ? 12 : 9;
  return base + (task == QS_TASK_RACING ? 9 : 0);
}

int qs_state_planes(int32_t model) {
  return model == QS_MODEL_FULL ? 4 : (model == QS_MODEL_SIMPLIFIED ? 5 : 3);
}

int qs_task_step_fwd(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_io* io,
                     void* stream) {
  return task_call(0, cfg, scene, io, nullptr, nullptr, stream);
}

int qs_task_step_bwd(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_grad* g,
                     void* stream) {
  return task_call(1, cfg, scene, g, nullptr, nullptr, stream);
}

int qs_task_spawn(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_io* io,
                  const uint8_t* env_mask, const qs_reset_table* table, void* stream) {
  return task_call(2, cfg, scene, io, env_mask, table, stream);
}

int qs_task_observe(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_io* io,
                    void* stream) {
  return task_call(3, cfg, scene, io, nullptr, nullptr, stream);
}

int qs_task_privileged(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_io* io, float* out,
                       void* stream) {
  if (!io || !out) return QS_ERR_BAD_ARGUMENT;
  qs_step_io o = *io;
  o.obs = out;
  return task_call(7, cfg, scene, &o, nullptr, nullptr, stream);
}

int qs_task_window_fwd(const qs_task_cfg* cfg, const qs_scene* scene, const qs_window_io* w,
                       void* stream) {
  if (cfg && cfg->reset_mode != 0) return QS_ERR_BAD_ARGUMENT;  // windows reset in-kernel
  return task_call(4, cfg, scene, w, nullptr, nullptr, stream);
}

int qs_task_window_bwd(const qs_task_cfg* cfg, const qs_scene* scene, const qs_window_io* w,
                       void* stream) {
  return task_call(5, cfg, scene, w, nullptr, nullptr, stream);
}

}  // extern "C"
