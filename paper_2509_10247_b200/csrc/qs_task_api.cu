// C ABI for the fused task step (include/quadsim_b200.h).
#include <climits>

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
// q/tasks.py:551-558 then q/dynamics.py:130-133: key = code << 27 | row, so
// atomicMin picks the lowest action row, else the lowest state row
template <int M>
__global__ void __launch_bounds__(256) k_task_validate(const qs_task_cfg cfg, const qs_step_io io) {
  constexpr int A = ModelTraits<M>::A;
  const long N = (long)cfg.n_envs * cfg.n_agents;
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  int key = INT_MAX;
  if (row < N) {
    bool act_ok = true;
#pragma unroll
    for (int k = 0; k < A; ++k) act_ok = act_ok && isfinite(__ldg(io.raw + row * A + k));
    const State s = load_state<M>(io.S_in, N, row);
    if (!act_ok)
      key = (QS_ERR_NONFINITE_ACTION << 27) | (int)row;
    else if (!state_finite<M>(s))
      key = (QS_ERR_NONFINITE_STATE << 27) | (int)row;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
  if ((threadIdx.x & 31) == 0 && key != INT_MAX) atomicMin(io.err + 2, key);
}

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

int qs_task_validate(const qs_task_cfg* cfg, const qs_step_io* io, void* stream) {
  if (!cfg || !io || !io->raw || !io->S_in || !io->err) return QS_ERR_BAD_ARGUMENT;
  const long N = (long)cfg->n_envs * cfg->n_agents;
  if (N <= 0) return QS_OK;
  if (N >= (1L << 27)) return QS_ERR_BAD_ARGUMENT;
  const int grid = (int)((N + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  switch (cfg->model) {
    case QS_MODEL_FULL: k_task_validate<QS_MODEL_FULL><<<grid, 256, 0, s>>>(*cfg, *io); break;
    case QS_MODEL_PM_CONTINUOUS: k_task_validate<QS_MODEL_PM_CONTINUOUS><<<grid, 256, 0, s>>>(*cfg, *io); break;
    case QS_MODEL_PM_DISCRETE: k_task_validate<QS_MODEL_PM_DISCRETE><<<grid, 256, 0, s>>>(*cfg, *io); break;
    case QS_MODEL_SIMPLIFIED: k_task_validate<QS_MODEL_SIMPLIFIED><<<grid, 256, 0, s>>>(*cfg, *io); break;
    default: return QS_ERR_BAD_ARGUMENT;
  }
  return cudaGetLastError() == cudaSuccess ? QS_OK : QS_ERR_LAUNCH;
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
