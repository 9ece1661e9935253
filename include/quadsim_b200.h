/*
 * quadsim_b200 — C ABI of the B200-native quadsim hot path.
 *
 * The reference (DiffAero re-implemented as the numpy package `quadsim`,
 * /root/reference/pkg/src/quadsim, cited below as q/) has NO native FFI: its
 * boundary is the Python env API.  Each entry point below replaces the
 * reference function named in its comment; the Python package
 * `paper_2509_10247_b200` binds them with ctypes.
 *
 * Rules shared by every entry point:
 *   - every pointer is a caller-owned, contiguous device buffer (fp32 unless
 *     stated), laid out as documented in DESIGN.md §3;
 *   - nothing allocates and nothing synchronises the host; work is enqueued
 *     on `stream` (a cudaStream_t passed as void*), so every call is
 *     CUDA-graph capturable;
 *   - the return value is a launch status (QS_OK or QS_ERR_*); data-dependent
 *     contract violations (non-finite action/state, failed reset sampling)
 *     are reported through the device error word `err` (int32[2] = {code,
 *     first offending row}, codes QS_ERR_*), read lazily by the host.
 */
#ifndef QUADSIM_B200_H
#define QUADSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QS_ABI_VERSION 1

/* status / device error codes (map to the reference's exceptions) */
#define QS_OK 0
#define QS_ERR_NONFINITE_ACTION 1 /* tk.TaskContractError  q/tasks.py:555-558 */
#define QS_ERR_NONFINITE_STATE 2  /* dyn.ContractError     q/dynamics.py:130-133 */
#define QS_ERR_GENERATION 3       /* wd.GenerationError    q/world.py:251,340,448 */
#define QS_ERR_BAD_ARGUMENT 4     /* shape / enum errors */
#define QS_ERR_LAUNCH 5           /* cudaGetLastError after launch */

/* dynamics models  (q/dynamics.py:34) */
#define QS_MODEL_FULL 0
#define QS_MODEL_PM_CONTINUOUS 1
#define QS_MODEL_PM_DISCRETE 2
#define QS_MODEL_SIMPLIFIED 3

/* tasks (q/tasks.py:30) */
#define QS_TASK_POSITION 0
#define QS_TASK_AVOIDANCE 1
#define QS_TASK_RACING 2

#define QS_MAX_AGENTS 8
#define QS_MAX_GATES 16

/* Reward weights, q/tasks.py:37-54 (RewardWeights). */
typedef struct qs_weights {
  float w_p, w_v, w_a, w_s, w_t, w_o, w_f, w_g;
  float near_radius, near_width, track_gain, v_max, sdf_sharpness;
  float gate_pass_bonus, gate_crash_penalty, goal_bonus;
} qs_weights;

/* Everything constant over a rollout: TaskConfig (q/tasks.py:67-106) +
 * QuadParams (q/dynamics.py:42-82) + RandomizationSpec (q/world.py:114-127)
 * + the IMU spec (q/sensors.py:508-530). */
typedef struct qs_task_cfg {
  int32_t model, task;
  int32_t n_envs;      /* local envs on this rank */
  int32_t n_agents;    /* rows per env; row = env * n_agents + agent */
  int32_t episode_len, action_dim, proprio_dim, n_gates;
  int64_t env_offset;  /* global id of local env 0 (sharding; RNG keys) */
  uint64_t seed;
  float dt, success_radius, hover_speed, collision_radius, d_min, d_safe;
  float yaw_ema_alpha, obs_clip, goal_dist;
  float g[3], drag_diag[3], rate_gains[3];
  float drag_coeff, lag_decay;          /* scalar params (no randomization) */
  float act_lo[4], act_hi[4];           /* model action box (q/dynamics.py:342-425) */
  float formation[QS_MAX_AGENTS][3];    /* template (q/world.py:386-406) */
  float form_ref[QS_MAX_AGENTS][QS_MAX_AGENTS]; /* |f_i - f_j| (q/tasks.py:188) */
  qs_weights w, w_rl;
  int32_t dr_enabled, dr_per_episode;
  float dr_drag[2], dr_latency[2], dr_scale[2];
  int32_t imu_enabled;
  float imu_accel_std, imu_gyro_std, imu_accel_rw, imu_gyro_rw;
  int32_t reset_mode;   /* 0: in-kernel Philox resets; 1: deferred (injected) */
  int32_t want_cam;     /* write camera yaw (cos,sin) per row for rendering */
  float act_center[4], act_half[4];  /* (lo+hi)/2, (hi-lo)/2 of act_lo/hi (host-computed) */
  float imu_sqrt_dt;                 /* sqrt(dt) */
  uint32_t rng_round_keys[20];       /* Philox round keys of `seed`: written by the library
                                        on its private copy, ignored on input */
  int32_t guard;  /* step forward: skip the whole launch when err[2] != INT32_MAX (set by
                     qs_task_validate), so a rejected step mutates nothing */
} qs_task_cfg;

/* Per-env scene data (read-only during a rollout).  Obstacles are packed
 * valid-first per env: counts[e] = {n_sph, n_box, n_cyl, has_ground}. */
typedef struct qs_scene {
  const float* bounds;      /* (E,2,4) scene bounds lo, hi (without the 1e-6 shrink) */
  const float* spawn_goal;  /* (E,2,4) scene.spawn, scene.goal */
  const float* spheres;     /* (E,Sm,4)  cx cy cz r */
  const float* boxes;       /* (E,Bm,8)  cx cy cz _ hx hy hz _ */
  const float* cylinders;   /* (E,Cm,8)  cx cy cz r hh _ _ _ */
  const int32_t* counts;    /* (E,4) */
  const float* ground_z;    /* (E,)  */
  const float* gates;       /* (E,G,8)  cx cy cz inner nx ny nz frame */
  int32_t Sm, Bm, Cm;
} qs_scene;

/* Mutable per-env / per-row buffers.  `*_in` are read, `*_out` written
 * (functional update: the *_in buffers are what the backward replays). */
typedef struct qs_step_io {
  /* differentiable state + v_ema in the pad lanes: (NP,N,4), NP = qs_state_planes(model):
     3 (pm), 4 (full), 5 (simplified) */
  const float* S_in;  float* S_out;
  const float* raw;                     /* (N,A) raw (pre-squash) action */
  const float* goal_in; float* goal_out;  /* (N,4) */
  const float* peff_in; float* peff_out;  /* (N,4) previous effort */
  const float* dr_in;   float* dr_out;    /* (N,4) drag, lag_decay, action scale, latency | NULL */
  int32_t* meta;        /* (E,4) steps_in_episode, episode index, tick, next_gate (in place) */
  float* ep_return;     /* (E,) (in place) */
  float* imu_bias;      /* (N,8) accel bias, gyro bias (in place) | NULL */
  const float* imu_noise; /* (4,N,3) injected normals (ba, bg, na, ng) | NULL = Philox */
  float* imu_out;       /* (N,6) accel xyz, gyro xyz | NULL */
  float* obs;           /* (N,P) proprio */
  float* r_ctrl; float* r_goal; float* r_rl;  /* (N,) */
  int8_t* terminated; uint8_t* truncated;     /* (N,) */
  int32_t* flags;       /* (N,) record for the backward: bit0 done, clamp masks, sdf argmin */
  float* cam;           /* (N,2) cos/sin of camera yaw | NULL */
  double* stats;        /* (4,) finished, successes, collisions, finished_return (atomic) */
  int32_t* err;         /* (2,) code, first row */
} qs_step_io;

typedef struct qs_step_grad {
  const float* S_in; const float* raw; const float* goal_in; const float* peff_in;
  const float* dr_in; const int32_t* flags;
  const float* g_S_out;   /* (NP,N,4) | NULL */
  const float* g_obs;     /* (N,P) | NULL */
  const float* g_rctrl;   /* (N,) | NULL */
  float* g_S_in;          /* (NP,N,4) */
  float* g_raw;           /* (N,A) */
} qs_step_grad;

/* Reset table for deferred/injected resets: rows of the done envs only need
 * valid data; layout (N,4) each.  dr may be NULL. */
typedef struct qs_reset_table {
  const uint8_t* env_mask;  /* (E,) 1 = respawn this env */
  const float* p; const float* v; const float* goal; const float* v_ema;
  const float* dr;          /* (N,4) drag, lag_decay, scale, latency | NULL */
  const int32_t* next_gate; /* (E,) | NULL */
} qs_reset_table;

/* A fused T-step window (open-loop actions, in-kernel resets): the env's
 * state stays in registers across the T steps.  Checkpoint slot 0 holds the
 * window's initial state; slot t+1 receives the state after step t (the
 * backward's checkpoints).  Per-step outputs are stacked on a leading T axis. */
typedef struct qs_window_io {
  int32_t T;
  float* S;          /* (T+1,NP,N,4) */
  float* goal;       /* (T+1,N,4) */
  float* peff;       /* (T+1,N,4) */
  float* dr;         /* (T+1,N,4) | NULL */
  const float* actions; /* (T,N,A) raw actions */
  int32_t* meta; float* ep_return; float* imu_bias;  /* in place, as qs_step_io */
  const float* imu_noise;  /* (T,4,N,3) | NULL */
  float* imu_out;    /* (T,N,6) | NULL */
  float* obs;        /* (T,N,P) | NULL (observation not materialised) */
  float* r;          /* (T,3,N) r_ctrl, r_goal, r_rl */
  int8_t* terminated; uint8_t* truncated; int32_t* flags;  /* (T,N) */
  double* stats; int32_t* err;
  /* backward: dL/dr_ctrl[t,row] = g_rctrl[t,row], or g_rctrl_scale * gamma^t when NULL */
  const float* g_rctrl; float g_rctrl_scale, gamma;
  const float* g_S_final;  /* (NP,N,4) | NULL */
  float* g_actions;        /* (T,N,A) */
  float* g_S0;             /* (NP,N,4) | NULL */
  /* fwd: loss += -(1/(T N)) sum_t gamma^t sum_rows r_ctrl[t]  (the BPTT loss,
   * q/learners.py:222,254); zeroed by qs_task_window_fwd.  NULL = skip */
  double* loss;
  /* bwd: after the reverse sweep copy checkpoint slot T into slot 0 (the next
   * window starts where this one ended) */
  int32_t carry;
} qs_window_io;

int qs_abi_version(void);
int qs_proprio_dim(int32_t model, int32_t task);
int qs_state_planes(int32_t model);

/* FlightTask.step (q/tasks.py:549-600): squash -> yaw frame -> dynamics ->
 * EMA -> rewards -> termination -> auto-reset -> observe, fused per env. */
int qs_task_step_fwd(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_io* io,
                     void* stream);
/* Contract check of FlightTask.step's inputs before anything is mutated
 * (q/tasks.py:551-558, q/dynamics.py:130-133): every row's raw action and
 * model state must be finite.  Writes atomicMin(err[2], code << 27 | row) --
 * the reference's precedence: the lowest non-finite action row
 * (QS_ERR_NONFINITE_ACTION), else the lowest non-finite state row
 * (QS_ERR_NONFINITE_STATE).  err must hold 3 ints, err[2] = INT32_MAX when
 * clean.  Paired with qs_task_cfg.guard = 1 on the step launched after it,
 * one host read of err[2] gives raise-before-mutate semantics. */
int qs_task_validate(const qs_task_cfg* cfg, const qs_step_io* io, void* stream);
/* Analytic VJP of qs_task_step_fwd (replaces the tape backward of the ops
 * recorded by FlightTask.step; subgradients per q/autodiff.py). */
int qs_task_step_bwd(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_grad* g,
                     void* stream);
/* privileged_state (q/tasks.py:500-545) of the state in io->S_out / io->goal_out:
 * out (N,14) = yaw-local goal offset, velocity, thrust; sdf clamped to +-5;
 * yaw-local clearance direction; goal distance (critic features). */
int qs_task_privileged(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_io* io, float* out,
                       void* stream);
/* collect_window + Tape.backward of the BPTT learner for open-loop actions
 * (q/learners.py:201-265): T fused steps forward / T analytic VJPs backward in
 * one launch each. */
int qs_task_window_fwd(const qs_task_cfg* cfg, const qs_scene* scene, const qs_window_io* w,
                       void* stream);
int qs_task_window_bwd(const qs_task_cfg* cfg, const qs_scene* scene, const qs_window_io* w,
                       void* stream);
/* _spawn_all (q/tasks.py:687-721, 789-815, 873-902) + _redraw_randomization
 * (:377-387) for masked envs, writing into io->S_out/goal_out/peff_out/dr_out
 * in place; table==NULL -> in-kernel Philox sampling. */
int qs_task_spawn(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_io* io,
                  const uint8_t* env_mask, const qs_reset_table* table, void* stream);
/* FlightTask.observe proprio (q/tasks.py:415-442, racing :904-915) of io->S_out. */
int qs_task_observe(const qs_task_cfg* cfg, const qs_scene* scene, const qs_step_io* io,
                    void* stream);

/* ---- sensing (q/sensors.py) ---- */
typedef struct qs_ray_cfg {
  int32_t kind;        /* 0 camera (frustum cull), 1 lidar (range-ball cull), 2 generic rays */
  int32_t n_rays;      /* rays per env */
  int32_t cull;         /* bit 0: conservative frustum / range cull (never changes an image);
                          bit 1 (qs_raycast_tiled): extended per-tile culling (exact box
                          azimuth intervals + vertical flags), for scenes with large boxes */
  float max_range;
  float tan_h, tan_v;  /* camera half-FOV tangents (cull planes) */
  float offset[3];     /* sensor offset in the body frame */
  int32_t n_agents;    /* rows per env (obstacles are per env) */
} qs_ray_cfg;

/* render_depth / render_lidar / raycast (q/sensors.py:245-269, 377-410):
 * rows (N), origin = pos + Rz(yaw) offset, dir = Rz(yaw) dirs_body[r]
 * (or dirs_world (N,R,4) for kind 2).  out (N,R) fp32 distances, hit (N,R)
 * u8 | NULL.  dT_dO (N,R,4) | NULL: analytic d t / d origin (opt-in depth VJP). */
int qs_raycast(const qs_ray_cfg* cfg, const qs_scene* scene, int32_t n_rows, const float* pos,
               int32_t pos_stride, const float* cam_cs, const float* dirs_body,
               const float* dirs_world, float* out, uint8_t* hit, float* dT_dO, void* stream);
/* Same images as qs_raycast (kinds 0/1) with per-warp culling: rays are
 * grouped into n_tiles tiles of tile_width = 32, 64 or 128 rays; tile_dirs
 * (n_tiles,tile_width,4) = body-frame unit direction xyz + ray index (as a
 * float; < 0 = empty slot), lane j of the tile's warp casting slots j, j+32,
 * ...  Each tile has a body-frame bounding cone and azimuth sector,
 * tile_cones (n_tiles,12) = unit axis xyz, cos(half-angle), sin(half-angle),
 * unit horizontal sector centre xy, cos(sector half-width) (< -1.5: no sector
 * test), sin(sector half-width), min and max direction z, 1 pad. */
int qs_raycast_tiled(const qs_ray_cfg* cfg, const qs_scene* scene, int32_t n_rows, const float* pos,
                     int32_t pos_stride, const float* cam_cs, const float* tile_dirs,
                     const float* tile_cones, int32_t n_tiles, int32_t tile_width, float* out,
                     uint8_t* hit, void* stream);
/* The depth VJP without dT_dO in memory: recasts the tiled rays, finds each
 * ray's hit surface and accumulates g_pos[row] += sum_r g_depth[row,r] *
 * (-n/(n.d)) (rays clamped at max_range contribute 0), one atomic per row.
 * Same tile tables and conventions as qs_raycast_tiled. */
int qs_raycast_tiled_vjp(const qs_ray_cfg* cfg, const qs_scene* scene, int32_t n_rows, const float* pos,
                         int32_t pos_stride, const float* cam_cs, const float* tile_dirs,
                         const float* tile_cones, int32_t n_tiles, int32_t tile_width, const float* g_depth,
                         float* g_pos, int32_t gpos_stride, void* stream);
/* d loss / d pos = sum_r g_depth[r] * dT_dO[r]  (N,3) accumulate into g_pos (N,4 stride pos_stride). */
int qs_raycast_vjp(int32_t n_rows, int32_t n_rays, const float* g_depth, const float* dT_dO,
                   float* g_pos, int32_t pos_stride, void* stream);

/* Learner side (config C5): one full-batch gradient of the privileged-state
 * value MLP pred = tanh(tanh((x*scale) W0 + b0) W1 + b1) w2 + b2 with hidden
 * width 128 (q/nets.py:259-274) for L = mean((pred - y)^2) (q/learners.py:
 * 232-245), forward and backward fused on the tensor cores (bf16 operands,
 * fp32 accumulation).  x (m,k) fp32 rows (k <= 16), y (m,); W0 (k,128), W1
 * (128,128), w2 (128,) fp32.  The gradients (caller-zeroed, same shapes) and
 * loss are ACCUMULATED.  n_sm: persistent CTAs (the SM count). */
int qs_mlp3_fit_grad(int64_t m, int32_t k, const float* x, const float* scale, const float* y, const float* W0,
                     const float* b0, const float* W1, const float* b1, const float* w2, const float* b2,
                     float* gW0, float* gb0, float* gW1, float* gb1, float* gw2, float* gb2, float* loss,
                     int32_t n_sm, void* stream);
/* The same fit step on the 5th-generation tensor cores (tcgen05.mma, TMEM
 * accumulators, one persistent 512-thread CTA per SM): k <= 14 (the two spare
 * input columns carry the bias gradients through the MMAs).  `work` holds
 * qs_mlp3_work_floats(n_sm) floats of scratch: each CTA writes its partial
 * gradients there and a second kernel sums them in CTA order, so the
 * gradients and the loss are bitwise reproducible (no float atomics). */
int qs_mlp3_fit_grad_tc(int64_t m, int32_t k, const float* x, const float* scale, const float* y, const float* W0,
                        const float* b0, const float* W1, const float* b1, const float* w2, const float* b2,
                        float* gW0, float* gb0, float* gW1, float* gb1, float* gw2, float* gb2, float* loss,
                        float* work, int64_t work_floats, int32_t n_sm, void* stream);
int64_t qs_mlp3_work_floats(int32_t n_sm);
/* TD(lambda) targets over a (T, n) window with termination cuts (q/learners.py:78-94):
 * r, values, done (uint8) are (T, n) row-major, bootstrap (n,); targets (T, n).
 * one_minus_lam: 1 - lam as the caller rounds it (torch: from double). */
int qs_td_lambda(int32_t T, int64_t n, const float* r, const float* values, const float* bootstrap,
                 const uint8_t* done, float gamma, float lam, float one_minus_lam, float* targets, void* stream);
/* The value MLP's forward only (the TD-lambda targets' values and bootstrap,
 * q/learners.py:286-292) on the same tcgen05 path: pred (m,) fp32, k <= 14. */
int qs_mlp3_forward_tc(int64_t m, int32_t k, const float* x, const float* scale, const float* W0, const float* b0,
                       const float* W1, const float* b1, const float* w2, const float* b2, float* pred,
                       int32_t n_sm, void* stream);

/* The policy's MLP trunk + Gaussian heads (q/nets.py:198-256; PolicyArch with
 * hidden 64, mlp (128, 128)) on tcgen05: y = tanh(tanh(tanh(h W0 + b0) W1 + b1)
 * W2 + b2) Wh + bh for h (n, 64) fp32; W0 (64,128), W1, W2 (128,128), Wh
 * (128, n_out) row-major fp32, n_out <= 8 (mu | log sigma). */
int qs_policy_trunk_fwd(int64_t n, int32_t n_out, const float* h, const float* W0, const float* b0, const float* W1,
                        const float* b1, const float* W2, const float* b2, const float* Wh, const float* bh, float* y,
                        int32_t n_sm, void* stream);
/* The bf16 weight image the kernels below can stage with bulk copies instead
 * of converting the fp32 weights in every CTA: W0 | W1 | W2 | Wh | Wi | Wh_g in
 * the kernels' blocked operand layout, qs_policy_image_bytes() bytes, 16-byte
 * aligned.  Build it once per set of weights (e.g. per rollout). */
int64_t qs_policy_image_bytes(void);
int qs_policy_pack_image(int32_t n_in, int32_t n_out, const float* Wi, const float* Wh_g, const float* W0,
                         const float* W1, const float* W2, const float* Wh, int32_t wh_planar, void* w_image,
                         void* stream);
/* Its backward: given dL/dy (n, n_out), recomputes the forward per tile,
 * writes dL/dh (n, 64) and every weight / bias gradient (same shapes as the
 * parameters; overwritten, not accumulated).  w_image: NULL, or the image of
 * the same weights.  Planar mode (dy_planar != 0): dy is (2, n, n_out / 2) --
 * the mu block, then the log-sigma block -- and the heads Wh / gWh are
 * (2, 128, n_out / 2) likewise ([W_mu | W_sigma] as two blocks). */
int qs_policy_trunk_bwd(int64_t n, int32_t n_out, const void* w_image, const float* h, const float* dy,
                        int32_t dy_planar, const float* W0, const float* b0,
                        const float* W1, const float* b1, const float* W2, const float* b2, const float* Wh,
                        float* dh, float* gW0, float* gb0, float* gW1, float* gb1, float* gW2, float* gb2,
                        float* gWh, float* gbh, float* work, int64_t work_floats, int32_t n_sm, void* stream);
/* The GRU cell (q/nets.py:107-132; Wi (n_in, 192), Wh_g (64, 192), gates
 * r|z|n) fused in front of the trunk: h_out (n, 64) = GRU(x' , h'),
 * y = trunk + heads of h_out, where x' = x (n, n_in) times the per-feature
 * x_scale (the policy's input scale, q/nets.py:241; NULL = 1) and h' = h with
 * the rows h_reset[i] != 0 zeroed (the trainer's episode-reset mask; may be
 * NULL).  y: (n, n_out), or with y_planar != 0 (2, n, n_out / 2) -- mu block,
 * then log-sigma block, and Wh is (2, 128, n_out / 2) likewise.  n_in <= 16. */
int qs_policy_gru_fwd(int64_t n, int32_t n_in, int32_t n_out, const void* w_image, const float* x,
                      const float* x_scale, const float* h, const uint8_t* h_reset,
                      const float* Wi, const float* bi, const float* Wh_g, const float* bh_g, const float* W0,
                      const float* b0, const float* W1, const float* b1, const float* W2, const float* b2,
                      const float* Wh, const float* bh, float* h_out, float* y, int32_t y_planar, int32_t n_sm,
                      void* stream);
/* The GRU cell's backward for dL/dh_out = dh_out_a + dh_out_b (b may be
 * NULL): writes dx (n, n_in; dL/dx through x_scale), dh (n, 64; 0 on h_reset
 * rows) and gWi, gbi, gWh_g, gbh_g (overwritten). */
int qs_policy_gru_bwd(int64_t n, int32_t n_in, const void* w_image, const float* x, const float* x_scale,
                      const float* h, const uint8_t* h_reset,
                      const float* dh_out_a, const float* dh_out_b, const float* Wi, const float* bi,
                      const float* Wh_g, const float* bh_g, float* dx, float* dh, float* gWi, float* gbi,
                      float* gWh_g, float* gbh_g, float* work, int64_t work_floats, int32_t n_sm, void* stream);
/* Scratch the gradient kernels above need (floats): which 0 = trunk backward,
 * 1 = GRU backward; each CTA writes its partial gradients there and a second
 * kernel sums them in CTA order, so the gradients are bitwise reproducible
 * (no float atomics).  -1 for a bad argument. */
int64_t qs_policy_work_floats(int32_t which, int32_t n_sm);

/* sdf_np / sdf_var (q/sensors.py:417-501): points (N,4); out (N,); grad (N,4) | NULL */
int qs_sdf(const qs_scene* scene, int32_t n_rows, int32_t n_agents, const float* pts, float* out,
           float* grad, void* stream);

/* ImuModel.read (q/sensors.py:540-555), batch rows: R (N,9) row-major body->world,
 * w (N,4) | NULL, vdot (N,4).  noise (4,N,3) injected | NULL (Philox keyed by
 * seed,row,tick).  bias (N,8) in place; out (N,6). */
int qs_imu_read(int32_t n_rows, const float* R, const float* w, const float* vdot, const float* g,
                float dt, float sa, float sg, float ra, float rg, uint64_t seed, int64_t tick,
                const float* noise, float* bias, float* out, void* stream);

/* DynamicsModel.step (q/dynamics.py:140-274) on squashed world-frame commands,
 * state planes (NP,N,4) -> (NP,N,4); per-row drag/decay (N,4) | NULL. */
int qs_dyn_step_fwd(int32_t model, int32_t n, const float* S_in, const float* act,
                    const float* dr, const qs_task_cfg* cfg, float* S_out, int32_t* err,
                    void* stream);
int qs_dyn_step_bwd(int32_t model, int32_t n, const float* S_in, const float* act,
                    const float* dr, const qs_task_cfg* cfg, const float* g_S_out, float* g_S_in,
                    float* g_act, void* stream);

/* reconstruct_attitude (q/sensors.py:569-606): a (N,4), v_ema (N,4) -> R (N,9). */
int qs_reconstruct_attitude(int32_t n, const float* a, const float* v_ema, float* R, void* stream);

/* Philox4x32-10 (Salmon et al., SC'11), the counter-based generator behind every
 * in-kernel draw (resets, DR, IMU, scenes), exposed for known-answer tests:
 * items (n,6) = ctr[4], key[2] -> out (n,8) = the block computed with the key
 * schedule on the fly, then with precomputed round keys (the two must agree). */
int qs_philox4x32_10(int32_t n, const uint32_t* ctr_key, uint32_t* out, void* stream);
/* tcgen05 self-test: D (128x128 fp32) = A (128x128) @ B (128x128), bf16 operands
 * staged K-major or MN-major (mode bit 0: A, bit 1: B) in shared memory */
int qs_probe_umma(int32_t mode, const float* A, const float* B, float* D, void* stream);
/* Philox4x32-7 (the IMU sensor-noise generator), same layout */
int qs_philox4x32_7(int32_t n, const uint32_t* ctr_key, uint32_t* out, void* stream);

/* Measurement aid (not part of the reference API): FP32 peak probe for the
 * ray-casting roofline.  n_blocks CTAs of 256 threads, each thread 8 independent
 * FMA chains x 16 x iters; mode 0 = FFMA, mode 1 = packed fma.rn.f32x2 (FFMA2).
 * FLOPs per launch = n_blocks * 256 * iters * 256 (mode 0), twice that (mode 1). */
int qs_probe_fp32(int32_t mode, int32_t n_blocks, int32_t iters, float* out, void* stream);

/* In-kernel obstacle-course generation with BFS feasibility
 * (q/world.py:207-340), Philox keyed by (seed, global env id, attempt). */
typedef struct qs_gen_cfg {
  float spawn[3], goal[3];
  float density, r_quad, clearance, corridor_halfwidth;
  int32_t indoor, max_attempts, Sm, Bm, Cm;
  uint64_t seed;
  int64_t env_offset;
  /* re-randomisation on reset: only envs with env_mask[e] != 0 are
   * regenerated (NULL = all), keyed additionally by episode[e * episode_stride]
   * (NULL = episode 0).  Lets a reset regenerate its obstacles on device. */
  const uint8_t* env_mask;
  const int32_t* episode;
  int32_t episode_stride;
} qs_gen_cfg;
int qs_gen_obstacle_course(const qs_gen_cfg* cfg, int32_t n_envs, float* bounds, float* spawn_goal,
                           float* spheres, float* boxes, float* cylinders, int32_t* counts,
                           float* ground_z, int32_t* err, void* stream);

/* In-kernel race-track generation (replaces the reference's per-env host
 * loop gen_race_track, q/world.py:347-379): gates chained along an open loop,
 * spacing U(4, spread), heading turns U(-pi/6, pi/6) after the first gate,
 * gate heights U(1, 2.5); Philox keyed by (seed, global env id, episode).
 * Writes bounds (E,2,4), spawn_goal (E,2,4), gates (E,G,8) = centre, inner
 * radius 0.8, normal, frame width 0.3; counts (E,4) = (0,0,0,1), ground_z 0.
 * env_mask / episode as in qs_gen_cfg (regeneration on reset). */
typedef struct qs_track_cfg {
  int32_t n_gates;
  float spread;
  uint64_t seed;
  int64_t env_offset;
  const uint8_t* env_mask;
  const int32_t* episode;
  int32_t episode_stride;
} qs_track_cfg;
int qs_gen_race_track(const qs_track_cfg* cfg, int32_t n_envs, float* bounds, float* spawn_goal, float* gates,
                      int32_t* counts, float* ground_z, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* QUADSIM_B200_H */
