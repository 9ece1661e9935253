// torch custom-op layer over the C ABI (include/quadsim_b200.h): the fused env
// step of FlightTask.step (q/tasks.py:549-600) as the dispatcher op
//
//   quadsim::task_step(Tensor cfg, Tensor[] scene, Tensor S_in, Tensor raw,
//                      Tensor[] bufs, Tensor? imu_noise, bool want_cam,
//                      bool strict, int proprio_dim) -> Tensor[]
//
// with a C++ autograd kernel (one node per step whose backward is the
// analytic VJP kernel qs_task_step_bwd) and a CUDA kernel; its fake (shape)
// implementation is registered from Python (_lib.ops), so torch sees the op
// under FakeTensor / torch.compile tracing.  A step costs one call instead of
// ctypes struct building and Python allocations.
//
//   cfg    CPU uint8 tensor holding a qs_task_cfg (built once per reset)
//   scene  [bounds, spawn_goal, spheres, boxes, cylinders, counts, ground_z, gates]
//   bufs   [goal, peff, dr | empty, meta, ep_return, imu_bias | empty, stats, err]
//          (meta, ep_return, imu_bias, stats, err are updated in place)
//   out    [S_out, obs, r_ctrl, r_goal, r_rl, terminated, truncated, flags,
//           goal_out, peff_out, dr_out | empty, cam | empty, imu_out | empty]
//   strict launches qs_task_validate first and guards the step on it: a
//          rejected step mutates nothing (one host read of err[2] decides).
//   proprio_dim  the observation width (= cfg's; the fake implementation
//          cannot read the cfg bytes under FakeTensor tracing)
#include <ATen/ATen.h>
#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAGuard.h>
#include <torch/autograd.h>
#include <torch/extension.h>
#include <torch/library.h>

#include "../../include/quadsim_b200.h"

namespace {

using torch::autograd::AutogradContext;
using torch::autograd::variable_list;

const qs_task_cfg& cfg_of(const at::Tensor& blob) {
  TORCH_CHECK(blob.device().is_cpu() && blob.scalar_type() == at::kByte && blob.is_contiguous() &&
                  blob.numel() == (int64_t)sizeof(qs_task_cfg),
              "quadsim::task_step: cfg must be a CPU uint8 tensor of sizeof(qs_task_cfg) bytes");
  return *reinterpret_cast<const qs_task_cfg*>(blob.data_ptr());
}

template <typename T = void>
T* ptr(const at::Tensor& t) {
  return t.defined() && t.numel() > 0 ? reinterpret_cast<T*>(t.data_ptr()) : nullptr;
}

qs_scene scene_of(at::TensorList sc) {
  TORCH_CHECK(sc.size() == 8, "quadsim::task_step: scene needs 8 tensors");
  qs_scene s{};
  s.bounds = ptr<const float>(sc[0]);
  s.spawn_goal = ptr<const float>(sc[1]);
  s.spheres = ptr<const float>(sc[2]);
  s.boxes = ptr<const float>(sc[3]);
  s.cylinders = ptr<const float>(sc[4]);
  s.counts = ptr<const int32_t>(sc[5]);
  s.ground_z = ptr<const float>(sc[6]);
  s.gates = ptr<const float>(sc[7]);
  s.Sm = (int32_t)sc[2].size(1);
  s.Bm = (int32_t)sc[3].size(1);
  s.Cm = (int32_t)sc[4].size(1);
  return s;
}

int planes_of(int model) { return model == QS_MODEL_FULL ? 4 : (model == QS_MODEL_SIMPLIFIED ? 5 : 3); }

void check_status(int st, const char* what) {
  TORCH_CHECK(st == QS_OK, "quadsim::", what, " failed with status ", st);
}

// output tensors of one step (shapes from the cfg), carved from two
// allocations (fp32 and int32 words) instead of thirteen: a step's host cost
// is dominated by allocator calls, not by the launch
std::vector<at::Tensor> alloc_outputs(const qs_task_cfg& c, const at::Tensor& S_in, bool has_dr, bool want_cam,
                                      bool has_imu) {
  const int64_t N = (int64_t)c.n_envs * c.n_agents, P = c.proprio_dim, NP = S_in.size(0);
  // fp32 words: S_out | obs | r_ctrl r_goal r_rl | goal_out | peff_out | dr_out | cam | imu_out
  const int64_t nS = NP * N * 4, nO = N * P, nD = has_dr ? 4 * N : 0, nC = want_cam ? 2 * N : 0,
                nI = has_imu ? 6 * N : 0;
  auto up = [](int64_t n) { return (n + 31) & ~int64_t(31); };
  const int64_t nf = up(nS) + up(nO) + 3 * up(N) + 2 * up(4 * N) + up(nD) + up(nC) + up(nI);
  // int32 words after the fp32 ones: flags | terminated (int8) + truncated (bool) bytes
  const int64_t nb = (2 * N + 3) / 4;
  // ONE allocation for every output (fp32 words, then the int32 words)
  const at::Tensor fbuf = at::empty({nf + N + nb}, S_in.options());
  // the pieces are tensors over the buffers' storage built directly (no
  // dispatcher round trip per narrow/view: ~1 us each, a third of a step)
  auto carve = [](const at::Tensor& base, int64_t byte_off, std::initializer_list<int64_t> sizes,
                  at::ScalarType st) {
    auto impl = c10::make_intrusive<c10::TensorImpl>(c10::Storage(base.storage()), base.key_set(),
                                                     c10::scalarTypeToTypeMeta(st));
    impl->set_sizes_contiguous(at::IntArrayRef(sizes));
    impl->set_storage_offset(byte_off / (int64_t)c10::elementSize(st));
    return at::Tensor(std::move(impl));
  };
  int64_t o = 0;  // fp32 word offset; every piece starts on a 128-byte boundary (16-byte vector stores)
  auto take = [&](int64_t n, std::initializer_list<int64_t> sizes) {
    at::Tensor t = carve(fbuf, 4 * o, sizes, at::kFloat);
    o += (n + 31) & ~int64_t(31);
    return t;
  };
  at::Tensor S_out = take(nS, {NP, N, 4});
  at::Tensor obs = take(nO, {N, P});
  at::Tensor rc = take(N, {N}), rg = take(N, {N}), rl = take(N, {N});
  at::Tensor goal = take(4 * N, {N, 4}), peff = take(4 * N, {N, 4});
  at::Tensor dr = has_dr ? take(nD, {N, 4}) : take(0, {0});
  at::Tensor cam = want_cam ? take(nC, {N, 2}) : take(0, {0});
  at::Tensor imu = has_imu ? take(nI, {N, 6}) : take(0, {0});
  at::Tensor flags = carve(fbuf, 4 * nf, {N}, at::kInt);
  at::Tensor term = carve(fbuf, 4 * (nf + N), {N}, at::kChar);
  at::Tensor trunc = carve(fbuf, 4 * (nf + N) + N, {N}, at::kBool);
  return {S_out, obs, rc, rg, rl, term, trunc, flags, goal, peff, dr, cam, imu};
}

std::vector<at::Tensor> task_step_cuda(const at::Tensor& cfg_blob, at::TensorList scene, const at::Tensor& S_in,
                                       const at::Tensor& raw, at::TensorList bufs,
                                       const std::optional<at::Tensor>& imu_noise, bool want_cam, bool strict,
                                       int64_t proprio_dim) {
  qs_task_cfg c = cfg_of(cfg_blob);
  TORCH_CHECK(proprio_dim == c.proprio_dim, "quadsim::task_step: proprio_dim does not match the cfg");
  TORCH_CHECK(bufs.size() == 8, "quadsim::task_step: bufs needs 8 tensors");
  TORCH_CHECK(S_in.is_cuda() && S_in.scalar_type() == at::kFloat && S_in.is_contiguous(), "S_in: CUDA fp32");
  TORCH_CHECK(raw.is_cuda() && raw.scalar_type() == at::kFloat && raw.is_contiguous(), "raw: CUDA fp32");
  const int64_t N = (int64_t)c.n_envs * c.n_agents;
  TORCH_CHECK(S_in.dim() == 3 && S_in.size(0) == planes_of(c.model) && S_in.size(1) == N && S_in.size(2) == 4,
              "S_in: (NP, N, 4)");
  TORCH_CHECK(raw.dim() == 2 && raw.size(0) == N && raw.size(1) == c.action_dim, "raw: (N, A)");
  const c10::cuda::CUDAGuard guard(S_in.device());
  const bool has_dr = bufs[2].numel() > 0, has_imu = bufs[5].numel() > 0;
  auto out = alloc_outputs(c, S_in, has_dr, want_cam, has_imu);
  const qs_scene sc = scene_of(scene);
  qs_step_io io{};
  io.S_in = S_in.data_ptr<float>();
  io.S_out = ptr<float>(out[0]);
  io.raw = raw.data_ptr<float>();
  io.goal_in = ptr<const float>(bufs[0]);
  io.goal_out = ptr<float>(out[8]);
  io.peff_in = ptr<const float>(bufs[1]);
  io.peff_out = ptr<float>(out[9]);
  io.dr_in = ptr<const float>(bufs[2]);
  io.dr_out = ptr<float>(out[10]);
  io.meta = ptr<int32_t>(bufs[3]);
  io.ep_return = ptr<float>(bufs[4]);
  io.imu_bias = ptr<float>(bufs[5]);
  io.imu_noise = imu_noise.has_value() ? ptr<const float>(*imu_noise) : nullptr;
  io.imu_out = ptr<float>(out[12]);
  io.obs = ptr<float>(out[1]);
  io.r_ctrl = ptr<float>(out[2]);
  io.r_goal = ptr<float>(out[3]);
  io.r_rl = ptr<float>(out[4]);
  io.terminated = ptr<int8_t>(out[5]);
  io.truncated = ptr<uint8_t>(out[6]);
  io.flags = ptr<int32_t>(out[7]);
  io.cam = ptr<float>(out[11]);
  io.stats = ptr<double>(bufs[6]);
  io.err = ptr<int32_t>(bufs[7]);
  void* stream = at::cuda::getCurrentCUDAStream(S_in.device().index()).stream();
  if (strict) {
    TORCH_CHECK(bufs[7].numel() >= 3, "strict steps need a 3-int error word");
    check_status(qs_task_validate(&c, &io, stream), "qs_task_validate");
    c.guard = 1;
  }
  check_status(qs_task_step_fwd(&c, &sc, &io, stream), "qs_task_step_fwd");
  return out;
}

// one env step as an autograd node: differentiable inputs S_in, raw;
// differentiable outputs S_out, obs, r_ctrl (q/tasks.py:549-600)
struct TaskStepFn : public torch::autograd::Function<TaskStepFn> {
  static variable_list forward(AutogradContext* ctx, const at::Tensor& S_in, const at::Tensor& raw,
                               const at::Tensor& cfg_blob, std::vector<at::Tensor> scene,
                               std::vector<at::Tensor> bufs, std::optional<at::Tensor> imu_noise, bool want_cam,
                               bool strict, int64_t proprio_dim, bool direct) {
    // direct (the pybind entry, real CUDA tensors): call the CUDA kernel
    // without a dispatcher round trip; otherwise redispatch below autograd --
    // the CUDA kernel for real tensors, the fake kernel under tracing
    if (direct) {
      auto out = task_step_cuda(cfg_blob, scene, S_in, raw, bufs, imu_noise, want_cam, strict, proprio_dim);
      ctx->save_for_backward({S_in, raw, bufs[0], bufs[1], bufs[2], out[7]});
      ctx->saved_data["cfg"] = cfg_blob;
      ctx->saved_data["scene"] = scene;
      ctx->mark_non_differentiable(variable_list(out.begin() + 3, out.end()));
      ctx->set_materialize_grads(false);
      return out;
    }
    static auto op = c10::Dispatcher::singleton()
                         .findSchemaOrThrow("quadsim::task_step", "")
                         .typed<std::vector<at::Tensor>(const at::Tensor&, at::TensorList, const at::Tensor&,
                                                        const at::Tensor&, at::TensorList,
                                                        const std::optional<at::Tensor>&, bool, bool, int64_t)>();
    at::AutoDispatchBelowADInplaceOrView g;
    auto out = op.call(cfg_blob, scene, S_in, raw, bufs, imu_noise, want_cam, strict, proprio_dim);
    // the step's checkpoint: pre-step state, action, goal, previous effort, DR
    // draw and the flag record; the scene the SDF penalty was evaluated on
    ctx->save_for_backward({S_in, raw, bufs[0], bufs[1], bufs[2], out[7]});
    ctx->saved_data["cfg"] = cfg_blob;
    ctx->saved_data["scene"] = scene;
    ctx->mark_non_differentiable(variable_list(out.begin() + 3, out.end()));  // one call: it replaces the set
    ctx->set_materialize_grads(false);
    return out;
  }

  static variable_list backward(AutogradContext* ctx, variable_list go) {
    const auto saved = ctx->get_saved_variables();
    const at::Tensor &S_in = saved[0], &raw = saved[1];
    const at::Tensor gS = go[0].defined() ? go[0].contiguous() : at::Tensor();
    const at::Tensor gobs = go[1].defined() ? go[1].contiguous() : at::Tensor();
    const at::Tensor gr = go[2].defined() ? go[2].contiguous() : at::Tensor();
    variable_list grads(10);
    if (!gS.defined() && !gobs.defined() && !gr.defined()) return grads;
    const c10::cuda::CUDAGuard guard(S_in.device());
    const qs_task_cfg& c = cfg_of(ctx->saved_data["cfg"].toTensor());
    const auto scene_t = ctx->saved_data["scene"].toTensorVector();
    const qs_scene sc = scene_of(scene_t);
    at::Tensor gS_in = at::empty_like(S_in), g_raw = at::empty_like(raw);
    qs_step_grad g{};
    g.S_in = S_in.data_ptr<float>();
    g.raw = raw.data_ptr<float>();
    g.goal_in = ptr<const float>(saved[2]);
    g.peff_in = ptr<const float>(saved[3]);
    g.dr_in = ptr<const float>(saved[4]);
    g.flags = ptr<const int32_t>(saved[5]);
    g.g_S_out = gS.defined() ? gS.data_ptr<float>() : nullptr;
    g.g_obs = gobs.defined() ? gobs.data_ptr<float>() : nullptr;
    g.g_rctrl = gr.defined() ? gr.data_ptr<float>() : nullptr;
    g.g_S_in = gS_in.data_ptr<float>();
    g.g_raw = g_raw.data_ptr<float>();
    check_status(qs_task_step_bwd(&c, &sc, &g, at::cuda::getCurrentCUDAStream(S_in.device().index()).stream()),
                 "qs_task_step_bwd");
    grads[0] = gS_in;
    grads[1] = g_raw;
    return grads;
  }
};

std::vector<at::Tensor> task_step_autograd(const at::Tensor& cfg_blob, at::TensorList scene, const at::Tensor& S_in,
                                           const at::Tensor& raw, at::TensorList bufs,
                                           const std::optional<at::Tensor>& imu_noise, bool want_cam, bool strict,
                                           int64_t proprio_dim) {
  return TaskStepFn::apply(S_in, raw, cfg_blob, scene.vec(), bufs.vec(), imu_noise, want_cam, strict,
                           proprio_dim, false);
}

}  // namespace

TORCH_LIBRARY(quadsim, m) {
  m.def(
      "task_step(Tensor cfg, Tensor[] scene, Tensor S_in, Tensor raw, Tensor[] bufs, Tensor? imu_noise, "
      "bool want_cam, bool strict, int proprio_dim) -> Tensor[]");
}

TORCH_LIBRARY_IMPL(quadsim, CUDA, m) { m.impl("task_step", task_step_cuda); }
TORCH_LIBRARY_IMPL(quadsim, Autograd, m) { m.impl("task_step", task_step_autograd); }

// The same kernel as a direct Python entry point: FlightTask.step calls it
// to skip the generic schema-driven argument boxing of torch.ops (measured
// ~10 us per call for this op's 18 tensor arguments); the dispatcher op above
// is what torch's tracing / FakeTensor machinery sees.
PYBIND11_MODULE(_qs_torch_ops, m) {
  m.def(
      "task_step",
      [](const at::Tensor& cfg_blob, const std::vector<at::Tensor>& scene, const at::Tensor& S_in,
         const at::Tensor& raw, const std::vector<at::Tensor>& bufs, const std::optional<at::Tensor>& imu_noise,
         bool want_cam, bool strict, int64_t proprio_dim) {
        // no autograd node when nothing needs a gradient; else the node with a
        // direct kernel call (no dispatcher round trip either way)
        if (!(at::GradMode::is_enabled() && (S_in.requires_grad() || raw.requires_grad()))) {
          at::AutoDispatchBelowADInplaceOrView g;
          return task_step_cuda(cfg_blob, scene, S_in, raw, bufs, imu_noise, want_cam, strict, proprio_dim);
        }
        return TaskStepFn::apply(S_in, raw, cfg_blob, scene, bufs, imu_noise, want_cam, strict, proprio_dim,
                                 true);
      },
      "quadsim::task_step (autograd path)");
}
