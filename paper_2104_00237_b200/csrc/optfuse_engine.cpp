// optfuse_engine.cpp -- native hook scheduler for forward- and backward-fusion.
//
// The reference schedules updates from Python (schedule.py:98-207) and
// overlaps them with backward through a Python thread pool (schedule.py:210-311).
// On B200 the per-layer host work must cost well under the ~5-10 us a small
// backward kernel takes, or the fused schedules become CPU-bound.  So the
// whole per-layer path lives here, in C++:
//
//   * backward fusion: a C++ PostAccumulateGradHook on every parameter (fires
//     once per iteration, after every contribution has been accumulated and
//     after the consuming node computed its input gradient from the old value
//     -- Appendix B.2's safety condition, schedule.py:54-59).  When the last
//     parameter of a launch group (a layer, or a bucket of consecutive layers
//     in backward order) is ready, the engine records an event on the
//     autograd stream, makes the high-priority update stream wait on it and
//     launches one multi-tensor update kernel there (liboptfuse_b200 C ABI).
//     The compute stream joins the update stream once, at finish().
//   * forward fusion: ff_layer(l), called from the layer's forward pre-hook,
//     launches the update of every pending, not-yet-updated parameter of that
//     layer on the compute stream right before the layer's kernels (the
//     `updated` latch of schedule.py:112-121; the frozen step index of :133).
//
// Gradients are read straight from the parameters (param.grad()); with
// release_grads the engine drops them after the launch (set-to-none), keeping
// them alive in `hold_` until the update stream has been joined.
#include <torch/extension.h>
#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDACachingAllocator.h>
#include <c10/cuda/CUDAGuard.h>
#include <torch/csrc/autograd/function_hook.h>
#include <torch/csrc/autograd/variable.h>

#include <cuda_runtime_api.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "optfuse_b200.h"

namespace {

namespace py = pybind11;
using torch::autograd::Variable;

int dtype_code(at::ScalarType t) {
  switch (t) {
    case at::kFloat: return OF_F32;
    case at::kDouble: return OF_F64;
    case at::kBFloat16: return OF_BF16;
    default: throw std::invalid_argument("optfuse: unsupported dtype for the update kernels");
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// A fixed list of parameters updated by one kernel launch.
struct Group {
  std::vector<int> members;
  std::vector<void*> p, g, s0, s1, sh;
  std::vector<int64_t> n;
  of_tensor_list list{};
  cudaEvent_t ready = nullptr;
  int64_t elems = 0;

  void bind() {
    const size_t k = members.size();
    p.resize(k); g.resize(k); s0.resize(k); s1.resize(k); sh.resize(k); n.resize(k);
    list.n = static_cast<int32_t>(k);
    list.param = p.data();
    list.grad = g.data();
    list.state0 = s0.data();
    list.state1 = s1.data();
    list.shadow = sh.data();
    list.numel = n.data();
  }
};

class Engine;

struct FusionHook : torch::autograd::PostAccumulateGradHook {
  std::weak_ptr<Engine> eng;
  int idx;
  FusionHook(std::weak_ptr<Engine> e, int i) : eng(std::move(e)), idx(i) {}
  void operator()(const Variable& tensor) override;
};

class Engine : public std::enable_shared_from_this<Engine> {
 public:
  Engine(std::vector<at::Tensor> params, std::vector<std::vector<int>> bf_groups,
         std::vector<std::vector<int>> layers, int64_t side_stream)
      : params_(std::move(params)), layers_(std::move(layers)), ff_units_(layers_),
        side_(reinterpret_cast<cudaStream_t>(side_stream)) {
    const int np = static_cast<int>(params_.size());
    s0_.assign(np, at::Tensor());
    s1_.assign(np, at::Tensor());
    master_.assign(np, at::Tensor());
    group_of_.assign(np, -1);
    pending_.assign(np, 0);
    updated_.assign(np, 0);
    for (auto& members : bf_groups) {
      Group G;
      G.members = members;
      G.bind();
      for (int idx : members) {
        if (idx < 0 || idx >= np) throw std::out_of_range("optfuse: group member out of range");
        if (group_of_[idx] != -1) throw std::invalid_argument("optfuse: parameter in two groups");
        group_of_[idx] = static_cast<int>(groups_.size());
        G.elems += params_[idx].numel();
      }
      if (side_) cuda_check(cudaEventCreateWithFlags(&G.ready, cudaEventDisableTiming), "cudaEventCreate");
      groups_.push_back(std::move(G));
    }
    ready_.assign(groups_.size(), 0);
    launched_.assign(groups_.size(), 0);
    if (side_) cuda_check(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming), "cudaEventCreate");
    hp_ = of_hparams{};
  }

  ~Engine() {
    remove_hooks();
    for (auto& G : groups_)
      if (G.ready) cudaEventDestroy(G.ready);
    if (join_) cudaEventDestroy(join_);
    for (auto e : prefetch_done_)
      if (e) cudaEventDestroy(e);
    if (prefetch_group_.ready) cudaEventDestroy(prefetch_group_.ready);
    clear_profile();
  }

  // -- configuration -------------------------------------------------------
  // History slots of parameter idx and, for mixed precision, its fp32 master
  // copy: the kernel then updates the master and writes the (bf16) parameter
  // as the shadow in the same pass.
  void set_slots(int idx, c10::optional<at::Tensor> a, c10::optional<at::Tensor> b,
                 c10::optional<at::Tensor> master) {
    s0_.at(idx) = a.has_value() ? *a : at::Tensor();
    s1_.at(idx) = b.has_value() ? *b : at::Tensor();
    master_.at(idx) = master.has_value() ? *master : at::Tensor();
    // static pointers of the BF groups
    const int gi = group_of_[idx];
    if (gi >= 0) refresh_static(groups_[gi]);
  }

  void set_hparams(int kind, double eta, double alpha, double wd, double eps, double b1, double b2,
                   double rho, double bc1, double bc2, int64_t flags, bool release_grads,
                   c10::optional<at::Tensor> grad_scale, int max_ctas,
                   c10::optional<at::Tensor> step_offset, c10::optional<at::Tensor> step_table,
                   int64_t t_base) {
    hp_.kind = kind;
    hp_.max_ctas = max_ctas;
    hp_.eta = eta;
    hp_.alpha = alpha;
    hp_.weight_decay = wd;
    hp_.epsilon = eps;
    hp_.beta1 = b1;
    hp_.beta2 = b2;
    hp_.rho = rho;
    hp_.bias_correction1 = bc1;
    hp_.bias_correction2 = bc2;
    flags_ = static_cast<uint32_t>(flags);
    release_ = release_grads;
    gscale_ = grad_scale.has_value() ? *grad_scale : at::Tensor();
    // OF_FLAG_DEVICE_STEP: step index read on the device (CUDA-graph replay)
    step_offset_ = step_offset.has_value() ? *step_offset : at::Tensor();
    step_table_ = step_table.has_value() ? *step_table : at::Tensor();
    hp_.step_offset_dev = step_offset_.defined() ? step_offset_.data_ptr<int64_t>() : nullptr;
    hp_.step_table_dev = step_table_.defined() ? step_table_.data_ptr<double>() : nullptr;
    hp_.step_table_rows = step_table_.defined() ? step_table_.size(0) : 0;
    hp_.t_base = t_base;
  }

  // (Re)installs this engine's hook on every grouped parameter, replacing
  // whatever post-accumulate-grad hook another engine of the graph had set.
  void install_hooks() {
    auto self = weak_from_this();
    for (size_t i = 0; i < params_.size(); ++i) {
      if (group_of_[i] < 0) continue;
      torch::autograd::impl::set_post_acc_grad_hooks(
          params_[i], std::make_unique<FusionHook>(self, static_cast<int>(i)));
    }
    hooks_installed_ = true;
  }

  void remove_hooks() {
    if (!hooks_installed_) return;
    for (auto& p : params_) {
      auto& h = torch::autograd::impl::post_acc_grad_hooks(p);
      auto* mine = h ? dynamic_cast<FusionHook*>(h.get()) : nullptr;
      if (mine && mine->eng.lock().get() == this) torch::autograd::impl::set_post_acc_grad_hooks(p, nullptr);
    }
    hooks_installed_ = false;
  }

  void set_callback(py::object cb) { callback_ = cb.is_none() ? py::object() : cb; }

  void set_debug_skip_ready_wait(bool on) { debug_skip_ready_wait_ = on; }

  // -- backward fusion -----------------------------------------------------
  // Arms the hooks for one backward pass.  launch=false only reports
  // gradient readiness to the callback (schedule tracing of the unfused
  // schedules).
  void bf_begin(bool launch) {
    std::fill(ready_.begin(), ready_.end(), 0);
    std::fill(launched_.begin(), launched_.end(), 0);
    armed_ = true;
    launch_ = launch;
  }

  void disarm() { armed_ = false; }

  void on_ready(int idx) {
    if (!armed_) return;
    if (callback_) {
      py::gil_scoped_acquire gil;
      callback_(idx);
    }
    const int gi = group_of_[idx];
    if (gi < 0) return;
    if (!launch_) {
      // readiness only: the group callback (data-parallel buckets) runs once
      // per complete group instead of Python once per parameter
      if (group_cb_ && ++ready_[gi] == static_cast<int>(groups_[gi].members.size())) {
        if (gi < static_cast<int>(views_.size()) && !views_[gi].empty()) gather_group(gi);
        py::gil_scoped_acquire gil;
        group_cb_(gi);
      }
      return;
    }
    if (++ready_[gi] == static_cast<int>(groups_[gi].members.size())) launch_group(gi);
  }

  void set_group_callback(py::object cb) { group_cb_ = cb.is_none() ? py::object() : cb; }

  // Data parallel: where group gi's gradients land (views into its flat
  // buffer, one per member, same strides as the parameter).  When the group
  // completes, its gradients are copied there on the side (communication)
  // stream with one of_copy_mt launch and released, before the Python
  // callback issues the collectives -- no Python per parameter.
  void set_group_views(int gi, std::vector<at::Tensor> views) {
    if (gi < 0 || gi >= static_cast<int>(groups_.size()))
      throw std::out_of_range("optfuse: group index out of range");
    if (views.size() != groups_[gi].members.size())
      throw std::invalid_argument("optfuse: one view per group member");
    if (views_.size() < groups_.size()) views_.resize(groups_.size());
    views_[gi] = std::move(views);
  }

  static bool same_layout(const at::Tensor& a, const at::Tensor& b) {
    if (a.scalar_type() != b.scalar_type() || a.sizes() != b.sizes()) return false;
    for (int64_t d = 0; d < a.dim(); ++d)
      if (a.size(d) > 1 && a.stride(d) != b.stride(d)) return false;
    return a.is_non_overlapping_and_dense() && b.is_non_overlapping_and_dense();
  }

  void gather_group(int gi) {
    Group& G = groups_[gi];
    cudaStream_t cur = current();
    cudaStream_t s = side_ ? side_ : cur;
    if (side_) {
      cuda_check(cudaEventRecord(G.ready, cur), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(side_, G.ready, 0), "cudaStreamWaitEvent");
    }
    const auto dev = params_[G.members[0]].device();
    c10::cuda::CUDAStream cs = c10::cuda::getStreamFromExternal(s, dev.index());
    c10::cuda::CUDAStreamGuard guard(cs);
    std::vector<void*> dst;
    std::vector<const void*> src;
    std::vector<int64_t> nbytes;
    std::vector<at::Tensor> used;
    const auto& views = views_[gi];
    for (size_t k = 0; k < G.members.size(); ++k) {
      at::Tensor& gr = params_[G.members[k]].mutable_grad();
      const at::Tensor& v = views[k];
      if (!gr.defined()) {          // no contribution this iteration: the reference steps with 0
        v.zero_();
        continue;
      }
      if (same_layout(v, gr)) {
        dst.push_back(v.data_ptr());
        src.push_back(gr.data_ptr());
        nbytes.push_back(v.numel() * static_cast<int64_t>(v.element_size()));
      } else {
        v.copy_(gr);
      }
      used.push_back(gr);
      gr = at::Tensor();
    }
    if (!dst.empty()) {
      const int st = of_copy_mt(dst.data(), src.data(), nbytes.data(), static_cast<int>(dst.size()), s);
      if (st != OF_OK)
        throw std::runtime_error(std::string("of_copy_mt: ") + of_status_string(st) + " (" +
                                 of_last_error() + ")");
    }
    // released on the compute stream's allocator, used on s: reuse waits for s
    for (auto& g : used) c10::cuda::CUDACachingAllocator::recordStream(g.storage().data_ptr(), cs);
  }

  // Launch every group that did not complete during backward (parameters
  // that received no gradient this iteration still step, with g = 0, as the
  // reference steps every parameter), then join the update stream.
  int bf_finish() {
    armed_ = false;
    int late = 0;
    for (size_t gi = 0; gi < groups_.size(); ++gi) {
      if (!launched_[gi]) {
        launch_group(static_cast<int>(gi));
        ++late;
      }
    }
    join();
    return late;
  }

  void join() {
    if (side_) {
      cuda_check(cudaEventRecord(join_, side_), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(current(), join_, 0), "cudaStreamWaitEvent");
    }
    hold_.clear();
  }

  // -- forward fusion ------------------------------------------------------
  void set_all_pending() {
    std::fill(pending_.begin(), pending_.end(), 1);
    std::fill(updated_.begin(), updated_.end(), 0);
  }
  void clear_updated() { std::fill(updated_.begin(), updated_.end(), 0); }
  bool is_pending(int idx) const { return pending_.at(idx) != 0; }
  bool is_updated(int idx) const { return updated_.at(idx) != 0; }
  void set_pending(int idx, bool v) { pending_.at(idx) = v; }
  void set_updated(int idx, bool v) { updated_.at(idx) = v; }
  int64_t num_pending() const {
    int64_t c = 0;
    for (auto v : pending_) c += v;
    return c;
  }

  // Forward-fusion units: by default one per layer; set_ff_units replaces
  // them by buckets of consecutive layers (execution order) whose updates
  // are issued together before the bucket's first layer.
  void set_ff_units(std::vector<std::vector<int>> units) { ff_units_ = std::move(units); }
  void reset_ff_units() { ff_units_ = layers_; }

  // Updates the pending, not yet updated parameters of forward-fusion unit
  // `li` on the current stream; returns how many were updated.
  int ff_layer(int li) {
    const auto& lp = ff_units_.at(li);
    scratch_.members.clear();
    for (int idx : lp)
      if (pending_[idx] && !updated_[idx]) scratch_.members.push_back(idx);
    if (scratch_.members.empty()) return 0;
    launch_dynamic(scratch_, current());
    for (int idx : scratch_.members) {
      updated_[idx] = 1;
      pending_[idx] = 0;
    }
    return static_cast<int>(scratch_.members.size());
  }

  // Forward fusion with one-unit lookahead (needs the side stream): the
  // update of unit u+1 is issued on the side stream when unit u's pre-hook
  // runs, so it overlaps unit u's forward instead of sitting on the compute
  // stream's critical path; unit u+1's pre-hook makes the compute stream wait
  // for it.  Nothing reads unit u+1's parameters in between (a parameter
  // belongs to the unit of the first layer that uses it, and the latch skips
  // parameters already updated), the previous backward is ordered before the
  // prefetch by an event, and the released gradients are held until the
  // compute stream has waited, so the allocator cannot hand them to the
  // forward while the side stream still reads them.
  int ff_unit_lookahead(int u, int depth = 1) {
    if (!side_) return ff_layer(u);
    const int nu = static_cast<int>(ff_units_.size());
    if (prefetch_done_.size() != static_cast<size_t>(nu)) {
      for (auto e : prefetch_done_)
        if (e) cudaEventDestroy(e);
      prefetch_done_.assign(nu, nullptr);
      prefetch_hold_.assign(nu, {});
      prefetched_.assign(nu, 0);
    }
    cudaStream_t cur = current();
    int n = 0;
    if (prefetched_.at(u)) {
      cuda_check(cudaStreamWaitEvent(cur, prefetch_done_[u], 0), "cudaStreamWaitEvent");
      prefetch_hold_[u].clear();
      prefetched_[u] = 0;
    } else {
      n = ff_layer(u);
    }
    // units u+1 .. u+depth (each issued once; prefetch_unit skips updated ones)
    for (int v = u + 1; v < nu && v <= u + depth; ++v)
      if (!prefetched_[v]) n += prefetch_unit(v, cur);
    return n;
  }

  // Joins every prefetched unit whose layer did not run this forward.
  void ff_join() {
    cudaStream_t cur = current();
    for (size_t u = 0; u < prefetched_.size(); ++u) {
      if (!prefetched_[u]) continue;
      cuda_check(cudaStreamWaitEvent(cur, prefetch_done_[u], 0), "cudaStreamWaitEvent");
      prefetch_hold_[u].clear();
      prefetched_[u] = 0;
    }
  }

  // Updates every pending parameter (layer order, each once) on the current
  // stream: forward-fusion leftovers and flush_pending_updates.
  int flush() {
    scratch_.members.clear();
    std::vector<uint8_t> seen(params_.size(), 0);
    for (const auto& lp : layers_)
      for (int idx : lp)
        if (pending_[idx] && !seen[idx]) {
          seen[idx] = 1;
          scratch_.members.push_back(idx);
        }
    if (scratch_.members.empty()) return 0;
    launch_dynamic(scratch_, current());
    for (int idx : scratch_.members) pending_[idx] = 0;
    return static_cast<int>(scratch_.members.size());
  }

  // -- profiling -----------------------------------------------------------
  void set_profile(bool on) { profile_ = on; }
  // A timing event: inside a CUDA-graph capture it becomes an event-record
  // node (cudaEventRecordExternal), re-recorded by every replay, so the launch
  // can be timed live inside the replayed iteration.
  static void record_timing(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing(s, &cs), "cudaStreamIsCapturing");
    if (cs == cudaStreamCaptureStatusActive)
      cuda_check(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal), "cudaEventRecordWithFlags");
    else
      cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
  }

  // The last `last` timed launches (ms, elements), events kept (a replayed
  // graph re-records them).
  std::vector<std::pair<double, int64_t>> peek_profile(int last) {
    std::vector<std::pair<double, int64_t>> out;
    const int n = static_cast<int>(prof_.size());
    for (int i = n - last < 0 ? 0 : n - last; i < n; ++i) {
      auto& r = prof_[i];
      cuda_check(cudaEventSynchronize(r.stop), "cudaEventSynchronize");
      float ms = 0.f;
      cuda_check(cudaEventElapsedTime(&ms, r.start, r.stop), "cudaEventElapsedTime");
      out.emplace_back(ms, r.elems);
    }
    return out;
  }

  std::vector<std::pair<double, int64_t>> take_profile() {
    std::vector<std::pair<double, int64_t>> out;
    for (auto& r : prof_) {
      cuda_check(cudaEventSynchronize(r.stop), "cudaEventSynchronize");
      float ms = 0.f;
      cuda_check(cudaEventElapsedTime(&ms, r.start, r.stop), "cudaEventElapsedTime");
      out.emplace_back(ms, r.elems);
    }
    clear_profile();
    return out;
  }

  // Launches group `gi` now, as its last gradient-ready hook would (sync: with
  // the event edge from the current stream; without it for back-to-back
  // timing replays on a stream the caller has already ordered).
  void launch_now(int gi, bool sync) { launch_group(gi, sync); }

  int64_t launches() const { return launches_; }
  int num_groups() const { return static_cast<int>(groups_.size()); }

 private:
  struct ProfRec {
    cudaEvent_t start, stop;
    int64_t elems;
  };

  static cudaStream_t current() { return at::cuda::getCurrentCUDAStream().stream(); }

  void refresh_static(Group& G) {
    for (size_t k = 0; k < G.members.size(); ++k) {
      const int idx = G.members[k];
      const bool mixed = master_[idx].defined();
      G.p[k] = mixed ? master_[idx].data_ptr() : params_[idx].data_ptr();
      G.s0[k] = s0_[idx].defined() ? s0_[idx].data_ptr() : nullptr;
      G.s1[k] = s1_[idx].defined() ? s1_[idx].data_ptr() : nullptr;
      G.sh[k] = mixed ? params_[idx].data_ptr() : nullptr;
      G.n[k] = params_[idx].numel();
    }
    const int first = G.members[0];
    G.list.param_dtype = dtype_code(master_[first].defined() ? master_[first].scalar_type()
                                                              : params_[first].scalar_type());
  }

  // Fills the grad pointers (allocating a zero gradient on the current stream
  // where none exists).  Returns false if the group is empty.
  void fill_grads(Group& G) {
    for (size_t k = 0; k < G.members.size(); ++k) {
      at::Tensor& gr = params_[G.members[k]].mutable_grad();
      if (!gr.defined()) gr = at::zeros_like(params_[G.members[k]]);
      G.g[k] = gr.data_ptr();
      if (release_) hold_.push_back(gr);
    }
    G.list.grad_dtype = dtype_code(params_[G.members[0]].mutable_grad().scalar_type());
  }

  void release(const Group& G) {
    if (!release_) return;
    for (int idx : G.members) params_[idx].mutable_grad() = at::Tensor();
  }

  void launch(Group& G, cudaStream_t s) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (profile_) {
      cuda_check(cudaEventCreate(&a), "cudaEventCreate");
      cuda_check(cudaEventCreate(&b), "cudaEventCreate");
      record_timing(a, s);
    }
    const void* gs = gscale_.defined() ? gscale_.data_ptr() : nullptr;
    const uint32_t fl = flags_ | (gscale_.defined() && gscale_.scalar_type() == at::kDouble
                                      ? OF_FLAG_SCALE_F64 : 0u);
    const int st = of_policy_step_mt(&G.list, &hp_, gs, fl, s);
    if (st != OF_OK)
      throw std::runtime_error(std::string("of_policy_step_mt: ") + of_status_string(st) + " (" +
                               of_last_error() + ")");
    if (profile_) {
      record_timing(b, s);
      prof_.push_back({a, b, G.elems});
    }
    ++launches_;
  }

  void launch_group(int gi, bool sync = true) {
    Group& G = groups_[gi];
    fill_grads(G);
    cudaStream_t cur = current();
    cudaStream_t s = side_ ? side_ : cur;
    if (side_ && sync && !debug_skip_ready_wait_) {
      // the device half of the Appendix B.2 guard: every kernel that reads
      // the old parameter (this layer's input-gradient computation) was
      // enqueued on `cur` before this hook fired, so the update waits for them
      cuda_check(cudaEventRecord(G.ready, cur), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(side_, G.ready, 0), "cudaStreamWaitEvent");
      s = side_;
    }
    launch(G, s);
    release(G);
    launched_[gi] = 1;
  }

  int prefetch_unit(int u, cudaStream_t cur) {
    Group& G = prefetch_group_;
    G.members.clear();
    for (int idx : ff_units_[u])
      if (pending_[idx] && !updated_[idx]) G.members.push_back(idx);
    if (G.members.empty()) return 0;
    G.bind();
    G.elems = 0;
    for (int idx : G.members) G.elems += params_[idx].numel();
    refresh_static(G);
    const size_t held = hold_.size();
    fill_grads(G);                       // (zero gradients, if any, on the compute stream)
    if (!G.ready) cuda_check(cudaEventCreateWithFlags(&G.ready, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventRecord(G.ready, cur), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(side_, G.ready, 0), "cudaStreamWaitEvent");
    launch(G, side_);
    release(G);
    if (!prefetch_done_[u])
      cuda_check(cudaEventCreateWithFlags(&prefetch_done_[u], cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventRecord(prefetch_done_[u], side_), "cudaEventRecord");
    // gradients this launch reads stay referenced until the compute stream waited
    prefetch_hold_[u].assign(hold_.begin() + held, hold_.end());
    hold_.resize(held);
    prefetched_[u] = 1;
    for (int idx : G.members) {
      updated_[idx] = 1;
      pending_[idx] = 0;
    }
    return static_cast<int>(G.members.size());
  }

  void launch_dynamic(Group& G, cudaStream_t s) {
    G.bind();
    G.elems = 0;
    for (int idx : G.members) G.elems += params_[idx].numel();
    refresh_static(G);
    fill_grads(G);
    launch(G, s);
    release(G);
    if (release_) hold_.clear();  // same-stream use: the allocator orders reuse after it
  }

  void clear_profile() {
    for (auto& r : prof_) {
      cudaEventDestroy(r.start);
      cudaEventDestroy(r.stop);
    }
    prof_.clear();
  }

  std::vector<at::Tensor> params_, s0_, s1_, master_;
  std::vector<std::vector<int>> layers_;
  std::vector<std::vector<int>> ff_units_;
  std::vector<Group> groups_;
  Group scratch_, prefetch_group_;
  std::vector<cudaEvent_t> prefetch_done_;
  std::vector<std::vector<at::Tensor>> prefetch_hold_;
  std::vector<uint8_t> prefetched_;
  std::vector<int> group_of_, ready_;
  std::vector<uint8_t> launched_, pending_, updated_;
  std::vector<at::Tensor> hold_;
  of_hparams hp_;
  uint32_t flags_ = 0;
  bool release_ = false;
  at::Tensor gscale_, step_offset_, step_table_;
  cudaStream_t side_ = nullptr;
  cudaEvent_t join_ = nullptr;
  bool armed_ = false;
  bool launch_ = true;
  bool hooks_installed_ = false;
  bool profile_ = false;
  // TEST ONLY (tests/test_race_guard_gpu.py): launch side-stream updates
  // without waiting for the gradient-ready event -- removes the guard so the
  // adversarial test can show that it is what keeps the old weights intact
  bool debug_skip_ready_wait_ = false;
  std::vector<ProfRec> prof_;
  int64_t launches_ = 0;
  py::object callback_, group_cb_;
  std::vector<std::vector<at::Tensor>> views_;
};

void FusionHook::operator()(const Variable&) {
  if (auto e = eng.lock()) e->on_ready(idx);
}

}  // namespace

PYBIND11_MODULE(_optfuse_engine, m) {
  m.doc() = "Native hook scheduler for forward/backward fusion (liboptfuse_b200 launches)";
  py::class_<Engine, std::shared_ptr<Engine>>(m, "Engine")
      .def(py::init<std::vector<at::Tensor>, std::vector<std::vector<int>>,
                    std::vector<std::vector<int>>, int64_t>(),
           py::arg("params"), py::arg("bf_groups"), py::arg("layers"), py::arg("side_stream"))
      .def("set_slots", &Engine::set_slots)
      .def("set_hparams", &Engine::set_hparams)
      .def("install_hooks", &Engine::install_hooks)
      .def("remove_hooks", &Engine::remove_hooks)
      .def("set_callback", &Engine::set_callback)
      .def("set_group_callback", &Engine::set_group_callback)
      .def("set_group_views", &Engine::set_group_views)
      .def("bf_begin", &Engine::bf_begin, py::arg("launch") = true)
      .def("disarm", &Engine::disarm)
      .def("bf_finish", &Engine::bf_finish)
      .def("join", &Engine::join)
      .def("set_all_pending", &Engine::set_all_pending)
      .def("clear_updated", &Engine::clear_updated)
      .def("is_pending", &Engine::is_pending)
      .def("is_updated", &Engine::is_updated)
      .def("set_pending", &Engine::set_pending)
      .def("set_updated", &Engine::set_updated)
      .def("num_pending", &Engine::num_pending)
      .def("ff_layer", &Engine::ff_layer)
      .def("ff_unit_lookahead", &Engine::ff_unit_lookahead, py::arg("u"), py::arg("depth") = 1)
      // forward pre-hooks without a Python frame: functools.partial(engine.ff_hook, u, depth)
      // is called by torch as hook(module, args) and returns None
      .def("ff_hook",
           [](Engine& e, int u, int depth, py::object, py::object) {
             if (depth > 0) e.ff_unit_lookahead(u, depth);
             else e.ff_layer(u);
             return py::none();
           })
      .def("ff_join", &Engine::ff_join)
      .def("set_ff_units", &Engine::set_ff_units)
      .def("reset_ff_units", &Engine::reset_ff_units)
      .def("flush", &Engine::flush)
      .def("set_profile", &Engine::set_profile)
      .def("_debug_skip_ready_wait", &Engine::set_debug_skip_ready_wait)
      .def("take_profile", &Engine::take_profile)
      .def("peek_profile", &Engine::peek_profile)
      .def("launch_group", &Engine::launch_now, py::arg("gi"), py::arg("sync") = true)
      .def_property_readonly("launches", &Engine::launches)
      .def_property_readonly("num_groups", &Engine::num_groups);
}
