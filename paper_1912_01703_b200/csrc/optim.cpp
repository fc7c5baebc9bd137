// optim.cpp — SGD: the fused multi-tensor
// step after backward (be_sgd_step), and the overlapped variant
// (be_sgd_overlap) that updates each parameter as soon as its gradient is
// final, on a side stream, while the rest of backward runs on the compute
// stream — the "optimizer step in the backward pass" pattern.  Both launch
// the same kernel on the same per-parameter values, so the updated
// parameters are bitwise identical (tests/test_gpu_runtime.py).
//
// Update (oracle/optim.py):
//   g' = scale·g + wd·p;  v ← μ·v + g' (v₁ = g');  p ← p − lr·v  (μ = 0: p ← p − lr·g')
// and the bf16 shadow of p is rewritten in the same pass (mixed precision).
#include "ops_common.h"

namespace be {
std::vector<Tensor*>& sparse_tables();
namespace {

k::SgdEntry sgd_entry(Tensor* p, float momentum, cudaStream_t s) {
  k::SgdEntry e{};
  e.p = p->ptr<float>();
  e.g = p->grad->ptr<float>();
  e.n = p->numel();
  if (momentum != 0.f) {
    if (!p->mom_block) {
      p->mom_block = ctx().alloc.allocate(sizeof(float) * std::max<int64_t>(1, e.n), s);
      p->mom = reinterpret_cast<float*>(p->mom_block->ptr);
      k::fill(p->mom, e.n, BE_F32, 0.0, s);  // v0 = 0 ⇒ v1 = g'
    }
    e.mom = p->mom;
  }
  // keep the bf16 shadow in lock-step when it exists (mixed precision)
  if (p->shadow && p->shadow_version == p->version()) e.shadow = p->shadow->ptr<uint16_t>();
  return e;
}

void bump_after_update(Tensor* p, const k::SgdEntry& e) {
  p->bump_version();
  if (e.shadow) { p->shadow->bump_version(); p->shadow_version = p->version(); }
}

// ---------------------------------------------------------------- overlapped SGD state
struct Overlap {
  bool active = false;
  float lr = 0.f, momentum = 0.f, wd = 0.f;
  std::vector<Tensor*> params;          // one ref each
  std::vector<Tensor*> group;           // final grads not yet launched
  int64_t group_numel = 0;
  bool launched = false;                // any update enqueued this backward
  cudaEvent_t done = nullptr;
  std::vector<cudaEvent_t> ready_pool;  // compute-stream "grad final" events
  size_t ready_used = 0;
};
Overlap& ov() {
  static Overlap o;
  return o;
}
// a group is launched once it holds this many parameters (or at the end of
// backward): fewer, larger launches keep the host ahead of the GPU
constexpr int64_t kGroupNumel = 1 << 21;

void launch_group_on(const std::vector<Tensor*>& ps, cudaStream_t s, float scale) {
  Overlap& o = ov();
  std::vector<k::SgdEntry> es;
  es.reserve(ps.size());
  for (Tensor* p : ps) {
    if (!p->grad) continue;
    es.push_back(sgd_entry(p, o.momentum, s));
  }
  if (es.empty()) return;
  // full-width grid: measured on B200 (tools/timeline.py, C2), a 1-block-per-SM
  // update co-resident with the backward GEMMs slows them ~2.7× (both stream
  // through L2), so the update takes the machine briefly instead
  k::sgd_multi(es.data(), (int)es.size(), o.lr, o.momentum, o.wd, scale, s);
  size_t j = 0;
  for (Tensor* p : ps)
    if (p->grad) bump_after_update(p, es[j++]);
  o.launched = true;
}

void flush_group() {
  Overlap& o = ov();
  if (o.group.empty()) return;
  Context& c = ctx();
  if (o.ready_used == o.ready_pool.size()) {
    cudaEvent_t e;
    BE_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    o.ready_pool.push_back(e);
  }
  cudaEvent_t ev = o.ready_pool[o.ready_used++];
  BE_CHECK_CUDA(cudaEventRecord(ev, c.stream));
  BE_CHECK_CUDA(cudaStreamWaitEvent(c.opt_stream, ev, 0));
  launch_group_on(o.group, c.opt_stream, 1.f);
  o.group.clear();
  o.group_numel = 0;
}
}  // namespace

std::vector<Tensor*>& sparse_tables() {
  static std::vector<Tensor*> t;
  return t;
}

// a registered table whose gradient arrived densely (e.g. looked up twice in
// one step): the same update p -= lr·g from that gradient, on the compute stream
void opt_sparse_dense_fallback(Tensor* leaf) {
  if (!leaf->grad) return;
  BE_REQUIRE(!ddp_active() || ddp_world() == 1, BE_E_UNSUPPORTED,
             "sgd_sparse: a table with several lookups per step under DDP (its dense gradient is not exchanged)");
  k::SgdEntry e{};
  e.p = leaf->ptr<float>();
  e.g = leaf->grad->ptr<float>();
  e.n = leaf->numel();
  k::sgd_multi(&e, 1, leaf->sparse_lr, 0.f, 0.f, 1.f, ctx().stream);
  leaf->bump_version();
  tensor_drop(leaf->grad);
  leaf->grad = nullptr;
}

bool opt_active() { return ov().active; }
bool opt_hparams(float* lr, float* mu, float* wd) {
  const Overlap& o = ov();
  *lr = o.lr; *mu = o.momentum; *wd = o.wd;
  return o.active;
}
bool opt_param(const Tensor* leaf) { return ov().active && leaf->opt_slot >= 0; }

void opt_on_grad_final(Tensor* leaf) {
  Overlap& o = ov();
  if (!o.active || leaf->opt_slot < 0 || !leaf->grad) return;
  o.group.push_back(leaf);
  o.group_numel += leaf->numel();
  if (o.group_numel >= kGroupNumel) flush_group();
}

bool opt_fuse_desc(Tensor* p, k::SgdFuse* f) {
  static const bool on = [] { const char* e = getenv("BE_FUSE_SGD"); return !(e && e[0] == '0'); }();
  Overlap& o = ov();
  if (!on || !o.active || p->opt_slot < 0 || p->grad) return false;
  cudaStream_t s = ctx().stream;
  *f = k::SgdFuse{};
  f->p = p->ptr<float>();
  if (o.momentum != 0.f) {
    if (!p->mom_block) {
      p->mom_block = ctx().alloc.allocate(sizeof(float) * std::max<int64_t>(1, p->numel()), s);
      p->mom = reinterpret_cast<float*>(p->mom_block->ptr);
      k::fill(p->mom, p->numel(), BE_F32, 0.0, s);  // v0 = 0 ⇒ v1 = g'
    }
    f->v = p->mom;
  }
  if (p->shadow && p->shadow_version == p->version()) f->shadow = p->shadow->ptr<uint16_t>();
  f->lr = o.lr; f->mu = o.momentum; f->wd = o.wd; f->scale = 1.f;
  return true;
}

void opt_fused_done(Tensor* p) {
  const bool sh = p->shadow && p->shadow_version == p->version();
  p->bump_version();
  if (sh) { p->shadow->bump_version(); p->shadow_version = p->version(); }
}

void opt_launch_params(const std::vector<Tensor*>& ps, cudaStream_t s, float scale) {
  std::vector<Tensor*> mine;
  for (Tensor* p : ps)
    if (p->opt_slot >= 0) mine.push_back(p);
  launch_group_on(mine, s, scale);
}

void opt_end_backward() {
  Overlap& o = ov();
  if (!o.active) return;
  Context& c = ctx();
  if (ddp_active()) {
    ddp_wait_all();  // stragglers reduced (+ updated on the comm stream); compute waits on every bucket
  } else {
    flush_group();
    if (o.launched) {
      BE_CHECK_CUDA(cudaEventRecord(o.done, c.opt_stream));
      BE_CHECK_CUDA(cudaStreamWaitEvent(c.stream, o.done, 0));
    }
  }
  o.launched = false;
  o.ready_used = 0;
}

}  // namespace be

using namespace be;
extern "C" {

be_status be_sgd_step(const be_tensor* params, int n, float lr, float momentum, float weight_decay) {
  BE_API_BEGIN
  std::vector<k::SgdEntry> es;
  es.reserve(n);
  std::vector<Tensor*> ts;
  for (int i = 0; i < n; ++i) {
    Tensor* p = check_handle(params[i]);
    BE_REQUIRE(p->dtype == BE_F32 && p->is_contiguous(), BE_E_DTYPE, "sgd: params must be contiguous f32");
    BE_REQUIRE(!opt_param(p) && !opt_sparse(p), BE_E_ARG, "sgd: parameter " + std::to_string(i) +
                                           " is registered for overlapped / sparse SGD (updated during backward)");
    BE_REQUIRE(p->grad != nullptr, BE_E_MISSING_GRAD, "sgd: parameter " + std::to_string(i) + " has no grad");
    es.push_back(sgd_entry(p, momentum, ctx().stream));
    ts.push_back(p);
  }
  if (ddp_active()) ddp_wait_all();
  // DDP buckets already hold the mean gradient (ncclAvg): scale 1
  k::sgd_multi(es.data(), (int)es.size(), lr, momentum, weight_decay, 1.f, ctx().stream);
  for (size_t i = 0; i < ts.size(); ++i) bump_after_update(ts[i], es[i]);
  BE_API_END
}

be_status be_sgd_momentum(be_tensor param, be_tensor* out) {
  BE_API_BEGIN
  Tensor* p = check_handle(param);
  BE_REQUIRE(out != nullptr, BE_E_ARG, "sgd_momentum: out is NULL");
  *out = nullptr;
  if (!p->mom) return BE_OK;
  TRef v = new_tensor(p->shape, p->rank, BE_F32);
  BE_CHECK_CUDA(cudaMemcpyAsync(v->data(), p->mom, sizeof(float) * p->numel(), cudaMemcpyDeviceToDevice,
                                ctx().stream));
  *out = reinterpret_cast<be_tensor>(v.release());
  BE_API_END
}

be_status be_sgd_sparse(const be_tensor* tables, int n, float lr) {
  BE_API_BEGIN
  BE_REQUIRE(ctx().inited, BE_E_NOT_INIT, "be_init() was not called");
  std::vector<Tensor*>& reg = sparse_tables();
  for (Tensor* p : reg) { p->sparse_lr = -1.f; tensor_drop(p); }
  reg.clear();
  BE_REQUIRE(lr >= 0.f, BE_E_ARG, "sgd_sparse: lr must be >= 0");
  for (int i = 0; i < n; ++i) {
    Tensor* p = check_handle(tables[i]);
    BE_REQUIRE(p->dtype == BE_F32 && p->rank == 2 && p->is_contiguous() && p->requires_grad && p->is_leaf(),
               BE_E_ARG, "sgd_sparse: tables must be contiguous f32 [V, D] leaves requiring grad");
    BE_REQUIRE(p->opt_slot < 0 && p->ddp_slot < 0, BE_E_ARG,
               "sgd_sparse: a table cannot also be registered for overlapped SGD or attached to DDP");
    BE_REQUIRE(!opt_sparse(p), BE_E_ARG, "sgd_sparse: table listed twice");
    p->retain();
    p->sparse_lr = lr;
    reg.push_back(p);
  }
  BE_API_END
}

be_status be_sgd_overlap(const be_tensor* params, int n, float lr, float momentum, float weight_decay) {
  BE_API_BEGIN
  Overlap& o = ov();
  Context& c = ctx();
  BE_REQUIRE(c.inited, BE_E_NOT_INIT, "be_init() was not called");
  for (Tensor* p : o.params) { p->opt_slot = -1; tensor_drop(p); }
  o.params.clear();
  o.group.clear();
  o.group_numel = 0;
  o.active = false;
  if (n == 0) return BE_OK;  // detach
  for (int i = 0; i < n; ++i) {
    Tensor* p = check_handle(params[i]);
    BE_REQUIRE(p->dtype == BE_F32 && p->is_contiguous() && p->requires_grad && p->is_leaf(), BE_E_ARG,
               "sgd_overlap: params must be contiguous f32 leaves requiring grad");
    BE_REQUIRE(p->opt_slot < 0, BE_E_ARG, "sgd_overlap: parameter listed twice");
    BE_REQUIRE(!ddp_active() || p->ddp_slot >= 0, BE_E_ARG,
               "sgd_overlap: with DDP attached every registered parameter must be DDP-attached");
    p->retain();
    p->opt_slot = i;
    o.params.push_back(p);
  }
  if (!c.opt_stream) {
    // lowest priority: when a GEMM and an update both have blocks pending,
    // the compute stream's go first
    int least = 0, greatest = 0;
    BE_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    BE_CHECK_CUDA(cudaStreamCreateWithPriority(&c.opt_stream, cudaStreamNonBlocking, least));
  }
  if (!o.done) BE_CHECK_CUDA(cudaEventCreateWithFlags(&o.done, cudaEventDisableTiming));
  o.lr = lr; o.momentum = momentum; o.wd = weight_decay;
  o.active = true;
  BE_API_END
}

}  // extern "C"
