// dist.cpp — data parallelism: NCCL communicator and bucketed gradient
// allreduce overlapped with backward (§5.4 "synchronize
// gradients using all-reduce style primitives").
//
// One process per GPU.  Parameters are broadcast from rank 0 at attach.
// Leaf gradients are VIEWS into flat fp32 buckets (~bucket_bytes each, in
// reverse registration order, i.e. the order backward produces them), so no
// gradient is ever copied.  When the last gradient of a bucket lands (the
// engine's leaf-finalize hook), the compute stream records an event, the comm
// stream waits on it and runs ncclAllReduce(avg) on the bucket — concurrently
// with the remaining backward kernels.  The bucket therefore holds the MEAN
// gradient (g = (1/R)·Σ_r g_r), so a second backward before
// the step (gradient accumulation) adds its local gradient to an identical
// mean on every rank and its re-reduction gives mean(g1) + mean(g2).  The end
// of every backward makes the compute stream wait for every bucket, so
// gradients read after be_backward are reduced.  Replicas stay bitwise
// identical because every rank applies the same reduced bytes.
//
// NCCL is resolved with dlopen (the torch-bundled libnccl.so.2 that
// torch.distributed already loaded), so the library has no link-time NCCL
// dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <vector>

#include "kernels.h"
#include "runtime.h"

namespace be {
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  const char* env = getenv("BE_NCCL_LIB");
  const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    if (!nm) continue;
    api.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
    if (!api.h) api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  BE_REQUIRE(api.h != nullptr, BE_E_NCCL, "cannot dlopen libnccl.so.2 (import torch.distributed first or set BE_NCCL_LIB)");
  api.getUniqueId = (decltype(api.getUniqueId))dlsym(api.h, "ncclGetUniqueId");
  api.commInitRank = (decltype(api.commInitRank))dlsym(api.h, "ncclCommInitRank");
  api.allReduce = (decltype(api.allReduce))dlsym(api.h, "ncclAllReduce");
  api.broadcast = (decltype(api.broadcast))dlsym(api.h, "ncclBroadcast");
  api.getErrorString = (decltype(api.getErrorString))dlsym(api.h, "ncclGetErrorString");
  api.commDestroy = (decltype(api.commDestroy))dlsym(api.h, "ncclCommDestroy");
  api.commCount = (decltype(api.commCount))dlsym(api.h, "ncclCommCount");
  api.allGather = (decltype(api.allGather))dlsym(api.h, "ncclAllGather");
  BE_REQUIRE(api.getUniqueId && api.commInitRank && api.allReduce && api.broadcast, BE_E_NCCL,
             "libnccl is missing required symbols");
  return api;
}
#define BE_CHECK_NCCL(expr)                                                                            \
  do {                                                                                                 \
    ncclResult_t r__ = (expr);                                                                         \
    if (r__ != ncclSuccess)                                                                            \
      ::be::fail(BE_E_NCCL, std::string(#expr) + ": " +                                                \
                                (nccl().getErrorString ? nccl().getErrorString(r__) : "nccl error")); \
  } while (0)

struct Bucket {
  Storage* storage = nullptr;  // flat fp32 buffer (DDP holds one ref)
  size_t numel = 0;
  std::vector<int> params;
  int pending = 0;
  bool launched = false;
  cudaEvent_t ready = nullptr, done = nullptr;
};
struct DDP {
  bool comm_ready = false;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  bool active = false;
  std::vector<Tensor*> params;
  std::vector<int> bucket_of;
  std::vector<size_t> offset_of;
  std::vector<char> ready;
  std::vector<Bucket> buckets;
  uint64_t allreduce_calls = 0;
};
DDP& ddp() {
  static DDP d;
  return d;
}

void launch_bucket(Bucket& b) {
  DDP& d = ddp();
  Context& c = ctx();
  BE_CHECK_CUDA(cudaEventRecord(b.ready, c.stream));
  BE_CHECK_CUDA(cudaStreamWaitEvent(c.comm_stream, b.ready, 0));
  BE_CHECK_NCCL(nccl().allReduce(b.storage->ptr, b.storage->ptr, b.numel, ncclFloat, ncclAvg, d.comm, c.comm_stream));
  if (opt_active()) {
    // overlapped SGD: the bucket's parameters are updated on the comm stream
    // right behind their allreduce
    std::vector<Tensor*> ps;
    for (int i : b.params)
      if (d.ready[i]) ps.push_back(d.params[i]);
    opt_launch_params(ps, c.comm_stream, 1.f);
  }
  BE_CHECK_CUDA(cudaEventRecord(b.done, c.comm_stream));
  b.launched = true;
  d.allreduce_calls++;
}
// Bucket plan: reverse registration order, 64-element aligned offsets, a new
// bucket once the current one reaches bucket_bytes of fp32.
void plan_buckets(const int64_t* numels, int n, size_t bucket_bytes, int* bucket_of, int64_t* offset_of,
                  int64_t* bucket_numel, int cap, int* n_buckets) {
  if (bucket_bytes == 0) bucket_bytes = 25u << 20;
  int nb = 0;
  int64_t cur = 0;
  bool open = false;
  for (int i = n - 1; i >= 0; --i) {
    const int64_t aligned = (cur + 63) / 64 * 64;
    offset_of[i] = aligned;
    bucket_of[i] = nb;
    cur = aligned + numels[i];
    open = true;
    if ((size_t)cur * 4 >= bucket_bytes) {
      BE_REQUIRE(nb < cap, BE_E_ARG, "ddp_plan: bucket capacity exceeded");
      bucket_numel[nb++] = cur;
      cur = 0;
      open = false;
    }
  }
  if (open) {
    BE_REQUIRE(nb < cap, BE_E_ARG, "ddp_plan: bucket capacity exceeded");
    bucket_numel[nb++] = cur;
  }
  *n_buckets = nb;
}
}  // namespace

bool ddp_active() { return ddp().active; }
int ddp_world() { return ddp().world; }

Tensor* ddp_grad_view(Tensor* leaf) {
  DDP& d = ddp();
  if (!d.active || leaf->ddp_slot < 0) return nullptr;
  const int slot = leaf->ddp_slot;
  Bucket& b = d.buckets[d.bucket_of[slot]];
  Tensor* t = new Tensor();
  t->storage = b.storage;
  b.storage->retain();
  t->offset = (int64_t)d.offset_of[slot];
  t->rank = leaf->rank;
  int64_t st = 1;
  for (int i = leaf->rank - 1; i >= 0; --i) { t->shape[i] = leaf->shape[i]; t->strides[i] = st; st *= leaf->shape[i]; }
  t->dtype = BE_F32;
  return t;
}

void ddp_begin_backward() {
  DDP& d = ddp();
  for (Bucket& b : d.buckets) { b.pending = (int)b.params.size(); b.launched = false; }
  std::fill(d.ready.begin(), d.ready.end(), 0);
}

void ddp_on_leaf_grad_ready(Tensor* leaf) {
  DDP& d = ddp();
  if (leaf->ddp_slot < 0) return;
  const int slot = leaf->ddp_slot;
  Bucket& b = d.buckets[d.bucket_of[slot]];
  if (d.ready[slot]) {
    BE_REQUIRE(!b.launched, BE_E_ARG, "DDP: a parameter received another gradient after its bucket was reduced");
    return;
  }
  d.ready[slot] = 1;
  if (--b.pending == 0) launch_bucket(b);
}

void ddp_allgather(const void* src, void* dst, size_t bytes, cudaStream_t s) {
  DDP& d = ddp();
  BE_REQUIRE(d.comm_ready && nccl().allGather, BE_E_NCCL, "allgather: no communicator");
  BE_CHECK_NCCL(nccl().allGather(src, dst, bytes, ncclChar, d.comm, s));
}

void ddp_wait_all() {
  DDP& d = ddp();
  for (Bucket& b : d.buckets) {
    if (!b.launched) {
      bool any = false;
      for (int p : b.params) any |= d.ready[p] != 0;
      if (!any) continue;
      launch_bucket(b);  // some params got no gradient this step: reduce what exists
    }
    BE_CHECK_CUDA(cudaStreamWaitEvent(ctx().stream, b.done, 0));
  }
}

}  // namespace be

using namespace be;
extern "C" {

be_status be_dist_unique_id(void* out128) {
  BE_API_BEGIN
  ncclUniqueId id;
  BE_CHECK_NCCL(nccl().getUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, sizeof(id));
  BE_API_END
}

be_status be_dist_init(int rank, int world, const void* id128) {
  BE_API_BEGIN
  BE_REQUIRE(ctx().inited, BE_E_NOT_INIT, "be_init() was not called");
  DDP& d = ddp();
  BE_REQUIRE(!d.comm_ready, BE_E_ARG, "be_dist_init called twice");
  BE_REQUIRE(world >= 1 && rank >= 0 && rank < world, BE_E_ARG, "bad rank/world");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  BE_CHECK_NCCL(nccl().commInitRank(&d.comm, world, id, rank));
  d.rank = rank;
  d.world = world;
  d.comm_ready = true;
  if (!ctx().comm_stream) BE_CHECK_CUDA(cudaStreamCreateWithFlags(&ctx().comm_stream, cudaStreamNonBlocking));
  BE_API_END
}

be_status be_ddp_attach(const be_tensor* params, int n, size_t bucket_bytes) {
  BE_API_BEGIN
  DDP& d = ddp();
  BE_REQUIRE(d.comm_ready, BE_E_NOT_INIT, "be_dist_init() was not called");
  BE_REQUIRE(!d.active, BE_E_ARG, "DDP already attached");
  if (bucket_bytes == 0) bucket_bytes = 25u << 20;
  Context& c = ctx();
  d.params.clear();
  // validate everything first so a failed attach leaves no parameter marked
  for (int i = 0; i < n; ++i) {
    Tensor* p = check_handle(params[i]);
    BE_REQUIRE(p->dtype == BE_F32 && p->is_contiguous() && p->requires_grad, BE_E_ARG,
               "DDP params must be contiguous f32 leaves requiring grad");
    BE_REQUIRE(p->ddp_slot < 0, BE_E_ARG, "parameter listed twice");
    for (int j = 0; j < i; ++j)
      BE_REQUIRE(params[j] != params[i], BE_E_ARG, "parameter listed twice");
  }
  for (int i = 0; i < n; ++i) {
    Tensor* p = check_handle(params[i]);
    p->retain();
    p->ddp_slot = i;
    d.params.push_back(p);
  }
  try {
    for (Tensor* p : d.params) {
      // replicas start identical: broadcast from rank 0
      BE_CHECK_NCCL(nccl().broadcast(p->data(), p->data(), (size_t)p->numel(), ncclFloat, 0, d.comm, c.stream));
      p->bump_version();
      if (p->grad) { tensor_drop(p->grad); p->grad = nullptr; }
    }
  } catch (...) {
    for (Tensor* p : d.params) { p->ddp_slot = -1; tensor_drop(p); }
    d.params.clear();
    throw;
  }
  d.bucket_of.assign(n, -1);
  d.offset_of.assign(n, 0);
  d.ready.assign(n, 0);
  d.buckets.clear();
  {
    std::vector<int64_t> numels(n), offs(n), bnum(n + 1);
    std::vector<int> bof(n);
    for (int i = 0; i < n; ++i) numels[i] = d.params[i]->numel();
    int nb = 0;
    plan_buckets(numels.data(), n, bucket_bytes, bof.data(), offs.data(), bnum.data(), n + 1, &nb);
    d.buckets.resize(nb);
    for (int b = 0; b < nb; ++b) d.buckets[b].numel = (size_t)bnum[b];
    for (int i = n - 1; i >= 0; --i) {  // params listed in the order gradients arrive
      d.bucket_of[i] = bof[i];
      d.offset_of[i] = (size_t)offs[i];
      d.buckets[bof[i]].params.push_back(i);
    }
  }
  for (Bucket& b : d.buckets) {
    Storage* st = new Storage();
    st->nbytes = std::max<size_t>(b.numel, 1) * 4;
    st->block = c.alloc.allocate(st->nbytes, c.stream);
    st->ptr = st->block->ptr;
    b.storage = st;
    BE_CHECK_CUDA(cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming));
    BE_CHECK_CUDA(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming));
  }
  d.active = true;
  BE_API_END
}

be_status be_ddp_detach(void) {
  BE_API_BEGIN
  DDP& d = ddp();
  if (!d.active) return BE_OK;
  BE_CHECK_CUDA(cudaStreamSynchronize(ctx().stream));
  if (ctx().comm_stream) BE_CHECK_CUDA(cudaStreamSynchronize(ctx().comm_stream));
  for (Tensor* p : d.params) {
    if (p->grad) { tensor_drop(p->grad); p->grad = nullptr; }
    p->ddp_slot = -1;
    tensor_drop(p);
  }
  for (Bucket& b : d.buckets) {
    b.storage->drop();
    cudaEventDestroy(b.ready);
    cudaEventDestroy(b.done);
  }
  d.buckets.clear();
  d.params.clear();
  d.active = false;
  BE_API_END
}

be_status be_ddp_sync_buffers(const be_tensor* bufs, int n) {
  BE_API_BEGIN
  DDP& d = ddp();
  BE_REQUIRE(d.comm_ready, BE_E_NOT_INIT, "be_dist_init() was not called");
  for (int i = 0; i < n; ++i) {
    Tensor* t = check_handle(bufs[i]);
    BE_REQUIRE(t->dtype == BE_F32 && t->is_contiguous(), BE_E_ARG, "ddp_sync_buffers: contiguous f32 buffers");
    BE_CHECK_NCCL(nccl().broadcast(t->data(), t->data(), (size_t)t->numel(), ncclFloat, 0, d.comm, ctx().stream));
    t->bump_version();
  }
  BE_API_END
}

be_status be_dist_world(int* rank, int* world) {
  BE_API_BEGIN
  DDP& d = ddp();
  BE_REQUIRE(d.comm_ready, BE_E_NOT_INIT, "be_dist_init() was not called");
  *rank = d.rank;
  *world = d.world;
  if (nccl().commCount) {  // the communicator's own rank count, not the argument we passed
    int nr = 0;
    BE_CHECK_NCCL(nccl().commCount(d.comm, &nr));
    *world = nr;
  }
  BE_API_END
}

be_status be_ddp_plan(const int64_t* numels, int n, size_t bucket_bytes, int* bucket_of, int64_t* offset_of,
                      int64_t* bucket_numel, int cap, int* n_buckets) {
  BE_API_BEGIN
  BE_REQUIRE(n >= 0 && numels && bucket_of && offset_of && bucket_numel && n_buckets, BE_E_ARG, "ddp_plan: bad args");
  plan_buckets(numels, n, bucket_bytes, bucket_of, offset_of, bucket_numel, cap, n_buckets);
  BE_API_END
}

be_status be_allreduce_(be_tensor h) {
  BE_API_BEGIN
  DDP& d = ddp();
  BE_REQUIRE(d.comm_ready, BE_E_NOT_INIT, "be_dist_init() was not called");
  Tensor* t = check_handle(h);
  BE_REQUIRE(t->is_contiguous(), BE_E_NONCONTIG, "allreduce needs a contiguous tensor");
  ncclDataType_t dt = t->dtype == BE_F32 ? ncclFloat : t->dtype == BE_BF16 ? ncclBfloat16 : ncclInt32;
  BE_REQUIRE(t->dtype == BE_F32 || t->dtype == BE_BF16 || t->dtype == BE_I32, BE_E_DTYPE, "allreduce dtype");
  BE_CHECK_NCCL(nccl().allReduce(t->data(), t->data(), (size_t)t->numel(), dt, ncclSum, d.comm, ctx().stream));
  t->bump_version();
  BE_API_END
}

}  // extern "C"
