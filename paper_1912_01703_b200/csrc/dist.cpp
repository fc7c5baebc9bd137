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

#include "ops_common.h"

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
// Peer-memory mode (be_p2p_attach / be_p2p_connect): buckets reduced by the
// fused allreduce + SGD kernel of p2p.cu over CUDA-IPC mappings of every
// rank's buckets, parameters and bf16 shadows instead of ncclAllReduce.
struct P2P {
  bool on = false, connected = false;
  std::vector<void*> exported;          // local allocation bases, in export order
  std::vector<void*> opened;            // IPC mappings of the peers' allocations
  Block* ctl = nullptr;                 // flags [nb][2][R] u64, counters [nb] u32, status i32
  Block* tables = nullptr;              // device pointer tables of every bucket
  std::vector<k::P2PBucketArgs> args;   // per bucket (device table pointers filled in)
  std::vector<unsigned long long> epoch;
  int blocks = 32;
};
struct DDP {
  P2P p2p;
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

void launch_bucket_p2p(Bucket& b) {
  DDP& d = ddp();
  Context& c = ctx();
  const int bi = (int)(&b - d.buckets.data());
  k::P2PBucketArgs a = d.p2p.args[bi];
  a.epoch = ++d.p2p.epoch[bi];
  float lr = 0.f, mu = 0.f, wd = 0.f;
  bool sgd = opt_hparams(&lr, &mu, &wd);
  for (int i : b.params) sgd = sgd && opt_param(d.params[i]);
  a.lr_on = sgd ? 1 : 0;
  a.lr = lr; a.mu = mu; a.wd = wd;
  k::p2p_allreduce_sgd(a, d.p2p.blocks, c.comm_stream);
  if (sgd) {
    // every rank's copy of these parameters (and shadows) was rewritten
    for (int i : b.params) {
      Tensor* p = d.params[i];
      const bool sh = p->shadow && p->shadow_version == p->version();
      p->bump_version();
      if (sh) { p->shadow->bump_version(); p->shadow_version = p->version(); }
    }
  }
}

void launch_bucket(Bucket& b) {
  DDP& d = ddp();
  Context& c = ctx();
  BE_CHECK_CUDA(cudaEventRecord(b.ready, c.stream));
  BE_CHECK_CUDA(cudaStreamWaitEvent(c.comm_stream, b.ready, 0));
  if (d.p2p.on) {
    launch_bucket_p2p(b);
    BE_CHECK_CUDA(cudaEventRecord(b.done, c.comm_stream));
    b.launched = true;
    d.allreduce_calls++;
    return;
  }
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

}  // extern "C"

namespace be {
namespace {
// Bucket the registered parameters (shared by the NCCL and the peer-memory
// modes).  broadcast: parameters start identical by an ncclBroadcast from
// rank 0 (the NCCL mode); the peer-memory mode requires identical initial
// parameters from the caller.
void attach_common(const be_tensor* params, int n, size_t bucket_bytes, bool broadcast) {
  DDP& d = ddp();
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
      if (broadcast) {
        BE_CHECK_NCCL(nccl().broadcast(p->data(), p->data(), (size_t)p->numel(), ncclFloat, 0, d.comm, c.stream));
        p->bump_version();
      }
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
}

constexpr uint32_t kP2PMagic = 0x32504542;  // "BEP2"
struct P2PHeader { uint32_t magic, rank, world, count; };
}  // namespace
}  // namespace be

extern "C" {

be_status be_ddp_attach(const be_tensor* params, int n, size_t bucket_bytes) {
  BE_API_BEGIN
  DDP& d = ddp();
  BE_REQUIRE(d.comm_ready, BE_E_NOT_INIT, "be_dist_init() was not called");
  attach_common(params, n, bucket_bytes, true);
  d.active = true;
  BE_API_END
}

be_status be_p2p_attach(const be_tensor* params, int n, size_t bucket_bytes, int rank, int world, void* blob,
                        size_t cap, size_t* blob_bytes) {
  BE_API_BEGIN
  Context& c = ctx();
  BE_REQUIRE(c.inited, BE_E_NOT_INIT, "be_init() was not called");
  BE_REQUIRE(world >= 1 && rank >= 0 && rank < world, BE_E_ARG, "p2p_attach: bad rank/world");
  DDP& d = ddp();
  BE_REQUIRE(!d.comm_ready || (d.rank == rank && d.world == world), BE_E_ARG,
             "p2p_attach: rank/world differ from be_dist_init's");
  attach_common(params, n, bucket_bytes, false);
  d.rank = rank;
  d.world = world;
  P2P& q = d.p2p;
  q = P2P();
  q.on = true;
  if (!c.comm_stream) BE_CHECK_CUDA(cudaStreamCreateWithFlags(&c.comm_stream, cudaStreamNonBlocking));
  const int nb = (int)d.buckets.size();
  // control block: flags [nb][2][world] u64, counters [nb] u32, status i32
  const size_t ctl_bytes = (size_t)nb * 2 * world * 8 + (size_t)nb * 4 + 16;
  q.ctl = c.alloc.allocate(ctl_bytes, c.stream);
  BE_CHECK_CUDA(cudaMemsetAsync(q.ctl->ptr, 0, ctl_bytes, c.stream));
  // bf16 shadows exist from the start (the kernel rewrites every rank's) and
  // the momentum buffers live with the parameters (be_sgd_momentum reads them)
  for (Tensor* p : d.params) {
    if (c.compute == BE_BF16) weight_operand(p);
    if (!p->mom_block) {
      p->mom_block = c.alloc.allocate(sizeof(float) * std::max<int64_t>(1, p->numel()), c.stream);
      p->mom = reinterpret_cast<float*>(p->mom_block->ptr);
      k::fill(p->mom, p->numel(), BE_F32, 0.0, c.stream);
    }
  }
  // export order: control block, buckets, params, shadows
  q.exported.push_back(q.ctl->ptr);
  for (Bucket& b : d.buckets) q.exported.push_back(b.storage->ptr);
  for (Tensor* p : d.params) {
    BE_REQUIRE(p->offset == 0 && p->storage->block && p->storage->ptr == p->storage->block->ptr, BE_E_ARG,
               "p2p_attach: parameters must own their allocation (not views)");
    q.exported.push_back(p->data());
  }
  for (Tensor* p : d.params) q.exported.push_back(p->shadow ? p->shadow->data() : nullptr);
  const size_t need = sizeof(P2PHeader) + q.exported.size() * sizeof(cudaIpcMemHandle_t);
  *blob_bytes = need;
  BE_CHECK_CUDA(cudaStreamSynchronize(c.stream));
  if (blob && cap >= need) {
    P2PHeader h{kP2PMagic, (uint32_t)rank, (uint32_t)world, (uint32_t)q.exported.size()};
    memcpy(blob, &h, sizeof(h));
    cudaIpcMemHandle_t* hs = reinterpret_cast<cudaIpcMemHandle_t*>(reinterpret_cast<char*>(blob) + sizeof(h));
    for (size_t i = 0; i < q.exported.size(); ++i) {
      memset(&hs[i], 0, sizeof(hs[i]));
      if (q.exported[i] && world > 1) BE_CHECK_CUDA(cudaIpcGetMemHandle(&hs[i], q.exported[i]));
    }
  }
  BE_API_END
}

// all: world blobs of blob_bytes each, rank-major (an all-gather of every
// rank's be_p2p_attach output, done by the caller over any transport)
be_status be_p2p_connect(const void* all, size_t blob_bytes) {
  BE_API_BEGIN
  DDP& d = ddp();
  P2P& q = d.p2p;
  Context& c = ctx();
  BE_REQUIRE(q.on && !q.connected, BE_E_ARG, "p2p_connect: call be_p2p_attach first (once)");
  const int R = d.world, me = d.rank, nb = (int)d.buckets.size(), n = (int)d.params.size();
  const size_t cnt = q.exported.size();
  BE_REQUIRE(blob_bytes == sizeof(P2PHeader) + cnt * sizeof(cudaIpcMemHandle_t), BE_E_ARG,
             "p2p_connect: blob size does not match this rank's (different models?)");
  // ptr[r][i]: allocation i of rank r mapped into this process
  std::vector<std::vector<char*>> ptr(R, std::vector<char*>(cnt, nullptr));
  for (int r = 0; r < R; ++r) {
    const char* b = reinterpret_cast<const char*>(all) + (size_t)r * blob_bytes;
    P2PHeader h;
    memcpy(&h, b, sizeof(h));
    BE_REQUIRE(h.magic == kP2PMagic && (int)h.rank == r && (int)h.world == R && h.count == cnt, BE_E_ARG,
               "p2p_connect: blob " + std::to_string(r) + " is not rank " + std::to_string(r) + "'s");
    const cudaIpcMemHandle_t* hs = reinterpret_cast<const cudaIpcMemHandle_t*>(b + sizeof(h));
    for (size_t i = 0; i < cnt; ++i) {
      if (r == me) { ptr[r][i] = reinterpret_cast<char*>(q.exported[i]); continue; }
      if (!q.exported[i]) continue;  // no shadow (f32 mode) on any rank
      void* m = nullptr;
      BE_CHECK_CUDA(cudaIpcOpenMemHandle(&m, hs[i], cudaIpcMemLazyEnablePeerAccess));
      q.opened.push_back(m);
      ptr[r][i] = reinterpret_cast<char*>(m);
    }
  }
  // device tables: per bucket seg_off, seg_n [nseg] i64; grad [R]; p, shadow [nseg·R]; mom [nseg];
  // flags_peer, flags_peer_done [R]
  std::vector<std::vector<int>> segs(nb);
  for (int b = 0; b < nb; ++b) segs[b] = d.buckets[b].params;  // ascending offsets
  size_t words = 0;
  for (int b = 0; b < nb; ++b) {
    const size_t ns = segs[b].size();
    words += 2 * ns + R + 2 * ns * R + ns + 2 * R;
  }
  std::vector<uint64_t> host(std::max<size_t>(words, 1));
  q.tables = c.alloc.allocate(host.size() * 8, c.stream);
  uint64_t* dbase = reinterpret_cast<uint64_t*>(q.tables->ptr);
  size_t w = 0;
  const size_t flags_per_bucket = 2 * (size_t)R;
  q.args.assign(nb, k::P2PBucketArgs());
  q.epoch.assign(nb, 0);
  for (int b = 0; b < nb; ++b) {
    const std::vector<int>& sg = segs[b];
    const int ns = (int)sg.size();
    k::P2PBucketArgs& a = q.args[b];
    a.rank = me; a.world = R; a.numel = (int64_t)d.buckets[b].numel; a.nseg = ns;
    auto take = [&](size_t k2) { uint64_t* p = dbase + w; w += k2; return p; };
    uint64_t* so = take(ns); uint64_t* sn = take(ns);
    for (int j = 0; j < ns; ++j) {
      host[(so - dbase) + j] = (uint64_t)d.offset_of[sg[j]];
      host[(sn - dbase) + j] = (uint64_t)d.params[sg[j]]->numel();
    }
    a.seg_off = reinterpret_cast<const int64_t*>(so);
    a.seg_n = reinterpret_cast<const int64_t*>(sn);
    uint64_t* gr = take(R);
    for (int r = 0; r < R; ++r) host[(gr - dbase) + r] = (uint64_t)(uintptr_t)ptr[r][1 + b];
    a.grad = reinterpret_cast<float* const*>(gr);
    uint64_t* pp = take((size_t)ns * R);
    uint64_t* sp = take((size_t)ns * R);
    bool any_shadow = false;
    for (int j = 0; j < ns; ++j)
      for (int r = 0; r < R; ++r) {
        host[(pp - dbase) + (size_t)j * R + r] = (uint64_t)(uintptr_t)ptr[r][1 + nb + sg[j]];
        char* shp = ptr[r][1 + nb + n + sg[j]];
        host[(sp - dbase) + (size_t)j * R + r] = (uint64_t)(uintptr_t)shp;
        any_shadow |= shp != nullptr;
      }
    a.p = reinterpret_cast<float* const*>(pp);
    a.shadow = any_shadow ? reinterpret_cast<uint16_t* const*>(sp) : nullptr;
    uint64_t* mp = take(ns);
    for (int j = 0; j < ns; ++j) host[(mp - dbase) + j] = (uint64_t)(uintptr_t)d.params[sg[j]]->mom;
    a.mom = reinterpret_cast<float* const*>(mp);
    uint64_t* fp = take(R);
    uint64_t* fd = take(R);
    for (int r = 0; r < R; ++r) {
      unsigned long long* fl = reinterpret_cast<unsigned long long*>(ptr[r][0]) + (size_t)b * flags_per_bucket;
      host[(fp - dbase) + r] = (uint64_t)(uintptr_t)fl;
      host[(fd - dbase) + r] = (uint64_t)(uintptr_t)(fl + R);
    }
    a.flags_peer = reinterpret_cast<unsigned long long* const*>(fp);
    a.flags_peer_done = reinterpret_cast<unsigned long long* const*>(fd);
    unsigned long long* lf = reinterpret_cast<unsigned long long*>(q.ctl->ptr) + (size_t)b * flags_per_bucket;
    a.flags_arrive = lf;
    a.flags_done = lf + R;
    a.counter = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(q.ctl->ptr) + (size_t)nb * flags_per_bucket * 8) + b;
    a.status = reinterpret_cast<int*>(reinterpret_cast<char*>(q.ctl->ptr) + (size_t)nb * flags_per_bucket * 8 +
                                      (size_t)nb * 4);
  }
  BE_CHECK_CUDA(cudaMemcpyAsync(dbase, host.data(), host.size() * 8, cudaMemcpyHostToDevice, c.stream));
  BE_CHECK_CUDA(cudaStreamSynchronize(c.stream));
  q.connected = true;
  d.active = true;
  BE_API_END
}

// 0 = healthy; 1 = a peer barrier timed out (10 s) in some bucket kernel
be_status be_p2p_status(int* status) {
  BE_API_BEGIN
  DDP& d = ddp();
  *status = 0;
  if (!d.p2p.on || !d.p2p.ctl) return BE_OK;
  const int nb = (int)d.buckets.size();
  const char* st = reinterpret_cast<const char*>(d.p2p.ctl->ptr) + (size_t)nb * 2 * d.world * 8 + (size_t)nb * 4;
  BE_CHECK_CUDA(cudaDeviceSynchronize());
  BE_CHECK_CUDA(cudaMemcpy(status, st, sizeof(int), cudaMemcpyDeviceToHost));
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
  if (d.p2p.on) {
    for (void* m : d.p2p.opened) cudaIpcCloseMemHandle(m);
    if (d.p2p.ctl) ctx().alloc.free(d.p2p.ctl);
    if (d.p2p.tables) ctx().alloc.free(d.p2p.tables);
    d.p2p = P2P();
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
