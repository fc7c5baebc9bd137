// runtime.h — internal C++ runtime of the be_* library (not part of the ABI).
// Tensor/Storage, caching allocator,
// tape nodes, global context (one device, one compute
// stream).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/be.h"

namespace be {

// ------------------------------------------------------------------ errors
struct BeException {
  int code;
  std::string msg;
};
void set_error(const std::string& m);
const char* last_error();

#define BE_API_BEGIN try {
#define BE_API_END                                      \
  return BE_OK;                                         \
  }                                                     \
  catch (const ::be::BeException& e) {                  \
    ::be::set_error(e.msg);                             \
    return e.code;                                      \
  }                                                     \
  catch (const std::exception& e) {                     \
    ::be::set_error(e.what());                          \
    return BE_E_ARG;                                    \
  }
[[noreturn]] void fail(int code, const std::string& msg);

#define BE_CHECK_CUDA(expr)                                                         \
  do {                                                                              \
    cudaError_t e__ = (expr);                                                       \
    if (e__ != cudaSuccess)                                                         \
      ::be::fail(BE_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__));   \
  } while (0)
#define BE_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) ::be::fail((code), (msg)); \
  } while (0)

size_t dtype_size(be_dtype d);
const char* dtype_name(be_dtype d);

// ------------------------------------------------------------------ allocator
struct Block {
  void* ptr = nullptr;
  size_t size = 0;               // rounded
  cudaStream_t stream = nullptr; // home stream (pool)
  std::vector<cudaStream_t> extra_streams;
  bool in_use = false;
};

class CachingAllocator {
 public:
  static constexpr size_t kQuantum = 512;
  static size_t round_size(size_t n) { return ((n == 0 ? 1 : n) + kQuantum - 1) / kQuantum * kQuantum; }
  Block* allocate(size_t nbytes, cudaStream_t s);
  void free(Block* b);
  void record_stream(Block* b, cudaStream_t s);
  size_t empty_cache();
  struct be_alloc_stats stats();
  void reset_peak();
  Block* find(void* ptr);
  bool poison = false;

 private:
  void process_deferred_locked();
  std::mutex mu_;
  // pool per stream: rounded size -> LIFO list (exact-size reuse)
  std::unordered_map<cudaStream_t, std::unordered_map<size_t, std::vector<Block*>>> pools_;
  struct Deferred { Block* b; std::vector<cudaEvent_t> events; };
  std::vector<Deferred> deferred_;
  std::unordered_map<void*, Block*> live_;
  struct be_alloc_stats st_{};
};

// ------------------------------------------------------------------ storage/tensor
struct Storage {
  std::atomic<int> refcount{1};
  void* ptr = nullptr;
  size_t nbytes = 0;
  Block* block = nullptr;              // null for external
  void (*release)(void*) = nullptr;    // external deleter
  void* release_ctx = nullptr;
  std::atomic<uint64_t> version{0};
  void retain() { refcount.fetch_add(1, std::memory_order_relaxed); }
  void drop();
};

struct Node;
void node_retain(Node* n);
void node_drop(Node* n);

struct Tensor {
  uint32_t magic = 0xBE7E5011u;
  std::atomic<int> refcount{1};
  Storage* storage = nullptr;
  int64_t offset = 0;  // elements
  int rank = 0;
  int64_t shape[6] = {0};
  int64_t strides[6] = {0};
  be_dtype dtype = BE_F32;
  bool requires_grad = false;
  Node* grad_fn = nullptr;  // strong
  int output_nr = 0;
  Tensor* grad = nullptr;   // strong (leaves)
  // bf16 shadow of an fp32 parameter (mixed precision; SGD refreshes it)
  Tensor* shadow = nullptr;
  uint64_t shadow_version = ~0ull;
  float* mom = nullptr;       // SGD momentum buffer (fp32), owned
  Block* mom_block = nullptr;
  int ddp_slot = -1;          // index in DDP param table
  int opt_slot = -1;          // index in the overlapped-SGD table
  float sparse_lr = -1.f;     // >= 0: embedding table updated on its touched rows inside backward (be_sgd_sparse)
  // per-channel Σ / Σx² partials of this tensor's values, produced by the
  // epilogue of the conv that wrote it (be_conv_attrs.bn_stats); valid while
  // the version is unchanged — batchnorm2d then skips its statistics pass
  Tensor* bn_stats = nullptr;
  int bn_stats_parts = 0;
  uint64_t bn_stats_version = ~0ull;
  // engine scratch for leaves (per backward pass): edges still to run into
  // this leaf (overlapped SGD / DDP readiness), and whether some already ran
  uint64_t bw_epoch = 0;
  int bw_uses = 0;
  bool bw_partial = false;

  int64_t numel() const {
    int64_t n = 1;
    for (int i = 0; i < rank; ++i) n *= shape[i];
    return n;
  }
  bool is_contiguous() const;
  void* data() const { return (char*)storage->ptr + offset * dtype_size(dtype); }
  template <class T> T* ptr() const { return reinterpret_cast<T*>(data()); }
  bool is_leaf() const { return grad_fn == nullptr; }
  uint64_t version() const { return storage->version.load(); }
  void bump_version() { storage->version.fetch_add(1); }
  void retain() { refcount.fetch_add(1, std::memory_order_relaxed); }
};
void tensor_drop(Tensor* t);

// Strong-reference smart pointer for internal use.
struct TRef {
  Tensor* t = nullptr;
  TRef() = default;
  explicit TRef(Tensor* x, bool adopt = true) : t(x) { if (t && !adopt) t->retain(); }
  TRef(const TRef& o) : t(o.t) { if (t) t->retain(); }
  TRef(TRef&& o) noexcept : t(o.t) { o.t = nullptr; }
  TRef& operator=(TRef o) { std::swap(t, o.t); return *this; }
  ~TRef() { if (t) tensor_drop(t); }
  Tensor* operator->() const { return t; }
  Tensor* get() const { return t; }
  Tensor* release() { Tensor* x = t; t = nullptr; return x; }
  explicit operator bool() const { return t != nullptr; }
};

TRef new_tensor(const int64_t* shape, int rank, be_dtype dt);
TRef new_tensor(std::initializer_list<int64_t> shape, be_dtype dt);
TRef make_view(Tensor* base, const int64_t* shape, int rank, const int64_t* strides, int64_t offset);
Tensor* check_handle(be_tensor h);

// ------------------------------------------------------------------ tape
struct SavedVar {
  Storage* storage = nullptr;  // strong (never the Tensor: avoids output→node cycles)
  int64_t offset = 0;
  int rank = 0;
  int64_t shape[6]{}, strides[6]{};
  be_dtype dtype = BE_F32;
  uint64_t version = 0;
  bool defined = false;
};

struct Edge {
  enum Kind { NONE, NODE, LEAF } kind = NONE;
  Node* node = nullptr;   // strong (NODE)
  int output_nr = 0;
  Tensor* leaf = nullptr; // strong (LEAF)
};

struct GradSink;
namespace k { struct SgdFuse; }
using VjpFn = void (*)(Node* n, GradSink& sink);

struct OutMeta {
  int rank = 0;
  int64_t shape[6]{};
  be_dtype dtype = BE_F32;
};

struct Node {
  std::atomic<int> refcount{1};
  const char* name = "";
  int op = 0;
  uint64_t seq = 0;
  VjpFn vjp = nullptr;
  std::vector<Edge> edges;          // one per differentiable input
  std::vector<SavedVar> saved;
  std::vector<OutMeta> outs;
  alignas(8) unsigned char attrs[64]{};
  int64_t iattr[8]{};
  bool consumed = false;
  bool upstream_is_ones = false;    // set by the engine for the root
  // engine scratch of the backward pass `bw_epoch` (reset when first reached)
  uint64_t bw_epoch = 0;
  int bw_deps = 0;
  std::vector<Tensor*> pend;        // pending output gradients (owned refs)
};

// The engine hands each VJP a sink: grads for input i are written into
// sink.dest(i) (allocated on demand with beta=0, or the existing buffer with
// beta=1 to accumulate); kernels that cannot accumulate call dest_fresh().
// All engine callbacks are plain member functions over the engine state of
// the running backward (no per-node closures: host enqueue cost).
struct Engine;
struct GradSink {
  Node* node = nullptr;
  Engine* eng = nullptr;
  std::vector<Tensor*> upstream;    // per output (borrowed)
  // returns nullptr when input i needs no grad
  Tensor* dest(int i, float* beta);
  Tensor* dest_fresh(int i);        // always zero-initialised fresh buffer semantics: caller writes all
  void commit(int i);               // finish: adds fresh buffers, notifies DDP for leaves
  // hand over an exclusively-owned tensor as input i's gradient (adopted
  // without a copy when nothing is pending yet, else accumulated)
  void give(int i, TRef t);
  bool needs(int i) const;
  bool upstream_ones() const { return node->upstream_is_ones; }
  bool retain = false;
  // Fused SGD (overlapped optimizer): true when input i is a parameter
  // registered with be_sgd_overlap whose gradient is complete with this one
  // contribution; *f then describes the update the VJP's weight-gradient GEMM
  // applies in its epilogue (no gradient tensor is stored), after which the
  // VJP calls fused(i).  Every reader of the parameter in this VJP must be
  // enqueued before that GEMM.
  bool fuse(int i, k::SgdFuse* f);
  void fused(int i);
  // Sparse SGD (be_sgd_sparse): true when input i is an embedding table
  // registered for the touched-rows update whose gradient is complete with this
  // one contribution; the VJP applies p[row] -= lr·g_row itself (no gradient
  // tensor) and then calls fused_sparse(i)
  bool fuse_sparse(int i, float* lr);
  void fused_sparse(int i);
  Tensor* leaf(int i) const { return node->edges[i].kind == Edge::LEAF ? node->edges[i].leaf : nullptr; }
  // engine internals
  struct Slot { Tensor* target = nullptr; Tensor* tmp = nullptr; bool acc = false; bool used = false; };
  std::vector<Slot> slots;
  Tensor* acquire(int i, bool* existing);
  bool adopt(int i, Tensor* t);
  void finalize(int i, Tensor* t);
};

Tensor* unpack(Node* n, int i, TRef& holder);   // version-checked view of saved[i]
void save(Node* n, Tensor* t);
void release_saved(Node* n);

// ------------------------------------------------------------------ context
struct Context {
  bool inited = false;
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t comm_stream = nullptr;
  cudaStream_t opt_stream = nullptr;   // overlapped SGD
  cudaStream_t sort_stream = nullptr;  // embedding id sorts issued at forward time
  cudaEvent_t sort_done = nullptr;     // re-recorded after every sort (the stream is in order)
  be_dtype compute = BE_F32;
  bool sync_mode = false;
  CachingAllocator alloc;
  std::atomic<uint64_t> seq{0};
  std::atomic<uint64_t> launches{0};
  uint64_t bw_epoch = 0;               // id of the current / last backward pass
};
Context& ctx();
bool grad_enabled();
// On-line variant autotuning (cudnn.benchmark-style, no synchronisation):
// the first n calls for `key` run variants 0..n-1 (warm-up), the next 3n
// run them again bracketed by events (returned in *ev0/*ev1, to be recorded
// around the launch by the caller); once all those events have completed,
// the variant with the fastest single timed run is returned for every later
// call.  BE_TUNE=0 pins variant `dflt`.
int tune_choose(const std::string& key, int n_variants, int dflt, cudaEvent_t* ev0, cudaEvent_t* ev1);
// GEMM launch profiling (be_prof_enable): returns a record index or -1
int prof_begin(const char* name, double flops, double bytes, int m, int n, int k, cudaStream_t s);
void prof_end(int idx, cudaStream_t s);
void after_launch(const char* what);   // counts + BE_SYNC + error check

// DDP hook (dist.cpp)
void ddp_on_leaf_grad_ready(Tensor* leaf);
bool ddp_active();
Tensor* ddp_grad_view(Tensor* leaf);     // bucket view for a param grad or nullptr
void ddp_wait_all();                     // compute stream waits on all bucket allreduces
int ddp_world();
void ddp_begin_backward();
// DDP: params of a reduced bucket (for the overlapped optimizer, launched on
// the comm stream right after the bucket's allreduce)
void opt_launch_params(const std::vector<Tensor*>& ps, cudaStream_t s, float scale);

// Overlapped SGD (optim.cpp; be_sgd_overlap): the engine reports each
// registered parameter whose gradient is final; its update runs on a side
// stream while backward continues.
bool opt_active();
bool opt_hparams(float* lr, float* mu, float* wd);  // the overlapped update's hyper-parameters
bool opt_param(const Tensor* leaf);      // registered for overlapped SGD
void opt_on_grad_final(Tensor* leaf);    // (non-DDP) grad complete for this backward
void opt_end_backward();                 // flush; compute stream waits for every update
bool opt_fuse_desc(Tensor* leaf, k::SgdFuse* f);  // fill the update-epilogue descriptor (BE_FUSE_SGD=0: off)
void opt_fused_done(Tensor* leaf);       // versions after the fused update was enqueued
// Sparse (touched-rows) SGD of embedding tables (be_sgd_sparse): μ = 0, wd = 0,
// applied by the embedding backward itself; a table whose gradient arrives
// densely instead (several lookups) is updated from it when final.
inline bool opt_sparse(const Tensor* leaf) { return leaf->sparse_lr >= 0.f; }
void opt_sparse_dense_fallback(Tensor* leaf);
// DDP: all-gather `bytes` from every rank into dst (rank-major) on stream s
void ddp_allgather(const void* src, void* dst, size_t bytes, cudaStream_t s);

}  // namespace be
