// runtime.cpp — context, errors, caching allocator, tensors/storage and the
// tensor part of the C ABI.
//
// Caching allocator (§5.3): sizes rounded up to 512 B; one
// pool per CUDA stream; a block freed on the host goes back to its stream's
// pool IMMEDIATELY and may be handed to the next allocation on the same
// stream before the GPU finished using it (stream FIFO order makes this
// safe); blocks also used on another stream (record_stream)
// are parked until an event recorded on that stream completes.
// Exact rounded-size reuse, LIFO; on cudaMalloc failure
// empty_cache() and retry once.
#include <execinfo.h>

#include "runtime.h"

#include <cstdio>
#include <cstdlib>
#include <stdexcept>

namespace be {

// ------------------------------------------------------------------ errors
static thread_local std::string t_last_error;

const char* last_error() { return t_last_error.c_str(); }
void set_error(const std::string& m) { t_last_error = m; }
void fail(int code, const std::string& msg) { throw BeException{code, msg}; }

size_t dtype_size(be_dtype d) {
  switch (d) {
    case BE_F32: return 4;
    case BE_F64: return 8;
    case BE_I64: return 8;
    case BE_BOOL: return 1;
    case BE_BF16: return 2;
    case BE_I32: return 4;
    case BE_U8: return 1;
  }
  return 0;
}
const char* dtype_name(be_dtype d) {
  switch (d) {
    case BE_F32: return "f32";
    case BE_F64: return "f64";
    case BE_I64: return "i64";
    case BE_BOOL: return "bool";
    case BE_BF16: return "bf16";
    case BE_I32: return "i32";
    case BE_U8: return "u8";
  }
  return "?";
}

Context& ctx() {
  static Context c;
  return c;
}
static thread_local bool t_grad_enabled = true;
bool grad_enabled() { return t_grad_enabled; }

void after_launch(const char* what) {
  Context& c = ctx();
  c.launches.fetch_add(1, std::memory_order_relaxed);
  if (c.sync_mode) {
    cudaError_t e = cudaStreamSynchronize(c.stream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) fail(BE_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  } else {
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(BE_E_CUDA, std::string(what) + " launch: " + cudaGetErrorString(e));
    }
  }
}

// ------------------------------------------------------------------ profiling
namespace {
struct ProfRec {
  std::string name;
  double flops, bytes;
  int m, n, k;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_ev_pool;
cudaEvent_t take_event() {
  if (!g_ev_pool.empty()) { cudaEvent_t e = g_ev_pool.back(); g_ev_pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

int prof_begin(const char* name, double flops, double bytes, int m, int n, int k, cudaStream_t s) {
  if (!g_prof_on) return -1;
  std::lock_guard<std::mutex> g(g_prof_mu);
  ProfRec r{name, flops, bytes, m, n, k, take_event(), take_event()};
  cudaEventRecord(r.a, s);
  g_prof.push_back(r);
  return (int)g_prof.size() - 1;
}
void prof_end(int idx, cudaStream_t s) {
  if (idx < 0) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  cudaEventRecord(g_prof[idx].b, s);
}

// ------------------------------------------------------------------ autotuning
namespace {
struct TuneState {
  int tried = 0;
  int choice = -1;
  std::vector<cudaEvent_t> ev;  // 2 per variant
};
std::mutex g_tune_mu;
std::unordered_map<std::string, TuneState> g_tune;
// BE_TUNE_FILE=path: decisions already in the file are replayed (no timing),
// new ones are appended — so a profiled run (ncu serialises and replays
// kernels, which distorts the timings) uses the choices of an unprofiled run
const char* tune_file() {
  static const char* f = getenv("BE_TUNE_FILE");
  return f && f[0] ? f : nullptr;
}
void tune_file_load_locked() {
  static bool loaded = false;
  if (loaded || !tune_file()) return;
  loaded = true;
  FILE* fp = fopen(tune_file(), "r");
  if (!fp) return;
  char key[512];
  int v;
  while (fscanf(fp, "%511s %d", key, &v) == 2) g_tune[key].choice = v;
  fclose(fp);
}
}  // namespace

int tune_choose(const std::string& key, int n, int dflt, cudaEvent_t* ev0, cudaEvent_t* ev1) {
  *ev0 = *ev1 = nullptr;
  static const int enabled = [] { const char* e = getenv("BE_TUNE"); return e ? atoi(e) : 1; }();
  if (!enabled || n <= 1) return dflt;
  // round 0 warms each variant up (first-touch allocations, descriptor
  // caches); rounds 1..kRounds are timed; a variant's score is its fastest
  // timed run (robust to a run that shared the GPU with other work)
  constexpr int kRounds = 3;
  std::lock_guard<std::mutex> lk(g_tune_mu);
  tune_file_load_locked();
  TuneState& t = g_tune[key];
  if (t.choice >= 0) return t.choice < n ? t.choice : dflt;
  if (t.tried < (1 + kRounds) * n) {
    const int v = t.tried % n, round = t.tried / n;
    ++t.tried;
    if (round >= 1) {
      t.ev.resize(2 * n * kRounds, nullptr);
      const int i = 2 * ((round - 1) * n + v);
      cudaEventCreate(&t.ev[i]);
      cudaEventCreate(&t.ev[i + 1]);
      *ev0 = t.ev[i];
      *ev1 = t.ev[i + 1];
    }
    return v;
  }
  for (size_t i = 1; i < t.ev.size(); i += 2)
    if (cudaEventQuery(t.ev[i]) != cudaSuccess) { cudaGetLastError(); return dflt; }
  static const bool log = [] { const char* e = getenv("BE_TUNE_LOG"); return e && e[0] == '1'; }();
  float best = 1e30f;
  int bv = dflt;
  std::string msg;
  for (int v = 0; v < n; ++v) {
    float vbest = 1e30f;
    for (int r = 0; r < kRounds; ++r) {
      float ms = 0.f;
      const int i = 2 * (r * n + v);
      cudaEventElapsedTime(&ms, t.ev[i], t.ev[i + 1]);
      vbest = std::min(vbest, ms);
      if (log) msg += (r ? "," : " [") + std::to_string((int)(ms * 1000.f)) + (r == kRounds - 1 ? "]" : "");
    }
    if (vbest < best) { best = vbest; bv = v; }
  }
  if (log) fprintf(stderr, "tune %s ->%d (us)%s\n", key.c_str(), bv, msg.c_str());
  for (cudaEvent_t e : t.ev) cudaEventDestroy(e);
  t.ev.clear();
  t.choice = bv;
  if (tune_file()) {
    if (FILE* fp = fopen(tune_file(), "a")) {
      fprintf(fp, "%s %d\n", key.c_str(), bv);
      fclose(fp);
    }
  }
  return bv;
}

// ------------------------------------------------------------------ allocator
void CachingAllocator::process_deferred_locked() {
  for (size_t i = 0; i < deferred_.size();) {
    bool done = true;
    for (cudaEvent_t e : deferred_[i].events)
      if (cudaEventQuery(e) != cudaSuccess) { done = false; break; }
    if (done) {
      for (cudaEvent_t e : deferred_[i].events) cudaEventDestroy(e);
      Block* b = deferred_[i].b;
      b->extra_streams.clear();
      pools_[b->stream][b->size].push_back(b);
      deferred_[i] = deferred_.back();
      deferred_.pop_back();
    } else {
      ++i;
    }
  }
  cudaGetLastError();  // clear cudaErrorNotReady
}

Block* CachingAllocator::allocate(size_t nbytes, cudaStream_t s) {
  std::lock_guard<std::mutex> g(mu_);
  const size_t sz = round_size(nbytes);
  if (!deferred_.empty()) process_deferred_locked();
  auto& pool = pools_[s];
  auto it = pool.find(sz);
  if (it != pool.end() && !it->second.empty()) {
    Block* b = it->second.back();
    it->second.pop_back();
    b->in_use = true;
    st_.cache_hit_count++;
    st_.bytes_cached -= sz;
    st_.bytes_in_use += sz;
    st_.peak_bytes_in_use = std::max(st_.peak_bytes_in_use, st_.bytes_in_use);
    if (poison) cudaMemsetAsync(b->ptr, 0xFF, sz, s);  // debug: stale data shows as NaN
    return b;
  }
  // A block of this size and stream still waiting on another stream's use
  // (record_stream) is reused in stream order instead of growing the pool:
  // stream s waits on that use's event, no host synchronisation (the host may
  // run ahead of the side streams, so their events are often still pending).
  for (size_t i = 0; i < deferred_.size(); ++i) {
    Block* b = deferred_[i].b;
    if (b->stream != s || b->size != sz) continue;
    for (cudaEvent_t e : deferred_[i].events) {
      cudaStreamWaitEvent(s, e, 0);
      cudaEventDestroy(e);
    }
    b->extra_streams.clear();
    deferred_[i] = deferred_.back();
    deferred_.pop_back();
    b->in_use = true;
    st_.cache_hit_count++;
    st_.bytes_cached -= sz;
    st_.bytes_in_use += sz;
    st_.peak_bytes_in_use = std::max(st_.peak_bytes_in_use, st_.bytes_in_use);
    if (poison) cudaMemsetAsync(b->ptr, 0xFF, sz, s);
    return b;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, sz);
  if (e != cudaSuccess) {
    cudaGetLastError();
    mu_.unlock();
    empty_cache();
    mu_.lock();
    e = cudaMalloc(&p, sz);
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(BE_E_OOM, "out of memory allocating " + std::to_string(sz) + " bytes");
    }
  }
  static const bool trace = getenv("BE_ALLOC_TRACE") != nullptr;
  if (trace) {  // debug: who grows the pool (size, stream, native call stack)
    size_t same_other = 0, defer_same = 0, defer_other = 0;
    for (auto& kv : pools_)
      if (kv.first != s) {
        auto it2 = kv.second.find(sz);
        if (it2 != kv.second.end()) same_other += it2->second.size();
      }
    for (auto& d : deferred_)
      if (d.b->size == sz) (d.b->stream == s ? defer_same : defer_other)++;
    fprintf(stderr, "be raw alloc #%llu: %zu B on stream %p (free on other streams %zu, deferred same-stream %zu, "
            "deferred other %zu, deferred total %zu)\n", (unsigned long long)st_.raw_alloc_count + 1, sz, (void*)s,
            same_other, defer_same, defer_other, deferred_.size());
    void* bt[16];
    backtrace_symbols_fd(bt, backtrace(bt, 16), 2);
  }
  Block* b = new Block();
  b->ptr = p;
  b->size = sz;
  b->stream = s;
  b->in_use = true;
  live_[p] = b;
  st_.raw_alloc_count++;
  st_.bytes_in_use += sz;
  st_.peak_bytes_in_use = std::max(st_.peak_bytes_in_use, st_.bytes_in_use);
  if (poison) cudaMemsetAsync(p, 0xFF, sz, s);
  return b;
}

void CachingAllocator::free(Block* b) {
  std::lock_guard<std::mutex> g(mu_);
  if (!b->in_use) fail(BE_E_DOUBLE_FREE, "double free of allocator block");
  b->in_use = false;
  st_.bytes_in_use -= b->size;
  st_.bytes_cached += b->size;
  if (b->extra_streams.empty()) {
    pools_[b->stream][b->size].push_back(b);  // immediate, CPU-side
  } else {
    Deferred d{b, {}};
    for (cudaStream_t s : b->extra_streams) {
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      cudaEventRecord(ev, s);
      d.events.push_back(ev);
    }
    deferred_.push_back(std::move(d));
  }
}

void CachingAllocator::record_stream(Block* b, cudaStream_t s) {
  std::lock_guard<std::mutex> g(mu_);
  if (s == b->stream) return;
  for (cudaStream_t x : b->extra_streams)
    if (x == s) return;
  b->extra_streams.push_back(s);
}

size_t CachingAllocator::empty_cache() {
  std::lock_guard<std::mutex> g(mu_);
  process_deferred_locked();
  size_t freed = 0;
  bool synced = false;
  for (auto& kv : pools_) {
    for (auto& kv2 : kv.second) {
      for (Block* b : kv2.second) {
        if (!synced) { cudaDeviceSynchronize(); synced = true; }
        cudaFree(b->ptr);
        live_.erase(b->ptr);
        freed += b->size;
        st_.raw_free_count++;
        st_.bytes_cached -= b->size;
        delete b;
      }
      kv2.second.clear();
    }
  }
  return freed;
}

struct be_alloc_stats CachingAllocator::stats() {
  std::lock_guard<std::mutex> g(mu_);
  return st_;
}
void CachingAllocator::reset_peak() {
  std::lock_guard<std::mutex> g(mu_);
  st_.peak_bytes_in_use = st_.bytes_in_use;
}
Block* CachingAllocator::find(void* ptr) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = live_.find(ptr);
  return it == live_.end() ? nullptr : it->second;
}

// ------------------------------------------------------------------ storage/tensor
void Storage::drop() {
  if (refcount.fetch_sub(1, std::memory_order_acq_rel) == 1) {
    if (block) ctx().alloc.free(block);       // back to the stream pool now
    else if (release) release(release_ctx);
    delete this;
  }
}

bool Tensor::is_contiguous() const {
  int64_t expect = 1;
  for (int i = rank - 1; i >= 0; --i) {
    if (shape[i] != 1 && strides[i] != expect) return false;
    expect *= shape[i];
  }
  return true;
}

void tensor_drop(Tensor* t) {
  if (t->refcount.fetch_sub(1, std::memory_order_acq_rel) == 1) {
    if (t->grad) tensor_drop(t->grad);
    if (t->shadow) tensor_drop(t->shadow);
    if (t->bn_stats) tensor_drop(t->bn_stats);
    if (t->mom_block) ctx().alloc.free(t->mom_block);
    if (t->grad_fn) node_drop(t->grad_fn);
    t->storage->drop();
    t->magic = 0;
    delete t;
  }
}

static void contiguous_strides(const int64_t* shape, int rank, int64_t* strides) {
  int64_t s = 1;
  for (int i = rank - 1; i >= 0; --i) { strides[i] = s; s *= shape[i]; }
}

TRef new_tensor(const int64_t* shape, int rank, be_dtype dt) {
  BE_REQUIRE(rank >= 0 && rank <= 6, BE_E_SHAPE, "rank must be in [0, 6]");
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) {
    BE_REQUIRE(shape[i] >= 0, BE_E_SHAPE, "negative dimension");
    n *= shape[i];
  }
  Storage* st = new Storage();
  st->nbytes = (size_t)n * dtype_size(dt);
  st->block = ctx().alloc.allocate(st->nbytes, ctx().stream);
  st->ptr = st->block->ptr;
  Tensor* t = new Tensor();
  t->storage = st;
  t->rank = rank;
  for (int i = 0; i < rank; ++i) t->shape[i] = shape[i];
  contiguous_strides(t->shape, rank, t->strides);
  t->dtype = dt;
  return TRef(t);
}
TRef new_tensor(std::initializer_list<int64_t> shape, be_dtype dt) {
  int64_t s[6];
  int r = 0;
  for (int64_t x : shape) s[r++] = x;
  return new_tensor(s, r, dt);
}
TRef make_view(Tensor* base, const int64_t* shape, int rank, const int64_t* strides, int64_t offset) {
  Tensor* t = new Tensor();
  t->storage = base->storage;
  base->storage->retain();
  t->offset = offset;
  t->rank = rank;
  for (int i = 0; i < rank; ++i) t->shape[i] = shape[i];
  if (strides) for (int i = 0; i < rank; ++i) t->strides[i] = strides[i];
  else contiguous_strides(t->shape, rank, t->strides);
  t->dtype = base->dtype;
  return TRef(t);
}

Tensor* check_handle(be_tensor h) {
  Tensor* t = reinterpret_cast<Tensor*>(h);
  BE_REQUIRE(t != nullptr && t->magic == 0xBE7E5011u, BE_E_BAD_HANDLE, "invalid or freed tensor handle");
  return t;
}

}  // namespace be

// ====================================================================== C ABI
using namespace be;

static void require_init() { BE_REQUIRE(ctx().inited, BE_E_NOT_INIT, "be_init() was not called"); }

extern "C" {

const char* be_last_error(void) { return be::last_error(); }

be_status be_init(int device, uint64_t cuda_stream) {
  BE_API_BEGIN
  Context& c = ctx();
  if (c.inited) {
    BE_REQUIRE(device == c.device, BE_E_ARG, "be_init: already initialised on another device");
    return BE_OK;
  }
  BE_CHECK_CUDA(cudaSetDevice(device));
  c.device = device;
  int sms = 0;
  BE_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  c.num_sms = sms;
  int major = 0;
  BE_CHECK_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  BE_REQUIRE(major == 10, BE_E_UNSUPPORTED, "this library is built for sm_100a (B200) only");
  if (cuda_stream) {
    c.stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    c.own_stream = false;
  } else {
    // highest priority: side streams (overlapped SGD, copies) yield to it
    int least = 0, greatest = 0;
    BE_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    BE_CHECK_CUDA(cudaStreamCreateWithPriority(&c.stream, cudaStreamNonBlocking, greatest));
    c.own_stream = true;
  }
  const char* sm = getenv("BE_SYNC");
  c.sync_mode = sm && sm[0] == '1';
  const char* pz = getenv("BE_ALLOC_POISON");
  c.alloc.poison = pz && pz[0] == '1';
  c.inited = true;
  BE_API_END
}

be_status be_get_stream(uint64_t* out) {
  BE_API_BEGIN
  require_init();
  *out = reinterpret_cast<uint64_t>(ctx().stream);
  BE_API_END
}

be_status be_launch_count(uint64_t* out) {
  BE_API_BEGIN
  *out = ctx().launches.load();
  BE_API_END
}

be_status be_tensor_create(const void* host, const int64_t* shape, int rank, be_dtype dtype, int requires_grad,
                           be_tensor* out) {
  BE_API_BEGIN
  require_init();
  BE_REQUIRE(out != nullptr, BE_E_ARG, "out is NULL");
  BE_REQUIRE(dtype_size(dtype) > 0, BE_E_DTYPE, "unknown dtype");
  BE_REQUIRE(!requires_grad || dtype == BE_F32, BE_E_DTYPE, "requires_grad needs an f32 tensor");
  TRef t = new_tensor(shape, rank, dtype);
  if (host && t->storage->nbytes)
    BE_CHECK_CUDA(cudaMemcpyAsync(t->data(), host, t->storage->nbytes, cudaMemcpyHostToDevice, ctx().stream));
  t->requires_grad = requires_grad != 0;
  *out = reinterpret_cast<be_tensor>(t.release());
  BE_API_END
}

be_status be_tensor_empty(const int64_t* shape, int rank, be_dtype dtype, be_tensor* out) {
  return be_tensor_create(nullptr, shape, rank, dtype, 0, out);
}

be_status be_tensor_from_device(void* dptr, const int64_t* shape, const int64_t* strides, int rank, be_dtype dtype,
                                void (*release)(void*), void* rctx, be_tensor* out) {
  BE_API_BEGIN
  require_init();
  BE_REQUIRE(rank >= 0 && rank <= 6, BE_E_SHAPE, "rank must be in [0, 6]");
  Storage* st = new Storage();
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) n *= shape[i];
  st->ptr = dptr;
  st->nbytes = (size_t)n * dtype_size(dtype);
  st->release = release;
  st->release_ctx = rctx;
  Tensor* t = new Tensor();
  t->storage = st;
  t->rank = rank;
  for (int i = 0; i < rank; ++i) t->shape[i] = shape[i];
  if (strides) for (int i = 0; i < rank; ++i) t->strides[i] = strides[i];
  else contiguous_strides(t->shape, rank, t->strides);
  t->dtype = dtype;
  *out = reinterpret_cast<be_tensor>(t);
  BE_API_END
}

be_status be_tensor_to_host(be_tensor h, void* dst, size_t nbytes) {
  BE_API_BEGIN
  Tensor* t = check_handle(h);
  const size_t es = dtype_size(t->dtype);
  BE_REQUIRE(nbytes >= (size_t)t->numel() * es, BE_E_ARG, "destination too small");
  if (t->is_contiguous()) {
    BE_CHECK_CUDA(cudaMemcpyAsync(dst, t->data(), t->numel() * es, cudaMemcpyDeviceToHost, ctx().stream));
    BE_CHECK_CUDA(cudaStreamSynchronize(ctx().stream));
  } else {
    // stride walk on the host over a copy of the spanned range
    int64_t lo = 0, hi = 0;
    for (int i = 0; i < t->rank; ++i) {
      if (t->shape[i] == 0) { BE_CHECK_CUDA(cudaStreamSynchronize(ctx().stream)); return BE_OK; }
      int64_t ext = (t->shape[i] - 1) * t->strides[i];
      if (ext < 0) lo += ext; else hi += ext;
    }
    std::vector<char> buf((size_t)(hi - lo + 1) * es);
    BE_CHECK_CUDA(cudaMemcpyAsync(buf.data(), (char*)t->data() + lo * (int64_t)es, buf.size(),
                                  cudaMemcpyDeviceToHost, ctx().stream));
    BE_CHECK_CUDA(cudaStreamSynchronize(ctx().stream));
    int64_t idx[6] = {0};
    const int64_t n = t->numel();
    for (int64_t k = 0; k < n; ++k) {
      int64_t off = -lo;
      for (int i = 0; i < t->rank; ++i) off += idx[i] * t->strides[i];
      memcpy((char*)dst + k * es, buf.data() + off * es, es);
      for (int i = t->rank - 1; i >= 0; --i) {
        if (++idx[i] < t->shape[i]) break;
        idx[i] = 0;
      }
    }
  }
  BE_API_END
}

be_status be_tensor_copy_from_host_async(be_tensor h, const void* src, size_t nbytes) {
  BE_API_BEGIN
  Tensor* t = check_handle(h);
  BE_REQUIRE(t->is_contiguous(), BE_E_NONCONTIG, "copy_from_host needs a contiguous tensor");
  BE_REQUIRE(nbytes == (size_t)t->numel() * dtype_size(t->dtype), BE_E_ARG, "size mismatch");
  BE_CHECK_CUDA(cudaMemcpyAsync(t->data(), src, nbytes, cudaMemcpyHostToDevice, ctx().stream));
  t->bump_version();
  BE_API_END
}

be_status be_tensor_copy_to_host_async(be_tensor h, void* dst, size_t nbytes) {
  BE_API_BEGIN
  Tensor* t = check_handle(h);
  BE_REQUIRE(t->is_contiguous(), BE_E_NONCONTIG, "copy_to_host needs a contiguous tensor");
  BE_REQUIRE(nbytes == (size_t)t->numel() * dtype_size(t->dtype), BE_E_ARG, "size mismatch");
  BE_CHECK_CUDA(cudaMemcpyAsync(dst, t->data(), nbytes, cudaMemcpyDeviceToHost, ctx().stream));
  BE_API_END
}

be_status be_tensor_info(be_tensor h, int* rank, int64_t* shape, int64_t* strides, be_dtype* dtype,
                         uint64_t* device_ptr) {
  BE_API_BEGIN
  Tensor* t = check_handle(h);
  if (rank) *rank = t->rank;
  for (int i = 0; i < t->rank; ++i) {
    if (shape) shape[i] = t->shape[i];
    if (strides) strides[i] = t->strides[i];
  }
  if (dtype) *dtype = t->dtype;
  if (device_ptr) *device_ptr = reinterpret_cast<uint64_t>(t->data());
  BE_API_END
}

be_status be_tensor_version(be_tensor h, uint64_t* out) {
  BE_API_BEGIN
  *out = check_handle(h)->version();
  BE_API_END
}

be_status be_tensor_requires_grad(be_tensor h, int* out) {
  BE_API_BEGIN
  *out = check_handle(h)->requires_grad ? 1 : 0;
  BE_API_END
}

be_status be_retain(be_tensor h) {
  BE_API_BEGIN
  check_handle(h)->retain();
  BE_API_END
}

be_status be_release(be_tensor h) {
  BE_API_BEGIN
  Tensor* t = reinterpret_cast<Tensor*>(h);
  BE_REQUIRE(t != nullptr, BE_E_BAD_HANDLE, "NULL handle");
  BE_REQUIRE(t->magic == 0xBE7E5011u, BE_E_DOUBLE_FREE, "tensor handle already released");
  tensor_drop(t);
  BE_API_END
}

be_status be_set_grad_enabled(int on) {
  t_grad_enabled = on != 0;
  return BE_OK;
}
be_status be_is_grad_enabled(int* out) {
  *out = t_grad_enabled ? 1 : 0;
  return BE_OK;
}
be_status be_set_compute_dtype(be_dtype d) {
  BE_API_BEGIN
  BE_REQUIRE(d == BE_F32 || d == BE_BF16, BE_E_UNSUPPORTED, "compute dtype must be f32 or bf16");
  ctx().compute = d;
  BE_API_END
}

be_status be_synchronize(void) {
  BE_API_BEGIN
  require_init();
  BE_CHECK_CUDA(cudaStreamSynchronize(ctx().stream));
  if (ctx().comm_stream) BE_CHECK_CUDA(cudaStreamSynchronize(ctx().comm_stream));
  BE_CHECK_CUDA(cudaGetLastError());
  BE_API_END
}

be_status be_item(be_tensor h, double* out) {
  BE_API_BEGIN
  Tensor* t = check_handle(h);
  BE_REQUIRE(t->numel() == 1, BE_E_SHAPE, "item() needs a 1-element tensor");
  char buf[8] = {0};
  BE_CHECK_CUDA(cudaMemcpyAsync(buf, t->data(), dtype_size(t->dtype), cudaMemcpyDeviceToHost, ctx().stream));
  BE_CHECK_CUDA(cudaStreamSynchronize(ctx().stream));
  switch (t->dtype) {
    case BE_F32: *out = *reinterpret_cast<float*>(buf); break;
    case BE_F64: *out = *reinterpret_cast<double*>(buf); break;
    case BE_I32: *out = *reinterpret_cast<int32_t*>(buf); break;
    case BE_I64: *out = (double)*reinterpret_cast<int64_t*>(buf); break;
    case BE_BF16: { uint32_t u = (uint32_t)(*reinterpret_cast<uint16_t*>(buf)) << 16; float f; memcpy(&f, &u, 4); *out = f; break; }
    default: *out = (double)(uint8_t)buf[0];
  }
  BE_API_END
}

static cudaStream_t as_stream(uint64_t s) { return s ? reinterpret_cast<cudaStream_t>(s) : ctx().stream; }

be_status be_stream_create(uint64_t* out) {
  BE_API_BEGIN
  require_init();
  cudaStream_t s;
  BE_CHECK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = reinterpret_cast<uint64_t>(s);
  BE_API_END
}
be_status be_stream_destroy(uint64_t s) {
  BE_API_BEGIN
  BE_REQUIRE(s != 0, BE_E_ARG, "cannot destroy the compute stream");
  BE_CHECK_CUDA(cudaStreamDestroy(reinterpret_cast<cudaStream_t>(s)));
  BE_API_END
}
be_status be_event_create(uint64_t* out) {
  BE_API_BEGIN
  cudaEvent_t e;
  BE_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  *out = reinterpret_cast<uint64_t>(e);
  BE_API_END
}
be_status be_event_destroy(uint64_t e) {
  BE_API_BEGIN
  BE_CHECK_CUDA(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(e)));
  BE_API_END
}
be_status be_event_record(uint64_t e, uint64_t s) {
  BE_API_BEGIN
  require_init();
  BE_CHECK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(e), as_stream(s)));
  BE_API_END
}
be_status be_stream_wait_event(uint64_t s, uint64_t e) {
  BE_API_BEGIN
  require_init();
  BE_CHECK_CUDA(cudaStreamWaitEvent(as_stream(s), reinterpret_cast<cudaEvent_t>(e), 0));
  BE_API_END
}
be_status be_tensor_copy_from_host_on(be_tensor h, const void* src, size_t nbytes, uint64_t s) {
  BE_API_BEGIN
  Tensor* t = check_handle(h);
  BE_REQUIRE(t->is_contiguous(), BE_E_NONCONTIG, "copy_from_host needs a contiguous tensor");
  BE_REQUIRE(nbytes == (size_t)t->numel() * dtype_size(t->dtype), BE_E_ARG, "size mismatch");
  BE_CHECK_CUDA(cudaMemcpyAsync(t->data(), src, nbytes, cudaMemcpyHostToDevice, as_stream(s)));
  t->bump_version();
  BE_API_END
}

be_status be_prof_enable(int on) {
  BE_API_BEGIN
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
  BE_API_END
}

be_status be_prof_read(be_prof_rec* out, int cap, int* n_out) {
  BE_API_BEGIN
  require_init();
  BE_CHECK_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> g(g_prof_mu);
  int n = 0;
  for (ProfRec& r : g_prof) {
    if (n < cap && out) {
      be_prof_rec& o = out[n];
      memset(&o, 0, sizeof(o));
      strncpy(o.name, r.name.c_str(), sizeof(o.name) - 1);
      o.flops = r.flops;
      o.bytes = r.bytes;
      o.m = r.m; o.n = r.n; o.k = r.k;
      cudaEventElapsedTime(&o.ms, r.a, r.b);
      cudaEventElapsedTime(&o.t_start_ms, g_prof.front().a, r.a);
    }
    ++n;
    g_ev_pool.push_back(r.a);
    g_ev_pool.push_back(r.b);
  }
  g_prof.clear();
  if (n_out) *n_out = std::min(n, cap);
  BE_API_END
}

be_status be_alloc_stats(struct be_alloc_stats* out) {
  BE_API_BEGIN
  *out = ctx().alloc.stats();
  BE_API_END
}
be_status be_alloc_reset_peak(void) {
  BE_API_BEGIN
  ctx().alloc.reset_peak();
  BE_API_END
}
be_status be_empty_cache(uint64_t* released) {
  BE_API_BEGIN
  size_t r = ctx().alloc.empty_cache();
  if (released) *released = r;
  BE_API_END
}
uint64_t be_round_size(uint64_t nbytes) { return CachingAllocator::round_size(nbytes); }

be_status be_record_stream(be_tensor h, uint64_t stream) {
  BE_API_BEGIN
  Tensor* t = check_handle(h);
  if (t->storage->block) ctx().alloc.record_stream(t->storage->block, reinterpret_cast<cudaStream_t>(stream));
  BE_API_END
}
be_status be_raw_alloc(uint64_t nbytes, uint64_t stream, uint64_t* dptr) {
  BE_API_BEGIN
  require_init();
  cudaStream_t s = stream ? reinterpret_cast<cudaStream_t>(stream) : ctx().stream;
  Block* b = ctx().alloc.allocate(nbytes, s);
  *dptr = reinterpret_cast<uint64_t>(b->ptr);
  BE_API_END
}
be_status be_raw_free(uint64_t dptr) {
  BE_API_BEGIN
  Block* b = ctx().alloc.find(reinterpret_cast<void*>(dptr));
  BE_REQUIRE(b != nullptr, BE_E_BAD_HANDLE, "unknown pointer");
  ctx().alloc.free(b);
  BE_API_END
}

}  // extern "C"
