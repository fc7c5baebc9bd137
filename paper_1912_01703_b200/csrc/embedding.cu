// embedding.cu — deterministic embedding backward:
//   dE[ids[b], :] += dRows[b, :]
// computed as: stable LSD radix sort of (id, position) pairs (single CTA,
// 6-bit digits), then one warp per segment of equal ids summing its rows in
// position order.  No floating-point atomics → bitwise reproducible.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "runtime.h"

namespace be { namespace k {
using namespace be::dev;

namespace {
constexpr int kSortThreads = 256;
constexpr int kDigitBits = 6;
constexpr int kBuckets = 1 << kDigitBits;

// One stable LSD pass: thread t owns the contiguous chunk [t*E, (t+1)*E).
__global__ void __launch_bounds__(kSortThreads) radix_pass(const uint32_t* __restrict__ kin,
                                                          const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
                                                          uint32_t* __restrict__ vout, int n, int shift) {
  pdl_entry();
  extern __shared__ uint32_t cnt[];  // [kBuckets][kSortThreads]
  const int t = threadIdx.x;
  const int E = (n + kSortThreads - 1) / kSortThreads;
  const int lo = min(n, t * E), hi = min(n, lo + E);
  for (int b = 0; b < kBuckets; ++b) cnt[b * kSortThreads + t] = 0;
  for (int i = lo; i < hi; ++i) cnt[((kin[i] >> shift) & (kBuckets - 1)) * kSortThreads + t]++;
  __syncthreads();
  // exclusive scan over the flattened [bucket][thread] array (bucket-major ⇒ stable)
  __shared__ uint32_t part[kSortThreads];
  const int per = kBuckets;  // entries per thread in the flattened order
  uint32_t s = 0;
  for (int j = 0; j < per; ++j) s += cnt[t * per + j];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    uint32_t run = 0;
    for (int j = 0; j < kSortThreads; ++j) { uint32_t v = part[j]; part[j] = run; run += v; }
  }
  __syncthreads();
  uint32_t run = part[t];
  for (int j = 0; j < per; ++j) { uint32_t v = cnt[t * per + j]; cnt[t * per + j] = run; run += v; }
  __syncthreads();
  for (int i = lo; i < hi; ++i) {
    const uint32_t k = kin[i];
    const uint32_t pos = cnt[((k >> shift) & (kBuckets - 1)) * kSortThreads + t]++;
    kout[pos] = k;
    vout[pos] = vin[i];
  }
}

// Whole sort in one CTA's shared memory (n ≤ kSmemSortMax): the same stable
// LSD passes as radix_pass, but keys/positions never leave smem between
// passes — one global read of the ids, one write of the sorted pairs.
constexpr int kSmemSortMax = 10240;
// counter (bucket b, thread t) lives at flattened f = b·T + t, skewed by f/64
// so both access patterns — a warp counting one digit (consecutive t) and a
// thread scanning its 64 consecutive flattened entries — avoid bank conflicts
__device__ __forceinline__ int cidx(int f) { return f + (f >> 6); }
// exclusive scan of one value per thread over the block (256 threads)
__device__ __forceinline__ uint32_t block_exscan(uint32_t v, uint32_t* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t tsum = lane < kSortThreads / 32 ? warp_tot[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, tsum, o);
      if (lane >= o) tsum += y;
    }
    if (lane < kSortThreads / 32) warp_tot[lane] = tsum;  // inclusive warp prefix
  }
  __syncthreads();
  const uint32_t before = w ? warp_tot[w - 1] : 0u;
  return before + x - v;
}
__global__ void __launch_bounds__(kSortThreads) radix_sort_smem(const int32_t* __restrict__ ids,
                                                               uint32_t* __restrict__ out_k,
                                                               uint32_t* __restrict__ out_v, int n, int bits) {
  pdl_entry();
  extern __shared__ uint32_t sm[];
  uint32_t* cnt = sm;                                              // skewed [kBuckets][kSortThreads]
  uint32_t* ka = cnt + kBuckets * kSortThreads + kBuckets * kSortThreads / 64;  // [n]
  uint32_t* va = ka + n;
  uint32_t* kb = va + n;
  uint32_t* vb = kb + n;
  __shared__ uint32_t warp_tot[kSortThreads / 32];
  const int t = threadIdx.x;
  for (int i = t; i < n; i += kSortThreads) { ka[i] = (uint32_t)ids[i]; va[i] = (uint32_t)i; }
  __syncthreads();
  const int E = (n + kSortThreads - 1) / kSortThreads;
  const int lo = min(n, t * E), hi = min(n, lo + E);
  for (int shift = 0; shift < bits; shift += kDigitBits) {
    for (int b = 0; b < kBuckets; ++b) cnt[cidx(b * kSortThreads + t)] = 0;
    for (int i = lo; i < hi; ++i) cnt[cidx(((ka[i] >> shift) & (kBuckets - 1)) * kSortThreads + t)]++;
    __syncthreads();
    uint32_t sacc = 0;
    for (int j = 0; j < kBuckets; ++j) sacc += cnt[cidx(t * kBuckets + j)];
    uint32_t run = block_exscan(sacc, warp_tot);
    for (int j = 0; j < kBuckets; ++j) {
      const int f = cidx(t * kBuckets + j);
      const uint32_t v = cnt[f];
      cnt[f] = run;
      run += v;
    }
    __syncthreads();
    for (int i = lo; i < hi; ++i) {
      const uint32_t k = ka[i];
      const uint32_t pos = cnt[cidx(((k >> shift) & (kBuckets - 1)) * kSortThreads + t)]++;
      kb[pos] = k;
      vb[pos] = va[i];
    }
    __syncthreads();
    uint32_t* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
  for (int i = t; i < n; i += kSortThreads) { out_k[i] = ka[i]; out_v[i] = va[i]; }
}

__global__ void init_pairs(const int32_t* ids, uint32_t* k, uint32_t* v, int n) {
  pdl_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    k[i] = (uint32_t)ids[i];
    v[i] = (uint32_t)i;
  }
}

// one warp per sorted element; segment heads sum their segment in order
__global__ void segment_sum(const uint32_t* keys, const uint32_t* pos, int n, const void* drows, be_dtype dd,
                            int64_t D, float* dtable, float beta) {
  pdl_entry();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  if (warp > 0 && keys[warp - 1] == keys[warp]) return;
  int end = warp + 1;
  while (end < n && keys[end] == keys[warp]) ++end;
  const int64_t row = keys[warp];
  for (int64_t d = lane; d < D; d += 32) {
    float acc = 0.f;
    for (int j = warp; j < end; ++j) acc += ld(drows, (int64_t)pos[j] * D + d, dd);
    float* o = dtable + row * D + d;
    *o = acc + (beta != 0.f ? *o : 0.f);
  }
}
// Sparse SGD (be_sgd_sparse): the same ordered segment sums, applied as the
// update of the touched rows only, p[row] ← p[row] − lr·(scale·Σ g) — no
// gradient table exists (μ = 0, wd = 0: untouched rows are unchanged, exactly
// as dense SGD with a zero gradient row leaves them)
__global__ void segment_sgd(const uint32_t* keys, const uint32_t* pos, int n, const void* drows, be_dtype dd,
                            int64_t D, float* table, float lr, float scale) {
  pdl_entry();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  if (warp > 0 && keys[warp - 1] == keys[warp]) return;
  int end = warp + 1;
  while (end < n && keys[end] == keys[warp]) ++end;
  const int64_t row = keys[warp];
  for (int64_t d = lane; d < D; d += 32) {
    float acc = 0.f;
    for (int j = warp; j < end; ++j) acc += ld(drows, (int64_t)pos[j] * D + d, dd);
    float* o = table + row * D + d;
    *o = __fsub_rn(*o, __fmul_rn(lr, __fmul_rn(scale, acc)));
  }
}
}  // namespace

void embedding_sgd_sorted(const void* drows, be_dtype dd, int64_t B, int64_t D, float* table, float lr, float scale,
                          const void* sorted, cudaStream_t s) {
  if (B == 0) return;
  const uint32_t* k0 = reinterpret_cast<const uint32_t*>(sorted);
  const uint32_t* v0 = k0 + B;
  const int64_t threads = B * 32;
  launch_pdl(segment_sgd, (int)((threads + 255) / 256), 256, 0, s, k0, v0, (int)B, drows, dd, D, table, lr, scale);
  after_launch("embedding_segment_sgd");
}

size_t embedding_bwd_scratch(int64_t B) { return (size_t)B * 16 + 64; }

// Sort phase only: (id, position) pairs sorted by id (stable) into
// sorted[0..B) = ids, sorted[B..2B) = positions.  `scratch` ≥ 16·B bytes; the
// result lives in its first 8·B bytes.
void embedding_sort(const int32_t* ids, int64_t B, int64_t V, void* scratch, cudaStream_t s);

void embedding_bwd(const void* drows, be_dtype dd, const int32_t* ids, int64_t B, int64_t D, float* dtable, int64_t V,
                   float beta, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  BE_REQUIRE(scratch_bytes >= embedding_bwd_scratch(B), BE_E_ARG, "embedding_bwd: scratch too small");
  embedding_sort(ids, B, V, scratch, s);
  embedding_bwd_sorted(drows, dd, B, D, dtable, V, beta, scratch, s);
}

void embedding_bwd_sorted(const void* drows, be_dtype dd, int64_t B, int64_t D, float* dtable, int64_t V, float beta,
                          const void* sorted, cudaStream_t s) {
  if (beta == 0.f) {  // untouched rows get 0
    BE_CHECK_CUDA(cudaMemsetAsync(dtable, 0, sizeof(float) * V * D, s));
    beta = 1.f;        // segments now accumulate onto zeros
  }
  if (B == 0) return;
  const uint32_t* k0 = reinterpret_cast<const uint32_t*>(sorted);
  const uint32_t* v0 = k0 + B;
  const int64_t threads = B * 32;
  launch_pdl(segment_sum, (int)((threads + 255) / 256), 256, 0, s, k0, v0, (int)B, drows, dd, D, dtable, beta);
  after_launch("embedding_segment_sum");
}

void embedding_sort(const int32_t* ids, int64_t B, int64_t V, void* scratch, cudaStream_t s) {
  BE_REQUIRE(B < (1LL << 31), BE_E_SHAPE, "embedding_bwd: batch too large");
  if (B == 0) return;
  uint32_t* k0 = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* v0 = k0 + B;
  uint32_t* k1 = v0 + B;
  uint32_t* v1 = k1 + B;
  if (B <= kSmemSortMax) {
    int bits = 1;
    while ((1LL << bits) < V) ++bits;
    const size_t cwords = (size_t)kBuckets * kSortThreads + (size_t)kBuckets * kSortThreads / 64;
    const size_t smem = sizeof(uint32_t) * (cwords + 4 * (size_t)B);
    static bool sattr = false;
    if (!sattr) {
      BE_CHECK_CUDA(cudaFuncSetAttribute(radix_sort_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(uint32_t) * (cwords + 4 * kSmemSortMax))));
      sattr = true;
    }
    launch_pdl(radix_sort_smem, 1, kSortThreads, smem, s, ids, k0, v0, (int)B, bits);
    after_launch("embedding_radix_sort_smem");
    return;
  }
  init_pairs<<<(int)std::min<int64_t>((B + 255) / 256, 1024), 256, 0, s>>>(ids, k0, v0, (int)B);
  after_launch("embedding_init_pairs");
  int bits = 1;
  while ((1LL << bits) < V) ++bits;
  const size_t smem = sizeof(uint32_t) * kBuckets * kSortThreads;
  static bool attr = false;
  if (!attr) {
    BE_CHECK_CUDA(cudaFuncSetAttribute(radix_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  for (int shift = 0; shift < bits; shift += kDigitBits) {
    launch_pdl(radix_pass, 1, kSortThreads, smem, s, k0, v0, k1, v1, (int)B, shift);
    after_launch("embedding_radix_pass");
    std::swap(k0, k1);
    std::swap(v0, v1);
  }
  uint32_t* base = reinterpret_cast<uint32_t*>(scratch);
  if (k0 != base)  // odd number of passes: result sits in the second half
    BE_CHECK_CUDA(cudaMemcpyAsync(base, k0, sizeof(uint32_t) * 2 * B, cudaMemcpyDeviceToDevice, s));
}

}}  // namespace be::k
