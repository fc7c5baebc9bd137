// pointwise.cu — memory-bound kernels of the hot path: elementwise ops with
// 128-bit vector I/O, deterministic column / full reductions (warp shuffles,
// fixed-order combination), fused softmax-cross-entropy, BCE, and the fused
// multi-tensor SGD.  All grids are sized in multiples of the SM count.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "sgd_math.cuh"
#include "kernels.h"
#include "runtime.h"

namespace be { namespace k {
using namespace be::dev;

namespace {
int ew_grid(int64_t n, int per_thread = 8) {
  int64_t blocks = (n + 256LL * per_thread - 1) / (256LL * per_thread);
  int64_t cap = (int64_t)ctx().num_sms * 8;
  return (int)std::max<int64_t>(1, std::min(blocks, cap));
}

// Generic vectorised unary/binary elementwise: op(i, a, b, y) on 8 lanes.
template <typename F>
__global__ void ew_kernel(int64_t n, bool vec, F f) {
  pdl_entry();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    const int64_t n8 = n / 8;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += stride) f.vec(i * 8);
    for (int64_t i = n8 * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) f.one(i);
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) f.one(i);
  }
}
template <typename F>
void launch_ew(int64_t n, bool vec, F f, cudaStream_t s, const char* name) {
  if (n <= 0) return;
  launch_pdl(ew_kernel<F>, ew_grid(n), 256, 0, s, n, vec, f);
  after_launch(name);
}

struct FillF {
  void* x; be_dtype dt; float v; int64_t iv;
  __device__ void one(int64_t i) const {
    if (dt == BE_I32) reinterpret_cast<int32_t*>(x)[i] = (int32_t)iv;
    else if (dt == BE_I64) reinterpret_cast<int64_t*>(x)[i] = iv;
    else if (dt == BE_U8 || dt == BE_BOOL) reinterpret_cast<uint8_t*>(x)[i] = (uint8_t)iv;
    else st(x, i, dt, v);
  }
  __device__ void vec(int64_t i) const { for (int j = 0; j < 8; ++j) one(i + j); }
};
struct CastF {
  const void* x; be_dtype xd; void* y; be_dtype yd;
  __device__ float get(int64_t i) const {
    if (xd == BE_I32) return (float)reinterpret_cast<const int32_t*>(x)[i];
    return ld(x, i, xd);
  }
  __device__ void one(int64_t i) const {
    float v = get(i);
    if (yd == BE_I32) reinterpret_cast<int32_t*>(y)[i] = (int32_t)v;
    else st(y, i, yd, v);
  }
  __device__ void vec(int64_t i) const {
    if ((xd == BE_F32 || xd == BE_BF16) && (yd == BE_F32 || yd == BE_BF16)) st8(y, i, yd, ld8(x, i, xd));
    else for (int j = 0; j < 8; ++j) one(i + j);
  }
};
struct SplitF {
  const float* x; float* hi; float* lo;
  __device__ void one(int64_t i) const {
    float v = x[i];
    uint32_t h, l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    float r = v - __uint_as_float(h);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
    hi[i] = __uint_as_float(h);
    lo[i] = __uint_as_float(l);
  }
  __device__ void vec(int64_t i) const { for (int j = 0; j < 8; ++j) one(i + j); }
};
struct ReluF {
  const void* x; void* y; be_dtype dt;
  __device__ void one(int64_t i) const { st(y, i, dt, fmaxf(ld(x, i, dt), 0.f)); }
  __device__ void vec(int64_t i) const {
    V8 a = ld8(x, i, dt);
    for (int j = 0; j < 8; ++j) a.v[j] = fmaxf(a.v[j], 0.f);
    st8(y, i, dt, a);
  }
};
struct ReluBwdF {
  const void* dy; const void* y; void* dx; be_dtype dt; float beta;
  __device__ void one(int64_t i) const {
    float g = ld(y, i, dt) > 0.f ? ld(dy, i, dt) : 0.f;
    if (beta != 0.f) g += ld(dx, i, dt);
    st(dx, i, dt, g);
  }
  __device__ void vec(int64_t i) const {
    V8 g = ld8(dy, i, dt), yy = ld8(y, i, dt);
    V8 o;
    if (beta != 0.f) o = ld8(dx, i, dt);
    for (int j = 0; j < 8; ++j) o.v[j] = (yy.v[j] > 0.f ? g.v[j] : 0.f) + (beta != 0.f ? o.v[j] : 0.f);
    st8(dx, i, dt, o);
  }
};
// residual add+ReLU backward: both inputs get dy·1[y>0] in one pass
struct ReluBwd2F {
  const void* dy; const void* y; void* d1; float b1; void* d2; float b2; be_dtype dt;
  __device__ void one(int64_t i) const {
    const float g = ld(y, i, dt) > 0.f ? ld(dy, i, dt) : 0.f;
    if (d1) st(d1, i, dt, g + (b1 != 0.f ? ld(d1, i, dt) : 0.f));
    if (d2) st(d2, i, dt, g + (b2 != 0.f ? ld(d2, i, dt) : 0.f));
  }
  __device__ void vec(int64_t i) const {
    V8 g = ld8(dy, i, dt), yy = ld8(y, i, dt);
#pragma unroll
    for (int j = 0; j < 8; ++j) g.v[j] = yy.v[j] > 0.f ? g.v[j] : 0.f;
    if (d1) {
      V8 o = g;
      if (b1 != 0.f) { V8 p = ld8(d1, i, dt); for (int j = 0; j < 8; ++j) o.v[j] += p.v[j]; }
      st8(d1, i, dt, o);
    }
    if (d2) {
      V8 o = g;
      if (b2 != 0.f) { V8 p = ld8(d2, i, dt); for (int j = 0; j < 8; ++j) o.v[j] += p.v[j]; }
      st8(d2, i, dt, o);
    }
  }
};
struct AddF {
  const void* a; const void* b; void* y; be_dtype dt; int act;
  __device__ void one(int64_t i) const {
    float v = ld(a, i, dt) + ld(b, i, dt);
    st(y, i, dt, act ? fmaxf(v, 0.f) : v);
  }
  __device__ void vec(int64_t i) const {
    V8 p = ld8(a, i, dt), q = ld8(b, i, dt);
    for (int j = 0; j < 8; ++j) { float v = p.v[j] + q.v[j]; p.v[j] = act ? fmaxf(v, 0.f) : v; }
    st8(y, i, dt, p);
  }
};
struct MulAccF {
  const void* a; const void* b; void* y; be_dtype dt; float beta;
  __device__ void one(int64_t i) const {
    float v = ld(a, i, dt) * ld(b, i, dt);
    if (beta != 0.f) v += ld(y, i, dt);
    st(y, i, dt, v);
  }
  __device__ void vec(int64_t i) const {
    V8 p = ld8(a, i, dt), q = ld8(b, i, dt), o;
    if (beta != 0.f) o = ld8(y, i, dt);
    for (int j = 0; j < 8; ++j) p.v[j] = p.v[j] * q.v[j] + (beta != 0.f ? o.v[j] : 0.f);
    st8(y, i, dt, p);
  }
};
struct AxpbyF {
  const void* x; be_dtype xd; void* y; be_dtype yd; float alpha, beta;
  __device__ void one(int64_t i) const {
    float v = alpha * ld(x, i, xd);
    if (beta != 0.f) v += beta * ld(y, i, yd);
    st(y, i, yd, v);
  }
  __device__ void vec(int64_t i) const {
    V8 p = ld8(x, i, xd), o;
    if (beta != 0.f) o = ld8(y, i, yd);
    for (int j = 0; j < 8; ++j) p.v[j] = alpha * p.v[j] + (beta != 0.f ? beta * o.v[j] : 0.f);
    st8(y, i, yd, p);
  }
};
struct ScaleDevF {
  const void* x; be_dtype xd; void* y; be_dtype yd; const float* s;
  __device__ void one(int64_t i) const { st(y, i, yd, ld(x, i, xd) * __ldg(s)); }
  __device__ void vec(int64_t i) const {
    float c = __ldg(s);
    V8 p = ld8(x, i, xd);
    for (int j = 0; j < 8; ++j) p.v[j] *= c;
    st8(y, i, yd, p);
  }
};
struct BcastScalarF {
  const float* g; void* dx; be_dtype dt; float scale, beta;
  __device__ void one(int64_t i) const {
    float v = __ldg(g) * scale;
    if (beta != 0.f) v += ld(dx, i, dt);
    st(dx, i, dt, v);
  }
  __device__ void vec(int64_t i) const { for (int j = 0; j < 8; ++j) one(i + j); }
};

__global__ void add_bcast_kernel(const void* a, const void* b, void* y, BcastDesc d, be_dtype dt, int act,
                                 int64_t n) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = i, oa = 0, ob = 0;
    for (int r = d.rank - 1; r >= 0; --r) {
      int64_t c = rem % d.shape[r];
      rem /= d.shape[r];
      oa += c * d.sa[r];
      ob += c * d.sb[r];
    }
    float v = ld(a, oa, dt) + ld(b, ob, dt);
    st(y, i, dt, act ? fmaxf(v, 0.f) : v);
  }
}

// ---- column sums: grid (col groups of 64, row splits); block = 8 warps.
// MODE 0: plain; MODE 1: dz = dy*[y>0] written, colsum(dz)
template <int MODE>
__global__ void colsum_kernel(const void* x, const void* yv, void* dz, int64_t rows, int64_t cols, be_dtype dt,
                              float* partial, int64_t rows_per_split) {
  pdl_entry();
  __shared__ float sm[8][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * 64 + lane * 2;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = min(rows, r0 + rows_per_split);
  float s0 = 0.f, s1 = 0.f;
  for (int64_t r = r0 + warp; r < r1; r += 8) {
    const int64_t base = r * cols + c;
    float a0 = 0.f, a1 = 0.f;
    if (c < cols) a0 = ld(x, base, dt);
    if (c + 1 < cols) a1 = ld(x, base + 1, dt);
    if (MODE == 1) {
      if (c < cols) { if (!(ld(yv, base, dt) > 0.f)) a0 = 0.f; st(dz, base, dt, a0); }
      if (c + 1 < cols) { if (!(ld(yv, base + 1, dt) > 0.f)) a1 = 0.f; st(dz, base + 1, dt, a1); }
    }
    s0 += a0; s1 += a1;
  }
  sm[warp][lane * 2] = s0;
  sm[warp][lane * 2 + 1] = s1;
  __syncthreads();
  if (warp == 0) {
    for (int j = 0; j < 2; ++j) {
      float t = 0.f;
      for (int w = 0; w < 8; ++w) t += sm[w][lane * 2 + j];
      int64_t cc = c + j;
      if (cc < cols) partial[(int64_t)blockIdx.y * cols + cc] = t;
    }
  }
}
// Vectorised variant (cols % 8 == 0, 16-B aligned): thread (tx, ty) owns 8
// consecutive columns (one 128-bit bf16 vector) and every 8th row of its
// split; 4 rows in flight per thread; fixed-order smem combine.
// The last block of each 256-column group to finish (arrival counter) also
// reduces that group's split partials into out[] (+ beta·out) in a fixed order
// — no separate finalize launch, and the result does not depend on which
// block arrived last.
template <int MODE>
__global__ void __launch_bounds__(256) colsum_v_kernel(const void* __restrict__ x, const void* __restrict__ yv,
                                                       void* __restrict__ dz, int64_t rows, int64_t cols, be_dtype dt,
                                                       float* __restrict__ partial, int64_t rows_per_split,
                                                       unsigned* __restrict__ counters, float* __restrict__ out,
                                                       float beta) {
  pdl_entry();
  __shared__ float sm[8][257];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c = ((int64_t)blockIdx.x * 32 + tx) * 8;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = min(rows, r0 + rows_per_split);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (c < cols) {
    int64_t r = r0 + ty;
    for (; r + 24 < r1; r += 32) {
      V8 a[4], m[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = ld8(x, (r + u * 8) * cols + c, dt);
      if (MODE == 1) {
#pragma unroll
        for (int u = 0; u < 4; ++u) m[u] = ld8(yv, (r + u * 8) * cols + c, dt);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (MODE == 1) {
#pragma unroll
          for (int j = 0; j < 8; ++j) a[u].v[j] = m[u].v[j] > 0.f ? a[u].v[j] : 0.f;
          st8(dz, (r + u * 8) * cols + c, dt, a[u]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += a[u].v[j];
      }
    }
    for (; r < r1; r += 8) {
      V8 a = ld8(x, r * cols + c, dt);
      if (MODE == 1) {
        V8 m = ld8(yv, r * cols + c, dt);
#pragma unroll
        for (int j = 0; j < 8; ++j) a.v[j] = m.v[j] > 0.f ? a.v[j] : 0.f;
        st8(dz, r * cols + c, dt, a);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += a.v[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) sm[ty][tx * 8 + j] = acc[j];
  __syncthreads();
  const int cc = threadIdx.x;  // 256 columns of this block
  const int64_t col = (int64_t)blockIdx.x * 256 + cc;
  if (col < cols) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += sm[w][cc];
    partial[(int64_t)blockIdx.y * cols + col] = t;
  }
  // ---- last arriving block of this column group: final fixed-order reduce
  __shared__ unsigned last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&counters[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int64_t rem = cols - (int64_t)blockIdx.x * 256;
  const int ncol = rem < 256 ? (int)rem : 256;
  const int per = 256 / ncol >= 8 ? 8 : (256 / ncol >= 4 ? 4 : (256 / ncol >= 2 ? 2 : 1));  // threads per column
  const int cidx = threadIdx.x / per, part = threadIdx.x % per;
  float t = 0.f;
  if (cidx < ncol) {
    const int64_t c2 = (int64_t)blockIdx.x * 256 + cidx;
    for (int sp = part; sp < (int)gridDim.y; sp += per) t += __ldcg(&partial[(int64_t)sp * cols + c2]);
  }
  __syncthreads();
  sm[0][threadIdx.x] = t;
  __syncthreads();
  if (part == 0 && cidx < ncol) {
    float u = 0.f;
    for (int k = 0; k < per; ++k) u += sm[0][threadIdx.x + k];
    const int64_t c2 = (int64_t)blockIdx.x * 256 + cidx;
    out[c2] = u + (beta != 0.f ? out[c2] : 0.f);
  }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0u;  // ready for the next launch
}

__global__ void colsum_finalize(const float* partial, int splits, int64_t cols, float* out, float beta) {
  pdl_entry();
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
    float t = 0.f;
    for (int s = 0; s < splits; ++s) t += partial[(int64_t)s * cols + c];
    out[c] = t + (beta != 0.f ? out[c] : 0.f);
  }
}

// Zero-initialised arrival counters (one per 256-column group), reset by the
// kernel itself; one buffer per process is enough because launches on the
// compute stream are serialised.
unsigned* colsum_counters(int64_t groups) {
  static unsigned* buf = nullptr;
  static int64_t cap = 0;
  if (groups > cap) {
    BE_CHECK_CUDA(cudaDeviceSynchronize());  // the old buffer may still be in use
    if (buf) cudaFree(buf);
    cap = std::max<int64_t>(groups, 4096);
    BE_CHECK_CUDA(cudaMalloc(&buf, sizeof(unsigned) * cap));
    BE_CHECK_CUDA(cudaMemset(buf, 0, sizeof(unsigned) * cap));
  }
  return buf;
}

void colsum_impl(int mode, const void* x, const void* y, void* dz, int64_t rows, int64_t cols, be_dtype dt,
                 float* out, float beta, cudaStream_t s) {
  if (cols == 0) return;
  if (rows > 0 && cols % 8 == 0 && aligned16(x) && (mode == 0 || (aligned16(y) && aligned16(dz)))) {
    const int64_t cg = (cols + 255) / 256;
    int64_t splits = std::max<int64_t>(1, std::min<int64_t>((rows + 31) / 32, (int64_t)ctx().num_sms * 4 / cg));
    const int64_t rps = (rows + splits - 1) / splits;
    splits = (rows + rps - 1) / rps;
    Block* tmp = ctx().alloc.allocate(sizeof(float) * splits * cols, s);
    float* partial = reinterpret_cast<float*>(tmp->ptr);
    dim3 grid((unsigned)cg, (unsigned)splits);
    unsigned* counters = colsum_counters(cg);
    if (mode == 0)
      launch_pdl(colsum_v_kernel<0>, grid, 256, 0, s, x, nullptr, nullptr, rows, cols, dt, partial, rps, counters, out, beta);
    else
      launch_pdl(colsum_v_kernel<1>, grid, 256, 0, s, x, y, dz, rows, cols, dt, partial, rps, counters, out, beta);
    after_launch(mode == 0 ? "colsum_v" : "relu_bwd_colsum_v");
    ctx().alloc.free(tmp);
    return;
  }
  const int64_t cgroups = (cols + 63) / 64;
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>((rows + 63) / 64, (int64_t)ctx().num_sms * 4 / cgroups));
  splits = std::min<int64_t>(splits, 4096);
  const int64_t rps = (rows + splits - 1) / splits;
  splits = rows == 0 ? 1 : (rows + rps - 1) / rps;
  Block* tmp = ctx().alloc.allocate(sizeof(float) * splits * cols, s);
  float* partial = reinterpret_cast<float*>(tmp->ptr);
  dim3 grid((unsigned)cgroups, (unsigned)splits);
  if (rows == 0) {
    cudaMemsetAsync(partial, 0, sizeof(float) * cols, s);
  } else if (mode == 0) {
    launch_pdl(colsum_kernel<0>, grid, 256, 0, s, x, nullptr, nullptr, rows, cols, dt, partial, rps);
    after_launch("colsum");
  } else {
    launch_pdl(colsum_kernel<1>, grid, 256, 0, s, x, y, dz, rows, cols, dt, partial, rps);
    after_launch("relu_bwd_colsum");
  }
  colsum_finalize<<<(unsigned)std::min<int64_t>((cols + 255) / 256, 1024), 256, 0, s>>>(partial, (int)splits, cols,
                                                                                          out, beta);
  after_launch("colsum_finalize");
  ctx().alloc.free(tmp);
}

// ---- full reduction: two-pass, deterministic
__global__ void reduce_partial(const void* x, int64_t n, be_dtype dt, float* partial) {
  pdl_entry();
  float s = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += ld(x, i, dt);
  s = warp_sum(s);
  __shared__ float sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? sm[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
  }
}
__global__ void reduce_final(const float* partial, int n, float* out, float scale) {
  pdl_entry();
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
  s = warp_sum(s);
  __shared__ float sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? sm[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) out[0] = t * scale;
  }
}

// ---- softmax cross-entropy: one block (256 thr) per row
__global__ void __launch_bounds__(256) xent_kernel(const void* z, be_dtype zd, int64_t ldz, const int32_t* y,
                                                   int64_t B, int64_t C, float* row_loss, void* dz, be_dtype dzd,
                                                   int32_t* am) {
  pdl_entry();
  const int64_t row = blockIdx.x;
  const void* zr = reinterpret_cast<const char*>(z) + row * ldz * (zd == BE_BF16 ? 2 : 4);
  __shared__ float smax[8], ssum[8];
  __shared__ int sidx[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float m = -INFINITY;
  int mi = 0x7fffffff;
  for (int64_t j = threadIdx.x; j < C; j += 256) {
    float v = ld(zr, j, zd);
    if (v > m || (v == m && j < mi) || (v != v && m == m)) { m = v; mi = (int)j; }
  }
  // (max, first index) warp reduce
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float om = __shfl_xor_sync(0xffffffffu, m, o);
    int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    if (om > m || (om == m && oi < mi)) { m = om; mi = oi; }
  }
  if (lane == 0) { smax[warp] = m; sidx[warp] = mi; }
  __syncthreads();
  m = smax[0]; mi = sidx[0];
  for (int w = 1; w < 8; ++w)
    if (smax[w] > m || (smax[w] == m && sidx[w] < mi)) { m = smax[w]; mi = sidx[w]; }
  float s = 0.f;
  for (int64_t j = threadIdx.x; j < C; j += 256) s += __expf(ld(zr, j, zd) - m);
  s = warp_sum(s);
  if (lane == 0) ssum[warp] = s;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < 8; ++w) tot += ssum[w];
  const float lse = m + logf(tot);
  const int lab = y[row];
  const float invB = 1.f / (float)B;
  for (int64_t j = threadIdx.x; j < C; j += 256) {
    float p = __expf(ld(zr, j, zd) - lse);
    st(dz, row * C + j, dzd, (p - (j == lab ? 1.f : 0.f)) * invB);
  }
  if (threadIdx.x == 0) {
    row_loss[row] = lse - ld(zr, lab, zd);
    if (am) am[row] = mi;
  }
}
__global__ void bce_kernel(const void* z, be_dtype zd, const int32_t* y, int64_t B, float* row_loss, void* dz,
                           be_dtype dzd) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B; i += (int64_t)gridDim.x * blockDim.x) {
    float v = ld(z, i, zd);
    float t = (float)y[i];
    // softplus(z) − t·z, stable; dz = (σ(z) − t)/B
    row_loss[i] = fmaxf(v, 0.f) - t * v + log1pf(__expf(-fabsf(v)));
    float sg = 1.f / (1.f + __expf(-v));
    st(dz, i, dzd, (sg - t) / (float)B);
  }
}

// ---- fused multi-tensor SGD
constexpr int kSgdMax = 256;
struct SgdTable {
  int n;
  int64_t start[kSgdMax + 1];  // prefix sums of chunks (in units of kSgdChunk elements)
  SgdEntry e[kSgdMax];
};
// One chunk = 4096 elements; each thread owns 4 float4 of it (stride 1024
// elements → coalesced) and issues all its loads before any arithmetic:
// ~192 B in flight per thread, so the kernel keeps HBM busy even with only a
// couple of blocks per SM (when it overlaps backward GEMMs, be_sgd_overlap).
constexpr int kSgdChunk = 4096;
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__global__ void __launch_bounds__(256) sgd_kernel(const __grid_constant__ SgdTable t, float lr, float mu, float wd,
                                                  float scale) {
  pdl_entry();
  const int64_t total_chunks = t.start[t.n];
  for (int64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
    int lo = 0, hi = t.n - 1;
    while (lo < hi) {  // last entry with start <= c
      int mid = (lo + hi + 1) >> 1;
      if (t.start[mid] <= c) lo = mid; else hi = mid - 1;
    }
    const SgdEntry& e = t.e[lo];
    const int64_t base = (c - t.start[lo]) * kSgdChunk;
    const int64_t end = min(e.n, base + kSgdChunk);
    const bool vec = ((reinterpret_cast<uintptr_t>(e.p) | reinterpret_cast<uintptr_t>(e.g) |
                       reinterpret_cast<uintptr_t>(e.mom)) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(e.shadow) & 7) == 0;
    if (vec && base + kSgdChunk <= e.n) {
      float4 p4[4], g4[4], m4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t i = base + (threadIdx.x + k * 256) * 4;
        p4[k] = ld4(e.p + i);
        g4[k] = ld4(e.g + i);
        m4[k] = e.mom ? ld4(e.mom + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t i = base + (threadIdx.x + k * 256) * 4;
        float pv[4] = {p4[k].x, p4[k].y, p4[k].z, p4[k].w}, gv[4] = {g4[k].x, g4[k].y, g4[k].z, g4[k].w};
        float mv[4] = {m4[k].x, m4[k].y, m4[k].z, m4[k].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) sgd_elem(pv[j], gv[j], mv[j], e.mom != nullptr, lr, mu, wd, scale);
        *reinterpret_cast<float4*>(e.p + i) = make_float4(pv[0], pv[1], pv[2], pv[3]);
        if (e.mom) *reinterpret_cast<float4*>(e.mom + i) = make_float4(mv[0], mv[1], mv[2], mv[3]);
        if (e.shadow) {
          uint2 u;
          u.x = (uint32_t)f2bf(pv[0]) | ((uint32_t)f2bf(pv[1]) << 16);
          u.y = (uint32_t)f2bf(pv[2]) | ((uint32_t)f2bf(pv[3]) << 16);
          *reinterpret_cast<uint2*>(e.shadow + i) = u;
        }
      }
    } else {
      for (int64_t i = base + threadIdx.x; i < end; i += 256) {
        float pv = e.p[i], mv = e.mom ? e.mom[i] : 0.f;
        sgd_elem(pv, e.g[i], mv, e.mom != nullptr, lr, mu, wd, scale);
        if (e.mom) e.mom[i] = mv;
        e.p[i] = pv;
        if (e.shadow) e.shadow[i] = f2bf(pv);
      }
    }
  }
}
}  // namespace

void fill(void* x, int64_t n, be_dtype dt, double v, cudaStream_t s) {
  launch_ew(n, false, FillF{x, dt, (float)v, (int64_t)v}, s, "fill");
}
void cast(const void* x, be_dtype xd, void* y, be_dtype yd, int64_t n, cudaStream_t s) {
  launch_ew(n, aligned16(x) && aligned16(y), CastF{x, xd, y, yd}, s, "cast");
}
void split_tf32(const float* x, float* hi, float* lo, int64_t n, cudaStream_t s) {
  launch_ew(n, true, SplitF{x, hi, lo}, s, "split_tf32");
}
void relu_fwd(const void* x, void* y, int64_t n, be_dtype dt, cudaStream_t s) {
  launch_ew(n, aligned16(x) && aligned16(y), ReluF{x, y, dt}, s, "relu");
}
void relu_bwd(const void* dy, const void* y, void* dx, int64_t n, be_dtype dt, float beta, cudaStream_t s) {
  launch_ew(n, aligned16(dy) && aligned16(y) && aligned16(dx), ReluBwdF{dy, y, dx, dt, beta}, s, "relu_bwd");
}
void relu_bwd2(const void* dy, const void* y, void* d1, float b1, void* d2, float b2, int64_t n, be_dtype dt,
               cudaStream_t s) {
  const bool vec = aligned16(dy) && aligned16(y) && (!d1 || aligned16(d1)) && (!d2 || aligned16(d2));
  launch_ew(n, vec, ReluBwd2F{dy, y, d1, b1, d2, b2, dt}, s, "relu_bwd2");
}
void add_same(const void* a, const void* b, void* y, int64_t n, be_dtype dt, int act, cudaStream_t s) {
  launch_ew(n, aligned16(a) && aligned16(b) && aligned16(y), AddF{a, b, y, dt, act}, s, "add");
}
void mul_same(const void* a, const void* b, void* y, int64_t n, be_dtype dt, cudaStream_t s) {
  launch_ew(n, aligned16(a) && aligned16(b) && aligned16(y), MulAccF{a, b, y, dt, 0.f}, s, "mul");
}
void mul_acc(const void* a, const void* b, void* y, int64_t n, be_dtype dt, float beta, cudaStream_t s) {
  launch_ew(n, aligned16(a) && aligned16(b) && aligned16(y), MulAccF{a, b, y, dt, beta}, s, "mul_acc");
}
void axpby(const void* x, be_dtype xd, void* y, be_dtype yd, int64_t n, float alpha, float beta, cudaStream_t s) {
  launch_ew(n, aligned16(x) && aligned16(y), AxpbyF{x, xd, y, yd, alpha, beta}, s, "axpby");
}
void scale_dev(const void* x, be_dtype xd, void* y, be_dtype yd, int64_t n, const float* sc, cudaStream_t s) {
  launch_ew(n, aligned16(x) && aligned16(y), ScaleDevF{x, xd, y, yd, sc}, s, "scale_dev");
}
void broadcast_scalar(const float* g, void* dx, be_dtype dt, int64_t n, float scale, float beta, cudaStream_t s) {
  launch_ew(n, false, BcastScalarF{g, dx, dt, scale, beta}, s, "broadcast_scalar");
}
void add_bcast(const void* a, const void* b, void* y, const BcastDesc& d, be_dtype dt, int act, cudaStream_t s) {
  int64_t n = 1;
  for (int i = 0; i < d.rank; ++i) n *= d.shape[i];
  if (n == 0) return;
  launch_pdl(add_bcast_kernel, ew_grid(n, 1), 256, 0, s, a, b, y, d, dt, act, n);
  after_launch("add_bcast");
}
void colsum(const void* x, int64_t rows, int64_t cols, be_dtype dt, float* out, float beta, cudaStream_t s) {
  colsum_impl(0, x, nullptr, nullptr, rows, cols, dt, out, beta, s);
}
bool relu_colsum_stream(const uint16_t* gy, const uint16_t* y, uint16_t* dz, int64_t rows, int C, float* out,
                        float beta, cudaStream_t s);  // bn_stream.cu
void relu_bwd_colsum(const void* dy, const void* y, void* dz, int64_t rows, int64_t cols, be_dtype dt, float* db,
                     float db_beta, int act, cudaStream_t s) {
  if (act && dt == BE_BF16 && (cols <= 2048 || (cols <= 16384 && rows >= 1024)) &&
      relu_colsum_stream(reinterpret_cast<const uint16_t*>(dy), reinterpret_cast<const uint16_t*>(y),
                         reinterpret_cast<uint16_t*>(dz), rows, (int)cols, db, db_beta, s))
    return;
  if (act) colsum_impl(1, dy, y, dz, rows, cols, dt, db, db_beta, s);
  else colsum_impl(0, dy, nullptr, nullptr, rows, cols, dt, db, db_beta, s);
}
void reduce_sum(const void* x, int64_t n, be_dtype dt, float* out, float scale, float* scratch, cudaStream_t s) {
  const int blocks = std::max(1, std::min<int>((int)((n + 2047) / 2048), 1024));
  launch_pdl(reduce_partial, blocks, 256, 0, s, x, n, dt, scratch);
  after_launch("reduce_partial");
  launch_pdl(reduce_final, 1, 1024, 0, s, scratch, blocks, out, scale);
  after_launch("reduce_final");
}
void softmax_xent(const void* z, be_dtype zd, int64_t ldz, const int32_t* y, int64_t B, int64_t C, float* row_loss,
                  float* loss_out, void* dz, be_dtype dzd, int32_t* am, cudaStream_t s) {
  if (B == 0) return;
  launch_pdl(xent_kernel, (unsigned)B, 256, 0, s, z, zd, ldz, y, B, C, row_loss, dz, dzd, am);
  after_launch("softmax_xent");
  launch_pdl(reduce_final, 1, 1024, 0, s, row_loss, (int)B, loss_out, 1.f / (float)B);
  after_launch("xent_mean");
}
void bce_logits(const void* z, be_dtype zd, const int32_t* y, int64_t B, float* row_loss, float* loss_out, void* dz,
                be_dtype dzd, cudaStream_t s) {
  if (B == 0) return;
  launch_pdl(bce_kernel, ew_grid(B, 1), 256, 0, s, z, zd, y, B, row_loss, dz, dzd);
  after_launch("bce");
  launch_pdl(reduce_final, 1, 1024, 0, s, row_loss, (int)B, loss_out, 1.f / (float)B);
  after_launch("bce_mean");
}
void sgd_multi(const SgdEntry* e, int n, float lr, float mu, float wd, float scale, cudaStream_t s, int blocks_per_sm) {
  for (int off = 0; off < n; off += kSgdMax) {
    SgdTable t;
    memset(&t, 0, sizeof(t));
    t.n = std::min(kSgdMax, n - off);
    t.start[0] = 0;
    for (int i = 0; i < t.n; ++i) {
      t.e[i] = e[off + i];
      t.start[i + 1] = t.start[i] + (t.e[i].n + kSgdChunk - 1) / kSgdChunk;
    }
    if (t.start[t.n] == 0) continue;
    const int grid = (int)std::min<int64_t>(t.start[t.n], (int64_t)ctx().num_sms * blocks_per_sm);
    double bytes = 0;
    for (int i = 0; i < t.n; ++i)
      bytes += (double)t.e[i].n * (12 + (t.e[i].mom ? 8 : 0) + (t.e[i].shadow ? 2 : 0));
    const int pidx = prof_begin("sgd", 0.0, bytes, t.n, 0, 0, s);
    launch_pdl(sgd_kernel, grid, 256, 0, s, t, lr, mu, wd, scale);
    prof_end(pidx, s);
    after_launch("sgd_multi");
  }
}

}}  // namespace be::k
