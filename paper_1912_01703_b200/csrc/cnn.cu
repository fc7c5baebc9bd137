// cnn.cu — memory-bound CNN kernels (NHWC): im2col / col2im feeding the
// tcgen05 GEMM (conv fwd / dgrad / wgrad as GEMMs),
// max / global-average pooling, batch-norm statistics / apply / backward,
// embedding gather, column concat / slice.
//
// Index conventions are those of the oracle's im2col table:
// row m = (n, p, q) row-major; column k = (r, u, c) row-major (KRSC order);
// h = p·stride − pad + r; w = q·stride − pad + u; padding reads 0.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "runtime.h"

namespace be { namespace k {
using namespace be::dev;

// bn_stream.cu: TMA-bulk streaming BN passes (bf16, C % 8 == 0, C ≤ 2048)
bool bn_stream_ok(const void* a, int64_t rows, int C);
int64_t bn_stream_splits(int64_t rows, int C, int64_t cap);
// (stats / reduce: true = the finalize ran inside the pass — no bn_finalize_v launch)
bool bn_stats_stream(const uint16_t* x, int64_t rows, int C, float* part0, float* part1, int64_t sp, cudaStream_t s,
                     float eps = 0.f, float* mean = nullptr, float* invstd = nullptr, float* run_mean = nullptr,
                     float* run_var = nullptr, float momentum = 0.f);
bool bn_reduce_stream(const uint16_t* x, const uint16_t* gy, int act, int64_t rows, int C, const float* mean,
                      const float* invstd, float* part0, float* part1, int64_t sp, const float* gam,
                      const float* bsh, const uint16_t* rmask, uint16_t* gout, cudaStream_t s,
                      const uint8_t* rbits = nullptr, float* sums = nullptr, float* dgamma = nullptr,
                      float* dbeta = nullptr, float gb_beta = 0.f);
// early = 1: x / res (apply) or gy / x (dx) were not written by the kernel
// launched just before on s — the pass may start streaming them before its
// PDL wait (bn_stream.cu pdl_entry_stream)
void bn_apply_stream(const uint16_t* x, uint16_t* y, int64_t rows, int C, const float* mean, const float* invstd,
                     const float* gamma, const float* beta, int act, const uint16_t* res, cudaStream_t s,
                     uint8_t* mbits = nullptr, int early = 0);
void bn_dx_stream(const uint16_t* gy, const uint16_t* x, int act, uint16_t* dx, int64_t rows, int C,
                  const float* mean, const float* invstd, const float* gamma, const float* sums, float dx_beta,
                  const float* bsh, cudaStream_t s, int early = 0);

namespace {
int grid_for(int64_t n, int per = 1) {
  int64_t b = (n + 256LL * per - 1) / (256LL * per);
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)ctx().num_sms * 16));
}

// Index arithmetic: the memory-bound CNN kernels decompose a flat item index
// into (n, h, w, c)-style coordinates with run-time divisors.  The launchers
// pick I = uint32_t whenever the item count fits (every C3/C4 shape): 64-bit
// integer division is a ~70-instruction software routine on the GPU and was
// the bottleneck of these kernels (e.g. conv1's wgrad im2col ran at 2 TB/s).
// Byte offsets stay 64-bit.  Each thread keeps UNR items' loads in flight.
constexpr int UNR = 4;

// ---- im2col: one item per (m, r, u, VEC-channel chunk); 16-B copies when C%8==0 (bf16) / C%4==0 (f32)
template <typename T, int VEC, typename I>
__global__ void __launch_bounds__(256) im2col_kernel(const T* __restrict__ x, T* __restrict__ cols, int64_t ldc,
                                                     ConvGeom g, I total) {
  pdl_entry();
  using VT = typename std::conditional<VEC * sizeof(T) == 16, uint4, T>::type;
  static_assert(VEC * sizeof(T) == 16 || VEC == 1, "im2col vector width");
  const I CV = (I)(g.C / VEC);
  const I stride = (I)gridDim.x * blockDim.x;
  for (I base = (I)blockIdx.x * blockDim.x + threadIdx.x; base < total; base += UNR * stride) {
    VT v[UNR];
    int64_t dst[UNR];
#pragma unroll
    for (int k = 0; k < UNR; ++k) {
      const I i = base + (I)k * stride;
      dst[k] = -1;
      if (i < total) {
        I t = i;
        const int cv = (int)(t % CV); t /= CV;
        const int u = (int)(t % (I)g.S); t /= (I)g.S;
        const int r = (int)(t % (I)g.R);
        const I m = t / (I)g.R;
        const int q = (int)(m % (I)g.Q);
        const I np = m / (I)g.Q;
        const int p = (int)(np % (I)g.P);
        const int n = (int)(np / (I)g.P);
        const int h = p * g.stride - g.pad + r, w = q * g.stride - g.pad + u;
        dst[k] = (int64_t)m * ldc + (int64_t)(r * g.S + u) * g.C + cv * VEC;
        if (h >= 0 && h < g.H && w >= 0 && w < g.W)
          v[k] = *reinterpret_cast<const VT*>(x + (((int64_t)n * g.H + h) * g.W + w) * g.C + cv * VEC);
        else
          v[k] = VT{};
      }
    }
#pragma unroll
    for (int k = 0; k < UNR; ++k)
      if (dst[k] >= 0) *reinterpret_cast<VT*>(cols + dst[k]) = v[k];
  }
}

// ---- im2col, tap loop: one item per (m, VEC-channel chunk); the (n, p, q)
// decomposition is done once per item and the R·S taps are copied with their
// loads batched (8 in flight).  The per-(m, r, u, chunk) form above spends
// ~6 run-time divisions per 16-B copy and ran ALU-bound (~2.9 TB/s on the
// ResNet layer-3 wgrad columns); consecutive threads take consecutive channel
// chunks of one pixel, so each tap's loads and stores stay coalesced.
template <typename T, int VEC>
__global__ void __launch_bounds__(256) im2col_taps_kernel(const T* __restrict__ x, T* __restrict__ cols, int64_t ldc,
                                                          ConvGeom g, uint32_t total) {
  pdl_entry();
  using VT = typename std::conditional<VEC * sizeof(T) == 16, uint4, T>::type;
  constexpr int B = 8;
  const uint32_t CV = (uint32_t)(g.C / VEC);
  const int RS = g.R * g.S;
  const uint32_t stride = gridDim.x * blockDim.x;
  if (RS == 1) {  // 1×1 (strided) convolution: a subsampling copy — batch the items instead of the taps
    for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += B * stride) {
      VT v[B];
      int64_t dst[B];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const uint32_t i = i0 + k * stride;
        dst[k] = -1;
        if (i < total) {
          const int cv = (int)(i % CV);
          const uint32_t m = i / CV;
          const int q = (int)(m % (uint32_t)g.Q);
          const uint32_t np = m / (uint32_t)g.Q;
          const int p = (int)(np % (uint32_t)g.P);
          const int n = (int)(np / (uint32_t)g.P);
          const int h = p * g.stride - g.pad, w = q * g.stride - g.pad;
          dst[k] = (int64_t)m * ldc + cv * VEC;
          v[k] = VT{};
          if (h >= 0 && h < g.H && w >= 0 && w < g.W)
            v[k] = *reinterpret_cast<const VT*>(x + (((int64_t)n * g.H + h) * g.W + w) * g.C + cv * VEC);
        }
      }
#pragma unroll
      for (int k = 0; k < B; ++k)
        if (dst[k] >= 0) *reinterpret_cast<VT*>(cols + dst[k]) = v[k];
    }
    return;
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int cv = (int)(i % CV);
    const uint32_t m = i / CV;
    const int q = (int)(m % (uint32_t)g.Q);
    const uint32_t np = m / (uint32_t)g.Q;
    const int p = (int)(np % (uint32_t)g.P);
    const int n = (int)(np / (uint32_t)g.P);
    const int h0 = p * g.stride - g.pad, w0 = q * g.stride - g.pad;
    const T* xn = x + (int64_t)n * g.H * g.W * g.C + cv * VEC;
    T* dst = cols + (int64_t)m * ldc + cv * VEC;
    for (int t0 = 0; t0 < RS; t0 += B) {
      VT v[B];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int t = t0 + k;
        const int r = t / g.S, u = t - r * g.S;
        const int h = h0 + r, w = w0 + u;
        v[k] = VT{};
        if (t < RS && h >= 0 && h < g.H && w >= 0 && w < g.W)
          v[k] = *reinterpret_cast<const VT*>(xn + ((int64_t)h * g.W + w) * g.C);
      }
#pragma unroll
      for (int k = 0; k < B; ++k)
        if (t0 + k < RS) *reinterpret_cast<VT*>(dst + (int64_t)(t0 + k) * g.C) = v[k];
    }
  }
}

// ---- col2im (gather form): dx[n,h,w,c] = Σ_{r,u: h=p·s−pad+r, w=q·s−pad+u} dcols[(n,p,q),(r,u,c)]
template <typename T>
__global__ void col2im_kernel(const T* __restrict__ dcols, int64_t ldc, T* __restrict__ dx, ConvGeom g, float beta,
                              int64_t total, be_dtype dt) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int c = (int)(t % g.C); t /= g.C;
    const int w = (int)(t % g.W); t /= g.W;
    const int h = (int)(t % g.H);
    const int n = (int)(t / g.H);
    float acc = 0.f;
    for (int r = 0; r < g.R; ++r) {
      const int ph = h + g.pad - r;
      if (ph < 0 || ph % g.stride) continue;
      const int p = ph / g.stride;
      if (p >= g.P) continue;
      for (int u = 0; u < g.S; ++u) {
        const int qw = w + g.pad - u;
        if (qw < 0 || qw % g.stride) continue;
        const int q = qw / g.stride;
        if (q >= g.Q) continue;
        const int64_t m = ((int64_t)n * g.P + p) * g.Q + q;
        acc += ld(dcols, m * ldc + (int64_t)(r * g.S + u) * g.C + c, dt);
      }
    }
    if (beta != 0.f) acc += ld(dx, i, dt);
    st(dx, i, dt, acc);
  }
}

// (n, h, w, cv) of a flat NHWC item index with 8-channel vectors
template <typename I>
__device__ __forceinline__ void nhwc8(I i, const ConvGeom& g, int H, int W, int& n, int& h, int& w, int& cv) {
  const I CV = (I)(g.C / 8);
  I t = i;
  cv = (int)(t % CV); t /= CV;
  w = (int)(t % (I)W); t /= (I)W;
  h = (int)(t % (I)H);
  n = (int)(t / (I)H);
}

// col2im, 8 channels per item (16-B loads of dcols / stores of dx).  The taps
// that reach input pixel (h, w) are enumerated by output row/column directly
// (p ∈ [p_lo, p_hi], r = h + pad − p·stride), summed in increasing (r, u)
// order (decreasing p, q) as the reference loop over taps.
template <typename I>
__global__ void __launch_bounds__(256) col2im_v(const void* __restrict__ dcols, int64_t ldc, void* __restrict__ dx,
                                                ConvGeom g, float beta, I nvec, be_dtype dt) {
  pdl_entry();
  const I stride = (I)gridDim.x * blockDim.x;
  for (I i = (I)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    int n, h, w, cv;
    nhwc8(i, g, g.H, g.W, n, h, w, cv);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // p·stride ∈ [h + pad − R + 1, h + pad]
    const int p_hi = min(g.P - 1, (h + g.pad) / g.stride);
    const int p_lo = max(0, (h + g.pad - g.R + g.stride) / g.stride);
    const int q_hi = min(g.Q - 1, (w + g.pad) / g.stride);
    const int q_lo = max(0, (w + g.pad - g.S + g.stride) / g.stride);
    for (int p = p_hi; p >= p_lo; --p) {
      const int r = h + g.pad - p * g.stride;
      for (int q = q_hi; q >= q_lo; --q) {
        const int u = w + g.pad - q * g.stride;
        const int64_t m = ((int64_t)n * g.P + p) * g.Q + q;
        V8 a = ld8(dcols, m * ldc + (int64_t)(r * g.S + u) * g.C + cv * 8, dt);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += a.v[j];
      }
    }
    V8 o;
    if (beta != 0.f) o = ld8(dx, (int64_t)i * 8, dt);
#pragma unroll
    for (int j = 0; j < 8; ++j) o.v[j] = acc[j] + (beta != 0.f ? o.v[j] : 0.f);
    st8(dx, (int64_t)i * 8, dt, o);
  }
}

// col2im for stride-2 R×R (R ∈ {1, 3}) bf16 convolutions (ResNet's
// down-sampling 1×1 and 3×3 dgrads): every pixel gets at most ⌈R/2⌉² taps, so
// all of an item's loads (2 items per thread) are issued before the sums,
// which run in the same increasing-(r, u) order as col2im_v.  When
// accumulating (beta ≠ 0) the pixels no tap reaches (3 of 4 for R = 1) are
// left untouched instead of read and rewritten.
template <int R>
__global__ void __launch_bounds__(256) col2im_s2_bf16(const uint16_t* __restrict__ dcols, int64_t ldc,
                                                      uint16_t* __restrict__ dx, ConvGeom g, float beta, uint32_t nvec) {
  pdl_entry();
  constexpr int T = (R + 1) / 2;  // taps per dimension
  constexpr int UNR = 2;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < nvec; base += stride * UNR) {
    uint4 a[UNR][T * T];
    int nt[UNR][2];
    uint32_t idx[UNR];
#pragma unroll
    for (int k = 0; k < UNR; ++k) {
      const uint32_t i = base + k * stride;
      idx[k] = i;
      nt[k][0] = nt[k][1] = 0;
      if (i >= nvec) continue;
      int n, h, w, cv;
      nhwc8(i, g, g.H, g.W, n, h, w, cv);
      const int p_hi = min(g.P - 1, (h + g.pad) >> 1), p_lo = max(0, (h + g.pad - R + 2) >> 1);
      const int q_hi = min(g.Q - 1, (w + g.pad) >> 1), q_lo = max(0, (w + g.pad - R + 2) >> 1);
      nt[k][0] = max(0, p_hi - p_lo + 1);
      nt[k][1] = max(0, q_hi - q_lo + 1);
#pragma unroll
      for (int dp = 0; dp < T; ++dp)
#pragma unroll
        for (int dq = 0; dq < T; ++dq) {
          const int p = p_hi - dp, q = q_hi - dq;
          if (dp < nt[k][0] && dq < nt[k][1]) {
            const int r = h + g.pad - 2 * p, u = w + g.pad - 2 * q;
            const int64_t m = ((int64_t)n * g.P + p) * g.Q + q;
            a[k][dp * T + dq] = __ldg(reinterpret_cast<const uint4*>(dcols + m * ldc + (int64_t)(r * R + u) * g.C + cv * 8));
          }
        }
    }
#pragma unroll
    for (int k = 0; k < UNR; ++k) {
      if (idx[k] >= nvec) continue;
      const bool none = nt[k][0] == 0 || nt[k][1] == 0;
      if (none && beta != 0.f) continue;  // dx += 0 (beta is an accumulate flag, as in col2im_v)
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int dp = 0; dp < T; ++dp)
#pragma unroll
        for (int dq = 0; dq < T; ++dq)
          if (dp < nt[k][0] && dq < nt[k][1]) {
            const uint16_t* hv = reinterpret_cast<const uint16_t*>(&a[k][dp * T + dq]);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += bf2f(hv[j]);
          }
      uint16_t* dst = dx + (int64_t)idx[k] * 8;
      if (beta != 0.f) {
        const uint4 o = *reinterpret_cast<const uint4*>(dst);
        const uint16_t* hv = reinterpret_cast<const uint16_t*>(&o);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += bf2f(hv[j]);
      }
      uint4 o;
      uint16_t* ho = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
      for (int j = 0; j < 8; ++j) ho[j] = f2bf(acc[j]);
      *reinterpret_cast<uint4*>(dst) = o;
    }
  }
}

// max pool, 8 channels per item; UNR items per thread, all window loads of an
// item issued before its compare chain
template <typename I>
__global__ void __launch_bounds__(256) maxpool_fwd_v(const void* __restrict__ x, void* __restrict__ y,
                                                     uint8_t* __restrict__ am, ConvGeom g, be_dtype dt, I nvec) {
  pdl_entry();
  const I stride = (I)gridDim.x * blockDim.x;
  for (I i = (I)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    int n, p, q, cv;
    nhwc8(i, g, g.P, g.Q, n, p, q, cv);
    float best[8];
    int bi[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { best[j] = -INFINITY; bi[j] = -1; }
    for (int r = 0; r < g.R; ++r) {
      const int h = p * g.stride - g.pad + r;
      if (h < 0 || h >= g.H) continue;
      for (int u = 0; u < g.S; ++u) {
        const int w = q * g.stride - g.pad + u;
        if (w < 0 || w >= g.W) continue;
        V8 a = ld8(x, (((int64_t)n * g.H + h) * g.W + w) * g.C + cv * 8, dt);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float v = a.v[j];
          if (bi[j] < 0 || v > best[j] || (v != v && best[j] == best[j])) { best[j] = v; bi[j] = r * g.S + u; }
        }
      }
    }
    V8 o;
    uint2 packed;
    uint8_t* pb = reinterpret_cast<uint8_t*>(&packed);
#pragma unroll
    for (int j = 0; j < 8; ++j) { o.v[j] = best[j]; pb[j] = (uint8_t)bi[j]; }
    st8(y, (int64_t)i * 8, dt, o);
    if (am) *reinterpret_cast<uint2*>(am + (int64_t)i * 8) = packed;
  }
}
// max-pool backward, gather form: dx[n,h,w,c] = Σ over the windows (p, q)
// containing (h, w) whose recorded winner is (h, w).  With R ≤ 2·stride and
// S ≤ 2·stride (every pool on the path) at most 2 × 2 windows: their 4
// (dy, argmax) loads are issued together, then summed in (p, q) order.
template <typename I, bool TWO>
__global__ void __launch_bounds__(256) maxpool_bwd_v(const void* __restrict__ dy, const uint8_t* __restrict__ am,
                                                     void* __restrict__ dx, ConvGeom g, be_dtype dt, float beta,
                                                     I nvec) {
  pdl_entry();
  const I stride = (I)gridDim.x * blockDim.x;
  for (I i = (I)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    int n, h, w, cv;
    nhwc8(i, g, g.H, g.W, n, h, w, cv);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int p_lo = max(0, (h + g.pad - g.R + g.stride) / g.stride);
    const int p_hi = min(g.P - 1, (h + g.pad) / g.stride);
    const int q_lo = max(0, (w + g.pad - g.S + g.stride) / g.stride);
    const int q_hi = min(g.Q - 1, (w + g.pad) / g.stride);
    if (TWO) {
      uint2 pk[4];
      V8 d[4];
      int widx[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int p = p_lo + (c >> 1), q = q_lo + (c & 1);
        widx[c] = -1;
        if (p <= p_hi && q <= q_hi) {
          const int64_t o = (((int64_t)n * g.P + p) * g.Q + q) * g.C + cv * 8;
          pk[c] = *reinterpret_cast<const uint2*>(am + o);
          d[c] = ld8(dy, o, dt);
          widx[c] = (h - (p * g.stride - g.pad)) * g.S + (w - (q * g.stride - g.pad));
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (widx[c] < 0) continue;
        const uint8_t* pb = reinterpret_cast<const uint8_t*>(&pk[c]);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += pb[j] == widx[c] ? d[c].v[j] : 0.f;
      }
    } else {
      for (int p = p_lo; p <= p_hi; ++p) {
        const int r = h - (p * g.stride - g.pad);
        for (int q = q_lo; q <= q_hi; ++q) {
          const int u = w - (q * g.stride - g.pad);
          const int64_t o = (((int64_t)n * g.P + p) * g.Q + q) * g.C + cv * 8;
          const uint2 packed = *reinterpret_cast<const uint2*>(am + o);
          const uint8_t* pb = reinterpret_cast<const uint8_t*>(&packed);
          V8 d = ld8(dy, o, dt);
          const int widx = r * g.S + u;
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += pb[j] == widx ? d.v[j] : 0.f;
        }
      }
    }
    V8 o2;
    if (beta != 0.f) o2 = ld8(dx, (int64_t)i * 8, dt);
#pragma unroll
    for (int j = 0; j < 8; ++j) o2.v[j] = acc[j] + (beta != 0.f ? o2.v[j] : 0.f);
    st8(dx, (int64_t)i * 8, dt, o2);
  }
}

__global__ void phase_zero_kernel(uint16_t* __restrict__ dx, ConvGeom g, uint32_t live, int64_t total) {
  pdl_entry();
  const int CV = g.C / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i / CV;
    const int w = (int)(t % g.W); t /= g.W;
    const int h = (int)(t % g.H);
    const int ph = (h % g.stride) * g.stride + (w % g.stride);
    if (!((live >> ph) & 1u)) *reinterpret_cast<uint4*>(dx + i * 8) = make_uint4(0u, 0u, 0u, 0u);
  }
}

// Index probe for be_debug_im2col_offsets: element i of the probe input holds
// the bits of the int32 i + 1 (the im2col kernel is a pure bit copy, so the
// column matrix it builds holds 1 + the NHWC offset it gathered, 0 = padding).
__global__ void iota1_kernel(int32_t* x, int64_t n) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (int32_t)(i + 1);
}
__global__ void cols_to_offsets_kernel(const int32_t* cols, int64_t* out, int64_t n) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)cols[i] - 1;
}

// ---- max pool NHWC; window scanned r outer, u inner; first strictly greater wins; NaN wins at first sight
__global__ void maxpool_fwd_kernel(const void* x, void* y, uint8_t* am, ConvGeom g, be_dtype dt, int64_t total) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int c = (int)(t % g.C); t /= g.C;
    const int q = (int)(t % g.Q); t /= g.Q;
    const int p = (int)(t % g.P);
    const int n = (int)(t / g.P);
    float best = -INFINITY;
    int bi = -1;
    for (int r = 0; r < g.R; ++r) {
      const int h = p * g.stride - g.pad + r;
      if (h < 0 || h >= g.H) continue;
      for (int u = 0; u < g.S; ++u) {
        const int w = q * g.stride - g.pad + u;
        if (w < 0 || w >= g.W) continue;
        const float v = ld(x, (((int64_t)n * g.H + h) * g.W + w) * g.C + c, dt);
        if (bi < 0 || v > best || (v != v && best == best)) { best = v; bi = r * g.S + u; }
      }
    }
    st(y, i, dt, best);
    if (am) am[i] = (uint8_t)bi;
  }
}
__global__ void maxpool_bwd_kernel(const void* dy, const uint8_t* am, void* dx, ConvGeom g, be_dtype dt, float beta,
                                   int64_t total) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int c = (int)(t % g.C); t /= g.C;
    const int w = (int)(t % g.W); t /= g.W;
    const int h = (int)(t % g.H);
    const int n = (int)(t / g.H);
    float acc = 0.f;
    // windows (p,q) with p·s−pad ≤ h < p·s−pad+R
    const int p_lo = max(0, (h + g.pad - g.R + g.stride) / g.stride);
    const int p_hi = min(g.P - 1, (h + g.pad) / g.stride);
    const int q_lo = max(0, (w + g.pad - g.S + g.stride) / g.stride);
    const int q_hi = min(g.Q - 1, (w + g.pad) / g.stride);
    for (int p = p_lo; p <= p_hi; ++p) {
      const int r = h - (p * g.stride - g.pad);
      if (r < 0 || r >= g.R) continue;
      for (int q = q_lo; q <= q_hi; ++q) {
        const int u = w - (q * g.stride - g.pad);
        if (u < 0 || u >= g.S) continue;
        const int64_t o = (((int64_t)n * g.P + p) * g.Q + q) * g.C + c;
        if (am[o] == r * g.S + u) acc += ld(dy, o, dt);
      }
    }
    if (beta != 0.f) acc += ld(dx, i, dt);
    st(dx, i, dt, acc);
  }
}

// ---- global average pool: block per (n, 64-channel group)
__global__ void avgpool_fwd_kernel(const void* x, void* y, int HW, int C, be_dtype dt) {
  pdl_entry();
  const int n = blockIdx.y;
  const int c = blockIdx.x * 64 + (threadIdx.x & 63);
  const int part = threadIdx.x >> 6;  // 4 parts
  __shared__ float sm[4][64];
  float s = 0.f;
  if (c < C)
    for (int i = part; i < HW; i += 4) s += ld(x, ((int64_t)n * HW + i) * C + c, dt);
  sm[part][threadIdx.x & 63] = s;
  __syncthreads();
  if (part == 0 && c < C) st(y, (int64_t)n * C + c, dt, (sm[0][threadIdx.x] + sm[1][threadIdx.x] + sm[2][threadIdx.x] + sm[3][threadIdx.x]) / (float)HW);
}
__global__ void avgpool_bwd_kernel(const void* dy, void* dx, int HW, int C, be_dtype dt, float beta, int64_t total) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t n = i / ((int64_t)HW * C);
    float v = ld(dy, n * C + c, dt) / (float)HW;
    if (beta != 0.f) v += ld(dx, i, dt);
    st(dx, i, dt, v);
  }
}

// ---- batch norm: per-channel reductions over rows with fixed-order partials
// partial layout: [splits][C] ; grid (ceil(C/64), splits), block 256 (4 row lanes x 64 channels)
template <int MODE>  // 0: Σx   1: Σ(x−mean)²   2: Σg', Σg'·x̂  (g' = g·[y>0] if act)
__global__ void bn_reduce_kernel(const void* x, const void* gy, const void* yv, int act, int64_t rows, int C,
                                 be_dtype dt, const float* mean, const float* invstd, float* part0, float* part1,
                                 int64_t rows_per_split) {
  pdl_entry();
  const int cl = threadIdx.x & 63, lane_r = threadIdx.x >> 6;
  const int c = blockIdx.x * 64 + cl;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split, r1 = min(rows, r0 + rows_per_split);
  float s0 = 0.f, s1 = 0.f;
  if (c < C) {
    const float mu = MODE >= 1 ? mean[c] : 0.f;
    const float is = MODE == 2 ? invstd[c] : 0.f;
    for (int64_t r = r0 + lane_r; r < r1; r += 4) {
      const int64_t o = r * C + c;
      const float v = ld(x, o, dt);
      if (MODE == 0) s0 += v;
      else if (MODE == 1) { float d = v - mu; s0 += d * d; }
      else {
        float g = ld(gy, o, dt);
        if (act && !act_pass(ld(yv, o, dt), act)) g = 0.f;
        s0 += g;
        s1 += g * (v - mu) * is;
      }
    }
  }
  __shared__ float sm0[4][64], sm1[4][64];
  sm0[lane_r][cl] = s0;
  sm1[lane_r][cl] = s1;
  __syncthreads();
  if (lane_r == 0 && c < C) {
    part0[(int64_t)blockIdx.y * C + c] = sm0[0][cl] + sm0[1][cl] + sm0[2][cl] + sm0[3][cl];
    if (MODE == 2) part1[(int64_t)blockIdx.y * C + c] = sm1[0][cl] + sm1[1][cl] + sm1[2][cl] + sm1[3][cl];
  }
}
__global__ void bn_mean_finalize(const float* part, int splits, int C, int64_t rows, float* mean) {
  pdl_entry();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float s = 0.f;
  for (int i = 0; i < splits; ++i) s += part[(int64_t)i * C + c];
  mean[c] = s / (float)rows;
}
__global__ void bn_var_finalize(const float* part, int splits, int C, int64_t rows, float eps, const float* mean,
                                float* invstd, float* run_mean, float* run_var, float momentum) {
  pdl_entry();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float s = 0.f;
  for (int i = 0; i < splits; ++i) s += part[(int64_t)i * C + c];
  const float var = s / (float)rows;  // biased (normalisation)
  invstd[c] = rsqrtf(var + eps);
  if (run_mean) run_mean[c] = (1.f - momentum) * run_mean[c] + momentum * mean[c];
  if (run_var) run_var[c] = (1.f - momentum) * run_var[c] + momentum * var * (float)rows / (float)(rows > 1 ? rows - 1 : 1);
}
__global__ void bn_grad_finalize(const float* p0, const float* p1, int splits, int C, float* dgamma, float* dbeta,
                                 float gb_beta, float* sums) {
  pdl_entry();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float s0 = 0.f, s1 = 0.f;
  for (int i = 0; i < splits; ++i) { s0 += p0[(int64_t)i * C + c]; s1 += p1[(int64_t)i * C + c]; }
  sums[c] = s0;       // Σg'
  sums[C + c] = s1;   // Σg'·x̂
  if (dbeta) dbeta[c] = s0 + (gb_beta != 0.f ? dbeta[c] : 0.f);
  if (dgamma) dgamma[c] = s1 + (gb_beta != 0.f ? dgamma[c] : 0.f);
}
__global__ void bn_apply_kernel(const void* x, void* y, int64_t total, int C, be_dtype dt, const float* mean,
                                const float* invstd, const float* gamma, const float* beta, int act,
                                const void* res) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    float v = gamma[c] * (ld(x, i, dt) - mean[c]) * invstd[c] + beta[c];
    if (res) v += ld(res, i, dt);
    v = act_apply(v, act);
    st(y, i, dt, v);
  }
}
__global__ void bn_dx_kernel(const void* gy, const void* x, const void* yv, int act, void* dx, int64_t total, int C,
                             int64_t rows, be_dtype dt, const float* mean, const float* invstd, const float* gamma,
                             const float* sums, float dx_beta) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    float g = ld(gy, i, dt);
    if (act && !act_pass(ld(yv, i, dt), act)) g = 0.f;
    const float is = invstd[c];
    const float xh = (ld(x, i, dt) - mean[c]) * is;
    const float inv_n = 1.f / (float)rows;
    float v = gamma[c] * is * (g - sums[c] * inv_n - xh * sums[C + c] * inv_n);
    if (dx_beta != 0.f) v += ld(dx, i, dt);
    st(dx, i, dt, v);
  }
}

// ---- vectorised BN (C % 8 == 0, 16-B aligned): thread owns 8 consecutive
// channels of one row; a block covers up to 2048 channels × (256/(C/8)) rows
// per iteration; fixed-order smem combine → deterministic partials.
constexpr int kBnCG = 2048;  // channels per block group
template <int MODE>  // 0: Σ(x−K), Σ(x−K)² with K = x[0,c] (shifted sums); 2: Σg', Σg'·x̂
__global__ void __launch_bounds__(256) bn_reduce_v(const void* __restrict__ x, const void* __restrict__ gy,
                                                   const void* __restrict__ yv, int act, int64_t rows, int C,
                                                   be_dtype dt, const float* __restrict__ mean,
                                                   const float* __restrict__ invstd, float* __restrict__ part0,
                                                   float* __restrict__ part1, int64_t rows_per_split,
                                                   const float* __restrict__ gam = nullptr,
                                                   const float* __restrict__ bsh = nullptr) {
  pdl_entry();
  // act with gam/bsh: the ReLU mask is recomputed as fma(x, γ·is, β − μ·γ·is) > 0
  // — the forward's exact expression — instead of reading the saved output.
  __shared__ float sm0[kBnCG], sm1[kBnCG];
  const int base = blockIdx.x * kBnCG;
  const int Cg = min(kBnCG, C - base);
  const int lanes = Cg / 8, rpi = 256 / lanes;
  const int t = threadIdx.x, v = t % lanes, rl = t / lanes;
  const int c = base + v * 8;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split, r1 = min(rows, r0 + rows_per_split);
  float s0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, s1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (rl < rpi) {
    float k[8], is[8], sc[8], sh[8];
    if (MODE == 0) {
      V8 kk = ld8(x, c, dt);
#pragma unroll
      for (int j = 0; j < 8; ++j) k[j] = kk.v[j];
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        k[j] = mean[c + j]; is[j] = invstd[c + j];
        sc[j] = gam ? gam[c + j] * is[j] : 0.f;
        sh[j] = gam ? bsh[c + j] - k[j] * sc[j] : 0.f;
      }
    }
    // two rows per iteration, all loads issued before any use (more bytes in
    // flight per thread; the duplicate load of a missing second row hits L1)
    auto accum = [&](const V8& a, V8 g, const V8& yy) {
      if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) { const float d = a.v[j] - k[j]; s0[j] += d; s1[j] += d * d; }
      } else {
        if (act && gam) {
#pragma unroll
          for (int j = 0; j < 8; ++j) g.v[j] = act_pass_st(fmaf(a.v[j], sc[j], sh[j]), act, dt == BE_BF16) ? g.v[j] : 0.f;
        } else if (act) {
#pragma unroll
          for (int j = 0; j < 8; ++j) g.v[j] = act_pass(yy.v[j], act) ? g.v[j] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) { s0[j] += g.v[j]; s1[j] += g.v[j] * (a.v[j] - k[j]) * is[j]; }
      }
    };
    for (int64_t r = r0 + rl; r < r1; r += 2 * rpi) {
      const bool two = r + rpi < r1;
      const int64_t o0 = r * C + c, o1 = two ? o0 + (int64_t)rpi * C : o0;
      V8 a0 = ld8(x, o0, dt), a1 = ld8(x, o1, dt), g0, g1, y0, y1;
      if (MODE != 0) {
        g0 = ld8(gy, o0, dt); g1 = ld8(gy, o1, dt);
        if (act && !gam) { y0 = ld8(yv, o0, dt); y1 = ld8(yv, o1, dt); }
      }
      accum(a0, g0, y0);
      if (two) accum(a1, g1, y1);
    }
  }
  // rpi·Cg ≤ 2048: every lane's partials fit; combine over row lanes in order
  if (rl < rpi) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { sm0[rl * Cg + v * 8 + j] = s0[j]; sm1[rl * Cg + v * 8 + j] = s1[j]; }
  }
  __syncthreads();
  for (int i = t; i < Cg; i += 256) {
    float a0 = 0.f, a1 = 0.f;
    for (int w = 0; w < rpi; ++w) { a0 += sm0[w * Cg + i]; a1 += sm1[w * Cg + i]; }
    part0[(int64_t)blockIdx.y * C + base + i] = a0;
    part1[(int64_t)blockIdx.y * C + base + i] = a1;
  }
}
__global__ void bn_stats_finalize_v(const float* p0, const float* p1, int splits, int C, int64_t rows, const void* x,
                                    be_dtype dt, float eps, float* mean, float* invstd, float* run_mean,
                                    float* run_var, float momentum) {
  pdl_entry();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double s1 = 0, s2 = 0;
  for (int i = 0; i < splits; ++i) { s1 += p0[(int64_t)i * C + c]; s2 += p1[(int64_t)i * C + c]; }
  const double n = (double)rows;
  const double ms = s1 / n;
  double var = s2 / n - ms * ms;  // biased (normalisation)
  if (var < 0) var = 0;
  const float mu = ld(x, c, dt) + (float)ms;
  mean[c] = mu;
  invstd[c] = rsqrtf((float)var + eps);
  if (run_mean) run_mean[c] = (1.f - momentum) * run_mean[c] + momentum * mu;
  if (run_var) run_var[c] = (1.f - momentum) * run_var[c] + momentum * (float)(var * n / (rows > 1 ? n - 1 : 1));
}
// Element-wise BN kernels with a 2-D mapping: thread t owns channel vector
// t % lanes for the whole launch (per-channel constants live in registers)
// and walks rows (t / lanes) + k·rpi of its row block.
__global__ void __launch_bounds__(256) bn_apply_v(const void* __restrict__ x, void* __restrict__ y, int64_t rows,
                                                  int C, be_dtype dt, const float* __restrict__ mean,
                                                  const float* __restrict__ invstd, const float* __restrict__ gamma,
                                                  const float* __restrict__ beta, int act, int64_t rows_per_block,
                                                  const void* __restrict__ res) {
  pdl_entry();
  const int base = blockIdx.x * kBnCG;
  const int Cg = min(kBnCG, C - base);
  const int lanes = Cg / 8, rpi = 256 / lanes;
  const int t = threadIdx.x, v = t % lanes, rl = t / lanes;
  if (rl >= rpi) return;
  const int c = base + v * 8;
  float sc[8], sh[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sc[j] = gamma[c + j] * invstd[c + j];
    sh[j] = beta[c + j] - mean[c + j] * sc[j];
  }
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  auto row = [&](int64_t o, V8 a, const V8& rr) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float val = fmaf(a.v[j], sc[j], sh[j]);
      if (res) val += rr.v[j];  // fused residual add (ResNet block output)
      a.v[j] = act_apply(val, act);
    }
    st8(y, o, dt, a);
  };
  for (int64_t r = r0 + rl; r < r1; r += 2 * rpi) {
    const bool two = r + rpi < r1;
    const int64_t o0 = r * C + c, o1 = two ? o0 + (int64_t)rpi * C : o0;
    V8 a0 = ld8(x, o0, dt), a1 = ld8(x, o1, dt), r0v, r1v;
    if (res) { r0v = ld8(res, o0, dt); r1v = ld8(res, o1, dt); }
    row(o0, a0, r0v);
    if (two) row(o1, a1, r1v);
  }
}
__global__ void __launch_bounds__(256) bn_dx_v(const void* __restrict__ gy, const void* __restrict__ x,
                                               const void* __restrict__ yv, int act, void* dx, int64_t rows, int C,
                                               be_dtype dt, const float* __restrict__ mean,
                                               const float* __restrict__ invstd, const float* __restrict__ gamma,
                                               const float* __restrict__ sums, float dx_beta, int64_t rows_per_block,
                                               const float* __restrict__ bsh = nullptr) {
  pdl_entry();
  const int base = blockIdx.x * kBnCG;
  const int Cg = min(kBnCG, C - base);
  const int lanes = Cg / 8, rpi = 256 / lanes;
  const int t = threadIdx.x, v = t % lanes, rl = t / lanes;
  if (rl >= rpi) return;
  const int c = base + v * 8;
  // dx = γ·is·(g' − Σg'/n − x̂·Σg'x̂/n),  x̂ = (x − μ)·is   ⇒  dx = k1·g' + k2·x + k3
  const float inv_n = 1.f / (float)rows;
  float k1[8], k2[8], k3[8], sc[8], sh[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float is = invstd[c + j], a = gamma[c + j] * is;
    sc[j] = a;
    sh[j] = bsh ? bsh[c + j] - mean[c + j] * a : 0.f;
    const float m1 = sums[c + j] * inv_n, m2 = sums[C + c + j] * inv_n;
    k1[j] = a;
    k2[j] = -a * m2 * is;
    k3[j] = -a * m1 + a * m2 * is * mean[c + j];
  }
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  auto row = [&](int64_t o, V8 g, const V8& a, const V8& yy, const V8& prev) {
    if (act && bsh) {
#pragma unroll
      for (int j = 0; j < 8; ++j) g.v[j] = act_pass_st(fmaf(a.v[j], sc[j], sh[j]), act, dt == BE_BF16) ? g.v[j] : 0.f;
    } else if (act) {
#pragma unroll
      for (int j = 0; j < 8; ++j) g.v[j] = act_pass(yy.v[j], act) ? g.v[j] : 0.f;
    }
    V8 out;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float val = fmaf(k1[j], g.v[j], fmaf(k2[j], a.v[j], k3[j]));
      out.v[j] = val + (dx_beta != 0.f ? prev.v[j] : 0.f);
    }
    st8(dx, o, dt, out);
  };
  // two rows per iteration, loads first (bytes in flight)
  for (int64_t r = r0 + rl; r < r1; r += 2 * rpi) {
    const bool two = r + rpi < r1;
    const int64_t o0 = r * C + c, o1 = two ? o0 + (int64_t)rpi * C : o0;
    V8 g0 = ld8(gy, o0, dt), a0 = ld8(x, o0, dt), g1 = ld8(gy, o1, dt), a1 = ld8(x, o1, dt), y0, y1, p0, p1;
    if (act && !bsh) { y0 = ld8(yv, o0, dt); y1 = ld8(yv, o1, dt); }
    if (dx_beta != 0.f) { p0 = ld8(dx, o0, dt); p1 = ld8(dx, o1, dt); }
    row(o0, g0, a0, y0, p0);
    if (two) row(o1, g1, a1, y1, p1);
  }
}
// ---- bf16 fast paths of the BN backward (the ResNet case): raw 16-B loads
// (4 registers per 8 values instead of 8) for 4 rows per iteration, issued
// before any arithmetic: twice the bytes in flight of the generic kernels at
// the same occupancy.  Same per-element arithmetic and summation structure
// per row as the generic kernels (reduce: each thread's rows in order).
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = (uint32_t)f2bf(f[2 * i]) | ((uint32_t)f2bf(f[2 * i + 1]) << 16);
  return make_uint4(w[0], w[1], w[2], w[3]);
}
constexpr int kBnU = 4;  // rows per iteration in the bf16 fast paths

// Σg', Σg'·x̂ (g' = gy masked by act(γx̂+β) > 0 recomputed from x when act)
__global__ void __launch_bounds__(256) bn_reduce_bf16(const uint16_t* __restrict__ x, const uint16_t* __restrict__ gy,
                                                      int act, int64_t rows, int C, const float* __restrict__ mean,
                                                      const float* __restrict__ invstd, float* __restrict__ part0,
                                                      float* __restrict__ part1, int64_t rows_per_split,
                                                      const float* __restrict__ gam, const float* __restrict__ bsh,
                                                      const uint16_t* __restrict__ rmask = nullptr,
                                                      uint16_t* __restrict__ gout = nullptr) {
  pdl_entry();
  __shared__ float sm0[kBnCG], sm1[kBnCG];
  const int base = blockIdx.x * kBnCG;
  const int Cg = min(kBnCG, C - base);
  const int lanes = Cg / 8, rpi = 256 / lanes;
  const int t = threadIdx.x, v = t % lanes, rl = t / lanes;
  const int c = base + v * 8;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split, r1 = min(rows, r0 + rows_per_split);
  float s0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, s1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (rl < rpi) {
    float k[8], is[8], sc[8], sh[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      k[j] = mean[c + j]; is[j] = invstd[c + j];
      sc[j] = act ? gam[c + j] * is[j] : 0.f;
      sh[j] = act ? bsh[c + j] - k[j] * sc[j] : 0.f;
    }
    for (int64_t r = r0 + rl; r < r1; r += kBnU * rpi) {
      uint4 xa[kBnU], ga[kBnU], ma[kBnU];
#pragma unroll
      for (int u = 0; u < kBnU; ++u) {
        const int64_t rr = r + (int64_t)u * rpi;
        const int64_t o = (rr < r1 ? rr : r) * C + c;
        xa[u] = *reinterpret_cast<const uint4*>(x + o);
        ga[u] = *reinterpret_cast<const uint4*>(gy + o);
        if (rmask) ma[u] = *reinterpret_cast<const uint4*>(rmask + o);
      }
#pragma unroll
      for (int u = 0; u < kBnU; ++u) {
        if (r + (int64_t)u * rpi >= r1) break;
        float a[8], g[8];
        unpack8(xa[u], a);
        if (rmask) {
          // residual block output y = relu(bn(x) + shortcut): g = gy·1[y > 0]
          // (bf16 y > 0 ⇔ bits in [1, 0x7f80]: positive, finite or +inf, not NaN), stored for the shortcut
          // and the dx pass — the ReLU backward fused into this read of gy
          const uint32_t gw[4] = {ga[u].x, ga[u].y, ga[u].z, ga[u].w};
          const uint32_t mw[4] = {ma[u].x, ma[u].y, ma[u].z, ma[u].w};
          uint32_t ow[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t ml = mw[i] & 0xffffu, mh = mw[i] >> 16;  // y > 0: 0 < bits ≤ +inf (0x7f80)
            const uint32_t lo = ml - 1u < 0x7f80u ? 0x0000ffffu : 0u;
            const uint32_t hi = mh - 1u < 0x7f80u ? 0xffff0000u : 0u;
            ow[i] = gw[i] & (lo | hi);
          }
          ga[u] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
          *reinterpret_cast<uint4*>(gout + (r + (int64_t)u * rpi) * C + c) = ga[u];
        }
        unpack8(ga[u], g);
        if (act) {
#pragma unroll
          for (int j = 0; j < 8; ++j) g[j] = act_pass_st(fmaf(a[j], sc[j], sh[j]), act, true) ? g[j] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) { s0[j] += g[j]; s1[j] += g[j] * (a[j] - k[j]) * is[j]; }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) { sm0[rl * Cg + v * 8 + j] = s0[j]; sm1[rl * Cg + v * 8 + j] = s1[j]; }
  }
  __syncthreads();
  for (int i = t; i < Cg; i += 256) {
    float a0 = 0.f, a1 = 0.f;
    for (int w = 0; w < rpi; ++w) { a0 += sm0[w * Cg + i]; a1 += sm1[w * Cg + i]; }
    part0[(int64_t)blockIdx.y * C + base + i] = a0;
    part1[(int64_t)blockIdx.y * C + base + i] = a1;
  }
}

// dx (+)= k1·g' + k2·x + k3
__global__ void __launch_bounds__(256) bn_dx_bf16(const uint16_t* __restrict__ gy, const uint16_t* __restrict__ x,
                                                  int act, uint16_t* dx, int64_t rows, int C,
                                                  const float* __restrict__ mean, const float* __restrict__ invstd,
                                                  const float* __restrict__ gamma, const float* __restrict__ sums,
                                                  float dx_beta, int64_t rows_per_block, const float* __restrict__ bsh) {
  pdl_entry();
  const int base = blockIdx.x * kBnCG;
  const int Cg = min(kBnCG, C - base);
  const int lanes = Cg / 8, rpi = 256 / lanes;
  const int t = threadIdx.x, v = t % lanes, rl = t / lanes;
  if (rl >= rpi) return;
  const int c = base + v * 8;
  const float inv_n = 1.f / (float)rows;
  float k1[8], k2[8], k3[8], sc[8], sh[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float is = invstd[c + j], a = gamma[c + j] * is;
    sc[j] = a;
    sh[j] = act ? bsh[c + j] - mean[c + j] * a : 0.f;
    const float m1 = sums[c + j] * inv_n, m2 = sums[C + c + j] * inv_n;
    k1[j] = a;
    k2[j] = -a * m2 * is;
    k3[j] = -a * m1 + a * m2 * is * mean[c + j];
  }
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  for (int64_t r = r0 + rl; r < r1; r += kBnU * rpi) {
    uint4 ga[kBnU], xa[kBnU], pa[kBnU];
#pragma unroll
    for (int u = 0; u < kBnU; ++u) {
      const int64_t rr = r + (int64_t)u * rpi;
      const int64_t o = (rr < r1 ? rr : r) * C + c;
      ga[u] = *reinterpret_cast<const uint4*>(gy + o);
      xa[u] = *reinterpret_cast<const uint4*>(x + o);
      if (dx_beta != 0.f) pa[u] = *reinterpret_cast<const uint4*>(dx + o);
    }
#pragma unroll
    for (int u = 0; u < kBnU; ++u) {
      const int64_t rr = r + (int64_t)u * rpi;
      if (rr >= r1) break;
      float g[8], a[8], o8[8];
      unpack8(ga[u], g);
      unpack8(xa[u], a);
      if (act) {
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = act_pass_st(fmaf(a[j], sc[j], sh[j]), act, true) ? g[j] : 0.f;
      }
      float pv[8];
      if (dx_beta != 0.f) unpack8(pa[u], pv);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float val = fmaf(k1[j], g[j], fmaf(k2[j], a[j], k3[j]));
        o8[j] = val + (dx_beta != 0.f ? pv[j] : 0.f);
      }
      *reinterpret_cast<uint4*>(dx + rr * C + c) = pack8(o8);
    }
  }
}

// forward statistics, bf16: shifted sums Σ(x−K), Σ(x−K)² with K = x[0,c]
__global__ void __launch_bounds__(256) bn_stats_bf16(const uint16_t* __restrict__ x, int64_t rows, int C,
                                                     float* __restrict__ part0, float* __restrict__ part1,
                                                     int64_t rows_per_split) {
  pdl_entry();
  __shared__ float sm0[kBnCG], sm1[kBnCG];
  const int base = blockIdx.x * kBnCG;
  const int Cg = min(kBnCG, C - base);
  const int lanes = Cg / 8, rpi = 256 / lanes;
  const int t = threadIdx.x, v = t % lanes, rl = t / lanes;
  const int c = base + v * 8;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split, r1 = min(rows, r0 + rows_per_split);
  float s0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, s1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (rl < rpi) {
    float k[8];
    unpack8(*reinterpret_cast<const uint4*>(x + c), k);
    for (int64_t r = r0 + rl; r < r1; r += kBnU * rpi) {
      uint4 xa[kBnU];
#pragma unroll
      for (int u = 0; u < kBnU; ++u) {
        const int64_t rr = r + (int64_t)u * rpi;
        xa[u] = *reinterpret_cast<const uint4*>(x + (rr < r1 ? rr : r) * C + c);
      }
#pragma unroll
      for (int u = 0; u < kBnU; ++u) {
        if (r + (int64_t)u * rpi >= r1) break;
        float a[8];
        unpack8(xa[u], a);
#pragma unroll
        for (int j = 0; j < 8; ++j) { const float d = a[j] - k[j]; s0[j] += d; s1[j] += d * d; }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) { sm0[rl * Cg + v * 8 + j] = s0[j]; sm1[rl * Cg + v * 8 + j] = s1[j]; }
  }
  __syncthreads();
  for (int i = t; i < Cg; i += 256) {
    float a0 = 0.f, a1 = 0.f;
    for (int w = 0; w < rpi; ++w) { a0 += sm0[w * Cg + i]; a1 += sm1[w * Cg + i]; }
    part0[(int64_t)blockIdx.y * C + base + i] = a0;
    part1[(int64_t)blockIdx.y * C + base + i] = a1;
  }
}

// y = act(γ·x̂ + β [+ res]) for bf16, 4 rows in flight per thread
__global__ void __launch_bounds__(256) bn_apply_bf16(const uint16_t* __restrict__ x, uint16_t* __restrict__ y,
                                                     int64_t rows, int C, const float* __restrict__ mean,
                                                     const float* __restrict__ invstd, const float* __restrict__ gamma,
                                                     const float* __restrict__ beta, int act, int64_t rows_per_block,
                                                     const uint16_t* __restrict__ res) {
  pdl_entry();
  const int base = blockIdx.x * kBnCG;
  const int Cg = min(kBnCG, C - base);
  const int lanes = Cg / 8, rpi = 256 / lanes;
  const int t = threadIdx.x, v = t % lanes, rl = t / lanes;
  if (rl >= rpi) return;
  const int c = base + v * 8;
  float sc[8], sh[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sc[j] = gamma[c + j] * invstd[c + j];
    sh[j] = beta[c + j] - mean[c + j] * sc[j];
  }
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  for (int64_t r = r0 + rl; r < r1; r += kBnU * rpi) {
    uint4 xa[kBnU], ra[kBnU];
#pragma unroll
    for (int u = 0; u < kBnU; ++u) {
      const int64_t rr = r + (int64_t)u * rpi;
      const int64_t o = (rr < r1 ? rr : r) * C + c;
      xa[u] = *reinterpret_cast<const uint4*>(x + o);
      if (res) ra[u] = *reinterpret_cast<const uint4*>(res + o);
    }
#pragma unroll
    for (int u = 0; u < kBnU; ++u) {
      const int64_t rr = r + (int64_t)u * rpi;
      if (rr >= r1) break;
      float a[8], rv[8];
      unpack8(xa[u], a);
      if (res) unpack8(ra[u], rv);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float val = fmaf(a[j], sc[j], sh[j]);
        if (res) val += rv[j];
        a[j] = act_apply(val, act);
      }
      *reinterpret_cast<uint4*>(y + rr * C + c) = pack8(a);
    }
  }
}

// Cooperative fixed-order finalize: 8 threads per channel each sum a strided
// subset of the split partials, then combine in lane order.
template <int MODE>  // 0: stats, 2: grads
__global__ void __launch_bounds__(1024) bn_finalize_v(const float* __restrict__ p0, const float* __restrict__ p1,
                                                      int splits, int C, int64_t rows, const void* x, be_dtype dt,
                                                      float eps, float* mean, float* invstd, float* run_mean,
                                                      float* run_var, float momentum, float* dgamma, float* dbeta,
                                                      float gb_beta, float* sums) {
  pdl_entry();
  // 8 channels × 128 sub-lanes: each sub-lane sums every 128th split with all
  // its loads in flight (≤ 4 per operand for the usual ≤ 592 splits), then a
  // fixed-order two-level sum over the sub-lanes (deterministic)
  __shared__ double s0[128][9], s1[128][9];
  const int cl = threadIdx.x & 7, sub = threadIdx.x >> 3;
  const int c = blockIdx.x * 8 + cl;
  double a0 = 0, a1 = 0;
  if (c < C) {
    int i = sub;
    for (; i + 384 < splits; i += 512) {
      const float x0 = p0[(int64_t)i * C + c], x1 = p0[(int64_t)(i + 128) * C + c];
      const float x2 = p0[(int64_t)(i + 256) * C + c], x3 = p0[(int64_t)(i + 384) * C + c];
      const float y0 = p1[(int64_t)i * C + c], y1 = p1[(int64_t)(i + 128) * C + c];
      const float y2 = p1[(int64_t)(i + 256) * C + c], y3 = p1[(int64_t)(i + 384) * C + c];
      a0 += (double)x0; a0 += (double)x1; a0 += (double)x2; a0 += (double)x3;
      a1 += (double)y0; a1 += (double)y1; a1 += (double)y2; a1 += (double)y3;
    }
    for (; i < splits; i += 128) { a0 += p0[(int64_t)i * C + c]; a1 += p1[(int64_t)i * C + c]; }
  }
  s0[sub][cl] = a0;
  s1[sub][cl] = a1;
  __syncthreads();
  if (sub < 8) {
    double u0 = 0, u1 = 0;
    for (int k = 0; k < 16; ++k) { u0 += s0[sub * 16 + k][cl]; u1 += s1[sub * 16 + k][cl]; }
    __syncwarp();
    s0[sub * 16][cl] = u0;
    s1[sub * 16][cl] = u1;
  }
  __syncthreads();
  if (sub != 0 || c >= C) return;
  double t0 = 0, t1 = 0;
  for (int k = 0; k < 8; ++k) { t0 += s0[k * 16][cl]; t1 += s1[k * 16][cl]; }
  if (MODE == 0) {
    const double n = (double)rows;
    const double ms = t0 / n;
    double var = t1 / n - ms * ms;  // biased (normalisation)
    if (var < 0) var = 0;
    const float mu = (x ? ld(x, c, dt) : 0.f) + (float)ms;  // x = nullptr: unshifted partials
    mean[c] = mu;
    invstd[c] = rsqrtf((float)var + eps);
    if (run_mean) run_mean[c] = (1.f - momentum) * run_mean[c] + momentum * mu;
    if (run_var) run_var[c] = (1.f - momentum) * run_var[c] + momentum * (float)(var * n / (rows > 1 ? n - 1 : 1));
  } else {
    sums[c] = (float)t0;
    sums[C + c] = (float)t1;
    if (dbeta) dbeta[c] = (float)t0 + (gb_beta != 0.f ? dbeta[c] : 0.f);
    if (dgamma) dgamma[c] = (float)t1 + (gb_beta != 0.f ? dgamma[c] : 0.f);
  }
}

// ---- embedding gather
__global__ void embedding_fwd_kernel(const float* table, int64_t D, const int32_t* ids, int64_t B, void* out,
                                     be_dtype od) {
  pdl_entry();
  const int64_t total = B * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / D, d = i % D;
    st(out, i, od, table[(int64_t)ids[b] * D + d]);
  }
}

// ---- concat / slice along columns
struct ConcatArgs { const void* x[8]; int64_t w[8]; int64_t off[9]; int n; };
__global__ void concat_kernel(ConcatArgs a, int64_t rows, void* y, be_dtype dt) {
  pdl_entry();
  const int64_t W = a.off[a.n];
  const int64_t total = rows * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / W, c = i % W;
    int j = 0;
    while (c >= a.off[j + 1]) ++j;
    st(y, i, dt, ld(a.x[j], r * a.w[j] + (c - a.off[j]), dt));
  }
}
__global__ void slice_kernel(const void* y, int64_t ldy, int64_t col0, int64_t width, int64_t rows, void* x,
                             be_dtype dt, float beta) {
  pdl_entry();
  const int64_t total = rows * width;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / width, c = i % width;
    float v = ld(y, r * ldy + col0 + c, dt);
    if (beta != 0.f) v += ld(x, i, dt);
    st(x, i, dt, v);
  }
}
// ---- max pool, bf16, one block row per output row (n, p): the window's
// input rows are uniform across the block, a thread owns one 8-channel vector
// of one output pixel and issues all R·S ≤ 9 window loads before comparing.
// Selection rule (as maxpool_fwd_v and the oracle): taps in (r, u) order,
// the first maximum wins (−0 == +0), a NaN wins over numbers and the first
// NaN is kept.  The compare runs on packed bf16 pairs (HSETP2 masks + LOP3
// selects of value and 16-bit tap index); a window holding a NaN takes the
// scalar path.
// Thread layout (no run-time divisions): threadIdx.x = channel vector,
// threadIdx.y = output column within the block, grid (Q tiles, P, N);
// STRIDE = 2 (every pool on the path) is a compile-time constant.
template <int STRIDE>
__global__ void __launch_bounds__(256) maxpool_fwd_rows(const uint16_t* __restrict__ x, uint16_t* __restrict__ y,
                                                        uint8_t* __restrict__ am, ConvGeom g) {
  pdl_entry();
  const int stride = STRIDE > 0 ? STRIDE : g.stride;
  const int cv = threadIdx.x;
  const int q = blockIdx.x * blockDim.y + threadIdx.y;
  if (q >= g.Q) return;
  const int n = blockIdx.z, p = blockIdx.y;
  const int h0 = p * stride - g.pad, w0 = q * stride - g.pad;
  // valid taps form the rectangle [r0, r1) × [u0, u1)
  const int r0 = max(0, -h0), r1 = min(g.R, g.H - h0), u0 = max(0, -w0), u1 = min(g.S, g.W - w0);
  uint4 a[9];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int t = r * 3 + u;
      if (r >= r0 && r < r1 && u >= u0 && u < u1)
        a[t] = __ldg(reinterpret_cast<const uint4*>(x + (((int64_t)n * g.H + h0 + r) * g.W + w0 + u) * g.C) + cv);
      else
        a[t] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  uint32_t nan = 0u;
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const uint32_t wv[4] = {a[t].x, a[t].y, a[t].z, a[t].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) nan |= __vcmpgtu2(wv[i] & 0x7fff7fffu, 0x7f807f80u);
  }
  uint32_t bv[4], bi[4];  // best value / tap index, two channels per word
  if (!nan) {
    const int tf = r0 * 3 + u0;  // first valid tap
#pragma unroll
    for (int i = 0; i < 4; ++i) bv[i] = 0u;
    // initialise from the first valid tap (selected by index: registers only)
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      if (t == tf) {
        bv[0] = a[t].x; bv[1] = a[t].y; bv[2] = a[t].z; bv[3] = a[t].w;
      }
    }
    const uint32_t i0 = (uint32_t)(r0 * g.S + u0) * 0x00010001u;
#pragma unroll
    for (int i = 0; i < 4; ++i) bi[i] = i0;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const int r = t / 3, u = t % 3;
      if (!(r >= r0 && r < r1 && u >= u0 && u < u1)) continue;
      const uint32_t ti = (uint32_t)(r * g.S + u) * 0x00010001u;
      const uint32_t wv[4] = {a[t].x, a[t].y, a[t].z, a[t].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 vv = *reinterpret_cast<const __nv_bfloat162*>(&wv[i]);
        __nv_bfloat162 bb = *reinterpret_cast<const __nv_bfloat162*>(&bv[i]);
        const uint32_t m = __hgt2_mask(vv, bb);
        bv[i] = (bv[i] & ~m) | (wv[i] & m);
        bi[i] = (bi[i] & ~m) | (ti & m);
      }
    }
  } else {
    float best[8];
    int bj[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { best[j] = -INFINITY; bj[j] = -1; }
    for (int t = 0; t < 9; ++t) {
      const int r = t / 3, u = t % 3;
      if (!(r >= r0 && r < r1 && u >= u0 && u < u1)) continue;
      float v[8];
      unpack8(a[t], v);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (bj[j] < 0 || v[j] > best[j] || (v[j] != v[j] && best[j] == best[j])) { best[j] = v[j]; bj[j] = r * g.S + u; }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      bv[i] = (uint32_t)f2bf(best[2 * i]) | ((uint32_t)f2bf(best[2 * i + 1]) << 16);
      bi[i] = (uint32_t)bj[2 * i] | ((uint32_t)bj[2 * i + 1] << 16);
    }
  }
  const int64_t o = (((int64_t)n * g.P + p) * g.Q + q) * g.C + cv * 8;
  *reinterpret_cast<uint4*>(y + o) = make_uint4(bv[0], bv[1], bv[2], bv[3]);
  // 16-bit index pairs → 8 bytes
  if (am)
    *reinterpret_cast<uint2*>(am + o) = make_uint2(__byte_perm(bi[0], bi[1], 0x6420), __byte_perm(bi[2], bi[3], 0x6420));
}
// ---- max-pool backward, bf16, one block per input row (n, h): the ≤ 2
// output rows whose windows contain h are uniform across the block; a thread
// owns one 8-channel vector of one input pixel, loads the ≤ 2 × 2 (dy,
// argmax) pairs together and sums the winners in (p, q) order in fp32 (as
// maxpool_bwd_v; losers contribute an exact +0).  Winner test on packed
// bytes (__vcmpeq4), byte masks widened to bf16 lanes with PRMT.  Requires
// R ≤ 2·stride and S ≤ 2·stride.
template <int STRIDE>
__global__ void __launch_bounds__(256) maxpool_bwd_rows(const uint16_t* __restrict__ dy,
                                                        const uint8_t* __restrict__ am, uint16_t* __restrict__ dx,
                                                        ConvGeom g, float beta) {
  pdl_entry();
  const int stride = STRIDE > 0 ? STRIDE : g.stride;
  const int cv = threadIdx.x;
  const int w = blockIdx.x * blockDim.y + threadIdx.y;
  if (w >= g.W) return;
  const int n = blockIdx.z, h = blockIdx.y;
  // (negative numerators: truncation and flooring both clamp to 0 below)
  const int p_lo = max(0, (h + g.pad - g.R + stride) / stride);
  const int p_hi = min(g.P - 1, (h + g.pad) / stride);
  const int q_lo = max(0, (w + g.pad - g.S + stride) / stride);
  const int q_hi = min(g.Q - 1, (w + g.pad) / stride);
  uint4 d[4];
  uint2 pk[4];
  uint32_t widx[4];
  // 64-bit image base once; the ≤ 4 candidates are 32-bit offsets from (p_lo, q_lo)
  const int64_t img = (int64_t)n * g.P * g.Q * g.C;
  const uint16_t* dyi = dy + img;
  const uint8_t* ami = am + img;
  const uint32_t o00 = ((uint32_t)p_lo * g.Q + q_lo) * g.C + cv * 8;
  const int w00 = (h - (p_lo * stride - g.pad)) * g.S + (w - (q_lo * stride - g.pad));
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int dp = c >> 1, dq = c & 1;
    d[c] = make_uint4(0u, 0u, 0u, 0u);
    pk[c] = make_uint2(0xffffffffu, 0xffffffffu);
    widx[c] = 0u;
    if (p_lo + dp <= p_hi && q_lo + dq <= q_hi) {
      const uint32_t o = o00 + (uint32_t)(dp * g.Q + dq) * g.C;
      d[c] = __ldg(reinterpret_cast<const uint4*>(dyi + o));
      pk[c] = __ldg(reinterpret_cast<const uint2*>(ami + o));
      widx[c] = (uint32_t)(w00 - dp * stride * g.S - dq * stride) * 0x01010101u;
    }
  }
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t m0 = __vcmpeq4(pk[c].x, widx[c]), m1 = __vcmpeq4(pk[c].y, widx[c]);
    uint4 v = d[c];
    v.x &= __byte_perm(m0, 0, 0x1100); v.y &= __byte_perm(m0, 0, 0x3322);
    v.z &= __byte_perm(m1, 0, 0x1100); v.w &= __byte_perm(m1, 0, 0x3322);
    float f[8];
    unpack8(v, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += f[j];
  }
  const int64_t o = (((int64_t)n * g.H + h) * g.W + w) * g.C + cv * 8;
  if (beta != 0.f) {
    float old[8];
    unpack8(*reinterpret_cast<const uint4*>(dx + o), old);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += old[j];
  }
  *reinterpret_cast<uint4*>(dx + o) = pack8(acc);
}
// ---- max-pool backward for the 3×3 / stride-2 pools (pad 1: ResNet's; pad 0:
// AlexNet's), one thread per 2×2 quad of input pixels h ∈ {2i−pad, 2i−pad+1}
// (likewise w): the
// quad's pixels are reached only by the windows (p, q) ∈ {i−1, i} × {j−1, j},
// whose (dy, argmax) pairs are loaded once for all four pixels (the per-pixel
// kernel loads ≤ 4 pairs per pixel and was issue-bound).  Each pixel sums
// its winners in (p, q) order in fp32, exactly as maxpool_bwd_rows: bitwise
// the same result.  Tap index of pixel (h, w) in window (p, q) = (h − 2p + 1)·3
// + (w − 2q + 1).
__global__ void __launch_bounds__(256) maxpool_bwd_quad(const uint16_t* __restrict__ dy,
                                                        const uint8_t* __restrict__ am, uint16_t* __restrict__ dx,
                                                        ConvGeom g, float beta) {
  pdl_entry();
  const int cv = threadIdx.x;
  const int j = blockIdx.x * blockDim.y + threadIdx.y;
  if (j > g.Q) return;
  const int n = blockIdx.z, i = blockIdx.y;
  const int64_t img = (int64_t)n * g.P * g.Q * g.C;
  uint4 d[2][2];
  uint2 pk[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int p = i - 1 + a, q = j - 1 + b;
      d[a][b] = make_uint4(0u, 0u, 0u, 0u);
      pk[a][b] = make_uint2(0xffffffffu, 0xffffffffu);
      if (p >= 0 && p < g.P && q >= 0 && q < g.Q) {
        const int64_t o = img + ((int64_t)p * g.Q + q) * g.C + cv * 8;
        d[a][b] = __ldg(reinterpret_cast<const uint4*>(dy + o));
        pk[a][b] = __ldg(reinterpret_cast<const uint2*>(am + o));
      }
    }
#pragma unroll
  for (int dh = 0; dh < 2; ++dh) {
    const int h = 2 * i - g.pad + dh;
    if (h < 0 || h >= g.H) continue;
#pragma unroll
    for (int dw = 0; dw < 2; ++dw) {
      const int w = 2 * j - g.pad + dw;
      if (w < 0 || w >= g.W) continue;
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      // windows reaching (h, w): odd h (dh = 0) ← p = i − 1 (r = 2), p = i (r = 0);
      // even h (dh = 1) ← p = i (r = 1); likewise w — in (p, q) order
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        if (dh == 1 && a == 0) continue;
        const int r = dh == 1 ? 1 : (a == 0 ? 2 : 0);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          if (dw == 1 && b == 0) continue;
          const int u = dw == 1 ? 1 : (b == 0 ? 2 : 0);
          const uint32_t tap = (uint32_t)(r * 3 + u) * 0x01010101u;
          const uint32_t m0 = __vcmpeq4(pk[a][b].x, tap), m1 = __vcmpeq4(pk[a][b].y, tap);
          uint4 v = d[a][b];
          v.x &= __byte_perm(m0, 0, 0x1100); v.y &= __byte_perm(m0, 0, 0x3322);
          v.z &= __byte_perm(m1, 0, 0x1100); v.w &= __byte_perm(m1, 0, 0x3322);
          float f[8];
          unpack8(v, f);
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] += f[k];
        }
      }
      const int64_t o = (((int64_t)n * g.H + h) * g.W + w) * g.C + cv * 8;
      if (beta != 0.f) {
        float old[8];
        unpack8(*reinterpret_cast<const uint4*>(dx + o), old);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += old[k];
      }
      *reinterpret_cast<uint4*>(dx + o) = pack8(acc);
    }
  }
}
// ---- max-pool backward for the 2×2 / stride-2 / pad-0 pool (VGG's): windows do
// not overlap, so one thread per window (8 channels) loads its (dy, index)
// once and writes the window's 4 input pixels (the winner gets dy, the rest
// +0 — the per-pixel kernel's result, each pixel reached by one window)
__global__ void __launch_bounds__(256) maxpool_bwd_2x2(const uint16_t* __restrict__ dy,
                                                       const uint8_t* __restrict__ am, uint16_t* __restrict__ dx,
                                                       ConvGeom g, float beta) {
  pdl_entry();
  const int cv = threadIdx.x;
  const int q = blockIdx.x * blockDim.y + threadIdx.y;
  if (q >= g.Q) return;
  const int n = blockIdx.z, p = blockIdx.y;
  const int64_t o = (((int64_t)n * g.P + p) * g.Q + q) * g.C + cv * 8;
  const uint4 d = __ldg(reinterpret_cast<const uint4*>(dy + o));
  const uint2 pk = __ldg(reinterpret_cast<const uint2*>(am + o));
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int h = 2 * p + a;
    if (h >= g.H) continue;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int w = 2 * q + b;
      if (w >= g.W) continue;
      const uint32_t tap = (uint32_t)(a * 2 + b) * 0x01010101u;
      const uint32_t m0 = __vcmpeq4(pk.x, tap), m1 = __vcmpeq4(pk.y, tap);
      uint4 v = d;
      v.x &= __byte_perm(m0, 0, 0x1100); v.y &= __byte_perm(m0, 0, 0x3322);
      v.z &= __byte_perm(m1, 0, 0x1100); v.w &= __byte_perm(m1, 0, 0x3322);
      const int64_t od = (((int64_t)n * g.H + h) * g.W + w) * g.C + cv * 8;
      if (beta != 0.f) {
        float f[8], old[8];
        unpack8(v, f);
        unpack8(*reinterpret_cast<const uint4*>(dx + od), old);
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = old[k] + f[k];
        *reinterpret_cast<uint4*>(dx + od) = pack8(f);
      } else {
        float f[8];
        unpack8(v, f);
        float z[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) z[k] = 0.f + f[k];  // as the gather kernel: +0 accumulator, one rounding
        *reinterpret_cast<uint4*>(dx + od) = pack8(z);
      }
    }
  }
}
}  // namespace

template <typename T, int VEC>
static void im2col_launch(const void* x, void* cols, int64_t ldc, const ConvGeom& g, int64_t total, cudaStream_t s) {
  const int64_t items = total / ((int64_t)g.R * g.S);
  if (VEC > 1 && items < (1LL << 31)) {  // tap-loop form (total = items · R·S)
    launch_pdl(im2col_taps_kernel<T, VEC>, grid_for(items, 2), 256, 0, s, (const T*)x, (T*)cols, ldc, g,
               (uint32_t)items);
    return;
  }
  const int grid = grid_for(total, UNR);
  if (total < (1LL << 31))
    launch_pdl(im2col_kernel<T, VEC, uint32_t>, grid, 256, 0, s, (const T*)x, (T*)cols, ldc, g, (uint32_t)total);
  else
    launch_pdl(im2col_kernel<T, VEC, int64_t>, grid, 256, 0, s, (const T*)x, (T*)cols, ldc, g, total);
}
void im2col(const void* x, void* cols, int64_t ldc, const ConvGeom& g, be_dtype dt, cudaStream_t s) {
  const int64_t M = (int64_t)g.N * g.P * g.Q;
  if (M == 0) return;
  const int64_t taps = M * g.R * g.S;
  if (dt == BE_BF16 && g.C % 8 == 0) im2col_launch<uint16_t, 8>(x, cols, ldc, g, taps * (g.C / 8), s);
  else if (dt == BE_F32 && g.C % 4 == 0) im2col_launch<float, 4>(x, cols, ldc, g, taps * (g.C / 4), s);
  else if (dt == BE_BF16) im2col_launch<uint16_t, 1>(x, cols, ldc, g, taps * g.C, s);
  else im2col_launch<float, 1>(x, cols, ldc, g, taps * g.C, s);
  after_launch("im2col");
}
void col2im(const void* dcols, int64_t ldc, void* dx, const ConvGeom& g, be_dtype dt, float beta, cudaStream_t s) {
  const int64_t total = (int64_t)g.N * g.H * g.W * g.C;
  if (total == 0) return;
  if (g.C % 8 == 0 && ldc % 8 == 0 && aligned16(dcols) && aligned16(dx)) {
    if (dt == BE_BF16 && g.stride == 2 && g.R == g.S && (g.R == 1 || g.R == 3) && total / 8 < (1LL << 31)) {
      const uint32_t nvec = (uint32_t)(total / 8);
      const int64_t blocks = std::min<int64_t>(((int64_t)nvec + 511) / 512, (int64_t)ctx().num_sms * 8);
      if (g.R == 1)
        launch_pdl(col2im_s2_bf16<1>, (unsigned)blocks, 256, 0, s, (const uint16_t*)dcols, ldc, (uint16_t*)dx, g, beta, nvec);
      else
        launch_pdl(col2im_s2_bf16<3>, (unsigned)blocks, 256, 0, s, (const uint16_t*)dcols, ldc, (uint16_t*)dx, g, beta, nvec);
      after_launch("col2im_s2");
      return;
    }
    if (total / 8 < (1LL << 31))
      launch_pdl(col2im_v<uint32_t>, grid_for(total / 8), 256, 0, s, dcols, ldc, dx, g, beta, (uint32_t)(total / 8), dt);
    else
      launch_pdl(col2im_v<int64_t>, grid_for(total / 8), 256, 0, s, dcols, ldc, dx, g, beta, total / 8, dt);
    after_launch("col2im_v");
    return;
  }
  if (dt == BE_BF16)
    launch_pdl(col2im_kernel<uint16_t>, grid_for(total), 256, 0, s, (const uint16_t*)dcols, ldc, (uint16_t*)dx, g, beta, total, dt);
  else
    launch_pdl(col2im_kernel<float>, grid_for(total), 256, 0, s, (const float*)dcols, ldc, (float*)dx, g, beta, total, dt);
  after_launch("col2im");
}
void conv_phase_zero(void* dx, const ConvGeom& g, const int* cr, const int* cs, cudaStream_t s) {
  uint32_t live = 0;
  for (int a = 0; a < g.stride; ++a)
    for (int b = 0; b < g.stride; ++b)
      if (cr[a] > 0 && cs[b] > 0) live |= 1u << (a * g.stride + b);
  const int64_t total = (int64_t)g.N * g.H * g.W * (g.C / 8);
  launch_pdl(phase_zero_kernel, grid_for(total), 256, 0, s, (uint16_t*)dx, g, live, total);
  after_launch("conv_phase_zero");
}
void im2col_offsets(const ConvGeom& g, int64_t* out, cudaStream_t s) {
  // the product's im2col kernel (f32 element path) run on an index-encoded input
  const int64_t nx = (int64_t)g.N * g.H * g.W * g.C;
  const int64_t total = (int64_t)g.N * g.P * g.Q * g.R * g.S * g.C;
  if (total == 0) return;
  BE_REQUIRE(nx < (1ll << 31) - 1, BE_E_ARG, "im2col_offsets: input too large for the int32 probe");
  int32_t *x = nullptr, *cols = nullptr;
  BE_CHECK_CUDA(cudaMallocAsync(&x, std::max<int64_t>(nx, 1) * 4, s));
  BE_CHECK_CUDA(cudaMallocAsync(&cols, total * 4, s));
  launch_pdl(iota1_kernel, grid_for(nx), 256, 0, s, x, nx);
  im2col(x, cols, (int64_t)g.R * g.S * g.C, g, BE_F32, s);
  launch_pdl(cols_to_offsets_kernel, grid_for(total), 256, 0, s, (const int32_t*)cols, out, total);
  after_launch("im2col_offsets");
  BE_CHECK_CUDA(cudaFreeAsync(x, s));
  BE_CHECK_CUDA(cudaFreeAsync(cols, s));
}
void maxpool_fwd(const void* x, void* y, uint8_t* am, const ConvGeom& g, be_dtype dt, cudaStream_t s) {
  const int64_t total = (int64_t)g.N * g.P * g.Q * g.C;
  if (total == 0) return;
  if (dt == BE_BF16 && g.C % 8 == 0 && g.R <= 3 && g.S <= 3 && g.C <= 2048 && g.N < 65536 && aligned16(x) &&
      aligned16(y) && (reinterpret_cast<uintptr_t>(am) & 7) == 0) {
    const int cvn = g.C / 8, wpb = std::max(1, 256 / cvn);
    dim3 grid((g.Q + wpb - 1) / wpb, g.P, g.N), block(cvn, wpb);
    if (g.stride == 2) launch_pdl(maxpool_fwd_rows<2>, grid, block, 0, s, (const uint16_t*)x, (uint16_t*)y, am, g);
    else launch_pdl(maxpool_fwd_rows<0>, grid, block, 0, s, (const uint16_t*)x, (uint16_t*)y, am, g);
    after_launch("maxpool_fwd_rows");
    return;
  }
  if (g.C % 8 == 0 && aligned16(x) && aligned16(y) && (reinterpret_cast<uintptr_t>(am) & 7) == 0) {
    if (total / 8 < (1LL << 31))
      launch_pdl(maxpool_fwd_v<uint32_t>, grid_for(total / 8), 256, 0, s, x, y, am, g, dt, (uint32_t)(total / 8));
    else
      launch_pdl(maxpool_fwd_v<int64_t>, grid_for(total / 8), 256, 0, s, x, y, am, g, dt, total / 8);
    after_launch("maxpool_fwd_v");
    return;
  }
  launch_pdl(maxpool_fwd_kernel, grid_for(total), 256, 0, s, x, y, am, g, dt, total);
  after_launch("maxpool_fwd");
}
void maxpool_bwd(const void* dy, const uint8_t* am, void* dx, const ConvGeom& g, be_dtype dt, float beta,
                 cudaStream_t s) {
  const int64_t total = (int64_t)g.N * g.H * g.W * g.C;
  if (total == 0) return;
  if (dt == BE_BF16 && g.C % 8 == 0 && g.R <= 2 * g.stride && g.S <= 2 * g.stride && g.C <= 2048 && g.N < 65536 &&
      (int64_t)g.P * g.Q * g.C < (1LL << 32) &&
      aligned16(dy) && aligned16(dx) && (reinterpret_cast<uintptr_t>(am) & 7) == 0) {
    const int cvn = g.C / 8, wpb = std::max(1, 256 / cvn);
    static const int quad_on = [] { const char* e = getenv("BE_MAXPOOL_QUAD"); return e ? atoi(e) : 1; }();
    if (quad_on && g.R == 2 && g.S == 2 && g.stride == 2 && g.pad == 0 && g.H <= 2 * g.P + 1 && g.W <= 2 * g.Q + 1) {
      // non-overlapping 2×2 windows (pixels past the last window get 0: H odd)
      if (beta == 0.f && (g.H > 2 * g.P || g.W > 2 * g.Q))
        BE_CHECK_CUDA(cudaMemsetAsync(dx, 0, sizeof(uint16_t) * (size_t)total, s));
      dim3 g2((g.Q + wpb - 1) / wpb, g.P, g.N), b2(cvn, wpb);
      launch_pdl(maxpool_bwd_2x2, g2, b2, 0, s, (const uint16_t*)dy, am, (uint16_t*)dx, g, beta);
      after_launch("maxpool_bwd_2x2");
      return;
    }
    if (quad_on && g.R == 3 && g.S == 3 && g.stride == 2 && (g.pad == 1 || g.pad == 0) && g.H <= 2 * g.P + 2 - g.pad &&
        g.W <= 2 * g.Q + 2 - g.pad) {
      // quads i ∈ [0, P], j ∈ [0, Q] cover h ∈ [−pad, 2P − pad + 1] (⊇ [0, H))
      dim3 gq((g.Q + 1 + wpb) / wpb, g.P + 1, g.N), bq(cvn, wpb);
      launch_pdl(maxpool_bwd_quad, gq, bq, 0, s, (const uint16_t*)dy, am, (uint16_t*)dx, g, beta);
      after_launch("maxpool_bwd_quad");
      return;
    }
    dim3 grid((g.W + wpb - 1) / wpb, g.H, g.N), block(cvn, wpb);
    if (g.stride == 2) launch_pdl(maxpool_bwd_rows<2>, grid, block, 0, s, (const uint16_t*)dy, am, (uint16_t*)dx, g, beta);
    else launch_pdl(maxpool_bwd_rows<0>, grid, block, 0, s, (const uint16_t*)dy, am, (uint16_t*)dx, g, beta);
    after_launch("maxpool_bwd_rows");
    return;
  }
  if (g.C % 8 == 0 && aligned16(dy) && aligned16(dx) && (reinterpret_cast<uintptr_t>(am) & 7) == 0) {
    const bool two = g.R <= 2 * g.stride && g.S <= 2 * g.stride;
    const int grid = grid_for(total / 8);
    if (total / 8 < (1LL << 31)) {
      if (two) launch_pdl(maxpool_bwd_v<uint32_t, true>, grid, 256, 0, s, dy, am, dx, g, dt, beta, (uint32_t)(total / 8));
      else launch_pdl(maxpool_bwd_v<uint32_t, false>, grid, 256, 0, s, dy, am, dx, g, dt, beta, (uint32_t)(total / 8));
    } else {
      if (two) launch_pdl(maxpool_bwd_v<int64_t, true>, grid, 256, 0, s, dy, am, dx, g, dt, beta, total / 8);
      else launch_pdl(maxpool_bwd_v<int64_t, false>, grid, 256, 0, s, dy, am, dx, g, dt, beta, total / 8);
    }
    after_launch("maxpool_bwd_v");
    return;
  }
  launch_pdl(maxpool_bwd_kernel, grid_for(total), 256, 0, s, dy, am, dx, g, dt, beta, total);
  after_launch("maxpool_bwd");
}
namespace {
// bf16, C % 8 == 0: one thread per (n, 8-channel vector); HW 16-B loads summed
// in the scalar kernel's order (i ≡ part mod 4 partial sums, combined 0+1+2+3)
__global__ void avgpool_fwd_v8(const uint16_t* __restrict__ x, uint16_t* __restrict__ y, int HW, int C, uint32_t total) {
  pdl_entry();
  const uint32_t CV = (uint32_t)C / 8;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const uint32_t n = t / CV, cv = t - n * CV;
    const uint16_t* xp = x + (int64_t)n * HW * C + cv * 8;
    float a[4][8] = {};
    int i = 0;
    for (; i + 4 <= HW; i += 4) {
      uint4 u[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) u[k] = __ldg(reinterpret_cast<const uint4*>(xp + (int64_t)(i + k) * C));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float v[8];
        unpack8(u[k], v);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[k][j] += v[j];
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (i + k < HW) {
        float v[8];
        unpack8(__ldg(reinterpret_cast<const uint4*>(xp + (int64_t)(i + k) * C)), v);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[k][j] += v[j];
      }
    }
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (a[0][j] + a[1][j] + a[2][j] + a[3][j]) / (float)HW;
    *reinterpret_cast<uint4*>(y + (int64_t)n * C + cv * 8) = pack8(o);
  }
}
// bf16, C % 8 == 0: one thread per (image, 8-channel vector) loads dy once and
// writes it (÷ HW) to the HW pixels (16-B stores; consecutive threads take
// consecutive channel vectors, so each pixel row is written coalesced)
__global__ void avgpool_bwd_v8(const uint16_t* __restrict__ dy, uint16_t* __restrict__ dx, int HW, int C, float beta,
                               uint32_t total) {
  pdl_entry();
  const uint32_t CV = (uint32_t)C / 8;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const uint32_t n = t / CV, cv = t - n * CV;
    float v[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(dy + (int64_t)n * C + cv * 8)), v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] /= (float)HW;
    const uint4 pv = pack8(v);
    uint16_t* base = dx + (int64_t)n * HW * C + cv * 8;
    for (int i = 0; i < HW; ++i) {
      uint4* o = reinterpret_cast<uint4*>(base + (int64_t)i * C);
      if (beta != 0.f) {
        float old[8], w[8];
        unpack8(*o, old);
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = v[j] + old[j];
        *o = pack8(w);
      } else {
        *o = pv;
      }
    }
  }
}
}  // namespace
void avgpool_fwd(const void* x, void* y, int N, int HW, int C, be_dtype dt, cudaStream_t s) {
  if (N == 0 || C == 0) return;
  const int64_t vecs = (int64_t)N * C / 8;
  if (dt == BE_BF16 && C % 8 == 0 && HW > 0 && aligned16(x) && aligned16(y) && vecs < (1LL << 31)) {
    launch_pdl(avgpool_fwd_v8, (int)std::max<int64_t>(1, (vecs + 127) / 128), 128, 0, s, (const uint16_t*)x,
               (uint16_t*)y, HW, C, (uint32_t)vecs);
    after_launch("avgpool_fwd_v8");
    return;
  }
  dim3 grid((C + 63) / 64, N);
  launch_pdl(avgpool_fwd_kernel, grid, 256, 0, s, x, y, HW, C, dt);
  after_launch("avgpool_fwd");
}
void avgpool_bwd(const void* dy, void* dx, int N, int HW, int C, be_dtype dt, float beta, cudaStream_t s) {
  const int64_t total = (int64_t)N * HW * C;
  if (total == 0) return;
  if (dt == BE_BF16 && C % 8 == 0 && aligned16(dy) && aligned16(dx) && total / 8 < (1LL << 31)) {
    const int64_t vecs = (int64_t)N * C / 8;
    launch_pdl(avgpool_bwd_v8, (int)std::max<int64_t>(1, (vecs + 127) / 128), 128, 0, s, (const uint16_t*)dy,
               (uint16_t*)dx, HW, C, beta, (uint32_t)vecs);
    after_launch("avgpool_bwd_v8");
    return;
  }
  launch_pdl(avgpool_bwd_kernel, grid_for(total), 256, 0, s, dy, dx, HW, C, dt, beta, total);
  after_launch("avgpool_bwd");
}

static int64_t bn_splits(int64_t rows, int C) {
  const int64_t cg = (C + 63) / 64;
  int64_t sp = std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, (int64_t)ctx().num_sms * 4 / cg));
  return std::min<int64_t>(sp, 2048);
}
static bool bn_vec_ok(const void* a, int C) { return C % 8 == 0 && aligned16(a); }
// 2-D grid for the element-wise BN kernels: ~16 row-iterations per thread,
// capped at 16 blocks per SM worth of row blocks.
static int64_t bn_rows_per_block(int64_t rows, int C, dim3* grid) {
  const int64_t cg = (C + kBnCG - 1) / kBnCG;
  const int64_t lanes = std::max(1, std::min(C, kBnCG) / 8);
  const int64_t rpi = std::max<int64_t>(1, 256 / lanes);
  int64_t rpb = rpi * 16;
  int64_t nb = (rows + rpb - 1) / rpb;
  const int64_t cap = (int64_t)ctx().num_sms * 16 / cg;
  if (nb > cap) { nb = cap; rpb = (rows + nb - 1) / nb; }
  *grid = dim3((unsigned)cg, (unsigned)std::max<int64_t>(1, nb));
  return rpb;
}
static int64_t bn_splits_v(int64_t rows, int C) {
  const int64_t cg = (C + kBnCG - 1) / kBnCG;
  const int64_t lanes = std::max(1, std::min(C, kBnCG) / 8);
  const int64_t rpi = std::max<int64_t>(1, 256 / lanes);
  // ≥ 8 rows per thread, ≈ 4 blocks per SM
  int64_t sp = std::max<int64_t>(1, std::min<int64_t>(rows / (rpi * 8) + 1, (int64_t)ctx().num_sms * 4 / cg));
  return std::min<int64_t>(sp, 4096);
}
void bn_stats(const void* x, int64_t rows, int C, be_dtype dt, float eps, float* mean, float* invstd, float* partial,
              float* run_mean, float* run_var, float momentum, cudaStream_t s) {
  if (bn_vec_ok(x, C)) {
    int64_t sp = bn_splits_v(rows, C);
    const bool stream = dt == BE_BF16 && bn_stream_ok(x, rows, C);
    if (stream) sp = bn_stream_splits(rows, C, sp);
    const int64_t rps = (rows + sp - 1) / sp;
    dim3 grid((C + kBnCG - 1) / kBnCG, (unsigned)sp);
    if (stream) {
      if (bn_stats_stream(reinterpret_cast<const uint16_t*>(x), rows, C, partial, partial + sp * C, sp, s, eps, mean,
                          invstd, run_mean, run_var, momentum))
        return;
    } else {
      if (dt == BE_BF16)
        launch_pdl(bn_stats_bf16, grid, 256, 0, s, reinterpret_cast<const uint16_t*>(x), rows, C, partial,
                   partial + sp * C, rps);
      else
        launch_pdl(bn_reduce_v<0>, grid, 256, 0, s, x, nullptr, nullptr, 0, rows, C, dt, nullptr, nullptr, partial,
                   partial + sp * C, rps, nullptr, nullptr);
      after_launch("bn_stats_v");
    }
    launch_pdl(bn_finalize_v<0>, (C + 7) / 8, 1024, 0, s, partial, partial + sp * C, (int)sp, C, rows, x, dt, eps, mean,
                                                    invstd, run_mean, run_var, momentum, nullptr, nullptr, 0.f,
                                                    nullptr);
    after_launch("bn_stats_finalize_v");
    return;
  }
  const int64_t sp = bn_splits(rows, C);
  const int64_t rps = (rows + sp - 1) / sp;
  dim3 grid((C + 63) / 64, (unsigned)sp);
  launch_pdl(bn_reduce_kernel<0>, grid, 256, 0, s, x, nullptr, nullptr, 0, rows, C, dt, nullptr, nullptr, partial, nullptr, rps);
  after_launch("bn_sum");
  launch_pdl(bn_mean_finalize, (C + 255) / 256, 256, 0, s, partial, (int)sp, C, rows, mean);
  after_launch("bn_mean");
  launch_pdl(bn_reduce_kernel<1>, grid, 256, 0, s, x, nullptr, nullptr, 0, rows, C, dt, mean, nullptr, partial, nullptr, rps);
  after_launch("bn_sqdev");
  launch_pdl(bn_var_finalize, (C + 255) / 256, 256, 0, s, partial, (int)sp, C, rows, eps, mean, invstd, run_mean, run_var,
                                                  momentum);
  after_launch("bn_var");
}
void bn_stats_from_partials(const float* partial, int parts, int64_t rows, int C, float eps, float* mean,
                            float* invstd, float* run_mean, float* run_var, float momentum, cudaStream_t s) {
  launch_pdl(bn_finalize_v<0>, (C + 7) / 8, 1024, 0, s, partial, partial + (int64_t)parts * C, parts, C, rows, nullptr,
                                                  BE_F32, eps, mean, invstd, run_mean, run_var, momentum, nullptr,
                                                  nullptr, 0.f, nullptr);
  after_launch("bn_stats_from_partials");
}
bool bn_mask_bits_ok(const void* x, const void* y, const void* res, int64_t rows, int C, be_dtype dt) {
  return dt == BE_BF16 && bn_stream_ok(x, rows, C) && aligned16(y) && (!res || aligned16(res));
}
void bn_apply(const void* x, void* y, int64_t rows, int C, be_dtype dt, const float* mean, const float* invstd,
              const float* gamma, const float* beta, int act, cudaStream_t s, const void* res, uint8_t* mbits,
              int early) {
  const int64_t total = rows * C;
  if (total == 0) return;
  if (dt == BE_BF16 && bn_stream_ok(x, rows, C) && aligned16(y) && (!res || aligned16(res))) {
    bn_apply_stream(reinterpret_cast<const uint16_t*>(x), reinterpret_cast<uint16_t*>(y), rows, C, mean, invstd, gamma,
                    beta, act, reinterpret_cast<const uint16_t*>(res), s, mbits, early);
    return;
  }
  if (bn_vec_ok(x, C) && aligned16(y) && (!res || aligned16(res))) {
    dim3 grid;
    const int64_t rpb = bn_rows_per_block(rows, C, &grid);
    if (dt == BE_BF16)
      launch_pdl(bn_apply_bf16, grid, 256, 0, s, reinterpret_cast<const uint16_t*>(x), reinterpret_cast<uint16_t*>(y), rows, C,
                                         mean, invstd, gamma, beta, act, rpb, reinterpret_cast<const uint16_t*>(res));
    else
      launch_pdl(bn_apply_v, grid, 256, 0, s, x, y, rows, C, dt, mean, invstd, gamma, beta, act, rpb, res);
    after_launch("bn_apply_v");
    return;
  }
  launch_pdl(bn_apply_kernel, grid_for(total), 256, 0, s, x, y, total, C, dt, mean, invstd, gamma, beta, act, res);
  after_launch("bn_apply");
}
void bn_bwd(const void* dy, const void* x, const void* y, int act, void* dx, int64_t rows, int C, be_dtype dt,
            const float* mean, const float* invstd, const float* gamma, float* dgamma, float* dbeta, float gb_beta,
            float dx_beta, float* partial, cudaStream_t s, const float* bn_beta, const void* rmask,
            void* gout, const uint8_t* rbits) {
  // partial must hold 2*splits*C + 2*C floats
  BE_REQUIRE(!rbits || (dt == BE_BF16 && bn_stream_ok(x, rows, C)), BE_E_ARG, "bn_bwd: bit mask needs the stream path");
  if (rmask || rbits) {
    // residual output mask: g = dy·1[rmask > 0] into gout, then the BN backward of g
    if (dt == BE_BF16 && !act && bn_vec_ok(x, C) && aligned16(dy) && (rbits || aligned16(rmask)) && aligned16(gout) &&
        (!dx || aligned16(dx))) {
      int64_t sp = bn_splits_v(rows, C);
      const bool stream = bn_stream_ok(x, rows, C);
      if (stream) sp = bn_stream_splits(rows, C, sp);
      const int64_t rps = (rows + sp - 1) / sp;
      float* p0 = partial;
      float* p1 = partial + sp * C;
      float* sums = partial + 2 * sp * C;
      dim3 grid((C + kBnCG - 1) / kBnCG, (unsigned)sp);
      bool folded = false;
      if (stream) {
        folded = bn_reduce_stream(reinterpret_cast<const uint16_t*>(x), reinterpret_cast<const uint16_t*>(dy), 0, rows,
                                  C, mean, invstd, p0, p1, sp, gamma, nullptr,
                                  reinterpret_cast<const uint16_t*>(rmask), reinterpret_cast<uint16_t*>(gout), s, rbits,
                                  sums, dgamma, dbeta, gb_beta);
      } else {
        launch_pdl(bn_reduce_bf16, grid, 256, 0, s, reinterpret_cast<const uint16_t*>(x), reinterpret_cast<const uint16_t*>(dy),
                                            0, rows, C, mean, invstd, p0, p1, rps, gamma, nullptr,
                                            reinterpret_cast<const uint16_t*>(rmask), reinterpret_cast<uint16_t*>(gout));
        after_launch("bn_bwd_reduce_mask_bf16");
      }
      if (!folded) {
        launch_pdl(bn_finalize_v<2>, (C + 7) / 8, 1024, 0, s, p0, p1, (int)sp, C, rows, nullptr, dt, 0.f, nullptr,
                   nullptr, nullptr, nullptr, 0.f, dgamma, dbeta, gb_beta, sums);
        after_launch("bn_bwd_finalize_v");
      }
      if (dx && stream) {
        bn_dx_stream(reinterpret_cast<const uint16_t*>(gout), reinterpret_cast<const uint16_t*>(x), 0,
                     reinterpret_cast<uint16_t*>(dx), rows, C, mean, invstd, gamma, sums, dx_beta, nullptr, s);
      } else if (dx) {
        dim3 g2;
        const int64_t rpb = bn_rows_per_block(rows, C, &g2);
        launch_pdl(bn_dx_bf16, g2, 256, 0, s, reinterpret_cast<const uint16_t*>(gout), reinterpret_cast<const uint16_t*>(x),
                                      0, reinterpret_cast<uint16_t*>(dx), rows, C, mean, invstd, gamma, sums, dx_beta,
                                      rpb, nullptr);
        after_launch("bn_bwd_dx_v");
      }
      return;
    }
    relu_bwd(dy, rmask, gout, rows * C, dt, 0.f, s);
    dy = gout;
  }
  if (bn_vec_ok(x, C) && aligned16(dy) && (!act || bn_beta || aligned16(y)) && (!dx || aligned16(dx))) {
    int64_t sp = bn_splits_v(rows, C);
    const bool fast = dt == BE_BF16 && (!act || bn_beta) && (!dx || aligned16(dx));
    const bool stream = fast && bn_stream_ok(x, rows, C);
    if (stream) sp = bn_stream_splits(rows, C, sp);
    const int64_t rps = (rows + sp - 1) / sp;
    float* p0 = partial;
    float* p1 = partial + sp * C;
    float* sums = partial + 2 * sp * C;
    dim3 grid((C + kBnCG - 1) / kBnCG, (unsigned)sp);
    bool folded = false;
    if (stream)
      folded = bn_reduce_stream(reinterpret_cast<const uint16_t*>(x), reinterpret_cast<const uint16_t*>(dy), act, rows,
                                C, mean, invstd, p0, p1, sp, gamma, bn_beta, nullptr, nullptr, s, nullptr, sums,
                                dgamma, dbeta, gb_beta);
    else if (fast)
      launch_pdl(bn_reduce_bf16, grid, 256, 0, s, reinterpret_cast<const uint16_t*>(x), reinterpret_cast<const uint16_t*>(dy),
                                          act, rows, C, mean, invstd, p0, p1, rps, gamma, bn_beta, nullptr, nullptr);
    else
      launch_pdl(bn_reduce_v<2>, grid, 256, 0, s, x, dy, y, act, rows, C, dt, mean, invstd, p0, p1, rps,
                                          bn_beta ? gamma : nullptr, bn_beta);
    if (!stream) after_launch("bn_bwd_reduce_v");
    if (!folded) {
      launch_pdl(bn_finalize_v<2>, (C + 7) / 8, 1024, 0, s, p0, p1, (int)sp, C, rows, nullptr, dt, 0.f, nullptr,
                 nullptr, nullptr, nullptr, 0.f, dgamma, dbeta, gb_beta, sums);
      after_launch("bn_bwd_finalize_v");
    }
    if (dx && stream) {
      // early: dy and x were written before the reduction just launched (which
      // writes only partial rows / sums)
      bn_dx_stream(reinterpret_cast<const uint16_t*>(dy), reinterpret_cast<const uint16_t*>(x), act,
                   reinterpret_cast<uint16_t*>(dx), rows, C, mean, invstd, gamma, sums, dx_beta, bn_beta, s, 1);
    } else if (dx) {
      dim3 g2;
      const int64_t rpb = bn_rows_per_block(rows, C, &g2);
      if (fast)
        launch_pdl(bn_dx_bf16, g2, 256, 0, s, reinterpret_cast<const uint16_t*>(dy), reinterpret_cast<const uint16_t*>(x), act,
                                      reinterpret_cast<uint16_t*>(dx), rows, C, mean, invstd, gamma, sums, dx_beta, rpb,
                                      bn_beta);
      else
        launch_pdl(bn_dx_v, g2, 256, 0, s, dy, x, y, act, dx, rows, C, dt, mean, invstd, gamma, sums, dx_beta, rpb, bn_beta);
      after_launch("bn_bwd_dx_v");
    }
    return;
  }
  const int64_t sp = bn_splits(rows, C);
  const int64_t rps = (rows + sp - 1) / sp;
  float* p0 = partial;
  float* p1 = partial + sp * C;
  float* sums = partial + 2 * sp * C;
  dim3 grid((C + 63) / 64, (unsigned)sp);
  launch_pdl(bn_reduce_kernel<2>, grid, 256, 0, s, x, dy, y, act, rows, C, dt, mean, invstd, p0, p1, rps);
  after_launch("bn_bwd_reduce");
  launch_pdl(bn_grad_finalize, (C + 255) / 256, 256, 0, s, p0, p1, (int)sp, C, dgamma, dbeta, gb_beta, sums);
  after_launch("bn_bwd_finalize");
  if (dx) {
    const int64_t total = rows * C;
    launch_pdl(bn_dx_kernel, grid_for(total), 256, 0, s, dy, x, y, act, dx, total, C, rows, dt, mean, invstd, gamma, sums,
                                                 dx_beta);
    after_launch("bn_bwd_dx");
  }
}
size_t bn_partial_floats(int64_t rows, int C) {
  return (size_t)(2 * std::max(bn_splits(rows, C), bn_splits_v(rows, C)) * C + 2 * C);
}

void embedding_fwd(const float* table, int64_t D, const int32_t* ids, int64_t B, void* out, be_dtype od,
                   cudaStream_t s) {
  if (B * D == 0) return;
  launch_pdl(embedding_fwd_kernel, grid_for(B * D), 256, 0, s, table, D, ids, B, out, od);
  after_launch("embedding_fwd");
}
void concat_cols(const void* const* xs, const int64_t* widths, int n, int64_t rows, void* y, be_dtype dt,
                 cudaStream_t s) {
  ConcatArgs a{};
  a.n = n;
  a.off[0] = 0;
  for (int i = 0; i < n; ++i) { a.x[i] = xs[i]; a.w[i] = widths[i]; a.off[i + 1] = a.off[i] + widths[i]; }
  if (rows * a.off[n] == 0) return;
  launch_pdl(concat_kernel, grid_for(rows * a.off[n]), 256, 0, s, a, rows, y, dt);
  after_launch("concat");
}
void slice_cols(const void* y, int64_t ldy, int64_t col0, int64_t width, int64_t rows, void* x, be_dtype dt,
                float beta, cudaStream_t s) {
  if (rows * width == 0) return;
  launch_pdl(slice_kernel, grid_for(rows * width), 256, 0, s, y, ldy, col0, width, rows, x, dt, beta);
  after_launch("slice");
}

}}  // namespace be::k
