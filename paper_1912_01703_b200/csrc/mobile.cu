// mobile.cu — the Table 1 CNN extras ("VGG-19", "MobileNet"):
// depthwise convolution over NHWC activations (forward, dgrad, wgrad) and
// inverted dropout whose mask is a counter-based Philox4x64-10 draw,
// regenerated in the backward pass from (seed, offset) — no mask tensor is
// stored or read (oracle: oracle/ops.py conv2d_depthwise, dropout).
//
// All three depthwise passes are HBM-bound streams (one read of each input,
// one write of the output; the R×S neighbourhood re-reads hit L1/L2): a
// thread owns 8 consecutive channels (one 16-B bf16 vector) of one pixel and
// consecutive threads walk consecutive channel groups, so every warp access
// is a contiguous run.  The weight gradient is a fixed-order two-level
// reduction (per-block partials, then one ordered sum per weight):
// deterministic, no atomics.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.h"
#include "runtime.h"

namespace be {
namespace dev {
namespace {

// ------------------------------------------------------------------ Philox4x64-10
// Salmon et al., SC'11; the same generator as oracle/ops.py philox4x64_10
// (written independently from the published round function).
__device__ __forceinline__ void philox4x64_10(uint64_t (&c)[4], uint64_t k0, uint64_t k1) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  constexpr uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += W0; k1 += W1; }
    const uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
}

// y = x · keep · scale for elements 4b .. 4b+3 of block b (one Philox call);
// keep_i = (word_i >> 32) >= thr.  Forward and backward are the same map.
template <typename T>
__global__ void dropout_kernel(const T* __restrict__ x, T* __restrict__ y, int64_t n, uint64_t seed,
                               uint64_t offset, uint64_t thr, float scale, float beta) {
  pdl_entry();
  const int64_t nb = (n + 3) / 4;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c[4] = {(uint64_t)b, offset, 0ull, 0ull};
    philox4x64_10(c, seed, 0ull);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t i = 4 * b + j;
      if (i >= n) break;
      const bool keep = (c[j] >> 32) >= thr;
      float v;
      if constexpr (sizeof(T) == 2) v = bf2f(reinterpret_cast<const uint16_t*>(x)[i]);
      else v = reinterpret_cast<const float*>(x)[i];
      v = keep ? v * scale : 0.f;
      if constexpr (sizeof(T) == 2) {
        if (beta != 0.f) v += bf2f(reinterpret_cast<uint16_t*>(y)[i]);
        reinterpret_cast<uint16_t*>(y)[i] = f2bf(v);
      } else {
        if (beta != 0.f) v += reinterpret_cast<float*>(y)[i];
        reinterpret_cast<float*>(y)[i] = v;
      }
    }
  }
}

// ------------------------------------------------------------------ depthwise conv
// x NHWC [N,H,W,C], w RSC [R,S,C] fp32, y NHWC [N,P,Q,C]; C % 8 == 0
__device__ __forceinline__ void ldw8(const float* __restrict__ w, int64_t i, float (&o)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(w + i), b = *reinterpret_cast<const float4*>(w + i + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}

__global__ void __launch_bounds__(256) dw_fwd_kernel(const void* __restrict__ x, const float* __restrict__ w,
                                                     void* __restrict__ y, k::ConvGeom g, be_dtype dt) {
  pdl_entry();
  const int C8 = g.C >> 3;
  const int64_t total = (int64_t)g.N * g.P * g.Q * C8;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t % C8) * 8;
    int64_t pix = t / C8;
    const int q = (int)(pix % g.Q);
    pix /= g.Q;
    const int p = (int)(pix % g.P);
    const int n = (int)(pix / g.P);
    float acc[8] = {};
    for (int r = 0; r < g.R; ++r) {
      const int h = p * g.stride - g.pad + r;
      if (h < 0 || h >= g.H) continue;
      for (int s = 0; s < g.S; ++s) {
        const int wc = q * g.stride - g.pad + s;
        if (wc < 0 || wc >= g.W) continue;
        const V8 xv = ld8(x, (((int64_t)n * g.H + h) * g.W + wc) * g.C + c, dt);
        float wv[8];
        ldw8(w, (int64_t)(r * g.S + s) * g.C + c, wv);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(xv.v[j], wv[j], acc[j]);
      }
    }
    V8 o;
#pragma unroll
    for (int j = 0; j < 8; ++j) o.v[j] = acc[j];
    st8(y, t * 8, dt, o);
  }
}

// dx[n,h,w,c] (+)= Σ_{r,s: (h+pad−r), (w+pad−s) divisible by stride, in range} dy[n,p,q,c]·w[r,s,c]
__global__ void __launch_bounds__(256) dw_dgrad_kernel(const void* __restrict__ dy, const float* __restrict__ w,
                                                       void* dx, k::ConvGeom g, be_dtype dt, float beta) {
  pdl_entry();
  const int C8 = g.C >> 3;
  const int64_t total = (int64_t)g.N * g.H * g.W * C8;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t % C8) * 8;
    int64_t pix = t / C8;
    const int wc = (int)(pix % g.W);
    pix /= g.W;
    const int h = (int)(pix % g.H);
    const int n = (int)(pix / g.H);
    float acc[8] = {};
    for (int r = 0; r < g.R; ++r) {
      const int ph = h + g.pad - r;
      if (ph < 0 || ph % g.stride) continue;
      const int p = ph / g.stride;
      if (p >= g.P) continue;
      for (int s = 0; s < g.S; ++s) {
        const int qw = wc + g.pad - s;
        if (qw < 0 || qw % g.stride) continue;
        const int q = qw / g.stride;
        if (q >= g.Q) continue;
        const V8 gv = ld8(dy, (((int64_t)n * g.P + p) * g.Q + q) * g.C + c, dt);
        float wv[8];
        ldw8(w, (int64_t)(r * g.S + s) * g.C + c, wv);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(gv.v[j], wv[j], acc[j]);
      }
    }
    V8 o;
    if (beta != 0.f) {
      const V8 prev = ld8(dx, t * 8, dt);
#pragma unroll
      for (int j = 0; j < 8; ++j) o.v[j] = acc[j] + prev.v[j];
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) o.v[j] = acc[j];
    }
    st8(dx, t * 8, dt, o);
  }
}

// dw partials: block b sums dy·x over its output-pixel range for every
// (r, s, c); thread (pl, c8) strides the range by npl pixels; the block then
// combines its npl lanes in lane order.  partial[b][(r·S + s)·C + c].
template <int RS>
__global__ void __launch_bounds__(256) dw_wgrad_partial_kernel(const void* __restrict__ dy,
                                                               const void* __restrict__ x, float* __restrict__ part,
                                                               k::ConvGeom g, be_dtype dt, int64_t ppb) {
  pdl_entry();
  extern __shared__ float red[];
  const int C8 = g.C >> 3, npl = blockDim.x / C8;
  const int c8 = threadIdx.x % C8, pl = threadIdx.x / C8;
  const int c = c8 * 8;
  const int64_t npq = (int64_t)g.N * g.P * g.Q;
  const int64_t p0 = blockIdx.x * ppb, p1 = min(npq, p0 + ppb);
  float acc[RS][8];
#pragma unroll
  for (int k = 0; k < RS; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[k][j] = 0.f;
  if (pl < npl) {
    for (int64_t pix = p0 + pl; pix < p1; pix += npl) {
      const int q = (int)(pix % g.Q);
      const int64_t np_ = pix / g.Q;
      const int p = (int)(np_ % g.P);
      const int n = (int)(np_ / g.P);
      const V8 gv = ld8(dy, pix * g.C + c, dt);
#pragma unroll
      for (int k = 0; k < RS; ++k) {
        const int r = k / g.S, s = k % g.S;
        const int h = p * g.stride - g.pad + r, wc = q * g.stride - g.pad + s;
        if (h < 0 || h >= g.H || wc < 0 || wc >= g.W) continue;
        const V8 xv = ld8(x, (((int64_t)n * g.H + h) * g.W + wc) * g.C + c, dt);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[k][j] = fmaf(gv.v[j], xv.v[j], acc[k][j]);
      }
    }
    float* mine = red + ((int64_t)pl * C8 + c8) * (RS * 8);
#pragma unroll
    for (int k = 0; k < RS; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) mine[k * 8 + j] = acc[k][j];
  }
  __syncthreads();
  const int per = C8 * RS * 8;
  for (int e = threadIdx.x; e < per; e += blockDim.x) {
    float sum = 0.f;
    for (int l = 0; l < npl; ++l) sum += red[(int64_t)l * per + e];
    const int cc = e / (RS * 8), k = (e / 8) % RS, j = e % 8;
    part[(int64_t)blockIdx.x * RS * g.C + (int64_t)k * g.C + cc * 8 + j] = sum;
  }
}

__global__ void __launch_bounds__(256) dw_wgrad_finalize_kernel(const float* __restrict__ part, int parts, int n,
                                                                float* dw, float beta) {
  pdl_entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int b = 0; b < parts; ++b) s += part[(int64_t)b * n + i];
  dw[i] = s + (beta != 0.f ? dw[i] : 0.f);
}

inline int grid_ew(int64_t items) {
  const int64_t b = (items + 255) / 256;
  return (int)std::min<int64_t>(std::max<int64_t>(b, 1), 148LL * 16);
}

}  // namespace
}  // namespace dev

namespace k {
using namespace be::dev;

void dropout_apply(const void* x, void* y, int64_t n, be_dtype dt, uint64_t seed, uint64_t offset, double p,
                   float beta, cudaStream_t s) {
  if (n <= 0) return;
  const uint64_t thr = p >= 1.0 ? (1ull << 32) : (uint64_t)std::floor(p * 4294967296.0);
  const float scale = p >= 1.0 ? 0.f : (float)(1.0 / (1.0 - p));
  const int grid = grid_ew((n + 3) / 4);
  if (dt == BE_BF16)
    launch_pdl(dropout_kernel<uint16_t>, grid, 256, 0, s, reinterpret_cast<const uint16_t*>(x),
               reinterpret_cast<uint16_t*>(y), n, seed, offset, thr, scale, beta);
  else
    launch_pdl(dropout_kernel<float>, grid, 256, 0, s, reinterpret_cast<const float*>(x),
               reinterpret_cast<float*>(y), n, seed, offset, thr, scale, beta);
  after_launch("dropout");
}

void dw_conv_fwd(const void* x, const float* w, void* y, const ConvGeom& g, be_dtype dt, cudaStream_t s) {
  const int64_t items = (int64_t)g.N * g.P * g.Q * (g.C / 8);
  if (items <= 0) return;
  launch_pdl(dw_fwd_kernel, grid_ew(items), 256, 0, s, x, w, y, g, dt);
  after_launch("dw_fwd");
}

void dw_conv_dgrad(const void* dy, const float* w, void* dx, const ConvGeom& g, be_dtype dt, float beta,
                   cudaStream_t s) {
  const int64_t items = (int64_t)g.N * g.H * g.W * (g.C / 8);
  if (items <= 0) return;
  launch_pdl(dw_dgrad_kernel, grid_ew(items), 256, 0, s, dy, w, dx, g, dt, beta);
  after_launch("dw_dgrad");
}

size_t dw_wgrad_partial_floats(const ConvGeom& g, int num_sms) {
  const int64_t npq = (int64_t)g.N * g.P * g.Q;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(4LL * num_sms, (npq + 63) / 64));
  return (size_t)blocks * g.R * g.S * g.C;
}

void dw_conv_wgrad(const void* dy, const void* x, float* dw, float* part, const ConvGeom& g, be_dtype dt,
                   float beta, int num_sms, cudaStream_t s) {
  const int64_t npq = (int64_t)g.N * g.P * g.Q;
  const int RSC = g.R * g.S * g.C;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(4LL * num_sms, (npq + 63) / 64));
  const int64_t ppb = (npq + blocks - 1) / blocks;
  const int C8 = g.C / 8;
  BE_REQUIRE(g.R == 3 && g.S == 3, BE_E_UNSUPPORTED, "depthwise conv: 3x3 filters only");
  BE_REQUIRE(C8 <= 256, BE_E_UNSUPPORTED, "depthwise conv: C <= 2048");
  const int npl = 256 / C8;
  const size_t smem = (size_t)npl * C8 * 9 * 8 * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dw_wgrad_partial_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  if (npq > 0) {
    launch_pdl(dw_wgrad_partial_kernel<9>, (unsigned)blocks, 256, smem, s, dy, x, part, g, dt, ppb);
    after_launch("dw_wgrad_partial");
  } else {
    cudaMemsetAsync(part, 0, (size_t)blocks * RSC * sizeof(float), s);
  }
  launch_pdl(dw_wgrad_finalize_kernel, (RSC + 255) / 256, 256, 0, s, (const float*)part, (int)blocks, RSC, dw, beta);
  after_launch("dw_wgrad_finalize");
}

}  // namespace k
}  // namespace be
