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
// x NHWC [N,H,W,C], w RSC [3,3,C] fp32, y NHWC [N,P,Q,C]; C % 8 == 0.
// Every kernel runs blocks of C/8 · ⌊256 / (C/8)⌋ threads and strides over
// pixels in multiples of C/8, so a thread owns ONE 8-channel group for its
// whole life: its 9 × 8 filter taps sit in registers, loaded once; per pixel
// the 9 neighbourhood vectors are issued back to back (predicated, fully
// unrolled) before any arithmetic.
__device__ __forceinline__ void ldw8(const float* __restrict__ w, int64_t i, float (&o)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(w + i), b = *reinterpret_cast<const float4*>(w + i + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
// 8 channels as loaded: bf16 stays packed (4 registers) until used
template <bool BF> struct Pk;
template <> struct Pk<true> {
  uint4 u;
  __device__ __forceinline__ float operator[](int j) const {
    const uint32_t w = j < 2 ? u.x : j < 4 ? u.y : j < 6 ? u.z : u.w;
    return __uint_as_float((j & 1) ? (w & 0xffff0000u) : (w << 16));
  }
};
template <> struct Pk<false> {
  float4 a, b;
  __device__ __forceinline__ float operator[](int j) const {
    const float4& h = j < 4 ? a : b;
    const int k = j & 3;
    return k == 0 ? h.x : k == 1 ? h.y : k == 2 ? h.z : h.w;
  }
};
template <bool BF>
__device__ __forceinline__ Pk<BF> ldpk(const void* p, int64_t i, bool ok) {
  Pk<BF> r;
  if constexpr (BF) {
    r.u = ok ? __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p) + i)) : make_uint4(0, 0, 0, 0);
  } else {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    r.a = ok ? __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p) + i)) : z;
    r.b = ok ? __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p) + i) + 1) : z;
  }
  return r;
}
// packed fp32 FMA (sm_100 FFMA2): two independent IEEE fp32 FMAs per
// instruction — per lane exactly fmaf's result, half the FMA issue slots
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  uint64_t d, a, b;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(d0), "f"(d1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}
template <bool BF>
__device__ __forceinline__ void stpk(void* p, int64_t i, const float (&o)[8]) {
  V8 v;
#pragma unroll
  for (int j = 0; j < 8; ++j) v.v[j] = o[j];
  st8(p, i, BF ? BE_BF16 : BE_F32, v);
}

template <int ST, bool BF>
__global__ void __launch_bounds__(256) dw_fwd_kernel(const void* __restrict__ x, const float* __restrict__ w,
                                                     void* __restrict__ y, k::ConvGeom g) {
  pdl_entry();
  const int C8 = g.C >> 3, ppb = blockDim.x / C8;
  if ((int)threadIdx.x >= ppb * C8) return;
  const int c = (threadIdx.x % C8) * 8;
  float wr[9][8];
#pragma unroll
  for (int t = 0; t < 9; ++t) ldw8(w, (int64_t)t * g.C + c, wr[t]);
  const int64_t npix = (int64_t)g.N * g.P * g.Q;
  for (int64_t pix = (int64_t)blockIdx.x * ppb + threadIdx.x / C8; pix < npix; pix += (int64_t)gridDim.x * ppb) {
    const int q = (int)(pix % g.Q);
    const int64_t np_ = pix / g.Q;
    const int p = (int)(np_ % g.P), n = (int)(np_ / g.P);
    const int h0 = p * ST - g.pad, w0 = q * ST - g.pad;
    const int64_t base = (((int64_t)n * g.H + h0) * g.W + w0) * g.C + c;
    Pk<BF> v[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int s2 = 0; s2 < 3; ++s2) {
        const bool ok = (unsigned)(h0 + r) < (unsigned)g.H && (unsigned)(w0 + s2) < (unsigned)g.W;
        v[r * 3 + s2] = ldpk<BF>(x, base + ((int64_t)r * g.W + s2) * g.C, ok);
      }
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int t = 0; t < 9; ++t) ffma2(a0, a1, v[t][j], v[t][j + 1], wr[t][j], wr[t][j + 1]);
      o[j] = a0; o[j + 1] = a1;
    }
    stpk<BF>(y, pix * g.C + c, o);
  }
}

// dx[n,h,w,c] (+)= Σ_{r,s: (h+pad−r), (w+pad−s) divisible by ST, in range} dy[n,p,q,c]·w[r,s,c]
template <int ST, bool BF>
__global__ void __launch_bounds__(256) dw_dgrad_kernel(const void* __restrict__ dy, const float* __restrict__ w,
                                                       void* dx, k::ConvGeom g, float beta) {
  pdl_entry();
  const int C8 = g.C >> 3, ppb = blockDim.x / C8;
  if ((int)threadIdx.x >= ppb * C8) return;
  const int c = (threadIdx.x % C8) * 8;
  float wr[9][8];
#pragma unroll
  for (int t = 0; t < 9; ++t) ldw8(w, (int64_t)t * g.C + c, wr[t]);
  const int64_t npix = (int64_t)g.N * g.H * g.W;
  for (int64_t pix = (int64_t)blockIdx.x * ppb + threadIdx.x / C8; pix < npix; pix += (int64_t)gridDim.x * ppb) {
    const int wc = (int)(pix % g.W);
    const int64_t nh = pix / g.W;
    const int h = (int)(nh % g.H), n = (int)(nh / g.H);
    const int64_t img = (int64_t)n * g.P * g.Q;
    Pk<BF> v[9];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int ph = h + g.pad - r;
      const int p = ph / ST;
      const bool rok = ph >= 0 && (ST == 1 || (ph & 1) == 0) && p < g.P;
#pragma unroll
      for (int s2 = 0; s2 < 3; ++s2) {
        const int qw = wc + g.pad - s2;
        const int q = qw / ST;
        const bool ok = rok && qw >= 0 && (ST == 1 || (qw & 1) == 0) && q < g.Q;
        v[r * 3 + s2] = ldpk<BF>(dy, (img + (int64_t)p * g.Q + q) * g.C + c, ok);
      }
    }
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int t = 0; t < 9; ++t) ffma2(a0, a1, v[t][j], v[t][j + 1], wr[t][j], wr[t][j + 1]);
      o[j] = a0; o[j + 1] = a1;
    }
    if (beta != 0.f) {
      const Pk<BF> prev = ldpk<BF>(dx, pix * g.C + c, true);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] += prev[j];
    }
    stpk<BF>(dx, pix * g.C + c, o);
  }
}

// stride 1, pad 1, 3×3 (forward, and dgrad = the same correlation of dY with
// the taps flipped): a thread owns a column strip of kVR output rows at one
// (n, q, 8 channels) and slides its 3×3 input window down the strip, loading
// the 3 vectors of one new input row per output row instead of 9 (the 9-load
// form is L1-wavefront bound); lanes walk channel groups then q, so every
// warp load is a contiguous run of one input row.
constexpr int kVR = 8;
template <bool BF, bool FLIP>
__global__ void __launch_bounds__(256, 2) dw_s1_strip_kernel(const void* __restrict__ x, const float* __restrict__ w,
                                                             void* y, k::ConvGeom g, float beta) {
  pdl_entry();
  const int C8 = g.C >> 3, ppb = blockDim.x / C8;
  if ((int)threadIdx.x >= ppb * C8) return;
  const int c = (threadIdx.x % C8) * 8;
  float wr[9][8];
#pragma unroll
  for (int t = 0; t < 9; ++t) ldw8(w, (int64_t)(FLIP ? 8 - t : t) * g.C + c, wr[t]);
  const unsigned segs = (g.H + kVR - 1) / kVR;
  const unsigned nitems = (unsigned)g.N * segs * g.W;  // host checks < 2^31
  const int64_t row = (int64_t)g.W * g.C;
  for (unsigned it = blockIdx.x * ppb + threadIdx.x / C8; it < nitems; it += gridDim.x * ppb) {
    const int q = (int)(it % g.W);
    const unsigned ns = it / g.W;
    const int p0 = (int)(ns % segs) * kVR, n = (int)(ns / segs);
    const bool lok = q > 0, rok = q + 1 < g.W;
    const int64_t b = (((int64_t)n * g.H + p0 - 1) * g.W + q) * g.C + c;  // input (p0 − 1, q)
    Pk<BF> v[3][3];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const bool ok = p0 - 1 + r >= 0;  // p0 − 1 + r ≤ p0 < H
      v[r + 1][0] = ldpk<BF>(x, b + r * row - g.C, ok && lok);
      v[r + 1][1] = ldpk<BF>(x, b + r * row, ok);
      v[r + 1][2] = ldpk<BF>(x, b + r * row + g.C, ok && rok);
    }
    // the next input row is loaded one output row ahead (a rolled loop keeps
    // the window + prefetch + taps in registers: no spills at 2 blocks / SM)
    Pk<BF> nx[3];
    {
      const bool ok = p0 + 1 < g.H;
      const int64_t bn = b + 2 * row;
      nx[0] = ldpk<BF>(x, bn - g.C, ok && lok);
      nx[1] = ldpk<BF>(x, bn, ok);
      nx[2] = ldpk<BF>(x, bn + g.C, ok && rok);
    }
    const int tend = min(kVR, g.H - p0);
#pragma unroll 1
    for (int t = 0; t < tend; ++t) {
      const int p = p0 + t;
#pragma unroll
      for (int s2 = 0; s2 < 3; ++s2) { v[0][s2] = v[1][s2]; v[1][s2] = v[2][s2]; v[2][s2] = nx[s2]; }
      {
        const bool ok = p + 2 < g.H;
        const int64_t bn = b + (int64_t)(t + 3) * row;
        nx[0] = ldpk<BF>(x, bn - g.C, ok && lok);
        nx[1] = ldpk<BF>(x, bn, ok);
        nx[2] = ldpk<BF>(x, bn + g.C, ok && rok);
      }
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int tt = 0; tt < 9; ++tt) ffma2(a0, a1, v[tt / 3][tt % 3][j], v[tt / 3][tt % 3][j + 1], wr[tt][j], wr[tt][j + 1]);
        o[j] = a0; o[j + 1] = a1;
      }
      const int64_t oi = b + (int64_t)(t + 1) * row;  // output (p, q): same layout as the input (P = H, Q = W)
      if (beta != 0.f) {
        const Pk<BF> prev = ldpk<BF>(y, oi, true);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] += prev[j];
      }
      stpk<BF>(y, oi, o);
    }
  }
}

// stride 2, pad 1: thread per 2×2 quad of dx, (2i..2i+1, 2j..2j+1).  Row 2i
// takes only tap r = 1 from dy row i; row 2i+1 takes r = 2 from row i and
// r = 0 from row i+1 (same for columns), so the quad reads 4 dy vectors and
// does 9 tap products — the per-pixel kernel above issues 36 predicated loads
// and 36 products (¾ of them zero) and 4 index divisions for the same quad.
template <bool BF>
__global__ void __launch_bounds__(256, 2) dw_dgrad_s2q_kernel(const void* __restrict__ dy, const float* __restrict__ w,
                                                           void* dx, k::ConvGeom g, float beta) {
  pdl_entry();
  const int C8 = g.C >> 3, ppb = blockDim.x / C8;
  if ((int)threadIdx.x >= ppb * C8) return;
  const int c = (threadIdx.x % C8) * 8;
  float wr[9][8];
#pragma unroll
  for (int t = 0; t < 9; ++t) ldw8(w, (int64_t)t * g.C + c, wr[t]);
  const unsigned Hq = (g.H + 1) >> 1, Wq = (g.W + 1) >> 1;
  const unsigned nq = (unsigned)g.N * Hq * Wq;  // host checks < 2^31
  for (unsigned qd = blockIdx.x * ppb + threadIdx.x / C8; qd < nq; qd += gridDim.x * ppb) {
    const unsigned j = qd % Wq, ni = qd / Wq;
    const unsigned i = ni % Hq, n = ni / Hq;
    const bool i1 = (int)i + 1 < g.P, j1 = (int)j + 1 < g.Q;
    const int64_t b00 = (((int64_t)n * g.P + i) * g.Q + j) * g.C + c;
    const Pk<BF> d00 = ldpk<BF>(dy, b00, true), d01 = ldpk<BF>(dy, b00 + g.C, j1),
                 d10 = ldpk<BF>(dy, b00 + (int64_t)g.Q * g.C, i1),
                 d11 = ldpk<BF>(dy, b00 + (int64_t)(g.Q + 1) * g.C, i1 && j1);
    float o00[8], o01[8], o10[8], o11[8];
    // taps t = r·3 + s
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      float a0 = 0.f, a1 = 0.f;
      ffma2(a0, a1, d00[k], d00[k + 1], wr[4][k], wr[4][k + 1]);
      o00[k] = a0; o00[k + 1] = a1;
      a0 = a1 = 0.f;
      ffma2(a0, a1, d00[k], d00[k + 1], wr[5][k], wr[5][k + 1]);
      ffma2(a0, a1, d01[k], d01[k + 1], wr[3][k], wr[3][k + 1]);
      o01[k] = a0; o01[k + 1] = a1;
      a0 = a1 = 0.f;
      ffma2(a0, a1, d00[k], d00[k + 1], wr[7][k], wr[7][k + 1]);
      ffma2(a0, a1, d10[k], d10[k + 1], wr[1][k], wr[1][k + 1]);
      o10[k] = a0; o10[k + 1] = a1;
      a0 = a1 = 0.f;
      ffma2(a0, a1, d00[k], d00[k + 1], wr[8][k], wr[8][k + 1]);
      ffma2(a0, a1, d01[k], d01[k + 1], wr[6][k], wr[6][k + 1]);
      ffma2(a0, a1, d10[k], d10[k + 1], wr[2][k], wr[2][k + 1]);
      ffma2(a0, a1, d11[k], d11[k + 1], wr[0][k], wr[0][k + 1]);
      o11[k] = a0; o11[k + 1] = a1;
    }
    const bool h1 = 2 * (int)i + 1 < g.H, w1 = 2 * (int)j + 1 < g.W;
    const int64_t x00 = (((int64_t)n * g.H + 2 * i) * g.W + 2 * j) * g.C + c, xrow = (int64_t)g.W * g.C;
    if (beta != 0.f) {
      const Pk<BF> p00 = ldpk<BF>(dx, x00, true), p01 = ldpk<BF>(dx, x00 + g.C, w1),
                   p10 = ldpk<BF>(dx, x00 + xrow, h1), p11 = ldpk<BF>(dx, x00 + xrow + g.C, h1 && w1);
#pragma unroll
      for (int k = 0; k < 8; ++k) { o00[k] += p00[k]; o01[k] += p01[k]; o10[k] += p10[k]; o11[k] += p11[k]; }
    }
    stpk<BF>(dx, x00, o00);
    if (w1) stpk<BF>(dx, x00 + g.C, o01);
    if (h1) stpk<BF>(dx, x00 + xrow, o10);
    if (h1 && w1) stpk<BF>(dx, x00 + xrow + g.C, o11);
  }
}

// dw partials: block b sums dy·x over its output-pixel range for every
// (r, s, c); thread (pl, c8) strides the range by ppb pixels with the 9
// neighbourhood loads of a pixel issued together; the block then combines
// its ppb lanes in lane order.  partial[b][(r·3 + s)·C + c].
template <int ST, bool BF>
__global__ void __launch_bounds__(256) dw_wgrad_partial_kernel(const void* __restrict__ dy,
                                                               const void* __restrict__ x, float* __restrict__ part,
                                                               k::ConvGeom g, int64_t pix_per_block) {
  pdl_entry();
  extern __shared__ float red[];
  const int C8 = g.C >> 3, ppb = blockDim.x / C8;
  const int c8 = threadIdx.x % C8, pl = threadIdx.x / C8;
  const int c = c8 * 8;
  const int64_t npq = (int64_t)g.N * g.P * g.Q;
  const int64_t p0 = blockIdx.x * pix_per_block, p1 = min(npq, p0 + pix_per_block);
  float acc[9][8];
#pragma unroll
  for (int k = 0; k < 9; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[k][j] = 0.f;
  if (pl < ppb) {
    for (int64_t pix = p0 + pl; pix < p1; pix += ppb) {
      const int q = (int)(pix % g.Q);
      const int64_t np_ = pix / g.Q;
      const int p = (int)(np_ % g.P), n = (int)(np_ / g.P);
      const int h0 = p * ST - g.pad, w0 = q * ST - g.pad;
      const int64_t base = (((int64_t)n * g.H + h0) * g.W + w0) * g.C + c;
      const Pk<BF> gv = ldpk<BF>(dy, pix * g.C + c, true);
      Pk<BF> v[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s2 = 0; s2 < 3; ++s2) {
          const bool ok = (unsigned)(h0 + r) < (unsigned)g.H && (unsigned)(w0 + s2) < (unsigned)g.W;
          v[r * 3 + s2] = ldpk<BF>(x, base + ((int64_t)r * g.W + s2) * g.C, ok);
        }
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float g0 = gv[j], g1 = gv[j + 1];
#pragma unroll
        for (int t = 0; t < 9; ++t) ffma2(acc[t][j], acc[t][j + 1], g0, g1, v[t][j], v[t][j + 1]);
      }
    }
    float* mine = red + ((int64_t)pl * C8 + c8) * 72;
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int j = 0; j < 8; ++j) mine[t * 8 + j] = acc[t][j];
  }
  __syncthreads();
  const int per = C8 * 72;
  for (int e = threadIdx.x; e < per; e += blockDim.x) {
    float sum = 0.f;
    for (int l = 0; l < ppb; ++l) sum += red[(int64_t)l * per + e];
    const int cc = e / 72, t = (e / 8) % 9, j = e % 8;
    part[(int64_t)blockIdx.x * 9 * g.C + (int64_t)t * g.C + cc * 8 + j] = sum;
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

static int dw_block(int C) {
  const int c8 = C / 8;
  return c8 * std::max(1, 256 / c8);
}
static int dw_grid(int64_t pixels, int C, int per_sm) {
  const int ppb = dw_block(C) / (C / 8);
  const int64_t want = (pixels + ppb - 1) / ppb;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, 148LL * per_sm));
}

static bool dw_strip_ok(const ConvGeom& g) {
  static const bool on = [] { const char* e = getenv("BE_DW_STRIP"); return !e || atoi(e) != 0; }();
  return on && g.stride == 1 && g.pad == 1 && g.P == g.H && g.Q == g.W &&
         (int64_t)g.N * ((g.H + kVR - 1) / kVR) * g.W < (1LL << 31);
}
static int dw_strip_grid(const ConvGeom& g) {
  return dw_grid((int64_t)g.N * ((g.H + kVR - 1) / kVR) * g.W, g.C, 2);
}

void dw_conv_fwd(const void* x, const float* w, void* y, const ConvGeom& g, be_dtype dt, cudaStream_t s) {
  const int64_t npix = (int64_t)g.N * g.P * g.Q;
  if (npix <= 0) return;
  BE_REQUIRE(g.R == 3 && g.S == 3 && (g.stride == 1 || g.stride == 2) && g.C / 8 <= 256, BE_E_UNSUPPORTED,
             "depthwise conv: 3x3, stride 1|2, C <= 2048");
  const bool bf = dt == BE_BF16;
  if (dw_strip_ok(g)) {
    if (bf) launch_pdl(dw_s1_strip_kernel<true, false>, dw_strip_grid(g), dw_block(g.C), 0, s, x, w, y, g, 0.f);
    else launch_pdl(dw_s1_strip_kernel<false, false>, dw_strip_grid(g), dw_block(g.C), 0, s, x, w, y, g, 0.f);
    after_launch("dw_fwd_strip");
    return;
  }
  const int grid = dw_grid(npix, g.C, 16), block = dw_block(g.C);
  if (g.stride == 1 && bf) launch_pdl(dw_fwd_kernel<1, true>, grid, block, 0, s, x, w, y, g);
  else if (g.stride == 1) launch_pdl(dw_fwd_kernel<1, false>, grid, block, 0, s, x, w, y, g);
  else if (bf) launch_pdl(dw_fwd_kernel<2, true>, grid, block, 0, s, x, w, y, g);
  else launch_pdl(dw_fwd_kernel<2, false>, grid, block, 0, s, x, w, y, g);
  after_launch("dw_fwd");
}

void dw_conv_dgrad(const void* dy, const float* w, void* dx, const ConvGeom& g, be_dtype dt, float beta,
                   cudaStream_t s) {
  const int64_t npix = (int64_t)g.N * g.H * g.W;
  if (npix <= 0) return;
  BE_REQUIRE(g.R == 3 && g.S == 3 && (g.stride == 1 || g.stride == 2) && g.C / 8 <= 256, BE_E_UNSUPPORTED,
             "depthwise conv: 3x3, stride 1|2, C <= 2048");
  const bool bf = dt == BE_BF16;
  const int64_t nquad = (int64_t)g.N * ((g.H + 1) / 2) * ((g.W + 1) / 2);
  static const bool quad_on = [] { const char* e = getenv("BE_DW_S2Q"); return !e || atoi(e) != 0; }();
  if (quad_on && g.stride == 2 && g.pad == 1 && nquad < (1LL << 31)) {
    // one wave of resident blocks (2 per SM at <= 128 registers): each
    // thread loads its 72 filter taps once and walks many quads
    // (measured on C7: 301 µs/step for the four stride-2 layers vs 347 µs at
    // 16 blocks per SM and 1089 µs with the per-pixel kernel)
    const int grid = dw_grid(nquad, g.C, 2), block = dw_block(g.C);
    if (bf) launch_pdl(dw_dgrad_s2q_kernel<true>, grid, block, 0, s, dy, w, dx, g, beta);
    else launch_pdl(dw_dgrad_s2q_kernel<false>, grid, block, 0, s, dy, w, dx, g, beta);
    after_launch("dw_dgrad_s2q");
    return;
  }
  if (dw_strip_ok(g)) {  // dx (H×W) = correlation of dY (P×Q = H×W) with the flipped taps
    if (bf) launch_pdl(dw_s1_strip_kernel<true, true>, dw_strip_grid(g), dw_block(g.C), 0, s, dy, w, dx, g, beta);
    else launch_pdl(dw_s1_strip_kernel<false, true>, dw_strip_grid(g), dw_block(g.C), 0, s, dy, w, dx, g, beta);
    after_launch("dw_dgrad_strip");
    return;
  }
  const int grid = dw_grid(npix, g.C, 16), block = dw_block(g.C);
  if (g.stride == 1 && bf) launch_pdl(dw_dgrad_kernel<1, true>, grid, block, 0, s, dy, w, dx, g, beta);
  else if (g.stride == 1) launch_pdl(dw_dgrad_kernel<1, false>, grid, block, 0, s, dy, w, dx, g, beta);
  else if (bf) launch_pdl(dw_dgrad_kernel<2, true>, grid, block, 0, s, dy, w, dx, g, beta);
  else launch_pdl(dw_dgrad_kernel<2, false>, grid, block, 0, s, dy, w, dx, g, beta);
  after_launch("dw_dgrad");
}

static int64_t dw_wgrad_blocks(const ConvGeom& g, int num_sms) {
  const int64_t npq = (int64_t)g.N * g.P * g.Q;
  return std::max<int64_t>(1, std::min<int64_t>(2LL * num_sms, (npq + 255) / 256));
}
size_t dw_wgrad_partial_floats(const ConvGeom& g, int num_sms) {
  return (size_t)dw_wgrad_blocks(g, num_sms) * g.R * g.S * g.C;
}

void dw_conv_wgrad(const void* dy, const void* x, float* dw, float* part, const ConvGeom& g, be_dtype dt,
                   float beta, int num_sms, cudaStream_t s) {
  const int64_t npq = (int64_t)g.N * g.P * g.Q;
  const int RSC = g.R * g.S * g.C;
  BE_REQUIRE(g.R == 3 && g.S == 3 && (g.stride == 1 || g.stride == 2), BE_E_UNSUPPORTED,
             "depthwise conv: 3x3 filters, stride 1|2");
  BE_REQUIRE(g.C / 8 <= 256, BE_E_UNSUPPORTED, "depthwise conv: C <= 2048");
  const int64_t blocks = dw_wgrad_blocks(g, num_sms);
  const int64_t ppb = (npq + blocks - 1) / blocks;
  const int block = dw_block(g.C);
  const size_t smem = (size_t)block * 72 * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dw_wgrad_partial_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(dw_wgrad_partial_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(dw_wgrad_partial_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(dw_wgrad_partial_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  if (npq > 0) {
    const bool bf = dt == BE_BF16;
    if (g.stride == 1 && bf) launch_pdl(dw_wgrad_partial_kernel<1, true>, (unsigned)blocks, block, smem, s, dy, x, part, g, ppb);
    else if (g.stride == 1) launch_pdl(dw_wgrad_partial_kernel<1, false>, (unsigned)blocks, block, smem, s, dy, x, part, g, ppb);
    else if (bf) launch_pdl(dw_wgrad_partial_kernel<2, true>, (unsigned)blocks, block, smem, s, dy, x, part, g, ppb);
    else launch_pdl(dw_wgrad_partial_kernel<2, false>, (unsigned)blocks, block, smem, s, dy, x, part, g, ppb);
    after_launch("dw_wgrad_partial");
  } else {
    cudaMemsetAsync(part, 0, (size_t)blocks * RSC * sizeof(float), s);
  }
  launch_pdl(dw_wgrad_finalize_kernel, (RSC + 255) / 256, 256, 0, s, (const float*)part, (int)blocks, RSC, dw, beta);
  after_launch("dw_wgrad_finalize");
}

}  // namespace k
}  // namespace be
