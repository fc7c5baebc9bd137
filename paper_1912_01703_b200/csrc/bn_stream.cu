// bn_stream.cu — batch-norm passes over bf16 NHWC activations as TMA-bulk
// streams (SURVEY §8(a) a5 forward statistics / apply, a9 backward reduce /
// dx; formulas: SURVEY §8(c)-6, oracle/ops.py batchnorm2d).
//
// The four passes are HBM-bound (ResNet-50 b256: 2.85 G activation elements
// per step through BN, ≈48 GB of traffic).  Each block owns a contiguous row
// range [r0, r1) of the [rows, C] tensor (C a multiple of 8, ≤ 2048), i.e. a
// contiguous byte range per input stream: one producer warp moves it into a
// shared-memory ring with 1-D cp.async.bulk copies (ITERS × 4 KB chunks per
// stream, NST stages, mbarrier complete_tx), so ≈64 KB per block (≈190 KB
// per SM) are in flight without any per-thread load issue; 8 consumer warps
// read their 16 B (8 channels of one row: thread t ↔ byte t·16 of every
// ⌊256/(C/8)⌋ rows, ≤ 4 KB; when C/8 does not divide 256 the last
// 256 mod (C/8) consumer threads idle — MobileNetV2's 24 … 1280 channels) from smem.  Outputs (y, dx, the masked gradient) are
// direct 16-B coalesced stores.  Reductions finish with the same fixed-order
// per-block combine as the register kernels (deterministic partials).
#include <cuda_runtime.h>

#include <algorithm>
#include <unordered_map>

#include "common.cuh"
#include "kernels.h"
#include "runtime.h"
#include "sm100.cuh"

namespace be { namespace k {
using namespace be::dev;

namespace {
constexpr int kCons = 256;              // consumer threads (8 warps)
constexpr int kThr = kCons + 32;        // + producer warp
constexpr int kIter = 4096;             // bytes per consumer iteration (16 B per thread)

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(sm100::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void unpack8s(uint4 v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 pack8s(const float (&f)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);  // RN-even
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <int NS, int ITERS, int NST>
struct Ring {
  static constexpr int CH = ITERS * kIter;
  static constexpr int SMEM = NST * NS * CH + 2 * NST * 8 + 128;
};

// Streams rows [r0, r1) of NS bf16 [rows, C] tensors through the ring; body(row,
// v[NS]) runs for each (row, 8-channel group) of this thread.  Returns after the
// last chunk (consumers) / last copy (producer); callers __syncthreads() before
// reusing the ring.
struct NoPre {
  __device__ __forceinline__ void operator()(int64_t) const {}
};
template <int NS, int ITERS, int NST, typename Body, typename Pre = NoPre>
__device__ __forceinline__ void stream_rows(const uint16_t* const (&src)[NS], int64_t r0, int64_t r1, int C,
                                            uint8_t* ring, Body&& body, int64_t ld = 0, Pre&& pre = Pre{}) {
  // ld (row stride, elements) > C: a column group of a wider tensor — one
  // bulk copy per row instead of one per chunk
  if (ld == 0) ld = C;
  using RG = Ring<NS, ITERS, NST>;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + NST * NS * RG::CH);
  uint64_t* empty = full + NST;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int lanes = C >> 3, rpi = kCons / lanes;   // rows per iteration (threads ≥ rpi·lanes idle when C ∤ 2048)
  const int iterb = rpi * C * 2;                    // bytes per iteration (4 KB when C | 2048)
  const int64_t crow = (int64_t)ITERS * rpi;
  const int64_t nchunks = r1 > r0 ? (r1 - r0 + crow - 1) / crow : 0;
  if (warp == kCons / 32) {
    // the producer initialises the ring barriers and signals the consumers
    // through named barrier 1 WITHOUT waiting for them (bar.arrive): with the
    // PDL early start its copies begin while the consumers are still in
    // griddepcontrol.wait
    if (lane == 0) {
      for (int s = 0; s < NST; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], kCons / 32); }
      sm100::fence_barrier_init();
    }
    __syncwarp();
    asm volatile("bar.arrive 1, %0;" ::"n"(kThr) : "memory");
    if (lane == 0) {
      for (int64_t i = 0; i < nchunks; ++i) {
        const int st = (int)(i % NST);
        sm100::mbar_wait(&empty[st], (uint32_t)((i / NST) & 1) ^ 1u);
        const int64_t rs = r0 + i * crow;
        const int nr = (int)min(crow, r1 - rs);
        const uint32_t bytes = (uint32_t)(nr * C * 2);
        sm100::mbar_arrive_expect_tx(&full[st], bytes * NS);
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          if (ld == C) {
            bulk_g2s(sm100::smem_u32(ring + (st * NS + k) * RG::CH), src[k] + rs * C, bytes, &full[st]);
          } else {
            for (int r = 0; r < nr; ++r)
              bulk_g2s(sm100::smem_u32(ring + (st * NS + k) * RG::CH + r * C * 2), src[k] + (rs + r) * ld,
                       (uint32_t)(C * 2), &full[st]);
          }
        }
      }
    }
    return;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kThr) : "memory");
  const int rin = t / lanes;
  const bool active = rin < rpi;
  for (int64_t i = 0; i < nchunks; ++i) {
    const int st = (int)(i % NST);
    pre(i);  // consumer-side loads for chunk i (+1) issued before waiting on the ring
    sm100::mbar_wait(&full[st], (uint32_t)((i / NST) & 1));
    const int64_t rs = r0 + i * crow;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t row = rs + it * rpi + rin;
      if (active && row < r1) {
        uint4 v[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k)
          v[k] = *reinterpret_cast<const uint4*>(ring + (st * NS + k) * RG::CH + it * iterb + t * 16);
        body(row, v);
      }
    }
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(&empty[st]);
  }
}

// fixed-order per-block combine of the consumers' per-row-slot sums → partial row blockIdx.x
__device__ __forceinline__ void combine_partials(const float (&s0)[8], const float (&s1)[8], int C, float* sm,
                                                 float* part0, float* part1, int Ctot = 0, int col0 = 0,
                                                 const float* __restrict__ scale1 = nullptr) {
  if (Ctot == 0) Ctot = C;
  const int t = threadIdx.x, lanes = C >> 3, rpi = kCons / lanes;
  if (t < rpi * lanes) {
    const int v = t % lanes, rl = t / lanes;
#pragma unroll
    for (int j = 0; j < 8; ++j) { sm[rl * C + v * 8 + j] = s0[j]; sm[kCons * 8 + rl * C + v * 8 + j] = s1[j]; }
  }
  __syncthreads();
  for (int i = t; i < C; i += blockDim.x) {
    float a0 = 0.f, a1 = 0.f;
    for (int w = 0; w < rpi; ++w) { a0 += sm[w * C + i]; a1 += sm[kCons * 8 + w * C + i]; }
    part0[(int64_t)blockIdx.x * Ctot + col0 + i] = a0;
    part1[(int64_t)blockIdx.x * Ctot + col0 + i] = scale1 ? a1 * scale1[col0 + i] : a1;
  }
}

// PDL entry of a stream pass whose streamed inputs were NOT written by its
// stream predecessor (early = 1: the apply after the statistics pass / its
// finalize, the dx pass after the backward reduction): the producer warp reads
// only those inputs and writes nothing, so it starts filling the ring without
// griddepcontrol.wait — the copies overlap the predecessor's reduction tail;
// consumers (which read the statistics / sums and write) wait as usual.  The
// inputs' own producers completed before the predecessor passed its wait,
// which is what launched this grid.
__device__ __forceinline__ void pdl_entry_stream(int early) {
  if (!(early && threadIdx.x >= kCons)) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
int early_on() {
  static const int on = [] { const char* e = getenv("BE_PDL_EARLY"); return e ? atoi(e) : 1; }();
  return on;
}

}  // namespace
// Finalize folded into the statistics / reduction pass (replaces the separate
// bn_finalize_v launch).  Every block writes its partial row, takes a ticket;
// the last nf blocks to arrive wait until all partial rows are written (all
// blocks of these grids are co-resident: ≤ 3 per SM, 3 fit) and each reduces
// 8-channel groups g ≡ (ticket − (sp − nf)) (mod nf): 32 sub-lanes per group sum
// every 32nd split in double, combined in sub-lane order — a fixed order, so
// the result does not depend on which blocks arrive last.  The last finalizer
// to depart resets the two counters for the next launch on this stream.
struct BnFin {
  int mode = 0;                 // 0: caller finalizes; 1: statistics; 2: backward sums
  unsigned int* ctr = nullptr;  // [0] arrivals, [1] departures
  int nf = 0;
  int64_t rows = 0;
  const uint16_t* shift = nullptr;  // mode 1: x (row 0 = the shift K)
  float eps = 0.f, momentum = 0.f;
  float* mean = nullptr;
  float* invstd = nullptr;
  float* run_mean = nullptr;
  float* run_var = nullptr;
  float* dgamma = nullptr;
  float* dbeta = nullptr;
  float* sums = nullptr;
  float gb_beta = 0.f;
};
namespace {
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ void fold_finalize(const BnFin& f, const float* __restrict__ p0, const float* __restrict__ p1, int C,
                              uint8_t* smem) {
  __shared__ unsigned int s_ticket;
  const int sp = (int)gridDim.x;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_ticket = atomicAdd(&f.ctr[0], 1u);
  __syncthreads();
  const int first = sp - f.nf;
  if ((int)s_ticket < first) return;
  const int fi = (int)s_ticket - first;
  if (threadIdx.x == 0)
    while (ld_acquire_u32(&f.ctr[0]) < (unsigned)sp) __nanosleep(32);
  __syncthreads();
  double* s0 = reinterpret_cast<double*>(smem);  // [32][8]
  double* s1 = s0 + 256;
  const int t = threadIdx.x, cl = t & 7, sub = t >> 3;
  const int groups = C >> 3;
  for (int g = fi; g < groups; g += f.nf) {
    const int c = g * 8 + cl;
    if (t < 256) {
      double a0 = 0, a1 = 0;
      int i = sub;
      for (; i + 96 < sp; i += 128) {
        const float x0 = __ldcg(p0 + (int64_t)i * C + c), x1 = __ldcg(p0 + (int64_t)(i + 32) * C + c);
        const float x2 = __ldcg(p0 + (int64_t)(i + 64) * C + c), x3 = __ldcg(p0 + (int64_t)(i + 96) * C + c);
        const float y0 = __ldcg(p1 + (int64_t)i * C + c), y1 = __ldcg(p1 + (int64_t)(i + 32) * C + c);
        const float y2 = __ldcg(p1 + (int64_t)(i + 64) * C + c), y3 = __ldcg(p1 + (int64_t)(i + 96) * C + c);
        a0 += (double)x0; a0 += (double)x1; a0 += (double)x2; a0 += (double)x3;
        a1 += (double)y0; a1 += (double)y1; a1 += (double)y2; a1 += (double)y3;
      }
      for (; i < sp; i += 32) { a0 += __ldcg(p0 + (int64_t)i * C + c); a1 += __ldcg(p1 + (int64_t)i * C + c); }
      s0[sub * 8 + cl] = a0;
      s1[sub * 8 + cl] = a1;
    }
    __syncthreads();
    if (t < 8) {
      double t0 = 0, t1 = 0;
      for (int k = 0; k < 32; ++k) { t0 += s0[k * 8 + cl]; t1 += s1[k * 8 + cl]; }
      if (f.mode == 1) {
        const double n = (double)f.rows;
        const double ms = t0 / n;
        double var = t1 / n - ms * ms;  // biased (normalisation)
        if (var < 0) var = 0;
        const float mu = bf2f(f.shift[c]) + (float)ms;
        f.mean[c] = mu;
        f.invstd[c] = rsqrtf((float)var + f.eps);
        if (f.run_mean) f.run_mean[c] = (1.f - f.momentum) * f.run_mean[c] + f.momentum * mu;
        if (f.run_var)
          f.run_var[c] = (1.f - f.momentum) * f.run_var[c] +
                         f.momentum * (float)(var * n / (f.rows > 1 ? n - 1 : 1));
      } else {
        f.sums[c] = (float)t0;
        f.sums[C + c] = (float)t1;
        if (f.dbeta) f.dbeta[c] = (float)t0 + (f.gb_beta != 0.f ? f.dbeta[c] : 0.f);
        if (f.dgamma) f.dgamma[c] = (float)t1 + (f.gb_beta != 0.f ? f.dgamma[c] : 0.f);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&f.ctr[1], 1u) == (unsigned)f.nf - 1u) {
      f.ctr[0] = 0u;
      f.ctr[1] = 0u;
    }
  }
}

// forward statistics: shifted sums Σ(x−K), Σ(x−K)² with K = x[0, c]
__global__ void __launch_bounds__(kThr, 3) bn_stats_stream_kernel(const uint16_t* __restrict__ x, int64_t rows, int C,
                                                               float* part0, float* part1, int64_t rps,
                                                               const __grid_constant__ BnFin fin) {
  pdl_entry();
  extern __shared__ __align__(128) uint8_t ring[];
  const int64_t r0 = (int64_t)blockIdx.x * rps, r1 = min(rows, r0 + rps);
  const int c = (threadIdx.x % (C >> 3)) * 8;
  float k[8], s0[8] = {}, s1[8] = {};
  unpack8s(*reinterpret_cast<const uint4*>(x + c), k);
  const uint16_t* src[1] = {x};
  stream_rows<1, 4, 4>(src, r0, r1, C, ring, [&](int64_t, const uint4 (&v)[1]) {
    float a[8];
    unpack8s(v[0], a);
#pragma unroll
    for (int j = 0; j < 8; ++j) { const float d = a[j] - k[j]; s0[j] += d; s1[j] += d * d; }
  });
  __syncthreads();
  combine_partials(s0, s1, C, reinterpret_cast<float*>(ring), part0, part1);
  if (fin.mode) fold_finalize(fin, part0, part1, C, ring);
}

// backward reduction Σg', Σg'·x̂ (g' = gy masked by act(γx̂+β) > 0 recomputed
// from x when ACT; with rmask: g = gy·1[rmask > 0] written to gout first)
// MASK 1: the residual mask read from the stored block output (bf16 y > 0);
// MASK 2: read from the forward's 1-bit mask (bit j of byte row·C/8 + c/8 =
// channel c + j passed the ReLU) — 1/16 of the bytes of y; the mask bytes of
// chunk i + 1 are loaded while chunk i is consumed (a dependent global load
// per row otherwise stalls every consumer warp on DRAM latency).
// Σg'·(x − μ) is accumulated per thread and scaled by invstd once per column
// when the block's partial row is written (registers: the residual variants
// spilled with the per-thread invstd copy).  ACT is a template parameter so
// the residual variants (ACT 0) carry no ReLU-recompute constants.
template <int MASK, int ACT>
__global__ void __launch_bounds__(kThr, 3) bn_reduce_stream_kernel(const uint16_t* __restrict__ x,
                                                                const uint16_t* __restrict__ gy,
                                                                int64_t rows, int C, const float* __restrict__ mean,
                                                                const float* __restrict__ invstd, float* part0,
                                                                float* part1, int64_t rps,
                                                                const float* __restrict__ gam,
                                                                const float* __restrict__ bsh,
                                                                const uint16_t* __restrict__ rmask,
                                                                uint16_t* __restrict__ gout,
                                                                const uint8_t* __restrict__ rbits,
                                                                const __grid_constant__ BnFin fin) {
  pdl_entry();
  extern __shared__ __align__(128) uint8_t ring[];
  const int64_t r0 = (int64_t)blockIdx.x * rps, r1 = min(rows, r0 + rps);
  const int c = (threadIdx.x % (C >> 3)) * 8;
  float k[8], sc[8], sh[8], s0[8] = {}, s1[8] = {};
  if (threadIdx.x < kCons) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      k[j] = mean[c + j];
      if (ACT) {
        sc[j] = gam[c + j] * invstd[c + j];
        sh[j] = bsh[c + j] - k[j] * sc[j];
      }
    }
  }
  // MASK 2: this thread's mask bytes for the rows of the current / next chunk
  constexpr int IT = 2;  // ITERS of the ring below
  const int lanes = C >> 3, rpi = kCons / lanes, rin = threadIdx.x / lanes;
  const int64_t crow = (int64_t)IT * rpi;
  uint32_t bcur[IT], bnext[IT];
  int64_t cb = r0;  // first row of the chunk being consumed
  auto load_bits = [&](int64_t i, uint32_t (&b)[IT]) {
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int64_t row = r0 + i * crow + it * rpi + rin;
      b[it] = (rin < rpi && row < r1) ? (uint32_t)__ldg(rbits + row * (C >> 3) + (c >> 3)) : 0u;
    }
  };
  if (MASK == 2) load_bits(0, bnext);
  auto pre = [&](int64_t i) {
    if (MASK == 2) {
#pragma unroll
      for (int it = 0; it < IT; ++it) bcur[it] = bnext[it];
      load_bits(i + 1, bnext);
      cb = r0 + i * crow;
    }
  };
  auto body = [&](int64_t row, const uint4* v) {
    float a[8], g[8];
    unpack8s(v[0], a);
    uint4 gv = v[1];
    if (MASK == 2) {
      const uint32_t b = (int)(row - cb - rin) >= rpi ? bcur[1] : bcur[0];
      uint32_t ow[4];
      const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        ow[i] = gw[i] & (((b >> (2 * i)) & 1u ? 0x0000ffffu : 0u) | ((b >> (2 * i + 1)) & 1u ? 0xffff0000u : 0u));
      gv = make_uint4(ow[0], ow[1], ow[2], ow[3]);
      *reinterpret_cast<uint4*>(gout + row * C + c) = gv;
    } else if (MASK == 1) {
      // residual block output y = relu(bn(x) + shortcut): g = gy·1[y > 0]
      // (bf16 y > 0 ⇔ bits in [1, 0x7f80]), stored for the shortcut and dx
      const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w};
      const uint32_t mw[4] = {v[2].x, v[2].y, v[2].z, v[2].w};
      uint32_t ow[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t ml = mw[i] & 0xffffu, mh = mw[i] >> 16;
        const uint32_t lo = ml - 1u < 0x7f80u ? 0x0000ffffu : 0u;
        const uint32_t hi = mh - 1u < 0x7f80u ? 0xffff0000u : 0u;
        ow[i] = gw[i] & (lo | hi);
      }
      gv = make_uint4(ow[0], ow[1], ow[2], ow[3]);
      *reinterpret_cast<uint4*>(gout + row * C + c) = gv;
    }
    unpack8s(gv, g);
    if (ACT) {
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = act_pass_st(fmaf(a[j], sc[j], sh[j]), ACT, true) ? g[j] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) { s0[j] += g[j]; s1[j] = fmaf(g[j], a[j] - k[j], s1[j]); }
  };
  if (MASK == 1) {
    const uint16_t* src[3] = {x, gy, rmask};
    stream_rows<3, 2, 3>(src, r0, r1, C, ring, [&](int64_t row, const uint4 (&v)[3]) { body(row, v); });
  } else {
    const uint16_t* src[2] = {x, gy};
    stream_rows<2, 2, 4>(src, r0, r1, C, ring, [&](int64_t row, const uint4 (&v)[2]) { body(row, v); }, 0, pre);
  }
  __syncthreads();
  combine_partials(s0, s1, C, reinterpret_cast<float*>(ring), part0, part1, 0, 0, invstd);
  if (fin.mode) fold_finalize(fin, part0, part1, C, ring);
}

// y = act(γ·x̂ + β [+ res])
template <bool RES>
__global__ void __launch_bounds__(kThr, 3) bn_apply_stream_kernel(const uint16_t* __restrict__ x, uint16_t* y,
                                                               int64_t rows, int C, const float* __restrict__ mean,
                                                               const float* __restrict__ invstd,
                                                               const float* __restrict__ gamma,
                                                               const float* __restrict__ beta, int act, int64_t rps,
                                                               const uint16_t* __restrict__ res,
                                                               uint8_t* __restrict__ mbits, int early) {
  pdl_entry_stream(early);
  extern __shared__ __align__(128) uint8_t ring[];
  const int64_t r0 = (int64_t)blockIdx.x * rps, r1 = min(rows, r0 + rps);
  const int c = (threadIdx.x % (C >> 3)) * 8;
  float sc[8], sh[8];
  if (threadIdx.x < kCons) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j] = gamma[c + j] * invstd[c + j];
      sh[j] = beta[c + j] - mean[c + j] * sc[j];
    }
  }
  auto body = [&](int64_t row, const uint4* v) {
    float a[8], o[8];
    unpack8s(v[0], a);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = fmaf(a[j], sc[j], sh[j]);
    if (RES) {
      float b[8];
      unpack8s(v[1], b);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] += b[j];
    }
    if (act) {
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = act_apply(o[j], act);
    }
    const uint4 pk = pack8s(o);
    *reinterpret_cast<uint4*>(y + row * C + c) = pk;
    if (mbits) {  // 1-bit mask of the stored value: bf16 bits in [1, 0x7f80] ⇔ y > 0
      const uint32_t w[4] = {pk.x, pk.y, pk.z, pk.w};
      uint32_t b = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        b |= ((w[i] & 0xffffu) - 1u < 0x7f80u ? 1u : 0u) << (2 * i);
        b |= ((w[i] >> 16) - 1u < 0x7f80u ? 1u : 0u) << (2 * i + 1);
      }
      mbits[row * (C >> 3) + (c >> 3)] = (uint8_t)b;
    }
  };
  if (RES) {
    const uint16_t* src[2] = {x, res};
    stream_rows<2, 2, 4>(src, r0, r1, C, ring, [&](int64_t row, const uint4 (&v)[2]) { body(row, v); });
  } else {
    const uint16_t* src[1] = {x};
    stream_rows<1, 4, 4>(src, r0, r1, C, ring, [&](int64_t row, const uint4 (&v)[1]) { body(row, v); });
  }
}

// y = act(γ·x̂ + β + γr·x̂r + βr): the ResNet projection block output with the
// shortcut's batch norm applied on the fly (no residual tensor written / read)
__global__ void __launch_bounds__(kThr, 3) bn_apply2_stream_kernel(const uint16_t* __restrict__ x, uint16_t* y,
                                                                int64_t rows, int C, const float* __restrict__ mean,
                                                                const float* __restrict__ invstd,
                                                                const float* __restrict__ gamma,
                                                                const float* __restrict__ beta, int act, int64_t rps,
                                                                const uint16_t* __restrict__ xr,
                                                                const float* __restrict__ mean_r,
                                                                const float* __restrict__ invstd_r,
                                                                const float* __restrict__ gamma_r,
                                                                const float* __restrict__ beta_r,
                                                                uint8_t* __restrict__ mbits, int early) {
  pdl_entry_stream(early);
  extern __shared__ __align__(128) uint8_t ring[];
  const int64_t r0 = (int64_t)blockIdx.x * rps, r1 = min(rows, r0 + rps);
  const int c = (threadIdx.x % (C >> 3)) * 8;
  float sc[8], sh[8], sr[8];
  if (threadIdx.x < kCons) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j] = gamma[c + j] * invstd[c + j];
      const float scr = gamma_r[c + j] * invstd_r[c + j];
      sr[j] = scr;
      // both shifts folded into one constant
      sh[j] = (beta[c + j] - mean[c + j] * sc[j]) + (beta_r[c + j] - mean_r[c + j] * scr);
    }
  }
  const uint16_t* src[2] = {x, xr};
  stream_rows<2, 2, 4>(src, r0, r1, C, ring, [&](int64_t row, const uint4 (&v)[2]) {
    float a[8], b[8], o[8];
    unpack8s(v[0], a);
    unpack8s(v[1], b);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = fmaf(a[j], sc[j], fmaf(b[j], sr[j], sh[j]));
    if (act) {
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = act_apply(o[j], act);
    }
    const uint4 pk = pack8s(o);
    *reinterpret_cast<uint4*>(y + row * C + c) = pk;
    if (mbits) {
      const uint32_t w[4] = {pk.x, pk.y, pk.z, pk.w};
      uint32_t bb = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        bb |= ((w[i] & 0xffffu) - 1u < 0x7f80u ? 1u : 0u) << (2 * i);
        bb |= ((w[i] >> 16) - 1u < 0x7f80u ? 1u : 0u) << (2 * i + 1);
      }
      mbits[row * (C >> 3) + (c >> 3)] = (uint8_t)bb;
    }
  });
}

// dx (+)= k1·g' + k2·x + k3 (ACT: the ReLU / ReLU6 mask recomputed from x)
template <bool ACC, int ACT>
__global__ void __launch_bounds__(kThr, 3) bn_dx_stream_kernel(const uint16_t* __restrict__ gy,
                                                            const uint16_t* __restrict__ x, uint16_t* dx,
                                                            int64_t rows, int C, const float* __restrict__ mean,
                                                            const float* __restrict__ invstd,
                                                            const float* __restrict__ gamma,
                                                            const float* __restrict__ sums, int64_t rps,
                                                            const float* __restrict__ bsh, int early) {
  pdl_entry_stream(early);
  extern __shared__ __align__(128) uint8_t ring[];
  const int64_t r0 = (int64_t)blockIdx.x * rps, r1 = min(rows, r0 + rps);
  const int c = (threadIdx.x % (C >> 3)) * 8;
  const float inv_n = 1.f / (float)rows;
  float k1[8], k2[8], k3[8], sc[8], sh[8];
  if (threadIdx.x < kCons) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float is = invstd[c + j], a = gamma[c + j] * is;
      sc[j] = a;
      sh[j] = ACT ? bsh[c + j] - mean[c + j] * a : 0.f;
      const float m1 = sums[c + j] * inv_n, m2 = sums[C + c + j] * inv_n;
      k1[j] = a;
      k2[j] = -a * m2 * is;
      k3[j] = -a * m1 + a * m2 * is * mean[c + j];
    }
  }
  auto body = [&](int64_t row, const uint4* v) {
    float g[8], a[8], o[8];
    unpack8s(v[0], g);
    unpack8s(v[1], a);
    if (ACT) {
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = act_pass_st(fmaf(a[j], sc[j], sh[j]), ACT, true) ? g[j] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = fmaf(k1[j], g[j], fmaf(k2[j], a[j], k3[j]));
    if (ACC) {
      float pv[8];
      unpack8s(v[2], pv);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] += pv[j];
    }
    *reinterpret_cast<uint4*>(dx + row * C + c) = pack8s(o);
  };
  if (ACC) {
    const uint16_t* src[3] = {gy, x, dx};
    stream_rows<3, 2, 3>(src, r0, r1, C, ring, [&](int64_t row, const uint4 (&v)[3]) { body(row, v); });
  } else {
    const uint16_t* src[2] = {gy, x};
    stream_rows<2, 2, 4>(src, r0, r1, C, ring, [&](int64_t row, const uint4 (&v)[2]) { body(row, v); });
  }
}

// fused ReLU backward + bias gradient: dz = gy·1[y > 0] (stored), Σ_rows dz per column
// (column group blockIdx.y of width Cg = C / gridDim.y)
__global__ void __launch_bounds__(kThr, 3) relu_colsum_stream_kernel(const uint16_t* __restrict__ gy,
                                                                 const uint16_t* __restrict__ y, uint16_t* dz,
                                                                 int64_t rows, int C, float* part, int64_t rps) {
  pdl_entry();
  extern __shared__ __align__(128) uint8_t ring[];
  const int Cg = C / gridDim.y, col0 = blockIdx.y * Cg;
  const int64_t r0 = (int64_t)blockIdx.x * rps, r1 = min(rows, r0 + rps);
  const int c = col0 + (threadIdx.x % (Cg >> 3)) * 8;
  float s0[8] = {}, s1[8] = {};
  const uint16_t* src[2] = {gy + col0, y + col0};
  stream_rows<2, 2, 4>(src, r0, r1, Cg, ring, [&](int64_t row, const uint4 (&v)[2]) {
    float g[8], m[8];
    unpack8s(v[0], g);
    unpack8s(v[1], m);
#pragma unroll
    for (int j = 0; j < 8; ++j) { g[j] = m[j] > 0.f ? g[j] : 0.f; s0[j] += g[j]; }
    *reinterpret_cast<uint4*>(dz + row * C + c) = pack8s(g);
  }, (int64_t)C);
  __syncthreads();
  combine_partials(s0, s1, Cg, reinterpret_cast<float*>(ring), part, part + (int64_t)gridDim.x * C, C, col0);
}
// out[c] = Σ_split part[split][c] (+ out[c] when beta ≠ 0): 8 columns × 32
// sub-lanes per block, each sub-lane sums every 32nd split, then a fixed-order
// combine over the sub-lanes (deterministic; ~14× fewer dependent loads per
// thread than one thread per column)
__global__ void __launch_bounds__(256) colsum_partials_finalize(const float* __restrict__ part, int splits, int C,
                                                                float* out, float beta) {
  pdl_entry();
  __shared__ float sm[32][9];
  const int cl = threadIdx.x & 7, sub = threadIdx.x >> 3;
  const int c = blockIdx.x * 8 + cl;
  float a0 = 0.f, a1 = 0.f;
  if (c < C) {
    int i = sub;
    for (; i + 32 < splits; i += 64) { a0 += part[(int64_t)i * C + c]; a1 += part[(int64_t)(i + 32) * C + c]; }
    if (i < splits) a0 += part[(int64_t)i * C + c];
  }
  sm[sub][cl] = a0 + a1;
  __syncthreads();
  if (sub == 0 && c < C) {
    float v = 0.f;
    for (int k = 0; k < 32; ++k) v += sm[k][cl];
    out[c] = v + (beta != 0.f ? out[c] : 0.f);
  }
}

template <typename K>
void set_smem(K kern, int bytes) {
  BE_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}
constexpr int kS1 = Ring<1, 4, 4>::SMEM;   // 64 KB ring: 3 blocks per SM
constexpr int kS2 = Ring<2, 2, 4>::SMEM;
constexpr int kS3 = Ring<3, 2, 3>::SMEM;
int stream_blocks(int per_sm) { return ctx().num_sms * per_sm; }
bool enabled() {
  static const int on = [] { const char* e = getenv("BE_BN_STREAM"); return e ? atoi(e) : 1; }();
  return on != 0;
}
}  // namespace

bool bn_stream_ok(const void* a, int64_t rows, int C) {
  return enabled() && C >= 8 && C <= 2048 && C % 8 == 0 && rows > 0 && aligned16(a);
}

bool relu_colsum_stream(const uint16_t* gy, const uint16_t* y, uint16_t* dz, int64_t rows, int C, float* out,
                        float beta, cudaStream_t s) {
  // column groups of ≤ 2048 (one consumer thread per 8 channels)
  const int groups = (C + 2047) / 2048;
  if (!enabled() || C < 8 || C % groups != 0 || (C / groups) % 8 != 0 || rows <= 0 || !aligned16(gy) ||
      !aligned16(y) || !aligned16(dz))
    return false;
  const int Cg = C / groups;
  static bool once = [] { set_smem(relu_colsum_stream_kernel, kS2); return true; }();
  (void)once;
  const int64_t rpi = kCons / (Cg / 8);
  const int64_t crow = 2 * rpi;
  const int64_t sp = std::max<int64_t>(1, std::min<int64_t>(rows / (crow * 4) + 1, stream_blocks(3) / groups));
  const int64_t rps = (rows + sp - 1) / sp;
  Block* tmp = ctx().alloc.allocate(sizeof(float) * 2 * sp * C, s);
  float* part = reinterpret_cast<float*>(tmp->ptr);
  launch_pdl(relu_colsum_stream_kernel, dim3((unsigned)sp, (unsigned)groups), kThr, kS2, s, gy, y, dz, rows, C, part,
             rps);
  after_launch("relu_colsum_stream");
  launch_pdl(colsum_partials_finalize, (C + 7) / 8, 256, 0, s, part, (int)sp, C, out, beta);
  after_launch("relu_colsum_finalize");
  ctx().alloc.free(tmp);
  return true;
}

int64_t bn_stream_splits(int64_t rows, int C, int64_t cap) {
  // ≥ 4 chunks per block; 3 blocks per SM; never more than the caller's partial rows
  const int64_t crow = 4LL * (kCons / (C >> 3));
  int64_t sp = std::min<int64_t>(rows / (crow * 4) + 1, stream_blocks(3));
  return std::max<int64_t>(1, std::min(sp, cap));
}

namespace {
// per-stream arrival / departure counters of the folded finalize (zeroed once;
// every launch leaves them zero)
unsigned int* fin_counters(cudaStream_t s) {
  static std::unordered_map<cudaStream_t, Block*> m;
  auto it = m.find(s);
  if (it != m.end()) return reinterpret_cast<unsigned int*>(it->second->ptr);
  Block* b = ctx().alloc.allocate(64, s);
  BE_CHECK_CUDA(cudaMemsetAsync(b->ptr, 0, 64, s));
  m[s] = b;
  return reinterpret_cast<unsigned int*>(b->ptr);
}
// BE_BN_FOLD=1 folds the finalize into the statistics / reduction pass; off
// by default: under PDL the separate bn_finalize_v launch is cheaper than the
// fold's tail on the critical path (C4 A/B, 3 pairs: 12.40k vs 12.34k mean)
bool fold_on() {
  static const int on = [] { const char* e = getenv("BE_BN_FOLD"); return e ? atoi(e) : 0; }();
  return on != 0;
}
void fin_setup(BnFin& f, int C, int64_t sp, cudaStream_t s) {
  f.ctr = fin_counters(s);
  f.nf = (int)std::min<int64_t>(sp, C / 8);
}
}  // namespace

bool bn_stats_stream(const uint16_t* x, int64_t rows, int C, float* part0, float* part1, int64_t sp, cudaStream_t s,
                     float eps, float* mean, float* invstd, float* run_mean, float* run_var, float momentum) {
  static bool once = [] { set_smem(bn_stats_stream_kernel, kS1); return true; }();
  (void)once;
  const int64_t rps = (rows + sp - 1) / sp;
  BnFin fin;
  if (fold_on() && mean) {
    fin_setup(fin, C, sp, s);
    fin.mode = 1;
    fin.rows = rows; fin.shift = x; fin.eps = eps; fin.momentum = momentum;
    fin.mean = mean; fin.invstd = invstd; fin.run_mean = run_mean; fin.run_var = run_var;
  }
  launch_pdl(bn_stats_stream_kernel, (unsigned)sp, kThr, kS1, s, x, rows, C, part0, part1, rps, fin);
  after_launch("bn_stats_stream");
  return fin.mode != 0;
}

bool bn_reduce_stream(const uint16_t* x, const uint16_t* gy, int act, int64_t rows, int C, const float* mean,
                      const float* invstd, float* part0, float* part1, int64_t sp, const float* gam,
                      const float* bsh, const uint16_t* rmask, uint16_t* gout, cudaStream_t s,
                      const uint8_t* rbits, float* sums, float* dgamma, float* dbeta, float gb_beta) {
  static bool once = [] {
    set_smem(bn_reduce_stream_kernel<0, 0>, kS2);
    set_smem(bn_reduce_stream_kernel<0, 1>, kS2);
    set_smem(bn_reduce_stream_kernel<0, 2>, kS2);
    set_smem(bn_reduce_stream_kernel<1, 0>, kS3);
    set_smem(bn_reduce_stream_kernel<2, 0>, kS2);
    return true;
  }();
  (void)once;
  BE_REQUIRE(act >= 0 && act <= 2 && (act == 0 || (!rbits && !rmask)), BE_E_ARG, "bn_reduce_stream: activation");
  const int64_t rps = (rows + sp - 1) / sp;
  BnFin fin;
  if (fold_on() && sums) {
    fin_setup(fin, C, sp, s);
    fin.mode = 2;
    fin.sums = sums; fin.dgamma = dgamma; fin.dbeta = dbeta; fin.gb_beta = gb_beta;
  }
  auto go = [&](auto kern, int smem, const uint16_t* rm, uint16_t* go_, const uint8_t* rb) {
    launch_pdl(kern, (unsigned)sp, kThr, smem, s, x, gy, rows, C, mean, invstd, part0, part1, rps, gam, bsh, rm, go_,
               rb, fin);
  };
  if (rbits) go(bn_reduce_stream_kernel<2, 0>, kS2, (const uint16_t*)nullptr, gout, rbits);
  else if (rmask) go(bn_reduce_stream_kernel<1, 0>, kS3, rmask, gout, (const uint8_t*)nullptr);
  else if (act == 1) go(bn_reduce_stream_kernel<0, 1>, kS2, (const uint16_t*)nullptr, (uint16_t*)nullptr, (const uint8_t*)nullptr);
  else if (act == 2) go(bn_reduce_stream_kernel<0, 2>, kS2, (const uint16_t*)nullptr, (uint16_t*)nullptr, (const uint8_t*)nullptr);
  else go(bn_reduce_stream_kernel<0, 0>, kS2, (const uint16_t*)nullptr, (uint16_t*)nullptr, (const uint8_t*)nullptr);
  after_launch("bn_reduce_stream");
  return fin.mode != 0;
}

void bn_apply_stream(const uint16_t* x, uint16_t* y, int64_t rows, int C, const float* mean, const float* invstd,
                     const float* gamma, const float* beta, int act, const uint16_t* res, cudaStream_t s,
                     uint8_t* mbits, int early) {
  static bool once = [] {
    set_smem(bn_apply_stream_kernel<false>, kS1);
    set_smem(bn_apply_stream_kernel<true>, kS2);
    return true;
  }();
  (void)once;
  const int64_t sp = bn_stream_splits(rows, C, 1 << 30);
  const int64_t rps = (rows + sp - 1) / sp;
  if (res)
    launch_pdl(bn_apply_stream_kernel<true>, (unsigned)sp, kThr, kS2, s, x, y, rows, C, mean, invstd, gamma, beta, act, rps,
               res, mbits, early && early_on());
  else
    launch_pdl(bn_apply_stream_kernel<false>, (unsigned)sp, kThr, kS1, s, x, y, rows, C, mean, invstd, gamma, beta, act, rps,
               (const uint16_t*)nullptr, mbits, early && early_on());
  after_launch("bn_apply_stream");
}

void bn_apply_stream2(const uint16_t* x, uint16_t* y, int64_t rows, int C, const float* mean, const float* invstd,
                      const float* gamma, const float* beta, int act, const uint16_t* xr, const float* mean_r,
                      const float* invstd_r, const float* gamma_r, const float* beta_r, cudaStream_t s,
                      uint8_t* mbits) {
  static bool once = [] { set_smem(bn_apply2_stream_kernel, kS2); return true; }();
  (void)once;
  const int64_t sp = bn_stream_splits(rows, C, 1 << 30);
  const int64_t rps = (rows + sp - 1) / sp;
  // early: x and xr were written before the statistics kernels just launched
  launch_pdl(bn_apply2_stream_kernel, (unsigned)sp, kThr, kS2, s, x, y, rows, C, mean, invstd, gamma, beta, act, rps, xr,
             mean_r, invstd_r, gamma_r, beta_r, mbits, early_on());
  after_launch("bn_apply2_stream");
}

void bn_dx_stream(const uint16_t* gy, const uint16_t* x, int act, uint16_t* dx, int64_t rows, int C,
                  const float* mean, const float* invstd, const float* gamma, const float* sums, float dx_beta,
                  const float* bsh, cudaStream_t s, int early) {
  static bool once = [] {
    set_smem(bn_dx_stream_kernel<false, 0>, kS2);
    set_smem(bn_dx_stream_kernel<false, 1>, kS2);
    set_smem(bn_dx_stream_kernel<false, 2>, kS2);
    set_smem(bn_dx_stream_kernel<true, 0>, kS3);
    set_smem(bn_dx_stream_kernel<true, 1>, kS3);
    set_smem(bn_dx_stream_kernel<true, 2>, kS3);
    return true;
  }();
  (void)once;
  BE_REQUIRE(act >= 0 && act <= 2, BE_E_ARG, "bn_dx_stream: activation");
  const int64_t sp = bn_stream_splits(rows, C, 1 << 30);
  const int64_t rps = (rows + sp - 1) / sp;
  auto go = [&](auto kern, int smem) {
    launch_pdl(kern, (unsigned)sp, kThr, smem, s, gy, x, dx, rows, C, mean, invstd, gamma, sums, rps, bsh,
               early && early_on());
  };
  if (dx_beta != 0.f) {
    if (act == 1) go(bn_dx_stream_kernel<true, 1>, kS3);
    else if (act == 2) go(bn_dx_stream_kernel<true, 2>, kS3);
    else go(bn_dx_stream_kernel<true, 0>, kS3);
  } else {
    if (act == 1) go(bn_dx_stream_kernel<false, 1>, kS2);
    else if (act == 2) go(bn_dx_stream_kernel<false, 2>, kS2);
    else go(bn_dx_stream_kernel<false, 0>, kS2);
  }
  after_launch("bn_dx_stream");
}

}}  // namespace be::k
