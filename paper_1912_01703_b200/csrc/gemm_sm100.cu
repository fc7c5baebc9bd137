// gemm_sm100.cu — persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
// Serves every dense contraction on the hot path:
// Linear fwd (Y = X·W, Listing 1), dgrad (dX = dY·Wᵀ) and wgrad
// (dW = Xᵀ·dY) of Linear and of convolutions, with operand majorness
// chosen at run time so none of the three needs a transpose kernel
// (tcgen05 accepts MN-major bf16/tf32 operands).
//
//   warp 0 (one lane) : TMA producer — cp.async.bulk.tensor into a ring of
//                       SW128-swizzled smem stages, mbarrier complete_tx
//   warp 1 (one lane) : MMA issuer — tcgen05.mma (M=128, N=BN, K=16|8) into a
//                       double-buffered TMEM accumulator, tcgen05.commit frees
//                       smem stages / signals the epilogue
//   warp 2            : TMEM allocator
//   warps 4..7        : epilogue — tcgen05.ld 32x32b rows, bias / ReLU /
//                       beta-accumulate / fp32→bf16 (RN-even), vector stores
//
// Precision: kind::f16 with bf16 operands, or "3xTF32" for the fp32 path:
// operands pre-split into tf32 hi = rna(x), lo = rna(x − hi) and
// D = Ahi·Bhi + Ahi·Blo + Alo·Bhi accumulated in fp32 TMEM (SURVEY §8(c)
// reading 12).  Shapes TMA cannot describe (global row stride not a multiple
// of 16 B) run a SIMT tile kernel instead (still on the GPU; counted).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <mutex>
#include <string>
#include <unordered_map>

#include "common.cuh"
#include "kernels.h"
#include "runtime.h"
#include "sgd_math.cuh"
#include "sm100.cuh"

namespace be { namespace k {
using be::dev::launch_pdl;
using be::dev::pdl_entry;

namespace {
std::atomic<uint64_t> g_tc_calls{0}, g_simt_calls{0};

constexpr int BM = 128;
constexpr int kThreads = 384;  // w0 TMA, w1 MMA, w2 TMEM, w3 idle, w4-11 epilogue (2 per TMEM lane quarter)
constexpr int kEpiWarps = 8;

struct __align__(64) GemmParams {
  CUtensorMap ta[2];
  CUtensorMap tb[2];
  int M, N, K;
  int a_kmajor, b_kmajor;
  int tiles_m, tiles_n;
  int splits, kb_per_split;   // split-K: tile index t → (split, tm, tn); split s covers k-blocks [s·kps, (s+1)·kps)
  long long split_stride;     // elements between split partial slabs (fp32 workspace)
  int split_rows;             // rows per slab (M rounded up to the tile height)
  void* D;
  long long ldd;
  int d_f32;
  float beta;
  const float* bias;
  int act;
  // implicit-GEMM convolution (A gathered from NHWC x; unused by plain GEMMs)
  const uint16_t* x;
  int cN, cH, cW, cC, cR, cS, cstride, cpad, cP, cQ;
  int use_im2col;             // conv A operand via TMA im2col map (ta[1]) instead of gather4 (ta[0])
  int b_im2col;               // conv wgrad: MN-major B operand = im2col(x) via TMA im2col map (tb[1])
  // conv wgrad, shifted-tile mode: the GEMM's K axis is blocks of 64 output
  // pixels = sh_hb output rows × sh_wb (≥ Q, power of 2) columns of image n;
  // A = dY through a 4-D [N,P,Q,K] tiled map (ta[0]), B chunk (tap r,s;
  // 64 channels) = x through a 4-D [N,H,W,C] tiled map with element strides
  // = conv stride (tb[1]); out-of-range pixels are zero-filled by TMA
  int b_shift, sh_wb, sh_hb, sh_pg;  // sh_pg = p-groups per image
  // TMA-store epilogue: D (or the split-K workspace) as [rows, N], box 32×32
  int tma_store;
  // epilogue split by tile instead of by column half (BN = 64, no stats): the
  // warp pair of each TMEM lane quarter takes alternate tiles, each pair owns
  // one accumulator buffer — two tiles' epilogues in flight for the narrow
  // outputs (MobileNet's 16–64-channel 1×1 convs) where a tile is one chunk
  int epi_split;
  // operand transform (XF kernels): v ← act(γ_c·(v − μ_c)·is_c + β_c) on the
  // A tile (xf_op 1: K-major, channel = k) or the B tile (xf_op 2: MN-major,
  // channel = n), channel c < xf_C (else 0)
  int xf_op, xf_act, xf_C;
  const float *xf_mean, *xf_invstd, *xf_gamma, *xf_beta;
  CUtensorMap td;
  // fused SGD epilogue (kernels.h SgdFuse): acc = gradient of P[M, N]
  int upd;
  float* upd_p;
  float* upd_v;
  uint16_t* upd_shadow;
  float lr, mu, wd, gscale;
  CUtensorMap tp[2];          // P, V as fp32 [M, N] maps, box 32 × 32 (fused-SGD epilogue loads)
  // per-column Σ / Σx² of the stored output (batch-norm statistics from the
  // epilogue): partial rows [gridDim.x·4][N] (Σ) then [gridDim.x·4][N] (Σx²);
  // row = CTA·4 + TMEM lane quarter; zeroed by the host before the launch
  float* stats;
  // phase-split patch convolution (conv_stem_kernel): L columns per phase,
  // phase block bytes, taps per (phase, row) padded even, patch buffers,
  // weight bytes
  int st_L, st_phb, st_taps, st_nbuf, st_wbytes;
  const uint16_t* st_w;       // KRSC weights (C = 8), copied into smem by every CTA
  // conv_tc_kernel: extra window offset on the w axis (w pad = cpad + cpad_w_off)
  int cpad_w_off;
  // phase store (stride-ph_st dgrad as ph_st² stride-1 phase convolutions):
  // output row m = (n, i, j) of the phase grid [N, cP, cQ] is stored to pixel
  // (n, ph_st·i + ph_h, ph_st·j + ph_w) of the [N, ph_H, ph_W] tensor D (ld = ldd)
  int ph_st, ph_h, ph_w, ph_H, ph_W;
  // data-gradient convolutions (conv_tc / conv_fwd_patch): B read in place from
  // the forward weights W[k, r, s, c] as an MN-major operand (tb[0] = W as
  // [K_fwd rows, R·S·C cols], box {64 c, 64 k}): GEMM tap (t_r, t_s) reads the
  // forward tap (bw_r0 + bw_rstep·t_r, bw_s0 + bw_sstep·t_s); no transposed /
  // flipped weight copy is materialised.  bw_S = forward S, N = forward C.
  int bw_inplace, bw_r0, bw_rstep, bw_s0, bw_sstep, bw_S;
};
constexpr int kEpiBytes = 32768;  // 8 epilogue warps × one 4 KB staging buffer

// Fused-SGD epilogue: 8 warps (two per TMEM lane quarter, alternating
// 16-column chunks of a tile), each with three 5 KB buffers; a buffer holds
// one 32 × 16 chunk of P (2 KB) and V (2 KB) in the TMA SW64 layout, updated
// in place, + its bf16 shadow (1 KB, SW32).  The update is latency-bound per
// warp (dependent smem round trips per chunk), so twice the warps over
// half-width chunks keep twice the chunks in flight in the same 120 KB.
constexpr int kUpdWarps = 8;
constexpr int kUpdBufs = 3;
constexpr int kUpdCW = 16;  // chunk width (columns)
constexpr int kUpdBufBytes = 2048 + 2048 + 1024;
constexpr int kUpdWarpBytes = kUpdBufs * kUpdBufBytes;
// BN ≥ 128 tiles: two buffers per warp (prefetch distance 1) so that one more
// mainloop stage fits (BN 256: 3 × 48 KB, BN 128: 4 × 32 KB) — with two
// stages the operand loads, not the update traffic, bound the kernel (ncu:
// the update warps waited on the accumulator 42 % of their time; 4096² K=1024
// launch 80 → 75 µs, BN 128 90 → 79 µs)
constexpr int upd_bufs(int bn) { return bn >= 128 ? 2 : kUpdBufs; }

// NSLOT: 2-KB bf16 staging slots per epilogue warp (TMA stores in flight per
// warp = NSLOT − 1).  4 for store-heavy short-K shapes (the 1×1 convs: the
// epilogue, not the mainloop, is the critical path), 2 otherwise (more
// mainloop stages for long K).
// XF: the operand-transform variant (a batch norm's normalise + activation
// applied to the A (K-major, channel = k) or B (MN-major, channel = n) tile in
// shared memory between the TMA load and the MMA; see gemm_tc_kernel).
template <int BN, bool X3, bool UPD = false, int NSLOT = 2, bool XF = false>
struct Cfg {
  static constexpr int ESIZE = X3 ? 4 : 2;
  static constexpr int BK = 128 / ESIZE;           // one 128-B swizzle row of K
  static constexpr int UMMA_K = X3 ? 8 : 16;
  static constexpr int NOPS = X3 ? 2 : 1;          // hi (+ lo)
  static constexpr int A_BYTES = BM * 128;         // BM rows x 128 B
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = NOPS * (A_BYTES + B_BYTES);
  static constexpr int EPI_BYTES = UPD ? kUpdWarps * upd_bufs(BN) * kUpdBufBytes : kEpiWarps * NSLOT * 2048;
  static constexpr int XF_BYTES = XF ? 8 * 8 + 2 * 2048 * 4 : 0;  // xfull barriers + per-channel scale/shift (C ≤ 2048)
  static constexpr int STAGES_RAW = (226 * 1024 - EPI_BYTES - XF_BYTES - 1280) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + XF_BYTES + 1024 + 256;
  static constexpr int CH = 128 / ESIZE;           // MN elements per 128-B chunk
};

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // RN-even (cvt.rn.bf16x2.f32)
  return *reinterpret_cast<uint32_t*>(&h);
}

// Epilogue for 32 accumulator columns of one output row held by this thread:
// bias, ReLU, beta-accumulate, fp32 or RN-even bf16 store.  Tails use
// predicated fully-unrolled loops (no local-memory spills).
__device__ __forceinline__ void epi_store32(const GemmParams& p, char* Dbase, bool vec_ok, int row, int col0,
                                            const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  const int ncol = min(32, p.N - col0);
  const bool full = ncol == 32;
  if (p.bias) {
    if (full && (reinterpret_cast<uintptr_t>(p.bias + col0) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j));
        v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < ncol) v[j] += __ldg(p.bias + col0 + j);
    }
  }
  if (p.act == 1) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
  }
  const bool acc = p.beta != 0.f;
  if (p.d_f32) {
    float* dst = reinterpret_cast<float*>(Dbase) + (long long)row * p.ldd + col0;
    if (full && vec_ok) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        if (acc) {
          float4 old = *reinterpret_cast<const float4*>(dst + j);
          o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
        }
        *reinterpret_cast<float4*>(dst + j) = o;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < ncol) dst[j] = v[j] + (acc ? dst[j] : 0.f);
    }
  } else {
    uint16_t* dst = reinterpret_cast<uint16_t*>(Dbase) + (long long)row * p.ldd + col0;
    if (full && vec_ok) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        if (acc) {
          uint4 old = *reinterpret_cast<const uint4*>(dst + j);
          const uint16_t* o16 = reinterpret_cast<const uint16_t*>(&old);
#pragma unroll
          for (int q = 0; q < 8; ++q) v[j + q] += bf16_bits_to_f32(o16[q]);
        }
        uint4 o;
        o.x = pack_bf16x2(v[j], v[j + 1]); o.y = pack_bf16x2(v[j + 2], v[j + 3]);
        o.z = pack_bf16x2(v[j + 4], v[j + 5]); o.w = pack_bf16x2(v[j + 6], v[j + 7]);
        *reinterpret_cast<uint4*>(dst + j) = o;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < ncol) {
          float x = v[j] + (acc ? bf16_bits_to_f32(dst[j]) : 0.f);
          __nv_bfloat16 h = __float2bfloat16_rn(x);
          dst[j] = *reinterpret_cast<uint16_t*>(&h);
        }
      }
    }
  }
}

// ---- column statistics of the stored output (BN statistics in the epilogue)
// lane = row of a 32 × 32 chunk: the value stored for (row, col0 + j) is the
// accumulator rounded to the output type (callers guarantee no bias / act /
// beta); rows ≥ M count 0.  A transpose-reduce (16+8+4+2+1 shuffles) leaves
// lane L with column col0 + L's sum over the 32 rows.
__device__ __forceinline__ float col_reduce32(float (&a)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < off; ++j) {
      const float send = up ? a[j] : a[j + off];
      const float keep = up ? a[j + off] : a[j];
      a[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return a[0];
}
__device__ __forceinline__ void colstats32(const GemmParams& p, const uint32_t (&r)[32], bool row_ok, int lane,
                                           float& s, float& q) {
  float a[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    float v = __uint_as_float(r[j]);
    if (!p.d_f32) v = __bfloat162float(__float2bfloat16_rn(v));
    a[j] = row_ok ? v : 0.f;
  }
  s = col_reduce32(a, lane);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    float v = __uint_as_float(r[j]);
    if (!p.d_f32) v = __bfloat162float(__float2bfloat16_rn(v));
    a[j] = row_ok ? v * v : 0.f;
  }
  q = col_reduce32(a, lane);
}
// per-warp running column sums over a CTA's tiles with the same column block
template <int NCH>
struct ColStats {
  float s[NCH], q[NCH];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int k = 0; k < NCH; ++k) { s[k] = 0.f; q[k] = 0.f; }
  }
  // write this warp's partial row for columns col_base + k·32 + lane, k < nch
  // (the warp's own 32-column chunks only)
  __device__ __forceinline__ void flush(const GemmParams& p, int part, int col_base, int lane, int nch) {
    const long long parts = (long long)gridDim.x * 4;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int col = col_base + k * 32 + lane;
      if (k < nch && col < p.N) {
        p.stats[(long long)part * p.N + col] = s[k];
        p.stats[(parts + part) * p.N + col] = q[k];
      }
    }
    reset();
  }
};

// Fused SGD epilogue for one 32-row × 32-column accumulator chunk held by a
// warp (lane = row): the accumulator is the fp32 gradient g of parameter
// elements P[row, col] (never stored).  All global traffic is TMA: the
// chunk's P and V (32 rows × 16 columns) arrive in smem in the SW64 layout (a
// lane reading its own row is bank-conflict-optimal), are updated in place
// with sgd_elem (the multi-tensor SGD kernel's arithmetic → bitwise the same
// parameters), the bf16 shadow row is written in the SW32 layout, and lane 0
// issues three bulk tensor stores (edges clipped by TMA).
// The caller waited for the loads (mbarrier) before calling.
__device__ __forceinline__ void epi_sgd16(const GemmParams& p, uint8_t* buf, int lane, int row0, int col0,
                                          const uint32_t (&r)[16]) {
  uint8_t* sp = buf;
  uint8_t* sv = buf + 2048;
  uint8_t* ss = buf + 4096;
  const bool mom = p.upd_v != nullptr;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    // SW64: the row's 16-B piece c sits at c ^ ((row >> 1) & 3)
    const int off = lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4);
    const float4 p4 = *reinterpret_cast<const float4*>(sp + off);
    const float4 v4 = mom ? *reinterpret_cast<const float4*>(sv + off) : make_float4(0.f, 0.f, 0.f, 0.f);
    float pv[4] = {p4.x, p4.y, p4.z, p4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) sgd_elem(pv[j], __uint_as_float(r[4 * c + j]), vv[j], mom, p.lr, p.mu, p.wd, p.gscale);
    *reinterpret_cast<float4*>(sp + off) = make_float4(pv[0], pv[1], pv[2], pv[3]);
    if (mom) *reinterpret_cast<float4*>(sv + off) = make_float4(vv[0], vv[1], vv[2], vv[3]);
    if (p.upd_shadow) {
      // 8 bf16 per 16-B SW32 piece (piece h at h ^ ((row >> 2) & 1)): fp32 pieces 2h, 2h+1 → bf16 piece h
      const int h = c >> 1;
      uint2* dst = reinterpret_cast<uint2*>(ss + lane * 32 + ((h ^ ((lane >> 2) & 1)) << 4) + (c & 1) * 8);
      *dst = make_uint2(pack_bf16x2(pv[0], pv[1]), pack_bf16x2(pv[2], pv[3]));
    }
  }
  sm100::fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    sm100::tma_store_2d(&p.tp[0], sp, col0, row0);
    if (mom) sm100::tma_store_2d(&p.tp[1], sv, col0, row0);
    if (p.upd_shadow) sm100::tma_store_2d(&p.td, ss, col0, row0);
    sm100::bulk_commit();
  }
}

// TMA-store epilogue for one 32-row × 32-column chunk held by a warp (lane =
// row): bias / ReLU / convert, write the lane's row into the warp's staging
// buffer in the store map's swizzle (bf16: 64-B rows, SW64 — chunk c at
// c ^ ((row>>1)&3); fp32: 128-B rows, SW128 — c ^ (row&7)), fence, and lane 0
// issues one bulk tensor store (out-of-range rows/columns are clipped by TMA).
// Each warp owns a 4 KB staging area: two 2 KB buffers alternating for bf16
// (the store issued from a buffer two chunks earlier must have read it), one
// 4 KB buffer for fp32.
// Column Σ / Σx² of a bf16 32 × 32 chunk staged in the SW64 layout (the
// stored values; rows ≥ nvalid count 0): lane l reads the 2-column pair
// (l & 15) of rows 2k + (l >> 4) as one 32-bit word (16 conflict-free LDS per
// chunk instead of a 31-step shuffle transpose per sum), the two row parities
// are combined, then lane l takes column l's sums.
__device__ __forceinline__ void colstats_staged(const uint8_t* buf, int lane, int nvalid, float* stq) {
  const int half = lane >> 4, cp = lane & 15;
  float s0 = 0.f, s1 = 0.f, q0 = 0.f, q1 = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int row = 2 * k + half;
    const uint32_t w = *reinterpret_cast<const uint32_t*>(buf + row * 64 + (((cp >> 2) ^ ((row >> 1) & 3)) << 4) +
                                                          (cp & 3) * 4);
    const float lo = row < nvalid ? __uint_as_float(w << 16) : 0.f;
    const float hi = row < nvalid ? __uint_as_float(w & 0xffff0000u) : 0.f;
    s0 += lo; q0 = fmaf(lo, lo, q0);
    s1 += hi; q1 = fmaf(hi, hi, q1);
  }
  s0 += __shfl_xor_sync(0xffffffffu, s0, 16); s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
  q0 += __shfl_xor_sync(0xffffffffu, q0, 16); q1 += __shfl_xor_sync(0xffffffffu, q1, 16);
  const float a0 = __shfl_sync(0xffffffffu, s0, lane >> 1), a1 = __shfl_sync(0xffffffffu, s1, lane >> 1);
  const float b0 = __shfl_sync(0xffffffffu, q0, lane >> 1), b1 = __shfl_sync(0xffffffffu, q1, lane >> 1);
  stq[0] = (lane & 1) ? a1 : a0;
  stq[1] = (lane & 1) ? b1 : b0;
}

template <int NSLOT = 2>
__device__ __forceinline__ void epi_tma32(const GemmParams& p, uint8_t* warp_buf, int& slot, int lane, int store_row,
                                          int col0, const uint32_t (&r)[32], int z = -1, float* stq = nullptr,
                                          int nvalid = 32) {
  static_assert(NSLOT == 2 || NSLOT == 4, "staging slots");
  uint8_t* buf = warp_buf;
  if (p.d_f32) {  // 4-KB fp32 chunks: NSLOT / 2 buffers
    buf += (slot % (NSLOT / 2)) * 4096;
    if (lane == 0) sm100::bulk_wait_read<NSLOT / 2 - 1>();
  } else {
    buf += slot * 2048;
    if (lane == 0) sm100::bulk_wait_read<NSLOT - 1>();
  }
  __syncwarp();
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (p.bias) {
    const int ncol = min(32, p.N - col0);
    if (ncol == 32 && (reinterpret_cast<uintptr_t>(p.bias + col0) & 15) == 0) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + j));
        v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < ncol) v[j] += __ldg(p.bias + col0 + j);
    }
  }
  if (p.act == 1) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
  }
  if (p.d_f32) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<float4*>(buf + lane * 128 + ((c ^ (lane & 7)) << 4)) =
          make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint4 o;
      o.x = pack_bf16x2(v[8 * c], v[8 * c + 1]); o.y = pack_bf16x2(v[8 * c + 2], v[8 * c + 3]);
      o.z = pack_bf16x2(v[8 * c + 4], v[8 * c + 5]); o.w = pack_bf16x2(v[8 * c + 6], v[8 * c + 7]);
      *reinterpret_cast<uint4*>(buf + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) = o;
    }
  }
  sm100::fence_proxy_async();
  __syncwarp();
  if (stq) colstats_staged(buf, lane, nvalid, stq);  // bf16 staging only (callers check d_f32)
  if (lane == 0) {
    if (z >= 0) {  // 3-D map (col, row, z)
      if (p.tma_store == 2) sm100::tma_reduce_add_3d(&p.td, buf, col0, store_row, z);
      else sm100::tma_store_3d(&p.td, buf, col0, store_row, z);
    } else if (p.tma_store == 2) {
      sm100::tma_reduce_add_2d(&p.td, buf, col0, store_row);  // beta = 1
    } else {
      sm100::tma_store_2d(&p.td, buf, col0, store_row);
    }
    sm100::bulk_commit();
  }
  slot = (slot + 1) % (p.d_f32 ? NSLOT / 2 : NSLOT);
}

// Fused-SGD epilogue of a persistent GEMM (warp = TMEM lane quarter eq, column
// parity half): 32 rows × the tile's 16-column chunks j ≡ half (mod 2), as a
// flat sequence over this CTA's tiles (t0, t0 + tstride, …).  Chunk i's P,V
// are TMA-loaded two chunks ahead into buffer i % 3 (no dependence on the
// accumulator), then updated in place and TMA-stored with the shadow
// (epi_sgd16).  CLUSTER: the accumulator-empty arrival goes to the pair
// leader's barrier.
template <int TILE_N, bool CLUSTER, int NBUF = kUpdBufs>
__device__ __forceinline__ void upd_epilogue(const GemmParams& p, uint8_t* epi_smem, uint64_t* ubar, uint64_t* tfull,
                                             uint64_t* tempty, uint32_t tempty_leader, uint32_t tmem_base, int uw,
                                             int lane, int t0, int tstride, int num_tiles, int mn_tiles, int tile_m,
                                             int row_off) {
  static_assert(NBUF == 2 || NBUF == 3, "update buffers");
  const int eq = uw & 3, half = uw >> 2;
  uint8_t* bufs = epi_smem + uw * NBUF * kUpdBufBytes;
  uint64_t* mb = ubar + uw * kUpdBufs;
  const uint32_t tx = p.upd_v ? 4096u : 2048u;
  const int cpt = (min(p.N, TILE_N) + kUpdCW - 1) / kUpdCW;  // chunks per tile (tail chunks past N skipped)
  const int cpw = (cpt - half + 1) / 2;                       // this warp's chunks per tile
  auto chunk_at = [&](int i, int* row0, int* col0, int* j) -> bool {
    const int t = t0 + (i / cpw) * tstride;
    if (t >= num_tiles) return false;
    const int tm = (t % mn_tiles) % p.tiles_m, tn = (t % mn_tiles) / p.tiles_m;
    *j = half + 2 * (i % cpw);
    *row0 = tm * tile_m + row_off + eq * 32;
    *col0 = tn * TILE_N + *j * kUpdCW;
    return true;
  };
  auto issue = [&](int i) {
    int r0, c0, j;
    if (!chunk_at(i, &r0, &c0, &j) || c0 >= p.N) return;
    if (lane == 0) {
      uint8_t* b = bufs + (i % NBUF) * kUpdBufBytes;
      uint64_t* bar = &mb[i % NBUF];
      sm100::mbar_arrive_expect_tx(bar, tx);
      sm100::tma_load_2d(&p.tp[0], bar, b, c0, r0);
      if (p.upd_v) sm100::tma_load_2d(&p.tp[1], bar, b + 2048, c0, r0);
    }
  };
  uint32_t uph = 0u;  // bit k: phase of buffer k
  issue(0);
  if (NBUF == 3) issue(1);
  int acc = 0; uint32_t acc_phase = 0;
  int i = 0;
  for (int t = t0; t < num_tiles; t += tstride) {
    sm100::mbar_wait(&tfull[acc], acc_phase);
    sm100::tc_fence_after();
    for (int q = 0; q < cpw; ++q, ++i) {
      int row0, col0, j;
      chunk_at(i, &row0, &col0, &j);
      const bool live = col0 < p.N;
      if (NBUF == 2) {
        // buffer (i+1) % 2 was last used by chunk i−1 (the latest commit
        // group): wait until its stores have read it, then refill
        if (lane == 0) sm100::bulk_wait_read<0>();
        __syncwarp();
        issue(i + 1);
      }
      if (live) {
        uint32_t ru[16];
        sm100::tmem_ld_32x32b_x16(tmem_base + acc * TILE_N + j * kUpdCW + ((uint32_t)(eq * 32) << 16), ru);
        sm100::tmem_ld_wait();
        const int k = i % NBUF;
        sm100::mbar_wait(&mb[k], (uph >> k) & 1u);
        uph ^= 1u << k;
        epi_sgd16(p, bufs + k * kUpdBufBytes, lane, row0, col0, ru);
      }
      if (NBUF == 3) {
        // buffer (i+2) % 3 was last used by chunk i−1, whose stores went out
        // one commit group ago: wait until they have read it, then refill
        if (lane == 0) {
          if (live) sm100::bulk_wait_read<1>();
          else sm100::bulk_wait_read<0>();
        }
        __syncwarp();
        issue(i + 2);
      }
    }
    sm100::tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (CLUSTER) sm100::mbar_arrive_cluster(tempty_leader + acc * 8);
      else sm100::mbar_arrive(&tempty[acc]);
    }
    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
  }
  if (lane == 0) sm100::bulk_wait<0>();  // stores complete before exit
}

template <int BN, bool X3, bool UPD = false, int NSLOT = 2, bool XF = false>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  using C = Cfg<BN, X3, UPD, NSLOT, XF>;
  static_assert(C::STAGES >= 2, "pipeline needs at least two stages");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + C::EPI_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ubar = tempty + 2;  // UPD: one barrier per P/V buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ubar + (UPD ? kUpdWarps * kUpdBufs : 0));
  uint64_t* xfull = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // XF: operand transformed
  float* xpar = reinterpret_cast<float*>(xfull + 8);              // XF: [channel][scale, shift]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    if (XF)
      for (int s = 0; s < C::STAGES; ++s) sm100::mbar_init(&xfull[s], 2);
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&tfull[a], 1);
      sm100::mbar_init(&tempty[a], UPD ? kUpdWarps : (p.epi_split ? kEpiWarps / 2 : kEpiWarps));
    }
    if (UPD)
      for (int i = 0; i < kUpdWarps * kUpdBufs; ++i) sm100::mbar_init(&ubar[i], 1);
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.ta[0]); sm100::tma_prefetch(&p.tb[0]);
    if (X3) { sm100::tma_prefetch(&p.ta[1]); sm100::tma_prefetch(&p.tb[1]); }
  }
  if (warp == 2) sm100::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int mn_tiles = p.tiles_m * p.tiles_n;
  const int num_tiles = mn_tiles * p.splits;
  const int kblocks_total = (p.K + C::BK - 1) / C::BK;

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA producer =====================
      int stage = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int mn = t % mn_tiles, sp = t / mn_tiles;
        const int tm = mn % p.tiles_m, tn = mn / p.tiles_m;
        const int m0 = tm * BM, n0 = tn * BN;
        const int kb0 = sp * p.kb_per_split, kb1 = min(kblocks_total, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          sm100::mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          uint8_t* sbase = smem + stage * C::STAGE_BYTES;
          const int k0 = kb * C::BK;
#pragma unroll
          for (int op = 0; op < C::NOPS; ++op) {
            uint8_t* sa = sbase + op * (C::A_BYTES + C::B_BYTES);
            uint8_t* sb = sa + C::A_BYTES;
            if (!X3 && p.b_shift) {
              // dY pixel block kb = (image n, p-group) as 64 MN-major rows
              const int ni = kb / p.sh_pg, pg = kb - ni * p.sh_pg;
#pragma unroll
              for (int j = 0; j < BM / C::CH; ++j)
                sm100::tma_load_4d(&p.ta[0], &full[stage], sa + j * C::BK * 128, m0 + j * C::CH, 0, pg * p.sh_hb, ni);
            } else if (p.a_kmajor) {
              sm100::tma_load_2d(&p.ta[op], &full[stage], sa, k0, m0);
            } else {
#pragma unroll
              for (int j = 0; j < BM / C::CH; ++j)
                sm100::tma_load_2d(&p.ta[op], &full[stage], sa + j * C::BK * 128, m0 + j * C::CH, k0);
            }
            if (p.b_kmajor) {
              sm100::tma_load_2d(&p.tb[op], &full[stage], sb, k0, n0);
            } else if (!X3 && p.b_shift) {
              // x for tap (r,s), 64 channels: window start (s−pad, p0·st+r−pad)
              const int ni = kb / p.sh_pg, pg = kb - ni * p.sh_pg;
              const int h0 = pg * p.sh_hb * p.cstride - p.cpad;
#pragma unroll
              for (int j = 0; j < BN / C::CH; ++j) {
                const int col = n0 + j * C::CH;
                const int tap = col / p.cC, cb = (col - tap * p.cC) / 64;
                const int r = tap / p.cS, sx = tap - r * p.cS;
                sm100::tma_load_4d(&p.tb[1], &full[stage], sb + j * C::BK * 128, cb * 64, sx - p.cpad, h0 + r, ni);
              }
            } else if (!X3 && p.b_im2col) {
              // conv wgrad: B = im2col(x) read in place — 64-pixel block k0 ×
              // 64 channels of one filter tap per MN chunk (TMA im2col map tb[1])
              const int q = k0 % p.cQ, pq = k0 / p.cQ;
              const int ws = q * p.cstride - p.cpad, hs = (pq % p.cP) * p.cstride - p.cpad, ni = pq / p.cP;
#pragma unroll
              for (int j = 0; j < BN / C::CH; ++j) {
                const int col = n0 + j * C::CH;
                const int tap = col / p.cC, cb = (col - tap * p.cC) / 64;
                sm100::tma_load_im2col_4d(&p.tb[1], &full[stage], sb + j * C::BK * 128, cb * 64, ws, hs, ni,
                                          (uint16_t)(tap % p.cS), (uint16_t)(tap / p.cS));
              }
            } else {
#pragma unroll
              for (int j = 0; j < BN / C::CH; ++j)
                sm100::tma_load_2d(&p.tb[op], &full[stage], sb + j * C::BK * 128, n0 + j * C::CH, k0);
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===================== MMA issuer =====================
      const uint32_t idesc = sm100::make_idesc(X3 ? 2u : 1u, BM, BN, p.a_kmajor ? 0 : 1, p.b_kmajor ? 0 : 1);
      // descriptor geometry
      const uint32_t a_lbo = p.a_kmajor ? 16u : (uint32_t)(C::BK * 128);
      const uint32_t b_lbo = p.b_kmajor ? 16u : (uint32_t)(C::BK * 128);
      const uint32_t a_kstep = p.a_kmajor ? 32u : (uint32_t)(C::UMMA_K * 128);
      const uint32_t b_kstep = p.b_kmajor ? 32u : (uint32_t)(C::UMMA_K * 128);
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int sp = t / mn_tiles;
        const int kb0 = sp * p.kb_per_split, kb1 = min(kblocks_total, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(XF ? &xfull[stage] : &full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sbase = sm100::smem_u32(smem + stage * C::STAGE_BYTES);
#pragma unroll
          for (int kk = 0; kk < C::BK / C::UMMA_K; ++kk) {
            const uint32_t en = ((kb - kb0) | kk) ? 1u : 0u;
            const uint32_t sa0 = sbase, sb0 = sbase + C::A_BYTES;
            const uint64_t ad = sm100::make_sw128_desc(sa0 + kk * a_kstep, a_lbo, 1024);
            const uint64_t bd = sm100::make_sw128_desc(sb0 + kk * b_kstep, b_lbo, 1024);
            if (X3) {
              const uint32_t sa1 = sbase + C::A_BYTES + C::B_BYTES, sb1 = sa1 + C::A_BYTES;
              const uint64_t ad1 = sm100::make_sw128_desc(sa1 + kk * a_kstep, a_lbo, 1024);
              const uint64_t bd1 = sm100::make_sw128_desc(sb1 + kk * b_kstep, b_lbo, 1024);
              sm100::mma_tf32(d_tmem, ad1, bd, idesc, en);   // lo·hi
              sm100::mma_tf32(d_tmem, ad, bd1, idesc, 1u);   // hi·lo
              sm100::mma_tf32(d_tmem, ad, bd, idesc, 1u);    // hi·hi
            } else {
              sm100::mma_bf16(d_tmem, ad, bd, idesc, en);
            }
          }
          sm100::mma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        sm100::mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (XF && (warp == 2 || warp == 3)) {
    // ===================== operand transform (BN apply) =====================
    // the 64 threads of warps 2–3: (1) once per CTA, scale/shift of every
    // channel into smem; (2) walk the producer's stage sequence: wait for the
    // TMA bytes, rewrite the operand tile in place (bf16 → fp32 affine → act →
    // RN-even bf16; the SW128 chunk at physical slot j of row r holds logical
    // chunk j ^ (r & 7)), four chunks per step with all loads first, make the
    // generic-proxy writes visible to the tensor core (fence.proxy.async) and
    // release the stage to the MMA warp
    const int tid = threadIdx.x - 64;
    for (int c = tid; c < p.xf_C; c += 64) {
      const float sc = p.xf_gamma[c] * p.xf_invstd[c];
      xpar[2 * c] = sc;
      xpar[2 * c + 1] = p.xf_beta[c] - p.xf_mean[c] * sc;
    }
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const int cmax = p.xf_C;
    int stage = 0; uint32_t phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int mn = t % mn_tiles, sp = t / mn_tiles;
      const int tn = mn / p.tiles_m;
      const int kb0 = sp * p.kb_per_split, kb1 = min(kblocks_total, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        sm100::mbar_wait(&full[stage], phase);
        uint8_t* sa = smem + stage * C::STAGE_BYTES;
        uint8_t* tile = p.xf_op == 1 ? sa : sa + C::A_BYTES;
        const int nchunks = p.xf_op == 1 ? BM * 8 : BN * 8;
        const int cbase = p.xf_op == 1 ? kb * C::BK : tn * BN;
        for (int id0 = tid; id0 < nchunks; id0 += 256) {
          uint4 u[4];
          int ch[4];
          uint4* q[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int id = id0 + 64 * v;
            int r, c0;
            if (p.xf_op == 1) {
              r = id >> 3;
              c0 = ((id & 7) ^ (r & 7)) * 8;
            } else {
              const int jb = id >> 9, rr = (id >> 3) & 63;
              r = jb * 64 + rr;
              c0 = jb * 64 + ((id & 7) ^ (rr & 7)) * 8;
            }
            ch[v] = cbase + c0;
            q[v] = reinterpret_cast<uint4*>(tile + (size_t)r * 128 + (id & 7) * 16);
            u[v] = id < nchunks ? *q[v] : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            if (id0 + 64 * v >= nchunks) break;
            uint32_t w[4] = {u[v].x, u[v].y, u[v].z, u[v].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int c = ch[v] + 2 * i;
              const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xffff0000u);
              const float a = c < cmax ? be::dev::act_apply(fmaf(lo, xpar[2 * c], xpar[2 * c + 1]), p.xf_act) : 0.f;
              const float b = c + 1 < cmax ? be::dev::act_apply(fmaf(hi, xpar[2 * c + 2], xpar[2 * c + 3]), p.xf_act)
                                           : 0.f;
              w[i] = pack_bf16x2(a, b);
            }
            *q[v] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        sm100::fence_proxy_async();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&xfull[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (UPD && warp >= 4 && warp < 4 + kUpdWarps) {
    upd_epilogue<BN, false, upd_bufs(BN)>(p, epi_smem, ubar, tfull, tempty, 0u, tmem_base, warp - 4, lane, blockIdx.x, gridDim.x,
                            num_tiles, mn_tiles, BM, 0);
  } else if (!UPD && warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp - 4;               // 0..7
    const int eq = warp & 3, eh = ew >> 2;  // TMEM lane quarter (= warp % 4), column half
    int slot = 0;
    int acc = 0; uint32_t acc_phase = 0;
    ColStats<(BN / 64 > 2 ? BN / 64 : 2)> cst;
    cst.reset();
    const bool vec_ok = (p.ldd % 8 == 0) && ((reinterpret_cast<uintptr_t>(p.D) & 15) == 0);
    if (BN == 64 && p.epi_split) {
      // tile-split epilogue: pair eh takes this CTA's tiles eh, eh + 2, … —
      // exactly the tiles the MMA warp accumulates into buffer eh
      uint32_t ph = 0;
      for (int t = blockIdx.x + eh * (int)gridDim.x; t < num_tiles; t += 2 * (int)gridDim.x, ph ^= 1u) {
        const int mn = t % mn_tiles, sp = t / mn_tiles;
        const int tm = mn % p.tiles_m, tn = mn / p.tiles_m;
        char* Dbase = reinterpret_cast<char*>(p.D) + (long long)sp * p.split_stride * 4;
        sm100::mbar_wait(&tfull[eh], ph);
        sm100::tc_fence_after();
        const int row = tm * BM + eq * 32 + lane;
        const bool row_ok = row < p.M;
        const int store_row = sp * p.split_rows + tm * BM + eq * 32;
        const int col0 = tn * BN, col1 = col0 + 32;
        const bool h1 = col1 < p.N;
        const uint32_t ta = tmem_base + eh * BN + ((uint32_t)(eq * 32) << 16);
        uint32_t r0[32], r1[32];
        sm100::tmem_ld_32x32b_x32(ta, r0);
        if (h1) sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&tempty[eh]);  // accumulator free before the stores
        if (p.tma_store) {
          epi_tma32<NSLOT>(p, epi_smem + ew * (NSLOT * 2048), slot, lane, store_row, col0, r0);
          if (h1) epi_tma32<NSLOT>(p, epi_smem + ew * (NSLOT * 2048), slot, lane, store_row, col1, r1);
        } else if (row_ok) {
          epi_store32(p, Dbase, vec_ok, row, col0, r0);
          if (h1) epi_store32(p, Dbase, vec_ok, row, col1, r1);
        }
      }
    } else
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int mn = t % mn_tiles, sp = t / mn_tiles;
      const int tm = mn % p.tiles_m, tn = mn / p.tiles_m;
      char* Dbase = reinterpret_cast<char*>(p.D) + (long long)sp * p.split_stride * 4;
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      const int row = tm * BM + eq * 32 + lane;
      const bool row_ok = row < p.M;
      const int store_row = sp * p.split_rows + tm * BM + eq * 32;
if (p.stats) {  // statistics epilogue: unrolled so the per-chunk sums stay in registers
      #pragma unroll
      for (int it = 0; it < (BN / 2 + 63) / 64; ++it) {
        const int c0 = eh * (BN / 2) + it * 64;
        // two TMEM loads in flight per wait (warp-uniform predicates)
        const int col0 = tn * BN + c0, col1 = col0 + 32;
        const bool h0 = col0 < p.N, h1 = col1 < p.N && c0 + 32 < (eh + 1) * (BN / 2);
        if (!h0) break;
        const uint32_t ta = tmem_base + acc * BN + c0 + ((uint32_t)(eq * 32) << 16);
        uint32_t r0[32], r1[32];
        sm100::tmem_ld_32x32b_x32(ta, r0);
        if (h1) sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        const bool sfast = p.tma_store && !p.d_f32;  // statistics from the bf16 staging buffer
        if (p.stats && !sfast) {  // batch-norm statistics of the stored values
          float s_, q_;
          colstats32(p, r0, row_ok, lane, s_, q_);
          cst.s[2 * it] += s_; cst.q[2 * it] += q_;
          if (h1) {
            colstats32(p, r1, row_ok, lane, s_, q_);
            cst.s[2 * it + 1] += s_; cst.q[2 * it + 1] += q_;
          }
        }
        if (p.tma_store) {
          float sq[2];
          const int nv = p.M - (row - lane);
          epi_tma32<NSLOT>(p, epi_smem + ew * (NSLOT * 2048), slot, lane, store_row, col0, r0, -1, sfast ? sq : nullptr, nv);
          if (sfast) { cst.s[2 * it] += sq[0]; cst.q[2 * it] += sq[1]; }
          if (h1) {
            epi_tma32<NSLOT>(p, epi_smem + ew * (NSLOT * 2048), slot, lane, store_row, col1, r1, -1, sfast ? sq : nullptr, nv);
            if (sfast) { cst.s[2 * it + 1] += sq[0]; cst.q[2 * it + 1] += sq[1]; }
          }
        } else if (row_ok) {
          epi_store32(p, Dbase, vec_ok, row, col0, r0);
          if (h1) epi_store32(p, Dbase, vec_ok, row, col1, r1);
        }
      }
      } else {
      // column pieces of 64 interleaved between the two warps of a lane
      // quarter (a ragged N such as 144 stays balanced); BN = 64: 32 each
      #pragma unroll 1
      for (int it = 0; it < (BN >= 128 ? BN / 128 : 1); ++it) {
        const int c0 = BN >= 128 ? (2 * it + eh) * 64 : eh * 32;
        // two TMEM loads in flight per wait (warp-uniform predicates)
        const int col0 = tn * BN + c0, col1 = col0 + 32;
        const bool h0 = col0 < p.N, h1 = BN >= 128 && col1 < p.N;
        if (!h0) break;
        const uint32_t ta = tmem_base + acc * BN + c0 + ((uint32_t)(eq * 32) << 16);
        uint32_t r0[32], r1[32];
        sm100::tmem_ld_32x32b_x32(ta, r0);
        if (h1) sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        if (p.tma_store) {
          epi_tma32<NSLOT>(p, epi_smem + ew * (NSLOT * 2048), slot, lane, store_row, col0, r0);
          if (h1) epi_tma32<NSLOT>(p, epi_smem + ew * (NSLOT * 2048), slot, lane, store_row, col1, r1);
        } else if (row_ok) {
          epi_store32(p, Dbase, vec_ok, row, col0, r0);
          if (h1) epi_store32(p, Dbase, vec_ok, row, col1, r1);
        }
      }
      }
      if (p.stats) {
        const int tn_next = t + (int)gridDim.x < num_tiles ? ((t + (int)gridDim.x) % mn_tiles) / p.tiles_m : -1;
        if (tn_next != tn) cst.flush(p, blockIdx.x * 4 + eq, tn * BN + eh * (BN / 2), lane, BN / 64 > 0 ? BN / 64 : 1);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) sm100::bulk_wait<0>();  // TMA stores complete before exit
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------- CTA-pair kernel
// cta_group::2, bf16: a cluster of 2 CTAs computes a 256×256 tile with
// M=256 MMAs issued by the leader; each CTA stages its own 128 rows of A and
// its own 128 rows (N-half) of B, so every byte is fetched from L2 once per
// pair (the 1-CTA 128×256 tile is L2-bandwidth bound, profiles/r01_summary).
namespace pair {
constexpr int TM = 256, TN = 256;         // pair tile
constexpr int HM = 128, HN = 128;         // per-CTA halves
constexpr int BK = 64;                    // bf16: one 128-B swizzle row
constexpr int A_BYTES = HM * 128, B_BYTES = HN * 128;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // 32 KB per CTA
constexpr int STAGES = 6;
constexpr int TMEM_COLS = 512;            // 2 accumulators × 256 columns
constexpr int SMEM = STAGES * STAGE_BYTES + kEpiBytes + 1024 + 256;
// fused-SGD variant: fewer stages, the 4-warp triple-buffered update epilogue
constexpr int STAGES_UPD = 3;
constexpr int SMEM_UPD = STAGES_UPD * STAGE_BYTES + kUpdWarps * kUpdWarpBytes + 1024 + 256;
}  // namespace pair

template <bool UPD = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  using namespace pair;
  constexpr int NST = UPD ? STAGES_UPD : STAGES;
  constexpr int EPI = UPD ? kUpdWarps * kUpdWarpBytes : kEpiBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + NST * STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + EPI);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint64_t* ubar = tempty + 2;  // UPD: one barrier per P/V buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ubar + (UPD ? kUpdWarps * kUpdBufs : 0));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&tfull[a], 1);
      sm100::mbar_init(&tempty[a], 2 * (UPD ? kUpdWarps : kEpiWarps));
    }
    if (UPD)
      for (int i = 0; i < kUpdWarps * kUpdBufs; ++i) sm100::mbar_init(&ubar[i], 1);
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.ta[0]); sm100::tma_prefetch(&p.tb[0]);
  }
  if (warp == 2) sm100::tmem_alloc_2sm<TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int mn_tiles = p.tiles_m * p.tiles_n;
  const int num_tiles = mn_tiles * p.splits;
  const int kblocks_total = (p.K + BK - 1) / BK;

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA producer (both CTAs) =====================
      int stage = 0; uint32_t phase = 0;
      for (int t = pair_id; t < num_tiles; t += npairs) {
        const int mn = t % mn_tiles, sp = t / mn_tiles;
        const int tm = mn % p.tiles_m, tn = mn / p.tiles_m;
        const int m0 = tm * TM + rank * HM, n0 = tn * TN + rank * HN;
        const int kb0 = sp * p.kb_per_split, kb1 = min(kblocks_total, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          if (leader) sm100::mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const int k0 = kb * BK;
          if (p.a_kmajor) {
            sm100::tma_load_2d_2sm(&p.ta[0], &full[stage], sa, k0, m0);
          } else {
#pragma unroll
            for (int j = 0; j < HM / 64; ++j) sm100::tma_load_2d_2sm(&p.ta[0], &full[stage], sa + j * BK * 128, m0 + j * 64, k0);
          }
          if (p.b_kmajor) {
            sm100::tma_load_2d_2sm(&p.tb[0], &full[stage], sb, k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < HN / 64; ++j) sm100::tma_load_2d_2sm(&p.tb[0], &full[stage], sb + j * BK * 128, n0 + j * 64, k0);
          }
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ===================== MMA issuer (leader CTA only) =====================
      const uint32_t idesc = sm100::make_idesc(1u, TM, TN, p.a_kmajor ? 0 : 1, p.b_kmajor ? 0 : 1);
      const uint32_t a_lbo = p.a_kmajor ? 16u : (uint32_t)(BK * 128);
      const uint32_t b_lbo = p.b_kmajor ? 16u : (uint32_t)(BK * 128);
      const uint32_t a_kstep = p.a_kmajor ? 32u : 16u * 128u;
      const uint32_t b_kstep = p.b_kmajor ? 32u : 16u * 128u;
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = pair_id; t < num_tiles; t += npairs) {
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TN;
        const int sp = t / mn_tiles;
        const int kb0 = sp * p.kb_per_split, kb1 = min(kblocks_total, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_u32(smem + stage * STAGE_BYTES), sb = sa + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = sm100::make_sw128_desc(sa + kk * a_kstep, a_lbo, 1024);
            const uint64_t bd = sm100::make_sw128_desc(sb + kk * b_kstep, b_lbo, 1024);
            sm100::mma_bf16_2sm(d_tmem, ad, bd, idesc, ((kb - kb0) | kk) ? 1u : 0u);
          }
          sm100::mma_commit_2sm(&empty[stage], 0x3);
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        sm100::mma_commit_2sm(&tfull[acc], 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (UPD && warp >= 4 && warp < 4 + kUpdWarps) {
    upd_epilogue<TN, true>(p, epi_smem, ubar, tfull, tempty, sm100::mapa(sm100::smem_u32(&tempty[0]), 0), tmem_base,
                           warp - 4, lane, pair_id, npairs, num_tiles, mn_tiles, TM, (int)rank * HM);
  } else if (!UPD && warp >= 4) {
    // ===================== epilogue (both CTAs, own TMEM half) =====================
    const int ew = warp - 4;               // 0..7
    const int eq = warp & 3, eh = ew >> 2;  // TMEM lane quarter (= warp % 4), column half
    int slot = 0;
    int acc = 0; uint32_t acc_phase = 0;
    ColStats<(TN / 64 > 2 ? TN / 64 : 2)> cst;
    cst.reset();
    const bool vec_ok = (p.ldd % 8 == 0) && ((reinterpret_cast<uintptr_t>(p.D) & 15) == 0);
    const uint32_t tempty_leader = sm100::mapa(sm100::smem_u32(&tempty[0]), 0);
    for (int t = pair_id; t < num_tiles; t += npairs) {
      const int mn = t % mn_tiles, sp = t / mn_tiles;
      const int tm = mn % p.tiles_m, tn = mn / p.tiles_m;
      char* Dbase = reinterpret_cast<char*>(p.D) + (long long)sp * p.split_stride * 4;
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      const int row = tm * TM + rank * HM + eq * 32 + lane;
      const bool row_ok = row < p.M;
      const int store_row = sp * p.split_rows + tm * TM + rank * HM + eq * 32;
if (p.stats) {  // statistics epilogue: unrolled so the per-chunk sums stay in registers
      #pragma unroll
      for (int it = 0; it < (TN / 2 + 63) / 64; ++it) {
        const int c0 = eh * (TN / 2) + it * 64;
        // two TMEM loads in flight per wait (warp-uniform predicates)
        const int col0 = tn * TN + c0, col1 = col0 + 32;
        const bool h0 = col0 < p.N, h1 = col1 < p.N && c0 + 32 < (eh + 1) * (TN / 2);
        if (!h0) break;
        const uint32_t ta = tmem_base + acc * TN + c0 + ((uint32_t)(eq * 32) << 16);
        uint32_t r0[32], r1[32];
        sm100::tmem_ld_32x32b_x32(ta, r0);
        if (h1) sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        const bool sfast = p.tma_store && !p.d_f32;  // statistics from the bf16 staging buffer
        if (p.stats && !sfast) {  // batch-norm statistics of the stored values
          float s_, q_;
          colstats32(p, r0, row_ok, lane, s_, q_);
          cst.s[2 * it] += s_; cst.q[2 * it] += q_;
          if (h1) {
            colstats32(p, r1, row_ok, lane, s_, q_);
            cst.s[2 * it + 1] += s_; cst.q[2 * it + 1] += q_;
          }
        }
        if (p.tma_store) {
          float sq[2];
          const int nv = p.M - (row - lane);
          epi_tma32(p, epi_smem + ew * 4096, slot, lane, store_row, col0, r0, -1, sfast ? sq : nullptr, nv);
          if (sfast) { cst.s[2 * it] += sq[0]; cst.q[2 * it] += sq[1]; }
          if (h1) {
            epi_tma32(p, epi_smem + ew * 4096, slot, lane, store_row, col1, r1, -1, sfast ? sq : nullptr, nv);
            if (sfast) { cst.s[2 * it + 1] += sq[0]; cst.q[2 * it + 1] += sq[1]; }
          }
        } else if (row_ok) {
          epi_store32(p, Dbase, vec_ok, row, col0, r0);
          if (h1) epi_store32(p, Dbase, vec_ok, row, col1, r1);
        }
      }
      } else {
      #pragma unroll 1
      for (int it = 0; it < (TN / 2 + 63) / 64; ++it) {
        const int c0 = eh * (TN / 2) + it * 64;
        // two TMEM loads in flight per wait (warp-uniform predicates)
        const int col0 = tn * TN + c0, col1 = col0 + 32;
        const bool h0 = col0 < p.N, h1 = col1 < p.N && c0 + 32 < (eh + 1) * (TN / 2);
        if (!h0) break;
        const uint32_t ta = tmem_base + acc * TN + c0 + ((uint32_t)(eq * 32) << 16);
        uint32_t r0[32], r1[32];
        sm100::tmem_ld_32x32b_x32(ta, r0);
        if (h1) sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        if (p.tma_store) {
          epi_tma32(p, epi_smem + ew * 4096, slot, lane, store_row, col0, r0);
          if (h1) epi_tma32(p, epi_smem + ew * 4096, slot, lane, store_row, col1, r1);
        } else if (row_ok) {
          epi_store32(p, Dbase, vec_ok, row, col0, r0);
          if (h1) epi_store32(p, Dbase, vec_ok, row, col1, r1);
        }
      }
      }
      if (p.stats) {
        const int tn_next = t + npairs < num_tiles ? ((t + npairs) % mn_tiles) / p.tiles_m : -1;
        if (tn_next != tn) cst.flush(p, blockIdx.x * 4 + eq, tn * TN + eh * (TN / 2), lane, TN / 64 > 0 ? TN / 64 : 1);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_cluster(tempty_leader + acc * 8);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) sm100::bulk_wait<0>();  // TMA stores complete before exit
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::cluster_sync();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------- implicit-GEMM convolution
// Y[m = (n,p,q), k] = Σ_{r,s,c} x[n, p·st−pad+r, q·st−pad+s, c] · W[k, r, s, c]
// without materialising im2col: 4 producer warps gather the A tile (one
// output pixel per thread, 8 × 16-B cp.async per 64-channel k-block, zero
// fill in the padding) straight into the SW128 layout UMMA expects (16-B
// chunk j of row r stored at j ^ (r & 7)); B (KRSC weights, K-major) comes
// by TMA; MMA issue / TMEM / epilogue as gemm_tc_kernel.  Requires C % 64 == 0
// so a k-block is 64 channels of one filter tap.
namespace conv {
constexpr int kThreads = 384;   // w0 TMA producer, w1 MMA, w2 TMEM, w4-11 epilogue
template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (226 * 1024 - kEpiBytes - 1280) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + kEpiBytes + 1024 + 256;
};
}  // namespace conv

template <int BN>
__global__ void __launch_bounds__(conv::kThreads, 1) conv_tc_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  using C = conv::Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + kEpiBytes);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    // full: 128 gather threads + 1 TMA expect_tx arrival
    for (int s = 0; s < C::STAGES; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { sm100::mbar_init(&tfull[a], 1); sm100::mbar_init(&tempty[a], kEpiWarps); }
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.ta[0]); sm100::tma_prefetch(&p.tb[0]);
  }
  if (warp == 2) sm100::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_tiles = p.tiles_m * p.tiles_n;
  const int CB = p.cC / 64;                          // k-blocks per tap
  const int kblocks = p.cR * p.cS * CB;

  if (warp == 0 && p.use_im2col) {
    // ===================== producer: A by TMA im2col, B by TMA tile =====================
    // one im2col op per k-block loads the tap (r,s) / 64-channel slice of the
    // tile's 128 output pixels (zero fill in the padding).
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int tm = t % p.tiles_m, tn = t / p.tiles_m;
        const int m0 = tm * BM;
        const int q0 = m0 % p.cQ, pq = m0 / p.cQ;
        const int p0 = pq % p.cP, n0 = pq / p.cP;
        const int ws = q0 * p.cstride - p.cpad - p.cpad_w_off, hs = p0 * p.cstride - p.cpad;
        for (int kb = 0; kb < kblocks; ++kb) {
          const int tap = kb / CB, cb = kb - tap * CB;
          const int r = tap / p.cS, s = tap - r * p.cS;
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          sm100::mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          uint8_t* sbase = smem + stage * C::STAGE_BYTES;
          if (p.bw_inplace) {  // W in place, MN-major: BN/64 boxes {64 c, 64 k} of forward tap (rf, sf)
            const int rf = p.bw_r0 + p.bw_rstep * r, sf = p.bw_s0 + p.bw_sstep * s;
            const int col = (rf * p.bw_S + sf) * p.N + tn * BN;
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              sm100::tma_load_2d(&p.tb[0], &full[stage], sbase + C::A_BYTES + j * 8192, col + j * 64, cb * 64);
          } else {
            sm100::tma_load_2d(&p.tb[0], &full[stage], sbase + C::A_BYTES, kb * 64, tn * BN);
          }
          sm100::tma_load_im2col_4d(&p.ta[1], &full[stage], sbase, cb * 64, ws, hs, n0, (uint16_t)s, (uint16_t)r);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 0) {
    // ===================== producer: A by TMA row-gather, B by TMA tile =====================
    // lane l owns tile rows 4l..4l+3; per k-block (tap r,s; 64 channels) it
    // issues one tile::gather4 of those rows (−1 = padding → zero fill).
    int stage = 0; uint32_t phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int tm = t % p.tiles_m, tn = t / p.tiles_m;
      int nb[4], hb[4], wb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = tm * BM + lane * 4 + i;
        if (m < p.M) {
          const int q = m % p.cQ, pq = m / p.cQ;
          const int pp = pq % p.cP;
          nb[i] = (pq / p.cP) * p.cH;
          hb[i] = pp * p.cstride - p.cpad;
          wb[i] = q * p.cstride - p.cpad - p.cpad_w_off;
        } else {
          nb[i] = 0; hb[i] = -(1 << 20); wb[i] = 0;  // always out of range
        }
      }
      for (int kb = 0; kb < kblocks; ++kb) {
        const int tap = kb / CB, cb = kb - tap * CB;
        const int r = tap / p.cS, s = tap - r * p.cS;
        int rc[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int h = hb[i] + r, w = wb[i] + s;
          rc[i] = (h >= 0 && h < p.cH && w >= 0 && w < p.cW) ? (nb[i] + h) * p.cW + w : -1;
        }
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          sm100::mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          if (p.bw_inplace) {
            const int rf = p.bw_r0 + p.bw_rstep * r, sf = p.bw_s0 + p.bw_sstep * s;
            const int col = (rf * p.bw_S + sf) * p.N + tn * BN;
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              sm100::tma_load_2d(&p.tb[0], &full[stage], smem + stage * C::STAGE_BYTES + C::A_BYTES + j * 8192,
                                 col + j * 64, cb * 64);
          } else {
            sm100::tma_load_2d(&p.tb[0], &full[stage], smem + stage * C::STAGE_BYTES + C::A_BYTES, kb * 64, tn * BN);
          }
        }
        __syncwarp();
        const uint32_t dst = sm100::smem_u32(smem + stage * C::STAGE_BYTES) + lane * 4 * 128;
        sm100::tma_gather4(&p.ta[0], &full[stage], dst, cb * 64, rc[0], rc[1], rc[2], rc[3]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===================== MMA issuer =====================
      const uint32_t idesc = sm100::make_idesc(1u, BM, BN, 0, p.bw_inplace ? 1 : 0);
      // B K-major (LBO 16, +32 B per K = 16) or MN-major in place (64-c chunks
      // 8 KB apart, +16 rows · 128 B per K = 16)
      const uint32_t b_lbo = p.bw_inplace ? 8192u : 16u, b_kstep = p.bw_inplace ? 2048u : 32u;
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_u32(smem + stage * C::STAGE_BYTES), sb = sa + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = sm100::make_sw128_desc(sa + kk * 32, 16, 1024);
            const uint64_t bd = sm100::make_sw128_desc(sb + kk * b_kstep, b_lbo, 1024);
            sm100::mma_bf16(d_tmem, ad, bd, idesc, (kb | kk) ? 1u : 0u);
          }
          sm100::mma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        sm100::mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp - 4;               // 0..7
    const int eq = warp & 3, eh = ew >> 2;  // TMEM lane quarter (= warp % 4), column half
    int slot = 0;
    int acc = 0; uint32_t acc_phase = 0;
    ColStats<(BN / 64 > 2 ? BN / 64 : 2)> cst;
    cst.reset();
    const bool vec_ok = (p.ldd % 8 == 0) && ((reinterpret_cast<uintptr_t>(p.D) & 15) == 0);
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int tm = t % p.tiles_m, tn = t / p.tiles_m;
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      const int row = tm * BM + eq * 32 + lane;
      const bool row_ok = row < p.M;
if (p.stats) {  // statistics epilogue: unrolled so the per-chunk sums stay in registers
      #pragma unroll
      for (int it = 0; it < (BN / 2 + 63) / 64; ++it) {
        const int c0 = eh * (BN / 2) + it * 64;
        // two TMEM loads in flight per wait (warp-uniform predicates)
        const int col0 = tn * BN + c0, col1 = col0 + 32;
        const bool h0 = col0 < p.N, h1 = col1 < p.N && c0 + 32 < (eh + 1) * (BN / 2);
        if (!h0) break;
        uint32_t r0[32], r1[32];
        const uint32_t ta = tmem_base + acc * BN + c0 + ((uint32_t)(eq * 32) << 16);
        sm100::tmem_ld_32x32b_x32(ta, r0);
        if (h1) sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        const bool sfast = p.tma_store && !p.d_f32;  // statistics from the bf16 staging buffer
        if (p.stats && !sfast) {  // batch-norm statistics of the stored values
          float s_, q_;
          colstats32(p, r0, row_ok, lane, s_, q_);
          cst.s[2 * it] += s_; cst.q[2 * it] += q_;
          if (h1) {
            colstats32(p, r1, row_ok, lane, s_, q_);
            cst.s[2 * it + 1] += s_; cst.q[2 * it + 1] += q_;
          }
        }
        if (p.tma_store) {
          float sq[2];
          const int nv = p.M - (row - lane);
          epi_tma32(p, epi_smem + ew * 4096, slot, lane, tm * BM + eq * 32, col0, r0, -1, sfast ? sq : nullptr, nv);
          if (sfast) { cst.s[2 * it] += sq[0]; cst.q[2 * it] += sq[1]; }
          if (h1) {
            epi_tma32(p, epi_smem + ew * 4096, slot, lane, tm * BM + eq * 32, col1, r1, -1, sfast ? sq : nullptr, nv);
            if (sfast) { cst.s[2 * it + 1] += sq[0]; cst.q[2 * it + 1] += sq[1]; }
          }
        } else if (row_ok) {
          epi_store32(p, reinterpret_cast<char*>(p.D), vec_ok, row, col0, r0);
          if (h1) epi_store32(p, reinterpret_cast<char*>(p.D), vec_ok, row, col1, r1);
        }
      }
      } else {
      // phase store: the row's pixel in the full-resolution output
      int orow = row;
      if (p.ph_st && row_ok) {
        const int j = row % p.cQ, ni = row / p.cQ;
        const int i = ni % p.cP, n = ni / p.cP;
        orow = (n * p.ph_H + p.ph_st * i + p.ph_h) * p.ph_W + p.ph_st * j + p.ph_w;
      }
      #pragma unroll 1
      for (int it = 0; it < (BN / 2 + 63) / 64; ++it) {
        const int c0 = eh * (BN / 2) + it * 64;
        // two TMEM loads in flight per wait (warp-uniform predicates)
        const int col0 = tn * BN + c0, col1 = col0 + 32;
        const bool h0 = col0 < p.N, h1 = col1 < p.N && c0 + 32 < (eh + 1) * (BN / 2);
        if (!h0) break;
        uint32_t r0[32], r1[32];
        const uint32_t ta = tmem_base + acc * BN + c0 + ((uint32_t)(eq * 32) << 16);
        sm100::tmem_ld_32x32b_x32(ta, r0);
        if (h1) sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        if (p.tma_store && p.ph_st) {
          // phase store through the 3-D [u][j][c] map: chunk rows m0.. = (u0, j0..)
          const int m0 = tm * BM + eq * 32, u0 = m0 / p.cQ, j0 = m0 - u0 * p.cQ;
          epi_tma32(p, epi_smem + ew * 4096, slot, lane, j0, col0, r0, u0);
          if (h1) epi_tma32(p, epi_smem + ew * 4096, slot, lane, j0, col1, r1, u0);
        } else if (p.tma_store) {
          epi_tma32(p, epi_smem + ew * 4096, slot, lane, tm * BM + eq * 32, col0, r0);
          if (h1) epi_tma32(p, epi_smem + ew * 4096, slot, lane, tm * BM + eq * 32, col1, r1);
        } else if (row_ok) {
          epi_store32(p, reinterpret_cast<char*>(p.D), vec_ok, orow, col0, r0);
          if (h1) epi_store32(p, reinterpret_cast<char*>(p.D), vec_ok, orow, col1, r1);
        }
      }
      }
      if (p.stats) {
        const int tn_next = t + (int)gridDim.x < num_tiles ? (t + (int)gridDim.x) / p.tiles_m : -1;
        if (tn_next != tn) cst.flush(p, blockIdx.x * 4 + eq, tn * BN + eh * (BN / 2), lane, BN / 64 > 0 ? BN / 64 : 1);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) sm100::bulk_wait<0>();  // TMA stores complete before exit
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------- small-C implicit-GEMM convolution
// Y[m, k] = Σ_{r,s,c} x[n, p·st−pad+r, q·st−pad+s, c] · W[k, r, s, c] for C ∈ {8, 16, 32}
// (the channel-padded image of conv1: C = 8).  A 64-wide k-block then spans
// 64/C filter taps, so neither TMA im2col (one tap per op, ~0.13 pixel/cycle)
// nor a materialised im2col (2.5 GB at ResNet conv1) fits.  4 gather warps own
// one output pixel (tile row) each and copy its eight 16-B chunks per k-block
// with cp.async (zero fill for padding and for taps past R·S) into the SW128
// layout (chunk j of row r at j ^ (r & 7)); a per-CTA table maps each 8-channel
// chunk kc of the K = R·S·C axis to (offset (r·W + s)·C + c0, r, s).  B (KRSC
// weights) by TMA; MMA / TMEM / epilogue as conv_tc_kernel.
namespace convs {
constexpr int kThreads = 512;   // w0-3 gather, w4 TMA, w5 MMA, w6 TMEM, w8-15 epilogue
constexpr int LAG = 3;          // cp.async groups in flight per gather thread
constexpr int kMaxChunks = 256; // R·S·C/8 ≤ 256
template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (226 * 1024 - kEpiBytes - 1280 - kMaxChunks * 16) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + kEpiBytes + kMaxChunks * 16 + 1024 + 256;
};
}  // namespace convs

template <int BN>
__global__ void __launch_bounds__(convs::kThreads, 1) conv_small_c_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  using C = convs::Cfg<BN>;
  static_assert(C::STAGES > convs::LAG, "gather pipeline needs more stages than cp.async groups in flight");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + C::STAGES * C::STAGE_BYTES;
  int4* chunk_tab = reinterpret_cast<int4*>(epi_smem + kEpiBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(chunk_tab + convs::kMaxChunks);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int RSC = p.cR * p.cS * p.cC;
  const int kblocks = (RSC + 63) / 64;
  const int lc = __ffs(p.cC) - 1;  // log2 C

  for (int kc = threadIdx.x; kc < kblocks * 8; kc += blockDim.x) {
    const int k0 = kc * 8, tap = k0 >> lc, c0 = k0 & (p.cC - 1);
    const int r = tap / p.cS, s = tap - r * p.cS;
    // taps past R·S: r = huge → always out of range → zero fill
    chunk_tab[kc] = tap < p.cR * p.cS ? make_int4((r * p.cW + s) * p.cC + c0, r, s, 0)
                                      : make_int4(0, 1 << 24, 0, 0);
  }
  if (threadIdx.x == 0) {
    // full: 128 gather threads + 1 TMA expect_tx arrival
    for (int s = 0; s < C::STAGES; ++s) { sm100::mbar_init(&full[s], 129); sm100::mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { sm100::mbar_init(&tfull[a], 1); sm100::mbar_init(&tempty[a], kEpiWarps); }
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.tb[0]);
  }
  if (warp == 6) sm100::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.tiles_m * p.tiles_n;

  if (warp < 4) {
    // ===================== A gather producers (one tile row per thread) =====================
    const int tid = threadIdx.x;
    int stage = 0; uint32_t phase = 0;
    int pend_stage[convs::LAG + 1];
    int npend = 0, head = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int tm = t % p.tiles_m;
      const int m = tm * BM + tid;
      const bool row_ok = m < p.M;
      int hb = -(1 << 25), wb = 0;
      long long base = 0;
      if (row_ok) {
        const int q = m % p.cQ, pq = m / p.cQ;
        const int pp = pq % p.cP, n = pq / p.cP;
        hb = pp * p.cstride - p.cpad;
        wb = q * p.cstride - p.cpad;
        base = (((long long)n * p.cH + hb) * p.cW + wb) * p.cC;
      }
      for (int kb = 0; kb < kblocks; ++kb) {
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t dst = sm100::smem_u32(smem + stage * C::STAGE_BYTES) + tid * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int4 e = chunk_tab[kb * 8 + j];
          const bool ok = (unsigned)(hb + e.y) < (unsigned)p.cH && (unsigned)(wb + e.z) < (unsigned)p.cW;
          const uint16_t* src = ok ? p.x + base + e.x : p.x;
          sm100::cp_async_16(dst + ((j ^ (tid & 7)) << 4), src, ok ? 16u : 0u);
        }
        sm100::cp_async_commit();
        pend_stage[(head + npend) % (convs::LAG + 1)] = stage;
        ++npend;
        if (npend > convs::LAG) {
          // oldest group complete → visible to the async proxy, then signal
          sm100::cp_async_wait<convs::LAG>();
          sm100::fence_proxy_async();
          sm100::mbar_arrive(&full[pend_stage[head]]);
          head = (head + 1) % (convs::LAG + 1);
          --npend;
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
    sm100::cp_async_wait<0>();
    sm100::fence_proxy_async();
    while (npend > 0) {
      sm100::mbar_arrive(&full[pend_stage[head]]);
      head = (head + 1) % (convs::LAG + 1);
      --npend;
    }
  } else if (warp == 4) {
    if (lane == 0) {
      // ===================== B (weights) TMA producer =====================
      int stage = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int tn = t / p.tiles_m;
        for (int kb = 0; kb < kblocks; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          sm100::mbar_arrive_expect_tx(&full[stage], C::B_BYTES);
          sm100::tma_load_2d(&p.tb[0], &full[stage], smem + stage * C::STAGE_BYTES + C::A_BYTES, kb * 64, tn * BN);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      // ===================== MMA issuer =====================
      const uint32_t idesc = sm100::make_idesc(1u, BM, BN, 0, 0);
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_u32(smem + stage * C::STAGE_BYTES), sb = sa + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = sm100::make_sw128_desc(sa + kk * 32, 16, 1024);
            const uint64_t bd = sm100::make_sw128_desc(sb + kk * 32, 16, 1024);
            sm100::mma_bf16(d_tmem, ad, bd, idesc, (kb | kk) ? 1u : 0u);
          }
          sm100::mma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        sm100::mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 8) {
    // ===================== epilogue =====================
    const int ew = warp - 8;               // 0..7
    const int eq = warp & 3, eh = ew >> 2;  // TMEM lane quarter (= warp % 4), column half
    int slot = 0;
    int acc = 0; uint32_t acc_phase = 0;
    ColStats<(BN / 64 > 2 ? BN / 64 : 2)> cst;
    cst.reset();
    const bool vec_ok = (p.ldd % 8 == 0) && ((reinterpret_cast<uintptr_t>(p.D) & 15) == 0);
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int tm = t % p.tiles_m, tn = t / p.tiles_m;
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      const int row = tm * BM + eq * 32 + lane;
      const bool row_ok = row < p.M;
if (p.stats) {  // statistics epilogue: unrolled so the per-chunk sums stay in registers
      #pragma unroll
      for (int it = 0; it < (BN / 2 + 63) / 64; ++it) {
        const int c0 = eh * (BN / 2) + it * 64;
        const int col0 = tn * BN + c0, col1 = col0 + 32;
        const bool h0 = col0 < p.N, h1 = col1 < p.N && c0 + 32 < (eh + 1) * (BN / 2);
        if (!h0) break;
        uint32_t r0[32], r1[32];
        const uint32_t ta = tmem_base + acc * BN + c0 + ((uint32_t)(eq * 32) << 16);
        sm100::tmem_ld_32x32b_x32(ta, r0);
        if (h1) sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        const bool sfast = p.tma_store && !p.d_f32;  // statistics from the bf16 staging buffer
        if (p.stats && !sfast) {  // batch-norm statistics of the stored values
          float s_, q_;
          colstats32(p, r0, row_ok, lane, s_, q_);
          cst.s[2 * it] += s_; cst.q[2 * it] += q_;
          if (h1) {
            colstats32(p, r1, row_ok, lane, s_, q_);
            cst.s[2 * it + 1] += s_; cst.q[2 * it + 1] += q_;
          }
        }
        if (p.tma_store) {
          float sq[2];
          const int nv = p.M - (row - lane);
          epi_tma32(p, epi_smem + ew * 4096, slot, lane, tm * BM + eq * 32, col0, r0, -1, sfast ? sq : nullptr, nv);
          if (sfast) { cst.s[2 * it] += sq[0]; cst.q[2 * it] += sq[1]; }
          if (h1) {
            epi_tma32(p, epi_smem + ew * 4096, slot, lane, tm * BM + eq * 32, col1, r1, -1, sfast ? sq : nullptr, nv);
            if (sfast) { cst.s[2 * it + 1] += sq[0]; cst.q[2 * it + 1] += sq[1]; }
          }
        } else if (row_ok) {
          epi_store32(p, reinterpret_cast<char*>(p.D), vec_ok, row, col0, r0);
          if (h1) epi_store32(p, reinterpret_cast<char*>(p.D), vec_ok, row, col1, r1);
        }
      }
      } else {
      #pragma unroll 1
      for (int it = 0; it < (BN / 2 + 63) / 64; ++it) {
        const int c0 = eh * (BN / 2) + it * 64;
        const int col0 = tn * BN + c0, col1 = col0 + 32;
        const bool h0 = col0 < p.N, h1 = col1 < p.N && c0 + 32 < (eh + 1) * (BN / 2);
        if (!h0) break;
        uint32_t r0[32], r1[32];
        const uint32_t ta = tmem_base + acc * BN + c0 + ((uint32_t)(eq * 32) << 16);
        sm100::tmem_ld_32x32b_x32(ta, r0);
        if (h1) sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        if (p.tma_store) {
          epi_tma32(p, epi_smem + ew * 4096, slot, lane, tm * BM + eq * 32, col0, r0);
          if (h1) epi_tma32(p, epi_smem + ew * 4096, slot, lane, tm * BM + eq * 32, col1, r1);
        } else if (row_ok) {
          epi_store32(p, reinterpret_cast<char*>(p.D), vec_ok, row, col0, r0);
          if (h1) epi_store32(p, reinterpret_cast<char*>(p.D), vec_ok, row, col1, r1);
        }
      }
      }
      if (p.stats) {
        const int tn_next = t + (int)gridDim.x < num_tiles ? (t + (int)gridDim.x) / p.tiles_m : -1;
        if (tn_next != tn) cst.flush(p, blockIdx.x * 4 + eq, tn * BN + eh * (BN / 2), lane, BN / 64 > 0 ? BN / 64 : 1);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) sm100::bulk_wait<0>();  // TMA stores complete before exit
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 6) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------- strided small-C convolution from a phase-split patch
// The stem convolutions (ResNet conv1 7×7/2) have C = 8 (channel-padded
// image) and stride st > 1: a 16-B gather per tap and output pixel uses half
// of every L2 sector and moves the 49 taps' worth of input per pixel through
// L2 (conv_small_c_kernel: L2-bound, 945 µs at b256).
// Here one tile is one output row (n, p) of Q ≤ 128 pixels (MMA rows ≥ Q are
// discarded).  Its input patch — R input rows × the columns the row's
// windows touch — is copied ONCE (coalesced 16-B cp.async along w, 4 copy
// warps), split by column phase φ = (w + pad) mod st: phase φ holds L
// columns j ↔ w = j·st + φ − pad as [r][j][8 channels] (16-B rows, zero-
// filled padding).  For tap (r, s) the A rows of output pixels q = 0,1,… are
// then CONSECUTIVE 16-B rows of phase s mod st starting at column ⌊s/st⌋,
// i.e. exactly a K-major SWIZZLE_NONE UMMA operand (8 contiguous 16-B rows
// per core matrix, SBO = 128 B): the MMA reads A straight from the patch,
// no im2col anywhere.  A K = 16 MMA covers two taps (its two core matrices
// along K are LBO apart): the taps of each (φ, r) are padded to an even count
// T (zero weights) so pair j of row (φ, r) is A = row base + 32·j with
// LBO = 16 and B = its weights + 2·j KB with LBO = 1 KB — descriptors are
// the row bases plus constants.  The weights sit in smem for the whole
// persistent CTA as [φ][r][T][k][8].  An N = 64 MMA runs 32 cycles, shorter
// than one thread's descriptor/issue chain, so two warps issue MMAs for
// alternate tiles into the two TMEM accumulators.  Output rows t·Q + q;
// epilogue as conv_small_c_kernel.
namespace stem {
constexpr int kThreads = 512;   // w0-3 patch copy (cp.async), w4-5 MMA, w6 TMEM, w8-15 epilogue
constexpr int kCopyThreads = 128;
constexpr int LAG = 3;          // cp.async groups (tiles) in flight per copy thread
constexpr int BN = 64;          // output channels (the stems' K)
constexpr int kZeroBytes = 4096;  // past the last patch buffer: discarded rows' overrun lands in zeros
constexpr int kSmemCap = 227 * 1024;
}  // namespace stem

__global__ void __launch_bounds__(stem::kThreads, 1) conv_stem_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nbuf = p.st_nbuf, st = p.cstride, R = p.cR, S = p.cS, L = p.st_L, T = p.st_taps;
  const int patch_bytes = st * p.st_phb;
  uint8_t* wsm = smem;                                   // [φ][r][T][BN][16 B]
  uint8_t* patch = wsm + p.st_wbytes;                    // nbuf × patch_bytes
  uint8_t* zero = patch + nbuf * patch_bytes;
  uint8_t* epi_smem = reinterpret_cast<uint8_t*>(        // 8 warps × 4 KB TMA-store staging (swizzle-aligned)
      (reinterpret_cast<uintptr_t>(zero + stem::kZeroBytes) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + kEpiBytes);
  uint64_t* empty = full + nbuf;
  uint64_t* tfull = empty + nbuf;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // weights (zeros for the padded taps s ≥ S); patch buffers and the zero
  // block zeroed once (phase-block gaps are never written, and padded taps /
  // discarded rows read them: must be finite)
  for (int idx = threadIdx.x; idx < st * R * T * stem::BN; idx += blockDim.x) {
    const int n = idx % stem::BN, sj = (idx / stem::BN) % T, r = (idx / (stem::BN * T)) % R;
    const int ph = idx / (stem::BN * T * R);
    const int s = sj * st + ph;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (s < S) v = __ldg(reinterpret_cast<const uint4*>(p.st_w + ((long long)(n * R + r) * S + s) * 8));
    *reinterpret_cast<uint4*>(wsm + idx * 16) = v;
  }
  for (int i = threadIdx.x; i < (nbuf * patch_bytes + stem::kZeroBytes) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(patch)[i] = make_uint4(0, 0, 0, 0);
  sm100::fence_proxy_async();  // generic-proxy smem writes → visible to the tensor core
  if (threadIdx.x == 0) {
    for (int b = 0; b < nbuf; ++b) {
      sm100::mbar_init(&full[b], stem::kCopyThreads);
      sm100::mbar_init(&empty[b], 1);
    }
    for (int a = 0; a < 2; ++a) { sm100::mbar_init(&tfull[a], 1); sm100::mbar_init(&tempty[a], kEpiWarps); }
    sm100::fence_barrier_init();
  }
  if (warp == 6) sm100::tmem_alloc<2 * stem::BN>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.cN * p.cP;

  if (warp < 4) {
    // ===================== patch copy: 16-B cp.async per (input row r, column w) =====================
    // each thread owns columns u = tid and tid + 128 of the span (≤ 256):
    // their phase offsets / bounds are tile-invariant, so the per-tile loop
    // is one row address + two predicated cp.async per input row
    const int tid = threadIdx.x;
    const int span = L * st;
    const int ua = tid, ub = tid + stem::kCopyThreads;
    const int wa = ua - p.cpad, wb = ub - p.cpad;
    const bool va = ua < span, vb = ub < span;
    const bool oka = va && (unsigned)wa < (unsigned)p.cW, okb = vb && (unsigned)wb < (unsigned)p.cW;
    const uint32_t da = (ua % st) * p.st_phb + (ua / st) * 16, db = (ub % st) * p.st_phb + (ub / st) * 16;
    const long long xa = oka ? (long long)wa * 8 : 0, xb = okb ? (long long)wb * 8 : 0;
    const uint32_t L16 = L * 16;
    int b = 0; uint32_t phase = 0;
    int pend[stem::LAG + 1];
    int npend = 0, head = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int n = t / p.cP, pp = t - n * p.cP;
      sm100::mbar_wait(&empty[b], phase ^ 1);
      uint32_t dst = sm100::smem_u32(patch + b * patch_bytes);
      const int h0 = pp * st - p.cpad;
      const uint16_t* img = p.x + (long long)n * p.cH * p.cW * 8;
      for (int r = 0; r < R; ++r, dst += L16) {
        const int h = h0 + r;
        const bool hok = (unsigned)h < (unsigned)p.cH;
        const uint16_t* srow = img + (long long)(hok ? h : 0) * p.cW * 8;
        if (va) sm100::cp_async_16(dst + da, hok && oka ? srow + xa : p.x, hok && oka ? 16u : 0u);
        if (vb) sm100::cp_async_16(dst + db, hok && okb ? srow + xb : p.x, hok && okb ? 16u : 0u);
      }
      sm100::cp_async_commit();
      pend[(head + npend) % (stem::LAG + 1)] = b;
      ++npend;
      if (npend > stem::LAG) {
        sm100::cp_async_wait<stem::LAG>();
        sm100::fence_proxy_async();
        sm100::mbar_arrive(&full[pend[head]]);
        head = (head + 1) % (stem::LAG + 1);
        --npend;
      }
      if (++b == nbuf) { b = 0; phase ^= 1; }
    }
    sm100::cp_async_wait<0>();
    sm100::fence_proxy_async();
    while (npend > 0) {
      sm100::mbar_arrive(&full[pend[head]]);
      head = (head + 1) % (stem::LAG + 1);
      --npend;
    }
  } else if (warp == 4 || warp == 5) {
    if (lane == 0) {
      // ===================== MMA issuers: warp 4+k takes tiles 2i+k, accumulator k =====================
      const int k = warp - 4;
      const uint32_t idesc = sm100::make_idesc(1u, BM, stem::BN, 0, 0);
      const uint64_t a0 = sm100::make_interleave_desc(sm100::smem_u32(patch), 16, 128);
      const uint64_t b0 = sm100::make_interleave_desc(sm100::smem_u32(wsm), stem::BN * 16, 128);
      const uint32_t rowA = (L * 16) >> 4, phA = p.st_phb >> 4;   // descriptor units (16 B)
      const uint32_t rowB = (T * stem::BN * 16) >> 4;
      uint32_t acc_phase = 0;
      int ti = k;
      for (int t = blockIdx.x + k * gridDim.x; t < num_tiles; t += 2 * gridDim.x, ti += 2) {
        const int b = ti % nbuf;
        sm100::mbar_wait(&tempty[k], acc_phase ^ 1);
        sm100::mbar_wait(&full[b], (uint32_t)(ti / nbuf) & 1u);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + k * stem::BN;
        uint64_t ad = a0 + (uint64_t)((b * patch_bytes) >> 4), bd = b0;
        uint32_t accum = 0;
        for (int ph = 0; ph < st; ++ph) {
          for (int r = 0; r < R; ++r) {
            for (int j = 0; j < T / 2; ++j) {
              sm100::mma_bf16(d_tmem, ad + 2 * j, bd + 128 * j, idesc, accum);
              accum = 1;
            }
            ad += rowA; bd += rowB;
          }
          ad += phA - R * rowA;
        }
        sm100::mma_commit(&empty[b]);
        sm100::mma_commit(&tfull[k]);
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 8) {
    // ===================== epilogue: warp (quarter eq, column half eh) =====================
    const int ew = warp - 8;
    const int eq = warp & 3, eh = ew >> 2;
    int acc = 0; uint32_t acc_phase = 0;
    int slot = 0;
    ColStats<1> cst;
    cst.reset();
    const bool vec_ok = (p.ldd % 8 == 0) && ((reinterpret_cast<uintptr_t>(p.D) & 15) == 0);
    const int qrow = eq * 32 + lane;
    const bool row_ok = qrow < p.cQ;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      uint32_t r0[32];
      sm100::tmem_ld_32x32b_x32(tmem_base + acc * stem::BN + eh * 32 + ((uint32_t)(eq * 32) << 16), r0);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      const bool sfast = p.stats && p.tma_store && !p.d_f32;  // statistics from the bf16 staging buffer
      if (p.stats && !sfast) {
        float s_, q_;
        colstats32(p, r0, row_ok, lane, s_, q_);
        cst.s[0] += s_; cst.q[0] += q_;
      }
      // TMA store of the warp's 32 × 32 box at (k = eh·32, q = eq·32, tile t):
      // full 128-B lines, rows q ≥ Q clipped by the map
      if (p.tma_store) {
        float sq[2];
        epi_tma32(p, epi_smem + ew * 4096, slot, lane, eq * 32, eh * 32, r0, t, sfast ? sq : nullptr, p.cQ - eq * 32);
        if (sfast) { cst.s[0] += sq[0]; cst.q[0] += sq[1]; }
      }
      else if (row_ok) epi_store32(p, reinterpret_cast<char*>(p.D), vec_ok, t * p.cQ + qrow, eh * 32, r0);
    }
    if (p.stats) cst.flush(p, blockIdx.x * 4 + eq, eh * 32, lane, 1);
    if (lane == 0) sm100::bulk_wait<0>();
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 6) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<2 * stem::BN>(tmem_base);
  }
}

// ---------------------------------------------------------------- conv wgrad from a shared input patch
// dW[k, r, s, c] = Σ_{n,p,q} dY[n,p,q,k] · x[n, p+r−pad, q+s−pad, c] for
// stride-1 convolutions with C = 64 and K = 64 (ResNet layer-1 3×3): the
// materialised / im2col-TMA / shifted-tile variants re-read x once per tap
// through L2 (≥ 9× the input), the L2→SM stream bounds them (≈350 µs at
// b256).  Here a tile is G = 128/W' output rows of one image at pitch W'
// (power of two ≥ Q + S − 1): slot m = dp·W' + q.  Per tile TMA loads
//   dY box {64 k, W', G, 1} → B operand (MN-major SW128, rows = slots; slots
//     with q ≥ Q or p ≥ P are zero-filled), and
//   x box {64 c, W', G+R−1, 1} at (−pad, p0−pad) → the patch: input pixel of
//     slot m for tap (r, s) is patch row m + r·W' + s.
// The A operand of tap (r, s) is the patch started at row r·W' + s: an
// MN-major SW128 operand whose start is not a multiple of the 8-row swizzle
// atom (valid: the swizzle is a function of the absolute smem address —
// tools/shift_probe.cu).  One M = 128 MMA covers two taps (A's two 64-channel
// M-atoms are LBO = their row distance apart; an odd last tap repeats itself,
// LBO = 0, and those D rows are dropped), N = 64 = k, K = 16 slots.  D for
// all ⌈RS/2⌉ tap pairs stays in TMEM (≤ 512 columns) for the CTA's whole
// slot range: no per-tile epilogue.  At the end each CTA writes its partial
// dWᵀ rows (D row = tap·64 + c, contiguous in KRSC) into an fp32 split-K slab
// [CTA][64][RSC]; the fixed-order splitk_reduce sums them (deterministic).
namespace wgp {
constexpr int kThreads = 384;   // w0 TMA, w1 + w3 MMA, w2 TMEM, w4-11 epilogue
constexpr int kSlack = 2048;    // zeroed tail after each x plane (discarded slots' overrun)
// geometry shared by host and device: C = 64·CP, K = 64·KP (CP, KP ∈ {1, 2});
// a unit = one M = 128 MMA row block = two taps (C = 64) or one tap (C = 128);
// units are split into ngroups groups of gs (≤ 512 / K accumulators per CTA)
struct Geo {
  int Wp, G, CP, KP, xps, yps, bufb, nbuf, units, ngroups, gs;
};
__host__ __device__ inline Geo geo(int Q, int R, int S, int C, int K) {
  Geo g{};
  g.Wp = 16;
  while (g.Wp < Q + S - 1) g.Wp *= 2;
  g.G = 128 / (g.Wp > 128 ? 128 : g.Wp);
  g.CP = C / 64; g.KP = K / 64;
  g.xps = ((g.G + R - 1) * g.Wp * 128 + kSlack + 1023) / 1024 * 1024;
  g.yps = (g.G * g.Wp * 128 + 1023) / 1024 * 1024;
  g.bufb = g.CP * g.xps + g.KP * g.yps;
  g.nbuf = (225 * 1024) / g.bufb;
  if (g.nbuf > 4) g.nbuf = 4;
  const int taps = R * S;
  g.units = g.CP == 1 ? (taps + 1) / 2 : taps;
  const int maxacc = 512 / K;
  g.ngroups = (g.units + maxacc - 1) / maxacc;
  g.gs = (g.units + g.ngroups - 1) / g.ngroups;
  return g;
}
}  // namespace wgp

__global__ void __launch_bounds__(wgp::kThreads, 1) conv_wgrad_patch_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const wgp::Geo gg = wgp::geo(p.cQ, p.cR, p.cS, p.cC, p.N);
  const int Wp = gg.Wp, G = gg.G, S = p.cS, taps = p.cR * p.cS, N = p.N;
  const int xbytes = (G + p.cR - 1) * Wp * 128, ybytes = G * Wp * 128;
  const int nbuf = gg.nbuf;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nbuf * gg.bufb);
  uint64_t* empty = full + nbuf;
  uint64_t* done = empty + nbuf;   // [2]: one per issuing warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // zero every x plane's slack once (TMA never writes it; discarded slots read it × dY = 0)
  for (int b = 0; b < nbuf; ++b)
    for (int c = 0; c < gg.CP; ++c)
      for (int i = threadIdx.x; i < (gg.xps - xbytes) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem + b * gg.bufb + c * gg.xps + xbytes)[i] = make_uint4(0, 0, 0, 0);
  sm100::fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int b = 0; b < nbuf; ++b) { sm100::mbar_init(&full[b], 1); sm100::mbar_init(&empty[b], 2); }
    sm100::mbar_init(&done[0], 1);
    sm100::mbar_init(&done[1], 1);
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.ta[0]);
    sm100::tma_prefetch(&p.tb[0]);
  }
  if (warp == 2) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int pg = (p.cP + G - 1) / G;       // row groups per image
  const int num_tiles = p.cN * pg;
  const int grp = blockIdx.x % gg.ngroups, split = blockIdx.x / gg.ngroups, splits = gridDim.x / gg.ngroups;
  const int u_lo = grp * gg.gs, u_hi = min(gg.units, u_lo + gg.gs);

  if (warp == 0) {
    if (lane == 0) {
      int b = 0; uint32_t phase = 0;
      for (int t = split; t < num_tiles; t += splits) {
        const int n = t / pg, p0 = (t - n * pg) * G;
        sm100::mbar_wait(&empty[b], phase ^ 1);
        sm100::mbar_arrive_expect_tx(&full[b], (uint32_t)(gg.CP * xbytes + gg.KP * ybytes));
        uint8_t* base = smem + b * gg.bufb;
        for (int c = 0; c < gg.CP; ++c)
          sm100::tma_load_4d(&p.ta[0], &full[b], base + c * gg.xps, c * 64, -p.cpad, p0 - p.cpad, n);
        for (int k = 0; k < gg.KP; ++k)
          sm100::tma_load_4d(&p.tb[0], &full[b], base + gg.CP * gg.xps + k * gg.yps, k * 64, 0, p0, n);
        if (++b == nbuf) { b = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // whole warp runs the issue loop (descriptors stay warp-uniform → uniform
    // registers, short issue chain); one elected lane issues.  Unit A
    // descriptors are built once: per tile / k-step only the start address
    // moves.  Two issuing warps own disjoint units (accumulators): an N = 64
    // MMA (32 cycles) is shorter than one warp's issue chain.
    const uint32_t idesc = sm100::make_idesc(1u, BM, N, 1, 1);
    const int half = (u_hi - u_lo + 1) / 2;
    const int a_lo = warp == 1 ? 0 : half, a_hi = warp == 1 ? half : u_hi - u_lo;
    uint64_t adesc[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int u = min(u_lo + a, gg.units - 1);
      int sh0, lbo;
      if (gg.CP == 1) {
        const int t0 = min(2 * u, taps - 1), t1 = min(2 * u + 1, taps - 1);
        sh0 = (t0 / S) * Wp + t0 % S;
        lbo = ((t1 / S) * Wp + t1 % S - sh0) * 128;       // second tap's 64 channels
      } else {
        sh0 = (u / S) * Wp + u % S;
        lbo = gg.xps;                                      // channels 64..127: the second plane
      }
      adesc[a] = sm100::make_sw128_desc(sm100::smem_u32(smem) + sh0 * 128, lbo, 1024);
    }
    const uint64_t bdesc0 = sm100::make_sw128_desc(sm100::smem_u32(smem + gg.CP * gg.xps), gg.yps, 1024);
    const int ksteps = G * Wp / 16;
    int b = 0; uint32_t phase = 0;
    uint32_t acc = 0;
    for (int t = split; t < num_tiles; t += splits) {
      sm100::mbar_wait(&full[b], phase);
      sm100::tc_fence_after();
      const uint64_t bo = (uint64_t)((b * gg.bufb) >> 4);
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t ko = (uint64_t)(ks * 128);  // 16 slots × 128 B >> 4
        const uint64_t bd = bdesc0 + bo + ko;
#pragma unroll
        for (int a = 0; a < 8; ++a)
          if (a >= a_lo && a < a_hi && sm100::elect_one())
            sm100::mma_bf16(tmem_base + a * N, adesc[a] + bo + ko, bd, idesc, acc);
        acc = 1;
      }
      if (sm100::elect_one()) sm100::mma_commit(&empty[b]);
      __syncwarp();
      if (++b == nbuf) { b = 0; phase ^= 1; }
    }
    if (sm100::elect_one()) sm100::mma_commit(&done[warp == 1 ? 0 : 1]);
    __syncwarp();
  } else if (warp >= 4) {
    // ===================== epilogue: partial dWᵀ rows into this split's slab =====================
    // D row r of unit u ↔ dW column 128·u + r (tap·C + c, contiguous in KRSC)
    const int ew = warp - 4, eq = warp & 3, eh = ew >> 2;
    const int RSC = taps * p.cC;
    float* slab = reinterpret_cast<float*>(p.D) + (long long)split * p.split_stride;
    const bool any = split < num_tiles && split < splits;
    if (any) {
      sm100::mbar_wait(&done[0], 0);
      sm100::mbar_wait(&done[1], 0);
      sm100::tc_fence_after();
    }
    if (split < splits) {
      for (int a = 0; a < u_hi - u_lo; ++a) {
        const int col = 128 * (u_lo + a) + eq * 32 + lane;
        for (int ch = 0; ch < N / 64; ++ch) {
          const int k0 = eh * (N / 2) + ch * 32;
          uint32_t r[32];
          if (any) {
            sm100::tmem_ld_32x32b_x32(tmem_base + a * N + k0 + ((uint32_t)(eq * 32) << 16), r);
            sm100::tmem_ld_wait();
          }
          if (col < RSC) {
#pragma unroll
            for (int j = 0; j < 32; ++j) slab[(long long)(k0 + j) * RSC + col] = any ? __uint_as_float(r[j]) : 0.f;
          }
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem_base);
  }
}

// ---------------------------------------------------------------- stride-1 conv from a shared input patch
// Y[n, p, q, k] = Σ_{r,s,c} x[n, p+r−pad, q+s−pad, c] · W[k, r, s, c] for
// stride-1 convolutions with C = K = 64 (ResNet layer 1: the 3×3 forward and,
// with flipped weights, its dgrad).  The im2col-TMA kernel loads one
// 128 × 64 A tile per tap (9× the input through L2: ≈190 B/clk/SM for an
// N = 64 MMA — L2-bound).  Here a tile is G = 128/W' output rows at pitch W'
// (slot m = dp·W' + q) whose input rows + halo are loaded once (TMA box
// {64 c, W', G+R−1, 1}); tap (r, s)'s A operand is the patch started at row
// r·W' + s — a K-major SW128 operand with an unaligned start (the swizzle
// follows the absolute address: tools/shift_probe.cu) — against the tap's
// 64 × 64 weight tile, resident in smem for the whole CTA.  Two MMA warps
// take alternate tiles (accumulator = tile parity); the epilogue stores each
// warp's 32 slots (one output row segment, W' ≥ 32) through a 3-D
// [N·P][Q][K] TMA map, clipping q ≥ Q; rows past P are skipped.
namespace cfp {
constexpr int kThreads = 384;   // w0 TMA, w1 + w3 MMA, w2 TMEM, w4-11 epilogue
constexpr int NBUF = 3;
constexpr int kSlack = 2048;
}  // namespace cfp

__global__ void __launch_bounds__(cfp::kThreads, 1) conv_fwd_patch_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int Wp = p.sh_wb, G = p.sh_hb, R = p.cR, S = p.cS, taps = R * S;
  const int xbytes = (G + R - 1) * Wp * 128;
  const int xstride = (xbytes + cfp::kSlack + 1023) / 1024 * 1024;
  uint8_t* wsm = smem;                                  // [tap][64 k][128 B] SW128
  uint8_t* xb = wsm + taps * 8192;
  uint8_t* epi_smem = xb + cfp::NBUF * xstride;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + kEpiBytes);
  uint64_t* empty = full + cfp::NBUF;
  uint64_t* tfull = empty + cfp::NBUF;
  uint64_t* tempty = tfull + 2;
  uint64_t* wbar = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wbar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = 0; b < cfp::NBUF; ++b)
    for (int i = threadIdx.x; i < (xstride - xbytes) / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(xb + b * xstride + xbytes)[i] = make_uint4(0, 0, 0, 0);
  sm100::fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int b = 0; b < cfp::NBUF; ++b) { sm100::mbar_init(&full[b], 1); sm100::mbar_init(&empty[b], 1); }
    for (int a = 0; a < 2; ++a) { sm100::mbar_init(&tfull[a], 1); sm100::mbar_init(&tempty[a], kEpiWarps); }
    sm100::mbar_init(wbar, 1);
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.ta[0]);
    sm100::tma_prefetch(&p.tb[0]);
  }
  if (warp == 2) sm100::tmem_alloc<128>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int pg = (p.cP + G - 1) / G;
  const int num_tiles = p.cN * pg;

  if (warp == 0) {
    if (lane == 0) {
      sm100::mbar_arrive_expect_tx(wbar, (uint32_t)(taps * 8192));
      for (int t = 0; t < taps; ++t) {
        if (p.bw_inplace) {  // W in place (MN-major box {64 c, 64 k} of the forward tap)
          const int rf = p.bw_r0 + p.bw_rstep * (t / S), sf = p.bw_s0 + p.bw_sstep * (t % S);
          sm100::tma_load_2d(&p.tb[0], wbar, wsm + t * 8192, (rf * p.bw_S + sf) * 64, 0);
        } else {
          sm100::tma_load_2d(&p.tb[0], wbar, wsm + t * 8192, t * 64, 0);
        }
      }
      int b = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int n = t / pg, p0 = (t - n * pg) * G;
        sm100::mbar_wait(&empty[b], phase ^ 1);
        sm100::mbar_arrive_expect_tx(&full[b], (uint32_t)xbytes);
        sm100::tma_load_4d(&p.ta[0], &full[b], xb + b * xstride, 0, -p.cpad, p0 - p.cpad, n);
        if (++b == cfp::NBUF) { b = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 || warp == 3) {
    const int k = warp == 1 ? 0 : 1;
    const uint32_t idesc = sm100::make_idesc(1u, BM, 64, 0, p.bw_inplace ? 1 : 0);
    const uint64_t a0 = sm100::make_sw128_desc(sm100::smem_u32(xb), 16, 1024);
    const uint64_t w0 = sm100::make_sw128_desc(sm100::smem_u32(wsm), p.bw_inplace ? 8192u : 16u, 1024);
    const uint64_t wk = p.bw_inplace ? 128u : 2u;  // descriptor step per K = 16 (2 KB MN-major / 32 B K-major, >> 4)
    sm100::mbar_wait(wbar, 0);
    int ti = k;
    for (int t = blockIdx.x + k * gridDim.x; t < num_tiles; t += 2 * gridDim.x, ti += 2) {
      const int b = ti % cfp::NBUF;
      sm100::mbar_wait(&tempty[k], (uint32_t)((ti >> 1) & 1) ^ 1u);
      sm100::mbar_wait(&full[b], (uint32_t)((ti / cfp::NBUF) & 1));
      sm100::tc_fence_after();
      const uint64_t ab = a0 + (uint64_t)((b * xstride) >> 4);
      const uint32_t d = tmem_base + k * 64;
      for (int tp = 0; tp < taps; ++tp) {
        const uint64_t ad = ab + (uint64_t)((((tp / S) * Wp + tp % S) * 128) >> 4);
        const uint64_t bd = w0 + (uint64_t)(tp * 512);  // 8 KB >> 4
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (sm100::elect_one()) sm100::mma_bf16(d, ad + 2 * kk, bd + wk * kk, idesc, (tp | kk) ? 1u : 0u);
      }
      if (sm100::elect_one()) {
        sm100::mma_commit(&empty[b]);
        sm100::mma_commit(&tfull[k]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int ew = warp - 4, eq = warp & 3, eh = ew >> 2;
    const int dp = (eq * 32) / Wp, q0 = (eq * 32) % Wp;
    int slot = 0, ti = 0;
    ColStats<1> cst;  // BN statistics of the stored bf16 values (p.stats; host: bf16 output only)
    cst.reset();
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++ti) {
      const int acc = ti & 1;
      const int n = t / pg, p0 = (t - n * pg) * G;
      sm100::mbar_wait(&tfull[acc], (uint32_t)((ti >> 1) & 1));
      sm100::tc_fence_after();
      uint32_t r[32];
      sm100::tmem_ld_32x32b_x32(tmem_base + acc * 64 + eh * 32 + ((uint32_t)(eq * 32) << 16), r);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (p0 + dp < p.cP && q0 < p.cQ) {
        float sq[2];
        epi_tma32(p, epi_smem + ew * 4096, slot, lane, q0, eh * 32, r, n * p.cP + p0 + dp, p.stats ? sq : nullptr,
                  p.cQ - q0);
        if (p.stats) { cst.s[0] += sq[0]; cst.q[0] += sq[1]; }
      }
    }
    if (p.stats) cst.flush(p, blockIdx.x * 4 + eq, eh * 32, lane, 1);
    if (lane == 0) sm100::bulk_wait<0>();
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<128>(tmem_base);
  }
}

// ---------------------------------------------------------------- conv wgrad, im2col gathered into smem
// dW[k, (r,s,c)] = Σ_{n,p,q} dY[n,p,q,k] · x[n, p·st−pad+r, q·st−pad+s, c] (C % 64 == 0, K % 128 == 0)
// as a split-K GEMM over pixel blocks of 64 without a materialised column
// matrix: A = dYᵀ by TMA (MN-major, boxes {64 k, 64 pixels}); B = the
// im2col slice [BN (tap, c) × 64 pixels] gathered by 4 warps with cp.async
// straight into the MN-major SW128 layout UMMA reads (thread = one pixel ×
// BN/2 channels: 16-B piece j of pixel row kk at (j ^ (kk & 7)) · 16; zero fill
// for padding and for pixels past the end).  The materialised variant spent
// ~40 % of its time writing 9× the input to HBM; TMA im2col (~0.13 px/clk)
// and the shifted 4-D tiles were 3–4× slower than the GEMM on the columns.
// Each CTA writes fp32 split slabs; the fixed-order splitk_reduce sums them.
namespace wgg {
constexpr int kThreads = 512;   // w0-3 gather, w4 TMA (A), w5 MMA, w6 TMEM, w8-15 epilogue
// cp.async groups in flight per gather thread before its stage is signalled
// full: the stages still available to the MMA are STAGES − LAG
template <int BN> constexpr int lag() { return BN == 256 ? 1 : 2; }
template <int BN>
struct Cfg {
  static constexpr int LAG = lag<BN>();
  static constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (226 * 1024 - kEpiBytes - 1280) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + kEpiBytes + 1024 + 256;
};
}  // namespace wgg

template <int BN>
__global__ void __launch_bounds__(wgg::kThreads, 1) conv_wgrad_gather_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  using C = wgg::Cfg<BN>;
  static_assert(C::STAGES > C::LAG, "gather pipeline needs more stages than cp.async groups in flight");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + kEpiBytes);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = (p.K + 63) / 64;
  const int mn_tiles = p.tiles_m * p.tiles_n;
  const int num_tiles = mn_tiles * p.splits;
  if (threadIdx.x == 0) {
    // full: 128 gather threads + 1 TMA expect_tx arrival
    for (int st = 0; st < C::STAGES; ++st) { sm100::mbar_init(&full[st], 129); sm100::mbar_init(&empty[st], 1); }
    for (int a = 0; a < 2; ++a) { sm100::mbar_init(&tfull[a], 1); sm100::mbar_init(&tempty[a], kEpiWarps); }
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.ta[0]);
  }
  if (warp == 6) sm100::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 4) {
    // ===================== B gather (pixel kk = tid / 2, channel half = tid % 2) =====================
    const int tid = threadIdx.x, kk = tid >> 1, half = tid & 1;
    constexpr int CPT = BN / 128;  // 64-channel chunks per thread
    int stage = 0; uint32_t phase = 0;
    int pend_stage[C::LAG + 1];
    int npend = 0, head = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int sp = t / mn_tiles, tn = (t % mn_tiles) / p.tiles_m;
      // the thread's chunks: global column n0 + 64·ch → tap, channel offset
      int coff[CPT], tr[CPT], ts[CPT];
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const int col = tn * BN + (half * CPT + i) * 64;
        const int tap = col / p.cC;
        coff[i] = col - tap * p.cC;
        tr[i] = tap / p.cS; ts[i] = tap - tr[i] * p.cS;
      }
      const int kb0 = sp * p.kb_per_split, kb1 = min(kblocks, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        const int m = kb * 64 + kk;  // pixel
        int hb = -(1 << 25), wb = 0;
        long long base = 0;
        if (m < p.K) {
          const int q = m % p.cQ, pq = m / p.cQ;
          const int pp = pq % p.cP, n = pq / p.cP;
          hb = pp * p.cstride - p.cpad;
          wb = q * p.cstride - p.cpad;
          base = ((long long)n * p.cH * p.cW) * p.cC;
        }
        sm100::mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t sbase = sm100::smem_u32(smem + stage * C::STAGE_BYTES) + C::A_BYTES + kk * 128;
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
          const int h = hb + tr[i], w = wb + ts[i];
          const bool ok = (unsigned)h < (unsigned)p.cH && (unsigned)w < (unsigned)p.cW;
          const uint16_t* src = ok ? p.x + base + ((long long)h * p.cW + w) * p.cC + coff[i] : p.x;
          const uint32_t dst = sbase + (half * CPT + i) * 8192;
#pragma unroll
          for (int j = 0; j < 8; ++j) sm100::cp_async_16(dst + ((j ^ (kk & 7)) << 4), src + j * 8, ok ? 16u : 0u);
        }
        sm100::cp_async_commit();
        pend_stage[(head + npend) % (C::LAG + 1)] = stage;
        ++npend;
        if (npend > C::LAG) {
          sm100::cp_async_wait<C::LAG>();
          sm100::fence_proxy_async();
          sm100::mbar_arrive(&full[pend_stage[head]]);
          head = (head + 1) % (C::LAG + 1);
          --npend;
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
    sm100::cp_async_wait<0>();
    sm100::fence_proxy_async();
    while (npend > 0) {
      sm100::mbar_arrive(&full[pend_stage[head]]);
      head = (head + 1) % (C::LAG + 1);
      --npend;
    }
  } else if (warp == 4) {
    if (lane == 0) {
      // ===================== A (dYᵀ, MN-major) TMA producer =====================
      int stage = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int sp = t / mn_tiles, tm = (t % mn_tiles) % p.tiles_m;
        const int kb0 = sp * p.kb_per_split, kb1 = min(kblocks, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          sm100::mbar_arrive_expect_tx(&full[stage], C::A_BYTES);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          sm100::tma_load_2d(&p.ta[0], &full[stage], sa, tm * BM, kb * 64);
          sm100::tma_load_2d(&p.ta[0], &full[stage], sa + 8192, tm * BM + 64, kb * 64);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      // ===================== MMA issuer (A and B MN-major) =====================
      const uint32_t idesc = sm100::make_idesc(1u, BM, BN, 1, 1);
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int sp = t / mn_tiles;
        const int kb0 = sp * p.kb_per_split, kb1 = min(kblocks, kb0 + p.kb_per_split);
        sm100::mbar_wait(&tempty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_u32(smem + stage * C::STAGE_BYTES), sb = sa + C::A_BYTES;
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const uint64_t ad = sm100::make_sw128_desc(sa + k4 * 2048, 8192, 1024);
            const uint64_t bd = sm100::make_sw128_desc(sb + k4 * 2048, 8192, 1024);
            sm100::mma_bf16(d_tmem, ad, bd, idesc, ((kb - kb0) | k4) ? 1u : 0u);
          }
          sm100::mma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        sm100::mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 8) {
    // ===================== epilogue: fp32 split slab by TMA store =====================
    const int ew = warp - 8;
    const int eq = warp & 3, eh = ew >> 2;
    int slot = 0;
    int acc = 0; uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int sp = t / mn_tiles, tm = (t % mn_tiles) % p.tiles_m, tn = (t % mn_tiles) / p.tiles_m;
      sm100::mbar_wait(&tfull[acc], acc_phase);
      sm100::tc_fence_after();
      const int store_row = sp * p.split_rows + tm * BM + eq * 32;
#pragma unroll 1
      for (int it = 0; it < BN / 128; ++it) {
        const int c0 = eh * (BN / 2) + it * 64;
        const int col0 = tn * BN + c0;
        uint32_t r0[32], r1[32];
        const uint32_t ta = tmem_base + acc * BN + c0 + ((uint32_t)(eq * 32) << 16);
        sm100::tmem_ld_32x32b_x32(ta, r0);
        sm100::tmem_ld_32x32b_x32(ta + 32, r1);
        sm100::tmem_ld_wait();
        epi_tma32(p, epi_smem + ew * 4096, slot, lane, store_row, col0, r0);
        epi_tma32(p, epi_smem + ew * 4096, slot, lane, store_row, col0 + 32, r1);
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) sm100::bulk_wait<0>();
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 6) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------- stem conv wgrad: im2col built in smem from the patch
// dW[k, r, s, c] = Σ_{n,p,q} dY[n,p,q,k] · x[n, p·st−pad+r, q·st−pad+s, c] for
// the C = 8 stem (ResNet conv1 7×7/2): the materialised im2col is 2.5 GB at
// b256 (≈0.9 ms to write + 0.45 ms for the GEMM to read).  Here a tile is one
// output row: its input patch is copied once into the stem kernel's
// phase-split layout (cp.async, 4 warps); 4 build warps then assemble, 16
// output pixels at a time, the im2col slice [16 pixels × R·S·8] in smem as an
// MN-major SW128 operand (M = (tap, c) — 8 taps of 8 channels per 128-B atom,
// K = pixels; 16-B smem→smem copies) — the columns never leave the SM.
// D[(tap, c), k] = Σ slice · dY slice (dY row by TMA, MN-major SW128, q ≥ Q
// zero-filled) accumulates in TMEM (⌈R·S·8/128⌉ M-tiles × 64 columns) over
// the CTA's rows; one fp32 split-K slab per CTA, fixed-order splitk_reduce.
namespace wgs {
constexpr int kThreads = 512;   // w0-3 patch copy, w4-7 slice build, w8 MMA, w9 dY TMA, w10 TMEM, w12-15 epilogue
constexpr int kCopy = 128;
constexpr int NY = 2;           // dY row buffers (16 KB each)
constexpr int kZeroBytes = 4096;
struct Geo { int L, phb, patch_bytes, Mt, slb, ns, np, smem; };
inline Geo geo(const ConvGeom& g) {
  Geo e{};
  e.L = g.Q + (g.S - 1) / g.stride;
  e.phb = (g.R * e.L * 16 + 127) / 128 * 128 + (128 / g.stride) / 16 * 16;
  e.patch_bytes = g.stride * e.phb;
  e.Mt = (g.R * g.S * 8 + 127) / 128;
  e.slb = e.Mt * 4096;
  const int fixed = 1024 + NY * 16384 + kZeroBytes + 512;
  // deep slice ring (the build → MMA → release loop is latency-bound), two patch buffers
  e.np = 2;
  e.ns = (227 * 1024 - fixed - e.np * e.patch_bytes) / e.slb;
  if (e.ns > 8) e.ns = 8;
  e.smem = fixed + e.ns * e.slb + e.np * e.patch_bytes;
  return e;
}
}  // namespace wgs

__global__ void __launch_bounds__(wgs::kThreads, 1) conv_wgrad_stem_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int st = p.cstride, R = p.cR, S = p.cS, L = p.st_L, taps = R * S;
  const int NS = p.st_nbuf & 0xff, NP = p.st_nbuf >> 8, Mt = p.st_taps, slb = Mt * 4096;
  const int patch_bytes = st * p.st_phb;
  uint8_t* slices = smem;                              // NS × Mt × [2 atoms × 16 rows × 128 B]
  uint8_t* ybuf = slices + NS * slb;                   // NY × 128 rows × 128 B
  uint8_t* patch = ybuf + wgs::NY * 16384;             // NP × patch_bytes
  uint8_t* zero = patch + NP * patch_bytes;
  int* tab = reinterpret_cast<int*>(zero + wgs::kZeroBytes);   // per tap: patch offset at q = 0
  uint64_t* full_p = reinterpret_cast<uint64_t*>(tab + 128);
  uint64_t* empty_p = full_p + 4;
  uint64_t* full_y = empty_p + 4;
  uint64_t* empty_y = full_y + wgs::NY;
  uint64_t* full_s = empty_y + wgs::NY;
  uint64_t* empty_s = full_s + 8;
  uint64_t* done = empty_s + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < (NS * slb) / 16; i += blockDim.x) reinterpret_cast<uint4*>(slices)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < (NP * patch_bytes + wgs::kZeroBytes) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(patch)[i] = make_uint4(0, 0, 0, 0);
  for (int t = threadIdx.x; t < taps; t += blockDim.x) {
    const int r = t / S, s_ = t % S;
    tab[t] = (s_ % st) * p.st_phb + (r * L + s_ / st) * 16;
  }
  sm100::fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int b = 0; b < NP; ++b) { sm100::mbar_init(&full_p[b], wgs::kCopy); sm100::mbar_init(&empty_p[b], 4); }
    for (int b = 0; b < wgs::NY; ++b) { sm100::mbar_init(&full_y[b], 1); sm100::mbar_init(&empty_y[b], 1); }
    for (int b = 0; b < NS; ++b) { sm100::mbar_init(&full_s[b], 4); sm100::mbar_init(&empty_s[b], 1); }
    sm100::mbar_init(done, 1);
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.tb[0]);
  }
  if (warp == 10) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.cN * p.cP;
  const int nks = (p.cQ + 15) / 16;

  if (warp < 4) {
    // ===================== patch copy (as conv_stem_kernel), one group in flight =====================
    const int tid = threadIdx.x, span = L * st;
    const int ua = tid, ub = tid + wgs::kCopy;
    const int wa = ua - p.cpad, wb = ub - p.cpad;
    const bool va = ua < span, vb = ub < span;
    const bool oka = va && (unsigned)wa < (unsigned)p.cW, okb = vb && (unsigned)wb < (unsigned)p.cW;
    const uint32_t da = (ua % st) * p.st_phb + (ua / st) * 16, db = (ub % st) * p.st_phb + (ub / st) * 16;
    const long long xa = oka ? (long long)wa * 8 : 0, xb = okb ? (long long)wb * 8 : 0;
    const uint32_t L16 = L * 16;
    int b = 0; uint32_t phase = 0;
    int prev = -1;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int n = t / p.cP, pp = t - n * p.cP;
      sm100::mbar_wait_sleep(&empty_p[b], phase ^ 1, 200);
      uint32_t dst = sm100::smem_u32(patch + b * patch_bytes);
      const int h0 = pp * st - p.cpad;
      const uint16_t* img = p.x + (long long)n * p.cH * p.cW * 8;
      for (int r = 0; r < R; ++r, dst += L16) {
        const int h = h0 + r;
        const bool hok = (unsigned)h < (unsigned)p.cH;
        const uint16_t* srow = img + (long long)(hok ? h : 0) * p.cW * 8;
        if (va) sm100::cp_async_16(dst + da, hok && oka ? srow + xa : p.x, hok && oka ? 16u : 0u);
        if (vb) sm100::cp_async_16(dst + db, hok && okb ? srow + xb : p.x, hok && okb ? 16u : 0u);
      }
      sm100::cp_async_commit();
      if (prev >= 0) {
        sm100::cp_async_wait<1>();
        sm100::fence_proxy_async();
        sm100::mbar_arrive(&full_p[prev]);
      }
      prev = b;
      if (++b == NP) { b = 0; phase ^= 1; }
    }
    sm100::cp_async_wait<0>();
    sm100::fence_proxy_async();
    if (prev >= 0) sm100::mbar_arrive(&full_p[prev]);
  } else if (warp < 8) {
    // ===================== im2col slice build: 16 pixels × taps × 16 B =====================
    // thread tid owns items idx = tid + 128·j (pixel i = idx & 15, tap = idx >> 4),
    // the same for every slice: its patch / slice offsets are computed once and
    // each slice is up to 16 independent ld.shared.v4 → st.shared.v4 pairs
    const int tid = threadIdx.x - 128;
    const int nitems = 16 * taps;
    uint32_t so[16], dof[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int idx = tid + 128 * j;
      const int i = idx & 15, tap = idx >> 4;
      so[j] = idx < nitems ? (uint32_t)(tab[tap] + i * 16) : 0u;
      dof[j] = idx < nitems ? (uint32_t)((tap >> 3) * 2048 + i * 128 + (((tap & 7) ^ (i & 7)) << 4)) : 0u;
    }
    const uint32_t patch_s = sm100::smem_u32(patch), slices_s = sm100::smem_u32(slices);
    int ti = 0, si = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++ti) {
      const int bp = ti % NP;
      sm100::mbar_wait(&full_p[bp], (uint32_t)((ti / NP) & 1));
      const uint32_t pb = patch_s + bp * patch_bytes;
      for (int ks = 0; ks < nks; ++ks, ++si) {
        const int sb = si % NS;
        sm100::mbar_wait(&empty_s[sb], (uint32_t)((si / NS) & 1) ^ 1u);
        const uint32_t src = pb + ks * 256, dst = slices_s + sb * slb;  // 16 pixels × 16 B per slice step
        uint4 v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (tid + 128 * j < nitems)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w) : "r"(src + so[j]));
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (tid + 128 * j < nitems)
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};"
                         :: "r"(dst + dof[j]), "r"(v[j].x), "r"(v[j].y), "r"(v[j].z), "r"(v[j].w) : "memory");
        sm100::fence_proxy_async();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&full_s[sb]);
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&empty_p[bp]);
    }
  } else if (warp == 8) {
    // ===================== MMA: per slice, Mt × (M = 128, N = 64, K = 16) =====================
    const uint32_t idesc = sm100::make_idesc(1u, BM, 64, 1, 1);
    const uint64_t a0 = sm100::make_sw128_desc(sm100::smem_u32(slices), 2048, 1024);
    const uint64_t b0 = sm100::make_sw128_desc(sm100::smem_u32(ybuf), 16, 1024);
    int ti = 0, si = 0;
    uint32_t acc = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++ti) {
      const int by = ti % wgs::NY;
      sm100::mbar_wait(&full_y[by], (uint32_t)((ti / wgs::NY) & 1));
      for (int ks = 0; ks < nks; ++ks, ++si) {
        const int sb = si % NS;
        sm100::mbar_wait(&full_s[sb], (uint32_t)((si / NS) & 1));
        sm100::tc_fence_after();
        const uint64_t bd = b0 + (uint64_t)((by * 16384 + ks * 2048) >> 4);
        const uint64_t ab = a0 + (uint64_t)((sb * slb) >> 4);
        for (int mt = 0; mt < Mt; ++mt)
          if (sm100::elect_one()) sm100::mma_bf16(tmem_base + mt * 64, ab + (uint64_t)(mt * 256), bd, idesc, acc);
        acc = 1;
        if (sm100::elect_one()) sm100::mma_commit(&empty_s[sb]);
        __syncwarp();
      }
      if (sm100::elect_one()) sm100::mma_commit(&empty_y[by]);
      __syncwarp();
    }
    if (sm100::elect_one()) sm100::mma_commit(done);
    __syncwarp();
  } else if (warp == 9) {
    if (lane == 0) {
      int ti = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++ti) {
        const int by = ti % wgs::NY, n = t / p.cP, pp = t - n * p.cP;
        sm100::mbar_wait(&empty_y[by], (uint32_t)((ti / wgs::NY) & 1) ^ 1u);
        sm100::mbar_arrive_expect_tx(&full_y[by], 16384u);
        sm100::tma_load_4d(&p.tb[0], &full_y[by], ybuf + by * 16384, 0, 0, pp, n);
      }
    }
  } else if (warp >= 12) {
    // ===================== epilogue: D row m = tap·8 + c → slab[k][m] =====================
    const int eq = warp & 3;
    const int RSC = taps * 8;
    float* slab = reinterpret_cast<float*>(p.D) + (long long)blockIdx.x * p.split_stride;
    sm100::mbar_wait_sleep(done, 0, 2000);
    sm100::tc_fence_after();
    for (int mt = 0; mt < Mt; ++mt) {
      const int m = mt * 128 + eq * 32 + lane;
      for (int h = 0; h < 2; ++h) {
        uint32_t r[32];
        sm100::tmem_ld_32x32b_x32(tmem_base + mt * 64 + h * 32 + ((uint32_t)(eq * 32) << 16), r);
        sm100::tmem_ld_wait();
        if (m < RSC) {
#pragma unroll
          for (int j = 0; j < 32; ++j) slab[(long long)(h * 32 + j) * RSC + m] = __uint_as_float(r[j]);
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 10) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem_base);
  }
}

// ---------------------------------------------------------------- stem conv wgrad, Hankel operand (no im2col)
// The same product as conv_wgrad_stem_kernel, with dY as the A operand
// (M = 64 output channels, MN-major SW128 straight from the TMA'd dY row) and
// the phase-split input patch itself as B: for filter row r and column phase
// φ, the taps s = φ + st·s' (s' = 0 … n_φ−1) of output pixel q read patch
// pixel q + s' of phase φ, i.e. B[n = (s', c), k = q] sits at
// φ·phb + (r·L + q + s')·16 + 2c — an MN-major SWIZZLE_NONE operand whose
// 8-channel core matrices step 16 B along N (SBO) and 128 B per 8 pixels
// along K (LBO): overlapping core matrices (a Hankel matrix), read in place.
// One tcgen05.mma (M = 64, N = 8·n_φ, K = 16 pixels) per (r, φ, 16 pixels);
// the R·S·8 accumulator columns stay in TMEM over all of the CTA's rows.
// Nothing is copied inside shared memory: the build warps of
// conv_wgrad_stem_kernel (its bottleneck) are gone.
namespace wgh {
constexpr int kThreads = 384;   // w0-3 patch copy, w4 MMA, w5 dY TMA, w6 TMEM, w8-11 epilogue
constexpr int kCopy = 128;
constexpr int NY = 4;           // dY row buffers (16 KB each)
constexpr int NP = 4;           // patch buffers
constexpr int kSlack = 2048;    // zeroed bytes after the last patch (ragged-Q reads past it)
inline int smem_bytes(const ConvGeom& g, int phb) { return 1024 + NY * 16384 + NP * g.stride * phb + kSlack + 1024; }
}  // namespace wgh

// KR, KS, KST: compile-time filter rows / columns / stride (the ResNet stem's
// 7, 7, 2) — the MMA issue loop then unrolls to one UTCHMMA per few
// instructions; 0, 0, 0: run-time geometry (an issue loop of ~20 uniform-
// datapath instructions per MMA, which bounds the kernel)
template <int KR, int KS, int KST>
__global__ void __launch_bounds__(wgh::kThreads, 1) conv_wgrad_hankel_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int st = KST ? KST : p.cstride, R = KR ? KR : p.cR, S = KS ? KS : p.cS, L = p.st_L;
  const int patch_bytes = st * p.st_phb;
  uint8_t* ybuf = smem;                                   // NY × 128 rows × 128 B
  uint8_t* patch = ybuf + wgh::NY * 16384;                // NP × patch_bytes
  uint64_t* full_p = reinterpret_cast<uint64_t*>(patch + wgh::NP * patch_bytes + wgh::kSlack);
  uint64_t* empty_p = full_p + wgh::NP;
  uint64_t* full_y = empty_p + wgh::NP;
  uint64_t* empty_y = full_y + wgh::NY;
  uint64_t* done = empty_y + wgh::NY;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);   // + 4 words, then the MMA tables (512 B)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // pixels past Q of the last 16-pixel step read patch bytes past the copied
  // row: zero them once (their dY rows are TMA zero-filled, 0 · finite = 0)
  for (int i = threadIdx.x; i < (wgh::NP * patch_bytes + wgh::kSlack) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(patch)[i] = make_uint4(0, 0, 0, 0);
  sm100::fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int b = 0; b < wgh::NP; ++b) { sm100::mbar_init(&full_p[b], wgh::kCopy); sm100::mbar_init(&empty_p[b], 1); }
    for (int b = 0; b < wgh::NY; ++b) { sm100::mbar_init(&full_y[b], 1); sm100::mbar_init(&empty_y[b], 1); }
    sm100::mbar_init(done, 1);
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.tb[0]);
  }
  if (warp == 6) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.cN * p.cP;
  const int nks = (p.cQ + 15) / 16;

  if (warp < 4) {
    // ===================== patch copy (phase-split rows, cp.async), one group in flight =====================
    const int tid = threadIdx.x, span = L * st;
    const int ua = tid, ub = tid + wgh::kCopy;
    const int wa = ua - p.cpad, wb = ub - p.cpad;
    const bool va = ua < span, vb = ub < span;
    const bool oka = va && (unsigned)wa < (unsigned)p.cW, okb = vb && (unsigned)wb < (unsigned)p.cW;
    const uint32_t da = (ua % st) * p.st_phb + (ua / st) * 16, db = (ub % st) * p.st_phb + (ub / st) * 16;
    const long long xa = oka ? (long long)wa * 8 : 0, xb = okb ? (long long)wb * 8 : 0;
    const uint32_t L16 = L * 16;
    int b = 0; uint32_t phase = 0;
    int prev = -1;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int n = t / p.cP, pp = t - n * p.cP;
      sm100::mbar_wait_sleep(&empty_p[b], phase ^ 1, 200);
      uint32_t dst = sm100::smem_u32(patch + b * patch_bytes);
      const int h0 = pp * st - p.cpad;
      const uint16_t* img = p.x + (long long)n * p.cH * p.cW * 8;
      for (int r = 0; r < R; ++r, dst += L16) {
        const int h = h0 + r;
        const bool hok = (unsigned)h < (unsigned)p.cH;
        const uint16_t* srow = img + (long long)(hok ? h : 0) * p.cW * 8;
        if (va && !(p.st_wbytes & 2)) sm100::cp_async_16(dst + da, hok && oka ? srow + xa : p.x, hok && oka ? 16u : 0u);
        if (vb && !(p.st_wbytes & 2)) sm100::cp_async_16(dst + db, hok && okb ? srow + xb : p.x, hok && okb ? 16u : 0u);
      }
      sm100::cp_async_commit();
      if (prev >= 0) {
        sm100::cp_async_wait<1>();
        sm100::fence_proxy_async();
        sm100::mbar_arrive(&full_p[prev]);
      }
      prev = b;
      if (++b == wgh::NP) { b = 0; phase ^= 1; }
    }
    sm100::cp_async_wait<0>();
    sm100::fence_proxy_async();
    if (prev >= 0) sm100::mbar_arrive(&full_p[prev]);
  } else if (warp == 4) {
    // ===================== MMA: per 16 pixels, one (M 64, N 8·n_φ, K 16) per (r, φ) =====================
    // descriptors by addition only, the warp converged (warp-uniform values
    // stay in uniform registers; one elected lane issues): per phase φ its
    // instruction descriptor, column count and byte offset; the B start steps
    // by one patch row (L pixels) per filter row r.  (A lane-0-only loop
    // that looked per-(r, φ) descriptors up in a table issued one MMA per
    // ~130 cycles.)
    {
      uint32_t idp[4], ncol[4];
      uint64_t dph[4];
#pragma unroll
      for (int ph = 0; ph < 4; ++ph) {
        const int nph = ph < st ? (S - ph + st - 1) / st : 0;
        ncol[ph] = nph > 0 ? 8u * nph : 0u;
        idp[ph] = sm100::make_idesc(1u, 64, nph > 0 ? 8 * nph : 8, 1, 1);
        dph[ph] = (uint64_t)((ph * p.st_phb) >> 4);
      }
      const uint64_t a0 = sm100::make_sw128_desc(sm100::smem_u32(ybuf), 16, 1024);
      const uint64_t b0 = sm100::make_interleave_desc(sm100::smem_u32(patch), 128, 16);
      int ti = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++ti) {
        const int by = ti % wgh::NY, bp = ti % wgh::NP;
        sm100::mbar_wait(&full_y[by], (uint32_t)((ti / wgh::NY) & 1));
        sm100::mbar_wait(&full_p[bp], (uint32_t)((ti / wgh::NP) & 1));
        sm100::tc_fence_after();
        for (int ks = 0; ks < nks; ++ks) {
          const uint64_t ad = a0 + (uint64_t)((by * 16384 + ks * 2048) >> 4);
          uint64_t brow = b0 + (uint64_t)((bp * patch_bytes) >> 4) + (uint64_t)(ks * 16);  // 16 pixels × 16 B
          const uint32_t accf = (ti | ks) ? 1u : 0u;
          const bool leader = sm100::elect_one();
          if constexpr (KR != 0) {
            if (leader) {
#pragma unroll
              for (int r = 0; r < KR; ++r)
#pragma unroll
                for (int ph = 0; ph < KST; ++ph) {
                  constexpr int dummy = 0;
                  (void)dummy;
                  // column of (r, φ): r·KS·8 + 8·(taps of phases < φ)
                  const uint32_t col = tmem_base + (uint32_t)(r * KS * 8 + 8 * (ph * (KS / KST) + (ph < KS % KST ? ph : KS % KST)));
                  sm100::mma_bf16(col, ad, brow + (uint64_t)(r * L) + dph[ph], idp[ph], accf);
                }
            }
          } else {
            uint32_t col = tmem_base;
            for (int r = 0; r < R; ++r, brow += (uint64_t)L) {
#pragma unroll
              for (int ph = 0; ph < 4; ++ph)
                if (ncol[ph]) {
                  if (leader && !(p.st_wbytes & 1)) sm100::mma_bf16(col, ad, brow + dph[ph], idp[ph], accf);
                  col += ncol[ph];
                }
            }
          }
          __syncwarp();
        }
        if (sm100::elect_one()) { sm100::mma_commit(&empty_p[bp]); sm100::mma_commit(&empty_y[by]); }
        __syncwarp();
      }
      if (sm100::elect_one()) sm100::mma_commit(done);
    }
    __syncwarp();
  } else if (warp == 5) {
    if (lane == 0) {
      int ti = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++ti) {
        const int by = ti % wgh::NY, n = t / p.cP, pp = t - n * p.cP;
        sm100::mbar_wait(&empty_y[by], (uint32_t)((ti / wgh::NY) & 1) ^ 1u);
        sm100::mbar_arrive_expect_tx(&full_y[by], 16384u);
        sm100::tma_load_4d(&p.tb[0], &full_y[by], ybuf + by * 16384, 0, 0, pp, n);
      }
    }
  } else if (warp >= 8) {
    // ===================== epilogue: D[k][(r, φ, s', c)] → slab[k][(r·S + φ + st·s')·8 + c] =====================
    // M = 64 accumulator: row i in TMEM lane (i / 16)·32 + i % 16 (lanes 0-15 of each quarter)
    const int eq = warp & 3;
    const int RSC = R * S * 8;
    const int k = eq * 16 + lane;
    float* slab = reinterpret_cast<float*>(p.D) + (long long)blockIdx.x * p.split_stride;
    sm100::mbar_wait_sleep(done, 0, 2000);
    sm100::tc_fence_after();
    uint32_t col = 0;
    for (int r = 0; r < R; ++r)
      for (int ph = 0; ph < st; ++ph) {
        const int nph = (S - ph + st - 1) / st;
        for (int sp = 0; sp < nph; ++sp, col += 8) {
          uint32_t v[8];
          sm100::tmem_ld_32x32b_x8(tmem_base + col + ((uint32_t)(eq * 32) << 16), v);
          sm100::tmem_ld_wait();
          if (lane < 16 && num_tiles > (int)blockIdx.x) {
            const int m0 = (r * S + ph + st * sp) * 8;
#pragma unroll
            for (int c = 0; c < 8; ++c) slab[(long long)k * RSC + m0 + c] = __uint_as_float(v[c]);
          }
        }
      }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 6) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem_base);
  }
}

// ---------------------------------------------------------------- stem wgrad, two output rows per MMA
// ResNet stem (7×7, stride 2, C = 8): output rows p and p+1 read input rows
// 2p−3 … 2p+5 — nine patch rows j, row p with filter row r = j, row p+1 with
// r = j − 2.  Stacking the two dY rows as the M = 128 A operand (M-atoms
// 16 KB apart) makes one tcgen05.mma per (patch row j, phase φ, 16 pixels)
// serve both rows: 126 MMAs per row pair instead of 196, at M = 128.  Both
// operands arrive by TMA, one stage per row pair: the dY rows (SW128) and
// the patch, each column phase φ one strided 4-D box (W traversal stride 2,
// start w = φ − pad, zero fill outside the image) landing in exactly the
// phase-split layout the Hankel descriptors read.  TMEM region j
// (56 columns): lanes 0-63 accumulate filter row j (row p), lanes 64-127
// filter row j − 2 (row p+1); the epilogue adds the two halves in a fixed
// order.  9 × 56 = 504 of the 512 columns.
namespace wgh2 {
constexpr int kThreads = 384;    // w0 TMA, w4 MMA, w6 TMEM, w8-11 epilogue
constexpr int NS = 3;            // stages (dY row pair + patch)
constexpr int RJ = 9;            // patch rows
constexpr int kSlack = 2048;
inline int phb(int L) { return (RJ * L * 16 + 64 + 511) / 512 * 512; }  // stages stay 1024-B aligned (SW128 dY)
inline int stage_bytes(int L) { return 32768 + 2 * phb(L); }
inline int smem_bytes(int L) { return 1024 + NS * stage_bytes(L) + kSlack + 1024; }
}  // namespace wgh2

__global__ void __launch_bounds__(wgh2::kThreads, 1) conv_wgrad_hankel2_kernel(const __grid_constant__ GemmParams p) {
  pdl_entry();
  constexpr int R = 7, S = 7, RJ = wgh2::RJ;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int L = p.st_L, phb = p.st_phb;
  const int sbytes = 32768 + 2 * phb;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + wgh2::NS * sbytes + wgh2::kSlack);
  uint64_t* empty = full + wgh2::NS;
  uint64_t* done = empty + wgh2::NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // the patch slack past each phase block (and past the last stage) is read
  // for pixels ≥ Q, whose dY rows are zero: zero it once (TMA never writes it)
  for (int i = threadIdx.x; i < (wgh2::NS * sbytes + wgh2::kSlack) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  sm100::fence_proxy_async();
  if (threadIdx.x == 0) {
    for (int b = 0; b < wgh2::NS; ++b) { sm100::mbar_init(&full[b], 1); sm100::mbar_init(&empty[b], 1); }
    sm100::mbar_init(done, 1);
    sm100::fence_barrier_init();
    sm100::tma_prefetch(&p.tb[0]);
    sm100::tma_prefetch(&p.ta[0]);
  }
  if (warp == 6) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int PP = (p.cP + 1) >> 1;
  const int num_tiles = p.cN * PP;
  const int nks = (p.cQ + 15) / 16;

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA: dY rows p, p+1 and the two patch phases =====================
      const uint32_t tx = 32768u + 2u * (uint32_t)(RJ * L * 16);
      int ti = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++ti) {
        const int b = ti % wgh2::NS, n = t / PP, p0 = (t - n * PP) * 2;
        sm100::mbar_wait(&empty[b], (uint32_t)((ti / wgh2::NS) & 1) ^ 1u);
        uint8_t* st = smem + b * sbytes;
        sm100::mbar_arrive_expect_tx(&full[b], tx);
        sm100::tma_load_4d(&p.tb[0], &full[b], st, 0, 0, p0, n);
        const int h0 = p0 * 2 - p.cpad;
        sm100::tma_load_4d(&p.ta[0], &full[b], st + 32768, 0, -p.cpad, h0, n);
        sm100::tma_load_4d(&p.ta[0], &full[b], st + 32768 + phb, 0, 1 - p.cpad, h0, n);
      }
    }
  } else if (warp == 4) {
    // ===================== MMA: (M 128 = two dY rows, N 32 | 24, K 16) per (j, φ, 16 pixels) =====================
    const uint32_t id0 = sm100::make_idesc(1u, 128, 32, 1, 1), id1 = sm100::make_idesc(1u, 128, 24, 1, 1);
    const uint64_t a0 = sm100::make_sw128_desc(sm100::smem_u32(smem), 16384, 1024);
    const uint64_t b0 = sm100::make_interleave_desc(sm100::smem_u32(smem + 32768), 128, 16);
    const uint64_t dph1 = (uint64_t)(phb >> 4);
    int ti = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++ti) {
      const int b = ti % wgh2::NS;
      sm100::mbar_wait(&full[b], (uint32_t)((ti / wgh2::NS) & 1));
      sm100::tc_fence_after();
      const uint64_t so = (uint64_t)((b * sbytes) >> 4);
      for (int ks = 0; ks < nks; ++ks) {
        const uint64_t ad = a0 + so + (uint64_t)(ks * 128);   // 16 pixels × 128 B
        const uint64_t brow = b0 + so + (uint64_t)(ks * 16);  // 16 pixels × 16 B
        const uint32_t accf = (ti | ks) ? 1u : 0u;
        if (sm100::elect_one()) {
#pragma unroll
          for (int j = 0; j < RJ; ++j) {
            sm100::mma_bf16(tmem_base + j * 56, ad, brow + (uint64_t)(j * L), id0, accf);
            sm100::mma_bf16(tmem_base + j * 56 + 32, ad, brow + (uint64_t)(j * L) + dph1, id1, accf);
          }
        }
        __syncwarp();
      }
      if (sm100::elect_one()) sm100::mma_commit(&empty[b]);
      __syncwarp();
    }
    if (sm100::elect_one()) sm100::mma_commit(done);
    __syncwarp();
  } else if (warp >= 8) {
    // ===================== epilogue: slab[k][(r·7 + s)·8 + c] = top[j = r] + bottom[j = r + 2] =====================
    const int eq = warp & 3, half = eq >> 1;
    const int k = (eq & 1) * 32 + lane;
    constexpr int RSC = R * S * 8;
    float* slab = reinterpret_cast<float*>(p.D) + (long long)blockIdx.x * p.split_stride;
    sm100::mbar_wait_sleep(done, 0, 2000);
    sm100::tc_fence_after();
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == half) {
        const int j0 = half ? 2 : 0;
        for (int j = j0; j < j0 + R; ++j) {
          const int r = j - j0;
          for (int g8 = 0; g8 < 7; ++g8) {   // column groups of region j: φ 0 (s' 0..3), φ 1 (s' 0..2)
            uint32_t v[8];
            sm100::tmem_ld_32x32b_x8(tmem_base + j * 56 + g8 * 8 + ((uint32_t)(eq * 32) << 16), v);
            sm100::tmem_ld_wait();
            const int sidx = g8 < 4 ? 2 * g8 : 2 * (g8 - 4) + 1;   // tap column s
            float* dst = slab + (long long)k * RSC + (r * S + sidx) * 8;
#pragma unroll
            for (int c = 0; c < 8; ++c) dst[c] = half ? dst[c] + __uint_as_float(v[c]) : __uint_as_float(v[c]);
          }
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 6) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem_base);
  }
}

// ---------------------------------------------------------------- SIMT path
// 64x64 tiles, 256 threads, 4x4 outputs per thread, fp32 accumulate.
template <typename TA>
__device__ __forceinline__ float ldv(const TA* p, long long i) {
  if constexpr (sizeof(TA) == 2) return bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(p)[i]);
  else return reinterpret_cast<const float*>(p)[i];
}
template <typename TA>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int M, int N, int K, const TA* A, long long lda, int akm,
                                                       const TA* B, long long ldb, int bkm, void* D, long long ldd,
                                                       int d_f32, float beta, const float* bias, int act,
                                                       int kchunk, float* ws) {
  // split-K over blockIdx.z when ws != null: partial sums to ws[z][M][N]
  // (reduced in fixed order by splitk_reduce, which then applies bias/act/beta)
  __shared__ float As[16][64 + 1];
  __shared__ float Bs[16][64 + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int kbeg = blockIdx.z * kchunk, kend = min(K, kbeg + kchunk);
  if (ws) {
    D = ws + (long long)blockIdx.z * M * N; ldd = N; d_f32 = 1; beta = 0.f; bias = nullptr; act = 0;
  }
  float acc[4][4] = {};
  for (int k0 = kbeg; k0 < kend; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      int kk = i / 64, mm = i % 64;
      int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < kend) ? ldv(A, akm ? (long long)m * lda + k : (long long)k * lda + m) : 0.f;
      int n = n0 + mm;
      Bs[kk][mm] = (n < N && k < kend) ? ldv(B, bkm ? (long long)n * ldb + k : (long long)k * ldb + n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j] + (bias ? bias[n] : 0.f);
      if (act == 1) v = fmaxf(v, 0.f);
      if (d_f32) {
        float* d = reinterpret_cast<float*>(D) + (long long)m * ldd + n;
        *d = v + (beta != 0.f ? *d : 0.f);
      } else {
        uint16_t* d = reinterpret_cast<uint16_t*>(D) + (long long)m * ldd + n;
        float x = v + (beta != 0.f ? bf16_bits_to_f32(*d) : 0.f);
        __nv_bfloat16 h = __float2bfloat16_rn(x);
        *d = *reinterpret_cast<uint16_t*>(&h);
      }
    }
  }
}

// Copy a [rows, cols] matrix (row stride lds) into a buffer with row stride
// ldd ≥ cols, zero-filling columns [cols, ldd): operands whose rows are not
// 16-byte multiples (e.g. an N = 10 head) become TMA-describable.
template <typename T>
__global__ void pad_rows_kernel(const T* __restrict__ src, long long lds, T* __restrict__ dst, long long ldd,
                                long long rows, long long cols) {
  pdl_entry();
  const long long total = rows * ldd;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ldd, c = i % ldd;
    dst[i] = c < cols ? src[r * lds + c] : T(0);
  }
}
__global__ void splitk_reduce(const float* __restrict__ ws, int splits, long long sstride, int M, int N, void* D, long long ldd,
                              int d_f32, float beta, const float* bias, int act) {
  pdl_entry();
  const long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int s = 0; s < splits; ++s) v += ws[(long long)s * sstride + i];
    const int m = (int)(i / N), n = (int)(i % N);
    if (bias) v += bias[n];
    if (act == 1) v = fmaxf(v, 0.f);
    if (d_f32) {
      float* d = reinterpret_cast<float*>(D) + (long long)m * ldd + n;
      *d = v + (beta != 0.f ? *d : 0.f);
    } else {
      uint16_t* d = reinterpret_cast<uint16_t*>(D) + (long long)m * ldd + n;
      float x = v + (beta != 0.f ? bf16_bits_to_f32(*d) : 0.f);
      __nv_bfloat16 h = __float2bfloat16_rn(x);
      *d = *reinterpret_cast<uint16_t*>(&h);
    }
  }
}

inline int splitk_blocks(long long total) {
  return (int)std::min<long long>((total + 255) / 256, (long long)ctx().num_sms * 16);
}
// fixed-order split-K reduction (a float4 variant with all splits' loads in
// flight measured slower: 10.6 vs 9.0 µs per C4 launch — fewer threads, and
// these launches are latency-bound)
void launch_splitk(const float* ws, int splits, long long sstride, int M, int N, void* D, long long ldd, int d_f32,
                   float beta, const float* bias, int act, cudaStream_t s) {
  const long long total = (long long)M * N;
  launch_pdl(splitk_reduce, splitk_blocks(total), 256, 0, s, ws, splits, sstride, M, N, D, ldd, d_f32, beta, bias,
             act);
}

// ---------------------------------------------------------------- skinny shapes (N = 1 / K = 1)
// Heads such as NCF's [B, 128]·[128, 1] have row strides TMA cannot describe
// (2 B) and almost no work; the 64×64 SIMT tiles wasted ≥ 98 % of their lanes
// (23 µs per call).  N = 1: a dot product per output row — K-major A: one
// warp per row, lanes stride over k, fixed-order shuffle reduce; MN-major A:
// lanes over 32 consecutive rows (coalesced), 8 warps over k, split over k
// across blocks with a fixed-order split-K reduce.  K = 1: an outer product.
template <typename TA>
__global__ void __launch_bounds__(256) gemv_kmajor_kernel(int M, int K, const TA* A, long long lda, const TA* B,
                                                          long long bstride, void* D, long long ldd, int d_f32,
                                                          float beta, const float* bias, int act) {
  pdl_entry();
  const int m = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (m >= M) return;
  float acc = 0.f;
  for (int k = lane; k < K; k += 32) acc = fmaf(ldv(A, (long long)m * lda + k), ldv(B, (long long)k * bstride), acc);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    float v = acc + (bias ? bias[0] : 0.f);
    if (act == 1) v = fmaxf(v, 0.f);
    if (d_f32) {
      float* d = reinterpret_cast<float*>(D) + (long long)m * ldd;
      *d = v + (beta != 0.f ? *d : 0.f);
    } else {
      uint16_t* d = reinterpret_cast<uint16_t*>(D) + (long long)m * ldd;
      const float x = v + (beta != 0.f ? bf16_bits_to_f32(*d) : 0.f);
      __nv_bfloat16 h = __float2bfloat16_rn(x);
      *d = *reinterpret_cast<uint16_t*>(&h);
    }
  }
}
// MN-major A (A(m, k) = A[k·lda + m]): partial sums over k-range split blockIdx.y → ws[split][m]
template <typename TA>
__global__ void __launch_bounds__(256) gemv_mnmajor_kernel(int M, int K, const TA* A, long long lda, const TA* B,
                                                           long long bstride, int kchunk, float* ws) {
  pdl_entry();
  __shared__ float sm[8][33];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = blockIdx.x * 32 + lane;
  const int kbeg = blockIdx.y * kchunk, kend = min(K, kbeg + kchunk);
  float acc = 0.f;
  if (m < M)
    for (int k = kbeg + w; k < kend; k += 8) acc = fmaf(ldv(A, (long long)k * lda + m), ldv(B, (long long)k * bstride), acc);
  sm[w][lane] = acc;
  __syncthreads();
  if (w == 0 && m < M) {
    float v = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) v += sm[j][lane];
    ws[(long long)blockIdx.y * M + m] = v;
  }
}
// K = 1: D[m, n] = A(m, 0)·B(0, n) (+ bias, act, beta)
template <typename TA>
__global__ void __launch_bounds__(256) outer_kernel(int M, int N, const TA* A, long long astride, const TA* B,
                                                    long long bstride, void* D, long long ldd, int d_f32, float beta,
                                                    const float* bias, int act) {
  pdl_entry();
  const long long total = (long long)M * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(i / N), n = (int)(i - (long long)m * N);
    float v = ldv(A, (long long)m * astride) * ldv(B, (long long)n * bstride) + (bias ? bias[n] : 0.f);
    if (act == 1) v = fmaxf(v, 0.f);
    if (d_f32) {
      float* d = reinterpret_cast<float*>(D) + (long long)m * ldd + n;
      *d = v + (beta != 0.f ? *d : 0.f);
    } else {
      uint16_t* d = reinterpret_cast<uint16_t*>(D) + (long long)m * ldd + n;
      const float x = v + (beta != 0.f ? bf16_bits_to_f32(*d) : 0.f);
      __nv_bfloat16 h = __float2bfloat16_rn(x);
      *d = *reinterpret_cast<uint16_t*>(&h);
    }
  }
}

// tf32 split into K-major hi/lo operands: out[mn, k] (ld2) from x (K-major
// x[mn*ldx + k] or MN-major x[k*ldx + mn]); 32x32 smem tiles keep both the
// read and the write coalesced.
__device__ __forceinline__ void tf32_split(float v, float& h, float& l) {
  uint32_t hb, lb;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
  const float r = v - __uint_as_float(hb);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(r));
  h = __uint_as_float(hb);
  l = __uint_as_float(lb);
}
__global__ void split_kmajor_kernel(const float* __restrict__ x, long long ldx, int src_kmajor, int MN, int K,
                                    float* __restrict__ hi, float* __restrict__ lo, long long ld2) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.x * 32, mn0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int j = ty; j < 32; j += 8) {
    if (src_kmajor) {
      const int mn = mn0 + j, k = k0 + tx;
      tile[j][tx] = (mn < MN && k < K) ? x[(long long)mn * ldx + k] : 0.f;
    } else {
      const int k = k0 + j, mn = mn0 + tx;
      tile[tx][j] = (mn < MN && k < K) ? x[(long long)k * ldx + mn] : 0.f;
    }
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    const int mn = mn0 + j, k = k0 + tx;
    if (mn < MN && k < ld2) {
      float h, l;
      tf32_split(tile[j][tx], h, l);
      hi[(long long)mn * ld2 + k] = h;
      lo[(long long)mn * ld2 + k] = l;
    }
  }
}
void split_tf32_kmajor(const float* x, long long ldx, bool src_kmajor, int MN, int K, float* hi, float* lo,
                       long long ld2, cudaStream_t s) {
  dim3 grid((unsigned)((ld2 + 31) / 32), (unsigned)((MN + 31) / 32));
  split_kmajor_kernel<<<grid, dim3(32, 8), 0, s>>>(x, ldx, src_kmajor ? 1 : 0, MN, K, hi, lo, ld2);
  after_launch("split_tf32_kmajor");
}

// ---------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(f);
  });
  return fn;
}

// 2-D map over a row-major matrix of `rows` x `cols` (cols contiguous), box
// {box_c, box_r}, SW128.
void encode_2d_sw(CUtensorMap* m, const void* ptr, be_dtype dt, uint64_t cols, uint64_t rows, uint64_t ld,
                  uint32_t box_c, uint32_t box_r, CUtensorMapSwizzle sw) {
  EncodeFn enc = get_encode();
  BE_REQUIRE(enc != nullptr, BE_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const size_t es = dtype_size(dt);
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * es};
  cuuint32_t box[2] = {box_c, box_r};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt == BE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BE_REQUIRE(r == CUDA_SUCCESS, BE_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}
// 4-D tiled bf16 map over an NHWC-like tensor dims {d0 (contiguous), d1, d2, d3}
// with element strides {1, es, es, 1}, box {b0, b1·es, b2·es, 1}, SW128.
bool encode_4d_tiled(CUtensorMap* m, const void* ptr, const uint64_t (&dims)[4], uint32_t b0, uint32_t b1, uint32_t b2,
                     uint32_t es) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t st[3] = {dims[0] * 2, dims[0] * dims[1] * 2, dims[0] * dims[1] * dims[2] * 2};
  cuuint32_t box[4] = {b0, b1 * es, b2 * es, 1};
  cuuint32_t estr[4] = {1, es, es, 1};
  if (box[1] > 256 || box[2] > 256) return false;
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), d, st, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
void encode_2d(CUtensorMap* m, const void* ptr, be_dtype dt, uint64_t cols, uint64_t rows, uint64_t ld,
               uint32_t box_c, uint32_t box_r) {
  encode_2d_sw(m, ptr, dt, cols, rows, ld, box_c, box_r, CU_TENSOR_MAP_SWIZZLE_128B);
}
// 4-D NHWC im2col map for a convolution's input (bf16): box = `pixels`
// output positions × `chans` channels, SW128; corners per CUTLASS's
// convention: lower = −pad, upper = pad − (R−1); traversal stride = conv stride.
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool encode_im2col_4d(CUtensorMap* m, const void* x, const ConvGeom& g, int chans, int pixels,
                      const int* corners = nullptr) {
  static EncodeIm2colFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeIm2colFn) nullptr;
    return reinterpret_cast<EncodeIm2colFn>(f);
  }();
  if (!fn || g.R - 1 - g.pad > 255 || g.S - 1 > 255) return false;
  cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
  cuuint64_t strides[3] = {(cuuint64_t)g.C * 2, (cuuint64_t)g.W * g.C * 2, (cuuint64_t)g.H * g.W * g.C * 2};
  int lower[2] = {-g.pad, -g.pad};
  int upper[2] = {g.pad - (g.S - 1), g.pad - (g.R - 1)};
  if (corners) {  // explicit {lower w, lower h, upper w, upper h}
    lower[0] = corners[0]; lower[1] = corners[1]; upper[0] = corners[2]; upper[1] = corners[3];
    if (lower[0] < -128 || lower[1] < -128 || upper[0] > 127 || upper[1] > 127) return false;
  }
  cuuint32_t es[4] = {1, (cuuint32_t)g.stride, (cuuint32_t)g.stride, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower, upper,
                  (cuuint32_t)chans, (cuuint32_t)pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// TMA-store epilogue map over the output (rows × N, row stride ld) when
// possible: 16-B aligned rows; beta = 0 → bulk tensor store, beta = 1 →
// bulk tensor reduce-add (one add per element: deterministic). Box 32×32 with
// SW128 (fp32, 128-B rows) or SW64 (bf16, 64-B rows) — epi_tma32's layout.
void setup_store(GemmParams& p, void* D, bool f32, long long rows, int N, long long ld) {
  p.tma_store = 0;
  static const int enabled = [] { const char* e = getenv("BE_TMA_STORE"); return e ? atoi(e) : 1; }();
  if (!enabled || (p.beta != 0.f && p.beta != 1.f)) return;
  const int es = f32 ? 4 : 2;
  if ((ld * es) % 16 != 0 || (reinterpret_cast<uintptr_t>(D) & 15) != 0 || rows <= 0 || N <= 0) return;
  encode_2d_sw(&p.td, D, f32 ? BE_F32 : BE_BF16, (uint64_t)N, (uint64_t)rows, (uint64_t)ld, 32, 32,
               f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
  p.tma_store = p.beta == 1.f ? 2 : 1;  // 2: bulk tensor reduce-add (D += result)
}

// Operand map: logical [MN, K]; kmajor → stored [MN rows, K cols]; else [K rows, MN cols].
void encode_operand(CUtensorMap* m, const void* ptr, be_dtype dt, int MN, int K, int64_t ld, bool kmajor,
                    int box_mn, int bk) {
  const uint32_t ch = 128 / dtype_size(dt);
  if (kmajor) encode_2d(m, ptr, dt, K, MN, ld, bk, box_mn);
  else encode_2d(m, ptr, dt, MN, K, ld, ch, bk);
}

bool tma_ok(const void* p, int64_t ld, be_dtype dt) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld * (int64_t)dtype_size(dt)) % 16 == 0;
}

// fused SGD epilogue parameters (GemmDesc::upd): P is [M, N] with ld = ldd
}  // namespace
bool gemm_update_ok(const GemmDesc& g) {
  if (!g.upd || g.ab != BE_BF16) return false;
  const uintptr_t pa = reinterpret_cast<uintptr_t>(g.upd->p), va = reinterpret_cast<uintptr_t>(g.upd->v),
                  sa = reinterpret_cast<uintptr_t>(g.upd->shadow);
  if (g.ldd % 8 != 0 || ((pa | va | sa) & 15) != 0) return false;  // TMA: 16-B aligned bases and row pitches
  // the update epilogue needs the whole K sum in one CTA (no split-K): a
  // small-output, long-K wgrad (NCF's 256×256 tower layers, K = 8192: 4–16
  // tiles on 148 SMs, 45 µs) runs faster as a split-K GEMM + the SGD kernel
  const long long tiles = (long long)((g.M + 127) / 128) * ((g.N + 127) / 128);
  return !(tiles * 4 < ctx().num_sms && g.K > 2048);
}
namespace {
void set_update(GemmParams& p, const GemmDesc& g) {
  BE_REQUIRE(gemm_update_ok(g), BE_E_ARG, "gemm: update epilogue needs 16-B aligned P/V rows, 8-B aligned shadow");
  // P / V chunks are TMA-loaded as 32 × 16 fp32 boxes (zero fill past the edges)
  encode_2d_sw(&p.tp[0], g.upd->p, BE_F32, (uint64_t)g.N, (uint64_t)g.M, (uint64_t)g.ldd, kUpdCW, 32,
               CU_TENSOR_MAP_SWIZZLE_64B);
  if (g.upd->v)
    encode_2d_sw(&p.tp[1], g.upd->v, BE_F32, (uint64_t)g.N, (uint64_t)g.M, (uint64_t)g.ldd, kUpdCW, 32,
                 CU_TENSOR_MAP_SWIZZLE_64B);
  if (g.upd->shadow)
    encode_2d_sw(&p.td, g.upd->shadow, BE_BF16, (uint64_t)g.N, (uint64_t)g.M, (uint64_t)g.ldd, kUpdCW, 32,
                 CU_TENSOR_MAP_SWIZZLE_32B);
  p.upd = 1;
  p.upd_p = g.upd->p; p.upd_v = g.upd->v; p.upd_shadow = g.upd->shadow;
  p.lr = g.upd->lr; p.mu = g.upd->mu; p.wd = g.upd->wd; p.gscale = g.upd->scale;
  p.ldd = g.ldd;
  p.tma_store = 0;
  p.D = nullptr;
}
// per parameter element: p read+write, v read+write (momentum), shadow write
// BN statistics epilogue (GemmDesc::stats)
void set_stats(GemmParams& p, const GemmDesc& g, int grid) {
  p.stats = nullptr;
  if (!g.stats) return;
  BE_REQUIRE(!g.bias && !g.act && g.beta == 0.f && p.splits == 1, BE_E_ARG,
             "gemm: statistics epilogue needs a plain (no bias/act/beta, unsplit) output");
  p.stats = g.stats;
  if (g.stats_parts) *g.stats_parts = grid * 4;
}
double update_bytes(const GemmDesc& g) {
  return 8.0 + (g.upd->v ? 8.0 : 0.0) + (g.upd->shadow ? 2.0 : 0.0);
}

template <int BN, bool X3, int NSLOT = 2, bool XF = false>
void launch_tc(const GemmDesc& g, const void* a_hi, const void* a_lo, const void* b_hi, const void* b_lo,
               cudaStream_t s, int force_splits = 0) {
  using C = Cfg<BN, X3, false, NSLOT, XF>;
  static bool attr_set = false;
  if (!attr_set) {
    BE_CHECK_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, X3, false, NSLOT, XF>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  GemmParams p;
  memset(&p, 0, sizeof(p));
  const be_dtype dt = X3 ? BE_F32 : BE_BF16;
  encode_operand(&p.ta[0], a_hi, dt, g.M, g.K, g.lda, g.a_kmajor, BM, C::BK);
  int Keff = g.K;  // the GEMM's reduction length as the kernel walks it
  if (!X3 && g.conv_x && g.conv_shift) {
    // wgrad, shifted-tile mode: pixel blocks of hb output rows × wb columns
    const ConvGeom& cg = g.conv_g;
    int wb = 1;
    while (wb < cg.Q) wb *= 2;
    BE_REQUIRE(wb <= 64 && cg.C % 64 == 0 && g.M % 8 == 0, BE_E_ARG, "shift wgrad: Q <= 64, C % 64, K % 8");
    const int hb = 64 / wb, pg = (cg.P + hb - 1) / hb;
    const uint64_t ddy[4] = {(uint64_t)g.M, (uint64_t)cg.Q, (uint64_t)cg.P, (uint64_t)cg.N};
    const uint64_t dx[4] = {(uint64_t)cg.C, (uint64_t)cg.W, (uint64_t)cg.H, (uint64_t)cg.N};
    BE_REQUIRE(encode_4d_tiled(&p.ta[0], g.A, ddy, 64, wb, hb, 1), BE_E_CUDA, "dY 4-D map encode failed");
    BE_REQUIRE(encode_4d_tiled(&p.tb[1], g.conv_x, dx, 64, wb, hb, cg.stride), BE_E_CUDA, "x 4-D map encode failed");
    encode_2d(&p.tb[0], g.conv_x, BE_BF16, (uint64_t)cg.C, (uint64_t)cg.N * cg.H * cg.W, (uint64_t)cg.C, 64, 64);
    p.b_shift = 1; p.sh_wb = wb; p.sh_hb = hb; p.sh_pg = pg;
    p.cN = cg.N; p.cH = cg.H; p.cW = cg.W; p.cC = cg.C; p.cR = cg.R; p.cS = cg.S;
    p.cstride = cg.stride; p.cpad = cg.pad; p.cP = cg.P; p.cQ = cg.Q;
    Keff = cg.N * pg * 64;
  } else if (!X3 && g.conv_x) {
    // wgrad B = im2col(x): tb[1] im2col map (64 pixels × 64 channels per op);
    // tb[0] = x as a plain 2-D map (only prefetched)
    const ConvGeom& cg = g.conv_g;
    BE_REQUIRE(encode_im2col_4d(&p.tb[1], g.conv_x, cg, 64, C::BK), BE_E_CUDA, "im2col map encode failed");
    encode_2d(&p.tb[0], g.conv_x, BE_BF16, (uint64_t)cg.C, (uint64_t)cg.N * cg.H * cg.W, (uint64_t)cg.C, 64, 64);
    p.b_im2col = 1;
    p.cN = cg.N; p.cH = cg.H; p.cW = cg.W; p.cC = cg.C; p.cR = cg.R; p.cS = cg.S;
    p.cstride = cg.stride; p.cpad = cg.pad; p.cP = cg.P; p.cQ = cg.Q;
  } else {
    encode_operand(&p.tb[0], b_hi, dt, g.N, g.K, g.ldb, g.b_kmajor, BN, C::BK);
  }
  if (X3) {
    encode_operand(&p.ta[1], a_lo, dt, g.M, g.K, g.lda, g.a_kmajor, BM, C::BK);
    encode_operand(&p.tb[1], b_lo, dt, g.N, g.K, g.ldb, g.b_kmajor, BN, C::BK);
  }
  p.M = g.M; p.N = g.N; p.K = Keff;
  p.a_kmajor = g.a_kmajor; p.b_kmajor = g.b_kmajor;
  p.tiles_m = (g.M + BM - 1) / BM;
  p.tiles_n = (g.N + BN - 1) / BN;
  const int sms = ctx().num_sms;
  const int mn = p.tiles_m * p.tiles_n;
  const int kblocks = (Keff + C::BK - 1) / C::BK;
  // split-K when the output tile grid cannot fill the machine (e.g. conv
  // wgrad: M·N tiny, K = N·P·Q up to 3.2 M); fp32 partials are summed in a
  // fixed order by splitk_reduce → deterministic.
  int splits = 1;
  if (g.upd || g.stats) splits = 1;  // the update / statistics epilogues need the complete result
  else if (force_splits > 0) splits = std::max(1, std::min(force_splits, kblocks));
  else if (mn * 2 <= sms && kblocks >= 8) splits = std::max(1, std::min(sms / mn, kblocks / 4));
  int kps = (kblocks + splits - 1) / splits;
  splits = (kblocks + kps - 1) / kps;
  p.splits = splits;
  p.kb_per_split = kps;
  Block* ws = nullptr;
  if (splits > 1) {
    // one slab per split, BM-row padded so a tile never spills into the next slab
    p.split_rows = p.tiles_m * BM;
    p.split_stride = (long long)p.split_rows * g.N;
    ws = ctx().alloc.allocate(sizeof(float) * (size_t)splits * p.split_stride, s);
    p.D = ws->ptr; p.ldd = g.N; p.d_f32 = 1; p.beta = 0.f; p.bias = nullptr; p.act = 0;
  } else {
    p.D = g.D; p.ldd = g.ldd; p.d_f32 = g.d == BE_F32; p.beta = g.beta; p.bias = g.bias; p.act = g.act;
    p.split_stride = 0;
    p.split_rows = 0;
  }
  if (g.upd) set_update(p, g);
  else setup_store(p, p.D, p.d_f32 != 0, splits > 1 ? (long long)splits * p.split_rows : g.M, g.N, p.ldd);
  const int grid = std::min(mn * splits, sms);
  set_stats(p, g, grid);
  static const int split_on = [] { const char* e = getenv("BE_EPI_SPLIT"); return e ? atoi(e) : 1; }();
  p.epi_split = (BN == 64 && !X3 && !g.upd && !p.stats && split_on) ? 1 : 0;
  if (XF) {
    p.xf_op = g.xf_op; p.xf_act = g.xf_act; p.xf_C = g.xf_C;
    p.xf_mean = g.xf_mean; p.xf_invstd = g.xf_invstd; p.xf_gamma = g.xf_gamma; p.xf_beta = g.xf_beta;
  }
  const double es = X3 ? 4.0 : 2.0, ds = g.d == BE_F32 ? 4.0 : 2.0;
  const double alg_bytes = ((double)g.M * g.K + (double)g.N * g.K) * es +
                           (double)g.M * g.N * (g.upd ? update_bytes(g) : ds * (g.beta != 0.f ? 2 : 1));
  const int pidx = prof_begin(g.upd ? "gemm_upd" : (X3 ? "gemm_tc_3xtf32" : "gemm_tc_bf16"), 2.0 * g.M * g.N * g.K,
                              alg_bytes, g.M, g.N, g.K, s);
  if (g.upd) {
    if constexpr (!X3) {
      using CU = Cfg<BN, false, true>;
      static bool upd_attr = false;
      if (!upd_attr) {
        BE_CHECK_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           CU::SMEM));
        upd_attr = true;
      }
      launch_pdl(gemm_tc_kernel<BN, false, true>, grid, kThreads, CU::SMEM, s, p);
    } else {
      fail(BE_E_ARG, "gemm: the update epilogue runs on the bf16 kernel");
    }
  } else {
    launch_pdl(gemm_tc_kernel<BN, X3, false, NSLOT, XF>, grid, kThreads, C::SMEM, s, p);
  }
  prof_end(pidx, s);
  after_launch("gemm_tc");
  if (ws) {
    const long long total = (long long)g.M * g.N;
    launch_splitk(reinterpret_cast<const float*>(ws->ptr), splits, p.split_stride, g.M, g.N, g.D, g.ldd,
                                         g.d == BE_F32, g.beta, g.bias, g.act, s);
    after_launch("gemm_splitk_reduce");
    ctx().alloc.free(ws);
  }
}

void launch_tc2(const GemmDesc& g, cudaStream_t s) {
  using namespace pair;
  static bool attr_set = false;
  if (!attr_set) {
    BE_CHECK_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    BE_CHECK_CUDA(cudaFuncSetAttribute(gemm_tc2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_UPD));
    attr_set = true;
  }
  GemmParams p;
  memset(&p, 0, sizeof(p));
  encode_operand(&p.ta[0], g.A, BE_BF16, g.M, g.K, g.lda, g.a_kmajor, HM, BK);
  encode_operand(&p.tb[0], g.B, BE_BF16, g.N, g.K, g.ldb, g.b_kmajor, HN, BK);
  p.M = g.M; p.N = g.N; p.K = g.K;
  p.a_kmajor = g.a_kmajor; p.b_kmajor = g.b_kmajor;
  p.tiles_m = (g.M + TM - 1) / TM;
  p.tiles_n = (g.N + TN - 1) / TN;
  const int pairs = ctx().num_sms / 2;
  const int mn = p.tiles_m * p.tiles_n;
  const int kblocks = (g.K + BK - 1) / BK;
  int splits = 1;
  if (!g.upd && !g.stats && mn * 2 <= pairs && kblocks >= 8) splits = std::max(1, std::min(pairs / mn, kblocks / 4));
  int kps = (kblocks + splits - 1) / splits;
  splits = (kblocks + kps - 1) / kps;
  p.splits = splits;
  p.kb_per_split = kps;
  Block* ws = nullptr;
  if (splits > 1) {
    p.split_rows = p.tiles_m * TM;
    p.split_stride = (long long)p.split_rows * g.N;
    ws = ctx().alloc.allocate(sizeof(float) * (size_t)splits * p.split_stride, s);
    p.D = ws->ptr; p.ldd = g.N; p.d_f32 = 1; p.beta = 0.f; p.bias = nullptr; p.act = 0;
  } else {
    p.D = g.D; p.ldd = g.ldd; p.d_f32 = g.d == BE_F32; p.beta = g.beta; p.bias = g.bias; p.act = g.act;
  }
  if (g.upd) set_update(p, g);
  else setup_store(p, p.D, p.d_f32 != 0, splits > 1 ? (long long)splits * p.split_rows : g.M, g.N, p.ldd);
  const int grid = 2 * std::min(mn * splits, pairs);
  set_stats(p, g, grid);
  const double ds = g.d == BE_F32 ? 4.0 : 2.0;
  const double alg_bytes = ((double)g.M * g.K + (double)g.N * g.K) * 2.0 +
                           (double)g.M * g.N * (g.upd ? update_bytes(g) : ds * (g.beta != 0.f ? 2 : 1));
  const int pidx = prof_begin(g.upd ? "gemm_upd2" : "gemm_tc2_bf16", 2.0 * g.M * g.N * g.K, alg_bytes, g.M, g.N, g.K, s);
  if (g.upd) launch_pdl(gemm_tc2_kernel<true>, grid, kThreads, SMEM_UPD, s, p);
  else launch_pdl(gemm_tc2_kernel<false>, grid, kThreads, SMEM, s, p);
  prof_end(pidx, s);
  after_launch("gemm_tc2");
  if (ws) {
    const long long total = (long long)g.M * g.N;
    launch_splitk(reinterpret_cast<const float*>(ws->ptr), splits, p.split_stride, g.M, g.N, g.D, g.ldd,
                                         g.d == BE_F32, g.beta, g.bias, g.act, s);
    after_launch("gemm_splitk_reduce");
    ctx().alloc.free(ws);
  }
}

// CTA-pair candidate: BE_GEMM_PAIR=0 drops it, =1 forces it where plausible;
// otherwise it is one of gemm()'s autotuned candidates (runtime.cpp tune_choose)
int pair_mode() {
  static int mode = [] { const char* e = getenv("BE_GEMM_PAIR"); return e ? atoi(e) : -1; }();
  return mode;
}
bool pair_plausible(const GemmDesc& g) {
  const long tiles = (long)((g.M + 255) / 256) * ((g.N + 255) / 256);
  return g.M >= 256 && g.N >= 192 && tiles >= 8;
}
std::string tune_key(const GemmDesc& g) {
  return std::to_string(g.M) + "x" + std::to_string(g.N) + "x" + std::to_string(g.K) + (g.a_kmajor ? "k" : "m") +
         (g.b_kmajor ? "k" : "m") + (g.d == BE_F32 ? "f" : "h");
}
int pick_bn(int M, int N, int sms, bool x3) {
  // Largest BN whose wave efficiency is within 10% of the best candidate.
  const int cands_bf16[3] = {256, 128, 64};
  const int cands_x3[2] = {128, 64};
  const int* c = x3 ? cands_x3 : cands_bf16;
  const int nc = x3 ? 2 : 3;
  double best = 0; int best_bn = c[nc - 1];
  double eff[3];
  for (int i = 0; i < nc; ++i) {
    long tiles = (long)((M + BM - 1) / BM) * ((N + c[i] - 1) / c[i]);
    long waves = (tiles + sms - 1) / sms;
    double useful = (double)M * N;
    double issued = (double)waves * sms * BM * c[i];
    eff[i] = useful / issued;
    if (eff[i] > best) best = eff[i];
  }
  for (int i = 0; i < nc; ++i)
    if (eff[i] >= 0.9 * best) { best_bn = c[i]; break; }
  return best_bn;
}

}  // namespace

template <int BN>
void launch_conv(GemmParams& p, cudaStream_t s, int* stats_parts) {
  using C = conv::Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    BE_CHECK_CUDA(cudaFuncSetAttribute(conv_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  p.tiles_m = (p.M + BM - 1) / BM;
  p.tiles_n = (p.N + BN - 1) / BN;
  const int grid = std::min(p.tiles_m * p.tiles_n, ctx().num_sms);
  if (p.stats && stats_parts) *stats_parts = grid * 4;
  launch_pdl(conv_tc_kernel<BN>, grid, conv::kThreads, C::SMEM, s, p);
}

template <int BN>
void launch_conv_small_c(GemmParams& p, cudaStream_t s, int* stats_parts) {
  using C = convs::Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    BE_CHECK_CUDA(cudaFuncSetAttribute(conv_small_c_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  p.tiles_m = (p.M + BM - 1) / BM;
  p.tiles_n = (p.N + BN - 1) / BN;
  const int grid = std::min(p.tiles_m * p.tiles_n, ctx().num_sms);
  if (p.stats && stats_parts) *stats_parts = grid * 4;
  launch_pdl(conv_small_c_kernel<BN>, grid, convs::kThreads, C::SMEM, s, p);
}

static bool conv_small_c(const void* x, const void* w, void* y, const ConvGeom& g, be_dtype yd, const float* bias,
                         int act, float beta, cudaStream_t s, float* stats, int* stats_parts) {
  const int RSC = g.R * g.S * g.C;
  if (!(g.C == 8 || g.C == 16 || g.C == 32) || g.K % 16 != 0 || (RSC + 63) / 64 * 8 > convs::kMaxChunks) return false;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(w) & 15)) return false;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.M = g.N * g.P * g.Q; p.N = g.K; p.K = RSC;
  p.a_kmajor = 1; p.b_kmajor = 1; p.splits = 1;
  p.D = y; p.ldd = g.K; p.d_f32 = yd == BE_F32; p.beta = beta; p.bias = bias; p.act = act;
  p.stats = (stats && !bias && !act && beta == 0.f) ? stats : nullptr;
  p.x = reinterpret_cast<const uint16_t*>(x);
  p.cN = g.N; p.cH = g.H; p.cW = g.W; p.cC = g.C; p.cR = g.R; p.cS = g.S;
  p.cstride = g.stride; p.cpad = g.pad; p.cP = g.P; p.cQ = g.Q;
  const int bn = g.K >= 128 ? 128 : 64;
  encode_operand(&p.tb[0], w, BE_BF16, g.K, RSC, RSC, true, bn, 64);
  const double flops = 2.0 * p.M * (double)g.K * RSC;
  const double bytes = ((double)g.N * g.H * g.W * g.C + (double)g.K * RSC) * 2.0 +
                       (double)p.M * g.K * (yd == BE_F32 ? 4 : 2);
  const int pidx = prof_begin("conv_tc_small_c", flops, bytes, p.M, g.K, RSC, s);
  setup_store(p, y, p.d_f32 != 0, p.M, g.K, g.K);
  if (bn == 128) launch_conv_small_c<128>(p, s, stats_parts);
  else launch_conv_small_c<64>(p, s, stats_parts);
  prof_end(pidx, s);
  after_launch("conv_tc_small_c");
  g_tc_calls++;
  return true;
}

bool conv_wgrad_patch(const void* dy, const void* x, void* dw, be_dtype dwt, const ConvGeom& g, float beta,
                      cudaStream_t s) {
  static const int on = [] { const char* e = getenv("BE_WGRAD_PATCH"); return e ? atoi(e) : 1; }();
  if (!on || g.stride != 1 || dwt != BE_F32 || g.R * g.S > 64) return false;
  if (!((g.C == 64 && g.K % 64 == 0 && g.K <= 256) || (g.C == 128 && g.K == 128))) return false;
  const wgp::Geo gg = wgp::geo(g.Q, g.R, g.S, g.C, g.K);
  if (gg.Wp > BM || gg.nbuf < 2 || gg.G + g.R - 1 > 256 || gg.gs > 8 || gg.ngroups * 2 > ctx().num_sms) return false;
  if ((reinterpret_cast<uintptr_t>(dy) & 15) || (reinterpret_cast<uintptr_t>(x) & 15)) return false;
  const int smem = 1024 + gg.nbuf * gg.bufb + 256;
  if (smem > 227 * 1024) return false;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  const uint64_t dx4[4] = {(uint64_t)g.C, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N};
  const uint64_t dy4[4] = {(uint64_t)g.K, (uint64_t)g.Q, (uint64_t)g.P, (uint64_t)g.N};
  if (!encode_4d_tiled(&p.ta[0], x, dx4, 64, gg.Wp, gg.G + g.R - 1, 1)) return false;
  if (!encode_4d_tiled(&p.tb[0], dy, dy4, 64, gg.Wp, gg.G, 1)) return false;
  p.cN = g.N; p.cH = g.H; p.cW = g.W; p.cC = g.C; p.cR = g.R; p.cS = g.S; p.cP = g.P; p.cQ = g.Q;
  p.cstride = 1; p.cpad = g.pad; p.N = g.K;
  const int RSC = g.R * g.S * g.C;
  const int tiles = g.N * ((g.P + gg.G - 1) / gg.G);
  const int splits = std::max(1, std::min(tiles, ctx().num_sms / gg.ngroups));
  const int grid = splits * gg.ngroups;
  p.split_stride = (long long)g.K * RSC;
  Block* ws = ctx().alloc.allocate(sizeof(float) * (size_t)splits * p.split_stride, s);
  p.D = ws->ptr;
  static bool attr = false;
  if (!attr) {
    BE_CHECK_CUDA(cudaFuncSetAttribute(conv_wgrad_patch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    attr = true;
  }
  const double flops = 2.0 * g.N * g.P * g.Q * (double)g.K * RSC;
  const double bytes = ((double)g.N * g.H * g.W * g.C + (double)g.N * g.P * g.Q * g.K) * 2.0 + 4.0 * g.K * RSC;
  const int pidx = prof_begin("conv_tc_wgrad_patch", flops, bytes, g.K, RSC, g.N * g.P * g.Q, s);
  launch_pdl(conv_wgrad_patch_kernel, grid, wgp::kThreads, smem, s, p);
  prof_end(pidx, s);
  after_launch("conv_wgrad_patch");
  g_tc_calls++;
  const long long total = (long long)g.K * RSC;
  launch_splitk(reinterpret_cast<const float*>(ws->ptr), splits, p.split_stride, g.K, RSC, dw,
                                       RSC, 1, beta, nullptr, 0, s);
  after_launch("conv_wgrad_patch_reduce");
  ctx().alloc.free(ws);
  return true;
}

// stem conv weight gradient (conv_wgrad_stem_kernel): C = 8, K = 64, Q ≤ 128,
// R·S ≤ 128; dw fp32 [64, R·S·8] (+)= dW; false when not applicable
// conv wgrad with the im2col slice gathered in smem (conv_wgrad_gather_kernel);
// false when the shape does not fit (C % 64, K % 128, (R·S·C) % BN)
bool conv_wgrad_gather(const void* dy, const void* x, void* dw, be_dtype dwt, const ConvGeom& g, float beta,
                       cudaStream_t s) {
  static const int on = [] { const char* e = getenv("BE_WGRAD_GATHER"); return e ? atoi(e) : 1; }();
  const int RSC = g.R * g.S * g.C;
  static const int bn_env = [] { const char* e = getenv("BE_WGG_BN"); return e ? atoi(e) : 0; }();
  const int bn = (bn_env != 128 && RSC % 256 == 0 && g.C % 256 == 0) ? 256 : 128;
  if (!on || dwt != BE_F32 || g.C % 64 != 0 || g.K % 128 != 0 || RSC % bn != 0 || (beta != 0.f && beta != 1.f))
    return false;
  if ((reinterpret_cast<uintptr_t>(dy) & 15) || (reinterpret_cast<uintptr_t>(x) & 15)) return false;
  const long long pixels = (long long)g.N * g.P * g.Q;
  if (pixels >= (1LL << 31) || (long long)g.N * g.H * g.W * g.C >= (1LL << 40)) return false;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.M = g.K; p.N = RSC; p.K = (int)pixels;
  p.x = reinterpret_cast<const uint16_t*>(x);
  p.cN = g.N; p.cH = g.H; p.cW = g.W; p.cC = g.C; p.cR = g.R; p.cS = g.S;
  p.cstride = g.stride; p.cpad = g.pad; p.cP = g.P; p.cQ = g.Q;
  encode_operand(&p.ta[0], dy, BE_BF16, g.K, (int)pixels, g.K, false, 64, 64);  // dY as [pixels, K]: MN-major A
  p.tiles_m = g.K / BM; p.tiles_n = RSC / bn;
  const int mn = p.tiles_m * p.tiles_n, sms = ctx().num_sms;
  const int kblocks = (int)((pixels + 63) / 64);
  int splits = std::max(1, std::min(2 * sms / mn, kblocks / 4));
  int kps = (kblocks + splits - 1) / splits;
  splits = (kblocks + kps - 1) / kps;
  p.splits = splits; p.kb_per_split = kps;
  p.split_rows = p.tiles_m * BM;
  p.split_stride = (long long)p.split_rows * RSC;
  Block* ws = ctx().alloc.allocate(sizeof(float) * (size_t)splits * p.split_stride, s);
  p.D = ws->ptr; p.ldd = RSC; p.d_f32 = 1; p.beta = 0.f;
  setup_store(p, ws->ptr, true, (long long)splits * p.split_rows, RSC, RSC);
  BE_REQUIRE(p.tma_store == 1, BE_E_CUDA, "conv_wgrad_gather: slab store map");
  const int grid = std::min(mn * splits, sms);
  const double flops = 2.0 * pixels * (double)g.K * RSC;
  const double bytes = ((double)g.N * g.H * g.W * g.C + (double)pixels * g.K) * 2.0 + 4.0 * g.K * RSC;
  const int pidx = prof_begin("conv_tc_wgrad_gather", flops, bytes, g.K, RSC, (int)pixels, s);
  if (bn == 256) {
    static bool a = false;
    if (!a) { BE_CHECK_CUDA(cudaFuncSetAttribute(conv_wgrad_gather_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, wgg::Cfg<256>::SMEM)); a = true; }
    launch_pdl(conv_wgrad_gather_kernel<256>, grid, wgg::kThreads, wgg::Cfg<256>::SMEM, s, p);
  } else {
    static bool a = false;
    if (!a) { BE_CHECK_CUDA(cudaFuncSetAttribute(conv_wgrad_gather_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, wgg::Cfg<128>::SMEM)); a = true; }
    launch_pdl(conv_wgrad_gather_kernel<128>, grid, wgg::kThreads, wgg::Cfg<128>::SMEM, s, p);
  }
  prof_end(pidx, s);
  after_launch("conv_wgrad_gather");
  g_tc_calls++;
  const long long total = (long long)g.K * RSC;
  launch_splitk(reinterpret_cast<const float*>(ws->ptr), splits,
             p.split_stride, g.K, RSC, dw, (long long)RSC, 1, beta, (const float*)nullptr, 0, s);
  after_launch("conv_wgrad_gather_reduce");
  ctx().alloc.free(ws);
  return true;
}

bool conv_wgrad_stem(const void* dy, const void* x, void* dw, be_dtype dwt, const ConvGeom& g, float beta,
                     cudaStream_t s) {
  static const int on = [] { const char* e = getenv("BE_WGRAD_STEM"); return e ? atoi(e) : 1; }();
  if (!on || g.C != 8 || g.K != 64 || dwt != BE_F32 || g.Q > BM || g.Q < 1 || g.R * g.S > 128) return false;
  const wgs::Geo e = wgs::geo(g);
  if (e.L * g.stride > 2 * wgs::kCopy || e.ns < 2 || e.smem > 227 * 1024) return false;
  if ((reinterpret_cast<uintptr_t>(dy) & 15) || (reinterpret_cast<uintptr_t>(x) & 15)) return false;
  // Hankel-operand kernel when the R·S·8 accumulator columns fit TMEM
  const bool hankel = on != 1 ? on == 2
                                : (g.R * g.S * 8 <= 512 && g.R * g.stride <= 32 && wgh::smem_bytes(g, e.phb) <= 227 * 1024);
  GemmParams p;
  memset(&p, 0, sizeof(p));
  const uint64_t dy4[4] = {(uint64_t)g.K, (uint64_t)g.Q, (uint64_t)g.P, (uint64_t)g.N};
  p.x = reinterpret_cast<const uint16_t*>(x);
  p.cN = g.N; p.cH = g.H; p.cW = g.W; p.cC = g.C; p.cR = g.R; p.cS = g.S; p.cP = g.P; p.cQ = g.Q;
  p.cstride = g.stride; p.cpad = g.pad;
  p.st_L = e.L; p.st_phb = e.phb; p.st_taps = e.Mt; p.st_nbuf = e.ns | (e.np << 8);
  // two output rows per MMA for the ResNet stem geometry
  bool two_rows = hankel && g.R == 7 && g.S == 7 && g.stride == 2 && on != 3 && wgh2::smem_bytes(e.L) <= 227 * 1024;
  if (hankel) {  // BE_HANKEL_DBG (timing experiments only): bit 0 skips the MMAs, bit 1 the patch copies
    static const int dbg = [] { const char* v = getenv("BE_HANKEL_DBG"); return v ? atoi(v) : 0; }();
    p.st_wbytes = dbg;
  }
  if (two_rows) {
    // patch map: x [N, H, W, 8] bf16, W traversed with stride 2 (one column
    // phase per load), box 8 × L × 9 rows, no swizzle (phase-split layout)
    EncodeFn enc = get_encode();
    cuuint64_t d[4] = {8, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
    cuuint64_t st4[3] = {16, (cuuint64_t)g.W * 16, (cuuint64_t)g.H * g.W * 16};
    cuuint32_t box[4] = {8, (cuuint32_t)(2 * e.L), (cuuint32_t)wgh2::RJ, 1};
    cuuint32_t estr[4] = {1, 2, 1, 1};
    if (!enc || 2 * e.L > 256 ||
        enc(&p.ta[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), d, st4, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      two_rows = false;
    else
      p.st_phb = wgh2::phb(e.L);
  }
  if (!encode_4d_tiled(&p.tb[0], dy, dy4, 64, 128, two_rows ? 2 : 1, 1)) return false;
  const int RSC = g.R * g.S * 8;
  const int grid = std::min(two_rows ? g.N * ((g.P + 1) / 2) : g.N * g.P, ctx().num_sms);
  p.split_stride = 64LL * RSC;
  Block* ws = ctx().alloc.allocate(sizeof(float) * (size_t)grid * p.split_stride, s);
  p.D = ws->ptr;
  static bool attr = false;
  if (!attr) {
    BE_CHECK_CUDA(cudaFuncSetAttribute(conv_wgrad_stem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    BE_CHECK_CUDA(cudaFuncSetAttribute(conv_wgrad_hankel_kernel<0, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    BE_CHECK_CUDA(cudaFuncSetAttribute(conv_wgrad_hankel_kernel<7, 7, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    BE_CHECK_CUDA(cudaFuncSetAttribute(conv_wgrad_hankel2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    attr = true;
  }
  const double flops = 2.0 * g.N * g.P * g.Q * 64.0 * RSC;
  const double bytes = ((double)g.N * g.H * g.W * 8 + (double)g.N * g.P * g.Q * 64) * 2.0 + 4.0 * 64 * RSC;
  const int pidx = prof_begin("conv_tc_wgrad_stem", flops, bytes, 64, RSC, g.N * g.P * g.Q, s);
  if (two_rows)
    launch_pdl(conv_wgrad_hankel2_kernel, grid, wgh2::kThreads, wgh2::smem_bytes(e.L), s, p);
  else if (hankel)
    launch_pdl(g.R == 7 && g.S == 7 && g.stride == 2 ? conv_wgrad_hankel_kernel<7, 7, 2> : conv_wgrad_hankel_kernel<0, 0, 0>,
               grid, wgh::kThreads, wgh::smem_bytes(g, e.phb), s, p);
  else
    launch_pdl(conv_wgrad_stem_kernel, grid, wgs::kThreads, e.smem, s, p);
  prof_end(pidx, s);
  after_launch("conv_wgrad_stem");
  g_tc_calls++;
  const long long total = 64LL * RSC;
  launch_splitk(reinterpret_cast<const float*>(ws->ptr), grid, p.split_stride, 64, RSC, dw, RSC,
                                       1, beta, nullptr, 0, s);
  after_launch("conv_wgrad_stem_reduce");
  ctx().alloc.free(ws);
  return true;
}

// stride-1 conv from a shared input patch (conv_fwd_patch_kernel): C = K = 64,
// ≤ 9 taps, W' = pow2 ≥ Q + S − 1 in [32, 128]; false when not applicable
static void set_bw(GemmParams& p, const void* w, const ConvGeom& g, const int* bw);
static bool conv_fwd_patch(const void* x, const void* w, void* y, const ConvGeom& g, be_dtype yd, const float* bias,
                           int act, float beta, cudaStream_t s, float* stats = nullptr, int* stats_parts = nullptr,
                           const int* bw = nullptr) {
  if (stats && (yd != BE_BF16 || bias || act || beta != 0.f)) return false;
  static const int on = [] { const char* e = getenv("BE_CONV_PATCH"); return e ? atoi(e) : 1; }();
  if (!on || g.stride != 1 || g.C != 64 || g.K != 64 || g.R * g.S > 9 || (beta != 0.f && beta != 1.f)) return false;
  int Wp = 32;
  while (Wp < g.Q + g.S - 1) Wp *= 2;
  if (Wp > BM) return false;
  const int G = BM / Wp;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(w) & 15) ||
      (reinterpret_cast<uintptr_t>(y) & 15))
    return false;
  const int xbytes = (G + g.R - 1) * Wp * 128;
  const int xstride = (xbytes + cfp::kSlack + 1023) / 1024 * 1024;
  const int smem = 1024 + g.R * g.S * 8192 + cfp::NBUF * xstride + kEpiBytes + 256;
  if (smem > 227 * 1024 || G + g.R - 1 > 256) return false;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  const uint64_t dx4[4] = {(uint64_t)g.C, (uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N};
  if (!encode_4d_tiled(&p.ta[0], x, dx4, 64, Wp, G + g.R - 1, 1)) return false;
  const int RSC = g.R * g.S * g.C;
  if (bw) set_bw(p, w, g, bw);
  else encode_operand(&p.tb[0], w, BE_BF16, g.K, RSC, RSC, true, 64, 64);
  const bool f32 = yd == BE_F32;
  {
    const cuuint64_t es = f32 ? 4 : 2;
    cuuint64_t od[3] = {(cuuint64_t)g.K, (cuuint64_t)g.Q, (cuuint64_t)g.N * g.P};
    cuuint64_t os[2] = {(cuuint64_t)g.K * es, (cuuint64_t)g.Q * g.K * es};
    cuuint32_t ob[3] = {32, 32, 1};
    cuuint32_t oe[3] = {1, 1, 1};
    EncodeFn enc = get_encode();
    if (!enc || enc(&p.td, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, y, od, os, ob,
                    oe, CU_TENSOR_MAP_INTERLEAVE_NONE, f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  p.tma_store = beta == 1.f ? 2 : 1;
  p.M = g.N * g.P * g.Q; p.N = g.K; p.K = RSC;
  p.D = y; p.ldd = g.K; p.d_f32 = f32; p.beta = beta; p.bias = bias; p.act = act;
  p.cN = g.N; p.cH = g.H; p.cW = g.W; p.cC = g.C; p.cR = g.R; p.cS = g.S; p.cP = g.P; p.cQ = g.Q;
  p.cstride = 1; p.cpad = g.pad; p.sh_wb = Wp; p.sh_hb = G;
  static bool attr = false;
  if (!attr) {
    BE_CHECK_CUDA(cudaFuncSetAttribute(conv_fwd_patch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    attr = true;
  }
  const int tiles = g.N * ((g.P + G - 1) / G);
  const int grid = std::min(tiles, ctx().num_sms);
  p.stats = stats;
  if (stats && stats_parts) *stats_parts = grid * 4;
  const double flops = 2.0 * p.M * (double)g.K * RSC;
  const double bytes = ((double)g.N * g.H * g.W * g.C + (double)g.K * RSC) * 2.0 + (double)p.M * g.K * (f32 ? 4 : 2);
  const int pidx = prof_begin("conv_tc_patch", flops, bytes, p.M, g.K, RSC, s);
  launch_pdl(conv_fwd_patch_kernel, grid, cfp::kThreads, smem, s, p);
  prof_end(pidx, s);
  after_launch("conv_tc_patch");
  g_tc_calls++;
  return true;
}

// Phase-split patch convolution (conv_stem_kernel): C = 8, K = 64, stride
// > 1, one output row (Q ≤ 128) per tile.  Returns false when the shape
// does not fit (caller falls back to the gather kernel).
static bool conv_stem(const void* x, const void* w, void* y, const ConvGeom& g, be_dtype yd, const float* bias,
                      int act, float beta, cudaStream_t s, float* stats, int* stats_parts) {
  static const int on = [] { const char* e = getenv("BE_CONV_STEM"); return e ? atoi(e) : 1; }();
  if (!on || g.C != 8 || g.K != stem::BN || g.stride < 2 || g.Q > BM || g.Q < 1) return false;
  const int taps = g.R * g.S;
  const int T = ((g.S + g.stride - 1) / g.stride + 1) / 2 * 2;  // taps per (phase, row), padded even
  const int L = g.Q + T - 1;                                      // columns per phase (padded taps included)
  if (L * g.stride > 2 * stem::kCopyThreads) return false;       // span: 2 columns per copy thread
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(w) & 15)) return false;
  // phase blocks offset by 128/st bytes mod 128: a warp's 16-B copies to the
  // st phases land in different banks
  const int phb = (g.R * L * 16 + 127) / 128 * 128 + (128 / g.stride) / 16 * 16;
  const int patch_bytes = g.stride * phb;
  const int wbytes = g.stride * g.R * T * stem::BN * 16;
  const int fixed = 2048 + stem::kZeroBytes + kEpiBytes + 256;
  const int nbuf = std::min(6, (stem::kSmemCap - fixed - wbytes) / patch_bytes);
  if (nbuf <= stem::LAG) return false;
  const int smem = fixed + wbytes + nbuf * patch_bytes;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.M = g.N * g.P * g.Q; p.N = g.K; p.K = taps * g.C;
  p.D = y; p.ldd = g.K; p.d_f32 = yd == BE_F32; p.beta = beta; p.bias = bias; p.act = act;
  p.stats = (stats && !bias && !act && beta == 0.f) ? stats : nullptr;
  p.x = reinterpret_cast<const uint16_t*>(x);
  p.cN = g.N; p.cH = g.H; p.cW = g.W; p.cC = g.C; p.cR = g.R; p.cS = g.S;
  p.cstride = g.stride; p.cpad = g.pad; p.cP = g.P; p.cQ = g.Q;
  p.st_L = L; p.st_phb = phb; p.st_taps = T; p.st_nbuf = nbuf; p.st_wbytes = wbytes;
  p.st_w = reinterpret_cast<const uint16_t*>(w);
  // output as 3-D [N·P tiles][Q][K]: 32 × 32 TMA-store boxes, q ≥ Q clipped
  static const int tma_on = [] { const char* e = getenv("BE_TMA_STORE"); return e ? atoi(e) : 1; }();
  if (tma_on && (beta == 0.f || beta == 1.f) && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
    const bool f32 = yd == BE_F32;
    const cuuint64_t es = f32 ? 4 : 2;
    cuuint64_t od[3] = {(cuuint64_t)g.K, (cuuint64_t)g.Q, (cuuint64_t)g.N * g.P};
    cuuint64_t os[2] = {(cuuint64_t)g.K * es, (cuuint64_t)g.Q * g.K * es};
    cuuint32_t ob[3] = {32, 32, 1};
    cuuint32_t oe[3] = {1, 1, 1};
    EncodeFn enc = get_encode();
    if (enc && enc(&p.td, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, y, od, os, ob,
                   oe, CU_TENSOR_MAP_INTERLEAVE_NONE, f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      p.tma_store = beta == 1.f ? 2 : 1;
  }
  static int attr_smem = 0;
  if (smem > attr_smem) {
    BE_CHECK_CUDA(cudaFuncSetAttribute(conv_stem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, stem::kSmemCap));
    attr_smem = stem::kSmemCap;
  }
  const int tiles = g.N * g.P;
  const int grid = std::min(tiles, ctx().num_sms);
  if (p.stats && stats_parts) *stats_parts = grid * 4;
  const double flops = 2.0 * p.M * (double)g.K * taps * g.C;
  const double bytes = ((double)g.N * g.H * g.W * g.C + (double)g.K * taps * g.C) * 2.0 +
                       (double)p.M * g.K * (yd == BE_F32 ? 4 : 2);
  const int pidx = prof_begin("conv_tc_stem", flops, bytes, p.M, g.K, taps * g.C, s);
  launch_pdl(conv_stem_kernel, grid, stem::kThreads, smem, s, p);
  prof_end(pidx, s);
  after_launch("conv_tc_stem");
  g_tc_calls++;
  return true;
}

// bw (data-gradient convolutions): {r0, rstep, s0, sstep, S_fwd, RSC_fwd} — w is the FORWARD weight
// W[g.C rows = K_fwd][RSC_fwd] read in place as the MN-major B operand (GemmParams::bw_inplace)
static void set_bw(GemmParams& p, const void* w, const ConvGeom& g, const int* bw) {
  encode_operand(&p.tb[0], w, BE_BF16, bw[5], g.C, bw[5], false, 64, 64);
  p.bw_inplace = 1;
  p.bw_r0 = bw[0]; p.bw_rstep = bw[1]; p.bw_s0 = bw[2]; p.bw_sstep = bw[3]; p.bw_S = bw[4];
}
bool conv_implicit(const void* x, const void* w, void* y, const ConvGeom& g, be_dtype yd, const float* bias, int act,
                   float beta, cudaStream_t s, float* stats, int* stats_parts, const int* bw) {
  if (g.C % 64 != 0) {
    const char* e = getenv("BE_CONV_SMALLC");
    if (e && e[0] == '0') return false;
    if (conv_stem(x, w, y, g, yd, bias, act, beta, s, stats, stats_parts)) return true;
    return conv_small_c(x, w, y, g, yd, bias, act, beta, s, stats, stats_parts);
  }
  if (g.K % 16 != 0) return false;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(w) & 15)) return false;
  if (conv_fwd_patch(x, w, y, g, yd, bias, act, beta, s, stats, stats_parts, bw)) return true;
  const char* e = getenv("BE_CONV_IMPLICIT");
  if (e && e[0] == '0') return false;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  const int RSC = g.R * g.S * g.C;
  p.M = g.N * g.P * g.Q; p.N = g.K; p.K = RSC;
  p.a_kmajor = 1; p.b_kmajor = 1; p.splits = 1;
  p.D = y; p.ldd = g.K; p.d_f32 = yd == BE_F32; p.beta = beta; p.bias = bias; p.act = act;
  p.stats = (stats && !bias && !act && beta == 0.f) ? stats : nullptr;
  p.x = reinterpret_cast<const uint16_t*>(x);
  p.cN = g.N; p.cH = g.H; p.cW = g.W; p.cC = g.C; p.cR = g.R; p.cS = g.S;
  p.cstride = g.stride; p.cpad = g.pad; p.cP = g.P; p.cQ = g.Q;
  const int bn = g.K >= 256 ? 256 : (g.K >= 128 ? 128 : 64);
  if (bw) set_bw(p, w, g, bw);
  else encode_operand(&p.tb[0], w, BE_BF16, g.K, RSC, RSC, true, bn, 64);
  // x as a 2-D [N·H·W, C] matrix; tile::gather4 needs box {64, 1}
  encode_2d(&p.ta[0], x, BE_BF16, (uint64_t)g.C, (uint64_t)g.N * g.H * g.W, (uint64_t)g.C, 64, 1);
  // x as 4-D NHWC im2col map: window starts from −pad to W+pad−R (stride), 128 pixels × 64 channels
  static const int im2col_on = [] { const char* e = getenv("BE_CONV_IM2COL"); return e ? atoi(e) : 1; }();
  if (im2col_on && encode_im2col_4d(&p.ta[1], x, g, 64, BM)) p.use_im2col = 1;
  const double flops = 2.0 * p.M * (double)g.K * RSC;
  const double bytes = ((double)g.N * g.H * g.W * g.C + (double)g.K * RSC) * 2.0 +
                       (double)p.M * g.K * (yd == BE_F32 ? 4 : 2);
  const int pidx = prof_begin("conv_tc_implicit", flops, bytes, p.M, g.K, RSC, s);
  setup_store(p, y, p.d_f32 != 0, p.M, g.K, g.K);
  if (bn == 256) launch_conv<256>(p, s, stats_parts);
  else if (bn == 128) launch_conv<128>(p, s, stats_parts);
  else launch_conv<64>(p, s, stats_parts);
  prof_end(pidx, s);
  after_launch("conv_tc_implicit");
  g_tc_calls++;
  return true;
}

// Taps of a stride-st convolution that reach input rows h ≡ rho (mod st):
// r = rho + pad − st·d for the d with 0 ≤ r < R; count and the smallest d.
static void phase_taps(int R, int st, int pad, int rho, int* cnt, int* dmin) {
  *cnt = 0; *dmin = 0;
  for (int r = R - 1; r >= 0; --r) {
    const int num = rho + pad - r;
    if (((num % st) + st) % st != 0) continue;
    if (*cnt == 0) *dmin = num / st;  // r descending → d ascending; first hit is the smallest
    ++*cnt;
  }
}

// Stride-st data gradient as st² stride-1 phase convolutions:
// for output rows h = st·i + ρh, dx[n, h, w, :] = Σ_{t_r, t_s} dY[n, i + dminh + t_r,
// j + dminw + t_s, :] · W[:, r(t_r), s(t_s), :] with r(t) = ρh + pad − st·(dminh + t)
// (likewise s) — every term of the transposed convolution, none of the
// zero-inserted ones.  Each phase is one conv_tc_kernel launch: A = dY through
// a TMA im2col map whose corners give the phase's window, B = the phase's
// taps of W read in place as the MN-major B operand (GemmParams::bw_*), and the epilogue
// stores row (n, i, j) straight to dx pixel (n, st·i + ρh, st·j + ρw) (beta 1:
// read-add-write).  Phases with no taps are zero-filled (beta 0) or left
// untouched (beta 1).  Replaces the dcols GEMM + col2im.
bool conv_dgrad_phases(const void* dy, const void* w, void* dx, const ConvGeom& g, float beta, cudaStream_t s) {
  static const int on = [] { const char* e = getenv("BE_DGRAD_PHASE"); return e ? atoi(e) : 1; }();
  const int st = g.stride;
  if (!on || st < 2 || st > 4 || g.K % 64 != 0 || g.C % 16 != 0 || (beta != 0.f && beta != 1.f)) return false;
  if ((reinterpret_cast<uintptr_t>(dy) & 15) || (reinterpret_cast<uintptr_t>(w) & 15) ||
      (reinterpret_cast<uintptr_t>(dx) & 15))
    return false;
  int cr[4], dr[4], cs[4], ds[4];
  for (int rho = 0; rho < st; ++rho) {
    phase_taps(g.R, st, g.pad, rho, &cr[rho], &dr[rho]);
    phase_taps(g.S, st, g.pad, rho, &cs[rho], &ds[rho]);
  }
  // every phase map must be encodable before anything is launched
  GemmParams ps[16];
  int nph = 0;
  bool zero_needed = false;
  const int bn = g.C >= 256 ? 256 : (g.C >= 128 ? 128 : 64);
  for (int rh = 0; rh < st; ++rh)
    for (int rw = 0; rw < st; ++rw) {
      const int Hp = (g.H - rh + st - 1) / st, Wp = (g.W - rw + st - 1) / st;
      if (Hp <= 0 || Wp <= 0) continue;
      if (cr[rh] == 0 || cs[rw] == 0) { zero_needed = true; continue; }
      GemmParams& p = ps[nph];
      memset(&p, 0, sizeof(p));
      ConvGeom t;  // the phase convolution over dY
      t.N = g.N; t.H = g.P; t.W = g.Q; t.C = g.K; t.K = g.C; t.R = cr[rh]; t.S = cs[rw];
      t.stride = 1; t.pad = -dr[rh]; t.P = Hp; t.Q = Wp;
      const int lw = dr[rw], lh = dr[rh];
      // TMA-store epilogue when the phase rows have a uniform pitch (H % st == 0):
      // each output row is padded to Qp base positions (a power of two ≤ 32, else a
      // multiple of 32; the extra positions read only padding → zero rows, clipped
      // by the store map) so every 32-row epilogue chunk is whole rows / one row piece
      const bool tma_ph = g.H % st == 0 && Hp * st == g.H;
      int Qp = Wp;
      if (tma_ph) { if (Wp <= 32) { Qp = 1; while (Qp < Wp) Qp *= 2; } else Qp = (Wp + 31) / 32 * 32; }
      t.Q = Qp;
      // window starts lower = dmin; base positions per row = Q_in + upper − lower = Qp
      const int corners[4] = {lw, lh, Qp - g.Q + lw, Hp - g.P + lh};
      if (!encode_im2col_4d(&p.ta[1], dy, t, 64, BM, corners)) return false;
      if (tma_ph) {
        // dx phase view [u = n·H/st + i][j][c]: strides st·W·C, st·C, 1; box {32 c, bj, 32/bj}
        const int bj = Qp < 32 ? Qp : 32;
        cuuint64_t od[3] = {(cuuint64_t)g.C, (cuuint64_t)Wp, (cuuint64_t)g.N * Hp};
        cuuint64_t os[2] = {(cuuint64_t)st * g.C * 2, (cuuint64_t)st * g.W * g.C * 2};
        cuuint32_t ob[3] = {32, (cuuint32_t)bj, (cuuint32_t)(32 / bj)};
        cuuint32_t oe[3] = {1, 1, 1};
        EncodeFn enc = get_encode();
        void* base = reinterpret_cast<uint16_t*>(dx) + ((int64_t)rh * g.W + rw) * g.C;
        if (!enc || enc(&p.td, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, od, os, ob, oe, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return false;
        p.tma_store = beta == 1.f ? 2 : 1;
      }
      encode_2d(&p.ta[0], dy, BE_BF16, (uint64_t)g.K, (uint64_t)g.N * g.P * g.Q, (uint64_t)g.K, 64, 1);
      const int RSC = t.R * t.S * t.C;
      // the phase's taps of W read in place: t_r ↔ r = ρh + pad − st·(dminh + t_r)
      const int bw[6] = {rh + g.pad - st * dr[rh], -st, rw + g.pad - st * ds[rw], -st, g.S, g.R * g.S * g.C};
      set_bw(p, w, t, bw);
      p.use_im2col = 1;
      p.M = t.N * t.P * t.Q; p.N = t.K; p.K = RSC;
      p.a_kmajor = 1; p.b_kmajor = 1; p.splits = 1;
      p.D = dx; p.ldd = g.C; p.d_f32 = 0; p.beta = beta;
      p.x = reinterpret_cast<const uint16_t*>(dy);
      p.cN = t.N; p.cH = t.H; p.cW = t.W; p.cC = t.C; p.cR = t.R; p.cS = t.S;
      p.cstride = 1; p.cpad = -lh; p.cpad_w_off = lh - lw; p.cP = t.P; p.cQ = t.Q;
      p.ph_st = st; p.ph_h = rh; p.ph_w = rw; p.ph_H = g.H; p.ph_W = g.W;
      ++nph;
    }
  if (zero_needed && beta == 0.f) conv_phase_zero(dx, g, cr, cs, s);
  for (int i = 0; i < nph; ++i) {  // one profiler record per launch (tools/ncu_class.py pairs them with ncu's list)
    const GemmParams& p = ps[i];
    const double flops = 2.0 * p.M * (double)p.N * p.K;
    const double bytes = ((double)g.N * g.P * g.Q * g.K + (double)p.N * p.K + (double)p.M * p.N * (beta != 0.f ? 2 : 1)) * 2.0;
    const int pidx = prof_begin("conv_tc_dgrad_phase", flops, bytes, p.M, p.N, p.K, s);
    if (bn == 256) launch_conv<256>(ps[i], s, nullptr);
    else if (bn == 128) launch_conv<128>(ps[i], s, nullptr);
    else launch_conv<64>(ps[i], s, nullptr);
    prof_end(pidx, s);
    g_tc_calls++;
  }
  after_launch("conv_tc_dgrad_phase");
  return true;
}

uint64_t gemm_tcgen05_calls() { return g_tc_calls.load(); }
uint64_t gemm_simt_calls() { return g_simt_calls.load(); }

bool gemm_tc_ok(const GemmDesc& g) {
  return g.K > 0 && g.M > 0 && g.N > 0 && (g.ab == BE_BF16 || g.ab == BE_F32) && tma_ok(g.A, g.lda, g.ab) &&
         tma_ok(g.B, g.ldb, g.ab) && g.conv_x == nullptr;
}

const char* gemm(const GemmDesc& g, cudaStream_t s) {
  BE_REQUIRE(g.ab == BE_BF16 || g.ab == BE_F32, BE_E_DTYPE, "gemm: operands must be bf16 or f32");
  BE_REQUIRE(g.d == BE_BF16 || g.d == BE_F32, BE_E_DTYPE, "gemm: output must be bf16 or f32");
  if (g.M == 0 || g.N == 0) return "empty";
  if (g.K == 0) {  // D = beta*D + bias (+act): handled by SIMT kernel with K=0 loop
  }
  const bool x3 = g.ab == BE_F32;
  const bool tc = g.K > 0 && tma_ok(g.A, g.lda, g.ab) && tma_ok(g.B, g.ldb, g.ab);
  BE_REQUIRE(!g.upd || (tc && !g.conv_x), BE_E_ARG, "gemm: the SGD update epilogue needs the tcgen05 path");
  if (tc) {
    g_tc_calls++;
    const void *ahi = g.A, *alo = nullptr, *bhi = g.B, *blo = nullptr;
    Block* tmp = nullptr;
    GemmDesc gx = g;
    if (x3) {
      // Split both operands into tf32 hi = rna(x), lo = rna(x − hi).  The
      // split pass also writes every operand K-major (transposing MN-major
      // ones): kind::tf32 with MN-major operands needs the 128B_BASE32B
      // swizzle atom, which this kernel does not implement.
      const int64_t lda2 = (g.K + 3) / 4 * 4, ldb2 = lda2;
      const int64_t na = (int64_t)g.M * lda2, nb = (int64_t)g.N * ldb2;
      size_t bytes = (size_t)(2 * na + 2 * nb) * 4 + 64;
      tmp = ctx().alloc.allocate(bytes, s);
      float* base = reinterpret_cast<float*>(tmp->ptr);
      float *ah = base, *al = ah + na, *bh = al + na, *bl = bh + nb;
      split_tf32_kmajor(reinterpret_cast<const float*>(g.A), g.lda, g.a_kmajor, g.M, g.K, ah, al, lda2, s);
      split_tf32_kmajor(reinterpret_cast<const float*>(g.B), g.ldb, g.b_kmajor, g.N, g.K, bh, bl, ldb2, s);
      ahi = ah; alo = al; bhi = bh; blo = bl;
      gx.lda = lda2; gx.ldb = ldb2; gx.a_kmajor = true; gx.b_kmajor = true;
    }
    const int bn = pick_bn(g.M, g.N, ctx().num_sms, x3);
    if (g.xf_op) {
      // BN-apply fused into the operand load: the 1-CTA kernel with its
      // transform warps (tile and split rule as the default candidate)
      BE_REQUIRE(!x3 && !g.upd && !g.conv_x && !g.stats && g.beta == 0.f &&
                     ((g.xf_op == 1 && g.a_kmajor) || (g.xf_op == 2 && !g.b_kmajor)),
                 BE_E_ARG, "gemm: operand transform needs bf16, K-major A (op 1) or MN-major B (op 2)");
      if (bn == 256) launch_tc<256, false, 2, true>(g, ahi, alo, bhi, blo, s);
      else if (bn == 128) launch_tc<128, false, 2, true>(g, ahi, alo, bhi, blo, s);
      else launch_tc<64, false, 2, true>(g, ahi, alo, bhi, blo, s);
      if (tmp) ctx().alloc.free(tmp);
      return "tcgen05";
    }
    if (x3) {
      if (bn == 128) launch_tc<128, true>(gx, ahi, alo, bhi, blo, s);
      else launch_tc<64, true>(gx, ahi, alo, bhi, blo, s);
    } else if (g.conv_x) {
      BE_REQUIRE(!g.b_kmajor && g.conv_g.C % 64 == 0, BE_E_ARG, "im2col B needs MN-major B and C % 64 == 0");
      if (bn == 256) launch_tc<256, false>(g, ahi, alo, bhi, blo, s);
      else if (bn == 128) launch_tc<128, false>(g, ahi, alo, bhi, blo, s);
      else launch_tc<64, false>(g, ahi, alo, bhi, blo, s);
    } else if (g.upd) {
      // fused SGD epilogue: 1-CTA kernel BN 256 / 128 / 64 or the CTA pair (autotuned)
      cudaEvent_t ev0 = nullptr, ev1 = nullptr;
      const int v = tune_choose("gemm:" + tune_key(g) + "u", 4, 0, &ev0, &ev1);
      if (ev0) cudaEventRecord(ev0, s);
      if (v == 3 && pair_plausible(g)) launch_tc2(g, s);
      else if (v == 0 || v == 3) launch_tc<256, false>(g, ahi, alo, bhi, blo, s);
      else if (v == 1) launch_tc<128, false>(g, ahi, alo, bhi, blo, s);
      else launch_tc<64, false>(g, ahi, alo, bhi, blo, s);
      if (ev1) cudaEventRecord(ev1, s);
    } else {
      // candidate list (autotuned per shape): the 1-CTA kernel
      // with pick_bn's tile and its default split rule; the CTA pair; and,
      // when the tile grid under-fills the 148 SMs, BN=256 / BN=128 with
      // split-K sized to fill the machine.
      struct Cand { int kind, bn, splits; };
      Cand cands[6];
      int nc = 0;
      cands[nc++] = {0, bn, 0};
      const int pm = pair_mode();
      if (pm != 0 && pair_plausible(g)) cands[nc++] = {1, 256, 0};
      const int sms = ctx().num_sms;
      const int kbl = (g.K + 63) / 64;
      // store-heavy short-K shapes (1×1 convs): the same tile with 4 staging
      // slots per epilogue warp (3 TMA stores in flight) for fewer stages
      // BE_GEMM_EPI4=0 drops the candidate, =1 forces it where it applies (tests)
      static const int epi4 = [] { const char* e = getenv("BE_GEMM_EPI4"); return e ? atoi(e) : -1; }();
      const int tiles_bn = ((g.M + BM - 1) / BM) * ((g.N + bn - 1) / bn);
      if (epi4 != 0 && kbl <= 8 && tiles_bn >= sms) cands[nc++] = {2, bn, 0};
      // short K, narrow N (MobileNet's 1×1 convs): one tile covering all of N
      // reads A once — the wave-efficiency rule counts MMA work, which these
      // HBM-bound shapes do not spend (N = 144 → three BN = 64 tiles re-read A)
      const int bn_cover = g.N <= 64 ? 64 : (g.N <= 128 ? 128 : 256);
      if (kbl <= 8 && g.N <= 256 && bn_cover != bn) cands[nc++] = {0, bn_cover, 0};
      for (int cbn : {256, 128}) {
        if (g.stats) break;  // split-K cannot carry the statistics epilogue
        const int tiles = ((g.M + BM - 1) / BM) * ((g.N + cbn - 1) / cbn);
        if (tiles < sms && kbl >= 16 && g.N > cbn / 2) {
          const int sp = std::max(2, std::min(sms / tiles, kbl / 4));
          if (!(cbn == bn && sp == 1)) cands[nc++] = {0, cbn, sp};
        }
      }
      int v = 0;
      cudaEvent_t ev0 = nullptr, ev1 = nullptr;
      int deep = -1;
      for (int i = 0; i < nc; ++i)
        if (cands[i].kind == 2) deep = i;
      if (epi4 == 1 && deep >= 0) v = deep;  // tests: force the 4-slot epilogue where it applies
      else if (pm == 1 && pair_plausible(g)) v = 1;
      else if (nc > 1) v = tune_choose("gemm:" + tune_key(g) + (g.stats ? "s" : ""), nc, 0, &ev0, &ev1);
      const Cand c = cands[v];
      if (ev0) cudaEventRecord(ev0, s);
      if (c.kind == 1) launch_tc2(g, s);
      else if (c.kind == 2 && c.bn == 256) launch_tc<256, false, 4>(g, ahi, alo, bhi, blo, s);
      else if (c.kind == 2 && c.bn == 128) launch_tc<128, false, 4>(g, ahi, alo, bhi, blo, s);
      else if (c.kind == 2) launch_tc<64, false, 4>(g, ahi, alo, bhi, blo, s);
      else if (c.bn == 256) launch_tc<256, false>(g, ahi, alo, bhi, blo, s, c.splits);
      else if (c.bn == 128) launch_tc<128, false>(g, ahi, alo, bhi, blo, s, c.splits);
      else launch_tc<64, false>(g, ahi, alo, bhi, blo, s, c.splits);
      if (ev1) cudaEventRecord(ev1, s);
    }
    if (tmp) ctx().alloc.free(tmp);  // stream-ordered reuse is safe
    return "tcgen05";
  }
  if (g.K > 0 && g.N > 1 && g.K > 1 && !g.conv_x && !g.upd) {
    // TMA-indescribable operand rows (not 16-B multiples, e.g. a 10-class
    // head): pad them into temporaries and stay on the tcgen05 path
    const int es = x3 ? 4 : 2, q = 16 / es;
    GemmDesc gp = g;
    Block* tmpa = nullptr;
    Block* tmpb = nullptr;
    auto pad = [&](const void* src, int64_t ld, bool kmajor, int MN, Block** blk, int64_t* ldo) -> const void* {
      const int64_t rows = kmajor ? MN : g.K, cols = kmajor ? g.K : MN;
      const int64_t ldp = (cols + q - 1) / q * q;
      *blk = ctx().alloc.allocate((size_t)(rows * ldp) * es, s);
      const int blocks = (int)std::min<long long>((rows * ldp + 255) / 256, (long long)ctx().num_sms * 16);
      if (x3)
        launch_pdl(pad_rows_kernel<float>, blocks, 256, 0, s, (const float*)src, (long long)ld, (float*)(*blk)->ptr,
                   (long long)ldp, (long long)rows, (long long)cols);
      else
        launch_pdl(pad_rows_kernel<uint16_t>, blocks, 256, 0, s, (const uint16_t*)src, (long long)ld,
                   (uint16_t*)(*blk)->ptr, (long long)ldp, (long long)rows, (long long)cols);
      after_launch("gemm_pad_operand");
      *ldo = ldp;
      return (*blk)->ptr;
    };
    if (!tma_ok(g.A, g.lda, g.ab)) gp.A = pad(g.A, g.lda, g.a_kmajor, g.M, &tmpa, &gp.lda);
    if (!tma_ok(g.B, g.ldb, g.ab)) gp.B = pad(g.B, g.ldb, g.b_kmajor, g.N, &tmpb, &gp.ldb);
    const char* r = gemm(gp, s);
    if (tmpa) ctx().alloc.free(tmpa);  // stream-ordered reuse is safe
    if (tmpb) ctx().alloc.free(tmpb);
    return r;
  }
  if (g.N == 1 || g.K == 1) {
    g_simt_calls++;
    const double es = g.ab == BE_F32 ? 4.0 : 2.0, ds = g.d == BE_F32 ? 4.0 : 2.0;
    const int pidx = prof_begin("gemm_skinny", 2.0 * g.M * g.N * g.K,
                                ((double)g.M * g.K + (double)g.N * g.K) * es + (double)g.M * g.N * ds, g.M, g.N, g.K, s);
    const bool bf = g.ab == BE_BF16;
    if (g.K == 1) {
      // A(m, 0) at m·(a_kmajor ? lda : 1); B(0, n) at n·(b_kmajor ? ldb : 1)
      const long long as = g.a_kmajor ? g.lda : 1, bs = g.b_kmajor ? g.ldb : 1;
      const long long total = (long long)g.M * g.N;
      const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)ctx().num_sms * 16);
      if (bf) launch_pdl(outer_kernel<uint16_t>, blocks, 256, 0, s, g.M, g.N, (const uint16_t*)g.A, as, (const uint16_t*)g.B, bs,
                         g.D, (long long)g.ldd, (int)(g.d == BE_F32), g.beta, g.bias, g.act);
      else launch_pdl(outer_kernel<float>, blocks, 256, 0, s, g.M, g.N, (const float*)g.A, as, (const float*)g.B, bs, g.D,
                      (long long)g.ldd, (int)(g.d == BE_F32), g.beta, g.bias, g.act);
      after_launch("gemm_outer");
    } else if (g.a_kmajor) {
      const long long bs = g.b_kmajor ? 1 : g.ldb;  // B(k, 0)
      const int blocks = (g.M + 7) / 8;
      if (bf) launch_pdl(gemv_kmajor_kernel<uint16_t>, blocks, 256, 0, s, g.M, g.K, (const uint16_t*)g.A, (long long)g.lda,
                         (const uint16_t*)g.B, bs, g.D, (long long)g.ldd, (int)(g.d == BE_F32), g.beta, g.bias, g.act);
      else launch_pdl(gemv_kmajor_kernel<float>, blocks, 256, 0, s, g.M, g.K, (const float*)g.A, (long long)g.lda,
                      (const float*)g.B, bs, g.D, (long long)g.ldd, (int)(g.d == BE_F32), g.beta, g.bias, g.act);
      after_launch("gemm_gemv");
    } else {
      const long long bs = g.b_kmajor ? 1 : g.ldb;
      const int mb = (g.M + 31) / 32;
      int splits = std::max(1, std::min<int>(ctx().num_sms * 2 / mb, g.K / 256));
      const int kchunk = (g.K + splits - 1) / splits;
      splits = (g.K + kchunk - 1) / kchunk;
      Block* ws = ctx().alloc.allocate(sizeof(float) * (size_t)splits * g.M, s);
      float* wsp = reinterpret_cast<float*>(ws->ptr);
      dim3 grid(mb, splits);
      if (bf) launch_pdl(gemv_mnmajor_kernel<uint16_t>, grid, 256, 0, s, g.M, g.K, (const uint16_t*)g.A, (long long)g.lda,
                         (const uint16_t*)g.B, bs, kchunk, wsp);
      else launch_pdl(gemv_mnmajor_kernel<float>, grid, 256, 0, s, g.M, g.K, (const float*)g.A, (long long)g.lda,
                      (const float*)g.B, bs, kchunk, wsp);
      after_launch("gemm_gemv_mn");
      launch_splitk((const float*)wsp, splits, (long long)g.M, g.M, 1, g.D, (long long)g.ldd,
                 (int)(g.d == BE_F32), g.beta, g.bias, g.act, s);
      after_launch("gemm_gemv_reduce");
      ctx().alloc.free(ws);
    }
    prof_end(pidx, s);
    return "skinny";
  }
  g_simt_calls++;
  const int tiles = ((g.N + 63) / 64) * ((g.M + 63) / 64);
  // split-K so small-output / long-K shapes (e.g. a [128 x 1] head's wgrad, K = batch) fill the GPU
  int splits = 1;
  if (tiles < ctx().num_sms && g.K >= 1024)
    splits = std::max(1, std::min<int>(std::min(ctx().num_sms * 2 / tiles, g.K / 256), 256));
  const int kchunk = ((g.K + splits - 1) / splits + 15) / 16 * 16;
  splits = std::max(1, (g.K + kchunk - 1) / kchunk);
  Block* ws = splits > 1 ? ctx().alloc.allocate(sizeof(float) * (size_t)splits * g.M * g.N, s) : nullptr;
  float* wsp = ws ? reinterpret_cast<float*>(ws->ptr) : nullptr;
  dim3 grid((g.N + 63) / 64, (g.M + 63) / 64, splits);
  const double es = g.ab == BE_F32 ? 4.0 : 2.0, ds = g.d == BE_F32 ? 4.0 : 2.0;
  const int pidx = prof_begin("gemm_simt", 2.0 * g.M * g.N * g.K,
                              ((double)g.M * g.K + (double)g.N * g.K) * es + (double)g.M * g.N * ds, g.M, g.N, g.K, s);
  if (g.ab == BE_BF16)
    gemm_simt_kernel<uint16_t><<<grid, 256, 0, s>>>(g.M, g.N, g.K, (const uint16_t*)g.A, g.lda, g.a_kmajor,
                                                    (const uint16_t*)g.B, g.ldb, g.b_kmajor, g.D, g.ldd,
                                                    g.d == BE_F32, g.beta, g.bias, g.act, kchunk, wsp);
  else
    gemm_simt_kernel<float><<<grid, 256, 0, s>>>(g.M, g.N, g.K, (const float*)g.A, g.lda, g.a_kmajor,
                                                 (const float*)g.B, g.ldb, g.b_kmajor, g.D, g.ldd, g.d == BE_F32,
                                                 g.beta, g.bias, g.act, kchunk, wsp);
  after_launch("gemm_simt");
  if (ws) {
    const long long total = (long long)g.M * g.N;
    launch_splitk(wsp, splits, total, g.M, g.N, g.D, g.ldd, g.d == BE_F32, g.beta, g.bias,
                                         g.act, s);
    after_launch("gemm_simt_splitk_reduce");
    ctx().alloc.free(ws);
  }
  prof_end(pidx, s);
  return "simt";
}

}}  // namespace be::k
