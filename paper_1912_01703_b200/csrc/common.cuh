// common.cuh — device helpers shared by the memory-bound kernels.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "../../include/be.h"

namespace be { namespace dev {

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may
// become resident while its stream predecessor is still finishing; it must
// execute pdl_entry() before touching global memory.  griddepcontrol.wait
// returns once the predecessor grid has completed and its writes are
// visible; launch_dependents then lets this kernel's own successor launch
// early.  (Hides the launch latency between the step's ~1.2 k dependent
// kernels.)  BE_PDL=0 launches everything conventionally.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ float bf2f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ uint16_t f2bf(float x) {
  __nv_bfloat16 h = __float2bfloat16_rn(x);  // round-to-nearest-even
  return *reinterpret_cast<uint16_t*>(&h);
}

// scalar load/store with run-time dtype (f32 / bf16)
__device__ __forceinline__ float ld(const void* p, int64_t i, be_dtype dt) {
  return dt == BE_BF16 ? bf2f(reinterpret_cast<const uint16_t*>(p)[i]) : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void st(void* p, int64_t i, be_dtype dt, float v) {
  if (dt == BE_BF16) reinterpret_cast<uint16_t*>(p)[i] = f2bf(v);
  else reinterpret_cast<float*>(p)[i] = v;
}

// 8-element vector I/O (16 B for bf16, 2x16 B for f32)
struct V8 { float v[8]; };
__device__ __forceinline__ V8 ld8(const void* p, int64_t i, be_dtype dt) {
  V8 r;
  if (dt == BE_BF16) {
    uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p) + i);
    const uint16_t* h = reinterpret_cast<const uint16_t*>(&u);
#pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = bf2f(h[j]);
  } else {
    const float4* q = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p) + i);
    float4 a = q[0], b = q[1];
    r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
    r.v[4] = b.x; r.v[5] = b.y; r.v[6] = b.z; r.v[7] = b.w;
  }
  return r;
}
__device__ __forceinline__ void st8(void* p, int64_t i, be_dtype dt, const V8& r) {
  if (dt == BE_BF16) {
    uint4 u;
    uint16_t* h = reinterpret_cast<uint16_t*>(&u);
#pragma unroll
    for (int j = 0; j < 8; ++j) h[j] = f2bf(r.v[j]);
    *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p) + i) = u;
  } else {
    float4* q = reinterpret_cast<float4*>(reinterpret_cast<float*>(p) + i);
    q[0] = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
    q[1] = make_float4(r.v[4], r.v[5], r.v[6], r.v[7]);
  }
}
__host__ __device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// activations fused after a BN / conv epilogue: act 1 = ReLU, 2 = ReLU6
// (MobileNetV2); act_pass is the backward mask (gradient 0 at the kinks)
__device__ __forceinline__ float act_apply(float v, int act) {
  return act == 2 ? fminf(fmaxf(v, 0.f), 6.f) : (act ? fmaxf(v, 0.f) : v);
}
__device__ __forceinline__ bool act_pass(float v, int act) { return act == 2 ? (v > 0.f && v < 6.f) : v > 0.f; }
// the mask decided from the value as STORED (the forward writes bf16(act(v))):
// for ReLU6 a pre-activation just below 6 that rounds to 6 has gradient 0, the
// same decision a reader of the stored output takes (SURVEY §8(c) reading 16);
// for ReLU rounding never changes the sign
__device__ __forceinline__ float bf16_round(float v) {
  return __bfloat162float(__float2bfloat16_rn(v));
}
__device__ __forceinline__ bool act_pass_st(float v, int act, bool bf16) {
  return act_pass(act == 2 && bf16 ? bf16_round(v) : v, act);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}}  // namespace be::dev

#include <cuda_runtime.h>
#include <cstdlib>
#include <utility>
namespace be { namespace dev {
inline bool pdl_enabled() {
  static const bool on = [] { const char* e = std::getenv("BE_PDL"); return !e || e[0] != '0'; }();
  return on;
}
// kernel<<<grid, block, smem, s>>>(args...) with the PDL attribute (the kernel
// must call pdl_entry() first)
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}}  // namespace be::dev

