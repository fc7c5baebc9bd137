// sgd_math.cuh — the per-element SGD update,
// shared by the multi-tensor SGD kernel (pointwise.cu) and the fused
// weight-gradient + update GEMM epilogue (gemm_sm100.cu) so both produce
// bitwise the same parameters.  Explicit _rn intrinsics: no FMA contraction,
// so the result cannot depend on which kernel the compiler inlined it into.
//   g' = scale·g + wd·p;   v ← μ·v + g' (momentum);   p ← p − lr·(momentum ? v : g')
#pragma once

__device__ __forceinline__ void sgd_elem(float& p, float g, float& v, bool momentum, float lr, float mu, float wd,
                                         float scale) {
  float gg = __fadd_rn(__fmul_rn(g, scale), __fmul_rn(wd, p));
  if (momentum) {
    v = __fadd_rn(__fmul_rn(mu, v), gg);
    gg = v;
  }
  p = __fsub_rn(p, __fmul_rn(lr, gg));
}
