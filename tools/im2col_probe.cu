// Probe cp.async.bulk.tensor.4d.im2col semantics on sm_100a: which input
// pixel lands in smem row i for a given start coordinate / filter offset.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

constexpr int PIX = 32, CH = 64;
__global__ void probe(const __grid_constant__ CUtensorMap m, int c0, int w0, int h0, int n0, int offw, int offh,
                      uint16_t* out) {
  __shared__ __align__(1024) uint16_t buf[PIX * CH];
  __shared__ __align__(8) uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t d = (uint32_t)__cvta_generic_to_shared(buf);
  for (int i = threadIdx.x; i < PIX * CH; i += blockDim.x) buf[i] = 0xFFFF;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(PIX * CH * 2));
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(d),
        "l"(reinterpret_cast<uint64_t>(&m)), "r"(b), "r"(c0), "r"(w0), "r"(h0), "r"(n0), "h"((uint16_t)offw),
        "h"((uint16_t)offh)
        : "memory");
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < PIX * CH; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int N = 2, H = 5, W = 6, C = 64;
  std::vector<uint16_t> h((size_t)N * H * W * C);
  for (int n = 0; n < N; ++n)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        for (int c = 0; c < C; ++c) h[(((size_t)n * H + y) * W + x) * C + c] = (uint16_t)(n * 1000 + y * 100 + x * 10 + (c % 10));
  uint16_t *dx, *dout;
  cudaMalloc(&dx, h.size() * 2);
  cudaMalloc(&dout, PIX * CH * 2);
  cudaMemcpy(dx, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q);
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill))f;
  for (int stride : {1, 2}) {
    const int R = 3, pad = 1;
    const int Q = (W + 2 * pad - R) / stride + 1, P = (H + 2 * pad - R) / stride + 1;
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    int lower[2] = {-pad, -pad}, upper[2] = {pad - (R - 1), pad - (R - 1)};
    cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, dx, dims, strides, lower, upper, CH, PIX, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("stride %d (P=%d Q=%d): encode %d\n", stride, P, Q, (int)r);
    if (r) continue;
    // tile starting at output pixel m0 = 4 : (n,p,q) = (0, 4/Q, 4%Q)
    const int m0 = 4, q0 = m0 % Q, p0 = (m0 / Q) % P, n0 = m0 / (Q * P);
    for (int tap = 0; tap < 2; ++tap) {
      const int offw = tap == 0 ? 0 : 2, offh = tap == 0 ? 0 : 1;
      probe<<<1, 128>>>(m, 0, q0 * stride - pad, p0 * stride - pad, n0, offw, offh, dout);
      cudaError_t e = cudaDeviceSynchronize();
      printf("  tap (offw=%d, offh=%d): %s\n   rows:", offw, offh, cudaGetErrorString(e));
      if (e) { cudaGetLastError(); continue; }
      std::vector<uint16_t> o(PIX * CH);
      cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
      for (int i = 0; i < 24; ++i) {
        // row i, swizzled 128B: chunk 0 of row i sits at chunk (0 ^ (i&7))
        int v = (int16_t)o[i * 64 + ((0 ^ (i & 7)) * 8)];
        printf(" %d", v);
      }
      printf("\n");
    }
  }
  return 0;
}
