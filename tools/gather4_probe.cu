// Probe the semantics of cp.async.bulk.tensor.2d.tile::gather4 on sm_100a:
// which boxDim the tensor map needs, the smem placement of the 4 rows (with
// SW128), and zero-fill for out-of-range row coordinates.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap m, int r0, int r1, int r2, int r3, uint16_t* out) {
  __shared__ __align__(1024) uint16_t buf[4 * 64 * 4];
  __shared__ __align__(8) uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t d = (uint32_t)__cvta_generic_to_shared(buf);
  for (int i = threadIdx.x; i < 4 * 64 * 4; i += blockDim.x) buf[i] = 0xFFFF;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4 * 128));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(d),
        "l"(reinterpret_cast<uint64_t>(&m)), "r"(b), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
    asm volatile(
        "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 64 * 4; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int rows = 100, cols = 64;
  std::vector<uint16_t> h(rows * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) h[r * cols + c] = (uint16_t)(r * 100 + c);
  uint16_t *dx, *dout;
  cudaMalloc(&dx, h.size() * 2);
  cudaMalloc(&dout, 4 * 64 * 4 * 2);
  cudaMemcpy(dx, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill))f;
  for (int boxr : {1, 4}) {
    for (int sw : {0, 1}) {
      CUtensorMap m;
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)boxr};
      cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("box rows %d swizzle %d: encode %d\n", boxr, sw, (int)r);
      if (r) continue;
      cudaMemset(dout, 0, 4 * 64 * 4 * 2);
      probe<<<1, 128>>>(m, 7, 3, -1, 150, dout);
      cudaError_t e = cudaDeviceSynchronize();
      printf("  launch: %s\n", cudaGetErrorString(e));
      if (e) { cudaGetLastError(); continue; }
      std::vector<uint16_t> o(4 * 64 * 4);
      cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
      for (int rr = 0; rr < 5; ++rr) {
        printf("  smem row %d:", rr);
        for (int c = 0; c < 12; ++c) printf(" %5d", (int)(int16_t)o[rr * 64 + c]);
        printf(" ... [8]=%d [56]=%d\n", (int)(int16_t)o[rr * 64 + 8], (int)(int16_t)o[rr * 64 + 56]);
      }
    }
  }
  return 0;
}
