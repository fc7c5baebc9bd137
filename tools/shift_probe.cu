// Probe: can a tcgen05.mma K-major SWIZZLE_128B operand start at a row offset
// that is not a multiple of the 8-row (1024-B) swizzle atom?  (A 3×3 conv /
// wgrad reading a shifted window of one smem patch instead of one TMA load per
// tap.)  The patch is written in the TMA SW128 layout relative to a 1024-B
// aligned base (row r, 16-B chunk j at r·128 + (j ^ (r & 7))·16); the MMA's A
// descriptor starts at base + s·128 (+ kk·32 along K) with descriptor
// base_offset field = 0 or (s & 7).  D = A_s[128×64] · B[64×64]ᵀ is compared
// with the host product of rows s..s+127.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/shift_probe tools/shift_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t boff) {
  uint64_t d = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
               ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)(boff & 7) << 49) |
               ((uint64_t)2 << 61);
  return d;
}

__global__ void probe(const uint16_t* A, const uint16_t* B, int shift, int use_boff, float* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* pa = sm;                // 144 rows × 128 B
  uint8_t* pb = sm + 144 * 128;    // 64 rows × 128 B (1024-aligned: 144·128 = 18 KB)
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int i = t; i < 144 * 8; i += blockDim.x) {
    const int r = i / 8, j = i % 8;
    *(uint4*)(pa + r * 128 + ((j ^ (r & 7)) << 4)) = *(const uint4*)(A + r * 64 + j * 8);
  }
  for (int i = t; i < 64 * 8; i += blockDim.x) {
    const int r = i / 8, j = i % 8;
    *(uint4*)(pb + r * 128 + ((j ^ (r & 7)) << 4)) = *(const uint4*)(B + r * 64 + j * 8);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ad = desc(su32(pa) + shift * 128 + kk * 32, 16, 1024, use_boff ? (shift & 7) : 0);
      const uint64_t bd = desc(su32(pb) + kk * 32, 16, 1024, 0);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"(kk) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  }
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < 64; c0 += 32) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tm + c0 + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * 64 + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)((u + 0x7fff + ((u >> 16) & 1)) >> 16); }
static float bf2f(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
  std::vector<uint16_t> hA(144 * 64), hB(64 * 64);
  for (size_t i = 0; i < hA.size(); ++i) hA[i] = f2bf((float)((i * 37) % 17) / 8.f - 1.f);
  for (size_t i = 0; i < hB.size(); ++i) hB[i] = f2bf((float)((i * 11) % 13) / 6.f - 1.f);
  uint16_t *dA, *dB; float* dO;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dO, 128 * 64 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<float> o(128 * 64);
  for (int boff = 0; boff < 2; ++boff)
    for (int s = 0; s < 9; ++s) {
      probe<<<1, 128, 64 * 1024>>>(dA, dB, s, boff, dO);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("shift %d boff %d: CUDA error %s\n", s, boff, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double ref = 0;
          for (int k = 0; k < 64; ++k) ref += (double)bf2f(hA[(m + s) * 64 + k]) * bf2f(hB[n * 64 + k]);
          maxerr = fmax(maxerr, fabs(ref - o[m * 64 + n]));
        }
      printf("shift %d base_offset_field %s: max |err| %.3g %s\n", s, boff ? "=shift&7" : "=0", maxerr,
             maxerr < 1e-2 ? "OK" : "MISMATCH");
    }
  return 0;
}
