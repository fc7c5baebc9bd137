// nvls_probe.cu — does this box support NVLink SHARP multicast for one GPU?
// Creates a 1-device multicast object, binds a cuMemCreate allocation, runs
// multimem.ld_reduce / multimem.st / multimem.red through the multicast
// mapping and checks the unicast view.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
  printf("FAIL %s -> %d %s\n", #x, (int)r_, s); return 1; } } while (0)

__global__ void probe(float* mc, float* uc, unsigned long long* mcf, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i < n) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc + i) : "memory");
    v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(mc + i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  }
  if (i == 0) asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" :: "l"(mcf), "l"(5ull) : "memory");
}

int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  int mcs = 0; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("MULTICAST_SUPPORTED=%d\n", mcs);
  if (!mcs) return 0;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR; mp.size = 0;
  size_t gmin = 0, grec = 0;
  mp.size = 2u << 20;
  CK(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&grec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("granularity min %zu rec %zu\n", gmin, grec);
  const size_t sz = ((4u << 20) + gmin - 1) / gmin * gmin;
  mp.size = sz;
  CUmemGenericAllocationHandle mc;
  for (unsigned nd = 1; nd <= 2; ++nd)
    for (int ht = 0; ht < 3; ++ht) {
      CUmulticastObjectProp t = mp;
      t.numDevices = nd;
      t.handleTypes = ht == 0 ? 0 : ht == 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_FABRIC;
      CUresult r = cuMulticastCreate(&mc, &t);
      printf("create numDevices=%u handleTypes=%d -> %d\n", nd, ht, (int)r);
      if (r == CUDA_SUCCESS) cuMemRelease(mc);
    }
  mp.handleTypes = 0;
  CK(cuMulticastCreate(&mc, &mp));
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t ag = 0; CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  printf("alloc granularity %zu\n", ag);
  CUmemGenericAllocationHandle mem; CK(cuMemCreate(&mem, sz, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, mem, 0, sz, 0));
  CUdeviceptr uva, mva;
  CK(cuMemAddressReserve(&uva, sz, gmin, 0, 0)); CK(cuMemMap(uva, sz, 0, mem, 0));
  CK(cuMemAddressReserve(&mva, sz, gmin, 0, 0)); CK(cuMemMap(mva, sz, 0, mc, 0));
  CUmemAccessDesc acc = {}; acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uva, sz, &acc, 1)); CK(cuMemSetAccess(mva, sz, &acc, 1));
  const int n = 1 << 20;
  std::vector<float> h(n);
  for (int i = 0; i < n; ++i) h[i] = (float)(i % 1000) * 0.5f;
  cudaMemcpy((void*)uva, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemset((void*)(uva + n * 4), 0, 8);
  probe<<<n / 4 / 256, 256>>>((float*)mva, (float*)uva, (unsigned long long*)(mva + n * 4), n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> o(n);
  unsigned long long f = 0;
  cudaMemcpy(o.data(), (void*)uva, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&f, (void*)(uva + n * 4), 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += o[i] != h[i] + 1.f;
  printf("mismatches %d flag %llu (expect 5)\n", bad, f);
  // timing: ld_reduce + st over 256 MB
  printf("NVLS_PROBE %s\n", (bad == 0 && f == 5) ? "OK" : "BAD");
  return 0;
}
