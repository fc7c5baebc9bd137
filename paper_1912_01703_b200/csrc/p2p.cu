// p2p.cu — the gradient allreduce fused with the SGD update over peer memory
// (§5.4 "synchronize gradients using all-reduce
// style primitives"): ONE kernel per gradient bucket and rank that
//   1. arrives on a cross-GPU barrier (a flag written into every peer's memory),
//   2. reduces ITS 1/R slice of the bucket by loading that slice from every
//      rank's bucket over NVLink (fixed rank order),
//   3. applies ×1/R and the SGD update (sgd_math.cuh, bitwise the update of
//      be_sgd_step) to the slice of the fp32 master and its momentum, and
//   4. stores the new fp32 master and its bf16 shadow into EVERY rank's copy,
// then signals completion and waits for every peer's — a reduce-scatter →
// SGD → all-gather of parameters in one pass.  Per GPU and bucket of S
// floats: reads (R−1)/R·S·4 B from peers, writes (R−1)/R·S·6 B to peers, as
// an NVLS allreduce, with the separate SGD pass and the collective launch
// gone; the replicas are bitwise identical by construction (one owner
// computes every element).  Without an optimizer the same kernel is a plain
// allreduce (the owner writes the mean gradient back into every bucket).
//
// The barrier spins on acquire loads of system-scope flags with a 10 s
// timeout (status word set, no hang).
#include "common.cuh"
#include "kernels.h"
#include "runtime.h"
#include "sgd_math.cuh"

namespace be {
namespace dev {
namespace {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// wait until flags[q] >= epoch for every rank q (10 s timeout → status)
__device__ bool wait_all(const unsigned long long* flags, int R, unsigned long long epoch, int* status) {
  const unsigned long long t0 = globaltimer();
  for (int q = 0; q < R; ++q) {
    while (ld_acquire_sys(flags + q) < epoch) {
      if (globaltimer() - t0 > 10000000000ull) {
        atomicExch(status, 1);
        return false;
      }
      __nanosleep(200);
    }
  }
  return true;
}

__global__ void __launch_bounds__(512) p2p_allreduce_sgd_kernel(const __grid_constant__ k::P2PBucketArgs a) {
  pdl_entry();
  const int R = a.world, me = a.rank;
  // 1. arrive: this rank's gradients for the bucket are complete (stream
  //    order) and, after the system fence, visible to the peers
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < R; ++q) st_release_sys(a.flags_peer[q] + me, a.epoch);
  }
  if (threadIdx.x == 0) wait_all(a.flags_arrive, R, a.epoch, a.status);
  __syncthreads();
  if (*reinterpret_cast<volatile int*>(a.status) != 0) return;
  // 2-4. my slice [lo, hi) of the bucket, 4 elements per thread step
  const int64_t per = (a.numel + R - 1) / R;
  const int64_t lo = min(a.numel, (int64_t)me * ((per + 63) / 64 * 64));
  const int64_t hi = min(a.numel, lo + (per + 63) / 64 * 64);
  const float inv_r = 1.f / (float)R;
  const bool mom = a.mu != 0.f;
  for (int64_t e0 = lo + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; e0 < hi;
       e0 += (int64_t)gridDim.x * blockDim.x * 4) {
    // segment of e0 (last seg_off <= e0)
    int s0 = 0, s1 = a.nseg - 1;
    while (s0 < s1) {
      const int mid = (s0 + s1 + 1) >> 1;
      if (a.seg_off[mid] <= e0) s0 = mid; else s1 = mid - 1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t e = e0 + j;
      if (e >= hi) break;
      int s = s0;
      while (s + 1 < a.nseg && a.seg_off[s + 1] <= e) ++s;
      const int64_t loc = e - a.seg_off[s];
      if (loc >= a.seg_n[s]) continue;  // alignment gap between parameters
      float g = 0.f;
      for (int q = 0; q < R; ++q) g += a.grad[q][e];  // fixed rank order
      if (a.lr_on) {
        float p = a.p[(int64_t)s * R + me][loc];
        float v = mom ? a.mom[s][loc] : 0.f;
        sgd_elem(p, g, v, mom, a.lr, a.mu, a.wd, inv_r);
        if (mom) a.mom[s][loc] = v;
        const uint16_t sh = f2bf(p);
        for (int q = 0; q < R; ++q) {
          a.p[(int64_t)s * R + q][loc] = p;
          if (a.shadow) {
            uint16_t* d = a.shadow[(int64_t)s * R + q];
            if (d) d[loc] = sh;
          }
        }
      } else {
        const float m = __fmul_rn(g, inv_r);
        for (int q = 0; q < R; ++q) a.grad[q][e] = m;
      }
    }
  }
  // 5. done: every block's peer stores are fenced before it counts itself;
  //    the last block signals every peer, then waits for all of them
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int old = atomicAdd(a.counter, 1u);
    if (old == (unsigned int)(a.epoch * gridDim.x - 1)) {
      for (int q = 0; q < R; ++q) st_release_sys(a.flags_peer_done[q] + me, a.epoch);
      wait_all(a.flags_done, R, a.epoch, a.status);
    }
  }
}

}  // namespace
}  // namespace dev

namespace k {
void p2p_allreduce_sgd(const P2PBucketArgs& a, int blocks, cudaStream_t s) {
  dev::p2p_allreduce_sgd_kernel<<<blocks, 512, 0, s>>>(a);
  after_launch("p2p_allreduce_sgd");
}
}  // namespace k
}  // namespace be
