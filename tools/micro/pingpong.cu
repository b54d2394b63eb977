// Micro-benchmark: mbarrier ping-pong round trip between two warps, same CTA vs the two
// CTAs of a cluster pair (remote arrive .relaxed.cluster / .release.cluster), and with the
// leader's return signal sent by tcgen05.commit (multicast) like the fused linear's A ring.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pingpong pingpong.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_par(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void arrive_local(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint64_t* b, uint32_t rank, int relaxed) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(sa(b)), "r"(rank));
  if (relaxed) asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
  else asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}

// mode 0: same CTA (warps 0 and 1 of CTA 0), local arrives
// mode 1: cross CTA, relaxed remote arrives both ways
// mode 2: cross CTA, release remote arrives
// mode 3: cross CTA, ping = remote relaxed arrive (peer -> leader), pong = tcgen05.commit multicast
__global__ void pingpong(int mode, int iters, unsigned long long* out) {
  __shared__ __align__(8) uint64_t bar_a, bar_b;
  __shared__ uint32_t tb;
  uint32_t rank = 0;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar_a)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar_b)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (mode == 3 && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(sa(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  // A = leader side (CTA 0 warp 1), B = other side (mode 0: CTA 0 warp 2; else CTA 1 warp 1)
  const bool isA = rank == 0 && warp == 1;
  const bool isB = mode == 0 ? (rank == 0 && warp == 2) : (rank == 1 && warp == 1);
  if ((isA || isB) && lane == 0) {
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t ph = i & 1;
      if (isB) {
        // ping: B -> A
        if (mode == 0) arrive_local(&bar_a);
        else arrive_remote(&bar_a, 0, mode != 2);
        wait_par(&bar_b, ph);  // pong from A
      } else {
        wait_par(&bar_a, ph);
        if (mode == 0) arrive_local(&bar_b);
        else if (mode == 3)
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(sa(&bar_b)), "h"((uint16_t)2));
        else arrive_remote(&bar_b, 1, mode != 2);
      }
    }
    long long c1 = clock64();
    if (isB) out[0] = c1 - c0;
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (mode == 3 && warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 32;" ::"r"(tb));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const char* names[] = {"same CTA, local arrives", "cross CTA, relaxed remote arrives",
                         "cross CTA, release remote arrives", "cross CTA, ping remote / pong tcgen05.commit multicast"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(96);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    const int iters = 10000;
    cudaError_t e = cudaLaunchKernelEx(&cfg, pingpong, mode, iters, d);
    if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-55s: %7.1f cycles per round trip\n", names[mode], (double)h / iters);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
