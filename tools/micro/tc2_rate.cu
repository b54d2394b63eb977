// Micro-benchmark: tcgen05.mma.cta_group::2 (M = 256 over a CTA pair) issue rate with
// 1..3 issuing warps in the leader CTA, vs cta_group::1 (M = 128) per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc2_rate tc2_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)128 << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
template <int CG>
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (CG == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
template <int CG>
__device__ __forceinline__ void mma_ss_el(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (CG == 2)
    asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
template <int CG>
__device__ __forceinline__ void mma_ts_el(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (CG == 2)
    asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
template <int CG>
__device__ __forceinline__ void mma_ts_i8_el(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}
template <int CG>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (CG == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}

template <int CG>
__global__ void bench(int N, int R, int nis, int ts, unsigned long long* out, int cmode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t dummy;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tb)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tb)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(nis));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&dummy)), "r"(1 << 19));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3F803F80u;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tb;
  const int M = CG == 2 ? 256 : 128;
  if (ts >= 4 && rank == 0 && warp >= 1 && warp <= nis) {
    const uint32_t a = sa(sm) + (warp - 1) * 16384, b = sa(sm + 65536) + (warp - 1) * 16384;
    const uint32_t id = idesc(M, N);
    const uint64_t da = sdesc(a), db = sdesc(b);
    const uint32_t d = t + (warp - 1) * 64;
    const uint32_t at = t + 256 + (warp - 1) * 64;
    long long c0 = clock64();
    for (int i = 0; i < R; i += 8) {
      if (ts == 6) {  // int8 TS: 4 MMAs of K=32 per 128-wide k-step; idesc D s32, A/B s8
        const uint32_t idi = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
#pragma unroll
        for (int j = 0; j < 4; ++j) mma_ts_i8_el<CG>(d, at + 8 * j, db + 16 * j, idi, (i | j) ? 1u : 0u);
      } else if (ts == 4) {
#pragma unroll
        for (int j = 0; j < 8; ++j) mma_ts_el<CG>(d, at + 8 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) mma_ss_el<CG>(d, da + 16 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
      }
      if (CG == 2)
        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(sa(&dummy)), "h"((uint16_t)3));
      else
        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(sa(&dummy)));
    }
    if ((threadIdx.x & 31) == 0) {
      if (CG == 2)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(sa(&bar)), "h"((uint16_t)3));
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
      long long c1 = clock64();
      asm volatile("{\n.reg .pred P1;\nWE:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra WE;\n}\n" ::"r"(sa(&bar)));
      long long c2 = clock64();
      if (warp == 1 && blockIdx.x == 0) { out[0] = c1 - c0; out[1] = c2 - c0; }
    }
  } else if (rank == 0 && warp >= 1 && warp <= nis && (threadIdx.x & 31) == 0) {
    const uint32_t a = sa(sm) + (warp - 1) * 16384, b = sa(sm + 65536) + (warp - 1) * 16384;
    const uint32_t id = idesc(M, N);
    const uint64_t da = sdesc(a), db = sdesc(b);
    const uint32_t d = t + (warp - 1) * 64;        // accumulators: cols [0, 192)
    const uint32_t at = t + 256 + (warp - 1) * 64; // TMEM A operands: cols [256, 448)
    long long c0 = clock64();
    for (int i = 0; i < R; i += 8) {
      if (ts == 3 && warp == 1) {  // mixed: warp 1 SS (base-like), others TS (delta-like)
#pragma unroll
        for (int j = 0; j < 8; ++j) mma_ss<CG>(d, da + 16 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
      } else if (ts) {
#pragma unroll
        for (int j = 0; j < 8; ++j) mma_ts<CG>(d, at + 8 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
      } else if (ts == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) mma_ss<CG>(d, da + 16 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
      }
      for (int c = 0; c < cmode; ++c) {  // commits per 8 MMAs
        if (CG == 2)
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(sa(&dummy)), "h"((uint16_t)3));
        else
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&dummy)));
      }
    }
    if (CG == 2)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(sa(&bar)), "h"((uint16_t)3));
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
    long long c1 = clock64();
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(sa(&bar)));
    long long c2 = clock64();
    if (warp == 1 && blockIdx.x == 0) { out[0] = c1 - c0; out[1] = c2 - c0; }
  }
  if (CG == 2 && rank == 1 && threadIdx.x == 0) {
    // the peer's barrier also receives nis multicast arrivals
    asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W2;\n}\n" ::"r"(sa(&bar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 32);
  const int R = 4096;
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  for (int ts : {4, 5})
    for (int cg = 2; cg <= 2; ++cg)
      for (int nis = 1; nis <= 1; ++nis)
        for (int N : {16, 64, 128, 256}) {
          const int cmode = 1;
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(cg == 2 ? 2 : 1);
          cfg.blockDim = dim3(128);
          cfg.dynamicSmemBytes = 131072;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cg; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
          cfg.attrs = at; cfg.numAttrs = 1;
          cudaError_t e = cg == 2 ? cudaLaunchKernelEx(&cfg, bench<2>, N, R, nis, ts, d, cmode)
                                  : cudaLaunchKernelEx(&cfg, bench<1>, N, R, nis, ts, d, cmode);
          if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
          unsigned long long h[2];
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
          printf("%s cta_group::%d issuers %d N=%2d (+1 commit/8): %7.1f cyc per 8-MMA group per issuer -> aggregate %5.1f cyc/MMA\n",
                 ts == 3 ? "mixed(SS w1,TS rest)" : ts == 4 ? "TS-warp" : ts == 6 ? "TS-i8-warp(4 MMA/kstep)" : ts == 5 ? "SS-warp" : (ts ? "TS" : "SS"), cg, nis, N, (double)h[1] / (R / 8), (double)h[1] / R / nis);
        }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
