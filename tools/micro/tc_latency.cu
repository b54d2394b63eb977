// Microbenchmark: tcgen05.mma issue rate on B200 (sm_100a).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ int g_swz;
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  if (g_swz)  // SWIZZLE_128B K-major: SBO = 1024 B (8 rows x 128 B), LBO ignored
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | (1ull << 46) | (2ull << 61);
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)128 << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc));
}

__global__ void bench(int M, int N, int R, unsigned long long* out, int ts, int nis) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(nis));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3F803F80u;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tb;
  if (warp >= 1 && warp <= nis) {
    const uint32_t a = smem_u32(sm) + (warp - 1) * 16384, b = smem_u32(sm + 65536) + (warp - 1) * 16384;
    const uint32_t id = idesc(M, N);
    const uint64_t da = sdesc(a), db = sdesc(b);
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
    long long c0 = clock64();
    const uint32_t t0 = t;
    if ((threadIdx.x & 31) == 0) {
      const uint32_t t = t0 + (warp - 1) * (N <= 128 ? 128 : 256);
      for (int i = 0; i < R; i += 8) {
        if (ts == 1) {
#pragma unroll
          for (int j = 0; j < 8; ++j) mma_ts(t, t + 256 + 8 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
        } else if (ts == 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j) mma_ss(t, da + (g_swz ? 2 * (j & 3) + 64 * (j >> 2) : 16 * j), db + (g_swz ? 2 * (j & 3) + 64 * (j >> 2) : 16 * j), id, (i | j) ? 1u : 0u);
        } else if (ts == 2) {  // alternate accumulators every 8 (SS)
          const uint32_t dd = t + ((i >> 3) & 1) * 64;
#pragma unroll
          for (int j = 0; j < 8; ++j) mma_ss(dd, da + 16 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
        } else if (ts == 3) {  // alternate SS / TS every 8, separate accumulators
          if ((i >> 3) & 1) {
#pragma unroll
            for (int j = 0; j < 8; ++j) mma_ts(t + 64, t + 256 + 8 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) mma_ss(t, da + 16 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
          }
        } else {  // ts == 4: alternate accumulators every MMA (SS)
#pragma unroll
          for (int j = 0; j < 8; ++j) mma_ss(t + (j & 1) * 64, da + 16 * j, db + 16 * j, id, (i | j) ? 1u : 0u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }

    __syncwarp();
    long long c1 = clock64();
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)));
    long long c2 = clock64();
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
    if (threadIdx.x == 32) { out[0] = c1 - c0; out[1] = c2 - c0; out[2] = g1 - g0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int R = 4096;
  int zero = 0;
  cudaMemcpyToSymbol(g_swz, &zero, sizeof(int));
  const char* nm[] = {"SS", "TS"};
  for (int ts = 0; ts < 2; ++ts)
    for (int nis : {1, 2})
      for (int M : {64, 128})
        for (int N : {16, 32, 64, 128, 256}) {
          if (nis == 2 && N > 128) continue;
          if (ts == 1 && N > 128) continue;
          bench<<<1, 128, 131072>>>(M, N, R, d, ts, nis);
          unsigned long long h[3];
          cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
          double macs = (double)M * N * 16 * nis;
          printf("%s issuers %d M=%3d N=%3d: issue %6.1f cyc/mma, complete %6.1f cyc/mma (per issuer), %7.0f MAC/cyc total\n",
                 nm[ts], nis, M, N, (double)h[0] / R, (double)h[1] / R, macs / ((double)h[1] / R));
        }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
