// Micro-benchmark: tcgen05.st (STTM) throughput on B200 for the K2 dequant pattern
// (each warp stores 32 lanes x C columns of 32-bit words, then waits).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sttm_rate sttm_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define R8(b) "r"(r[b + 0]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3]), "r"(r[b + 4]), "r"(r[b + 5]), "r"(r[b + 6]), "r"(r[b + 7])
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {"
      "%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      R8(0), R8(8), R8(16), R8(24)
      : "memory");
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {"
      "%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      R8(0), R8(8)
      : "memory");
}

// mode 0: x32 store + wait each iteration; 1: x32 stores, wait every 4; 2: x16 + wait each
__global__ void bench(int R, int mode, unsigned long long* out) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tb;
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = lane * 131 + i * 7 + warp;
  const uint32_t col = (uint32_t)((warp >> 2) * 64) % 512;
  const uint32_t addr = t + (((uint32_t)(warp & 3) * 32) << 16) + col;
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < R; ++i) {
    if (mode == 2) {
      st16(addr + (i & 1) * 16, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else {
      st32(addr + (i & 1) * 32, r);
      if (mode == 0 || (i & 3) == 3) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
#pragma unroll
    for (int k = 0; k < 32; ++k) r[k] += 1;
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  long long c1 = clock64();
  __syncthreads();
  if (lane == 0) out[blockIdx.x * 32 + warp] = (unsigned long long)(c1 - c0);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 32 * 8);
  unsigned long long h[148 * 32];
  const int R = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 12, 16}) {
      bench<<<148, warps * 32>>>(R, mode, d);
      cudaDeviceSynchronize();
      bench<<<148, warps * 32>>>(R, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
      const double bytes = (double)warps * R * 32 * (mode == 2 ? 16 : 32) * 4;
      printf("mode %d (%s) warps %2d: %8llu cycles, %.1f B/cycle/SM, %.0f cycles per 32 KB job-equivalent\n", mode,
             mode == 0 ? "x32+wait" : (mode == 1 ? "x32, wait/4" : "x16+wait"), warps, mx, bytes / mx,
             32768.0 / (bytes / mx));
    }
  return 0;
}
