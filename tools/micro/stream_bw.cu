// Micro-benchmark: achievable HBM streaming rate of the weight-tile producer pattern
// (cp.async.bulk of contiguous tiles into an smem ring, one consumer thread releasing
// slots).  Variants: tile size, ring depth, L2 evict_first hint, paired CTAs with relay.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bw stream_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}

__device__ int PDL_DUMMY;
#define PDL_LAUNCH 1
template <bool HINT>
__global__ void stream_kernel(const uint8_t* src, size_t total, int tile, int depth, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16];
  const size_t ntiles = total / tile;
  const size_t t0 = blockIdx.x * ntiles / gridDim.x, t1 = (blockIdx.x + 1) * ntiles / gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (PDL_LAUNCH) asm volatile("griddepcontrol.launch_dependents;");
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (threadIdx.x == 0) {
    int st = 0; uint32_t ph = 0; bool first = true;
    for (size_t t = t0; t < t1; ++t) {
      if (!first) mbar_wait(&empty[st], ph ^ 1);
      expect_tx(&full[st], tile);
      if (HINT)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(sa(smem + (size_t)st * tile)), "l"(src + t * tile), "r"(tile), "r"(sa(&full[st])), "l"(pol) : "memory");
      else
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(smem + (size_t)st * tile)), "l"(src + t * tile), "r"(tile), "r"(sa(&full[st])) : "memory");
      if (++st == depth) { st = 0; ph ^= 1; first = false; }
    }
  } else if (threadIdx.x == 32) {
    int st = 0; uint32_t ph = 0;
    for (size_t t = t0; t < t1; ++t) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == depth) { st = 0; ph ^= 1; }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // dependent data would be read here
  }
}

int main() {
  const size_t total = (size_t)4096 * 14336 * 2;  // 117 MB (one Mistral FFN projection)
  uint8_t* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  uint8_t* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  int tiles[] = {16384, 32768, 65536};
  int depths[] = {3, 6};
  for (int hint = 0; hint < 2; ++hint)
    for (int ti = 0; ti < 3; ++ti)
      for (int di = 0; di < 2; ++di) {
        const int tile = tiles[ti], depth = depths[di];
        if ((size_t)tile * depth > 200 * 1024) continue;
        for (int grid : {148, 296}) {
          if (grid == 296 && (size_t)tile * depth > 100 * 1024) continue;
          auto k = hint ? stream_kernel<true> : stream_kernel<false>;
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
          float best = 1e9;
          for (int it = 0; it < 6; ++it) {
            cudaMemsetAsync(flush, it, 256 << 20);
            cudaEventRecord(a);
            k<<<grid, 64, (size_t)tile * depth>>>(src, total, tile, depth, nullptr);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best) best = ms;
          }
          printf("hint %d tile %6d depth %d grid %d: %7.2f us  %7.1f GB/s\n", hint, tile, depth, grid, best * 1e3,
                 total / (best * 1e-3) / 1e9);
        }
      }
  // sequences of 8 launches over 8 different 117 MB buffers (a decode layer's worth)
  uint8_t* big;
  cudaMalloc(&big, total * 8);
  cudaMemset(big, 1, total * 8);
  auto k = stream_kernel<true>;
  for (int pdl = 0; pdl < 2; ++pdl) {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaMemsetAsync(flush, it, 256 << 20);
      cudaEventRecord(a);
      for (int l = 0; l < 8; ++l) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = 32768 * 6;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = pdl;
        cudaLaunchKernelEx(&cfg, k, (const uint8_t*)(big + l * total), total, 32768, 6, (unsigned long long*)nullptr);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 0 && ms < best) best = ms;
    }
    printf("8 launches pdl %d: %7.2f us per launch  %7.1f GB/s\n", pdl, best * 1e3 / 8, 8 * total / (best * 1e-3) / 1e9);
  }
  {
    float best = 1e9;
    for (int it = 0; it < 4; ++it) {
      cudaEventRecord(a);
      k<<<148, 64, 32768 * 6>>>(big, total * 8, 32768, 6, nullptr);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 0 && ms < best) best = ms;
    }
    printf("one launch over 940 MB: %7.1f GB/s\n", 8 * total / (best * 1e-3) / 1e9);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
