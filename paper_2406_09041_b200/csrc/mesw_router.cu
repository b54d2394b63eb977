// K4: batched model-level router forward (multinomial Naive Bayes over hashed character
// 2/3-grams); hashing and summation order pinned in oracle/router.py.
//
// One warp per query.  The warp walks the query's n-grams (all 2-grams, then all 3-grams)
// 32 at a time: lane j hashes n-gram j (FNV-1a over its UTF-8 bytes, low 16 bits), then
// the buckets are broadcast in order and lane d accumulates f64(loglik[d][bucket]) (and
// domain d + 32's, D <= 64) sequentially -- the same additions, in the same order, as the
// CPU restatement, so the argmax (ties -> lowest id) is bit-identical.  The tables
// (D x 2^16 f32, 256 KiB per domain) stay L2-resident across queries.

#include <math.h>

#include "mesw_common.cuh"
#include "mesw_host.h"

namespace mesw {

constexpr int kRouterBuckets = 1 << 16;
constexpr int kRouterMaxDomains = 64;  // two domains per lane
constexpr int kRouterWarps = 4;  // queries per block

__device__ __forceinline__ uint32_t fnv_byte(uint32_t h, uint32_t b) { return (h ^ b) * 16777619u; }

// Fold one code point's UTF-8 encoding into the running FNV-1a state.
__device__ __forceinline__ uint32_t fnv_codepoint(uint32_t h, uint32_t cp) {
  if (cp < 0x80u) return fnv_byte(h, cp);
  if (cp < 0x800u) return fnv_byte(fnv_byte(h, 0xC0u | (cp >> 6)), 0x80u | (cp & 0x3Fu));
  if (cp < 0x10000u)
    return fnv_byte(fnv_byte(fnv_byte(h, 0xE0u | (cp >> 12)), 0x80u | ((cp >> 6) & 0x3Fu)), 0x80u | (cp & 0x3Fu));
  return fnv_byte(fnv_byte(fnv_byte(fnv_byte(h, 0xF0u | (cp >> 18)), 0x80u | ((cp >> 12) & 0x3Fu)),
                           0x80u | ((cp >> 6) & 0x3Fu)),
                  0x80u | (cp & 0x3Fu));
}

__global__ void __launch_bounds__(kRouterWarps * 32) router_classify_kernel(
    const int32_t* __restrict__ cps, const int64_t* __restrict__ offsets, int B, const float* __restrict__ loglik,
    const float* __restrict__ logprior, int D, int32_t* __restrict__ out_domain, float* __restrict__ out_conf,
    int32_t* __restrict__ out_prior_only) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int qi = blockIdx.x * kRouterWarps + (threadIdx.x >> 5);
  if (qi >= B) return;
  const int64_t c0 = offsets[qi];
  const int L = (int)(offsets[qi + 1] - c0);
  const int n2 = L >= 2 ? L - 1 : 0, n3 = L >= 3 ? L - 2 : 0;
  const int G = n2 + n3;
  // lane owns domains d0 = lane and d1 = lane + 32 (D <= 64); each summed sequentially in f64
  const int d0 = lane, d1 = lane + 32;
  const float* row0 = loglik + (size_t)(d0 < D ? d0 : 0) * kRouterBuckets;
  const float* row1 = loglik + (size_t)(d1 < D ? d1 : 0) * kRouterBuckets;
  double s0 = d0 < D ? (double)logprior[d0] : 0.0;
  double s1 = d1 < D ? (double)logprior[d1] : 0.0;
  for (int g0 = 0; g0 < G; g0 += 32) {
    const int g = g0 + lane;
    uint32_t bucket = 0;
    if (g < G) {
      const int n = g < n2 ? 2 : 3;
      const int i = g < n2 ? g : g - n2;
      uint32_t h = 2166136261u;
      for (int t = 0; t < n; ++t) h = fnv_codepoint(h, (uint32_t)cps[c0 + i + t]);
      bucket = h & (kRouterBuckets - 1);
    }
    const int cnt = min(32, G - g0);
    // gather this lane's 32 terms first (independent loads), then add them in order
    float v0[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t b = __shfl_sync(0xffffffffu, bucket, j);
      v0[j] = (j < cnt && d0 < D) ? __ldg(row0 + b) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < cnt) s0 += (double)v0[j];
    if (D > 32) {  // warp-uniform
      float v1[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t b = __shfl_sync(0xffffffffu, bucket, j);
        v1[j] = (j < cnt && d1 < D) ? __ldg(row1 + b) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < cnt) s1 += (double)v1[j];
    }
  }
  // argmax over domains 0..D-1 in id order (ties -> lowest id), then softmax of the winner
  double best = 0.0;
  int win = 0;
  for (int d = 0; d < D; ++d) {
    const double sd = __shfl_sync(0xffffffffu, d < 32 ? s0 : s1, d & 31);
    if (d == 0 || sd > best) { best = sd; win = d; }
  }
  double z = 0.0;
  for (int d = 0; d < D; ++d) z += exp(__shfl_sync(0xffffffffu, d < 32 ? s0 : s1, d & 31) - best);
  if (lane == 0) {
    out_domain[qi] = win;
    out_conf[qi] = (float)(1.0 / z);
    if (out_prior_only) out_prior_only[qi] = G == 0 ? 1 : 0;
  }
}

}  // namespace mesw

using namespace mesw;

extern "C" int mesw_router_classify(const int32_t* d_codepoints, const int64_t* d_offsets, int B,
                                    const float* d_loglik, const float* d_logprior, int D, int32_t* d_domain,
                                    float* d_conf, int32_t* d_prior_only, void* stream) {
  if (B < 0 || D < 1 || D > kRouterMaxDomains) return mesw_fail(MESW_ERR_VALUE, "router: 1..64 domains");
  if (!d_offsets || !d_loglik || !d_logprior || !d_domain || !d_conf)
    return mesw_fail(MESW_ERR_VALUE, "router: null buffer");
  if (B == 0) return MESW_OK;
  mesw_launch(router_classify_kernel, dim3((B + kRouterWarps - 1) / kRouterWarps), dim3(kRouterWarps * 32), 0,
              (cudaStream_t)stream, d_codepoints, d_offsets, B, d_loglik, d_logprior, D, d_domain, d_conf,
              d_prior_only);
  return mesw_check_launch("router_classify");
}
