// K5: decoder glue for the Mistral-7B-shaped multi-expert decode step (sm_100a).
//
// The reference toy model has no attention (toylm.py:1-8); these kernels are
// the standard Mistral decoder pieces around the fused multi-expert linears:
// embedding gather, RMSNorm, RoPE + KV-cache append, GQA decode attention,
// SwiGLU and the greedy argmax (first maximum, toylm.py:247 / np.argmax).
// All HBM-bound and tiny next to the linears; f32 arithmetic, bf16 storage.

#include <math.h>

#include "mesw_common.cuh"
#include "mesw_host.h"

namespace mesw {

// Canonical activation layout of mesw.h (consumed by the fused linear).
__device__ __forceinline__ size_t canon_index(int t, int k, int NP) {
  return (size_t)(k >> 7) * NP * 128 + (size_t)((t >> 3) & 1) * (NP / 2) * 128 + (size_t)(t >> 4) * 1024 +
         ((k & 127) >> 3) * 64 + (t & 7) * 8 + (k & 7);
}

// Output address of element (t, k): row-major with ld, or canonical when np > 0.
// Offset-code bias weight of input k (mesw.h x_corr): pair l = ((k % 64) / 2) % 8 ->
// 130 (l in {0,3,6}), 34 ({1,4,7}), 10 ({2,5}).
__device__ __forceinline__ float corr_w(int k) {
  const int l = ((k & 63) >> 1) & 7;
  const int m = l < 6 ? l % 3 : l - 6;
  return m == 0 ? 130.f : (m == 1 ? 34.f : 10.f);
}

// sum over the 16-lane half-warp holding one k-step (fixed tree order: deterministic)
__device__ __forceinline__ float sum16(float v) {
#pragma unroll
  for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ size_t out_index(int t, int k, int ld, int np) {
  return np > 0 ? canon_index(t, k, np) : (size_t)t * ld + k;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum for blockDim.x <= 1024; `red` has >= 32 floats.
__device__ __forceinline__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = lane < nw ? red[lane] : 0.f;
  return warp_sum(t);
}

__device__ __forceinline__ float block_max(float v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = lane < nw ? red[lane] : -INFINITY;
  return warp_max(t);
}

__global__ void embed_kernel(const int32_t* __restrict__ ids, const uint16_t* __restrict__ table,
                             int H, uint16_t* __restrict__ out, int ld_out) {
  pdl_trigger();
  pdl_wait();  // inputs may come from the previous kernel in the stream
  const int b = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(table + (size_t)ids[b] * H);
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)b * ld_out);
  for (int i = threadIdx.x; i < H / 8; i += blockDim.x) dst[i] = src[i];
}

// y = x * rsqrt(mean(x^2) + eps) * w   (one CTA per token; row held in registers,
// one 16-byte load per 8 elements, single global pass)
#ifndef MESW_NORM_THREADS
#define MESW_NORM_THREADS 256
#endif
constexpr int kNormThreads = MESW_NORM_THREADS;
// 16-byte vectors per thread: 8192 channels = 1024 vectors of 8 over the block
constexpr int kNormMaxVec = 1024 / MESW_NORM_THREADS;
static_assert(1024 % MESW_NORM_THREADS == 0, "MESW_NORM_THREADS must divide 1024");
__global__ void __launch_bounds__(kNormThreads) rmsnorm_kernel(const uint16_t* __restrict__ x, int ldx,
                                                               const uint16_t* __restrict__ w, int H, float eps,
                                                               uint16_t* __restrict__ y, int ldy, int ynp,
                                                               float* __restrict__ corr, int corr_ld) {
  pdl_trigger();
  __shared__ float red[32];
  const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t)blockIdx.x * ldx);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  const int nvec = H / 8;
  uint4 gw[kNormMaxVec];  // the norm weights are static: read them while the producer drains
#pragma unroll
  for (int j = 0; j < kNormMaxVec; ++j) {
    const int i = threadIdx.x + j * kNormThreads;
    if (i < nvec) gw[j] = __ldg(wr + i);
  }
  pdl_wait();  // x comes from the previous kernel in the stream
  uint4 v[kNormMaxVec];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kNormMaxVec; ++j) {
    const int i = threadIdx.x + j * kNormThreads;
    if (i < nvec) {
      v[j] = xr[i];
      const uint32_t* e = reinterpret_cast<const uint32_t*>(&v[j]);
#pragma unroll
      for (int q = 0; q < 4; ++q) ss = fmaf(bf16_lo(e[q]), bf16_lo(e[q]), fmaf(bf16_hi(e[q]), bf16_hi(e[q]), ss));
    }
  }
  const float r = rsqrtf(block_sum(ss, red) / (float)H + eps);
#pragma unroll
  for (int j = 0; j < kNormMaxVec; ++j) {
    const int i = threadIdx.x + j * kNormThreads;
    float c = 0.f;
    if (i < nvec) {
      const uint4 g4 = gw[j];
      const uint32_t* e = reinterpret_cast<const uint32_t*>(&v[j]);
      const uint32_t* g = reinterpret_cast<const uint32_t*>(&g4);
      uint4 o;
      uint32_t* oo = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        __nv_bfloat162 t = __floats2bfloat162_rn(bf16_lo(e[q]) * r * bf16_lo(g[q]), bf16_hi(e[q]) * r * bf16_hi(g[q]));
        oo[q] = *reinterpret_cast<uint32_t*>(&t);
      }
      *reinterpret_cast<uint4*>(y + out_index(blockIdx.x, i * 8, ldy, ynp)) = o;
#pragma unroll
      for (int q = 0; q < 4; ++q) c += corr_w(i * 8 + 2 * q) * (bf16_lo(oo[q]) + bf16_hi(oo[q]));
    }
    if (corr) {  // 16 consecutive threads hold the 16 chunks of one k-step (H % 128 == 0)
      c = sum16(c);
      if (i < nvec && (i & 15) == 0) corr[(size_t)blockIdx.x * corr_ld + i / 16] = c;
    }
  }
}

// RoPE (rotate-half pairs (i, i+D/2)) on q in place and on k, then append k and v
// to the cache at each token's position.  qkv row: [q heads | k heads | v heads].
// grid (B, n_heads + n_kv_heads), block D/2.
__global__ void rope_append_kernel(uint16_t* __restrict__ qkv, int ld_qkv, const int32_t* __restrict__ pos,
                                   int n_heads, int n_kv, int D, float theta,
                                   uint16_t* __restrict__ kc, uint16_t* __restrict__ vc, int ctx_max) {
  pdl_trigger();
  pdl_wait();  // inputs may come from the previous kernel in the stream
  const int b = blockIdx.x, h = blockIdx.y, i = threadIdx.x, half = D / 2;
  const int p = pos[b];
  const float inv = powf(theta, -2.0f * (float)i / (float)D);
  float sn, cs;
  sincosf((float)p * inv, &sn, &cs);
  uint16_t* row = qkv + (size_t)b * ld_qkv;
  const bool is_q = h < n_heads;
  const int kvh = h - n_heads;
  uint16_t* v = row + (size_t)(is_q ? h : n_heads + kvh) * D;
  const float x0 = bf16_to_f32(v[i]), x1 = bf16_to_f32(v[i + half]);
  const float r0 = x0 * cs - x1 * sn, r1 = x1 * cs + x0 * sn;
  const uint16_t o0 = __bfloat16_as_ushort(__float2bfloat16_rn(r0));
  const uint16_t o1 = __bfloat16_as_ushort(__float2bfloat16_rn(r1));
  if (is_q) {
    v[i] = o0;
    v[i + half] = o1;
  } else {
    const size_t base = (((size_t)b * ctx_max + p) * n_kv + kvh) * D;
    kc[base + i] = o0;
    kc[base + i + half] = o1;
    const uint16_t* vv = row + (size_t)(n_heads + n_kv + kvh) * D;
    vc[base + i] = vv[i];
    vc[base + i + half] = vv[i + half];
  }
}

// GQA decode attention: one CTA per (token, kv head); the G = n_heads / n_kv query
// heads sharing the kv head are processed together.  K and V rows of the context
// are staged in shared memory with coalesced 16-byte loads (rows padded to 272 B:
// conflict-free 128-bit accesses), then
//   scores: thread t owns position t (all G heads, 128-dim dot from smem),
//   softmax: block reductions per head (fixed order),
//   P.V: thread = (4-dim group, position slice), slices reduced through smem.
// GQA decode attention, split over the context (flash-decoding): CTA (b, kv head g, split s)
// handles positions [P s, P s + P) (P = kAttnSplit) for the G query heads of kv head g and writes a
// partial (running max, sum of exponentials, unnormalised output) per head; a second
// kernel merges the splits.  Many small CTAs stream the KV cache at full occupancy
// (the cache is read once per step: an HBM-bound pass).  D must be 128.
constexpr int kAttnThreads = 128;
#ifndef MESW_ATTN_SPLIT
#define MESW_ATTN_SPLIT 32  // measured on C2 (B=32, ctx 129-256): 32 > 64 (+0.5-1 %) > 16
#endif
constexpr int kAttnSplit = MESW_ATTN_SPLIT;  // positions per CTA
constexpr int kAttnRow = 136;      // bf16 per staged row (128 + 8 pad: conflict-free row reads)
constexpr int kAttnPart = 2 + 128; // floats per (b, head, split) partial: m, l, o[128]

// ROPE: fused decode form (rope_append folded in).  q holds the new token's fused qkv row
// ([q heads | k heads | v heads], q and k not yet rotated); the new token sits at position
// len[b] - 1 (the engine keeps len = pos + 1).  Every split rotates its q heads on load
// (same arithmetic and bf16 rounding as rope_append_kernel); the split holding the new
// position rotates k, stages the new k / v row from registers and appends it to the caches
// (no other split reads that position in this launch).
template <int G, bool ROPE>
__global__ void __launch_bounds__(kAttnThreads) attn_partial_kernel(
    const uint16_t* __restrict__ q, int ld_q, uint16_t* __restrict__ kc, uint16_t* __restrict__ vc,
    const int32_t* __restrict__ len, int n_kv, int ctx_max, float scale, float* __restrict__ part, int S,
    float theta) {
  pdl_trigger();
  // ROPE (the decode engine's fused form): len and the cached rows were written by earlier
  // decode steps, only the new token's q / k / v row comes from the previous kernel -- the
  // K / V stream starts before the wait, under the tail of the qkv linear
  if (!ROPE) pdl_wait();  // inputs may come from the previous kernel in the stream
  constexpr int D = 128;
  __shared__ __align__(16) uint16_t Ks[kAttnSplit * kAttnRow];
  __shared__ __align__(16) uint16_t Vs[kAttnSplit * kAttnRow];
  __shared__ __align__(16) float qs[G * D];
  __shared__ float ps[G][kAttnSplit];
  const int b = blockIdx.x, g = blockIdx.y, sp = blockIdx.z, tid = threadIdx.x;
  const int L = len[b];
  const int t0 = sp * kAttnSplit;
  if (t0 >= L) return;  // beyond this request's context: the merge ignores the split
  const int n = min(kAttnSplit, L - t0);
  const size_t kv_stride = (size_t)n_kv * D;
  const uint16_t* kb = kc + (((size_t)b * ctx_max + t0) * n_kv + g) * D;
  const uint16_t* vb = vc + (((size_t)b * ctx_max + t0) * n_kv + g) * D;
  const int n_cached = ROPE && t0 + n == L ? n - 1 : n;  // ROPE: the last row is the new token
  // cp.async: every thread's 16-byte K / V copies are in flight together (one wait below)
  for (int i = tid; i < n_cached * 16; i += kAttnThreads) {
    const int t = i >> 4, c = i & 15;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(Ks + t * kAttnRow + c * 8)),
                 "l"(kb + t * kv_stride + c * 8) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(Vs + t * kAttnRow + c * 8)),
                 "l"(vb + t * kv_stride + c * 8) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  const uint16_t* qrow = q + (size_t)b * ld_q;
  if (ROPE) {
    const int p = L - 1;
    constexpr int half = D / 2;
    constexpr int NQ = (G * half + kAttnThreads - 1) / kAttnThreads;  // (head, pair)s per thread
    // the rotation angles depend only on the position: computed before the PDL wait, then
    // every input element of the new row is requested at once (one round trip)
    float qcs[NQ], qsn[NQ];
#pragma unroll
    for (int r = 0; r < NQ; ++r) {
      const int i = tid + r * kAttnThreads, j = i % half;
      qcs[r] = 1.f; qsn[r] = 0.f;
      if (i < G * half) {
        const float inv = powf(theta, -2.0f * (float)j / (float)D);
        sincosf((float)p * inv, &qsn[r], &qcs[r]);
      }
    }
    const bool new_row = n_cached < n;  // this split holds the new position: rotate k, stage + append k / v
    float kcs = 1.f, ksn = 0.f;
    if (new_row && tid < half) {
      const float inv = powf(theta, -2.0f * (float)tid / (float)D);
      sincosf((float)p * inv, &ksn, &kcs);
    }
    pdl_wait();  // the new token's fused qkv row
    float x0[NQ], x1[NQ];
#pragma unroll
    for (int r = 0; r < NQ; ++r) {
      const int i = tid + r * kAttnThreads, hh = i / half, j = i % half;
      x0[r] = x1[r] = 0.f;
      if (i < G * half) {
        const uint16_t* v = qrow + (size_t)(g * G + hh) * D;
        x0[r] = bf16_to_f32(v[j]);
        x1[r] = bf16_to_f32(v[j + half]);
      }
    }
    const int n_heads = G * n_kv;
    uint16_t e0 = 0, e1 = 0;
    if (new_row) {
      const int j = tid < half ? tid : tid - half;
      const uint16_t* v = qrow + (size_t)(tid < half ? n_heads + g : n_heads + n_kv + g) * D;
      e0 = v[j];
      e1 = v[j + half];
    }
#pragma unroll
    for (int r = 0; r < NQ; ++r) {
      const int i = tid + r * kAttnThreads, hh = i / half, j = i % half;
      if (i < G * half) {
        qs[hh * D + j] = __bfloat162float(__float2bfloat16_rn(x0[r] * qcs[r] - x1[r] * qsn[r])) * scale;
        qs[hh * D + j + half] = __bfloat162float(__float2bfloat16_rn(x1[r] * qcs[r] + x0[r] * qsn[r])) * scale;
      }
    }
    if (new_row) {
      const int t = n - 1;
      const size_t cbase = (((size_t)b * ctx_max + p) * n_kv + g) * D;
      if (tid < half) {
        const int j = tid;
        const float k0 = bf16_to_f32(e0), k1 = bf16_to_f32(e1);
        const uint16_t o0 = __bfloat16_as_ushort(__float2bfloat16_rn(k0 * kcs - k1 * ksn));
        const uint16_t o1 = __bfloat16_as_ushort(__float2bfloat16_rn(k1 * kcs + k0 * ksn));
        Ks[t * kAttnRow + j] = o0;
        Ks[t * kAttnRow + j + half] = o1;
        kc[cbase + j] = o0;
        kc[cbase + j + half] = o1;
      } else {
        const int j = tid - half;
        Vs[t * kAttnRow + j] = e0;
        Vs[t * kAttnRow + j + half] = e1;
        vc[cbase + j] = e0;
        vc[cbase + j + half] = e1;
      }
    }
  } else {
    for (int i = tid; i < G * D; i += kAttnThreads)
      qs[i] = bf16_to_f32(qrow[(size_t)g * G * D + i]) * scale;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // scores: thread -> (head h, positions t, t + 32 ...) with 128 / G threads per head
  constexpr int TPH = kAttnThreads / G;
  {
    const int h = tid / TPH, j = tid % TPH;
    for (int t = j; t < n; t += TPH) {
      float acc = 0.f;
#pragma unroll 4
      for (int c = 0; c < 16; ++c) {
        const uint4 k4 = *reinterpret_cast<const uint4*>(Ks + t * kAttnRow + c * 8);
        const uint32_t* kk = reinterpret_cast<const uint32_t*>(&k4);
        const float4 qa = *reinterpret_cast<const float4*>(qs + h * D + c * 8);
        const float4 qb = *reinterpret_cast<const float4*>(qs + h * D + c * 8 + 4);
        acc = fmaf(qa.x, bf16_lo(kk[0]), acc); acc = fmaf(qa.y, bf16_hi(kk[0]), acc);
        acc = fmaf(qa.z, bf16_lo(kk[1]), acc); acc = fmaf(qa.w, bf16_hi(kk[1]), acc);
        acc = fmaf(qb.x, bf16_lo(kk[2]), acc); acc = fmaf(qb.y, bf16_hi(kk[2]), acc);
        acc = fmaf(qb.z, bf16_lo(kk[3]), acc); acc = fmaf(qb.w, bf16_hi(kk[3]), acc);
      }
      ps[h][t] = acc;
    }
  }
  __syncthreads();
  // per-head max / exp / sum: warp w handles heads w, w + 4, ...
  const int warp = tid >> 5, lane = tid & 31;
  float* outp = part + (((size_t)b * gridDim.y + g) * G) * (size_t)S * kAttnPart;
  for (int h = warp; h < G; h += kAttnThreads / 32) {
    float m = -INFINITY;
    for (int t = lane; t < n; t += 32) m = fmaxf(m, ps[h][t]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.f;
    for (int t = lane; t < n; t += 32) {
      const float e = __expf(ps[h][t] - m);
      ps[h][t] = e;
      l += e;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      float* pp = outp + ((size_t)h * S + sp) * kAttnPart;
      pp[0] = m;
      pp[1] = l;
    }
  }
  __syncthreads();
  // P.V: thread = output dim d, all G heads
  {
    const int d = tid;
    float o[G];
#pragma unroll
    for (int h = 0; h < G; ++h) o[h] = 0.f;
    for (int t = 0; t < n; ++t) {
      const float v = bf16_to_f32(Vs[t * kAttnRow + d]);
#pragma unroll
      for (int h = 0; h < G; ++h) o[h] = fmaf(ps[h][t], v, o[h]);
    }
#pragma unroll
    for (int h = 0; h < G; ++h) outp[((size_t)h * S + sp) * kAttnPart + 2 + d] = o[h];
  }
}

// Merge the splits of one (request, head): out = sum_s e^{m_s - M} o_s / sum_s e^{m_s - M} l_s.
// PRE (the fused decode form): len is complete before the launch (see attn_partial_kernel),
// so it is read before the PDL wait and only the partials after it.
template <bool PRE>
__global__ void __launch_bounds__(128) attn_merge_kernel(const float* __restrict__ part, const int32_t* __restrict__ len,
                                                         int n_heads, int S, uint16_t* __restrict__ out, int ld_out,
                                                         int out_np, float* __restrict__ corr, int corr_ld) {
  __shared__ float red[4];
  pdl_trigger();
  if (!PRE) pdl_wait();
  const int b = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  const int Sb = (len[b] + kAttnSplit - 1) / kAttnSplit;
  if (PRE) pdl_wait();
  const float* pp = part + ((size_t)b * n_heads + h) * (size_t)S * kAttnPart;
  float M = -INFINITY;
  float num = 0.f, den = 0.f;
  if (Sb <= 8) {  // every split's (m, l, o[d]) requested at once: one L2 round trip
    float ms[8], ls[8], os[8];
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2)
      if (s2 < Sb) {
        ms[s2] = pp[(size_t)s2 * kAttnPart];
        ls[s2] = pp[(size_t)s2 * kAttnPart + 1];
        os[s2] = pp[(size_t)s2 * kAttnPart + 2 + d];
      }
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2)
      if (s2 < Sb) M = fmaxf(M, ms[s2]);
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2)
      if (s2 < Sb) {
        const float w = __expf(ms[s2] - M);
        den = fmaf(w, ls[s2], den);
        num = fmaf(w, os[s2], num);
      }
  } else {
    for (int s2 = 0; s2 < Sb; ++s2) M = fmaxf(M, pp[(size_t)s2 * kAttnPart]);
    for (int s2 = 0; s2 < Sb; ++s2) {
      const float w = __expf(pp[(size_t)s2 * kAttnPart] - M);
      den = fmaf(w, pp[(size_t)s2 * kAttnPart + 1], den);
      num = fmaf(w, pp[(size_t)s2 * kAttnPart + 2 + d], num);
    }
  }
  const __nv_bfloat16 ob = __float2bfloat16_rn(num / den);
  out[out_index(b, h * 128 + d, ld_out, out_np)] = __bfloat16_as_ushort(ob);
  if (corr) {  // one head = one k-step of o_proj
    float c = corr_w(d) * __bfloat162float(ob);
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((d & 31) == 0) red[d >> 5] = c;
    __syncthreads();
    if (d == 0) corr[(size_t)b * corr_ld + h] = (red[0] + red[1]) + (red[2] + red[3]);
  }
}

// out = silu(gate) * up, gate/up halves of a [B][2I] row.
__global__ void swiglu_kernel(const uint16_t* __restrict__ gu, int ld_gu, int I, uint16_t* __restrict__ out,
                              int ld_out, int out_np, float* __restrict__ corr, int corr_ld) {
  pdl_trigger();
  pdl_wait();  // inputs may come from the previous kernel in the stream
  // 4 outputs per thread: a warp covers 128 consecutive outputs = one k-step of the next linear
  const int b = blockIdx.y;
  const uint16_t* r = gu + (size_t)b * ld_gu;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4; i < I; i += gridDim.x * blockDim.x * 4) {
    const uint2 g4 = *reinterpret_cast<const uint2*>(r + i);
    const uint2 u4 = *reinterpret_cast<const uint2*>(r + I + i);
    const uint32_t gg[2] = {g4.x, g4.y}, uu[2] = {u4.x, u4.y};
    uint32_t o[2];
    float c = 0.f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float g0 = bf16_lo(gg[h]), g1 = bf16_hi(gg[h]);
      const float s0 = g0 / (1.f + __expf(-g0)), s1 = g1 / (1.f + __expf(-g1));
      __nv_bfloat162 v = __floats2bfloat162_rn(s0 * bf16_lo(uu[h]), s1 * bf16_hi(uu[h]));
      o[h] = *reinterpret_cast<uint32_t*>(&v);
      c += corr_w(i + 2 * h) * (bf16_lo(o[h]) + bf16_hi(o[h]));
    }
    *reinterpret_cast<uint2*>(out + out_index(b, i, ld_out, out_np)) = make_uint2(o[0], o[1]);
    if (corr) {
#pragma unroll
      for (int q = 16; q; q >>= 1) c += __shfl_xor_sync(0xffffffffu, c, q);
      if ((threadIdx.x & 31) == 0) corr[(size_t)b * corr_ld + i / 128] = c;
    }
  }
}

// argmax over a row with ties to the lowest index (np.argmax); f32 or bf16 logits.
__global__ void argmax_kernel(const void* __restrict__ logits, int is_bf16, int V, int ld,
                              int32_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();  // inputs may come from the previous kernel in the stream
  __shared__ float bv[32];
  __shared__ int bi[32];
  const int b = blockIdx.x;
  float best = -INFINITY;
  int bidx = 0x7fffffff;
  if (is_bf16 && V % 8 == 0 && ld % 8 == 0) {  // 16-byte loads: 8 logits per thread per pass
    const uint4* row = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(logits) + (size_t)b * ld);
    for (int c = threadIdx.x; c < V / 8; c += blockDim.x) {
      const uint4 q = __ldg(row + c);
      const uint32_t* e = reinterpret_cast<const uint32_t*>(&q);
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // ascending index inside the chunk: ties keep the first
        const float v = (k & 1) ? bf16_hi(e[k >> 1]) : bf16_lo(e[k >> 1]);
        if (bidx == 0x7fffffff || v > best) { best = v; bidx = 8 * c + k; }
      }
    }
  } else {
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
      const float v = is_bf16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(logits)[(size_t)b * ld + i])
                              : reinterpret_cast<const float*>(logits)[(size_t)b * ld + i];
      if (bidx == 0x7fffffff || v > best) { best = v; bidx = i; }  // i ascending: ties keep the first
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { bv[w] = best; bi[w] = bidx; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? bv[lane] : -INFINITY;
    bidx = lane < nw ? bi[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
    }
    if (lane == 0) out[b] = bidx == 0x7fffffff ? 0 : bidx;
  }
}

// Row-major -> canonical (one thread per 16-byte chunk of 8 k); zero padding.  src (optional):
// canonical row t takes x row src[t] (-1: a zero padding row) -- the expert-grouping gather of
// the public me_linear path, done on the device.
__global__ void pack_x_kernel(const uint16_t* __restrict__ x, int B, int m, int ldx, uint16_t* __restrict__ xc,
                              int NP, int n_ks, float* __restrict__ corr, int corr_ld,
                              const int32_t* __restrict__ src) {
  pdl_trigger();
  pdl_wait();  // inputs may come from the previous kernel in the stream
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)n_ks * NP * 16;
  if (tid >= total) return;  // (total is a multiple of 16: k-step groups never straddle the exit)
  const int kc = (int)(tid % 16);
  const int t = (int)((tid / 16) % NP);
  const int ks = (int)(tid / (16LL * NP));
  const int k0 = ks * 128 + kc * 8;
  uint4 v = make_uint4(0, 0, 0, 0);
  const int r = src ? (t < B ? src[t] : -1) : (t < B ? t : -1);
  if (r >= 0) {
    if (k0 + 8 <= m && (ldx % 8) == 0) {
      v = *reinterpret_cast<const uint4*>(x + (size_t)r * ldx + k0);
    } else {
      uint16_t e[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) e[i] = (k0 + i < m) ? x[(size_t)r * ldx + k0 + i] : (uint16_t)0;
      v = make_uint4(e[0] | (uint32_t(e[1]) << 16), e[2] | (uint32_t(e[3]) << 16), e[4] | (uint32_t(e[5]) << 16),
                     e[6] | (uint32_t(e[7]) << 16));
    }
  }
  *reinterpret_cast<uint4*>(xc + canon_index(t, k0, NP)) = v;
  if (corr) {
    const uint32_t* e = reinterpret_cast<const uint32_t*>(&v);
    float c = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) c += corr_w(k0 + 2 * q) * (bf16_lo(e[q]) + bf16_hi(e[q]));
    c = sum16(c);
    if (kc == 0) corr[(size_t)t * corr_ld + ks] = c;
  }
}

__global__ void unpack_x_kernel(const uint16_t* __restrict__ xc, int B, int m, int NP, uint16_t* __restrict__ y,
                                int ldy) {
  pdl_trigger();
  pdl_wait();  // inputs may come from the previous kernel in the stream
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)B * m) return;
  const int t = (int)(tid / m), k = (int)(tid % m);
  y[(size_t)t * ldy + k] = xc[canon_index(t, k, NP)];
}

// Advance every request by one position (pos += 1, len = pos + 1).  wrap_to >= 0: a request
// that reaches the end of its cache window wraps back to `wrap_to` (bench steady state only);
// wrap_to < 0 (serving): no wrap -- the host refuses a step that would pass the window.
__global__ void advance_kernel(int32_t* __restrict__ pos, int32_t* __restrict__ len, int B, int ctx_max,
                               int wrap_to) {
  // no early trigger: the next step's kernels launch only after the positions are written,
  // so the whole previous step (and len) is complete before any of them starts -- the fused
  // decode attention reads len and the cached rows before its PDL wait
  pdl_wait();  // inputs may come from the previous kernel in the stream
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int p = pos[b] + 1;
  if (p >= ctx_max && wrap_to >= 0) p = wrap_to;
  pos[b] = p;
  len[b] = p + 1;
}

}  // namespace mesw

using namespace mesw;

extern "C" int mesw_advance_positions(int32_t* d_pos, int32_t* d_len, int B, int ctx_max, int wrap_to,
                                      void* stream) {
  if (B <= 0 || wrap_to >= ctx_max) return mesw_fail(MESW_ERR_VALUE, "advance: bad args");
  mesw_launch(advance_kernel, dim3((B + 127) / 128), dim3(128), 0, (cudaStream_t)stream, d_pos, d_len, B, ctx_max, wrap_to);
  return mesw_check_launch("advance_positions");
}

extern "C" int mesw_embed(const int32_t* d_ids, int B, const uint16_t* d_table, int H, uint16_t* d_out,
                          int ld_out, void* stream) {
  if (B <= 0 || H % 8) return mesw_fail(MESW_ERR_VALUE, "embed: H must be a multiple of 8");
  mesw_launch(embed_kernel, dim3(B), dim3(128), 0, (cudaStream_t)stream, d_ids, d_table, H, d_out, ld_out);
  return mesw_check_launch("embed");
}

extern "C" int mesw_rmsnorm(const uint16_t* d_x, int ldx, const uint16_t* d_w, int B, int H, float eps,
                            uint16_t* d_y, int ldy, int y_np, float* d_corr, int corr_ld, void* stream) {
  if (d_corr && (H % 128 || corr_ld < H / 128)) return mesw_fail(MESW_ERR_VALUE, "rmsnorm: corr table needs H % 128 == 0");
  if (B <= 0 || H % 8 || H > kNormThreads * kNormMaxVec * 8 || ldx % 8 || ldy % 8)
    return mesw_fail(MESW_ERR_VALUE, "rmsnorm: H and strides must be multiples of 8, H <= 8192");
  if (y_np > 0 && (y_np % 16 || y_np < B)) return mesw_fail(MESW_ERR_VALUE, "rmsnorm: canonical rows must be >= B, multiple of 16");
  mesw_launch(rmsnorm_kernel, dim3(B), dim3(kNormThreads), 0, (cudaStream_t)stream, d_x, ldx, d_w, H, eps, d_y, ldy, y_np,
              d_corr, corr_ld);
  return mesw_check_launch("rmsnorm");
}

extern "C" int mesw_rope_append(uint16_t* d_qkv, int ld_qkv, const int32_t* d_pos, int B, int n_heads,
                                int n_kv, int head_dim, float theta, uint16_t* d_kcache, uint16_t* d_vcache,
                                int ctx_max, void* stream) {
  if (B <= 0 || head_dim % 2 || head_dim > 2048) return mesw_fail(MESW_ERR_VALUE, "rope: bad shape");
  dim3 grid(B, n_heads + n_kv);
  mesw_launch(rope_append_kernel, dim3(grid), dim3(head_dim / 2), 0, (cudaStream_t)stream, d_qkv, ld_qkv, d_pos, n_heads, n_kv, head_dim, theta, d_kcache, d_vcache, ctx_max);
  return mesw_check_launch("rope_append");
}

extern "C" uint64_t mesw_attention_workspace_bytes(int B, int n_heads, int ctx_max) {
  const int S = (ctx_max + kAttnSplit - 1) / kAttnSplit;
  return (uint64_t)B * n_heads * S * kAttnPart * sizeof(float);
}

static int attention_decode(const uint16_t* d_q, int ld_q, uint16_t* d_kcache, uint16_t* d_vcache,
                            const int32_t* d_len, int B, int n_heads, int n_kv, int head_dim, int ctx_max,
                            uint16_t* d_out, int ld_out, int out_np, void* d_workspace, uint64_t workspace_bytes,
                            float* d_corr, int corr_ld, bool rope, float theta, void* stream) {
  if (B <= 0 || n_kv <= 0 || n_heads % n_kv || ctx_max <= 0) return mesw_fail(MESW_ERR_VALUE, "attention: bad shape");
  if (head_dim != 128) return mesw_fail(MESW_ERR_UNSUPPORTED, "attention: head_dim must be 128");
  if (!d_workspace || workspace_bytes < mesw_attention_workspace_bytes(B, n_heads, ctx_max))
    return mesw_fail(MESW_ERR_VALUE, "attention: workspace too small (mesw_attention_workspace_bytes)");
  if (d_corr && corr_ld < n_heads) return mesw_fail(MESW_ERR_VALUE, "attention: corr_ld too small");
  const int G = n_heads / n_kv;
  const int S = (ctx_max + kAttnSplit - 1) / kAttnSplit;
  const float scale = 1.0f / sqrtf((float)head_dim);
  dim3 grid(B, n_kv, S);
  cudaStream_t s = (cudaStream_t)stream;
  float* part = reinterpret_cast<float*>(d_workspace);
  cudaError_t e;
#define MESW_ATTN_CASE(GG)                                                                                     \
  case GG:                                                                                                     \
    e = rope ? mesw_launch(attn_partial_kernel<GG, true>, grid, dim3(kAttnThreads), 0, s, d_q, ld_q, d_kcache,   \
                           d_vcache, d_len, n_kv, ctx_max, scale, part, S, theta)                              \
             : mesw_launch(attn_partial_kernel<GG, false>, grid, dim3(kAttnThreads), 0, s, d_q, ld_q, d_kcache,  \
                           d_vcache, d_len, n_kv, ctx_max, scale, part, S, theta);                             \
    break;
  switch (G) {
    MESW_ATTN_CASE(1)
    MESW_ATTN_CASE(2)
    MESW_ATTN_CASE(4)
    MESW_ATTN_CASE(8)
    default:
      return mesw_fail(MESW_ERR_UNSUPPORTED, "attention: heads per kv head must be 1, 2, 4 or 8");
  }
#undef MESW_ATTN_CASE
  if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
  e = rope ? mesw_launch(attn_merge_kernel<true>, dim3(B, n_heads), dim3(128), 0, s, (const float*)part, d_len, n_heads,
                         S, d_out, ld_out, out_np, d_corr, corr_ld)
           : mesw_launch(attn_merge_kernel<false>, dim3(B, n_heads), dim3(128), 0, s, (const float*)part, d_len,
                         n_heads, S, d_out, ld_out, out_np, d_corr, corr_ld);
  if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
  return mesw_check_launch("attention_decode");
}

extern "C" int mesw_attention_decode(const uint16_t* d_q, int ld_q, const uint16_t* d_kcache,
                                     const uint16_t* d_vcache, const int32_t* d_len, int B, int n_heads,
                                     int n_kv, int head_dim, int ctx_max, uint16_t* d_out, int ld_out,
                                     int out_np, void* d_workspace, uint64_t workspace_bytes, float* d_corr,
                                     int corr_ld, void* stream) {
  // read-only caches (the non-ROPE instance never writes them)
  return attention_decode(d_q, ld_q, const_cast<uint16_t*>(d_kcache), const_cast<uint16_t*>(d_vcache), d_len, B,
                          n_heads, n_kv, head_dim, ctx_max, d_out, ld_out, out_np, d_workspace, workspace_bytes,
                          d_corr, corr_ld, false, 0.f, stream);
}

extern "C" int mesw_attention_decode_rope(const uint16_t* d_qkv, int ld_qkv, uint16_t* d_kcache,
                                          uint16_t* d_vcache, const int32_t* d_len, int B, int n_heads, int n_kv,
                                          int head_dim, float theta, int ctx_max, uint16_t* d_out, int ld_out,
                                          int out_np, void* d_workspace, uint64_t workspace_bytes, float* d_corr,
                                          int corr_ld, void* stream) {
  return attention_decode(d_qkv, ld_qkv, d_kcache, d_vcache, d_len, B, n_heads, n_kv, head_dim, ctx_max, d_out,
                          ld_out, out_np, d_workspace, workspace_bytes, d_corr, corr_ld, true, theta, stream);
}

extern "C" int mesw_swiglu(const uint16_t* d_gu, int ld_gu, int B, int I, uint16_t* d_out, int ld_out,
                           int out_np, float* d_corr, int corr_ld, void* stream) {
  if (B <= 0 || I % 128 || ld_gu % 4 || (out_np == 0 && ld_out % 4)) return mesw_fail(MESW_ERR_VALUE, "swiglu: I must be a multiple of 128");
  if (d_corr && corr_ld < I / 128) return mesw_fail(MESW_ERR_VALUE, "swiglu: corr_ld too small");
  dim3 grid((I / 4 + 255) / 256 < 64 ? (I / 4 + 255) / 256 : 64, B);
  mesw_launch(swiglu_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, d_gu, ld_gu, I, d_out, ld_out, out_np,
              d_corr, corr_ld);
  return mesw_check_launch("swiglu");
}

extern "C" int mesw_argmax(const void* d_logits, int is_bf16, int B, int V, int ld, int32_t* d_out,
                           void* stream) {
  if (B <= 0 || V <= 0) return mesw_fail(MESW_ERR_VALUE, "argmax: bad shape");
  mesw_launch(argmax_kernel, dim3(B), dim3(1024), 0, (cudaStream_t)stream, d_logits, is_bf16, V, ld, d_out);
  return mesw_check_launch("argmax");
}

extern "C" int mesw_pack_x(const uint16_t* d_x, int B, int m, int ldx, uint16_t* d_xc, float* d_corr, int corr_ld,
                           void* stream) {
  if (B <= 0 || m <= 0 || ldx < m) return mesw_fail(MESW_ERR_VALUE, "pack_x: bad shape");
  const int NP = (B + 15) & ~15, n_ks = (m + 127) / 128;
  const long long total = (long long)n_ks * NP * 16;
  if (d_corr && corr_ld < n_ks) return mesw_fail(MESW_ERR_VALUE, "pack_x: corr_ld too small");
  mesw_launch(pack_x_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, d_x, B, m, ldx, d_xc,
              NP, n_ks, d_corr, corr_ld, (const int32_t*)nullptr);
  return mesw_check_launch("pack_x");
}

extern "C" int mesw_pack_x_gather(const uint16_t* d_x, int ldx, const int32_t* d_src, int rows, int m, uint16_t* d_xc,
                                  float* d_corr, int corr_ld, void* stream) {
  if (rows <= 0 || m <= 0 || ldx < m || !d_src) return mesw_fail(MESW_ERR_VALUE, "pack_x_gather: bad arguments");
  const int NP = (rows + 15) & ~15, n_ks = (m + 127) / 128;
  const long long total = (long long)n_ks * NP * 16;
  if (d_corr && corr_ld < n_ks) return mesw_fail(MESW_ERR_VALUE, "pack_x_gather: corr_ld too small");
  mesw_launch(pack_x_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, d_x, rows, m,
              ldx, d_xc, NP, n_ks, d_corr, corr_ld, d_src);
  return mesw_check_launch("pack_x_gather");
}

extern "C" int mesw_unpack_x(const uint16_t* d_xc, int B, int m, uint16_t* d_y, int ldy, void* stream) {
  if (B <= 0 || m <= 0 || ldy < m) return mesw_fail(MESW_ERR_VALUE, "unpack_x: bad shape");
  const int NP = (B + 15) & ~15;
  const long long total = (long long)B * m;
  mesw_launch(unpack_x_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, d_xc, B, m, NP, d_y, ldy);
  return mesw_check_launch("unpack_x");
}
