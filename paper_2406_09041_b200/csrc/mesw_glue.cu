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
  const int b = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(table + (size_t)ids[b] * H);
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)b * ld_out);
  for (int i = threadIdx.x; i < H / 8; i += blockDim.x) dst[i] = src[i];
}

// y = x * rsqrt(mean(x^2) + eps) * w   (one CTA per token)
__global__ void rmsnorm_kernel(const uint16_t* __restrict__ x, int ldx, const uint16_t* __restrict__ w,
                               int H, float eps, uint16_t* __restrict__ y, int ldy) {
  __shared__ float red[32];
  const uint16_t* xr = x + (size_t)blockIdx.x * ldx;
  float ss = 0.f;
  for (int i = threadIdx.x * 2; i < H; i += blockDim.x * 2) {
    const uint32_t v = *reinterpret_cast<const uint32_t*>(xr + i);
    const float a = bf16_lo(v), b = bf16_hi(v);
    ss = fmaf(a, a, fmaf(b, b, ss));
  }
  const float tot = block_sum(ss, red);
  const float r = rsqrtf(tot / (float)H + eps);
  uint16_t* yr = y + (size_t)blockIdx.x * ldy;
  for (int i = threadIdx.x * 2; i < H; i += blockDim.x * 2) {
    const uint32_t v = *reinterpret_cast<const uint32_t*>(xr + i);
    const uint32_t g = *reinterpret_cast<const uint32_t*>(w + i);
    __nv_bfloat162 o = __floats2bfloat162_rn(bf16_lo(v) * r * bf16_lo(g), bf16_hi(v) * r * bf16_hi(g));
    *reinterpret_cast<__nv_bfloat162*>(yr + i) = o;
  }
}

// RoPE (rotate-half pairs (i, i+D/2)) on q in place and on k, then append k and v
// to the cache at each token's position.  qkv row: [q heads | k heads | v heads].
// grid (B, n_heads + n_kv_heads), block D/2.
__global__ void rope_append_kernel(uint16_t* __restrict__ qkv, int ld_qkv, const int32_t* __restrict__ pos,
                                   int n_heads, int n_kv, int D, float theta,
                                   uint16_t* __restrict__ kc, uint16_t* __restrict__ vc, int ctx_max) {
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

// GQA decode attention: one CTA per (token, kv head); G = n_heads / n_kv query heads
// share the kv head.  scores in smem (f32), softmax per head, then P.V.
// block = D threads (D = 128), dynamic smem = G * ctx_max floats + G*D floats.
template <int G>
__global__ void attn_decode_kernel(const uint16_t* __restrict__ q, int ld_q, const uint16_t* __restrict__ kc,
                                   const uint16_t* __restrict__ vc, const int32_t* __restrict__ len,
                                   int n_kv, int D, int ctx_max, float scale, uint16_t* __restrict__ out,
                                   int ld_out) {
  extern __shared__ float sm[];
  __shared__ float red[32];
  const int b = blockIdx.x, g = blockIdx.y, tid = threadIdx.x;
  const int L = len[b];
  float* qs = sm;                 // [G][D]
  float* sc = sm + G * D;         // [G][ctx_max]
  for (int i = tid; i < G * D; i += blockDim.x) {
    const int hh = i / D, d = i % D;
    qs[i] = bf16_to_f32(q[(size_t)b * ld_q + (size_t)(g * G + hh) * D + d]) * scale;
  }
  __syncthreads();
  const size_t kv_stride = (size_t)n_kv * D;
  const uint16_t* kb = kc + ((size_t)b * ctx_max * n_kv + g) * D;
  const uint16_t* vb = vc + ((size_t)b * ctx_max * n_kv + g) * D;
  // scores: warp per position, lanes over D
  const int lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  for (int t = w; t < L; t += nw) {
    const uint16_t* kr = kb + (size_t)t * kv_stride;
    float acc[G];
#pragma unroll
    for (int hh = 0; hh < G; ++hh) acc[hh] = 0.f;
    for (int d = lane * 2; d < D; d += 64) {
      const uint32_t kv2 = *reinterpret_cast<const uint32_t*>(kr + d);
      const float k0 = bf16_lo(kv2), k1 = bf16_hi(kv2);
#pragma unroll
      for (int hh = 0; hh < G; ++hh) acc[hh] = fmaf(qs[hh * D + d], k0, fmaf(qs[hh * D + d + 1], k1, acc[hh]));
    }
#pragma unroll
    for (int hh = 0; hh < G; ++hh) {
      const float s = warp_sum(acc[hh]);
      if (lane == 0) sc[hh * ctx_max + t] = s;
    }
  }
  __syncthreads();
  // softmax per head (block-wide, fixed order)
  for (int hh = 0; hh < G; ++hh) {
    float mx = -INFINITY;
    for (int t = tid; t < L; t += blockDim.x) mx = fmaxf(mx, sc[hh * ctx_max + t]);
    mx = block_max(mx, red);
    float sum = 0.f;
    for (int t = tid; t < L; t += blockDim.x) {
      const float e = __expf(sc[hh * ctx_max + t] - mx);
      sc[hh * ctx_max + t] = e;
      sum += e;
    }
    sum = block_sum(sum, red);
    const float inv = 1.f / sum;
    for (int t = tid; t < L; t += blockDim.x) sc[hh * ctx_max + t] *= inv;
    __syncthreads();
  }
  // out[h][d] = sum_t p[h][t] v[t][d]; thread = dim d
  for (int d = tid; d < D; d += blockDim.x) {
    float acc[G];
#pragma unroll
    for (int hh = 0; hh < G; ++hh) acc[hh] = 0.f;
    for (int t = 0; t < L; ++t) {
      const float vv = bf16_to_f32(vb[(size_t)t * kv_stride + d]);
#pragma unroll
      for (int hh = 0; hh < G; ++hh) acc[hh] = fmaf(sc[hh * ctx_max + t], vv, acc[hh]);
    }
#pragma unroll
    for (int hh = 0; hh < G; ++hh)
      out[(size_t)b * ld_out + (size_t)(g * G + hh) * D + d] = __bfloat16_as_ushort(__float2bfloat16_rn(acc[hh]));
  }
}

// out = silu(gate) * up, gate/up halves of a [B][2I] row.
__global__ void swiglu_kernel(const uint16_t* __restrict__ gu, int ld_gu, int I, uint16_t* __restrict__ out,
                              int ld_out) {
  const int b = blockIdx.y;
  const uint16_t* r = gu + (size_t)b * ld_gu;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2; i < I; i += gridDim.x * blockDim.x * 2) {
    const uint32_t g2 = *reinterpret_cast<const uint32_t*>(r + i);
    const uint32_t u2 = *reinterpret_cast<const uint32_t*>(r + I + i);
    const float g0 = bf16_lo(g2), g1 = bf16_hi(g2);
    const float s0 = g0 / (1.f + __expf(-g0)), s1 = g1 / (1.f + __expf(-g1));
    *reinterpret_cast<__nv_bfloat162*>(out + (size_t)b * ld_out + i) =
        __floats2bfloat162_rn(s0 * bf16_lo(u2), s1 * bf16_hi(u2));
  }
}

// argmax over a row with ties to the lowest index (np.argmax); f32 or bf16 logits.
__global__ void argmax_kernel(const void* __restrict__ logits, int is_bf16, int V, int ld,
                              int32_t* __restrict__ out) {
  __shared__ float bv[32];
  __shared__ int bi[32];
  const int b = blockIdx.x;
  float best = -INFINITY;
  int bidx = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = is_bf16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(logits)[(size_t)b * ld + i])
                            : reinterpret_cast<const float*>(logits)[(size_t)b * ld + i];
    if (bidx == 0x7fffffff || v > best) { best = v; bidx = i; }  // i ascending: ties keep the first
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

// Advance every request by one position (pos += 1, len = pos + 1); a request that
// reaches the end of its cache window wraps back to `wrap_to` (bench steady state).
__global__ void advance_kernel(int32_t* __restrict__ pos, int32_t* __restrict__ len, int B, int ctx_max,
                               int wrap_to) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int p = pos[b] + 1;
  if (p >= ctx_max) p = wrap_to;
  pos[b] = p;
  len[b] = p + 1;
}

}  // namespace mesw

using namespace mesw;

extern "C" int mesw_advance_positions(int32_t* d_pos, int32_t* d_len, int B, int ctx_max, int wrap_to,
                                      void* stream) {
  if (B <= 0 || wrap_to < 0 || wrap_to >= ctx_max) return mesw_fail(MESW_ERR_VALUE, "advance: bad args");
  advance_kernel<<<(B + 127) / 128, 128, 0, (cudaStream_t)stream>>>(d_pos, d_len, B, ctx_max, wrap_to);
  return mesw_check_launch("advance_positions");
}

extern "C" int mesw_embed(const int32_t* d_ids, int B, const uint16_t* d_table, int H, uint16_t* d_out,
                          int ld_out, void* stream) {
  if (B <= 0 || H % 8) return mesw_fail(MESW_ERR_VALUE, "embed: H must be a multiple of 8");
  embed_kernel<<<B, 128, 0, (cudaStream_t)stream>>>(d_ids, d_table, H, d_out, ld_out);
  return mesw_check_launch("embed");
}

extern "C" int mesw_rmsnorm(const uint16_t* d_x, int ldx, const uint16_t* d_w, int B, int H, float eps,
                            uint16_t* d_y, int ldy, void* stream) {
  if (B <= 0 || H % 2) return mesw_fail(MESW_ERR_VALUE, "rmsnorm: bad shape");
  rmsnorm_kernel<<<B, 256, 0, (cudaStream_t)stream>>>(d_x, ldx, d_w, H, eps, d_y, ldy);
  return mesw_check_launch("rmsnorm");
}

extern "C" int mesw_rope_append(uint16_t* d_qkv, int ld_qkv, const int32_t* d_pos, int B, int n_heads,
                                int n_kv, int head_dim, float theta, uint16_t* d_kcache, uint16_t* d_vcache,
                                int ctx_max, void* stream) {
  if (B <= 0 || head_dim % 2 || head_dim > 2048) return mesw_fail(MESW_ERR_VALUE, "rope: bad shape");
  dim3 grid(B, n_heads + n_kv);
  rope_append_kernel<<<grid, head_dim / 2, 0, (cudaStream_t)stream>>>(d_qkv, ld_qkv, d_pos, n_heads, n_kv,
                                                                      head_dim, theta, d_kcache, d_vcache,
                                                                      ctx_max);
  return mesw_check_launch("rope_append");
}

extern "C" int mesw_attention_decode(const uint16_t* d_q, int ld_q, const uint16_t* d_kcache,
                                     const uint16_t* d_vcache, const int32_t* d_len, int B, int n_heads,
                                     int n_kv, int head_dim, int ctx_max, uint16_t* d_out, int ld_out,
                                     void* stream) {
  if (B <= 0 || n_kv <= 0 || n_heads % n_kv || head_dim % 64)
    return mesw_fail(MESW_ERR_VALUE, "attention: bad shape");
  const int G = n_heads / n_kv;
  const size_t smem = (size_t)G * (ctx_max + head_dim) * sizeof(float);
  if (smem > 200 * 1024) return mesw_fail(MESW_ERR_UNSUPPORTED, "attention: context too long");
  const float scale = 1.0f / sqrtf((float)head_dim);
  dim3 grid(B, n_kv);
  cudaStream_t s = (cudaStream_t)stream;
#define MESW_ATTN(GG)                                                                                  \
  case GG: {                                                                                           \
    static bool cfg = false;                                                                           \
    if (!cfg) {                                                                                        \
      cudaFuncSetAttribute(attn_decode_kernel<GG>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                           200 * 1024);                                                                \
      cfg = true;                                                                                      \
    }                                                                                                  \
    attn_decode_kernel<GG><<<grid, 128, smem, s>>>(d_q, ld_q, d_kcache, d_vcache, d_len, n_kv, head_dim, \
                                                   ctx_max, scale, d_out, ld_out);                     \
    break;                                                                                             \
  }
  switch (G) {
    MESW_ATTN(1)
    MESW_ATTN(2)
    MESW_ATTN(4)
    MESW_ATTN(8)
    default:
      return mesw_fail(MESW_ERR_UNSUPPORTED, "attention: heads per kv head must be 1, 2, 4 or 8");
  }
#undef MESW_ATTN
  return mesw_check_launch("attention_decode");
}

extern "C" int mesw_swiglu(const uint16_t* d_gu, int ld_gu, int B, int I, uint16_t* d_out, int ld_out,
                           void* stream) {
  if (B <= 0 || I % 2) return mesw_fail(MESW_ERR_VALUE, "swiglu: bad shape");
  dim3 grid((I / 2 + 255) / 256 < 64 ? (I / 2 + 255) / 256 : 64, B);
  swiglu_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_gu, ld_gu, I, d_out, ld_out);
  return mesw_check_launch("swiglu");
}

extern "C" int mesw_argmax(const void* d_logits, int is_bf16, int B, int V, int ld, int32_t* d_out,
                           void* stream) {
  if (B <= 0 || V <= 0) return mesw_fail(MESW_ERR_VALUE, "argmax: bad shape");
  argmax_kernel<<<B, 1024, 0, (cudaStream_t)stream>>>(d_logits, is_bf16, V, ld, d_out);
  return mesw_check_launch("argmax");
}
