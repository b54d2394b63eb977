// f2: delta compression on the GPU, bit-exact with the reference's compress_layer
// (compress.py:178-215, metric "reconstruction"; restated in oracle/compress.py):
//   steps0 = init_step_sizes(delta)            per column: max|x|/Q_P in f64 (1-bit: mean|x|,
//                                              rows accumulated in order in f64), 0 -> TINY_F32
//   codes0 = clip(round_half_away(x/s))        f64 division (quant.py:111-120)
//   score_i = f32(E_i * sum_j (x - q*s)^2)     f64, numpy's pairwise order over j (salient.py:119)
//   S = top-k(score)                           ties -> lower index (stable argsort), sorted
//   steps = init_step_sizes(delta[~S]); codes of ~S rows re-quantised, S rows 0
//   rows = f16(delta[S]) (RNE, overflow -> inf); codes packed LSB-first per column run
// One thread per column / row / output byte: the passes are light next to the reference's
// host time (~7 s per 4096x14336 layer) and every reduction keeps the reference's order.

#include <float.h>
#include <math.h>

#include "mesw_common.cuh"
#include "mesw_host.h"

namespace mesw {

constexpr float kTinyF32 = 1.1754944e-38f;  // numerics.py:26

__device__ __forceinline__ void code_range_dev(int bits, int& qn, int& qp) {
  if (bits == 1) { qn = 1; qp = 1; return; }
  qn = 1 << (bits - 1);
  qp = (1 << (bits - 1)) - 1;
}

// quant.quantize_codes for one element (quant.py:111-120)
__device__ __forceinline__ int quantize_one(float x, float s, int bits) {
  if (bits == 1) return x < 0.f ? -1 : 1;
  int qn, qp;
  code_range_dev(bits, qn, qp);
  const double u = (double)x / (double)s;
  double r = copysign(floor(fabs(u) + 0.5), u);
  if (r < -qn) r = -qn;
  if (r > qp) r = qp;
  return (int)r;
}

// init_step_sizes over the rows with skip[i] == 0 (skip == nullptr: all rows)
__global__ void steps_kernel(const float* __restrict__ x, int m, int n, int bits, const uint8_t* __restrict__ skip,
                             int count, float* __restrict__ steps) {
  pdl_trigger();
  pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double raw;
  if (count == 0) {
    raw = 0.0;
  } else if (bits == 1) {
    double acc = 0.0;  // numpy mean(axis=0, dtype=f64): rows accumulated in order
    for (int i = 0; i < m; ++i)
      if (!skip || !skip[i]) acc += (double)fabsf(x[(size_t)i * n + j]);
    raw = acc / (double)count;
  } else {
    float mx = 0.f;
    for (int i = 0; i < m; ++i)
      if (!skip || !skip[i]) mx = fmaxf(mx, fabsf(x[(size_t)i * n + j]));
    int qn, qp;
    code_range_dev(bits, qn, qp);
    raw = (double)mx / (double)qp;
  }
  steps[j] = raw <= 0.0 ? kTinyF32 : (float)raw;
}

// squared reconstruction error of element j of row `row` (f64), as numpy forms it
__device__ __forceinline__ double err2(const float* __restrict__ row, const float* __restrict__ steps0, int j, int bits) {
  const float s = steps0[j];
  const float approx = (float)quantize_one(row[j], s, bits) * s;  // dequantize: f32 product
  const double e = (double)row[j] - (double)approx;
  return e * e;
}

// numpy pairwise_sum over [lo, lo + len) of err2 (loops_utils.h: 8-way blocks <= 128, split
// at a multiple of 8); explicit stack instead of recursion
__device__ double pairwise_err(const float* __restrict__ row, const float* __restrict__ steps0, int n, int bits) {
  // iterative post-order over the split tree: (lo, len, state)
  int st_lo[24], st_len[24], st_state[24];
  double st_left[24];
  int sp = 0;
  st_lo[0] = 0; st_len[0] = n; st_state[0] = 0;
  double ret = 0.0;
  for (;;) {
    const int lo = st_lo[sp], len = st_len[sp];
    if (len <= 128) {  // leaf
      double res;
      if (len < 8) {
        res = 0.0;
        for (int i = 0; i < len; ++i) res += err2(row, steps0, lo + i, bits);
      } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = err2(row, steps0, lo + j, bits);
        int i = 8;
        for (; i < len - (len % 8); i += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) r[j] += err2(row, steps0, lo + i + j, bits);
        }
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < len; ++i) res += err2(row, steps0, lo + i, bits);
      }
      // return res to the parent
      for (;;) {
        if (sp == 0) return res;
        --sp;
        if (st_state[sp] == 1) {  // left child done: run the right child
          st_left[sp] = res;
          st_state[sp] = 2;
          int n2 = st_len[sp] / 2;
          n2 -= n2 % 8;
          ++sp;
          st_lo[sp] = st_lo[sp - 1] + n2;
          st_len[sp] = st_len[sp - 1] - n2;
          st_state[sp] = 0;
          break;
        }
        res = st_left[sp] + res;  // right child done
      }
      continue;
    }
    // internal node: descend left
    int n2 = len / 2;
    n2 -= n2 % 8;
    st_state[sp] = 1;
    ++sp;
    st_lo[sp] = lo;
    st_len[sp] = n2;
    st_state[sp] = 0;
  }
  return ret;
}

__global__ void score_kernel(const float* __restrict__ x, int m, int n, int bits, const float* __restrict__ steps0,
                             const float* __restrict__ energy, float* __restrict__ scores) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double row_err = pairwise_err(x + (size_t)i * n, steps0, n, bits);
  scores[i] = (float)((double)energy[i] * row_err);
}

// top-k of scores (descending, ties -> lower index), indices ascending; one block
__global__ void topk_kernel(const float* __restrict__ scores, int m, int k, uint8_t* __restrict__ sel,
                            int32_t* __restrict__ idx_out) {
  pdl_trigger();
  pdl_wait();
  __shared__ float bv[32];
  __shared__ int bi[32];
  __shared__ int pick;
  for (int i = threadIdx.x; i < m; i += blockDim.x) sel[i] = 0;
  __syncthreads();
  for (int r = 0; r < k; ++r) {
    float best = -INFINITY;
    int bidx = 0x7fffffff;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      if (sel[i]) continue;
      const float v = scores[i];
      if (v > best || (v == best && i < bidx)) { best = v; bidx = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const float v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (v2 > best || (v2 == best && i2 < bidx)) { best = v2; bidx = i2; }
    }
    if ((threadIdx.x & 31) == 0) { bv[threadIdx.x >> 5] = best; bi[threadIdx.x >> 5] = bidx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      float b = bv[0];
      int ix = bi[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (bv[w] > b || (bv[w] == b && bi[w] < ix)) { b = bv[w]; ix = bi[w]; }
      if (ix == 0x7fffffff) {  // only -inf / NaN left: lowest unselected index
        for (ix = 0; ix < m && sel[ix]; ++ix) {}
      }
      sel[ix] = 1;
      pick = ix;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {  // ascending indices
    int c = 0;
    for (int i = 0; i < m && c < k; ++i)
      if (sel[i]) idx_out[c++] = i;
  }
  (void)pick;
}

// packed byte `b` of column j's run (LSB-first bit stream, quant.py:195-213)
__global__ void pack_kernel(const float* __restrict__ x, int m, int n, int bits, const float* __restrict__ steps,
                            const uint8_t* __restrict__ sel, uint8_t* __restrict__ packed, int run) {
  pdl_trigger();
  pdl_wait();
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)run * n) return;
  const int j = (int)(t / run), b = (int)(t % run);
  int qn, qp;
  code_range_dev(bits, qn, qp);
  uint32_t byte = 0;
  int last_row = -1;
  uint32_t u = 0;
  for (int bit = 0; bit < 8; ++bit) {
    const long long g = (long long)b * 8 + bit;
    const int i = (int)(g / bits);
    if (i >= m) break;
    if (i != last_row) {
      const int q = sel[i] ? 0 : quantize_one(x[(size_t)i * n + j], steps[j], bits);
      u = bits == 1 ? (uint32_t)((q + 1) / 2) : (uint32_t)(q + qn);
      last_row = i;
    }
    byte |= ((u >> (int)(g % bits)) & 1u) << bit;
  }
  packed[(size_t)j * run + b] = (uint8_t)byte;
}

__global__ void salient_rows_kernel(const float* __restrict__ x, int n, const int32_t* __restrict__ idx, int k,
                                    uint16_t* __restrict__ rows) {
  pdl_trigger();
  pdl_wait();
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)k * n) return;
  const int r = (int)(t / n), j = (int)(t % n);
  rows[t] = __half_as_ushort(__float2half_rn(x[(size_t)idx[r] * n + j]));
}

}  // namespace mesw

using namespace mesw;

extern "C" uint64_t mesw_compress_workspace_bytes(uint32_t m, uint32_t n) {
  return ((uint64_t)n * 4 + 255) / 256 * 256 + ((uint64_t)m * 4 + 255) / 256 * 256 + ((uint64_t)m + 255) / 256 * 256;
}

extern "C" int mesw_compress_layer(const float* d_delta, uint32_t m, uint32_t n, const float* d_energy, uint32_t bits,
                                   uint32_t k, float* d_steps, int32_t* d_sal_idx, uint16_t* d_sal_rows,
                                   uint8_t* d_packed, void* d_workspace, uint64_t workspace_bytes, void* stream) {
  if (m == 0 || n == 0) return mesw_fail(MESW_ERR_VALUE, "compress: empty matrix");
  if (!(bits == 1 || bits == 2 || bits == 3 || bits == 4 || bits == 8))
    return mesw_fail(MESW_ERR_VALUE, "compress: bits must be one of (1, 2, 3, 4, 8)");
  if (k > m) return mesw_fail(MESW_ERR_VALUE, "compress: salient_k exceeds the input channels");
  if (bits == 1 && k > 0)
    return mesw_fail(MESW_ERR_VALUE, "compress: 1-bit codes cannot hold the zero code of salient rows");
  if (!d_delta || !d_energy || !d_steps || !d_packed || (k && (!d_sal_idx || !d_sal_rows)))
    return mesw_fail(MESW_ERR_VALUE, "compress: null buffer");
  if (!d_workspace || workspace_bytes < mesw_compress_workspace_bytes(m, n))
    return mesw_fail(MESW_ERR_VALUE, "compress: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* ws = reinterpret_cast<uint8_t*>(d_workspace);
  float* steps0 = reinterpret_cast<float*>(ws);
  float* scores = reinterpret_cast<float*>(ws + ((uint64_t)n * 4 + 255) / 256 * 256);
  uint8_t* sel = ws + ((uint64_t)n * 4 + 255) / 256 * 256 + ((uint64_t)m * 4 + 255) / 256 * 256;
  const int M = (int)m, N = (int)n, B = (int)bits, K = (int)k;
  cudaError_t e;
#define MESW_CK(x) do { e = (x); if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e)); } while (0)
  MESW_CK(mesw_launch(steps_kernel, dim3((N + 127) / 128), dim3(128), 0, s, d_delta, M, N, B,
                      (const uint8_t*)nullptr, M, steps0));
  MESW_CK(mesw_launch(score_kernel, dim3((M + 127) / 128), dim3(128), 0, s, d_delta, M, N, B, (const float*)steps0,
                      d_energy, scores));
  MESW_CK(mesw_launch(topk_kernel, dim3(1), dim3(1024), 0, s, (const float*)scores, M, K, sel, d_sal_idx));
  MESW_CK(mesw_launch(steps_kernel, dim3((N + 127) / 128), dim3(128), 0, s, d_delta, M, N, B, (const uint8_t*)sel,
                      M - K, d_steps));
  const int run = (int)(((uint64_t)m * bits + 7) / 8);
  const long long nbytes = (long long)run * n;
  MESW_CK(mesw_launch(pack_kernel, dim3((unsigned)((nbytes + 255) / 256)), dim3(256), 0, s, d_delta, M, N, B,
                      (const float*)d_steps, (const uint8_t*)sel, d_packed, run));
  if (K > 0)
    MESW_CK(mesw_launch(salient_rows_kernel, dim3((unsigned)(((long long)K * N + 255) / 256)), dim3(256), 0, s,
                        d_delta, N, (const int32_t*)d_sal_idx, K, d_sal_rows));
#undef MESW_CK
  return mesw_check_launch("compress_layer");
}
