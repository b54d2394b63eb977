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

// fl64(x / s) for f32 x, s from a per-column reciprocal r = RN(1/s): u0 = RN(x r), the
// exact residual e = x - u0 s (one FMA), u = RN(u0 + e r).  The pre-rounding error is
// ~2^-106 relative while a quotient of two 24-bit significands lies >= ~2^-77 (relative)
// from any f64 rounding midpoint, so u is the correctly rounded quotient -- the f64
// division of the reference (quant.py:118) at 3 FP64 ops per element.
__device__ __forceinline__ double quot_f64(float x, double sd, double r) {
  const double xd = (double)x;
  const double u0 = __dmul_rn(xd, r);
  const double e = __fma_rn(-u0, sd, xd);
  return __fma_rn(e, r, u0);
}

__device__ __forceinline__ int quantize_one_r(float x, double sd, double r, int bits) {
  if (bits == 1) return x < 0.f ? -1 : 1;
  int qn, qp;
  code_range_dev(bits, qn, qp);
  const double u = quot_f64(x, sd, r);
  double q = copysign(floor(fabs(u) + 0.5), u);
  if (q < -qn) q = -qn;
  if (q > qp) q = qp;
  return (int)q;
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

// ------------------------------------------------------------------------------------
// f3: step-size distillation (compress.py:331-378, toylm.py:357-447; oracle/distill.py).
// The reductions and updates keep the reference's f64 operation order with explicit
// _rn intrinsics (no FMA contraction), so given the same inputs they are bit-exact.

namespace mesw {

// W_eff = base + reconstruct(steps): codes * steps in f32 (quant.dequantize), salient rows
// replaced by their fp16-rounded values (toylm.py:379-384); base == nullptr -> reconstruction.
// Thread per column (reciprocal of its step once) over a kRecRows-row strip; warps read
// 128 contiguous bytes per row.
constexpr int kRecRows = 64;

__global__ void __launch_bounds__(256) ste_reconstruct_kernel(const float* __restrict__ delta, int m, int n,
                                                              const float* __restrict__ steps, int bits,
                                                              const int32_t* __restrict__ row_slot,
                                                              const float* __restrict__ sal_rows,
                                                              const float* __restrict__ base, float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i0 = blockIdx.y * kRecRows, i1 = min(m, i0 + kRecRows);
  if (j >= n) return;
  const float sf = steps[j];
  const double sd = (double)sf, r = __drcp_rn(sd);
  for (int ib = i0; ib < i1; ib += 8) {  // batch the loads of 8 rows ahead of the math
    float xv[8], bv[8];
    int rs[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = ib + q;
      const bool ok = i < i1;
      const size_t t = (size_t)(ok ? i : i0) * n + j;
      xv[q] = delta[t];
      bv[q] = base ? base[t] : 0.f;
      rs[q] = (row_slot && ok) ? row_slot[i] : -1;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = ib + q;
      if (i >= i1) break;
      const float v = rs[q] >= 0 ? sal_rows[(size_t)rs[q] * n + j]
                                 : __fmul_rn((float)quantize_one_r(xv[q], sd, r, bits), sf);
      out[(size_t)i * n + j] = base ? __fadd_rn(bv[q], v) : v;
    }
  }
}

// grad[j] = f32(sum_i up[i,j] * local[i,j]) in f64, rows in order (numpy axis-0 sum);
// local = round_half_away(u) - u inside the clamp range, -Q_N / Q_P outside, sign(x)
// for 1-bit (quant.py:142-169); salient rows (row_slot >= 0) have zero upstream.
// A CTA owns kGC columns: all 256 threads compute a kGR-row tile of f64 products from
// coalesced loads (the next tile's loads in flight during the fold), then one thread per
// column folds the tile into its running sum in row order (the only serial part).
// Measured (tools/distill_bench.py, 4096x14336): 215 us; barrier- and latency-bound
// (ncu: FP64 pipe ~16% active) -- a dedicated folder warp with a double-buffered ring
// measured slower (334 us).
constexpr int kGC = 16, kGR = 64, kGT = 256, kGQ = kGR / (kGT / kGC);

__device__ __forceinline__ void ste_grad_load(const float* __restrict__ delta, const float* __restrict__ up,
                                              const int32_t* __restrict__ row_slot, int m, int n, int i0, int rl,
                                              int j, float* xs, float* gs) {
#pragma unroll
  for (int q = 0; q < kGQ; ++q) {
    const int i = i0 + rl + q * (kGT / kGC);
    const bool ok = i < m && j < n;
    xs[q] = ok ? delta[(size_t)i * n + j] : 0.f;
    gs[q] = ok ? up[(size_t)i * n + j] : 0.f;
    if (ok && row_slot && row_slot[i] >= 0) gs[q] = 0.f;
  }
}

__global__ void __launch_bounds__(kGT) ste_grad_kernel(const float* __restrict__ delta, int m, int n,
                                                       const float* __restrict__ steps, int bits,
                                                       const int32_t* __restrict__ row_slot,
                                                       const float* __restrict__ up, float* __restrict__ grad) {
  pdl_trigger();
  pdl_wait();
  __shared__ double prod[kGR][kGC + 1];
  const int c = threadIdx.x % kGC, rl = threadIdx.x / kGC;  // column lane, row lane
  const int j = blockIdx.x * kGC + c;
  int qn, qp;
  code_range_dev(bits, qn, qp);
  const double s = j < n ? (double)steps[j] : 1.0, rcp = __drcp_rn(s);
  double acc = 0.0;
  float xs[kGQ], gs[kGQ];
  ste_grad_load(delta, up, row_slot, m, n, 0, rl, j, xs, gs);
  for (int i0 = 0; i0 < m; i0 += kGR) {
#pragma unroll
    for (int q = 0; q < kGQ; ++q) {
      const int r = rl + q * (kGT / kGC);
      double local;
      if (bits == 1) {
        local = xs[q] < 0.f ? -1.0 : 1.0;
      } else {
        const double u = quot_f64(xs[q], s, rcp);
        local = __dsub_rn(copysign(floor(__dadd_rn(fabs(u), 0.5)), u), u);
        if (u < -qn) local = -(double)qn;
        if (u > qp) local = (double)qp;
      }
      prod[r][c] = __dmul_rn((double)gs[q], local);
    }
    __syncthreads();
    if (i0 + kGR < m) ste_grad_load(delta, up, row_slot, m, n, i0 + kGR, rl, j, xs, gs);
    if (threadIdx.x < kGC) {
      const int rn = min(kGR, m - i0);
      int r = 0;
      for (; r + 16 <= rn; r += 16) {  // 16 smem loads in flight, then the in-order adds
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = prod[r + q][c];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc = (i0 == 0 && r + q == 0) ? v[0] : __dadd_rn(acc, v[q]);
      }
      for (; r < rn; ++r) acc = (i0 == 0 && r == 0) ? prod[0][c] : __dadd_rn(acc, prod[r][c]);
    }
    __syncthreads();
  }
  if (threadIdx.x < kGC && j < n) grad[j] = (float)acc;
}

// AdamW rule, weight decay 0 (compress.py:288-302), then the positive clamp (compress.py:375)
__global__ void adam_kernel(float* __restrict__ p, double* __restrict__ m1, double* __restrict__ v1,
                            const float* __restrict__ grad, int n, double lr, double b1, double omb1, double b2,
                            double omb2, double bc1, double bc2, double eps, float floor_v) {
  pdl_trigger();
  pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double g = (double)grad[j];
  const double m = __dadd_rn(__dmul_rn(b1, m1[j]), __dmul_rn(omb1, g));
  const double v = __dadd_rn(__dmul_rn(b2, v1[j]), __dmul_rn(__dmul_rn(omb2, g), g));
  m1[j] = m;
  v1[j] = v;
  const double mh = __ddiv_rn(m, bc1), vh = __ddiv_rn(v, bc2);
  const double upd = __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps));
  const float np_ = (float)__dsub_rn((double)p[j], upd);
  p[j] = np_ > floor_v ? np_ : (np_ == np_ ? floor_v : np_);  // np.maximum (NaN propagates)
}

}  // namespace mesw

using namespace mesw;

extern "C" int mesw_ste_reconstruct(const float* d_delta, uint32_t m, uint32_t n, const float* d_steps, uint32_t bits,
                                    const int32_t* d_row_slot, const float* d_sal_rows, const float* d_base,
                                    float* d_out, void* stream) {
  if (m == 0 || n == 0 || !d_delta || !d_steps || !d_out) return mesw_fail(MESW_ERR_VALUE, "ste_reconstruct: bad args");
  if (d_row_slot && !d_sal_rows) return mesw_fail(MESW_ERR_VALUE, "ste_reconstruct: salient rows missing");
  cudaError_t e = mesw_launch(ste_reconstruct_kernel, dim3((n + 255) / 256, (m + kRecRows - 1) / kRecRows), dim3(256), 0,
                              (cudaStream_t)stream, d_delta, (int)m, (int)n, d_steps, (int)bits, d_row_slot, d_sal_rows,
                              d_base, d_out);
  if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
  return mesw_check_launch("ste_reconstruct");
}

extern "C" int mesw_ste_step_grad(const float* d_delta, uint32_t m, uint32_t n, const float* d_steps, uint32_t bits,
                                  const int32_t* d_row_slot, const float* d_upstream, float* d_grad, void* stream) {
  if (m == 0 || n == 0 || !d_delta || !d_steps || !d_upstream || !d_grad)
    return mesw_fail(MESW_ERR_VALUE, "ste_step_grad: bad args");
  cudaError_t e = mesw_launch(ste_grad_kernel, dim3((n + kGC - 1) / kGC), dim3(kGT), 0, (cudaStream_t)stream, d_delta,
                              (int)m, (int)n, d_steps, (int)bits, d_row_slot, d_upstream, d_grad);
  if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
  return mesw_check_launch("ste_step_grad");
}

extern "C" int mesw_adam_step(float* d_steps, double* d_m, double* d_v, const float* d_grad, uint32_t n, double lr,
                              double beta1, double beta2, double eps, double bias_corr1, double bias_corr2,
                              float step_floor, void* stream) {
  if (n == 0 || !d_steps || !d_m || !d_v || !d_grad) return mesw_fail(MESW_ERR_VALUE, "adam_step: bad args");
  cudaError_t e = mesw_launch(adam_kernel, dim3((n + 255) / 256), dim3(256), 0, (cudaStream_t)stream, d_steps, d_m,
                              d_v, d_grad, (int)n, lr, beta1, 1.0 - beta1, beta2, 1.0 - beta2, bias_corr1, bias_corr2,
                              eps, step_floor);
  if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
  return mesw_check_launch("adam_step");
}

extern "C" int mesw_quantize_pack(const float* d_delta, uint32_t m, uint32_t n, const float* d_steps, uint32_t bits,
                                  const uint8_t* d_salient_mask, uint8_t* d_packed, void* stream) {
  if (m == 0 || n == 0 || !d_delta || !d_steps || !d_salient_mask || !d_packed)
    return mesw_fail(MESW_ERR_VALUE, "quantize_pack: bad args");
  const int run = (int)(((uint64_t)m * bits + 7) / 8);
  const long long nbytes = (long long)run * n;
  cudaError_t e = mesw_launch(pack_kernel, dim3((unsigned)((nbytes + 255) / 256)), dim3(256), 0, (cudaStream_t)stream,
                              d_delta, (int)m, (int)n, (int)bits, d_steps, d_salient_mask, d_packed, run);
  if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
  return mesw_check_launch("quantize_pack");
}
