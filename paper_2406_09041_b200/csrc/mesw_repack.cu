// K1 loader kernels (MESW packed codes / bf16 weights -> device fragment layouts)
// and K6 debug kernels (device layouts -> reference-orientation dense arrays).
//
// Reference semantics: quant.unpack_codes (quant.py:216-236) for the code
// stream, CompressedDelta.reconstruct (compress.py:115-121) for the dense
// delta.  See include/mesw.h for the layouts.

#include "mesw_common.cuh"
#include "mesw_host.h"
#include "mesw_layout.cuh"

namespace mesw {

// Code of (row i, col j) from a MESW column-major, LSB-first stream.
__device__ __forceinline__ int read_mesw_code(const uint8_t* packed, uint32_t bpc, uint32_t i,
                                              uint32_t j, uint32_t bits) {
  const uint8_t* run = packed + (size_t)j * bpc;
  const uint32_t bit = i * bits;
  const uint32_t byte = bit >> 3, sh = bit & 7;
  uint32_t win = run[byte];
  if (sh + bits > 8) win |= uint32_t(run[byte + 1]) << 8;
  const int u = (win >> sh) & ((1u << bits) - 1u);
  if (bits == 1) return 2 * u - 1;               // quant.py:232-233
  return u - (1 << (bits - 1));                 // quant.py:234-235
}

__device__ __forceinline__ bool is_salient(const int32_t* idx, uint32_t k, uint32_t i) {
  uint32_t lo = 0, hi = k;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint32_t v = (uint32_t)idx[mid];
    if (v == i) return true;
    if (v < i) lo = mid + 1; else hi = mid;
  }
  return false;
}

// One thread per 32-bit device code word (layout: mesw_layout.cuh).
template <int DB>
__global__ void repack_codes_kernel(const uint8_t* __restrict__ packed, uint32_t m, uint32_t n,
                                    uint32_t bits, const int32_t* __restrict__ sal, uint32_t k,
                                    uint32_t* __restrict__ dst, uint32_t n_ks, uint32_t cg0,
                                    uint32_t n_cg_blk, uint32_t col_base) {
  constexpr int PW = 16 / DB;                  // pairs per word
  constexpr int WPU = kUnitN * kUnitK * DB / 32;  // words per unit
  constexpr int WPC = 2 * DB;                  // words per (kh, m) chunk
  constexpr int OFF = DB == 2 ? 2 : (DB == 4 ? 8 : 128);
  const uint64_t total = (uint64_t)n_cg_blk * n_ks * WPU;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  const int wi = (int)(tid % WPU);
  const uint64_t ul = tid / WPU;  // unit index within the block's column groups
  const uint32_t ks = (uint32_t)(ul % n_ks);
  const uint32_t cg = cg0 + (uint32_t)(ul / n_ks);
  const int w = wi % WPC, mrow = (wi / WPC) % kUnitN, kh = wi / (WPC * kUnitN);
  const uint32_t bpc = (m * bits + 7) / 8;
  const int64_t jl = (int64_t)cg * kUnitN + mrow - col_base;
  uint32_t out = 0;
#pragma unroll
  for (int loc = 0; loc < PW; ++loc) {
    const int p = w * PW + loc;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t i = ks * kUnitK + kh * 64 + 2 * p + h;
      int d = OFF;  // padding and salient rows decode to q = 0
      if (i < m && jl >= 0 && jl < (int64_t)n && !is_salient(sal, k, i))
        d = read_mesw_code(packed, bpc, i, (uint32_t)jl, bits) + OFF;
      out |= uint32_t(d) << (DB * loc + (h ? 16 : 0));
    }
  }
  dst[((uint64_t)cg * n_ks + ks) * WPU + wi] = out;
}

// One thread per 16-byte core-matrix row (8 bf16 along k of one output channel).
__global__ void repack_weight_kernel(const uint16_t* __restrict__ src, uint32_t m, uint32_t n,
                                     uint32_t ld, int transposed, uint8_t* __restrict__ dst,
                                     uint32_t n_ks, uint32_t cg0, uint32_t n_cg_blk,
                                     uint32_t col_base) {
  const uint64_t total = (uint64_t)n_cg_blk * n_ks * kUnitN * (kUnitK / 8);
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  const int kc = (int)(tid % (kUnitK / 8));
  const int mrow = (int)((tid / (kUnitK / 8)) % kUnitN);
  const uint64_t ul = tid / (kUnitN * (kUnitK / 8));
  const uint32_t ks = (uint32_t)(ul % n_ks);
  const uint32_t cg = cg0 + (uint32_t)(ul / n_ks);
  const int64_t jl = (int64_t)cg * kUnitN + mrow - col_base;
  uint32_t v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t pair = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t i = ks * kUnitK + kc * 8 + 2 * q + h;
      uint16_t e = 0;
      if (i < m && jl >= 0 && jl < (int64_t)n)
        e = transposed ? src[(uint64_t)jl * ld + i] : src[(uint64_t)i * ld + jl];
      pair |= uint32_t(e) << (h ? 16 : 0);
    }
    v[q] = pair;
  }
  uint8_t* unit = dst + ((uint64_t)cg * n_ks + ks) * kUnitWBytes;
  *reinterpret_cast<uint4*>(unit + w_byte_in_unit(mrow, kc * 8)) = make_uint4(v[0], v[1], v[2], v[3]);
}

__device__ __forceinline__ int device_code_at(const uint8_t* codes, int db, uint32_t i, uint32_t jg,
                                              uint32_t n_ks) {
  const uint32_t cg = jg / kUnitN, mrow = jg % kUnitN;
  const uint32_t ks = i / kUnitK, kk = i % kUnitK;
  uint32_t wb;
  int bit;
  code_loc(db, (int)mrow, (int)kk, wb, bit);
  const uint64_t unit = (uint64_t)cg * n_ks + ks;
  const uint32_t word = *reinterpret_cast<const uint32_t*>(codes + unit * (uint64_t)(kUnitN * kUnitK * db / 8) + wb);
  const int d = (word >> bit) & ((1 << db) - 1);
  return d - code_off(db);
}

__global__ void unpack_codes_kernel(const uint8_t* __restrict__ codes, int db, uint32_t m,
                                    uint32_t n, uint32_t n_ks, uint32_t col_base,
                                    int8_t* __restrict__ out) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (uint64_t)m * n) return;
  const uint32_t i = tid / n, j = tid % n;
  out[tid] = (int8_t)device_code_at(codes, db, i, col_base + j, n_ks);
}

__global__ void dequant_kernel(const uint8_t* __restrict__ codes, int db,
                               const float* __restrict__ steps, const int32_t* __restrict__ sal_off,
                               const int32_t* __restrict__ sal_idx,
                               const uint16_t* __restrict__ sal_rows, uint32_t m, uint32_t n,
                               uint32_t n_ks, uint32_t col_base, float* __restrict__ out) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (uint64_t)m * n) return;
  const uint32_t i = tid / n, j = tid % n;
  const uint32_t jg = col_base + j;
  const uint32_t cg = jg / kUnitN;
  float v = (float)device_code_at(codes, db, i, jg, n_ks) * steps[jg];
  for (int r = sal_off[cg]; r < sal_off[cg + 1]; ++r)
    if ((uint32_t)sal_idx[r] == i)
      v = __half2float(__ushort_as_half(sal_rows[(uint64_t)r * kUnitN + jg % kUnitN]));
  out[tid] = v;
}

__global__ void unpack_weight_kernel(const uint8_t* __restrict__ w, uint32_t m, uint32_t n,
                                     uint32_t n_ks, uint32_t col_base, uint16_t* __restrict__ out) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (uint64_t)m * n) return;
  const uint32_t i = tid / n, j = tid % n;
  const uint32_t jg = col_base + j;
  const uint64_t unit = (uint64_t)(jg / kUnitN) * n_ks + i / kUnitK;
  out[tid] = *reinterpret_cast<const uint16_t*>(w + unit * kUnitWBytes +
                                                w_byte_in_unit((int)(jg % kUnitN), (int)(i % kUnitK)));
}

}  // namespace mesw

using namespace mesw;

static inline unsigned grid_for(uint64_t total, int block) {
  return (unsigned)((total + block - 1) / block);
}

extern "C" int mesw_repack_codes(const uint8_t* d_packed, uint32_t m, uint32_t n, uint32_t bits,
                                 const int32_t* d_sal_idx, uint32_t k, uint8_t* d_codes,
                                 uint32_t m_pad, uint32_t n_total_pad, uint32_t col_base,
                                 void* stream) {
  const int db = mesw_device_code_bits(bits);
  if (!db) return mesw_fail(MESW_ERR_VALUE, "bits must be one of (1, 2, 3, 4, 8)");
  if (m_pad % kTileK || n_total_pad % kTileN || col_base % kTileN || m > m_pad ||
      col_base + n > n_total_pad)
    return mesw_fail(MESW_ERR_VALUE, "repack_codes: bad geometry");
  if (bits == 1 && k > 0)
    return mesw_fail(MESW_ERR_VALUE,
                     "1-bit layer with salient rows is not constructible (compress.py:205-214)");
  if (m == 0 || n == 0) return MESW_OK;
  const uint32_t n_ks = m_pad / kTileK;
  const uint32_t cg0 = col_base / kTileN;
  const uint32_t n_cg_blk = (n + kTileN - 1) / kTileN;
  const uint64_t words = (uint64_t)n_cg_blk * n_ks * (kUnitN * kUnitK * db / 32);
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t* dst = reinterpret_cast<uint32_t*>(d_codes);
  if (db == 2)
    repack_codes_kernel<2><<<grid_for(words, 256), 256, 0, s>>>(d_packed, m, n, bits, d_sal_idx, k,
                                                                dst, n_ks, cg0, n_cg_blk, col_base);
  else if (db == 4)
    repack_codes_kernel<4><<<grid_for(words, 256), 256, 0, s>>>(d_packed, m, n, bits, d_sal_idx, k,
                                                                dst, n_ks, cg0, n_cg_blk, col_base);
  else
    repack_codes_kernel<8><<<grid_for(words, 256), 256, 0, s>>>(d_packed, m, n, bits, d_sal_idx, k,
                                                                dst, n_ks, cg0, n_cg_blk, col_base);
  return mesw_check_launch("repack_codes");
}

extern "C" int mesw_repack_weight(const uint16_t* d_src, uint32_t m, uint32_t n, uint32_t ld,
                                  int transposed, uint16_t* d_w, uint32_t m_pad,
                                  uint32_t n_total_pad, uint32_t col_base, void* stream) {
  if (m_pad % kTileK || n_total_pad % kTileN || col_base % kTileN || m > m_pad ||
      col_base + n > n_total_pad)
    return mesw_fail(MESW_ERR_VALUE, "repack_weight: bad geometry");
  if (m == 0 || n == 0) return MESW_OK;
  const uint32_t n_ks = m_pad / kTileK;
  const uint32_t n_cg_blk = (n + kTileN - 1) / kTileN;
  const uint64_t rows16 = (uint64_t)n_cg_blk * n_ks * kUnitN * (kUnitK / 8);
  repack_weight_kernel<<<grid_for(rows16, 256), 256, 0, (cudaStream_t)stream>>>(
      d_src, m, n, ld, transposed, reinterpret_cast<uint8_t*>(d_w), n_ks, col_base / kTileN,
      n_cg_blk, col_base);
  return mesw_check_launch("repack_weight");
}

extern "C" int mesw_unpack_codes_debug(const uint8_t* d_codes, uint32_t code_bits, uint32_t m,
                                       uint32_t n, uint32_t m_pad, uint32_t n_total_pad,
                                       uint32_t col_base, int8_t* d_out, void* stream) {
  if (code_bits != 2 && code_bits != 4 && code_bits != 8)
    return mesw_fail(MESW_ERR_VALUE, "code_bits must be 2, 4 or 8");
  if (m_pad % kTileK || n_total_pad % kTileN || m > m_pad || col_base + n > n_total_pad)
    return mesw_fail(MESW_ERR_VALUE, "unpack_codes_debug: bad geometry");
  if (m == 0 || n == 0) return MESW_OK;
  unpack_codes_kernel<<<grid_for((uint64_t)m * n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_codes, code_bits, m, n, m_pad / kTileK, col_base, d_out);
  return mesw_check_launch("unpack_codes_debug");
}

extern "C" int mesw_dequant_debug(const uint8_t* d_codes, uint32_t code_bits, const float* d_steps,
                                  const int32_t* d_sal_off, const int32_t* d_sal_idx,
                                  const uint16_t* d_sal_rows, uint32_t m, uint32_t n,
                                  uint32_t m_pad, uint32_t n_total_pad, uint32_t col_base,
                                  float* d_out, void* stream) {
  if (code_bits != 2 && code_bits != 4 && code_bits != 8)
    return mesw_fail(MESW_ERR_VALUE, "code_bits must be 2, 4 or 8");
  if (m_pad % kTileK || n_total_pad % kTileN || m > m_pad || col_base + n > n_total_pad)
    return mesw_fail(MESW_ERR_VALUE, "dequant_debug: bad geometry");
  if (m == 0 || n == 0) return MESW_OK;
  dequant_kernel<<<grid_for((uint64_t)m * n, 256), 256, 0, (cudaStream_t)stream>>>(
      d_codes, code_bits, d_steps, d_sal_off, d_sal_idx, d_sal_rows, m, n, m_pad / kTileK,
      col_base, d_out);
  return mesw_check_launch("dequant_debug");
}

extern "C" int mesw_unpack_weight_debug(const uint16_t* d_w, uint32_t m, uint32_t n,
                                        uint32_t m_pad, uint32_t n_total_pad, uint32_t col_base,
                                        uint16_t* d_out, void* stream) {
  if (m_pad % kTileK || n_total_pad % kTileN || m > m_pad || col_base + n > n_total_pad)
    return mesw_fail(MESW_ERR_VALUE, "unpack_weight_debug: bad geometry");
  if (m == 0 || n == 0) return MESW_OK;
  unpack_weight_kernel<<<grid_for((uint64_t)m * n, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const uint8_t*>(d_w), m, n, m_pad / kTileK, col_base, d_out);
  return mesw_check_launch("unpack_weight_debug");
}
