// K1 loader kernels (MESW packed codes / bf16 weights -> device fragment layouts)
// and K6 debug kernels (device layouts -> reference-orientation dense arrays).
//
// Reference semantics: quant.unpack_codes (quant.py:216-236) for the code
// stream, CompressedDelta.reconstruct (compress.py:115-121) for the dense
// delta.  See include/mesw.h for the layouts.

#include "mesw_common.cuh"
#include "mesw_host.h"

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

// One thread per 32-bit device code word.
template <int DB>
__global__ void repack_codes_kernel(const uint8_t* __restrict__ packed, uint32_t m, uint32_t n,
                                    uint32_t bits, const int32_t* __restrict__ sal, uint32_t k,
                                    uint32_t* __restrict__ dst, uint32_t n_ks, uint32_t cg0,
                                    uint32_t n_cg_blk, uint32_t col_base) {
  constexpr int WPL = 2 * DB;   // words per lane per k-step
  constexpr int PW = 16 / DB;   // pairs per word
  constexpr int OFF = DB == 2 ? 2 : (DB == 4 ? 8 : 128);
  const uint64_t total = (uint64_t)n_cg_blk * n_ks * kTilesPerCg * 32 * WPL;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  const int word = tid % WPL;
  uint64_t r = tid / WPL;
  const int lane = r % 32; r /= 32;
  const int tile = r % kTilesPerCg; r /= kTilesPerCg;
  const uint32_t ks = r % n_ks;
  const uint32_t cg = cg0 + (uint32_t)(r / n_ks);
  const uint32_t bpc = (m * bits + 7) / 8;
  uint32_t out = 0;
#pragma unroll
  for (int loc = 0; loc < PW; ++loc) {
    const int p = word * PW + loc;
    const int kb = p >> 2, reg = p & 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int row, col;
      frag_coord(lane, reg, h, row, col);
      const uint32_t i = ks * kTileK + kb * 16 + col;
      const int64_t jl = (int64_t)cg * kTileN + tile * 16 + row - col_base;
      int d = OFF;  // padding and salient rows decode to q = 0
      if (i < m && jl >= 0 && jl < (int64_t)n && !is_salient(sal, k, i))
        d = read_mesw_code(packed, bpc, i, (uint32_t)jl, bits) + OFF;
      out |= uint32_t(d) << (DB * loc + (h ? 16 : 0));
    }
  }
  dst[((((uint64_t)cg * n_ks + ks) * kTilesPerCg + tile) * 32 + lane) * WPL + word] = out;
}

// One thread per lane-fragment (8 bf16 = 16 bytes).
__global__ void repack_weight_kernel(const uint16_t* __restrict__ src, uint32_t m, uint32_t n,
                                     uint32_t ld, int transposed, uint4* __restrict__ dst,
                                     uint32_t n_ks, uint32_t cg0, uint32_t n_cg_blk,
                                     uint32_t col_base) {
  const uint64_t total = (uint64_t)n_cg_blk * n_ks * kTilesPerCg * kKbPerKs * 32;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= total) return;
  uint64_t r = tid;
  const int lane = r % 32; r /= 32;
  const int kb = r % kKbPerKs; r /= kKbPerKs;
  const int tile = r % kTilesPerCg; r /= kTilesPerCg;
  const uint32_t ks = r % n_ks;
  const uint32_t cg = cg0 + (uint32_t)(r / n_ks);
  uint32_t v[4];
#pragma unroll
  for (int reg = 0; reg < 4; ++reg) {
    uint32_t pair = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int row, col;
      frag_coord(lane, reg, h, row, col);
      const uint32_t i = ks * kTileK + kb * 16 + col;
      const int64_t jl = (int64_t)cg * kTileN + tile * 16 + row - col_base;
      uint16_t e = 0;
      if (i < m && jl >= 0 && jl < (int64_t)n)
        e = transposed ? src[(uint64_t)jl * ld + i] : src[(uint64_t)i * ld + jl];
      pair |= uint32_t(e) << (h ? 16 : 0);
    }
    v[reg] = pair;
  }
  dst[((((uint64_t)cg * n_ks + ks) * kTilesPerCg + tile) * kKbPerKs + kb) * 32 + lane] =
      make_uint4(v[0], v[1], v[2], v[3]);
}

// Locate element (i, j_global) inside the fragment layouts.
struct FragLoc {
  uint64_t unit;  // cg * n_ks + ks
  int tile, kb, lane, reg, h;
};

__device__ __forceinline__ FragLoc locate(uint32_t i, uint32_t jg, uint32_t n_ks) {
  FragLoc L;
  const uint32_t cg = jg / kTileN, jj = jg % kTileN;
  const uint32_t ks = i / kTileK, ii = i % kTileK;
  L.unit = (uint64_t)cg * n_ks + ks;
  L.tile = jj / 16;
  const int row = jj % 16;
  L.kb = ii / 16;
  const int col = ii % 16;
  const int g = row & 7, t = (col & 7) >> 1;
  L.h = col & 1;
  L.lane = g * 4 + t;
  L.reg = (row >> 3) + 2 * (col >> 3);
  return L;
}

__device__ __forceinline__ int device_code_at(const uint8_t* codes, int db, uint32_t i, uint32_t jg,
                                              uint32_t n_ks) {
  const FragLoc L = locate(i, jg, n_ks);
  const int wpl = 2 * db, pw = 16 / db;
  const int p = L.kb * 4 + L.reg;
  const int word = p / pw, loc = p % pw;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(codes) +
                      ((L.unit * kTilesPerCg + L.tile) * 32 + L.lane) * wpl + word;
  const int d = (*w >> (db * loc + (L.h ? 16 : 0))) & ((1 << db) - 1);
  return d - code_offset(db);
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
  const uint32_t cg = jg / kTileN;
  float v = (float)device_code_at(codes, db, i, jg, n_ks) * steps[jg];
  for (int r = sal_off[cg]; r < sal_off[cg + 1]; ++r)
    if ((uint32_t)sal_idx[r] == i)
      v = __half2float(__ushort_as_half(sal_rows[(uint64_t)r * kTileN + jg % kTileN]));
  out[tid] = v;
}

__global__ void unpack_weight_kernel(const uint16_t* __restrict__ w, uint32_t m, uint32_t n,
                                     uint32_t n_ks, uint32_t col_base, uint16_t* __restrict__ out) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (uint64_t)m * n) return;
  const uint32_t i = tid / n, j = tid % n;
  const FragLoc L = locate(i, col_base + j, n_ks);
  const uint64_t lane_base =
      (((L.unit * kTilesPerCg + L.tile) * kKbPerKs + L.kb) * 32 + L.lane) * 8;
  out[tid] = w[lane_base + L.reg * 2 + L.h];
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
  const uint64_t words = (uint64_t)n_cg_blk * n_ks * kTilesPerCg * 32 * 2 * db;
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
  const uint64_t frags = (uint64_t)n_cg_blk * n_ks * kTilesPerCg * kKbPerKs * 32;
  repack_weight_kernel<<<grid_for(frags, 256), 256, 0, (cudaStream_t)stream>>>(
      d_src, m, n, ld, transposed, reinterpret_cast<uint4*>(d_w), n_ks, col_base / kTileN,
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
      d_w, m, n, m_pad / kTileK, col_base, d_out);
  return mesw_check_launch("unpack_weight_debug");
}
