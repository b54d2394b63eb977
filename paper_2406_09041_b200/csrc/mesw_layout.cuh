// Device layouts of the fused multi-expert linear (tcgen05 version).
//
// A linear (m inputs, n outputs) is padded to m_pad = ceil128(m), n_pad = ceil128(n)
// and cut into units (cg = 128 output channels, ks = 128 input channels), stored
// cg-major: unit = cg * n_ks + ks.
//
// Base weight unit (32 KiB, bf16): the UMMA K-major SWIZZLE_NONE canonical tile
// for A = W^T (M = 128 output channels, K = 128 inputs), so one bulk copy lands it
// ready for tcgen05.mma:
//   byte(m, k) = (m/8)*2048 + (k/8)*128 + (m%8)*16 + (k%8)*2
//   (8x16-byte core matrices; LBO = 128 B between k-chunks, SBO = 2048 B between
//    8-row groups)
//
// Delta code unit (2048*DB bytes): thread m (output channel) of the dequant warpgroup
// reads its codes for k in [64*kh, 64*kh+64) as 8*DB contiguous bytes:
//   chunk(kh, m) at byte ((kh*128) + m) * 8*DB
// Inside a chunk, bf16x2 pair p (k = 64*kh + 2p, 2p+1; p < 32) lives in 32-bit word
// p / PW (PW = 16/DB pairs per word), lo code at bit DB*(p%PW), hi code at bit
// 16 + DB*(p%PW).  Codes are offsets d = q + OFF (OFF = 2, 8, 128 for DB = 2, 4, 8).
#pragma once

#include <stdint.h>

namespace mesw {

constexpr int kUnitN = 128;
constexpr int kUnitK = 128;
constexpr int kUnitWBytes = kUnitN * kUnitK * 2;

__host__ __device__ inline uint32_t w_byte_in_unit(int m, int k) {
  return (uint32_t)((m >> 3) * 2048 + (k >> 3) * 128 + (m & 7) * 16 + (k & 7) * 2);
}

__host__ __device__ inline int code_off(int db) { return db == 2 ? 2 : (db == 4 ? 8 : 128); }

// Location of code (m, k) of a unit: byte offset of its 32-bit word and bit position.
__host__ __device__ inline void code_loc(int db, int m, int k, uint32_t& word_byte, int& bit) {
  const int kh = k >> 6, kk = k & 63, p = kk >> 1, h = kk & 1;
  const int pw = 16 / db;
  const int w = p / pw, loc = p % pw;
  word_byte = (uint32_t)(((kh * 128) + m) * 8 * db + w * 4);
  bit = db * loc + (h ? 16 : 0);
}

}  // namespace mesw
