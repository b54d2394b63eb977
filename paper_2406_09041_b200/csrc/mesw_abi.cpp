// Host side of the C ABI: MESW container parsing, geometry, salient tables.
//
// The container format and validation order follow compress.serialize_artifact /
// deserialize_artifact (compress.py:481-549); byte accounting follows
// quant.packed_nbytes (quant.py:190-192) and compress.layer_block_nbytes
// (compress.py:589-597).

#include <cstdio>
#include <cstring>
#include <string>

#include "mesw_host.h"

static thread_local std::string g_last_error;

int mesw_fail(int code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}

int mesw_check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    return mesw_fail(MESW_ERR_CUDA, buf);
  }
  return MESW_OK;
}

extern "C" int mesw_abi_version(void) { return 2; }  // 2: mesw_linear_args gained the SwiGLU epilogue fields

static int g_pdl = 1;
int mesw_pdl_enabled() { return g_pdl; }
extern "C" int mesw_set_pdl(int enable) {
  const int prev = g_pdl;
  g_pdl = enable ? 1 : 0;
  return prev;
}

extern "C" const char* mesw_last_error(void) { return g_last_error.c_str(); }

extern "C" int mesw_device_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return sms;
}

extern "C" uint64_t mesw_packed_nbytes(uint32_t rows, uint32_t cols, uint32_t bits) {
  return (uint64_t)cols * (((uint64_t)rows * bits + 7) / 8);
}

extern "C" uint64_t mesw_layer_block_nbytes(uint32_t m, uint32_t n, uint32_t bits, uint32_t k) {
  // codes + salient halves + f32 steps + u32 indices + 13-byte header + 4-byte length prefix
  return mesw_packed_nbytes(m, n, bits) + 2ull * k * n + 4ull * n + 4ull * k + 17ull;
}

extern "C" int mesw_device_code_bits(uint32_t bits) {
  switch (bits) {
    case 2: return 2;
    case 1: case 3: case 4: return 4;
    case 8: return 8;
    default: return 0;
  }
}

extern "C" uint64_t mesw_codes_device_bytes(uint32_t m_pad, uint32_t n_pad, uint32_t code_bits) {
  return (uint64_t)m_pad * n_pad * code_bits / 8;
}

extern "C" uint64_t mesw_weight_device_bytes(uint32_t m_pad, uint32_t n_pad) {
  return (uint64_t)m_pad * n_pad * 2;
}

namespace {
struct Cursor {
  const uint8_t* buf;
  uint64_t len, pos;
  // Returns false (and records a TruncatedArtifactError) if fewer than n bytes remain.
  bool take(uint64_t n, const uint8_t** out) {
    if (n > len - pos) {
      char msg[160];
      snprintf(msg, sizeof(msg), "need %llu bytes at offset %llu, only %llu left",
               (unsigned long long)n, (unsigned long long)pos,
               (unsigned long long)(len - pos));
      mesw_fail(MESW_ERR_TRUNCATED, msg);
      return false;
    }
    *out = buf + pos;
    pos += n;
    return true;
  }
};

template <typename T>
T rd(const uint8_t* p) {  // little-endian load (x86/ARM hosts are LE)
  T v;
  memcpy(&v, p, sizeof(T));
  return v;
}
}  // namespace

extern "C" int mesw_parse_header(const uint8_t* h_buf, uint64_t len, uint64_t* manifest_off,
                                 uint32_t* manifest_len) {
  if (!h_buf && len) return mesw_fail(MESW_ERR_VALUE, "null buffer");
  Cursor c{h_buf, len, 0};
  const uint8_t* p;
  if (!c.take(4, &p)) return MESW_ERR_TRUNCATED;
  if (memcmp(p, "MESW", 4) != 0) {
    char msg[96];
    snprintf(msg, sizeof(msg), "bad magic %02x%02x%02x%02x, expected 'MESW'", p[0], p[1], p[2], p[3]);
    return mesw_fail(MESW_ERR_BAD_MAGIC, msg);
  }
  if (!c.take(2, &p)) return MESW_ERR_TRUNCATED;
  const uint16_t version = rd<uint16_t>(p);
  if (version != 1) {
    char msg[64];
    snprintf(msg, sizeof(msg), "unsupported artifact version %u", (unsigned)version);
    return mesw_fail(MESW_ERR_UNSUPPORTED_VERSION, msg);
  }
  if (!c.take(4, &p)) return MESW_ERR_TRUNCATED;
  const uint32_t mlen = rd<uint32_t>(p);
  const uint64_t off = c.pos;
  if (!c.take(mlen, &p)) return MESW_ERR_TRUNCATED;
  *manifest_off = off;
  *manifest_len = mlen;
  return MESW_OK;
}

extern "C" int mesw_parse_layers(const uint8_t* h_buf, uint64_t len, uint64_t first_off,
                                 uint32_t layer_count, mesw_layer_view* views) {
  if (first_off > len) return mesw_fail(MESW_ERR_TRUNCATED, "layer offset past end");
  Cursor c{h_buf, len, first_off};
  const uint8_t* p;
  for (uint32_t l = 0; l < layer_count; ++l) {
    mesw_layer_view v{};
    if (!c.take(13, &p)) return MESW_ERR_TRUNCATED;
    v.m = rd<uint32_t>(p);
    v.n = rd<uint32_t>(p + 4);
    v.bits = p[8];
    v.k = rd<uint32_t>(p + 9);
    v.idx_off = c.pos;
    if (!c.take(4ull * v.k, &p)) return MESW_ERR_TRUNCATED;
    v.rows_off = c.pos;
    if (!c.take(2ull * v.k * v.n, &p)) return MESW_ERR_TRUNCATED;
    v.steps_off = c.pos;
    if (!c.take(4ull * v.n, &p)) return MESW_ERR_TRUNCATED;
    if (!c.take(4, &p)) return MESW_ERR_TRUNCATED;
    const uint32_t plen = rd<uint32_t>(p);
    const uint64_t expected = mesw_packed_nbytes(v.m, v.n, v.bits);
    if (plen != expected) {
      char msg[128];
      snprintf(msg, sizeof(msg), "packed block declares %u bytes, format requires %llu", plen,
               (unsigned long long)expected);
      return mesw_fail(MESW_ERR_TRUNCATED, msg);
    }
    v.codes_off = c.pos;
    v.codes_len = plen;
    if (!c.take(plen, &p)) return MESW_ERR_TRUNCATED;
    views[l] = v;
  }
  if (c.pos != len) {
    char msg[96];
    snprintf(msg, sizeof(msg), "%llu trailing bytes after last block",
             (unsigned long long)(len - c.pos));
    return mesw_fail(MESW_ERR_TRUNCATED, msg);
  }
  return MESW_OK;
}

extern "C" int mesw_build_salient_tables(uint32_t m, uint32_t n_blocks, const uint32_t* col_base,
                                         const uint32_t* n, const uint32_t* k,
                                         const uint32_t* const* h_idx,
                                         const uint16_t* const* h_rows, uint32_t n_total_pad,
                                         int32_t* h_sal_off, int32_t* h_sal_idx,
                                         uint16_t* h_sal_rows, uint64_t* total) {
  if (n_total_pad % MESW_TILE_N) return mesw_fail(MESW_ERR_VALUE, "n_total_pad % 128 != 0");
  const uint32_t n_cg = n_total_pad / MESW_TILE_N;
  for (uint32_t b = 0; b < n_blocks; ++b)
    for (uint32_t r = 0; r < k[b]; ++r) {
      // an out-of-range index would make the fused kernel read x outside the row
      if (h_idx[b][r] >= m) return mesw_fail(MESW_ERR_INDEX, "salient index out of range");
      if (r && h_idx[b][r] <= h_idx[b][r - 1]) return mesw_fail(MESW_ERR_VALUE, "salient indices must ascend");
    }
  uint64_t acc = 0;
  for (uint32_t cg = 0; cg < n_cg; ++cg) {
    const uint64_t c0 = (uint64_t)cg * MESW_TILE_N;
    int blk = -1;
    for (uint32_t b = 0; b < n_blocks; ++b)
      if (c0 >= col_base[b] && c0 < (uint64_t)col_base[b] + n[b]) blk = (int)b;
    if (h_sal_off) h_sal_off[cg] = (int32_t)acc;
    if (blk < 0) continue;
    for (uint32_t r = 0; r < k[blk]; ++r) {
      if (h_sal_idx) h_sal_idx[acc] = (int32_t)h_idx[blk][r];
      if (h_sal_rows) {
        for (uint32_t cc = 0; cc < MESW_TILE_N; ++cc) {
          const uint64_t jl = c0 + cc - col_base[blk];
          h_sal_rows[acc * MESW_TILE_N + cc] =
              jl < n[blk] ? h_rows[blk][(uint64_t)r * n[blk] + jl] : (uint16_t)0;
        }
      }
      ++acc;
    }
  }
  if (h_sal_off) h_sal_off[n_cg] = (int32_t)acc;
  if (total) *total = acc;
  return MESW_OK;
}
