// Device CRC-32 (IEEE / zlib, reflected polynomial 0xEDB88320) and kind-1 frame
// assembly.  The reference computes the frame CRC on the host
// with zlib (proj/src/core/crc32.cpp:7-20, frame.cpp:9-25) at ~2 GB/s; here it is a
// two-kernel reduction over the frame bytes in HBM:
//
//   crc_chunks_kernel : warp per 4 KiB chunk; lane l runs slicing-by-8 over its
//                       128-byte segment from a zero register, the warp folds the
//                       32 segment CRCs with byte-sliced "append 2^j x 128 zero
//                       bytes" operators.  A short last chunk is front-padded with
//                       zero bytes (R(0, 0^k || X) = R(0, X)).
//   crc_final_kernel  : one CTA folds the chunk CRCs (front-padded to a power-of-two
//                       run per thread, then a tree with the 2^k-byte shift
//                       matrices), appends the tail chunk and applies zlib's
//                       pre/post conditioning: crc = ~(R(0, D) ^ shift(~0, |D|)).
//
// R(c, D) is the raw register update; it is linear: R(c, A||B) = shift(R(c, A), |B|)
// ^ R(0, B), where shift(c, n) = R(c, 0^n) is a GF(2)-linear map (a 32x32 matrix).
#pragma once

#include <cstdint>

namespace isf {
namespace crc {

constexpr int kChunk = 4096;       // bytes per warp
constexpr int kSeg = kChunk / 32;  // bytes per lane
constexpr int kPow2 = 48;          // shift matrices for 2^0 .. 2^47 zero bytes

struct Tables {
  uint32_t slice[8][256];        // slicing-by-8
  uint32_t warpop[5][4][256];    // byte-sliced shift by kSeg * 2^j bytes, j = 0..4
  uint32_t op4k[4][256];         // byte-sliced shift by kChunk bytes
  uint32_t pow2[kPow2][32];      // columns of the shift-by-2^k-bytes matrices
};

__device__ Tables g_tables;

__host__ __device__ inline uint32_t mat_apply(const uint32_t* m, uint32_t v) {
  uint32_t r = 0;
  for (int i = 0; v; ++i, v >>= 1)
    if (v & 1u) r ^= m[i];
  return r;
}

// shift(c, n): append n zero bytes to the register
__device__ inline uint32_t shift_bytes(uint32_t c, uint64_t n) {
  for (int k = 0; n && c; ++k, n >>= 1)
    if (n & 1u) c = mat_apply(g_tables.pow2[k], c);
  return c;
}

__device__ __forceinline__ uint32_t sliced(const uint32_t (*t)[256], uint32_t c) {
  return t[0][c & 255u] ^ t[1][(c >> 8) & 255u] ^ t[2][(c >> 16) & 255u] ^ t[3][c >> 24];
}

// Host: build all tables (called once per device).
inline void build_tables(Tables& T) {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1u) ? (c >> 1) ^ 0xEDB88320u : c >> 1;
    T.slice[0][i] = c;
  }
  for (int s = 1; s < 8; ++s)
    for (int i = 0; i < 256; ++i) T.slice[s][i] = (T.slice[s - 1][i] >> 8) ^ T.slice[0][T.slice[s - 1][i] & 255u];
  // one zero bit: c -> (c >> 1) ^ (c & 1 ? poly : 0)
  uint32_t bit[32], a[32], b[32];
  bit[0] = 0xEDB88320u;
  for (int i = 1; i < 32; ++i) bit[i] = 1u << (i - 1);
  auto square = [](const uint32_t* m, uint32_t* out) {
    for (int i = 0; i < 32; ++i) out[i] = mat_apply(m, m[i]);
  };
  square(bit, a);  // 2 bits
  square(a, b);    // 4 bits
  square(b, a);    // 8 bits = 1 byte
  for (int i = 0; i < 32; ++i) T.pow2[0][i] = a[i];
  for (int k = 1; k < kPow2; ++k) square(T.pow2[k - 1], T.pow2[k]);
  auto sliced_of = [&](int k, uint32_t (*out)[256]) {
    for (int s = 0; s < 4; ++s)
      for (uint32_t v = 0; v < 256; ++v) out[s][v] = mat_apply(T.pow2[k], v << (8 * s));
  };
  for (int j = 0; j < 5; ++j) sliced_of(7 + j, T.warpop[j]);  // kSeg = 128 = 2^7
  sliced_of(12, T.op4k);                                       // kChunk = 2^12
}

// n_dev (if non-null) holds the byte count; data 16-B aligned unless `unaligned`.
__global__ void __launch_bounds__(256) crc_chunks_kernel(const uint8_t* __restrict__ data, const uint64_t* n_dev,
                                                         uint64_t n_host, uint32_t* __restrict__ chunk_crc) {
  __shared__ uint32_t S[8][256];
  __shared__ uint32_t O[5][4][256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&S[0][0])[i] = (&g_tables.slice[0][0])[i];
  for (int i = threadIdx.x; i < 5 * 4 * 256; i += blockDim.x) (&O[0][0][0])[i] = (&g_tables.warpop[0][0][0])[i];
  __syncthreads();
  const uint64_t n = n_dev ? *n_dev : n_host;
  const uint64_t nch = (n + kChunk - 1) / kChunk;
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t W = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const bool aligned = ((uintptr_t)data & 15u) == 0;
  for (uint64_t c = gw; c < nch; c += W) {
    const uint64_t base = c * kChunk;
    const uint64_t len = n - base < (uint64_t)kChunk ? n - base : (uint64_t)kChunk;
    uint32_t r = 0;
    if (len == (uint64_t)kChunk && aligned) {
      const uint4* p = reinterpret_cast<const uint4*>(data + base + (uint64_t)kSeg * lane);
#pragma unroll 4
      for (int i = 0; i < kSeg / 16; ++i) {
        const uint4 q = __ldg(p + i);
        uint32_t lo = q.x ^ r, hi = q.y;
        r = S[7][lo & 255u] ^ S[6][(lo >> 8) & 255u] ^ S[5][(lo >> 16) & 255u] ^ S[4][lo >> 24] ^
            S[3][hi & 255u] ^ S[2][(hi >> 8) & 255u] ^ S[1][(hi >> 16) & 255u] ^ S[0][hi >> 24];
        lo = q.z ^ r;
        hi = q.w;
        r = S[7][lo & 255u] ^ S[6][(lo >> 8) & 255u] ^ S[5][(lo >> 16) & 255u] ^ S[4][lo >> 24] ^
            S[3][hi & 255u] ^ S[2][(hi >> 8) & 255u] ^ S[1][(hi >> 16) & 255u] ^ S[0][hi >> 24];
      }
    } else {  // short last chunk (front-padded with zeros) or unaligned data: bytewise
      const int64_t pad = (int64_t)kChunk - (int64_t)len;
      for (int i = 0; i < kSeg; ++i) {
        const int64_t pos = (int64_t)kSeg * lane + i - pad;
        const uint32_t byte = pos >= 0 ? data[base + (uint64_t)pos] : 0u;
        r = (r >> 8) ^ S[0][(r ^ byte) & 255u];
      }
    }
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const uint32_t right = __shfl_down_sync(0xffffffffu, r, 1 << j);
      if ((lane & ((2 << j) - 1)) == 0) r = sliced(O[j], r) ^ right;
    }
    if (lane == 0) chunk_crc[c] = r;
  }
}

// One CTA of 1024 threads.  Writes the zlib CRC of the n bytes to *out (u32) and, if
// frame_tail is non-null, little-endian at frame_tail + n (the frame trailer).
constexpr int kFinalThreads = 1024;
__global__ void __launch_bounds__(kFinalThreads) crc_final_kernel(const uint32_t* __restrict__ chunk_crc,
                                                                  const uint64_t* n_dev, uint64_t n_host,
                                                                  uint32_t* out, uint8_t* frame_tail) {
  __shared__ uint32_t part[kFinalThreads];
  const uint64_t n = n_dev ? *n_dev : n_host;
  const uint64_t nfull = n / kChunk, tail = n % kChunk;
  // per-thread run length: a power of two with per * threads >= nfull (front-padded)
  uint64_t per = 1;
  int lg = 0;
  while (per * kFinalThreads < nfull) { per <<= 1; ++lg; }
  const uint64_t pad = per * kFinalThreads - nfull;
  const int t = threadIdx.x;
  uint32_t r = 0;
  for (uint64_t v = (uint64_t)t * per; v < (uint64_t)(t + 1) * per; ++v) {
    if (v < pad) continue;  // leading zero chunks: R(0, zeros) = 0
    r = sliced(g_tables.op4k, r) ^ chunk_crc[v - pad];
  }
  part[t] = r;
  __syncthreads();
  // tree: level j joins runs of per * 2^j chunks = 2^(12 + lg + j) bytes
  for (int j = 0; (1 << j) < kFinalThreads; ++j) {
    const int step = 2 << j;
    if ((t & (step - 1)) == 0) part[t] = mat_apply(g_tables.pow2[12 + lg + j], part[t]) ^ part[t + (1 << j)];
    __syncthreads();
  }
  if (t == 0) {
    uint32_t x = part[0];
    if (tail) x = shift_bytes(x, tail) ^ chunk_crc[nfull];
    const uint32_t crc = ~(x ^ shift_bytes(0xFFFFFFFFu, n));
    if (out) *out = crc;
    if (frame_tail)
      for (int b = 0; b < 4; ++b) frame_tail[n + b] = (uint8_t)(crc >> (8 * b));
  }
}

// Kind-1 frame (frame.hpp:3-11, frame.cpp:9-25) with the SPEC.md:282 payload, built
// from the mask stream:
//   header | kept_count u32[n_el] | index u32[K] | value f64[K] | codec u16 = 0 |
//   coded length u64 = 0 | (CRC-32 written afterwards by crc_final_kernel)
// index = component * P^3 + j (j = kx + P (ky + P kz)), ascending inside the element,
// so the values keep the stream's order and are one straight copy.  One warp per
// element for the counts and the indices (a mask word's set bits ranked by popcount,
// two bits per lane; block value offsets `off` from block_offsets8_kernel), all
// threads for the value copy (the payload's value array is only 4-byte aligned).
// n_out = bytes the CRC covers (0 and ISF_STATUS_OVERFLOW when frame_cap is short).
__global__ void spec_frame_kernel(uint8_t* frame, uint64_t frame_cap, const uint8_t* stream, const uint64_t* off,
                                  uint64_t n_el, uint32_t E, uint32_t P, uint32_t comps, const uint64_t* kept_dev,
                                  uint64_t step, double sim_time, uint64_t* n_out, unsigned long long* flags) {
  const uint64_t K = *kept_dev;
  const uint64_t payload = 4 * n_el + 12 * K + 10;
  if (48 + payload + 4 > frame_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicOr(flags, 4ull);  // ISF_STATUS_OVERFLOW
      *n_out = 0;
    }
    return;
  }
  const uint32_t P3 = P * P * P, W = (P3 + 63) / 64;
  const uint64_t B = n_el * comps;
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(stream);
  const uint64_t mask_off = (4 * B + 15) & ~15ull;
  const uint64_t* masks = reinterpret_cast<const uint64_t*>(stream + mask_off);
  const uint64_t* vals = reinterpret_cast<const uint64_t*>(stream + mask_off + 8ull * W * B);
  uint8_t* pl = frame + 48;
  uint32_t* cnt_out = reinterpret_cast<uint32_t*>(pl);
  uint32_t* idx_out = reinterpret_cast<uint32_t*>(pl + 4 * n_el);
  uint32_t* val_out = reinterpret_cast<uint32_t*>(pl + 4 * n_el + 4 * K);
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t p2 = 2 * lane;
  for (uint64_t e = gw; e < n_el; e += nw) {
    uint32_t ce = 0;
    for (uint32_t c = 0; c < comps; ++c) {
      const uint64_t b = e * comps + c;
      ce += counts[b];
      uint64_t base = off[b];
      for (uint32_t w = 0; w < W; ++w) {
        const uint64_t m = masks[b * W + w];
        if (m == 0) continue;  // warp-uniform
        const uint32_t r0 = (uint32_t)__popcll(m & ((1ull << p2) - 1ull));
        const uint32_t b0 = (uint32_t)(m >> p2) & 1u, b1 = (uint32_t)(m >> (p2 + 1)) & 1u;
        const uint32_t j = c * P3 + 64 * w + p2;
        if (b0) idx_out[base + r0] = j;
        if (b1) idx_out[base + r0 + b0] = j + 1;
        base += (uint64_t)__popcll(m);
      }
    }
    if (lane == 0) cnt_out[e] = ce;
  }
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < K; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = vals[i];
    val_out[2 * i] = (uint32_t)v;
    val_out[2 * i + 1] = (uint32_t)(v >> 32);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    auto put = [&](uint64_t o, uint64_t v, int nb) {
      for (int k = 0; k < nb; ++k) frame[o + k] = (uint8_t)(v >> (8 * k));
    };
    put(0, 0x31465349ull, 4);  // "ISF1"
    put(4, 1, 2);              // version
    put(6, 1, 2);              // payload_kind = CompressedBlock
    put(8, step, 8);
    put(16, (uint64_t)__double_as_longlong(sim_time), 8);
    put(24, E, 4);
    put(28, P, 4);
    put(32, comps, 4);
    put(36, 0, 4);  // reserved
    put(40, payload, 8);
    put(48 + payload - 10, 0, 2);  // codec id 0 (no lossless stage yet)
    put(48 + payload - 8, 0, 8);   // coded length 0
    *n_out = 48 + payload;
  }
}

}  // namespace crc
}  // namespace isf
