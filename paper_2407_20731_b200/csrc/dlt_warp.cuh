// dlt_warp.cuh -- warp-per-block decompress for lx != 8 (scalar fields, no error
// report).
//
// The generic decompress (dlt_kernels.cuh) runs one block per CTA with CTA-wide
// barriers between the gather and the three sweeps; this kernel gives each warp its own
// blocks (round-robin, no barriers) with the lx = 8 decompress structure carried over
// to any order:
//
//  * header (count, mask words, value offset) prefetched one block ahead, then a
//    batched gather of the kept values into a padded work buffer (row stride lx + 1
//    for even lx: every sweep's 64-bit accesses are bank-conflict free per half warp);
//  * paired-lane line transforms: a round covers 16 lines, lane l and lane l + 16 share
//    line 16 rd + (l & 15); the low half sums the even coefficients (E_i), the high
//    half the odd ones (O_i), one shuffle exchanges them and out[i] = E + O (low),
//    out[lx-1-i] = E - O (high).  Both halves run one instruction stream: the per-lane
//    constants C[i][q] = B[i][2q + half] sit in registers and the high half's operand
//    sign is flipped on the integer pipe (dsub(a, b) == dadd(a, -b) bitwise; IEEE
//    addition commutes).  For odd lx the absent terms are fma(-0, +0, acc) == acc
//    exactly (signed zeros included), so every value is computed with exactly the
//    pinned operation sequence of inv_line (dlt_common.cuh; oracle/isf_oracle.c);
//  * inverse sweeps x, y in place and z straight to global memory (each store
//    instruction writes two 128-B runs of one plane).
// Used for the orders where it measured faster than decompress_generic (isf_lossy.cu
// use_warp; profiles/r2_summary.md).  The matching warp-per-block compress (TMA stage,
// same paired sweeps, binned selection) measured slower than compress_generic at every
// order (occupancy: ~36 KB of shared memory per warp at lx 12) and was dropped.
#pragma once
#include "dlt_fast8.cuh"

#ifndef ISF_DW_BATCH
#define ISF_DW_BATCH 8
#endif

namespace isf {
namespace dev {

__host__ __device__ constexpr size_t wal16(size_t x) { return (x + 15) & ~size_t(15); }

template <int LX>
struct WG {
  static constexpr int N2 = LX * LX, N3 = LX * LX * LX;
  static constexpr int H = LX / 2, Q = (LX + 1) / 2;
  static constexpr int RS = (LX & 1) ? LX : LX + 1;  // padded row stride (odd)
  static constexpr int PN = N2 * RS;
  static constexpr int NL = (N2 + 15) / 16;  // line rounds of a sweep
  static constexpr int W = (N3 + 63) / 64;   // 64-bit mask words
  static constexpr int NWD = 4;              // warps per CTA
  // decompress, per warp
  static constexpr size_t d_mw = wal16((size_t)PN * 8);
  static constexpr size_t d_pre = d_mw + (size_t)W * 8;
  static constexpr size_t d_bytes = wal16(d_pre + (size_t)W * 4);
};

template <int LX>
__device__ __forceinline__ int padj(int j) {
  if constexpr (LX & 1) return j;
  else return j + j / LX;
}
__device__ __forceinline__ double flip_sign(double v, uint32_t sgn) {
  return __hiloint2double(__double2hiint(v) ^ (int)sgn, __double2loint(v));
}

// inverse, paired lanes: v[q] = coefficient 2q + half of the line; out[i] = value i
// (low half) or LX - 1 - i (high half); out[H] (odd lx, low half) = the middle value
template <int LX>
__device__ __forceinline__ void inv_pair(const double (&v)[WG<LX>::Q], const double (&C)[WG<LX>::Q][WG<LX>::Q],
                                         uint32_t sgn, double (&out)[WG<LX>::Q]) {
  constexpr int H = LX / 2, Q = (LX + 1) / 2;
  double acc[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    double a = __dmul_rn(C[i][0], v[0]);
#pragma unroll
    for (int q = 1; q < Q; ++q) a = __fma_rn(C[i][q], v[q], a);
    acc[i] = a;  // E_i (low half) | O_i (high half)
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const double r = __shfl_xor_sync(0xffffffffu, acc[i], 16);
    out[i] = __dadd_rn(r, flip_sign(acc[i], sgn));  // O + E == E + O | E - O
  }
  if constexpr (LX & 1) out[H] = acc[H];
}

template <int LX>
__global__ void __launch_bounds__(WG<LX>::NWD * 32) decompress_w(DecompressArgs A) {
  using G = WG<LX>;
  constexpr int N2 = G::N2, N3 = G::N3, H = G::H, Q = G::Q, RS = G::RS, NL = G::NL, W = G::W;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wb = smem + (size_t)warp * G::d_bytes;
  double* P = reinterpret_cast<double*>(wb);
  uint64_t* mwd = reinterpret_cast<uint64_t*>(wb + G::d_mw);
  uint32_t* wpre = reinterpret_cast<uint32_t*>(wb + G::d_pre);
  const bool hi_half = lane >= 16;
  const int li = lane & 15, half = hi_half ? 1 : 0;
  const uint32_t sgn = hi_half ? 0x80000000u : 0u;
  // per-lane inverse constants: value i, coefficient k = 2q + half
  double C[Q][Q];
#pragma unroll
  for (int i = 0; i < Q; ++i)
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int kq = 2 * q + half;
      C[i][q] = kq < LX ? c_ops[op_offset(LX) + LX * LX + i * LX + kq] : -0.0;
    }
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(A.stream);
  const uint64_t* masks = reinterpret_cast<const uint64_t*>(A.stream + A.mask_off);
  const double* vals = reinterpret_cast<const double*>(A.stream + A.val_off);
  const uint64_t nvals_avail = A.stream_bytes > A.val_off ? (A.stream_bytes - A.val_off) / 8 : 0;
  constexpr uint64_t lastmask = (N3 % 64) ? ((1ull << (N3 % 64)) - 1ull) : ~0ull;
  const uint64_t B = A.nblocks;
  const uint64_t Wt = (uint64_t)gridDim.x * G::NWD;
  const uint64_t gw = (uint64_t)blockIdx.x * G::NWD + warp;
  uint64_t m0 = 0, m1 = 0, off = 0;
  uint32_t cnt = 0;
  auto load_hdr = [&](uint64_t blk) {
    m0 = m1 = 0;
    cnt = 0;
    off = 0;
    if (blk < B) {
      if (lane < W) m0 = __ldg(masks + blk * W + lane);
      if (lane + 32 < W) m1 = __ldg(masks + blk * W + lane + 32);
      cnt = __ldg(counts + blk);
      off = __ldg(A.off + blk);
    }
  };
  load_hdr(gw);
  for (uint64_t blk = gw; blk < B; blk += Wt) {
    uint64_t a0 = m0, a1 = m1;
    const uint32_t c = cnt;
    const uint64_t prefix = off;
    load_hdr(blk + Wt);  // next block's header in flight during this one
    if (lane == W - 1 && (a0 & ~lastmask)) { atomicOr(A.ws.flags, kFlagShape); a0 &= lastmask; }
    if (lane + 32 == W - 1 && (a1 & ~lastmask)) { atomicOr(A.ws.flags, kFlagShape); a1 &= lastmask; }
    const uint32_t c0 = (uint32_t)__popcll(a0), c1 = (uint32_t)__popcll(a1);
    uint32_t i0 = c0, i1 = c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t0 = __shfl_up_sync(0xffffffffu, i0, o), t1 = __shfl_up_sync(0xffffffffu, i1, o);
      if (lane >= o) { i0 += t0; i1 += t1; }
    }
    const uint32_t tot0 = __shfl_sync(0xffffffffu, i0, 31);
    const uint32_t pc = tot0 + __shfl_sync(0xffffffffu, i1, 31);
    const bool bad = pc != c || prefix + c > nvals_avail;
    if (bad && lane == 0) atomicOr(A.ws.flags, kFlagShape);
    if (lane < W) { mwd[lane] = bad ? 0ull : a0; wpre[lane] = i0 - c0; }
    if (lane + 32 < W) { mwd[lane + 32] = bad ? 0ull : a1; wpre[lane + 32] = tot0 + i1 - c1; }
    __syncwarp();
    // ---- gather into P: word w, this lane's bits 2 lane and 2 lane + 1 (ranks by popcount)
    constexpr int kB = ISF_DW_BATCH;
    const uint64_t lowm = (1ull << (2 * lane)) - 1ull;
#pragma unroll 1
    for (int w0 = 0; w0 < W; w0 += kB) {
      double v0[kB], v1[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        v0[u] = 0.0;
        v1[u] = 0.0;
        const int w = w0 + u;
        if (w < W) {
          const uint64_t m = mwd[w];
          const uint32_t b0 = (uint32_t)(m >> (2 * lane)) & 1u, b1 = (uint32_t)(m >> (2 * lane + 1)) & 1u;
          const uint64_t r0 = prefix + wpre[w] + (uint32_t)__popcll(m & lowm);
          if (b0) v0[u] = __ldg(vals + r0);
          if (b1) v1[u] = __ldg(vals + r0 + b0);
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int p0 = 64 * (w0 + u) + 2 * lane;
        if (p0 < N3) P[padj<LX>(p0)] = v0[u];
        if (p0 + 1 < N3) P[padj<LX>(p0 + 1)] = v1[u];
      }
    }
    __syncwarp();
    // ---- x sweep (in place); row l
#pragma unroll 1
    for (int rd = 0; rd < NL; ++rd) {
      const int l = 16 * rd + li;
      const bool ok = l < N2;
      const int lc = ok ? l : 0;
      double* b = P + RS * lc;
      double v[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) v[q] = (2 * q + 1 < LX || !hi_half) ? b[half + 2 * q] : 0.0;
      double out[Q];
      inv_pair<LX>(v, C, sgn, out);
      if (ok) {
#pragma unroll
        for (int i = 0; i < H; ++i) b[hi_half ? LX - 1 - i : i] = out[i];
        if constexpr (LX & 1) if (!hi_half) b[H] = out[H];
      }
    }
    __syncwarp();
    // ---- y sweep (in place); line l = x + lx z
#pragma unroll 1
    for (int rd = 0; rd < NL; ++rd) {
      const int l = 16 * rd + li;
      const bool ok = l < N2;
      const int lc = ok ? l : 0;
      double* b = P + (lc % LX) + RS * LX * (lc / LX);
      double v[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) v[q] = (2 * q + 1 < LX || !hi_half) ? b[(half + 2 * q) * RS] : 0.0;
      double out[Q];
      inv_pair<LX>(v, C, sgn, out);
      if (ok) {
#pragma unroll
        for (int i = 0; i < H; ++i) b[(hi_half ? LX - 1 - i : i) * RS] = out[i];
        if constexpr (LX & 1) if (!hi_half) b[H * RS] = out[H];
      }
    }
    __syncwarp();
    // ---- z sweep: line l = x + lx y, values to global (zero results as +0)
    double* gout = A.out + blk * (uint64_t)N3;
#pragma unroll 1
    for (int rd = 0; rd < NL; ++rd) {
      const int l = 16 * rd + li;
      const bool ok = l < N2;
      const int lc = ok ? l : 0;
      const double* b = P + (lc % LX) + RS * (lc / LX);
      double v[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) v[q] = (2 * q + 1 < LX || !hi_half) ? b[(half + 2 * q) * RS * LX] : 0.0;
      double out[Q];
      inv_pair<LX>(v, C, sgn, out);
      if (ok) {
        double* g = gout + lc;
#pragma unroll
        for (int i = 0; i < H; ++i) __stcs(g + (hi_half ? LX - 1 - i : i) * N2, __dadd_rn(out[i], 0.0));
        if constexpr (LX & 1) if (!hi_half) __stcs(g + H * N2, __dadd_rn(out[H], 0.0));
      }
    }
    __syncwarp();  // P is rewritten by the next gather
  }
}

}  // namespace dev
}  // namespace isf
