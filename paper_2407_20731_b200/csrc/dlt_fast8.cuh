// dlt_fast8.cuh -- lx = 8, scalar-field fast path (the north_star configuration).
//
// One warp processes one (element, component) block of 8^3 fp64 values at a time;
// warps take blocks round-robin (block = gw, gw + W, ...), so there is no
// inter-warp dependency inside the hot kernels.  Per warp a ring of shared-memory
// stages is filled by the TMA engine (cp.async.bulk issued by one lane, mbarrier
// completion) blocks ahead.
//
// Register layouts (lane l, 16 values per lane):
//   z-lines : lane = (y = l>>2, q = l&3) holds x = 2q, 2q+1 at row y for all z
//   y-lines : compress lane = (q = l>>3, kz = l&7); decompress lane = (kz = l>>2, q = l&3)
//             both hold x = 2q, 2q+1 for all y at plane kz
//   x-lines : lane = (kz = l>>2, p = l&3) holds ky = 2p, 2p+1 for all x at plane kz
// so after the forward x sweep lane l owns coefficients 16 l .. 16 l + 15.
// Compress: z -> y through the stage (padded 33-chunk planes), y -> x through TMEM
// (tcgen05 16x256b, a two-bit lane/register exchange).  Decompress: both re-layouts
// through the stage with the padded address kz * 36 + 4 ky + ky / 2 + xq.  All
// access patterns are bank-conflict free with immediate offsets.
// Forward sweeps z, y, x; inverse x, y, z (the pinned order of oracle/isf_oracle.c).
#pragma once
#include "dlt_kernels.cuh"

namespace isf {
namespace dev {

#ifndef ISF_C8_WARPS
#define ISF_C8_WARPS 16
#endif
#ifndef ISF_D8_WARPS  // decompress8 warps per CTA (profiles/r2_summary.md, with the TMA block store:
#define ISF_D8_WARPS 20  // 16 / 18 / 20 / 21 / 22 / 24 -> 5.99 / 5.73 / 6.25 / 5.62 / 5.66 / 6.07 TB/s on TGV)
#endif
#ifndef ISF_D8E_WARPS
#define ISF_D8E_WARPS 16
#endif
constexpr int kC8Warps = ISF_C8_WARPS;  // compress warps per CTA
constexpr int kD8Warps = ISF_D8_WARPS;    // decompress warps per CTA (plain decode: 68 registers)
constexpr int kD8WarpsErr = ISF_D8E_WARPS;  // ... with the error report (more live state)
template <bool ERR>
__host__ __device__ constexpr int d8_warps() { return ERR ? kD8WarpsErr : kD8Warps; }
constexpr int kF8Stages = 2;   // TMA ring depth per warp (decompress)
#ifndef ISF_C8_STAGES
#define ISF_C8_STAGES 2
#endif
constexpr int kC8Stages = ISF_C8_STAGES;  // TMA ring depth per warp (compress)


// warp sum of per-lane values < 2^58 via three 32-bit REDUX.SUM (exact)
__device__ __forceinline__ uint64_t warp_sum_u58(uint64_t x) {
  const uint32_t a = (uint32_t)(x & 0x3FFFFFFull);
  const uint32_t b = (uint32_t)((x >> 26) & 0x3FFFFFFull);
  const uint32_t c = (uint32_t)(x >> 52);
  const uint64_t sa = __reduce_add_sync(0xffffffffu, a);
  const uint64_t sb = __reduce_add_sync(0xffffffffu, b);
  const uint64_t sc = __reduce_add_sync(0xffffffffu, c);
  return sa + (sb << 26) + (sc << 52);
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t x) {
  const uint32_t hi = (uint32_t)(x >> 32);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t lo = hi == mh ? (uint32_t)x : 0u;
  return ((uint64_t)mh << 32) | __reduce_max_sync(0xffffffffu, lo);
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t x) {
  const uint32_t hi = (uint32_t)(x >> 32);
  const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
  const uint32_t lo = hi == mh ? (uint32_t)x : 0xffffffffu;
  return ((uint64_t)mh << 32) | __reduce_min_sync(0xffffffffu, lo);
}
// exclusive prefix of per-lane counts v <= 31 without a dependent shuffle chain:
// five independent ballots over the bits of v
// (the total by one REDUX: callers that only need it drop the ballots entirely)
__device__ __forceinline__ uint32_t warp_exscan_small(uint32_t v, int lane, uint32_t& total) {
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t pre = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    const uint32_t bal = __ballot_sync(0xffffffffu, (v >> b) & 1u);
    pre += (uint32_t)__popc(bal & lt) << b;
  }
  total = __reduce_add_sync(0xffffffffu, v);
  return pre;
}
__device__ __forceinline__ uint32_t warp_exscan_u32(uint32_t v, int lane) {
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  return x - v;
}

// ---------------------------------------------------------------------------
// General-path exact selection over the warp's 512 coefficients held 16 per lane
// (same algorithm as radix_select in dlt_common.cuh, elements in registers).
// out = {t*, icut, discarded hi-sum}.
// ---------------------------------------------------------------------------
__device__ __noinline__ void radix_select16(uint32_t tpark, int lane, uint64_t R, double f, double sB, double pre,
                                            unsigned long long* hist, uint64_t* out) {
  double v[16];  // the parked coefficients (TMEM); pre: exact tiny-block pre-scale (else 1)
  tmem_wait_st();
  tmem_load16(tpark, v);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = __dmul_rn(v[r], pre);
  uint64_t klo = ~0ull, khi = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint64_t k = abs_bits(v[r]);
    klo = k < klo ? k : klo;
    khi = k > khi ? k : khi;
  }
  klo = warp_min_u64(klo);
  khi = warp_max_u64(khi);
  uint64_t dsum = 0;
  for (;;) {
    const uint64_t span = khi - klo;
    if (span == 0) {
      const uint64_t h = hi_v2(__longlong_as_double((long long)klo), f, sB);
      uint32_t cnt = 0;
#pragma unroll
      for (int r = 0; r < 16; ++r) cnt += (abs_bits(v[r]) == klo);
      const uint32_t gcount = __reduce_add_sync(0xffffffffu, cnt);
      uint64_t rr = (h == 0) ? gcount : (R / h);
      if (rr > gcount) rr = gcount;
      dsum += rr * h;
      uint32_t icut;
      if (rr == gcount) {
        icut = 0;
      } else if (rr == 0) {
        icut = 0xffffffffu;
      } else {
        // keep the (gcount - rr) smallest indices; tied elements are in ascending
        // (lane, register) = index order
        const uint32_t want = gcount - (uint32_t)rr;
        const uint32_t below = warp_exscan_u32(cnt, lane);
        uint32_t mine = 0xffffffffu, seen = 0;
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if (abs_bits(v[r]) == klo) {
            if (below + seen == want) mine = (uint32_t)(16 * lane + r);
            ++seen;
          }
        icut = __reduce_min_sync(0xffffffffu, mine);
      }
      out[0] = klo;
      out[1] = icut;
      out[2] = dsum;
      return;
    }
    const int bits = 64 - __clzll((long long)span);
    const int shift = bits > 6 ? bits - 6 : 0;
    // 64 bins of energy sums as three 21-bit digit planes of native 32-bit shared
    // atomics (each value <= 2^52, 512 values: every plane sum stays < 2^31)
    uint32_t* h32 = reinterpret_cast<uint32_t*>(hist);
#pragma unroll
    for (int j = 0; j < 6; ++j) h32[lane + 32 * j] = 0u;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint64_t k = abs_bits(v[r]);
      if (k >= klo && k <= khi) {
        const uint32_t bin = (uint32_t)((k - klo) >> shift);
        const uint64_t h = hi_v2(v[r], f, sB);
        atomicAdd(&h32[bin], (uint32_t)(h & 0x1FFFFFu));
        atomicAdd(&h32[64 + bin], (uint32_t)((h >> 21) & 0x1FFFFFu));
        atomicAdd(&h32[128 + bin], (uint32_t)(h >> 42));
      }
    }
    __syncwarp();
    const uint64_t b0 = (uint64_t)h32[2 * lane] + ((uint64_t)h32[64 + 2 * lane] << 21) +
                        ((uint64_t)h32[128 + 2 * lane] << 42);
    const uint64_t b1 = (uint64_t)h32[2 * lane + 1] + ((uint64_t)h32[64 + 2 * lane + 1] << 21) +
                        ((uint64_t)h32[128 + 2 * lane + 1] << 42);
    __syncwarp();
    const uint64_t run = b0 + b1;
    uint64_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    const uint64_t base = x - run;
    const uint64_t total = __shfl_sync(0xffffffffu, x, 31);
    uint32_t dloc = 64;
    uint64_t exloc = 0;
    if (base + b0 + b1 > R) { dloc = 2 * lane + 1; exloc = base + b0; }
    if (base + b0 > R) { dloc = 2 * lane; exloc = base; }
    const uint32_t d = __reduce_min_sync(0xffffffffu, dloc);
    if (d == 64) {
      dsum += total;
      out[0] = khi;
      out[1] = 0;
      out[2] = dsum;
      return;
    }
    const uint64_t ex = __shfl_sync(0xffffffffu, exloc, (int)(d >> 1));
    R -= ex;
    dsum += ex;
    const uint64_t nlo = klo + ((uint64_t)d << shift);
    const uint64_t nhi_full = nlo + ((1ull << shift) - 1);
    const uint64_t nhi = nhi_full < khi ? nhi_full : khi;
    uint64_t mn = ~0ull, mx = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint64_t k = abs_bits(v[r]);
      if (k >= nlo && k <= nhi) { mn = k < mn ? k : mn; mx = k > mx ? k : mx; }
    }
    klo = warp_min_u64(mn);
    khi = warp_max_u64(mx);
  }
}

#ifdef ISF_PATHSTATS
__device__ unsigned long long g_pathstats[16];
#define ISF_PATH(P_) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_pathstats[P_], 1ull); } while (0)
#else
#define ISF_PATH(P_) do {} while (0)
#endif
// ---------------------------------------------------------------------------
// General-path exact selection, binned (the common general case for turbulent
// spectra).  Any monotone function of the key |a| orders bins like the discard
// order; 256 quarter-binades of |a| below the block maximum are used.  One pass of native u32 shared atomics (three 21-bit digit planes) gives
// the exact energy of every bin; the cut lies in the first bin whose cumulative sum
// exceeds R.  If that bin holds <= 32 coefficients they are sorted across the warp
// (one key per lane, bitonic) and the cut is found with a warp prefix sum of their
// hi; ties at the cut key keep the smallest indices (SPEC.md:225 stable order).
// Returns false (nothing written) when the cut bin is too crowded: the caller falls
// back to radix_select16.  out = {t*, icut, discarded hi-sum}, as radix_select16.
// smem: bins = 3 x 256 u32, cand = 32 u64.
// ---------------------------------------------------------------------------
constexpr int kSelBins = 256;
__device__ __noinline__ bool select_bins16(uint32_t tpark, int lane, uint64_t R, double f, double sB, double pre,
                                           uint32_t* bins, uint64_t* cand, uint64_t* out) {
  uint64_t kk[16], hv[16];
  uint32_t bn[16];
  {
    double v[16];
    tmem_wait_st();
    tmem_load16(tpark, v);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const double a = __dmul_rn(v[r], pre);
      kk[r] = abs_bits(a);
      hv[r] = hi_v2(a, f, sB);  // in [1, 2^52]
    }
    // bins: quarter binades of |a| (exponent and the next two bits: kk >> 50, a
    // monotone function of the key) counted down from the block maximum; the lowest
    // 64 binades of |a| (128 of energy) share bin 0
    uint32_t top = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) top = ::max(top, (uint32_t)(kk[r] >> 50));
    top = __reduce_max_sync(0xffffffffu, top);
    const int base = (int)top - (kSelBins - 1);
#pragma unroll
    for (int r = 0; r < 16; ++r) bn[r] = (uint32_t)::max((int)(kk[r] >> 50) - base, 0);
  }
#pragma unroll
  for (int j = 0; j < 3 * kSelBins / 32; ++j) bins[lane + 32 * j] = 0u;
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    atomicAdd(&bins[bn[r]], (uint32_t)(hv[r] & 0x1FFFFFu));
    atomicAdd(&bins[kSelBins + bn[r]], (uint32_t)((hv[r] >> 21) & 0x1FFFFFu));
    atomicAdd(&bins[2 * kSelBins + bn[r]], (uint32_t)(hv[r] >> 42));
  }
  __syncwarp();
  // lane l owns bins 8l .. 8l+7
  uint64_t bs[8];
  uint64_t lsum = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int b = 8 * lane + q;
    bs[q] = (uint64_t)bins[b] + ((uint64_t)bins[kSelBins + b] << 21) + ((uint64_t)bins[2 * kSelBins + b] << 42);
    lsum += bs[q];
  }
  uint64_t x = lsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  uint64_t run = x - lsum;  // exclusive prefix of this lane's first bin
  uint32_t dloc = kSelBins;
  uint64_t exloc = 0;
#pragma unroll
  for (int q = 7; q >= 0; --q) {  // first bin (lowest q) whose inclusive sum exceeds R
    uint64_t pre_q = run;
#pragma unroll
    for (int w = 0; w < q; ++w) pre_q += bs[w];
    if (pre_q + bs[q] > R) { dloc = 8 * lane + q; exloc = pre_q; }
  }
  const uint32_t d = __reduce_min_sync(0xffffffffu, dloc);
  if (d == kSelBins) {  // everything fits: discard all (t* = largest key, none kept at it)
    uint64_t mx = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) mx = kk[r] > mx ? kk[r] : mx;
    out[0] = warp_max_u64(mx);
    out[1] = 0;
    out[2] = __shfl_sync(0xffffffffu, x, 31);
    return true;
  }
  const uint64_t ex = __shfl_sync(0xffffffffu, exloc, (int)(d >> 3));
  // candidates: the coefficients of bin d
  uint32_t cm = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) cm |= (bn[r] == d) ? (1u << r) : 0u;
  uint32_t ncand;
  const uint32_t pos = warp_exscan_small((uint32_t)__popc(cm), lane, ncand);
  if (ncand > 32) {
    ISF_PATH(15);
    return false;
  }
  __syncwarp();
  {
    uint32_t p = pos;
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if ((cm >> r) & 1u) cand[p++] = kk[r];
  }
  __syncwarp();
  uint64_t key = lane < (int)ncand ? cand[lane] : ~0ull;
  __syncwarp();
  // bitonic sort ascending by lane of the first NS keys, NS the power of two >= ncand
  // (warp-uniform): partners stay inside NS-lane groups and the lanes past ncand hold
  // the largest key, so the live lanes end sorted exactly as with all 32
  const int NS = ncand <= 2 ? 2 : ncand <= 4 ? 4 : ncand <= 8 ? 8 : ncand <= 16 ? 16 : 32;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
    if (k > NS) break;
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, key, j);
      const bool up = ((lane & k) == 0);
      const bool lower = ((lane & j) == 0);
      key = (lower == up) ? (o < key ? o : key) : (o > key ? o : key);
    }
  }
  const uint64_t h = lane < (int)ncand ? hi_v2(__longlong_as_double((long long)key), f, sB) : 0ull;
  uint64_t cs = h;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(0xffffffffu, cs, o);
    if (lane >= o) cs += t;
  }
  // first sorted candidate that does not fit: the cut (it exists: bin d overflows)
  const uint64_t Rr = R - ex;
  const uint32_t over = __ballot_sync(0xffffffffu, lane < (int)ncand && cs > Rr);
  const int ic = __ffs(over) - 1;
  const uint64_t K = __shfl_sync(0xffffffffu, key, ic);
  const uint64_t dis = __shfl_sync(0xffffffffu, cs - h, ic);  // candidates before the cut
  // discarded tied members at K: those sorted before the cut
  const uint32_t tiedbefore = __popc(__ballot_sync(0xffffffffu, lane < ic && key == K));
  uint32_t icut = 0xffffffffu;
  if (tiedbefore) {
    // keep the (gcount - tiedbefore) smallest indices among the coefficients with key K
    uint32_t cnt = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) cnt += (kk[r] == K);
    const uint32_t gcount = __reduce_add_sync(0xffffffffu, cnt);
    const uint32_t want = gcount - tiedbefore;
    const uint32_t below = warp_exscan_u32(cnt, lane);
    uint32_t mine = 0xffffffffu, seen = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (kk[r] == K) {
        if (below + seen == want) mine = (uint32_t)(16 * lane + r);
        ++seen;
      }
    icut = __reduce_min_sync(0xffffffffu, mine);
  }
  out[0] = K;
  out[1] = icut;
  out[2] = ex + dis;
  return true;
}

struct Sel16 {
  uint32_t mask;   // kept bits of this lane's 16 coefficients
  uint64_t T;      // block total at scale A (rule v2)
  uint64_t hdisc;  // hi-sum of the discarded set at scale B
  int eT, eD;      // energy = T 2^eT = hdisc 2^eD
  bool nonfinite;
};

// sqrt(2) - 1 in units of 2^-20, floor: the 20 leading fraction bits of max|a| decide
// whether its energy lies below 2^51 (h = 1) except for this one value
constexpr uint32_t kSqrt2F20 = 434334u;

// v[r] = coefficient 16*lane + r of the warp's block (consumed: only pass 0/1 read
// it); tpark = the same coefficients parked in tensor memory (32x32b, lane = thread,
// columns 2r, 2r+1), re-read by the one-move and general paths and by the encoder.
// Truncation rule v2 (oracle/isf_oracle.c select_impl).
__device__ __forceinline__ Sel16 select16(double (&v)[16], int lane, uint64_t eps_m, int eps_e,
                                          unsigned long long* hist, uint32_t tpark) {
  Sel16 s{0u, 0ull, 0ull, 0, 0, false};
  uint32_t hm = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) hm = ::max(hm, (uint32_t)__double2hiint(v[r]) & 0x7fffffffu);
  hm = __reduce_max_sync(0xffffffffu, hm);
  if (hm >= 0x7ff00000u) { s.nonfinite = true; return s; }
  constexpr int EM = energy_EM(8), HM = EM / 2;  // 52, 26
  int sexp, h;
  const uint32_t f20 = hm & 0xFFFFFu;
  if (hm >= 0x00100000u && f20 != kSqrt2F20) {
    sexp = (int)(hm >> 20) - 1022;
    h = f20 < kSqrt2F20 ? 1 : 0;  // max energy (m 2^25)^2 < 2^51  <=>  m < sqrt 2
  } else {  // subnormal maximum, all-zero block, or the undecided leading bits (rare)
    uint64_t mb = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) { const uint64_t b = abs_bits(v[r]); mb = b > mb ? b : mb; }
    mb = warp_max_u64(mb);
    if (mb == 0) return s;  // all-zero block keeps nothing
    sexp = hm >= 0x00100000u ? (int)(hm >> 20) - 1022 : 64 - __clzll((long long)mb) - 1074;
    const int kk = HM - sexp;
    const double am = __longlong_as_double((long long)mb);
    const double xm = kk > 1023 ? __dmul_rn(__dmul_rn(am, pow2d(kk - 1023)), pow2d(1023)) : __dmul_rn(am, pow2d(kk));
    h = (EM - 2 * HM) + (__dmul_rd(xm, xm) < pow2d(2 * HM - 1) ? 1 : 0);
  }
  int k = HM - sexp;
  const int k0 = k;
  // |a| < 2^-998: exact pre-scale by 2^(k-1023) (applied to every read below)
  const double pre = k > 1023 ? pow2d(k - 1023) : 1.0;
  if (k > 1023) {
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = __dmul_rn(v[r], pre);
    k = 1023;
  }
  const double f = pow2d(k);
  const double sA = h ? 2.0 : 1.0;
  // e_r = RD(x_r^2); scale A: 2^52 + floor(e_r 2^h) exactly (round-down fma), its bit
  // pattern is C52 + floor(e_r 2^h)
  constexpr uint64_t C52 = 0x4330000000000000ull;
  double t[16];
  uint64_t t0 = 0, t1 = 0;
  // f = 2^k folded into the scale constants: RD((a f)^2) = RD(a^2) 2^(2k) exactly while
  // a^2 is normal; when it is subnormal, both sides stay below 2^-22 after scaling by
  // at most 2^1000, so the floors agree (0)
  const bool fold = 2 * k + h <= 1000;
  if (fold) {
    const double fA = pow2d(2 * k + h);
#pragma unroll
    for (int r = 0; r < 16; r += 2) {
      t[r] = __dmul_rd(v[r], v[r]);
      t[r + 1] = __dmul_rd(v[r + 1], v[r + 1]);
      t0 += (uint64_t)__double_as_longlong(__fma_rd(t[r], fA, kTwo52));
      t1 += (uint64_t)__double_as_longlong(__fma_rd(t[r + 1], fA, kTwo52));
    }
  } else {
#pragma unroll
  for (int r = 0; r < 16; r += 2) {
    const double xa = __dmul_rn(v[r], f), xb = __dmul_rn(v[r + 1], f);
    t[r] = __dmul_rd(xa, xa);
    t[r + 1] = __dmul_rd(xb, xb);
    t0 += (uint64_t)__double_as_longlong(__fma_rd(t[r], sA, kTwo52));
    t1 += (uint64_t)__double_as_longlong(__fma_rd(t[r + 1], sA, kTwo52));
  }
  }
  const uint64_t T = warp_sum_u58(t0 + t1 - 16 * C52);
  s.T = T;
  int G;
  const uint64_t thr = thr_v2(T, eps_m, eps_e, h, G);
  s.eT = -2 * k0 - h;
  s.eD = -2 * k0 - h - G;
  const double sB = pow2d(h + G);
  // scale B: t_r = 2^52 + floor(e_r 2^(h+G)) (>= 2^53: saturated, never discardable)
  if (fold && 2 * k + h + G <= 1000) {
    const double fB = pow2d(2 * k + h + G);
#pragma unroll
    for (int r = 0; r < 16; ++r) t[r] = __fma_rd(t[r], fB, kTwo52);
  } else if (fold) {  // (rare) the folded scale would exceed 2^1000: recompute from the parked copy
    double c16[16];
    tmem_wait_st();
    tmem_load16(tpark, c16);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const double x = __dmul_rn(c16[r], f);
      t[r] = __fma_rd(__dmul_rd(x, x), sB, kTwo52);
    }
  } else {
#pragma unroll
  for (int r = 0; r < 16; ++r) t[r] = __fma_rd(t[r], sB, kTwo52);
  }
  // kept-above-threshold set H: hi = lo + 1 > thr  <=>  lo >= thr  <=>  t >= 2^52 + thr
  const double tthr = __longlong_as_double((long long)(C52 + thr));  // thr < 2^52
  uint32_t mH = 0;
  uint64_t n0 = 0, n1 = 0;
#pragma unroll
  for (int r = 0; r < 16; r += 2) {
    if (t[r] >= tthr) mH |= 1u << r; else n0 += (uint64_t)__double_as_longlong(t[r]);
    if (t[r + 1] >= tthr) mH |= 1u << (r + 1); else n1 += (uint64_t)__double_as_longlong(t[r + 1]);
  }
  const uint32_t nN = 16u - (uint32_t)__popc(mH);
  // sum of hi = lo + 1 over the rest (each lo < thr < 2^52: per-lane sum < 2^56)
  const uint64_t SN = warp_sum_u58(n0 + n1 - nN * C52 + nN);
  if (SN <= thr) {
    ISF_PATH(1);
    s.mask = mH;
    s.hdisc = SN;
    return s;
  }
  // Few-move path: the last element of the non-kept prefix (largest |a|, smallest
  // index among ties) joins the kept set, repeated until the rest fits under thr
  // (the next elements of the pinned order, so the result is the exact rule's).
  // t is monotone in |a|: the largest t among the non-kept gives the candidates (its
  // lo + 1 is the hi to move); ties in t are resolved by |a|, then the smallest index.
  // More than kMaxMoves moves (rare: TGV needs <= 4) go to the radix select.
  constexpr int kMaxMoves = 6;
  uint32_t mK = mH;
  uint64_t SNc = SN;
#pragma unroll 1
  for (int mv = 0; mv < kMaxMoves; ++mv) {
    uint64_t tm = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint64_t tb = ((mK >> r) & 1u) ? 0ull : (uint64_t)__double_as_longlong(t[r]);
      tm = tb > tm ? tb : tm;
    }
    const uint64_t gtm = warp_max_u64(tm);
    // t >= 2^52 > 0 and finite: double equality == bit-pattern equality, one DSETP per
    // candidate test instead of the two-word integer compare
    const double gtmd = __longlong_as_double((long long)gtm);
    // every remaining move removes at most this hi: give up early (exactly) when the
    // moves left cannot cover the excess (turbulent spectra need hundreds of moves)
    if (SNc - thr > (uint64_t)(kMaxMoves - mv) * (gtm - C52 + 1ull)) break;
    uint32_t cm = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (!((mK >> r) & 1u) && t[r] == gtmd) cm |= 1u << r;
    const uint32_t ncand = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(cm));
    if (ncand == 0) break;  // defensive (cannot happen while SNc > thr)
    uint32_t gidx;
    if (ncand == 1) {
      gidx = __reduce_min_sync(0xffffffffu, cm ? (uint32_t)(16 * lane + __ffs(cm) - 1) : 0xffffu);
    } else {
      uint64_t mk = 0;
      int mi = 16;
      double c16[16];
      tmem_wait_st();
      tmem_load16(tpark, c16);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint64_t kk = ((cm >> r) & 1u) ? abs_bits(c16[r]) + 1ull : 0ull;  // +1: zeros count
        if (kk > mk) { mk = kk; mi = r; }
      }
      const uint64_t gmk = warp_max_u64(mk);
      gidx = __reduce_min_sync(0xffffffffu, (mk == gmk && mi < 16) ? (uint32_t)(16 * lane + mi) : 0xffffu);
    }
    mK |= ((int)(gidx >> 4) == lane) ? (1u << (gidx & 15)) : 0u;
    SNc -= gtm - C52 + 1ull;
    if (SNc <= thr) {
      s.mask = mK;
      s.hdisc = SNc;
      ISF_PATH(2);
      return s;
    }
  }
  uint64_t res[3];
  if (!select_bins16(tpark, lane, thr, f, sB, pre, reinterpret_cast<uint32_t*>(hist) + 64,
                     reinterpret_cast<uint64_t*>(hist), res))
    radix_select16(tpark, lane, thr, f, sB, pre, hist, res);
  const uint64_t tstar = res[0];
  const uint32_t icut = (uint32_t)res[1];
  uint32_t mk2 = 0;
  double c16[16];
  tmem_load16(tpark, c16);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint64_t kk = abs_bits(__dmul_rn(c16[r], pre));
    const uint32_t j = (uint32_t)(16 * lane + r);
    if (kk > tstar || (kk == tstar && j < icut)) mk2 |= 1u << r;
  }
  s.mask = mk2;
#ifdef ISF_PATHSTATS
  {
    const uint32_t kk = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(mk2)) - NH;
    ISF_PATH(3);
    ISF_PATH(kk < 8 ? 4 + kk : (kk < 16 ? 12 : (kk < 64 ? 13 : 14)));
  }
#endif
  s.hdisc = res[2];
  return s;
}

// --------------------------- compress ---------------------------------------
// stage: the block's 4 KiB as loaded by the TMA engine, re-used in place for the z -> y
// re-layout with a plane stride of 33 16-B chunks (528 B; conflict free both ways)
constexpr int kC8Stage = 33 * 8 * 16;
// stages | selection scratch (radix: 3 x 64 u32; binned: 32 u64 candidates, then
// 3 x 256 u32 bins at byte 256) | mbarriers
constexpr int kC8Scratch = 32 * 8 + 3 * kSelBins * 4;
static_assert(kC8Scratch >= 768, "radix_select16 needs 3 x 64 u32");
constexpr int kC8WarpBytes = kC8Stages * kC8Stage + kC8Scratch + 128;
constexpr int kC8Smem = kC8Warps * kC8WarpBytes;
// TMEM columns per warp: [0, 32) y->x re-layout buffer, then the parked coefficients
// (one 32-column slot; three for the single-pass kernel, whose value writes trail the
// selection by two rounds); the four warps of a lane quadrant (warp % 4) sit side by side.
__host__ __device__ constexpr uint32_t pow2_ceil(uint32_t v) { return v <= 32u ? 32u : 2u * pow2_ceil((v + 1u) / 2u); }
template <bool SP>
__host__ __device__ constexpr uint32_t c8_tmem_cols() { return pow2_ceil((SP ? 128u : 64u) * (kC8Warps / 4)); }
static_assert(kC8Warps % 4 == 0 && c8_tmem_cols<true>() <= 512, "TMEM budget");

__device__ void finalize_cta(const FinalizeArgs& A, double* s_red);
__device__ __forceinline__ bool last_cta(uint32_t* done);

// Single-pass compress (SP): no value slots and no compaction kernel.  A block's value
// offset is (values of all earlier rounds) + (values of the earlier CTAs in its round) +
// (values of the earlier warps of its CTA): each CTA publishes its round aggregate
// (epoch-tagged) once its 16 warps have selected, and every warp writes the values of
// its block of round i - 2 while it works on round i, from the coefficients it parked
// in TMEM (three slots), by which time the round's aggregates are normally published.
struct Sp8Args {
  uint64_t* rstat;       // [round][cta] (epoch << 40) | kept count of the CTA's 16 blocks
  uint32_t epoch;
  uint32_t nrounds;      // ceil(B / W): every warp runs all rounds (empty ones too)
  double* vals;          // the stream's value region
  uint64_t cap_vals;
  uint64_t* total_out;   // total kept (read by the finalize)
  FinalizeArgs fin;
};

template <bool SP, bool VEC = false>
__global__ void __launch_bounds__(kC8Warps * 32) compress8_kernel(CompressArgs A, Sp8Args S) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t s_tmem;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wbase = smem + warp * kC8WarpBytes;
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(wbase + kC8Stages * kC8Stage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + kC8Stages * kC8Stage + kC8Scratch);
  const int yoff = (lane & 7) * 33 + (lane >> 3);  // y-line role (plane kz = l%8, x pair q = l/8)
  uint32_t* counts = reinterpret_cast<uint32_t*>(A.stream);
  uint16_t* masks16 = reinterpret_cast<uint16_t*>(A.stream + A.mask_off);
  const uint64_t W = (uint64_t)gridDim.x * kC8Warps;
  const uint64_t gw = (uint64_t)blockIdx.x * kC8Warps + warp;
  const uint64_t B = A.nblocks;
  __shared__ uint32_t s_kept[4][kC8Warps];  // SP: per-warp kept counts of the last rounds
  __shared__ uint32_t s_arrive[4];
  __shared__ uint32_t s_rstate[4];  // SP: round-total slots (codes in deferred())
  __shared__ uint64_t s_rtot[4], s_rpre[4];
  __shared__ double s_red[4 * kC8Warps];
  if (warp == 0) tmem_alloc<c8_tmem_cols<SP>()>(&s_tmem);
  if (threadIdx.x < 4) {
    s_arrive[threadIdx.x] = 0u;
    s_rstate[threadIdx.x] = 2u * threadIdx.x + 2u;  // READY(q - 4): slot q first serves round q
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kC8Stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = s_tmem;
  pdl_wait();  // the field / stream / workspace may come from the previous kernel
  pdl_launch_dependents();
  const uint32_t tx = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (SP ? 128u : 64u) * (uint32_t)(warp >> 2);
  const uint32_t wbase_a = smem_u32(wbase), bars_a = smem_u32(bars);  // hoisted shared-window addresses
  const uint64_t pol_stream = l2_policy_evict_first();  // the field is read once
  // vector fields (components = 3, element -> point -> component): a block is every
  // third double of its element, so each lane gathers 16 of them with 8-byte cp.async
  // into the same dense stage the TMA engine fills for scalar fields (one commit group
  // per stage, empty past the end so the group count stays in step)
  auto issue = [&](uint64_t blk, int st) {
    if constexpr (VEC) {
      if (blk < B) {
        const double* src = A.field + (blk / 3) * 1536 + (blk % 3);
        const uint32_t dst = wbase_a + (uint32_t)(st * kC8Stage);
#pragma unroll
        for (int k = 0; k < 16; ++k) cp_async8(dst + 8u * (uint32_t)(lane + 32 * k), src + 3 * (lane + 32 * k));
      }
      cp_async_commit();
      return;
    }
    if (lane == 0 && blk < B) {
      mbar_arrive_tx_a(bars_a + 8u * st, 4096u);
      bulk_g2s_hint_a(wbase_a + (uint32_t)(st * kC8Stage), A.field + blk * 512, 4096u, bars_a + 8u * st, pol_stream);
    }
  };
#pragma unroll
  for (int s = 0; s < kC8Stages; ++s) issue(gw + s * W, s);
  double tot_acc = 0.0, disc_acc = 0.0;
  int st = 0;
  uint32_t ph = 0;
  // SP state: masks / counts of the two rounds whose values are still to be written,
  // and the value offset of the first block of round i - 2
  uint32_t m1 = 0, m2 = 0, k1 = 0, k2 = 0;
  uint64_t vbase = 0;
  // SP: write the values of this warp's block of round j (mask mj, kept kj) from TMEM
  auto deferred = [&](uint32_t j, uint32_t mj, uint32_t kj) {
    // the round's totals over all CTAs: gathered once per CTA (by the first warp to
    // need them) and shared through shared memory
    volatile uint32_t* rs = s_rstate + (j & 3);
    uint32_t claim = 0;
    // slot codes: READY(r) = 2 r + 10, BUSY(r) = 2 r + 9; round j takes the slot over
    // from round j - 4, which no warp of the CTA needs any more (bounded skew: this warp
    // saw every warp of every CTA arrive at round j - 1)
    if (lane == 0) claim = atomicCAS(const_cast<uint32_t*>(rs), 2u * j + 2u, 2u * j + 9u) == 2u * j + 2u;
    claim = __shfl_sync(0xffffffffu, claim, 0);
    if (claim) {
      uint64_t tot = 0, pre = 0;
      for (uint32_t c = lane; c < gridDim.x; c += 32) {
        const uint64_t* wp = S.rstat + (uint64_t)j * gridDim.x + c;
        uint64_t w = ld_relaxed(wp);
        while ((uint32_t)(w >> 40) != S.epoch) {
          __nanosleep(32);
          w = ld_relaxed(wp);
        }
        const uint64_t a = w & ((1ull << 40) - 1);
        tot += a;
        pre += (c < blockIdx.x) ? a : 0ull;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        tot += __shfl_xor_sync(0xffffffffu, tot, o);
        pre += __shfl_xor_sync(0xffffffffu, pre, o);
      }
      if (lane == 0) {
        s_rtot[j & 3] = tot;
        s_rpre[j & 3] = pre;
        __threadfence_block();
        *rs = 2u * j + 10u;  // READY(j)
      }
      __syncwarp();
    } else {
      while (*rs != 2u * j + 10u) __nanosleep(32);
      __threadfence_block();
    }
    const uint64_t tot = *(volatile uint64_t*)&s_rtot[j & 3];
    const uint64_t pre = *(volatile uint64_t*)&s_rpre[j & 3];
    uint64_t pw = 0;  // earlier warps of this CTA (their counts are in: the CTA published)
    for (int w = 0; w < warp; ++w) pw += s_kept[j & 3][w];
    const uint64_t o0 = vbase + pre + pw;
    vbase += tot;
    if (kj == 0) return;
    if (o0 + kj > S.cap_vals) {
      if (lane == 0) atomicOr(A.ws.flags, kFlagOverflow);
      return;
    }
    uint32_t kk;
    const uint32_t lo = warp_exscan_small((uint32_t)__popc(mj), lane, kk);
    tmem_wait_st();
    double c16[16];
    tmem_load16(tx + 32u + 32u * (j % 3u), c16);
    double* dst = S.vals + o0 + lo;
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if ((mj >> r) & 1u) *dst++ = c16[r];
  };
  const uint32_t nrounds = SP ? S.nrounds : (gw < B ? (uint32_t)((B - gw + W - 1) / W) : 0u);
  for (uint32_t it = 0; it < nrounds; ++it) {
    const uint64_t blk = gw + (uint64_t)it * W;
    const uint32_t tpark = tx + 32u + (SP ? 32u * (it % 3u) : 0u);
    uint32_t mask = 0, kept = 0;
    if (!SP || blk < B) {  // warp-uniform
    double2* sb = reinterpret_cast<double2*>(wbase + st * kC8Stage);
    if constexpr (VEC) {
      static_assert(kC8Stages == 2, "one group in flight behind the consumed stage");
      cp_async_wait<1>();
      __syncwarp();
    } else {
      mbar_wait_a(bars_a + 8u * st, (ph >> st) & 1u);
      ph ^= 1u << st;
    }
    double v[16];
    // z-lines: lane = (y = l/4, q = l%4) holds x = 2q, 2q+1 of row y for all z
#pragma unroll
    for (int z = 0; z < 8; ++z) {
      const double2 t = sb[z * 32 + lane];
      v[2 * z] = t.x;
      v[2 * z + 1] = t.y;
    }
    // all-zero block (+-0 only): its coefficients are all zero, so it keeps nothing
    // -- skip the transform and the selection.  NaN / Inf / subnormal
    // bits are non-zero and take the normal path.
    uint32_t zlo = 0, zhi = 0;
#pragma unroll
    for (int r = 0; r < 16; r += 2) {
      zlo |= (uint32_t)__double2loint(v[r]) | (uint32_t)__double2loint(v[r + 1]);
      zhi |= (uint32_t)__double2hiint(v[r]) | (uint32_t)__double2hiint(v[r + 1]);
    }
    const bool zblk = !__any_sync(0xffffffffu, (zlo | (zhi & 0x7fffffffu)) != 0u);
    __syncwarp();
    if (zblk) {
      fence_proxy_async();
      __syncwarp();
      issue(blk + kC8Stages * W, st);
      st = (st + 1 == kC8Stages) ? 0 : st + 1;
      if (lane == 0) counts[blk] = 0u;
      masks16[blk * 32 + lane] = (uint16_t)0;
    } else {
#ifndef ISF_EXP_NOXFORM
    lines8<0, 2, 0, 1, 2, false>(v);  // z sweep
#endif
    // z -> y re-layout through the stage (in place): 16-B chunk c of plane kz at
    // kz * 33 + c (all reads of the stage are done)
#pragma unroll
    for (int kz = 0; kz < 8; ++kz) sb[kz * 33 + lane] = make_double2(v[2 * kz], v[2 * kz + 1]);
    __syncwarp();
    // y-lines: lane = (q = l/8, kz = l%8) holds x = 2q, 2q+1 for all y at plane kz
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const double2 t = sb[yoff + 4 * y];
      v[2 * y] = t.x;
      v[2 * y + 1] = t.y;
    }
    fence_proxy_async();
    __syncwarp();
    issue(blk + kC8Stages * W, st);  // the stage is free: refill it now
    st = (st + 1 == kC8Stages) ? 0 : st + 1;
#ifndef ISF_EXP_NOXFORM
    lines8<1, 2, 0, 1, 2, false>(v);  // y sweep: v[2 ky + x0]
#endif
    // y -> x re-layout through TMEM: store 32x32b with column pair
    // c = (ky0, x0, ky2, ky1) [bits 3..0], re-read 16x256b at lanes 0 and 16.  Reader
    // lane u gets (source lane bits 2..0, c bits 1..0) = (kz, ky2 ky1): the x-line
    // role; its double (g, j, h) of instruction g, rep j, half h holds
    // x2 = g, x1 = h, ky0 = j1, x0 = j0.
    {
      uint32_t r[32];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int ky = ((c >> 1) & 1) * 4 + (c & 1) * 2 + (c >> 3), x0 = (c >> 2) & 1;
        r[2 * c] = (uint32_t)__double2loint(v[2 * ky + x0]);
        r[2 * c + 1] = (uint32_t)__double2hiint(v[2 * ky + x0]);
      }
      tmem_st_32x32b_x32(tx, r);
      tmem_wait_st();
      uint32_t a0[16], a1[16];
      tmem_ld_16x256b_x4(tx, a0);
      tmem_ld_16x256b_x4(tx + (16u << 16), a1);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int dst = (j >> 1) * 8 + h * 2 + (j & 1);  // kyi * 8 + x, x = 4 g + 2 h + j0
          v[dst] = __hiloint2double((int)a0[4 * j + 2 * h + 1], (int)a0[4 * j + 2 * h]);
          v[dst + 4] = __hiloint2double((int)a1[4 * j + 2 * h + 1], (int)a1[4 * j + 2 * h]);
        }
    }
#ifndef ISF_EXP_NOXFORM
    lines8<2, 1, 0, 8, 2, false>(v);  // x sweep: v[r] = coefficient 16*lane + r
#endif
    // park the coefficients in TMEM (one column pair per double: no register
    // marshalling); the registers are then free for the selection
    tmem_park16(tpark, v);
#ifdef ISF_EXP_NOSEL
    Sel16 sel{0u, 1ull, 0ull, 0, false};
    if (__double_as_longlong(v[0]) == 0x1234) sel.mask = 1;
#else
    const Sel16 sel = select16(v, lane, A.eps_m, A.eps_e, hist, tpark);
#endif
    if (sel.nonfinite && lane == 0) atomicOr(A.ws.flags, kFlagNonFinite);
    mask = sel.nonfinite ? 0u : sel.mask;
    const uint32_t off = warp_exscan_small((uint32_t)__popc(mask), lane, kept);
    if (lane == 0) {
      counts[blk] = kept;  // the 16-B pad is zeroed by compact8_kernel / the last CTA
      if (!SP && kept) atomicAdd(reinterpret_cast<unsigned long long*>(A.ws.csum + (blk >> 10)), (unsigned long long)kept);
    }
    // mask words and slots are plain stores: an evict_last hint here (for
    // compact8_kernel's gather) left lines pinned in L2 that cost the next decompress
    // 9 % and this kernel 2 % (profiles/r2_summary.md)
    masks16[blk * 32 + lane] = (uint16_t)mask;
    // kept values from the parked copy into the block's slot at their natural index
    // (slot[j] = a_j for kept j): one TMEM load and sixteen predicated stores with
    // immediate offsets; compact8_kernel gathers them in index order via the mask
    if (!SP && __any_sync(0xffffffffu, mask != 0u)) {
      tmem_wait_st();
      double c16[16];
      tmem_load16(tpark, c16);
      // slot layout: natural index (j = 16 lane + r at j) for sparse blocks (<= 16 kept:
      // the few kept values share sectors), [r][lane] for dense ones (every store a
      // contiguous 256 B); compact8_kernel picks the same layout from the count
      if (kept <= 16) {
        double* dst = A.vslot + blk * 512 + 16 * lane;
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if ((mask >> r) & 1u)
            dst[r] = c16[r];
      } else {
        double* dst = A.vslot + blk * 512 + lane;
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if ((mask >> r) & 1u)
            dst[32 * r] = c16[r];
      }
    }
    if (!sel.nonfinite && sel.T) {
      if (sel.eT >= -1022 && sel.eT <= 1023 && sel.eD >= -1022 && sel.eD <= 1023) {  // exact power-of-two scales
        tot_acc = __fma_rn((double)sel.T, pow2d(sel.eT), tot_acc);
        disc_acc = __fma_rn((double)sel.hdisc, pow2d(sel.eD), disc_acc);
      } else {
        tot_acc += ldexp((double)sel.T, sel.eT);
        disc_acc += ldexp((double)sel.hdisc, sel.eD);
      }
    }
    (void)off;
    }  // non-zero block
    }  // live block
    if constexpr (SP) {
      // this CTA's aggregate of round it: the last of its 16 warps publishes it
      if (lane == 0) {
        s_kept[it & 3][warp] = kept;
        __threadfence_block();
        if (atomicAdd(&s_arrive[it & 3], 1u) == kC8Warps - 1) {
          __threadfence_block();
          uint64_t agg = 0;
          for (int w = 0; w < kC8Warps; ++w) agg += *(volatile uint32_t*)&s_kept[it & 3][w];
          s_arrive[it & 3] = 0u;
          st_relaxed(S.rstat + (uint64_t)it * gridDim.x + blockIdx.x, ((uint64_t)S.epoch << 40) | agg);
        }
      }
      __syncwarp();
      if (it >= 2) deferred(it - 2, m2, k2);
      m2 = m1; k2 = k1;
      m1 = mask; k1 = kept;
    }
  }
  if constexpr (SP) {  // the last two rounds
    if (nrounds >= 2) deferred(nrounds - 2, m2, k2);
    if (nrounds >= 1) deferred(nrounds - 1, m1, k1);
  }
  if (lane == 0) {
    A.ws.partials[gw * 4 + 0] = tot_acc;
    A.ws.partials[gw * 4 + 1] = disc_acc;
  }
  if constexpr (SP) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *S.total_out = vbase;  // every warp agrees on it
    if (last_cta(A.ws.counter + 1)) {
      if (threadIdx.x == 0) {
        uint32_t* wcounts = counts;
        for (uint64_t pb = B; pb < ((B + 3) & ~3ull); ++pb) wcounts[pb] = 0;  // pad to 16 B
        *S.total_out = vbase;
        if (vbase > S.cap_vals) atomicOr(A.ws.flags, kFlagOverflow);
        __threadfence_block();
      }
      __syncthreads();
      if (S.fin.stats) finalize_cta(S.fin, s_red);
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<c8_tmem_cols<SP>()>(tbase);
}

// --------------------------- block offsets / compact passes -----------------
// Decompress prologue: off[b] = sum of the stored counts of blocks < b (exclusive),
// off[B] = total.  CTA chunks of 1024 blocks (4 per thread) chained by a decoupled
// look-back on ws.status with a dynamic chunk claim (deadlock free).
constexpr int kOffThreads = 256;
constexpr int kOffPerThread = 4;
constexpr int kOffChunk = kOffThreads * kOffPerThread;
static_assert(kOffChunk == 1024, "compress8_kernel accumulates the chunk sums with blk >> 10");

// Deterministic reduction of the per-warp partials into isf_lossy_stats by one CTA.
__device__ void finalize_cta(const FinalizeArgs& A, double* s_red /* 4 * warps */) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double a0 = 0.0, a1 = 0.0;
  unsigned long long x0 = 0, x1 = 0;
  for (uint64_t i = tid; i < A.nparts; i += blockDim.x) {
    a0 = __dadd_rn(a0, A.partials[i * 4 + 0]);
    a1 = __dadd_rn(a1, A.partials[i * 4 + 1]);
    if (A.mode == 1) {
      unsigned long long v = (unsigned long long)__double_as_longlong(A.partials[i * 4 + 2]);
      x0 = v > x0 ? v : x0;
      v = (unsigned long long)__double_as_longlong(A.partials[i * 4 + 3]);
      x1 = v > x1 ? v : x1;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a0 = __dadd_rn(a0, __shfl_xor_sync(0xffffffffu, a0, o));
    a1 = __dadd_rn(a1, __shfl_xor_sync(0xffffffffu, a1, o));
    unsigned long long t = __shfl_xor_sync(0xffffffffu, x0, o);
    x0 = t > x0 ? t : x0;
    t = __shfl_xor_sync(0xffffffffu, x1, o);
    x1 = t > x1 ? t : x1;
  }
  if (lane == 0) {
    s_red[warp * 4 + 0] = a0;
    s_red[warp * 4 + 1] = a1;
    s_red[warp * 4 + 2] = __longlong_as_double((long long)x0);
    s_red[warp * 4 + 3] = __longlong_as_double((long long)x1);
  }
  __syncthreads();
  if (tid == 0) {
    double s0 = 0.0, s1 = 0.0;
    unsigned long long m0 = 0, m1 = 0;
    for (int w = 0; w < nw; ++w) {
      s0 = __dadd_rn(s0, s_red[w * 4]);
      s1 = __dadd_rn(s1, s_red[w * 4 + 1]);
      const unsigned long long t0 = (unsigned long long)__double_as_longlong(s_red[w * 4 + 2]);
      const unsigned long long t1 = (unsigned long long)__double_as_longlong(s_red[w * 4 + 3]);
      m0 = t0 > m0 ? t0 : m0;
      m1 = t1 > m1 ? t1 : m1;
    }
    double* st = reinterpret_cast<double*>(A.stats);
    uint64_t* su = reinterpret_cast<uint64_t*>(A.stats);
    const uint64_t total = *A.total_ptr;
    for (int i = 0; i < 12; ++i) su[i] = 0;
    if (A.mode == 0) {
      st[4] = s1;  // disc2
      st[5] = s0;  // tot2
    } else if (A.with_error) {
      st[0] = s0;
      st[1] = s1;
      st[2] = __longlong_as_double((long long)m0);
      st[3] = __longlong_as_double((long long)m1);
    }
    su[6] = total;
    su[7] = A.nblocks;
    if (A.density) {  // zero-copy into pinned host memory: read (stale-tolerant) by the next call
      A.density[1] = A.nblocks * 512ull;
      A.density[0] = total;
    }
    su[8] = A.val_off + 8 * total;
    su[9] = A.field_bytes;
    su[10] = *A.flags;
    *A.flags = 0;
  }
}

// Last-CTA election for the fused finalize; `done` is reset by the winner.
__device__ __forceinline__ bool last_cta(uint32_t* done) {
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    if (s_last) {
      *done = 0;
      __threadfence();
    }
  }
  __syncthreads();
  return s_last != 0;
}

__global__ void __launch_bounds__(kOffThreads) block_offsets8_kernel(const uint8_t* stream, uint64_t nblocks,
                                                                    uint64_t* off, Workspace ws, FinalizeArgs fin) {
  __shared__ uint64_t wsum[kOffThreads / 32];
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_chunk;
  __shared__ double s_red[4 * (kOffThreads / 32)];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(stream);
  const uint32_t nchunks = (uint32_t)((nblocks + kOffChunk - 1) / kOffChunk);
  pdl_wait();
  pdl_launch_dependents();
  for (;;) {
    if (tid == 0) {
      const uint32_t c = atomicAdd(ws.counter, 1u);
      if (c == nchunks + ws.total_warps - 1) *ws.counter = 0;
      s_chunk = c;
    }
    __syncthreads();
    const uint32_t chunk = s_chunk;
    if (chunk >= nchunks) break;
    const uint64_t b0 = (uint64_t)chunk * kOffChunk + (uint64_t)tid * kOffPerThread;
    uint4 c4 = make_uint4(0, 0, 0, 0);
    if (b0 < nblocks) c4 = *(reinterpret_cast<const uint4*>(counts) + b0 / 4);  // counts padded to 16 B
    if (b0 + 1 >= nblocks) c4.y = 0;
    if (b0 + 2 >= nblocks) c4.z = 0;
    if (b0 + 3 >= nblocks) c4.w = 0;
    const uint64_t v = (uint64_t)c4.x + c4.y + c4.z + c4.w;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint64_t wex = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < kOffThreads / 32; ++w) {
      wex += (w < warp) ? wsum[w] : 0ull;
      agg += wsum[w];
    }
    if (warp == 0) {
      const uint64_t pre = warp_lookback(ws.status, chunk, agg, ws.epoch);
      if (lane == 0) s_prefix = pre;
    }
    __syncthreads();
    const uint64_t e0 = s_prefix + wex + x - v;
    const uint64_t e1 = e0 + c4.x, e2 = e1 + c4.y, e3 = e2 + c4.z;
    if (b0 < nblocks) {  // off[] is 8-byte aligned only: scalar stores
      off[b0] = e0;
      if (b0 + 1 < nblocks) off[b0 + 1] = e1;
      if (b0 + 2 < nblocks) off[b0 + 2] = e2;
      if (b0 + 3 < nblocks) off[b0 + 3] = e3;
      if (b0 + 4 >= nblocks) off[nblocks] = e0 + v;
    }
    __syncthreads();
  }
  if (fin.stats && last_cta(ws.counter + 1)) finalize_cta(fin, s_red);
}

// Compress epilogue: pack the kept values from their per-block slots into the value
// region of the stream.  CTA c < nchunks owns chunk c (1024 blocks, one per thread):
// its value offset is the sum of the per-chunk kept counts compress8_kernel
// accumulated in csum (no look-back chain), the in-chunk offsets a block scan.  CTA
// nchunks clears the other csum buffer (used by the next call) and reduces the
// statistics, concurrently with the copies.
// Compress epilogue: one CTA per 1024-block chunk, 512 threads, two blocks per thread
// (64 registers: every mask word and value load of a sparse block in flight at once;
// the 1024-thread / 32-register version walked the mask words in dependent rounds).
constexpr int kCompactThreads = 512;
static_assert(2 * kCompactThreads == kOffChunk, "two blocks of a chunk per thread");

// up to 16 kept values of a sparse block (slot in natural index order): all mask words,
// then all loads, then all stores
__device__ __forceinline__ void sparse_copy16(const double* src, const uint4* m4, double* dst, uint32_t c) {
  uint64_t mw[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 t = m4[q];  // plain load: the masks stay in L2 for the decompress that follows
    mw[2 * q] = ((uint64_t)t.y << 32) | t.x;
    mw[2 * q + 1] = ((uint64_t)t.w << 32) | t.z;
  }
  uint32_t nz = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) nz |= (mw[w] ? 1u : 0u) << w;
  uint64_t mm = 0;
  int wb = 0;
  double v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    v[k] = 0.0;
    if ((uint32_t)k < c) {
      if (mm == 0) {  // next non-empty word (a select chain: no dynamic register index)
        const int w = __ffs(nz) - 1;
        nz &= nz - 1;
        uint64_t t = mw[0];
#pragma unroll
        for (int q = 1; q < 8; ++q) t = w == q ? mw[q] : t;
        mm = t;
        wb = 64 * w;
      }
      const int j = wb + __ffsll((long long)mm) - 1;
      mm &= mm - 1;
      v[k] = __ldcs(src + j);
    }
  }
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if ((uint32_t)k < c) dst[k] = v[k];
}

__global__ void __launch_bounds__(kCompactThreads, 2) compact8_kernel(uint8_t* stream, uint64_t nblocks, uint64_t mask_off,
                                                                  const uint64_t* csum, uint64_t* csum_next,
                                                                  const double* vslot, double* vals,
                                                                  uint64_t cap_vals, uint64_t* total_out,
                                                                  uint32_t nclear, FinalizeArgs fin) {
  constexpr int NW = kCompactThreads / 32;
  __shared__ uint64_t s_w[2 * NW];
  __shared__ uint64_t s_prefix;
  __shared__ double s_red[4 * NW];
  __shared__ uint64_t s_off[2 * kCompactThreads];  // dense list: value offsets
  __shared__ uint16_t s_dense[2 * kCompactThreads];
  __shared__ uint32_t s_ndense;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nchunks = (uint32_t)((nblocks + kOffChunk - 1) / kOffChunk);
  const uint32_t chunk = blockIdx.x;
  pdl_wait();
  pdl_launch_dependents();
  if (chunk == nchunks) {
    for (uint32_t c = tid; c < nclear; c += kCompactThreads) csum_next[c] = 0;  // high-water mark of all calls
    uint64_t a = 0;
    for (uint32_t c = tid; c < nchunks; c += kCompactThreads) a += csum[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) s_w[warp] = a;
    __syncthreads();
    if (tid == 0) {
      uint64_t t = 0;
      for (int w = 0; w < NW; ++w) t += s_w[w];
      *total_out = t;
      if (t > cap_vals) atomicOr(fin.flags, kFlagOverflow);
      uint32_t* counts = reinterpret_cast<uint32_t*>(stream);
      for (uint64_t pb = nblocks; pb < ((nblocks + 3) & ~3ull); ++pb) counts[pb] = 0;  // 16-B pad
      __threadfence_block();
    }
    __syncthreads();
    if (fin.stats) finalize_cta(fin, s_red);
    return;
  }
  if (warp == 0) {  // chunk prefix: the sum of the earlier chunks' kept counts
    uint64_t a = 0;
#pragma unroll 8
    for (uint32_t c = lane; c < chunk; c += 32) a += csum[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
      s_prefix = a;
      s_ndense = 0;
    }
  }
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(stream);
  const uint16_t* masks16 = reinterpret_cast<const uint16_t*>(stream + mask_off);  // 32 words per block
  const uint64_t b0 = (uint64_t)chunk * kOffChunk + tid, b1 = b0 + kCompactThreads;
  const uint32_t c0 = b0 < nblocks ? counts[b0] : 0u, c1 = b1 < nblocks ? counts[b1] : 0u;
  uint32_t x0 = c0, x1 = c1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t0 = __shfl_up_sync(0xffffffffu, x0, o), t1 = __shfl_up_sync(0xffffffffu, x1, o);
    if (lane >= o) {
      x0 += t0;
      x1 += t1;
    }
  }
  if (lane == 31) {
    s_w[warp] = x0;
    s_w[NW + warp] = x1;
  }
  __syncthreads();
  uint64_t w0 = 0, w1 = 0, t0 = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    w0 += w < warp ? s_w[w] : 0ull;
    w1 += w < warp ? s_w[NW + w] : 0ull;
    t0 += s_w[w];
  }
  const uint64_t e0 = s_prefix + w0 + x0 - c0, e1 = s_prefix + t0 + w1 + x1 - c1;  // the blocks' first values
  // Sparse blocks (<= 16 kept, slot in natural index order) are copied by their thread.
  // Dense blocks (slot layout [r][lane]) go to a list that whole warps pack below
  // (thread-serial copies of hundreds of values would dominate).
  if (c0 > 16 && e0 + c0 <= cap_vals) {
    const uint32_t k = atomicAdd(&s_ndense, 1u);
    s_dense[k] = (uint16_t)tid;
    s_off[k] = e0;
  }
  if (c1 > 16 && e1 + c1 <= cap_vals) {
    const uint32_t k = atomicAdd(&s_ndense, 1u);
    s_dense[k] = (uint16_t)(tid + kCompactThreads);
    s_off[k] = e1;
  }
  if (c0 && c0 <= 16 && e0 + c0 <= cap_vals)
    sparse_copy16(vslot + b0 * 512, reinterpret_cast<const uint4*>(masks16 + b0 * 32), vals + e0, c0);
  if (c1 && c1 <= 16 && e1 + c1 <= cap_vals)
    sparse_copy16(vslot + b1 * 512, reinterpret_cast<const uint4*>(masks16 + b1 * 32), vals + e1, c1);
  __syncthreads();
  // dense blocks: lane l owns the block's coefficients 16 l .. 16 l + 15 (mask word l),
  // so the slot reads and the packed writes of a warp are both contiguous
  const uint32_t nd = s_ndense;
  for (uint32_t i = warp; i < nd; i += NW) {
    const uint64_t bb = (uint64_t)chunk * kOffChunk + s_dense[i];
    const uint32_t m = masks16[bb * 32 + lane];
    uint32_t kept;
    const uint32_t off = warp_exscan_small((uint32_t)__popc(m), lane, kept);
    const double* src = vslot + bb * 512 + lane;
    double* dst = vals + s_off[i] + off;
    double v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = ((m >> r) & 1u) ? __ldcs(src + 32 * r) : 0.0;
    int k = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if ((m >> r) & 1u) dst[k++] = v[r];
  }
}

// Two inverse lines (offsets O0, O1, stride S) of lx = 8 whose coefficients at
// positions 4..7 are all zero (the common case after truncation): the pinned
// even/odd chains of inv_line restricted to k = 0..3, started from +0 with an fma.
// Leaving out terms b*(+-0) and replacing the first product by fma(b, a, +0) change
// nothing but the sign of zero: every intermediate keeps the real value of the
// dense chain, sweep after sweep, and the +0 canonicalisation of the reconstruction
// (applied by the oracle too) makes the bits identical.
// One line of inv2_low8 (same chains).
template <int S, int O, int T, int N>
__device__ __forceinline__ void inv1_low8(double (&v)[N]) {
  const double a[4] = {v[O], v[O + S], v[O + 2 * S], v[O + 3 * S]};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double e = __fma_rn(Bm<8, T>(i, 2), a[2], __fma_rn(Bm<8, T>(i, 0), a[0], 0.0));
    const double d = __fma_rn(Bm<8, T>(i, 3), a[3], __fma_rn(Bm<8, T>(i, 1), a[1], 0.0));
    v[O + i * S] = __dadd_rn(e, d);
    v[O + (7 - i) * S] = __dsub_rn(e, d);
  }
}
template <int S, int O0, int O1, int T, int N>
__device__ __forceinline__ void inv2_low8(double (&v)[N]) {
  const double a0[4] = {v[O0], v[O0 + S], v[O0 + 2 * S], v[O0 + 3 * S]};
  const double a1[4] = {v[O1], v[O1 + S], v[O1 + 2 * S], v[O1 + 3 * S]};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double e0 = __fma_rn(Bm<8, T>(i, 2), a0[2], __fma_rn(Bm<8, T>(i, 0), a0[0], 0.0));
    const double d0 = __fma_rn(Bm<8, T>(i, 3), a0[3], __fma_rn(Bm<8, T>(i, 1), a0[1], 0.0));
    const double e1 = __fma_rn(Bm<8, T>(i, 2), a1[2], __fma_rn(Bm<8, T>(i, 0), a1[0], 0.0));
    const double d1 = __fma_rn(Bm<8, T>(i, 3), a1[3], __fma_rn(Bm<8, T>(i, 1), a1[1], 0.0));
    v[O0 + i * S] = __dadd_rn(e0, d0);
    v[O0 + (7 - i) * S] = __dsub_rn(e0, d0);
    v[O1 + i * S] = __dadd_rn(e1, d1);
    v[O1 + (7 - i) * S] = __dsub_rn(e1, d1);
  }
}

// --------------------------- decompress -------------------------------------
// stage: [96, ...) the block's values (16-B aligned bulk copy); [0, 96) unused
constexpr int kD8Stage = 8 * 36 * 16;  // >= 96 + 4096 + 32 (values) and the re-layout planes
constexpr int kD8StageBytes = (kD8Stage + 127) & ~127;
constexpr int kD8WarpBytes = kF8Stages * kD8StageBytes + 128;  // stages | mbarriers
template <bool ERR>
__host__ __device__ constexpr int d8_smem() { return d8_warps<ERR>() * kD8WarpBytes; }
// vector fields (components = 3): 15 warps per CTA = the 3 components of 5 elements per
// round, reconstructed into a shared-memory copy of those elements (point-major,
// component-minor) and written out with coalesced 128-bit stores (12 warps with a
// double buffer and one barrier per round measured 7 % slower: fewer warps)
// plain scalar decode: each block's reconstruction leaves through one TMA bulk store
// (evict-first) from the stage instead of eight 128-bit streaming stores per lane
// (decompress 5.95 -> 6.06 TB/s, profiles/r2_summary.md)
#ifndef ISF_D8_TMASTORE
#define ISF_D8_TMASTORE 1
#endif
#ifndef ISF_D8V_WARPS
#define ISF_D8V_WARPS 15
#endif
#ifndef ISF_D8V_TMA
#define ISF_D8V_TMA 1
#endif
constexpr int kD8VecWarps = ISF_D8V_WARPS;
constexpr int kD8VecElems = kD8VecWarps / 3;
constexpr int kD8VecBufs = kD8VecWarps <= 12 ? 2 : 1;  // element buffers per element (double buffer if it fits)
constexpr int d8_vec_smem() { return kD8VecWarps * kD8WarpBytes + kD8VecBufs * kD8VecElems * 1536 * 8; }

struct Decompress8Args {
  DecompressArgs d;
  const uint64_t* off;  // block value offsets (block_offsets8_kernel), off[B] = total
  FinalizeArgs fin;     // fused finalize by the last CTA
};

// ERR: also read the original and accumulate the error report (separate instantiation
// so the plain decode does not carry the accumulators' registers)
template <bool ERR, bool VEC = false>
__global__ void __launch_bounds__((VEC ? kD8VecWarps : d8_warps<ERR>()) * 32) decompress8_kernel(Decompress8Args P) {
  constexpr int kNW = VEC ? kD8VecWarps : d8_warps<ERR>();
  static_assert(!(VEC && ERR), "the error report of vector fields takes the strided path");
  const DecompressArgs& A = P.d;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wbase = smem + warp * kD8WarpBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + kF8Stages * kD8StageBytes);
  const int kzp = lane >> 2, qp = lane & 3;
  const int q = lane & 3, y = lane >> 2;
  // re-layout addresses: 16-B chunk (kz, ky, x pair xq) at kz * 36 + 4 ky + ky / 2 + xq,
  // conflict free for the x-line stores, y-line loads / stores and z-line loads and
  // affine in every loop index (immediate offsets from one base per role)
  const int xoff = kzp * 36 + 9 * qp;            // x-lines: ky = 2 qp + kyi
  const int yoff = kzp * 36 + qp;                // y-lines: + 4 ky + ky / 2
  const int zoff = 4 * y + (y >> 1) + q;         // z-lines: + 36 z
  const uint64_t W = (uint64_t)gridDim.x * kNW;
  const uint64_t gw = (uint64_t)blockIdx.x * kNW + warp;
  const uint64_t B = A.nblocks;
  const uint64_t sb_floor16 = A.stream_bytes & ~15ull;
  const double wxy0 = __dmul_rn(Wg<8>(2 * q), Wg<8>(y));
  const double wxy1 = __dmul_rn(Wg<8>(2 * q + 1), Wg<8>(y));
  double e2 = 0.0, n2 = 0.0;
  uint64_t einf = 0, uinf = 0;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kF8Stages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  pdl_wait();
  pdl_launch_dependents();
  const uint64_t pol_out = l2_policy_evict_first();  // output and staged values are streamed
  // the TMA stage only carries the block's value range; offsets (from the counts) and
  // the lane's 16-bit mask word travel in registers, loaded two blocks ahead
  auto issue = [&](uint64_t blk, int st, uint64_t o0, uint64_t o1) {
    if (lane == 0 && blk < B) {
      unsigned char* sp = wbase + st * kD8StageBytes;
      const uint64_t a0 = (A.val_off + 8 * o0) & ~15ull;
      uint64_t a1 = (A.val_off + 8 * o1 + 15) & ~15ull;
      if (a1 > sb_floor16) a1 = sb_floor16;
      const uint32_t vbytes = (a1 > a0 && o1 - o0 <= 512) ? (uint32_t)(a1 - a0) : 0u;
      mbar_arrive_tx(&bars[st], vbytes);
      // the values are read once: evict-first, as the output (+0.8 % decompress)
      if (vbytes) bulk_g2s_hint(sp + 96, A.stream + a0, vbytes, &bars[st], pol_out);
    }
  };
  const uint16_t* masks16 = reinterpret_cast<const uint16_t*>(A.stream + A.mask_off);
  static_assert(kF8Stages == 2, "offset pipeline assumes two stages");
  // offsets and masks of the current block and the next one (loaded one iteration ahead)
  uint64_t o0 = 0, o1 = 0, p0 = 0, p1 = 0;
  uint32_t mc = 0, mn = 0;
  if (gw < B) { o0 = P.off[gw]; o1 = P.off[gw + 1]; mc = __ldg(masks16 + gw * 32 + lane); }
  if (gw + W < B) { p0 = P.off[gw + W]; p1 = P.off[gw + W + 1]; mn = __ldg(masks16 + (gw + W) * 32 + lane); }
  issue(gw, 0, o0, o1);
  issue(gw + W, 1, p0, p1);
  int st = 0;
  uint32_t ph = 0;
  // VEC: every warp runs every round (the CTA writes its 5 elements after a barrier)
  double* obuf = reinterpret_cast<double*>(smem + kNW * kD8WarpBytes);
  __shared__ uint64_t s_ebar[VEC ? kD8VecElems : 1];  // VEC + TMA store: element buffer free
  if constexpr (VEC) {
    if (threadIdx.x < kD8VecElems) mbar_init(&s_ebar[threadIdx.x], 1);
    fence_mbar_init();
    __syncthreads();
  }
  const uint64_t nrounds = VEC ? (B + W - 1) / W : 0;
  for (uint64_t it = 0, blk = gw; VEC ? it < nrounds : blk < B; ++it, blk += W) {
    if (!VEC || blk < B) {
    unsigned char* sp = wbase + st * kD8StageBytes;
    uint64_t r0 = 0, r1 = 0;  // offsets / mask of blk + 2W, consumed by the refill below
    uint32_t mr = 0;
    if (blk + 2 * W < B) {
      r0 = P.off[blk + 2 * W];
      r1 = P.off[blk + 2 * W + 1];
      mr = __ldg(masks16 + (blk + 2 * W) * 32 + lane);
    }
    mbar_wait(&bars[st], (ph >> st) & 1u);
    ph ^= 1u << st;
    uint32_t m = mc;
    const uint32_t pc = (uint32_t)__popc(m);
    uint32_t tot;  // pc <= 16: five independent ballots instead of a dependent shuffle scan
    const uint32_t inoff = warp_exscan_small(pc, lane, tot);
    // o1 - o0 is the block's stored count (block_offsets8_kernel scanned the counts)
    const bool ok = tot == o1 - o0 && A.val_off + 8 * o1 <= A.stream_bytes;
    if (!ok) {
      if (lane == 0) atomicOr(A.ws.flags, kFlagShape);
      m = 0;
    }
    // Occupied Legendre indices of the block (warp-uniform): lane l holds kz = l/4,
    // ky = 2(l%4) (mask bits 0-7) and 2(l%4)+1 (bits 8-15), kx = bit % 8.  Sweeps skip
    // the all-zero index planes 4..7 when they can; inv2_low8 says why that is exact.
    const uint32_t occ = __reduce_or_sync(
        0xffffffffu, ((m | (m >> 8)) & 0xffu) | (((m & 0xffu) ? 1u : 0u) << (8 + 2 * qp)) |
                         (((m >> 8) ? 1u : 0u) << (9 + 2 * qp)) | ((m ? 1u : 0u) << (16 + kzp)));
    const uint32_t Kx = occ & 0xffu, Ky = (occ >> 8) & 0xffu, Kz = occ >> 16;
    // the final 8 bytes of a stream whose length is 8 mod 16 are not in the bulk copy
    const double* sv0 = reinterpret_cast<const double*>(sp + 96) + (((A.val_off + 8 * o0) & 15ull) >> 3);
    if (Kz && A.val_off + 8 * o1 > sb_floor16) {
      if (lane == 0)
        const_cast<double*>(sv0)[o1 - 1 - o0] =
            reinterpret_cast<const double*>(A.stream + A.val_off)[(A.stream_bytes - A.val_off) / 8 - 1];
      __syncwarp();
    }
    double v[16];
    const bool lowz = Kz < 16u;
    if (!ERR && (Kx | Ky | Kz) < 16u) {  // (the error-report instantiation keeps the
      // general path: the extra live state would spill)
      // Low cube (the common smooth case): every kept coefficient has kx, ky, kz < 4.
      // The inverse then runs on 16 x-lines, 32 y-lines and 64 z-lines instead of 64
      // each, one line per lane for x and y (the same pinned chains as inv2_low8),
      // with two small padded shared-memory re-layouts: line m at 10 m + (m >> 3), which
      // keeps every half-warp's 16 doubles in distinct bank pairs for the x-line stores,
      // the y-line loads and stores and the z-line loads (a stride of 9 was 2-way
      // conflicted on the y-line loads and the z-line loads).
      double* fx = reinterpret_cast<double*>(sp);  // [16 x-lines (kz, ky)]: 10 L + (L >> 3) + x
      double* fy = fx + 160;                       // [32 y-lines (kz, x)]:  10 M + (M >> 3) + y
      {
        const int L = lane & 15, lky = L & 3;
        const int ml = 4 * (L >> 2) + (lky >> 1);  // mask lane of the line (kz, ky)
        const uint32_t mw = __shfl_sync(0xffffffffu, m, ml);
        const uint32_t bse = __shfl_sync(0xffffffffu, inoff, ml);
        const uint32_t lb = (lky & 1) ? 8u : 0u;
        double a8[8];
        // running offset over this line's four mask bits (one popcount for the low half)
        const uint32_t mh = mw >> lb;
        const double* sl = sv0 + bse + (lb ? (uint32_t)__popc(mw & 0xffu) : 0u);
#pragma unroll
        for (int kx = 0; kx < 4; ++kx) {
          const uint32_t b = (mh >> kx) & 1u;
          a8[kx] = b ? *sl : 0.0;
          sl += b;
        }
        inv1_low8<1, 0, 0>(a8);  // inverse x sweep
        __syncwarp();            // the values region is read: reuse the stage
        if (lane < 16) {
#pragma unroll
          for (int x = 0; x < 8; ++x) fx[L * 10 + (L >> 3) + x] = a8[x];
        }
      }
      __syncwarp();
      {
        const int ykz = lane >> 3, yx = lane & 7;
        double b8[8];
#pragma unroll
        for (int ky = 0; ky < 4; ++ky) b8[ky] = fx[(4 * ykz + ky) * 10 + (ykz >> 1) + yx];
        inv1_low8<1, 0, 1>(b8);  // inverse y sweep
#pragma unroll
        for (int yy = 0; yy < 8; ++yy) fy[(8 * ykz + yx) * 10 + ykz + yy] = b8[yy];
      }
      __syncwarp();
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        v[2 * z] = fy[(8 * z + 2 * q) * 10 + z + y];
        v[2 * z + 1] = fy[(8 * z + 2 * q + 1) * 10 + z + y];
      }
    } else {
    const double* sv = sv0 + inoff;
    if (Kx < 16u) {  // warp-uniform: only kx 0..3 occupied
      int o = 0;  // running value index (bits 4..7 and 12..15 are clear here)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool b = (m >> k) & 1u;
        v[k] = b ? sv[o] : 0.0;
        o += b;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool b = (m >> (8 + k)) & 1u;
        v[8 + k] = b ? sv[o] : 0.0;
        o += b;
      }
      __syncwarp();
      inv2_low8<1, 0, 8, 0>(v);
    } else {
      int o = 0;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = ((m >> r) & 1u) ? sv[o++] : 0.0;
      __syncwarp();
      lines8<0, 1, 0, 8, 2, true>(v);
    }
    double2* sb = reinterpret_cast<double2*>(sp);
    // Rows that are all zero and never read again are not moved: with Ky < 16 the
    // y-lines only read ky < 4, with Kz < 16 the z-lines only read planes kz < 4, so
    // lanes of planes kz >= 4 skip their stores and loads (their sweeps run on stale
    // registers whose results are dropped) -- fewer shared-memory wavefronts.
    const bool zlive = !lowz || kzp < 4;
#pragma unroll
    for (int kyi = 0; kyi < 2; ++kyi)
#pragma unroll
      for (int qq = 0; qq < 4; ++qq)
        if (zlive && (Ky >= 16u || 2 * qp + kyi < 4))
          sb[xoff + 4 * kyi + qq] = make_double2(v[kyi * 8 + 2 * qq], v[kyi * 8 + 2 * qq + 1]);
    __syncwarp();
    if (Ky < 16u) {
#pragma unroll
      for (int ky = 0; ky < 4; ++ky)
        if (zlive) {
          const double2 t = sb[yoff + 4 * ky + (ky >> 1)];
          v[2 * ky] = t.x;
          v[2 * ky + 1] = t.y;
        }
      __syncwarp();
      inv2_low8<2, 0, 1, 1>(v);
    } else {
#pragma unroll
      for (int ky = 0; ky < 8; ++ky)
        if (zlive) {
          const double2 t = sb[yoff + 4 * ky + (ky >> 1)];
          v[2 * ky] = t.x;
          v[2 * ky + 1] = t.y;
        }
      __syncwarp();
      lines8<1, 2, 0, 1, 2, true>(v);
    }
#pragma unroll
    for (int yy = 0; yy < 8; ++yy)
      if (zlive) sb[yoff + 4 * yy + (yy >> 1)] = make_double2(v[2 * yy], v[2 * yy + 1]);
    __syncwarp();
#pragma unroll
    for (int z = 0; z < 8; ++z)
      if (z < 4 || !lowz) {
        const double2 t = sb[z * 36 + zoff];
        v[2 * z] = t.x;
        v[2 * z + 1] = t.y;
      }
    }
    // TS (scalar plain decode): the stage also carries the reconstruction out through
    // one TMA bulk store, so its refill waits for that store's read
    constexpr bool TS = ISF_D8_TMASTORE && !ERR && !VEC;
    const int st_cur = st;
    if constexpr (!TS) {
      fence_proxy_async();
      __syncwarp();
      issue(blk + 2 * W, st, r0, r1);
    }
    st ^= 1;
    o0 = p0; o1 = p1;
    const uint64_t rr0 = r0, rr1 = r1;
    p0 = r0; p1 = r1;
    mc = mn; mn = mr;
    if (lowz) inv2_low8<2, 0, 1, 2>(v); else lines8<2, 2, 0, 1, 2, true>(v);  // inverse z sweep
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = __dadd_rn(v[r], 0.0);  // zeros as +0
    if constexpr (TS) {
      double2* so = reinterpret_cast<double2*>(wbase + st_cur * kD8StageBytes);
      __syncwarp();  // every lane's z-line loads of the stage are done
#pragma unroll
      for (int z = 0; z < 8; ++z) so[z * 32 + lane] = make_double2(v[2 * z], v[2 * z + 1]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        bulk_s2g_hint(A.out + blk * 512, so, 4096u, pol_out);  // (no hint: -15 %)
        bulk_commit();
      }
      // the stage is read: refill it (waiting here measured faster than deferring the
      // wait and the refill to the next block's start: 6.06 vs 6.00 TB/s)
      if (lane == 0) bulk_wait_read0();
      issue(blk + 2 * W, st_cur, rr0, rr1);
    }
    // vector field (the block is every third double of its element): VEC stages the
    // CTA's elements in shared memory; the error-report instantiation stores strided
    const bool vec = ERR && A.comps == 3;
    if constexpr (VEC) {
#if ISF_D8V_TMA
      // the element buffer's previous store has been read (one-way: the issuing thread
      // arrived after its bulk read; a whole block of work ago, so this rarely waits)
      if (kD8VecBufs == 1 && it > 0) mbar_wait(&s_ebar[warp / 3], (uint32_t)((it - 1) & 1));
#endif
      // element warp / 3 of the CTA's round, component warp % 3 (the round's first block
      // is a multiple of 3: 15 blocks per CTA, 15 x grid per round)
      double* ov = obuf + ((kD8VecBufs == 2 ? (it & 1) * kD8VecElems : 0) + warp / 3) * 1536 + (warp % 3) + 3 * (2 * q + 8 * y);
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        ov[192 * z] = v[2 * z];
        ov[192 * z + 3] = v[2 * z + 1];
      }
    } else if (vec) {
      double* dv = A.out + (blk / 3) * 1536 + (blk % 3) + 3 * (2 * q + 8 * y);
#pragma unroll
      for (int z = 0; z < 8; ++z) {  // plain stores: L2 merges the three components' sectors
        dv[192 * z] = v[2 * z];
        dv[192 * z + 3] = v[2 * z + 1];
      }
    } else if (!ISF_D8_TMASTORE || ERR) {
      double2* dst = reinterpret_cast<double2*>(A.out + blk * 512) + lane;
#pragma unroll
      for (int z = 0; z < 8; ++z) stg_stream(dst + z * 32, make_double2(v[2 * z], v[2 * z + 1]));
    }
    if (ERR) {
      const double2* src = reinterpret_cast<const double2*>(A.orig + blk * 512) + lane;
      const double* sv3 = A.orig + (blk / 3) * 1536 + (blk % 3) + 3 * (2 * q + 8 * y);
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        const double2 o = vec ? make_double2(__ldcs(sv3 + 192 * z), __ldcs(sv3 + 192 * z + 3)) : ldg_stream(src + z * 32);
        const double wz = Wg<8>(z);
        const double w0 = __dmul_rn(wxy0, wz), w1 = __dmul_rn(wxy1, wz);
        const double da = __dsub_rn(o.x, v[2 * z]), db = __dsub_rn(o.y, v[2 * z + 1]);
        e2 = __fma_rn(__dmul_rn(w0, da), da, e2);
        e2 = __fma_rn(__dmul_rn(w1, db), db, e2);
        n2 = __fma_rn(__dmul_rn(w0, o.x), o.x, n2);
        n2 = __fma_rn(__dmul_rn(w1, o.y), o.y, n2);
        uint64_t t;
        t = abs_bits(da); einf = t > einf ? t : einf;
        t = abs_bits(db); einf = t > einf ? t : einf;
        t = abs_bits(o.x); uinf = t > uinf ? t : uinf;
        t = abs_bits(o.y); uinf = t > uinf ? t : uinf;
      }
    }
    }  // live block
    if constexpr (VEC) {
      // the 3 warps of element warp / 3 meet on their own named barrier (96 threads), so
      // elements proceed independently: the element is in obuf -> its 12 KiB go out with
      // 128-bit stores by those 96 threads -> the buffer is free for the next round
      const uint32_t le = (uint32_t)warp / 3u;
      const uint64_t e = (blockIdx.x * (uint64_t)kNW + it * W) / 3 + le;
#if ISF_D8V_TMA
      // one bulk copy (TMA engine) per element: the writers' generic-proxy stores are
      // made visible to the async proxy, then one thread of the element's first warp
      // issues the 12 KiB store and, before the buffer is rewritten, waits for its reads
      fence_proxy_async();
      // double buffer: the previous round's store (its buffer is rewritten next round,
      // after this barrier) has finished reading
      if constexpr (kD8VecBufs == 2) {
        if (warp % 3 == 0 && lane == 0) bulk_wait_read0();
      }
      asm volatile("bar.sync %0, 96;" ::"r"(1u + le) : "memory");
      if (warp % 3 == 0 && lane == 0) {
        if (e < B / 3) {
          bulk_s2g_hint(A.out + e * 1536, obuf + ((kD8VecBufs == 2 ? (it & 1) * kD8VecElems : 0) + le) * 1536, 1536 * 8,
                        pol_out);  // streamed like the scalar path's block stores
          bulk_commit();
        }
        if constexpr (kD8VecBufs == 1) {
          bulk_wait_read0();
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s_ebar[le])) : "memory");
        }
      }
#else
      asm volatile("bar.sync %0, 96;" ::"r"(1u + le) : "memory");
      if (e < B / 3) {
        const double2* src = reinterpret_cast<const double2*>(
            obuf + ((kD8VecBufs == 2 ? (it & 1) * kD8VecElems : 0) + le) * 1536);
        double2* dst = reinterpret_cast<double2*>(A.out + e * 1536);
        const uint32_t t = (uint32_t)(warp % 3) * 32u + (uint32_t)lane;
#pragma unroll
        for (int i = 0; i < 8; ++i) stg_stream(dst + t + 96 * i, src[t + 96 * i]);
      }
#endif
#if !ISF_D8V_TMA
      // single buffer: wait until the element is out before the next round overwrites it
      // (double buffer: the next round's barrier already orders it)
      if constexpr (kD8VecBufs == 1) asm volatile("bar.sync %0, 96;" ::"r"(1u + le) : "memory");
#endif
    }
  }
  if (ERR) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      e2 = __dadd_rn(e2, __shfl_xor_sync(0xffffffffu, e2, o));
      n2 = __dadd_rn(n2, __shfl_xor_sync(0xffffffffu, n2, o));
      uint64_t t = __shfl_xor_sync(0xffffffffu, einf, o); einf = t > einf ? t : einf;
      t = __shfl_xor_sync(0xffffffffu, uinf, o); uinf = t > uinf ? t : uinf;
    }
    if (lane == 0) {
      A.ws.partials[gw * 4 + 0] = e2;
      A.ws.partials[gw * 4 + 1] = n2;
      A.ws.partials[gw * 4 + 2] = __longlong_as_double((long long)einf);
      A.ws.partials[gw * 4 + 3] = __longlong_as_double((long long)uinf);
    }
  }
#if ISF_D8V_TMA
  if constexpr (VEC) {
    if (warp % 3 == 0 && lane == 0) bulk_wait0();  // the element stores are complete
  }
#endif
  if constexpr (ISF_D8_TMASTORE && !ERR && !VEC) {
    if (lane == 0) bulk_wait0();  // the block stores are complete
  }
  __shared__ double s_red[4 * kNW];
  if (last_cta(A.ws.counter + 1)) finalize_cta(P.fin, s_red);
}

}  // namespace dev
}  // namespace isf
