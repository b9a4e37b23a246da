// dlt_kernels.cuh -- the sm_100a kernels of the hot path.
//
//  (the lx = 8 scalar-field fast path lives in dlt_fast8.cuh)
//  compress_generic / decompress_generic : any lx in [2,16], components 1 or 3; one
//      CTA per block, sweeps through shared memory, selection on warp 0.
//  finalize_kernel : deterministic fixed-tree reduction of per-tile partials.
#pragma once
#include "dlt_common.cuh"

namespace isf {
namespace dev {

struct Workspace {
  uint64_t* status;            // look-back descriptors, one per tile
  double* partials;            // per-tile partial sums (4 doubles per tile)
  uint32_t* counter;           // dynamic tile counter
  unsigned long long* flags;   // ISF_STATUS_* bits (reset by finalize)
  uint32_t epoch;
  uint32_t ntiles;
  uint32_t total_warps;        // warps (fast) or CTAs (generic) claiming tiles
  uint64_t* csum = nullptr;    // lx = 8 compress: kept count per 1024-block chunk (zero between calls)
};

struct CompressArgs {
  const double* field;
  uint64_t nblocks;
  int comps;
  uint8_t* stream;
  uint64_t cap;
  uint64_t mask_off;  // byte offset of masks
  uint64_t val_off;   // byte offset of values
  uint64_t eps_m;     // RD(eps^2) = eps_m * 2^eps_e, eps_m < 2^53 (truncation rule v2)
  int eps_e;
  double eps;         // max_error (RelativeLInf budget)
  int norm;           // ISF_NORM_RELATIVE_L2 (0) or ISF_NORM_RELATIVE_LINF (1; generic kernels)
  double* vslot;      // lx=8 fast path: per-tile value slots (2048 doubles per tile)
  Workspace ws;
};

struct DecompressArgs {
  const uint8_t* stream;
  uint64_t stream_bytes;
  uint64_t nblocks;
  int comps;
  uint64_t mask_off;
  uint64_t val_off;
  double* out;
  const double* orig;
  Workspace ws;
  const uint64_t* off = nullptr;  // per-block value offsets (block_offsets8_kernel); else look-back
};

constexpr unsigned long long kFlagNonFinite = 1, kFlagShape = 2, kFlagOverflow = 4;

// --------------------------- helpers ---------------------------------------
template <int LX, int S, int O0, int DO, int CNT, bool INV, int N, int T = -1>
__device__ __forceinline__ void lines(double (&v)[N]) {
  if constexpr (CNT > 0) {
    if constexpr (INV) inv_line<LX, S, O0, N, T>(v); else fwd_line<LX, S, O0, N, T>(v);
    lines<LX, S, O0 + DO, DO, CNT - 1, INV, N, T>(v);
  }
}
// lx = 8 sweep with its own constant table (see c_f8 / c_b8)
template <int T, int S, int O0, int DO, int CNT, bool INV, int N>
__device__ __forceinline__ void lines8(double (&v)[N]) {
  lines<8, S, O0, DO, CNT, INV, N, T>(v);
}
template <int LX, int S, int O0, int DO1, int CNT1, int DO2, int CNT2, bool INV, int N>
__device__ __forceinline__ void lines2(double (&v)[N]) {
  if constexpr (CNT2 > 0) {
    lines<LX, S, O0, DO1, CNT1, INV>(v);
    lines2<LX, S, O0 + DO2, DO1, CNT1, DO2, CNT2 - 1, INV>(v);
  }
}

// forward line on a strided pointer (generic kernels), returning the max |a| bits of
// its outputs (the selection's block maximum comes out of the x sweep)
template <int LX>
__device__ __forceinline__ uint64_t fwd_line_ptr_mb(double* p, int stride) {
  double v[LX];
#pragma unroll
  for (int i = 0; i < LX; ++i) v[i] = p[i * stride];
  fwd_line<LX, 1, 0>(v);
  uint64_t mb = 0;
#pragma unroll
  for (int i = 0; i < LX; ++i) {
    p[i * stride] = v[i];
    const uint64_t b = abs_bits(v[i]);
    mb = b > mb ? b : mb;
  }
  return mb;
}

__device__ __forceinline__ double2 ldg_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ uint32_t claim_tile(uint32_t* counter) {
  uint32_t t = 0;
  if ((threadIdx.x & 31) == 0) t = atomicAdd(counter, 1u);
  return __shfl_sync(0xffffffffu, t, 0);
}

// --------------------------- generic (any lx, comps) ------------------------

// compress_generic: one warp per block (selection is one warp's job, so wider CTAs idle;
// 64 and 128 threads measured slower on the cfg4 sweep)
constexpr int kGenCThreads = 32;
// decompress_generic CTA width per lx (measured on the cfg4 sweep, profiles/r1_summary.md):
// small blocks want more CTAs, large ones more threads per block
template <int LX>
__host__ __device__ constexpr int gen_dthreads() {
#ifdef ISF_GEN_DTHREADS
  return ISF_GEN_DTHREADS;
#else
  return LX <= 7 ? 64 : LX <= 11 ? 128 : 256;
#endif
}

#ifndef ISF_GEN_SELECT_BIN
#define ISF_GEN_SELECT_BIN 1
#endif
// orders whose compress uses select_bin (measured against select_generic on the cfg4
// spectra, eps 1e-2 / 1e-5: lx 4 +10 / -4 %, 5 +20 / +1 %, 6 +7..12 %, 7 +10 / +3 %,
// 9..12 +5..17 %; lx 3 -6 %); its 21-bit bin planes are exact for lx^3 <= 2048 candidates
__host__ __device__ constexpr bool gen_select_bin(int lx) {
  return ISF_GEN_SELECT_BIN && lx >= 4 && lx <= 12;
}
// select_bin's bins below the block maximum: 128 quarter binades of |a| up to lx 10
// (less to clear and scan: +2.5..8 %), 256 eighth binades at lx 11 / 12 (quarter
// binades crowd the cut bin past 32 candidates at eps 1e-5 there: -18 / -30 %)
__host__ __device__ constexpr int gen_bins(int lx) { return lx >= 11 ? 256 : 128; }
__host__ __device__ constexpr int gen_bin_shift(int lx) { return gen_bins(lx) == 256 ? 49 : 50; }

template <int LX>
struct GenSmem {
  static constexpr int N3 = LX * LX * LX;
  static constexpr int W = (N3 + 63) / 64;
  static constexpr size_t u_off = 0;
  static constexpr size_t idx_off = u_off + sizeof(double) * N3;
  static constexpr size_t hist_off = ((idx_off + sizeof(uint16_t) * N3) + 15) & ~size_t(15);
  // selection scratch: the binned cut search (3 x gen_bins u32 bins; the 32 cut-bin keys and
  // indices reuse them once read); the radix fallback reuses the first 512 B as 64 u64 bins
  static constexpr size_t hist_bytes = gen_select_bin(LX) ? (3 * gen_bins(LX) * 4 > 512 ? 3 * gen_bins(LX) * 4 : 512) : 64 * 8;
  static constexpr size_t mask_off = hist_off + hist_bytes;
  static constexpr size_t misc_off = mask_off + 64 * 8;
  static constexpr size_t bytes = misc_off + 64;
};

// decompress_generic: the block, per-word prefix popcounts, mask words, misc and the
// per-warp error partials (no selection scratch, so more resident CTAs)
template <int LX>
struct GenDSmem {
  static constexpr int N3 = LX * LX * LX;
  static constexpr size_t u_off = 0;
  static constexpr size_t wpre_off = sizeof(double) * N3;
  static constexpr size_t mask_off = wpre_off + 64 * 4;
  static constexpr size_t misc_off = mask_off + 64 * 8;
  static constexpr size_t red_off = misc_off + 64;
  static constexpr size_t bytes = red_off + (gen_dthreads<LX>() / 32) * 4 * 8;
};

// selection on warp 0 over the coefficients in smem u[]
template <int LX>
__device__ void select_generic(double* u, uint64_t eps_m, int eps_e, uint16_t* cidx,
                               unsigned long long* hist, uint64_t* maskw, uint64_t& T_out,
                               uint64_t& hdisc_out, int& eT_out, int& eD_out, bool& nonfinite) {
  constexpr int N3 = LX * LX * LX;
  constexpr int W = (N3 + 63) / 64;
  constexpr int NR = (N3 + 31) / 32;
  const LaneGroup<32> g;
  const int lane = g.rank;
  for (int w = lane; w < 64; w += 32) maskw[w] = 0ull;
  T_out = 0; hdisc_out = 0; eT_out = 0; eD_out = 0; nonfinite = false;
  uint64_t mb = 0;
  for (int p = lane; p < N3; p += 32) { const uint64_t b = abs_bits(u[p]); mb = b > mb ? b : mb; }
  mb = g.max(mb);
  __syncwarp();
  if (mb >= 0x7ff0000000000000ull) { nonfinite = true; return; }
  if (mb == 0) return;
  int s;
  {
    const uint32_t hm = (uint32_t)(mb >> 32);
    s = hm >= 0x00100000u ? (int)(hm >> 20) - 1022 : 64 - __clzll((long long)mb) - 1074;
  }
  constexpr int EM = energy_EM(LX), HM = EM / 2;
  int k = HM - s;
  const int k0 = k;
  const bool tiny = k > 1023;
  if (tiny) {
    const double pre = pow2d(k - 1023);
    for (int p = lane; p < N3; p += 32) u[p] = __dmul_rn(u[p], pre);
    k = 1023;
  }
  const double f = pow2d(k);
  // h from the largest energy (the key maximum): e_max 2^h in [2^(EM-1), 2^EM)
  int h;
  {
    const double xm = __dmul_rn(__longlong_as_double((long long)mb), tiny ? pow2d(k0 - 1023) : 1.0);
    const double xs = __dmul_rn(xm, f);
    h = (EM - 2 * HM) + (__dmul_rd(xs, xs) < pow2d(2 * HM - 1) ? 1 : 0);
  }
  const double sA = pow2d(h);
  uint64_t T = 0;
  for (int p = lane; p < N3; p += 32) {
    const double x = __dmul_rn(u[p], f);
    T += low52(__fma_rd(__dmul_rd(x, x), sA, kTwo52));
  }
  T = g.sum(T);
  T_out = T;
  int G;
  const uint64_t thr = thr_v2(T, eps_m, eps_e, h, G);
  const double sB = pow2d(h + G);
  eT_out = -2 * k0 - h;
  eD_out = -2 * k0 - h - G;
  // one pass: the sure-kept mask (e > thr), the discardable sum SN, and, in case SN
  // exceeds the budget, the sure-discarded sum SL (e <= thr / N3) with the candidates
  // in between compacted by index for the radix select
  const uint64_t thrn = thr / (uint64_t)N3;
  uint64_t SN = 0, SL = 0;
  uint32_t base = 0;
  for (int r = 0; r < NR; ++r) {
    const int p = r * 32 + lane;
    bool sure = false, cand = false;
    if (p < N3) {
      const uint64_t h = hi_v2(u[p], f, sB);
      sure = h > thr;
      if (!sure) {
        SN += h;
        if (h <= thrn) SL += h; else cand = true;
      }
    }
    const unsigned bk = __ballot_sync(0xffffffffu, sure);
    const unsigned bc = __ballot_sync(0xffffffffu, cand);
    if (lane == 0) maskw[r >> 1] |= (uint64_t)bk << (32 * (r & 1));
    if (cand) cidx[base + __popc(bc & ((1u << lane) - 1u))] = (uint16_t)p;
    base += __popc(bc);
  }
  SN = g.sum(SN);
  if (SN <= thr) {
    hdisc_out = SN;
  } else {
    SL = g.sum(SL);
    __syncwarp();
    uint64_t tstar, dsum;
    uint32_t icut;
    radix_select<32>(g, SrcIndirect{u, cidx}, (int)base, thr - SL, f, sB, hist, tstar, icut, dsum);
    // the cut (tstar, icut) is a candidate key (>= 1 candidate here, since SL <= thr < SN)
    // and hi_v2 is monotone in |a|: sure-discarded coefficients lie strictly below it, sure-
    // kept ones above, so the key comparison alone decides every coefficient
    for (int r = 0; r < NR; ++r) {
      const int p = r * 32 + lane;
      bool kept = false;
      if (p < N3) {
        const uint64_t kk = abs_bits(u[p]);
        kept = kk > tstar || (kk == tstar && (uint32_t)p < icut);
      }
      const unsigned b = __ballot_sync(0xffffffffu, kept);
      if (lane == 0) maskw[r >> 1] |= (uint64_t)b << (32 * (r & 1));
    }
    hdisc_out = SL + dsum;
  }
  if (tiny) {
    const double un = pow2d(1023 - k0);
    for (int p = lane; p < N3; p += 32) u[p] = __dmul_rn(u[p], un);
  }
  (void)W;
  __syncwarp();
}

// radix-select source with the tiny-block pre-scale applied on the fly (select_bin's
// fallback; keys of the pre-scaled coefficients, as select_generic)
struct SrcIndirectPre {
  static constexpr bool kCompact = true;
  const double* a;
  uint16_t* idxs;
  double pre;
  __device__ __forceinline__ void operator()(int p, uint64_t& k, uint32_t& ix) const {
    ix = idxs[p];
    k = abs_bits(__dmul_rn(a[ix], pre));
  }
  __device__ __forceinline__ void set(int p, uint32_t ix) const { idxs[p] = (uint16_t)ix; }
};

// Truncation rule v2 on warp 0 over the block's coefficients u[] (natural order), the
// same result as select_generic with fewer passes: the block maximum mb comes from the
// x sweep, the 2^k scale is folded into the energy constants (RD((a 2^k)^2) == RD(a^2)
// 2^2k while a^2 is normal; below, both floors are 0), and when the sure-kept set does
// not settle the block the cut is found by a binned search over the compacted
// candidates only (gen_bins quarter / eighth binades of |a| below the maximum, exact 21-bit-plane u32
// shared atomics, then a warp bitonic sort of the <= 32 cut-bin candidates), with the
// radix select as the fallback for crowded bins and tiny blocks.  Kept bits are OR-ed
// into mw[] (one u32 per 32 coefficients, zero on entry).  mb > 0, finite.
template <int LX>
__device__ __noinline__ void select_bin(const double* u, uint64_t mb, uint64_t eps_m, int eps_e, uint16_t* cidx,
                                        uint32_t* bins, uint64_t* ckey, uint32_t* cix, uint32_t* mw, uint64_t& T_out,
                                        uint64_t& hd_out, int& eT_out, int& eD_out) {
  constexpr int N3 = LX * LX * LX, NR = (N3 + 31) / 32;
  constexpr uint64_t C52 = 0x4330000000000000ull;
  const LaneGroup<32> g;
  const int lane = g.rank;
  const uint32_t lt = (1u << lane) - 1u;
  constexpr int EM = energy_EM(LX), HM = EM / 2;
  int s;
  {
    const uint32_t hm = (uint32_t)(mb >> 32);
    s = hm >= 0x00100000u ? (int)(hm >> 20) - 1022 : 64 - __clzll((long long)mb) - 1074;
  }
  int k = HM - s;
  const int k0 = k;
  const bool tiny = k > 1023;
  const double pre = tiny ? pow2d(k - 1023) : 1.0;
  if (tiny) k = 1023;
  const double f = pow2d(k);
  int h;
  {
    const double xm = __dmul_rn(__longlong_as_double((long long)mb), pre);
    const double xs = __dmul_rn(xm, f);
    h = (EM - 2 * HM) + (__dmul_rd(xs, xs) < pow2d(2 * HM - 1) ? 1 : 0);
  }
  const double sA = pow2d(h);
  const bool fold = !tiny && 2 * k + h <= 1000;
  uint64_t tl = 0;
  if (fold) {
    const double fA = pow2d(2 * k + h);
#pragma unroll 4
    for (int p = lane; p < N3; p += 32) {
      const double a = u[p];
      tl += (uint64_t)__double_as_longlong(__fma_rd(__dmul_rd(a, a), fA, kTwo52)) - C52;
    }
  } else {
#pragma unroll 4
    for (int p = lane; p < N3; p += 32) {
      const double x = __dmul_rn(__dmul_rn(u[p], pre), f);
      tl += (uint64_t)__double_as_longlong(__fma_rd(__dmul_rd(x, x), sA, kTwo52)) - C52;
    }
  }
  const uint64_t T = g.sum(tl);
  T_out = T;
  int Gs;
  const uint64_t thr = thr_v2(T, eps_m, eps_e, h, Gs);
  const double sB = pow2d(h + Gs);
  eT_out = -2 * k0 - h;
  eD_out = -2 * k0 - h - Gs;
  const bool foldB = fold && 2 * k + h + Gs <= 1000;
  const double fB = foldB ? pow2d(2 * k + h + Gs) : 1.0;
  // scale B: t = 2^52 + floor(e 2^(h+G)) (>= 2^53: saturated, always kept)
  auto tB = [&](double a) -> double {
    if (foldB) return __fma_rd(__dmul_rd(a, a), fB, kTwo52);
    const double x = __dmul_rn(__dmul_rn(a, pre), f);
    return __fma_rd(__dmul_rd(x, x), sB, kTwo52);
  };
  const double tthr = __longlong_as_double((long long)(C52 + thr));  // hi > thr  <=>  t >= tthr
  const uint64_t thrn = thr / (uint64_t)N3;
  uint64_t SN = 0, SL = 0;
  uint32_t nc = 0;
  for (int rr = 0; rr < NR; ++rr) {
    const int p = 32 * rr + lane;
    bool sure = false, cand = false;
    if (p < N3) {
      const double t = tB(u[p]);
      if (t >= tthr) {
        sure = true;
      } else {
        const uint64_t hv = (uint64_t)__double_as_longlong(t) - C52 + 1ull;
        SN += hv;
        if (hv <= thrn) SL += hv; else cand = true;
      }
    }
    const uint32_t bk = __ballot_sync(0xffffffffu, sure);
    const uint32_t bc = __ballot_sync(0xffffffffu, cand);
    if (lane == 0) mw[rr] = bk;
    if (cand) cidx[nc + __popc(bc & lt)] = (uint16_t)p;
    nc += __popc(bc);
  }
  SN = g.sum(SN);
  if (SN <= thr) {
    hd_out = SN;
    __syncwarp();
    return;
  }
  SL = g.sum(SL);
  const uint64_t R = thr - SL;
  constexpr int NB = gen_bins(LX), BPL = NB / 32, SH = gen_bin_shift(LX);
  const int bbase = (int)(mb >> SH) - (NB - 1);
  if (!tiny) {
#pragma unroll
    for (int j = 0; j < 3 * NB / 32; ++j) bins[lane + 32 * j] = 0u;
    __syncwarp();
    for (int c = lane; c < (int)nc; c += 32) {
      const double a = u[cidx[c]];
      const uint64_t kk = abs_bits(a);
      const uint64_t hv = (uint64_t)__double_as_longlong(tB(a)) - C52 + 1ull;
      const int bn = ::max((int)(kk >> SH) - bbase, 0);
      atomicAdd(&bins[bn], (uint32_t)(hv & 0x1FFFFFu));
      atomicAdd(&bins[NB + bn], (uint32_t)((hv >> 21) & 0x1FFFFFu));
      atomicAdd(&bins[2 * NB + bn], (uint32_t)(hv >> 42));
    }
    __syncwarp();
    uint64_t bs[BPL];
    uint64_t lsum = 0;
#pragma unroll
    for (int q = 0; q < BPL; ++q) {
      const int b = BPL * lane + q;
      bs[q] = (uint64_t)bins[b] + ((uint64_t)bins[NB + b] << 21) + ((uint64_t)bins[2 * NB + b] << 42);
      lsum += bs[q];
    }
    __syncwarp();  // bins are read: the cut-bin candidates below reuse their storage
    uint64_t x = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    const uint64_t run = x - lsum;
    uint32_t dloc = NB;
    uint64_t exloc = 0;
#pragma unroll
    for (int q = BPL - 1; q >= 0; --q) {
      uint64_t pq = run;
#pragma unroll
      for (int w2 = 0; w2 < q; ++w2) pq += bs[w2];
      if (pq + bs[q] > R) { dloc = BPL * lane + q; exloc = pq; }
    }
    const uint32_t d = g.min(dloc);
    if (d < (uint32_t)NB) {
      const uint64_t ex = __shfl_sync(0xffffffffu, exloc, (int)(d / BPL));
      uint32_t ncd = 0;  // the cut bin's candidates (key, index)
      for (int c0 = 0; c0 < (int)nc; c0 += 32) {
        const int c = c0 + lane;
        uint64_t kk = 0;
        uint32_t ix = 0;
        bool in = false;
        if (c < (int)nc) {
          ix = cidx[c];
          kk = abs_bits(u[ix]);
          in = ::max((int)(kk >> SH) - bbase, 0) == (int)d;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, in);
        const uint32_t pos = ncd + __popc(bal & lt);
        if (in && pos < 32) { ckey[pos] = kk; cix[pos] = ix; }
        ncd += __popc(bal);
      }
      __syncwarp();
      if (ncd <= 32) {
        uint64_t key = lane < (int)ncd ? ckey[lane] : ~0ull;
        uint32_t kix = lane < (int)ncd ? cix[lane] : 0xffffffffu;
        // bitonic sort by key (the index rides along) of the first NS lanes only, NS the
        // power of two >= ncd (warp-uniform): partners stay inside NS-lane groups and the
        // lanes past ncd hold the largest key, so the live lanes end sorted as with 32
        const int NS = ncd <= 2 ? 2 : ncd <= 4 ? 4 : ncd <= 8 ? 8 : ncd <= 16 ? 16 : 32;
#pragma unroll
        for (int kb = 2; kb <= 32; kb <<= 1) {
          if (kb > NS) break;
#pragma unroll
          for (int j = kb >> 1; j > 0; j >>= 1) {
            const uint64_t o = __shfl_xor_sync(0xffffffffu, key, j);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, kix, j);
            const bool up = ((lane & kb) == 0), lower = ((lane & j) == 0);
            const bool sw = (lower == up) ? (o < key) : (o > key);
            if (sw) { key = o; kix = oi; }
          }
        }
        const bool live = lane < (int)ncd;
        const uint64_t hv =
            live ? (uint64_t)__double_as_longlong(tB(__longlong_as_double((long long)key))) - C52 + 1ull : 0ull;
        uint64_t cs = hv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint64_t t = __shfl_up_sync(0xffffffffu, cs, o);
          if (lane >= o) cs += t;
        }
        const uint32_t over = __ballot_sync(0xffffffffu, live && cs > R - ex);
        if (over) {
          const int ic = __ffs(over) - 1;
          const uint64_t K = __shfl_sync(0xffffffffu, key, ic);
          const uint64_t dis = __shfl_sync(0xffffffffu, cs - hv, ic);
          const bool tied = live && key == K;
          const uint32_t tiedbefore = __popc(__ballot_sync(0xffffffffu, tied && lane < ic));
          uint32_t icut = 0xffffffffu;
          if (tiedbefore) {
            // keep the (gcount - tiedbefore) smallest indices among the tied (SPEC.md:225
            // stable order): icut = the tied index of that rank
            const uint32_t gcount = __popc(__ballot_sync(0xffffffffu, tied));
            const uint32_t want = gcount - tiedbefore;
            uint32_t rank = 0;
#pragma unroll 1
            for (int j = 0; j < 32; ++j) {
              const uint32_t oj = __shfl_sync(0xffffffffu, kix, j);
              const uint64_t kj = __shfl_sync(0xffffffffu, key, j);
              rank += (j < (int)ncd && kj == K && oj < kix) ? 1u : 0u;
            }
            icut = g.min((tied && rank == want) ? kix : 0xffffffffu);
          }
          hd_out = SL + ex + dis;
          for (int c = lane; c < (int)nc; c += 32) {
            const uint32_t ix = cidx[c];
            const uint64_t kk = abs_bits(u[ix]);
            if (kk > K || (kk == K && ix < icut)) atomicOr(&mw[ix >> 5], 1u << (ix & 31));
          }
          __syncwarp();
          return;
        }
      }
    }
  }
  // crowded cut bin / tiny block: the radix select over the candidates (exact, any case)
  __syncwarp();
  uint64_t tstar, dsum;
  uint32_t icut;
  radix_select<32>(g, SrcIndirectPre{u, cidx, pre}, (int)nc, R, f, sB, reinterpret_cast<unsigned long long*>(bins),
                   tstar, icut, dsum);
  for (int rr = 0; rr < NR; ++rr) {
    const int p = 32 * rr + lane;
    bool kept = false;
    if (p < N3) {
      const uint64_t kk = abs_bits(__dmul_rn(u[p], pre));
      kept = kk > tstar || (kk == tstar && (uint32_t)p < icut);
    }
    const uint32_t b = __ballot_sync(0xffffffffu, kept);
    if (lane == 0) mw[rr] = b;
  }
  hd_out = SL + dsum;
  __syncwarp();
}

// RelativeLInf selection on warp 0 (dlt_common.cuh radix_select_w)
template <int LX>
__device__ void select_linf(const double* u, double umax, double eps, unsigned long long* hist, uint64_t* maskw,
                            bool& nonfinite) {
  constexpr int N3 = LX * LX * LX;
  constexpr int NR = (N3 + 31) / 32;
  const LaneGroup<32> g;
  const int lane = g.rank;
  for (int w = lane; w < 64; w += 32) maskw[w] = 0ull;
  nonfinite = false;
  uint64_t mb = 0, xm = 0;
  for (int p = lane; p < N3; p += 32) {
    const uint64_t b = abs_bits(u[p]);
    mb = b > mb ? b : mb;
    const uint64_t xb = (uint64_t)__double_as_longlong(__dmul_ru(fabs(u[p]), linf_bmax<LX>(p)));
    xm = xb > xm ? xb : xm;
  }
  mb = g.max(mb);
  xm = g.max(xm);
  __syncwarp();
  if (mb >= 0x7ff0000000000000ull || xm >= 0x7ff0000000000000ull) { nonfinite = true; return; }
  if (xm == 0) return;  // all-zero block keeps nothing
  int s;
  {
    const uint32_t hm = (uint32_t)(xm >> 32);
    s = hm >= 0x00100000u ? (int)(hm >> 20) - 1022 : 64 - __clzll((long long)xm) - 1074;
  }
  const int k = linf_K(LX) - s;
  auto wt = [&](uint64_t key, uint32_t ix) -> uint64_t {
    return linf_weight(__dmul_ru(__longlong_as_double((long long)key), linf_bmax<LX>((int)ix)), k);
  };
  double tb = scale2(__dmul_rd(eps, umax), k);
  tb = floor(tb);
  const uint64_t thr = tb >= 9223372036854775808.0 ? (1ull << 63) : (uint64_t)tb;
  uint64_t tot = 0;
  for (int p = lane; p < N3; p += 32) tot += wt(abs_bits(u[p]), (uint32_t)p);
  tot = g.sum(tot);
  if (tot <= thr) return;  // the whole block fits in the budget
  uint64_t tstar, dsum;
  uint32_t icut;
  radix_select_w<32>(g, SrcDense{u}, wt, N3, thr, hist, tstar, icut, dsum);
  for (int r = 0; r < NR; ++r) {
    const int p = r * 32 + lane;
    bool kept = false;
    if (p < N3) {
      const uint64_t kk = abs_bits(u[p]);
      kept = kk > tstar || (kk == tstar && (uint32_t)p < icut);
    }
    const unsigned b = __ballot_sync(0xffffffffu, kept);
    if (lane == 0) maskw[r >> 1] |= (uint64_t)b << (32 * (r & 1));
  }
  __syncwarp();
}

template <int LX>
__global__ void __launch_bounds__(kGenCThreads) compress_generic(CompressArgs A) {
  constexpr int N = LX, N2 = LX * LX, N3 = LX * LX * LX;
  constexpr int W = (N3 + 63) / 64;
  using L = GenSmem<LX>;
  extern __shared__ __align__(128) unsigned char smem[];
  double* u = reinterpret_cast<double*>(smem + L::u_off);
  uint16_t* cidx = reinterpret_cast<uint16_t*>(smem + L::idx_off);
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(smem + L::hist_off);
  uint64_t* maskw = reinterpret_cast<uint64_t*>(smem + L::mask_off);
  uint64_t* misc = reinterpret_cast<uint64_t*>(smem + L::misc_off);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* counts = reinterpret_cast<uint32_t*>(A.stream);
  uint64_t* masks = reinterpret_cast<uint64_t*>(A.stream + A.mask_off);
  // block tickets one ahead: the next block's atomic is in flight while this one runs
  uint32_t next = 0;
  if (lane == 0) next = atomicAdd(A.ws.counter, 1u);
  next = __shfl_sync(0xffffffffu, next, 0);
  // small scalar RelativeL2 blocks (lx <= 7): the next block's values are loaded into
  // registers while this one is transformed and selected (ceil(lx^3 / 32) doubles per
  // lane), so the block loop does not wait on DRAM at its start
  constexpr bool kPf = LX <= 7;
  constexpr int NPF = kPf ? (N3 + 31) / 32 : 1;
  const bool pf_on = kPf && A.comps == 1 && !A.norm;
  double pf[NPF];
  if (pf_on && next < A.ws.ntiles) {
    const double* s0 = A.field + (uint64_t)next * N3;
#pragma unroll
    for (int i = 0; i < NPF; ++i) pf[i] = (tid + 32 * i < N3) ? s0[tid + 32 * i] : 0.0;
  }
  for (;;) {
    const uint32_t tile = next;
    if (tile >= A.ws.ntiles) {
      if (lane == 0 && tile == A.ws.ntiles + A.ws.total_warps - 1) *A.ws.counter = 0;
      break;
    }
    if (lane == 0) next = atomicAdd(A.ws.counter, 1u);
    __syncwarp();  // the previous block's smem is consumed
    const uint64_t blk = tile;
    const uint64_t e = blk / A.comps, c = blk % A.comps;
    const double* src = A.field + e * (uint64_t)N3 * A.comps + c;
    uint64_t um = 0;
    // scalar field, RelativeL2: plain contiguous copy, 4 loads in flight (lx <= 10;
    // at lx = 12 this variant measured 7 % slower, so it keeps the general loop)
    if (pf_on) {
#pragma unroll
      for (int i = 0; i < NPF; ++i)
        if (tid + 32 * i < N3) u[tid + 32 * i] = pf[i];
    } else if (LX <= 10 && A.comps == 1 && !A.norm) {
#pragma unroll 4
      for (int p = tid; p < N3; p += kGenCThreads) u[p] = src[p];
    } else {  // (also for RelativeL2 at lx > 10: a loop without the maximum measured 8-10 % slower)
      for (int p = tid; p < N3; p += kGenCThreads) {
        const double x = src[(uint64_t)p * A.comps];
        u[p] = x;
        const uint64_t b = abs_bits(x);
        um = b > um ? b : um;
      }
    }
    if (A.norm) {  // RelativeLInf needs max|u| of the block
      if (tid == 0) misc[3] = 0;
      __syncthreads();
      atomicMax(reinterpret_cast<unsigned long long*>(&misc[3]), (unsigned long long)um);
    }
    __syncthreads();
    for (int l = tid; l < N2; l += kGenCThreads) fwd_line_ptr<LX>(u + l, N2);                       // z
    __syncthreads();
    for (int l = tid; l < N2; l += kGenCThreads) fwd_line_ptr<LX>(u + (l / N) * N2 + (l % N), N);  // y
    __syncthreads();
    uint64_t mbl = 0;  // the block maximum, from the x sweep's outputs
    for (int l = tid; l < N2; l += kGenCThreads) {
      const uint64_t m = fwd_line_ptr_mb<LX>(u + l * N, 1);  // x
      mbl = m > mbl ? m : mbl;
    }
    if (pf_on) {  // the next block's values (its ticket is back by now)
      const uint32_t nt = __shfl_sync(0xffffffffu, next, 0);
      if (nt < A.ws.ntiles) {
        const double* s0 = A.field + (uint64_t)nt * N3;
#pragma unroll
        for (int i = 0; i < NPF; ++i) pf[i] = (tid + 32 * i < N3) ? s0[tid + 32 * i] : 0.0;
      }
    }
    __syncthreads();
    if (kGenCThreads == 32 || warp == 0) {  // single-warp CTA: no divergent region
      uint64_t T, hd;
      int eT, eD;
      bool nf;
      if (A.norm) {
        select_linf<LX>(u, __longlong_as_double((long long)misc[3]), A.eps, hist, maskw, nf);
        T = hd = 0;
        eT = eD = 0;
      } else {
        if constexpr (gen_select_bin(LX)) {
        const uint64_t mb = LaneGroup<32>().max(mbl);
        for (int w = lane; w < 64; w += 32) maskw[w] = 0ull;
        T = hd = 0;
        eT = eD = 0;
        nf = mb >= 0x7ff0000000000000ull;
        __syncwarp();
        if (!nf && mb != 0)
          select_bin<LX>(u, mb, A.eps_m, A.eps_e, cidx, reinterpret_cast<uint32_t*>(hist),
                         reinterpret_cast<uint64_t*>(hist),  // cut-bin keys / indices: in the read bins
                         reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(hist) + 32 * 8),
                         reinterpret_cast<uint32_t*>(maskw), T, hd, eT, eD);
        } else {
        (void)mbl;
        select_generic<LX>(u, A.eps_m, A.eps_e, cidx, hist, maskw, T, hd, eT, eD, nf);
        }
      }
      if (nf) {
        for (int w = lane; w < W; w += 32) maskw[w] = 0ull;
        if (lane == 0) atomicOr(A.ws.flags, kFlagNonFinite);
      }
      __syncwarp();
      uint32_t nk = 0;
      for (int w = lane; w < W; w += 32) nk += __popcll(maskw[w]);
      const LaneGroup<32> g;
      nk = g.sum(nk);
      // values go to the block's slot at their natural index (A.vslot, always set by the
      // host) and are packed afterwards by compact_generic_kernel, which also checks the
      // stream capacity
      if (lane == 0) {
        counts[blk] = nk;
        if (blk + 1 == A.nblocks) for (uint64_t pb = A.nblocks; pb < ((A.nblocks + 3) & ~3ull); ++pb) counts[pb] = 0;
        A.ws.partials[blk * 4 + 0] = nf ? 0.0 : ldexp((double)T, eT);
        A.ws.partials[blk * 4 + 1] = nf ? 0.0 : ldexp((double)hd, eD);
      }
      for (int w = lane; w < W; w += 32) masks[blk * W + w] = maskw[w];
    }
    __syncthreads();
    double* slot = A.vslot + blk * (uint64_t)N3;
    static_assert(kGenCThreads == 32, "one 32-bit mask half per round");
    const uint32_t* mw32 = reinterpret_cast<const uint32_t*>(maskw);
    for (int r = 0; 32 * r < N3; ++r) {
      const uint32_t m = mw32[r];
      if (m == 0u) continue;  // warp-uniform: the round keeps nothing
      if ((m >> tid) & 1u) slot[32 * r + tid] = u[32 * r + tid];
    }
    next = __shfl_sync(0xffffffffu, next, 0);
  }
}

// Generic compress epilogue: pack the slots (natural index, N3 doubles per block) into
// the value region.  One warp per block: the block's mask words (lane l holds words l
// and l + 32) and its offsets arrive in one round of loads and their prefix counts by
// a warp scan; then the non-empty words are walked four at a time with every value
// load of a group in flight before its stores (lane l moves bits 2l and 2l + 1 of each word, so
// reads and writes stay contiguous for dense blocks).  The earlier loop loaded one mask
// word, then its values, then stored, word after word: ~2 W dependent round trips per
// block.
__global__ void __launch_bounds__(256) compact_generic_kernel(const uint8_t* stream, uint64_t nblocks,
                                                            uint64_t mask_off, int W, int N3, const uint64_t* off,
                                                            const double* __restrict__ vslot,
                                                            double* __restrict__ vals, uint64_t cap_vals,
                                                            unsigned long long* flags) {
  const int lane = threadIdx.x & 31;
  const uint64_t* masks = reinterpret_cast<const uint64_t*>(stream + mask_off);
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const int p2 = 2 * lane;  // this lane's two bits of every 64-bit mask word
  const uint64_t lowm = (1ull << p2) - 1ull;
  for (uint64_t b = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nblocks; b += nw) {
    const uint64_t e = off[b], e1 = off[b + 1];
    const uint64_t m0 = lane < W ? masks[b * W + lane] : 0ull;
    const uint64_t m1 = lane + 32 < W ? masks[b * W + lane + 32] : 0ull;
    const uint64_t cnt = e1 - e;
    if (b + 1 == nblocks && lane == 0 && off[nblocks] > cap_vals) atomicOr(flags, kFlagOverflow);
    if (cnt == 0 || e + cnt > cap_vals) continue;  // warp-uniform
    // exclusive prefix of the words' popcounts (words 0..31, then 32..63)
    const uint32_t c0 = (uint32_t)__popcll(m0), c1 = (uint32_t)__popcll(m1);
    uint32_t x0 = c0, x1 = c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t0 = __shfl_up_sync(0xffffffffu, x0, o), t1 = __shfl_up_sync(0xffffffffu, x1, o);
      if (lane >= o) {
        x0 += t0;
        x1 += t1;
      }
    }
    const uint32_t tot0 = __shfl_sync(0xffffffffu, x0, 31);
    x0 -= c0;
    x1 += tot0 - c1;
    const double* src = vslot + b * (uint64_t)N3;
    double* dst = vals + e;
    // non-empty words only, four at a time (warp-uniform word indices)
    uint64_t nz = (uint64_t)__ballot_sync(0xffffffffu, m0 != 0ull) |
                  ((uint64_t)__ballot_sync(0xffffffffu, m1 != 0ull) << 32);
    while (nz) {
      uint64_t m[4];
      uint32_t wb[4];
      int wi[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int w = nz ? __ffsll((long long)nz) - 1 : 0;
        const bool live = nz != 0ull;
        nz &= nz - 1;
        const uint64_t a = __shfl_sync(0xffffffffu, m0, w & 31), c = __shfl_sync(0xffffffffu, m1, w & 31);
        const uint32_t ba = __shfl_sync(0xffffffffu, x0, w & 31), bc = __shfl_sync(0xffffffffu, x1, w & 31);
        m[q] = live ? (w < 32 ? a : c) : 0ull;
        wb[q] = w < 32 ? ba : bc;
        wi[q] = w;
      }
      double v[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[2 * q] = ((m[q] >> p2) & 1ull) ? __ldcs(src + 64 * wi[q] + p2) : 0.0;
        v[2 * q + 1] = ((m[q] >> (p2 + 1)) & 1ull) ? __ldcs(src + 64 * wi[q] + p2 + 1) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t r0 = wb[q] + (uint32_t)__popcll(m[q] & lowm);
        const uint32_t b0 = (uint32_t)(m[q] >> p2) & 1u;
        if (b0) dst[r0] = v[2 * q];
        if ((m[q] >> (p2 + 1)) & 1ull) dst[r0 + b0] = v[2 * q + 1];
      }
    }
  }
}

template <int LX>
__global__ void __launch_bounds__(gen_dthreads<LX>()) decompress_generic(DecompressArgs A) {
  constexpr int N = LX, N2 = LX * LX, N3 = LX * LX * LX;
  constexpr int kT = gen_dthreads<LX>();
  constexpr int W = (N3 + 63) / 64;
  using L = GenDSmem<LX>;
  extern __shared__ __align__(128) unsigned char smem[];
  double* u = reinterpret_cast<double*>(smem + L::u_off);
  uint64_t* maskw = reinterpret_cast<uint64_t*>(smem + L::mask_off);
  uint32_t* wpre = reinterpret_cast<uint32_t*>(smem + L::wpre_off);  // prefix popcounts per word
  uint64_t* misc = reinterpret_cast<uint64_t*>(smem + L::misc_off);
  double* red = reinterpret_cast<double*>(smem + L::red_off);        // warps x 4
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(A.stream);
  const uint64_t* masks = reinterpret_cast<const uint64_t*>(A.stream + A.mask_off);
  const double* vals = reinterpret_cast<const double*>(A.stream + A.val_off);
  const uint64_t nvals_avail = A.stream_bytes > A.val_off ? (A.stream_bytes - A.val_off) / 8 : 0;
  constexpr uint64_t lastmask = (N3 % 64) ? ((1ull << (N3 % 64)) - 1ull) : ~0ull;
  double e2 = 0.0, n2 = 0.0;
  uint64_t einf = 0, uinf = 0;
  // static round-robin over the blocks (uniform cost; value offsets come from the
  // block_offsets8_kernel scan, A.off, which the host always provides)
  for (uint64_t blk = blockIdx.x; blk < A.ws.ntiles; blk += gridDim.x) {
    __syncthreads();  // the previous block's smem is consumed
    if (warp == 0) {
      const uint32_t cnt = counts[blk];
      // mask words lane and lane + 32 (W <= 64), per-word exclusive popcount prefix
      uint64_t m0 = 0, m1 = 0;
      if (lane < W) m0 = masks[blk * W + lane];
      if (lane + 32 < W) m1 = masks[blk * W + lane + 32];
      if (lane == W - 1 && (m0 & ~lastmask)) { atomicOr(A.ws.flags, kFlagShape); m0 &= lastmask; }
      if (lane + 32 == W - 1 && (m1 & ~lastmask)) { atomicOr(A.ws.flags, kFlagShape); m1 &= lastmask; }
      const uint32_t c0 = (uint32_t)__popcll(m0), c1 = (uint32_t)__popcll(m1);
      uint32_t i0 = c0, i1 = c1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t0 = __shfl_up_sync(0xffffffffu, i0, o), t1 = __shfl_up_sync(0xffffffffu, i1, o);
        if (lane >= o) { i0 += t0; i1 += t1; }
      }
      const uint32_t tot0 = __shfl_sync(0xffffffffu, i0, 31);
      const uint32_t pc = tot0 + __shfl_sync(0xffffffffu, i1, 31);
      if (lane < W) { maskw[lane] = m0; wpre[lane] = i0 - c0; }
      if (lane + 32 < W) { maskw[lane + 32] = m1; wpre[lane + 32] = tot0 + i1 - c1; }
      const uint64_t prefix = A.off[blk];
      const bool bad = pc != cnt || prefix + cnt > nvals_avail;
      if (lane == 0) {
        if (bad) atomicOr(A.ws.flags, kFlagShape);
        misc[1] = prefix;
        misc[2] = bad;
      }
    }
    __syncthreads();
    const uint64_t prefix = misc[1];
    const bool bad = misc[2] != 0;
    // the gather's global loads are independent: batches of 8 in flight per thread
    constexpr int kG = 8;
    for (int p0 = tid; p0 < N3; p0 += kG * kT) {
      double val[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const int p = p0 + g * kT;
        val[g] = 0.0;
        if (p < N3) {
          const uint64_t mw = maskw[p >> 6];
          if (!bad && ((mw >> (p & 63)) & 1ull))
            val[g] = vals[prefix + wpre[p >> 6] + __popcll(mw & ((1ull << (p & 63)) - 1ull))];
        }
      }
#pragma unroll
      for (int g = 0; g < kG; ++g)
        if (p0 + g * kT < N3) u[p0 + g * kT] = val[g];
    }
    __syncthreads();
    for (int l = tid; l < N2; l += kT) inv_line_ptr<LX>(u + l * N, 1);                     // x
    __syncthreads();
    for (int l = tid; l < N2; l += kT) inv_line_ptr<LX>(u + (l / N) * N2 + (l % N), N);  // y
    __syncthreads();
    for (int l = tid; l < N2; l += kT) inv_line_ptr<LX>(u + l, N2);                       // z
    __syncthreads();
    const uint64_t e = blk / A.comps, c = blk % A.comps;
    double* dst = A.out + e * (uint64_t)N3 * A.comps + c;
    const double* org = A.orig ? A.orig + e * (uint64_t)N3 * A.comps + c : nullptr;
    for (int p = tid; p < N3; p += kT) {
      const double val = __dadd_rn(u[p], 0.0);  // zero results are written as +0
      __stcs(dst + (uint64_t)p * A.comps, val);  // streaming: the field is not re-read here
      if (org) {
        const int x = p % N, yy = (p / N) % N, z = p / N2;
        const double w3 = __dmul_rn(__dmul_rn(Wg<LX>(x), Wg<LX>(yy)), Wg<LX>(z));
        const double o = org[(uint64_t)p * A.comps];
        const double d = __dsub_rn(o, val);
        e2 = __fma_rn(__dmul_rn(w3, d), d, e2);
        n2 = __fma_rn(__dmul_rn(w3, o), o, n2);
        uint64_t t = abs_bits(d); einf = t > einf ? t : einf;
        t = abs_bits(o); uinf = t > uinf ? t : uinf;
      }
    }
  }
  if (A.orig) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      e2 = __dadd_rn(e2, __shfl_xor_sync(0xffffffffu, e2, o));
      n2 = __dadd_rn(n2, __shfl_xor_sync(0xffffffffu, n2, o));
      uint64_t t = __shfl_xor_sync(0xffffffffu, einf, o); einf = t > einf ? t : einf;
      t = __shfl_xor_sync(0xffffffffu, uinf, o); uinf = t > uinf ? t : uinf;
    }
    __syncthreads();
    if (lane == 0) {
      red[warp * 4 + 0] = e2; red[warp * 4 + 1] = n2;
      red[warp * 4 + 2] = __longlong_as_double((long long)einf);
      red[warp * 4 + 3] = __longlong_as_double((long long)uinf);
    }
    __syncthreads();
    if (tid == 0) {
      double se = 0, sn = 0;
      uint64_t me = 0, mu = 0;
      for (int w = 0; w < kT / 32; ++w) {
        se = __dadd_rn(se, red[w * 4]); sn = __dadd_rn(sn, red[w * 4 + 1]);
        uint64_t t = (uint64_t)__double_as_longlong(red[w * 4 + 2]); me = t > me ? t : me;
        t = (uint64_t)__double_as_longlong(red[w * 4 + 3]); mu = t > mu ? t : mu;
      }
      const uint64_t slot = blockIdx.x;
      A.ws.partials[slot * 4 + 0] = se;
      A.ws.partials[slot * 4 + 1] = sn;
      A.ws.partials[slot * 4 + 2] = __longlong_as_double((long long)me);
      A.ws.partials[slot * 4 + 3] = __longlong_as_double((long long)mu);
    }
  }
}

// --------------------------- finalize ---------------------------------------
struct FinalizeArgs {
  int mode;                 // 0 compress, 1 decompress
  const double* partials;
  uint64_t nparts;          // number of partial slots
  const uint64_t* status;   // look-back descriptors (total = inclusive of last tile)
  const uint64_t* total_ptr;  // if non-null: plain u64 total (tile-offset table end)
  uint32_t ntiles;
  unsigned long long* flags;
  void* stats;              // isf_lossy_stats*
  uint64_t nblocks, field_bytes, val_off;
  int with_error;
  volatile uint64_t* density = nullptr;  // host-mapped: (kept, coefficients) of this call (lx = 8 auto schedule)
};

constexpr int kFinThreads = 512;
constexpr int kFinChunks = 256;  // first-level CTAs of finalize_pre_kernel

// CTA-wide fixed-order reduction of records [begin, end) (sums of .0/.1, max of the bit
// patterns of .2/.3 when mode == 1); the results are in s0[0], s1[0], m0[0], m1[0]
__device__ __forceinline__ void reduce_records(const double* partials, uint64_t begin, uint64_t end, int mode,
                                               double* s0, double* s1, unsigned long long* m0,
                                               unsigned long long* m1) {
  const int t = threadIdx.x;
  double a0 = 0.0, a1 = 0.0;
  unsigned long long x0 = 0, x1 = 0;
  // 8 records in flight per thread, summed in the same sequential order as the tail loop
  // (the statistics stay bit-identical to a plain strided loop; the generic compress
  // path reduces one record per block here)
  const double2* rec = reinterpret_cast<const double2*>(partials);
  uint64_t i0 = begin + t;
  constexpr int U = 8;
  for (; i0 + (uint64_t)(U - 1) * kFinThreads < end; i0 += (uint64_t)U * kFinThreads) {
    double2 lo[U], hi[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      lo[j] = rec[(i0 + (uint64_t)j * kFinThreads) * 2];
      if (mode == 1) hi[j] = rec[(i0 + (uint64_t)j * kFinThreads) * 2 + 1];
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      a0 = __dadd_rn(a0, lo[j].x);
      a1 = __dadd_rn(a1, lo[j].y);
      if (mode == 1) {
        unsigned long long v = (unsigned long long)__double_as_longlong(hi[j].x);
        x0 = v > x0 ? v : x0;
        v = (unsigned long long)__double_as_longlong(hi[j].y);
        x1 = v > x1 ? v : x1;
      }
    }
  }
  for (uint64_t i = i0; i < end; i += kFinThreads) {
    a0 = __dadd_rn(a0, partials[i * 4 + 0]);
    a1 = __dadd_rn(a1, partials[i * 4 + 1]);
    if (mode == 1) {
      unsigned long long v = (unsigned long long)__double_as_longlong(partials[i * 4 + 2]);
      x0 = v > x0 ? v : x0;
      v = (unsigned long long)__double_as_longlong(partials[i * 4 + 3]);
      x1 = v > x1 ? v : x1;
    }
  }
  s0[t] = a0; s1[t] = a1; m0[t] = x0; m1[t] = x1;
  __syncthreads();
  for (int o = kFinThreads / 2; o; o >>= 1) {
    if (t < o) {
      s0[t] = __dadd_rn(s0[t], s0[t + o]);
      s1[t] = __dadd_rn(s1[t], s1[t + o]);
      m0[t] = m0[t + o] > m0[t] ? m0[t + o] : m0[t];
      m1[t] = m1[t + o] > m1[t] ? m1[t + o] : m1[t];
    }
    __syncthreads();
  }
}

// First level of the statistics reduction when there is one record per block (generic
// compress): CTA c reduces the fixed record range [c * CH, (c + 1) * CH) into record c of
// `out`, which finalize_kernel then reduces (a deterministic two-level tree)
__global__ void __launch_bounds__(kFinThreads) finalize_pre_kernel(const double* partials, uint64_t nparts, int mode,
                                                                  double* out) {
  __shared__ double s0[kFinThreads], s1[kFinThreads];
  __shared__ unsigned long long m0[kFinThreads], m1[kFinThreads];
  const uint64_t ch = (nparts + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = (uint64_t)blockIdx.x * ch, hi = lo + ch < nparts ? lo + ch : nparts;
  reduce_records(partials, lo < nparts ? lo : nparts, hi, mode, s0, s1, m0, m1);
  if (threadIdx.x == 0) {
    out[blockIdx.x * 4 + 0] = s0[0];
    out[blockIdx.x * 4 + 1] = s1[0];
    out[blockIdx.x * 4 + 2] = __longlong_as_double((long long)m0[0]);
    out[blockIdx.x * 4 + 3] = __longlong_as_double((long long)m1[0]);
  }
}

__global__ void __launch_bounds__(kFinThreads) finalize_kernel(FinalizeArgs A) {
  __shared__ double s0[kFinThreads], s1[kFinThreads];
  __shared__ unsigned long long m0[kFinThreads], m1[kFinThreads];
  const int t = threadIdx.x;
  reduce_records(A.partials, 0, A.nparts, A.mode, s0, s1, m0, m1);
  if (t == 0) {
    double* st = reinterpret_cast<double*>(A.stats);
    uint64_t* su = reinterpret_cast<uint64_t*>(A.stats);
    uint64_t total;
    if (A.total_ptr) {
      total = *A.total_ptr;
    } else {
      const uint64_t last = A.ntiles ? ld_relaxed(A.status + (A.ntiles - 1)) : 0ull;
      total = last & ((1ull << 38) - 1);
    }
    for (int i = 0; i < 12; ++i) su[i] = 0;
    if (A.mode == 0) {
      st[4] = s1[0];  // disc2
      st[5] = s0[0];  // tot2
    } else if (A.with_error) {
      st[0] = s0[0];
      st[1] = s1[0];
      st[2] = __longlong_as_double((long long)m0[0]);
      st[3] = __longlong_as_double((long long)m1[0]);
    }
    su[6] = total;
    su[7] = A.nblocks;
    su[8] = A.val_off + 8 * total;
    su[9] = A.field_bytes;
    su[10] = *A.flags;
    *A.flags = 0;
  }
}

}  // namespace dev
}  // namespace isf
