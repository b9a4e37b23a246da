// dlt_common.cuh -- device building blocks shared by the sm_100a kernels:
// GLL operators in constant memory, the pinned even/odd line transforms,
// lane-group primitives, decoupled look-back and the exact selection rule.
//
// Pinned numerics: every product/sum is an explicit __dmul_rn /
// __dadd_rn / __fma_rn in the same order as oracle/isf_oracle.c, so the
// coefficients, masks and streams are bit-identical to the CPU restatement of
// SPEC.md:222-239.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

namespace isf {
namespace dev {

constexpr int kMaxLx = 16;

// Packed operator table: for each lx in [2,16], F (lx*lx, [k][i]) then B (lx*lx, [i][k]).
// offset(lx) = 2 * sum_{m=2}^{lx-1} m^2.
__host__ __device__ constexpr int op_offset(int lx) {
  int o = 0;
  for (int m = 2; m < lx; ++m) o += 2 * m * m;
  return o;
}
constexpr int kOpTableSize = op_offset(kMaxLx + 1);
__host__ __device__ constexpr int w_offset(int lx) { return (lx * (lx - 1)) / 2 - 1; }  // sum_{m=2}^{lx-1} m
constexpr int kWTableSize = w_offset(kMaxLx + 1);

// single translation unit (isf_lossy.cu) -> defined here
__constant__ double c_ops[kOpTableSize];
__constant__ double c_w[kWTableSize];
__constant__ double c_x[kWTableSize];
__constant__ double c_bm[kWTableSize];  // RelativeLInf: max_i |B[i][k]| per lx (w_offset layout)

// lx = 8: one private copy of F and of B per sweep (T = 0, 1, 2).  With a single
// table the compiler keeps the 32 shared constants of the three sweeps live across
// the loop and falls back to per-use LDC into vector registers; with a table per
// sweep each sweep's constants go to uniform registers (LDCU) and feed the DFMAs
// directly.  Same values, same arithmetic order: results are unchanged.
__constant__ double c_f8[3][64];
__constant__ double c_b8[3][64];

template <int LX, int T = -1>
__device__ __forceinline__ double Fm(int k, int i) {
  if constexpr (LX == 8 && T >= 0) return c_f8[T][k * 8 + i];
  else return c_ops[op_offset(LX) + k * LX + i];
}
template <int LX, int T = -1>
__device__ __forceinline__ double Bm(int i, int k) {
  if constexpr (LX == 8 && T >= 0) return c_b8[T][i * 8 + k];
  else return c_ops[op_offset(LX) + LX * LX + i * LX + k];
}
template <int LX>
__device__ __forceinline__ double Wg(int i) { return c_w[w_offset(LX) + i]; }

// ---------------------------------------------------------------------------
// Pinned line transforms on register arrays: v[O + i*S], i = 0..LX-1.
// forward: s_i = u_i + u_{n-1-i}, d_i = u_i - u_{n-1-i}; a_k = F[k][0]*v_0 then
// ascending fma over the even (k even) / odd (k odd) half; middle node last.
// ---------------------------------------------------------------------------
template <int LX, int S, int O, int N, int T = -1>
__device__ __forceinline__ void fwd_line(double (&v)[N]) {
  constexpr int H = LX / 2;
  double s[H], d[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const double x0 = v[O + i * S], x1 = v[O + (LX - 1 - i) * S];
    s[i] = __dadd_rn(x0, x1);
    d[i] = __dsub_rn(x0, x1);
  }
  const double m = (LX & 1) ? v[O + H * S] : 0.0;
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    double acc = __dmul_rn(Fm<LX, T>(k, 0), (k & 1) ? d[0] : s[0]);
#pragma unroll
    for (int i = 1; i < H; ++i) acc = __fma_rn(Fm<LX, T>(k, i), (k & 1) ? d[i] : s[i], acc);
    if ((LX & 1) && !(k & 1)) acc = __fma_rn(Fm<LX, T>(k, H), m, acc);
    v[O + k * S] = acc;
  }
}

template <int LX, int S, int O, int N, int T = -1>
__device__ __forceinline__ void inv_line(double (&v)[N]) {
  constexpr int H = LX / 2;
  double out[LX];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    double E = __dmul_rn(Bm<LX, T>(i, 0), v[O]);
#pragma unroll
    for (int k = 2; k < LX; k += 2) E = __fma_rn(Bm<LX, T>(i, k), v[O + k * S], E);
    double Od = __dmul_rn(Bm<LX, T>(i, 1), v[O + S]);
#pragma unroll
    for (int k = 3; k < LX; k += 2) Od = __fma_rn(Bm<LX, T>(i, k), v[O + k * S], Od);
    out[i] = __dadd_rn(E, Od);
    out[LX - 1 - i] = __dsub_rn(E, Od);
  }
  if (LX & 1) {
    double E = __dmul_rn(Bm<LX, T>(H, 0), v[O]);
#pragma unroll
    for (int k = 2; k < LX; k += 2) E = __fma_rn(Bm<LX, T>(H, k), v[O + k * S], E);
    out[H] = E;
  }
#pragma unroll
  for (int i = 0; i < LX; ++i) v[O + i * S] = out[i];
}

// Line transform on a pointer with runtime stride (generic kernels; same order).
template <int LX>
__device__ __forceinline__ void fwd_line_ptr(double* p, int stride) {
  double v[LX];
#pragma unroll
  for (int i = 0; i < LX; ++i) v[i] = p[i * stride];
  fwd_line<LX, 1, 0>(v);
#pragma unroll
  for (int i = 0; i < LX; ++i) p[i * stride] = v[i];
}
template <int LX>
__device__ __forceinline__ void inv_line_ptr(double* p, int stride) {
  double v[LX];
#pragma unroll
  for (int i = 0; i < LX; ++i) v[i] = p[i * stride];
  inv_line<LX, 1, 0>(v);
#pragma unroll
  for (int i = 0; i < LX; ++i) p[i * stride] = v[i];
}

// ---------------------------------------------------------------------------
// Truncation rule v2 (oracle/isf_oracle.c select_impl):
//   x_j = |a_j| 2^k (k = EM/2 - s), e_j = RD(x_j^2), T = sum floor(e_j 2^h)  (scale A)
//   thr = floor(T * RD(eps^2) * 2^G) in [2^51, 2^52)                          (scale B)
//   hi_j = floor(e_j 2^(h+G)) + 1 (saturated to 2^52: never discardable)
// floor(y) for 0 <= y < 2^52 is the low mantissa of RD(y + 2^52): one fma_rd each.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int ceil_log2(int v) {
  int r = 0;
  while ((1 << r) < v) ++r;
  return r;
}
// max scale-A energy exponent: e_max 2^h in [2^(EM-1), 2^EM), sum of lx^3 < 2^63
__host__ __device__ constexpr int energy_EM(int lx) {
  return (63 - ceil_log2(lx * lx * lx)) < 52 ? (63 - ceil_log2(lx * lx * lx)) : 52;
}
__host__ __device__ constexpr int linf_K(int lx) { return 63 - ceil_log2(lx * lx * lx); }
__device__ __forceinline__ uint64_t low52(double t) {
  return (uint64_t)__double_as_longlong(t) & 0x000FFFFFFFFFFFFFull;
}
__device__ __forceinline__ double pow2d(int e) {  // 2^e for e in [-1022, 1023]
  return __longlong_as_double((long long)(e + 1023) << 52);
}
__device__ __forceinline__ uint64_t abs_bits(double a) {
  return (uint64_t)__double_as_longlong(a) & 0x7FFFFFFFFFFFFFFFull;
}
constexpr double kTwo52 = 4503599627370496.0;
constexpr double kTwo53 = 9007199254740992.0;
constexpr uint64_t kHiSat = 1ull << 52;  // saturated hi: larger than any threshold
// scale-B upper bound of the energy of a (already pre-scaled), f = 2^k, sB = 2^(h+G)
__device__ __forceinline__ uint64_t hi_v2(double a, double f, double sB) {
  const double x = __dmul_rn(a, f);
  const double t = __fma_rd(__dmul_rd(x, x), sB, kTwo52);
  return t < kTwo53 ? low52(t) + 1ull : kHiSat;
}
// thr and G from T (scale A) and RD(eps^2) = eps_m 2^eps_e (eps_m < 2^53), h
__device__ __forceinline__ uint64_t thr_v2(uint64_t T, uint64_t eps_m, int eps_e, int h, int& G) {
  const uint64_t plo = T * eps_m, phi = __umul64hi(T, eps_m);
  if ((plo | phi) == 0ull) { G = 0; return 0ull; }
  const int L = phi ? 128 - __clzll((long long)phi) : 64 - __clzll((long long)plo);
  int g = 52 - L - eps_e;
  g = g > 1023 - h ? 1023 - h : g;
  G = g;
  const int sh = g + eps_e;  // thr = floor(P 2^sh)
  if (sh >= 0) return plo << sh;  // L + sh <= 52: P < 2^64 here
  const int r = -sh;
  if (r >= 128) return 0ull;
  if (r >= 64) return phi >> (r - 64);
  return (plo >> r) | (r ? (phi << (64 - r)) : 0ull);
}
// x * 2^e, exact for results in the normal range (cheap common case of ldexp)
__device__ __forceinline__ double scale2(double x, int e) {
  return (e >= -1022 && e <= 1023) ? __dmul_rn(x, pow2d(e)) : ldexp(x, e);
}

// ---------------------------------------------------------------------------
// Lane groups: G consecutive lanes of one warp (G | 32), xor-shuffle reductions.
// ---------------------------------------------------------------------------
template <int G>
struct LaneGroup {
  unsigned mask;  // member mask of this group
  int rank;       // lane index inside the group
  __device__ __forceinline__ LaneGroup() {
    const int lane = threadIdx.x & 31;
    rank = lane & (G - 1);
    mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  __device__ __forceinline__ uint64_t sum(uint64_t v) const {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(mask, v, o);
    return v;
  }
  __device__ __forceinline__ uint32_t sum(uint32_t v) const {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(mask, v, o);
    return v;
  }
  __device__ __forceinline__ double sumd(double v) const {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(mask, v, o));
    return v;
  }
  __device__ __forceinline__ uint64_t max(uint64_t v) const {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) { uint64_t t = __shfl_xor_sync(mask, v, o); v = t > v ? t : v; }
    return v;
  }
  __device__ __forceinline__ uint64_t min(uint64_t v) const {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) { uint64_t t = __shfl_xor_sync(mask, v, o); v = t < v ? t : v; }
    return v;
  }
  __device__ __forceinline__ uint32_t max(uint32_t v) const {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v = ::max(v, __shfl_xor_sync(mask, v, o));
    return v;
  }
  __device__ __forceinline__ uint32_t min(uint32_t v) const {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v = ::min(v, __shfl_xor_sync(mask, v, o));
    return v;
  }
  __device__ __forceinline__ double maxd(double v) const {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v = fmax(v, __shfl_xor_sync(mask, v, o));
    return v;
  }
  // exclusive prefix sum inside the group
  __device__ __forceinline__ uint32_t exscan(uint32_t v) const {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      uint32_t t = __shfl_up_sync(mask, x, o, G);
      if (rank >= o) x += t;
    }
    return x - v;
  }
  __device__ __forceinline__ uint64_t exscan(uint64_t v) const {
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
      uint64_t t = __shfl_up_sync(mask, x, o, G);
      if (rank >= o) x += t;
    }
    return x - v;
  }
  template <class T>
  __device__ __forceinline__ T bcast(T v, int src_rank) const {
    return __shfl_sync(mask, v, src_rank, G);
  }
};

// ---------------------------------------------------------------------------
// Exact selection, general path: MSB radix select with 64 energy-sum bins.
// Finds the boundary key t* and the index cut of a tie group so that
//   kept  <=>  key > t*  ||  (key == t* && idx < icut)
// and the discarded set is the longest prefix of the discard order (|a| asc,
// index desc) with sum(hi) <= R.  `src(p, key, idx)` yields element p < n.
// Group = G lanes of one warp.  hist: 64 u64 in shared memory.
// ---------------------------------------------------------------------------
template <int G, class Src>
__device__ __forceinline__ void radix_select(const LaneGroup<G>& g, const Src& src, int n, uint64_t R,
                                             double f, double sB, unsigned long long* hist, uint64_t& tstar,
                                             uint32_t& icut, uint64_t& dsum) {
  uint64_t klo = ~0ull, khi = 0;
  for (int p = g.rank; p < n; p += G) {
    uint64_t k; uint32_t ix;
    src(p, k, ix);
    klo = k < klo ? k : klo;
    khi = k > khi ? k : khi;
  }
  klo = g.min(klo);
  khi = g.max(khi);
  dsum = 0;
  for (;;) {
    const uint64_t span = khi - klo;
    if (span == 0) {
      // tie group: every undecided element has key == klo
      const uint64_t h = hi_v2(__longlong_as_double((long long)klo), f, sB);
      uint32_t cnt = 0;
      for (int p = g.rank; p < n; p += G) { uint64_t k; uint32_t ix; src(p, k, ix); cnt += (k == klo); }
      const uint32_t gcount = g.sum(cnt);
      uint64_t r = (h == 0) ? gcount : (R / h);
      if (r > gcount) r = gcount;
      dsum += r * h;
      tstar = klo;
      if (r == gcount) {
        icut = 0;  // all tied discarded
      } else if (r == 0) {
        icut = 0xffffffffu;  // all tied kept
      } else {
        // keep the (gcount - r) smallest indices: icut = index of rank (gcount - r)
        const uint32_t want = gcount - (uint32_t)r;
        uint32_t mine = 0xffffffffu;
        for (int p = g.rank; p < n; p += G) {
          uint64_t k; uint32_t ip;
          src(p, k, ip);
          if (k != klo) continue;
          uint32_t rank = 0;
          for (int q = 0; q < n; ++q) { uint64_t kq; uint32_t iq; src(q, kq, iq); rank += (kq == klo && iq < ip); }
          if (rank == want) mine = ip;
        }
        icut = g.min(mine);
      }
      return;
    }
    const int bits = 64 - __clzll((long long)span);
    const int shift = bits > 6 ? bits - 6 : 0;
    for (int b = g.rank; b < 64; b += G) hist[b] = 0ull;
    g.sync();
    for (int p = g.rank; p < n; p += G) {
      uint64_t k; uint32_t ix;
      src(p, k, ix);
      if (k >= klo && k <= khi)
        atomicAdd(&hist[(k - klo) >> shift], (unsigned long long)hi_v2(__longlong_as_double((long long)k), f, sB));
    }
    g.sync();
    constexpr int BPL = 64 / G;
    uint64_t loc[BPL];
    uint64_t run = 0;
#pragma unroll
    for (int j = 0; j < BPL; ++j) { run += hist[g.rank * BPL + j]; loc[j] = run; }
    const uint64_t base = g.exscan(run);
    const uint64_t total = g.bcast(base + run, G - 1);
    g.sync();  // hist is reused by the next round
    uint32_t dloc = 64;
    uint64_t exloc = 0;
#pragma unroll
    for (int j = BPL - 1; j >= 0; --j) {
      if (base + loc[j] > R) { dloc = g.rank * BPL + j; exloc = base + (j ? loc[j - 1] : 0); }
    }
    const uint32_t d = g.min(dloc);
    if (d == 64) {  // everything undecided fits: discard it all
      dsum += total;
      tstar = khi;
      icut = 0;
      return;
    }
    const uint64_t ex = g.bcast(exloc, (int)(d / BPL));
    R -= ex;
    dsum += ex;
    const uint64_t nlo = klo + ((uint64_t)d << shift);
    const uint64_t nhi_full = nlo + ((1ull << shift) - 1);
    const uint64_t nhi = nhi_full < khi ? nhi_full : khi;
    uint64_t mn = ~0ull, mx = 0;
    if constexpr (Src::kCompact && G == 32) {
      // keep only the candidates of the cut bin (in place: a chunk's survivors land at
      // or before the chunk), so the next passes scan the survivors alone
      int w = 0;
      for (int p0 = 0; p0 < n; p0 += 32) {
        const int p = p0 + g.rank;
        uint64_t k = 0; uint32_t ix = 0;
        if (p < n) src(p, k, ix);
        const bool keep = p < n && k >= nlo && k <= nhi;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) {
          src.set(w + __popc(bal & ((1u << g.rank) - 1u)), ix);
          mn = k < mn ? k : mn;
          mx = k > mx ? k : mx;
        }
        w += __popc(bal);
      }
      n = w;
      __syncwarp();
    } else {
      for (int p = g.rank; p < n; p += G) {
        uint64_t k; uint32_t ix;
        src(p, k, ix);
        if (k >= nlo && k <= nhi) { mn = k < mn ? k : mn; mx = k > mx ? k : mx; }
      }
    }
    klo = g.min(mn);
    khi = g.max(mx);
  }
}

// ---------------------------------------------------------------------------
// RelativeLInf truncation.
// |u - u~|(x) <= sum_{j discarded} |a_j| * Bmax_j with Bmax_j = max|B(kx)| max|B(ky)|
// max|B(kz)|.  Exact integer form (upper bounds for the discarded terms, a lower
// bound for the budget):
//   x_j = RU(|a_j| * RU(RU(bm_kx * bm_ky) * bm_kz)),   m = max_j x_j = f 2^s, f in [.5,1)
//   k   = 53 - s,   w_j = x_j == 0 ? 0 : max(1, ceil(x_j 2^k))  (< 2^53)
//   thr = floor(RD(eps * max|u|) 2^k)
// and the discarded set is the longest prefix of the discard order (|a| asc, index
// desc) with sum w <= thr; an all-zero block keeps nothing.
// ---------------------------------------------------------------------------
template <int LX>
__device__ __forceinline__ double linf_bmax(int j) {
  const int kx = j % LX, ky = (j / LX) % LX, kz = j / (LX * LX);
  const int o = w_offset(LX);
  return __dmul_ru(__dmul_ru(c_bm[o + kx], c_bm[o + ky]), c_bm[o + kz]);
}
__device__ __forceinline__ uint64_t linf_weight(double x, int k) {
  if (x == 0.0) return 0;
  const double c = ceil(scale2(x, k));
  return c < 1.0 ? 1ull : (uint64_t)c;
}

// radix select over all n elements with per-element weights (general weights: the
// tie group is resolved in index-descending order element by element)
template <int G, class Src, class Wt>
__device__ void radix_select_w(const LaneGroup<G>& g, const Src& src, const Wt& wt, int n, uint64_t R,
                               unsigned long long* hist, uint64_t& tstar, uint32_t& icut, uint64_t& dsum) {
  uint64_t klo = ~0ull, khi = 0;
  for (int p = g.rank; p < n; p += G) {
    uint64_t k; uint32_t ix;
    src(p, k, ix);
    klo = k < klo ? k : klo;
    khi = k > khi ? k : khi;
  }
  klo = g.min(klo);
  khi = g.max(khi);
  dsum = 0;
  for (;;) {
    const uint64_t span = khi - klo;
    if (span == 0) {
      // tie group (key == klo): discard in index-descending order while the sum fits
      uint32_t mine = 0xffffffffu;
      uint64_t dloc = 0;
      for (int p = g.rank; p < n; p += G) {
        uint64_t k; uint32_t ip;
        src(p, k, ip);
        if (k != klo) continue;
        uint64_t S = wt(k, ip);
        const uint64_t own = S;
        for (int q = 0; q < n; ++q) {
          uint64_t kq; uint32_t iq;
          src(q, kq, iq);
          if (kq == klo && iq > ip) S += wt(kq, iq);
        }
        if (S <= R) { mine = ip < mine ? ip : mine; dloc += own; }
      }
      icut = (uint32_t)g.min((uint64_t)mine);
      dsum += g.sum(dloc);
      tstar = klo;
      return;
    }
    const int bits = 64 - __clzll((long long)span);
    const int shift = bits > 6 ? bits - 6 : 0;
    for (int b = g.rank; b < 64; b += G) hist[b] = 0ull;
    g.sync();
    for (int p = g.rank; p < n; p += G) {
      uint64_t k; uint32_t ix;
      src(p, k, ix);
      if (k >= klo && k <= khi) atomicAdd(&hist[(k - klo) >> shift], (unsigned long long)wt(k, ix));
    }
    g.sync();
    constexpr int BPL = 64 / G;
    uint64_t loc[BPL];
    uint64_t run = 0;
#pragma unroll
    for (int j = 0; j < BPL; ++j) { run += hist[g.rank * BPL + j]; loc[j] = run; }
    const uint64_t base = g.exscan(run);
    const uint64_t total = g.bcast(base + run, G - 1);
    g.sync();
    uint32_t dl = 64;
    uint64_t exloc = 0;
#pragma unroll
    for (int j = BPL - 1; j >= 0; --j) {
      if (base + loc[j] > R) { dl = g.rank * BPL + j; exloc = base + (j ? loc[j - 1] : 0); }
    }
    const uint32_t d = g.min(dl);
    if (d == 64) {
      dsum += total;
      tstar = khi;
      icut = 0;
      return;
    }
    const uint64_t ex = g.bcast(exloc, (int)(d / BPL));
    R -= ex;
    dsum += ex;
    const uint64_t nlo = klo + ((uint64_t)d << shift);
    const uint64_t nhi_full = nlo + ((1ull << shift) - 1);
    const uint64_t nhi = nhi_full < khi ? nhi_full : khi;
    uint64_t mn = ~0ull, mx = 0;
    if constexpr (Src::kCompact && G == 32) {
      // keep only the candidates of the cut bin (in place: a chunk's survivors land at
      // or before the chunk), so the next passes scan the survivors alone
      int w = 0;
      for (int p0 = 0; p0 < n; p0 += 32) {
        const int p = p0 + g.rank;
        uint64_t k = 0; uint32_t ix = 0;
        if (p < n) src(p, k, ix);
        const bool keep = p < n && k >= nlo && k <= nhi;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) {
          src.set(w + __popc(bal & ((1u << g.rank) - 1u)), ix);
          mn = k < mn ? k : mn;
          mx = k > mx ? k : mx;
        }
        w += __popc(bal);
      }
      n = w;
      __syncwarp();
    } else {
      for (int p = g.rank; p < n; p += G) {
        uint64_t k; uint32_t ix;
        src(p, k, ix);
        if (k >= nlo && k <= nhi) { mn = k < mn ? k : mn; mx = k > mx ? k : mx; }
      }
    }
    klo = g.min(mn);
    khi = g.max(mx);
  }
}

// element sources for radix_select
struct SrcIndirect {  // candidate indices into the block's coefficients (generic kernels)
  static constexpr bool kCompact = true;  // radix_select narrows the list in place
  const double* a;
  uint16_t* idxs;
  __device__ __forceinline__ void operator()(int p, uint64_t& k, uint32_t& ix) const { ix = idxs[p]; k = abs_bits(a[ix]); }
  __device__ __forceinline__ void set(int p, uint32_t ix) const { idxs[p] = (uint16_t)ix; }
};
struct SrcDense {  // raw coefficients in natural order, index = position (fast kernels)
  static constexpr bool kCompact = false;
  const double* a;
  __device__ __forceinline__ void operator()(int p, uint64_t& k, uint32_t& ix) const { k = abs_bits(a[p]); ix = (uint32_t)p; }
};

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA engine, cp.async.bulk) helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// programmatic dependent launch: wait until the stream predecessor grid has completed
// and its memory is visible (a no-op when the kernel was launched without the attribute)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// bulk shared -> global copy (TMA engine; bulk async-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// per-thread 8-byte async copies (vector fields: a block's stride-3 gather into the
// dense stage) and their commit / wait groups
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// shared-window (u32) address forms, for addresses hoisted out of the block loops
__device__ __forceinline__ void mbar_arrive_tx_a(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                                uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------------------
// Tensor memory (tcgen05) as a second on-chip buffer beside shared memory.
// The lx = 8 kernels use it for register re-layouts and to park coefficients: its
// datapath is separate from the shared-memory banks (128 B/clk/SM, the limit of the
// smem-only design) and a 4 KiB store + 16x256b re-read runs at ~358 B/clk/SM
// (tools/probe/tmem_bw.cu).  Thread <-> (lane, column) maps measured by
// tools/probe/tmem_probe.cu:
//   32x32b : thread t <-> lane t, register i <-> column i
//   16x256b.xN at lane L : register 4j + 2h + e <-> lane L + 8h + t/4,
//                          column 2(t%4) + e + 8j
// A warp may only touch lanes 32 (warp % 4) .. + 31.
// ---------------------------------------------------------------------------
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)), "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

#define ISF_R8(b) "r"(r[b]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3]), "r"(r[b + 4]), "r"(r[b + 5]), "r"(r[b + 6]), "r"(r[b + 7])
#define ISF_W8(b) "=r"(r[b]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), "=r"(r[b + 4]), "=r"(r[b + 5]), "=r"(r[b + 6]), "=r"(r[b + 7])
// 32x32b.x32: thread t's 32 words -> lane t, columns 0..31 (16 doubles as lo/hi pairs)
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t ta, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
      ISF_R8(0), ISF_R8(8), ISF_R8(16), ISF_R8(24)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t ta, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : ISF_W8(0), ISF_W8(8), ISF_W8(16), ISF_W8(24)
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void tmem_st_16x256b_x4(uint32_t ta, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      ISF_R8(0), ISF_R8(8)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t ta, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : ISF_W8(0), ISF_W8(8)
      : "r"(ta)
      : "memory");
}
// 16 doubles -> column pairs 0..15 of the thread's lane: one asm block, so the base
// address goes to a uniform register once (separate statements each get their own
// R2UR) and every double stays in its own aligned register pair (no marshalling)
__device__ __forceinline__ void tmem_park16(uint32_t ta, const double (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+0], {%1,%2};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+2], {%3,%4};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+4], {%5,%6};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+6], {%7,%8};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+8], {%9,%10};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+10], {%11,%12};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+12], {%13,%14};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+14], {%15,%16};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+16], {%17,%18};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+18], {%19,%20};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+20], {%21,%22};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+22], {%23,%24};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+24], {%25,%26};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+26], {%27,%28};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+28], {%29,%30};\n"
      "tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+30], {%31,%32};\n"
      ::"r"(ta), "r"((uint32_t)__double2loint(v[0])), "r"((uint32_t)__double2hiint(v[0])), "r"((uint32_t)__double2loint(v[1])), "r"((uint32_t)__double2hiint(v[1])), "r"((uint32_t)__double2loint(v[2])), "r"((uint32_t)__double2hiint(v[2])), "r"((uint32_t)__double2loint(v[3])), "r"((uint32_t)__double2hiint(v[3])), "r"((uint32_t)__double2loint(v[4])), "r"((uint32_t)__double2hiint(v[4])), "r"((uint32_t)__double2loint(v[5])), "r"((uint32_t)__double2hiint(v[5])), "r"((uint32_t)__double2loint(v[6])), "r"((uint32_t)__double2hiint(v[6])), "r"((uint32_t)__double2loint(v[7])), "r"((uint32_t)__double2hiint(v[7])), "r"((uint32_t)__double2loint(v[8])), "r"((uint32_t)__double2hiint(v[8])), "r"((uint32_t)__double2loint(v[9])), "r"((uint32_t)__double2hiint(v[9])), "r"((uint32_t)__double2loint(v[10])), "r"((uint32_t)__double2hiint(v[10])), "r"((uint32_t)__double2loint(v[11])), "r"((uint32_t)__double2hiint(v[11])), "r"((uint32_t)__double2loint(v[12])), "r"((uint32_t)__double2hiint(v[12])), "r"((uint32_t)__double2loint(v[13])), "r"((uint32_t)__double2hiint(v[13])), "r"((uint32_t)__double2loint(v[14])), "r"((uint32_t)__double2hiint(v[14])), "r"((uint32_t)__double2loint(v[15])), "r"((uint32_t)__double2hiint(v[15]))
      : "memory");
}
#undef ISF_R8
#undef ISF_W8
// 16 doubles parked at columns 0..31 of the thread's lane -> registers (waits)
__device__ __forceinline__ void tmem_load16(uint32_t ta, double (&c)[16]) {
  uint32_t r[32];
  tmem_ld_32x32b_x32(ta, r);
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}

// ---------------------------------------------------------------------------
// Decoupled look-back over warp tiles (single-pass variable-length output).
// status word: [63:40] epoch, [39:38] flag (1 aggregate, 2 inclusive), [37:0] value
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t lb_pack(uint32_t epoch, uint32_t flag, uint64_t v) {
  return ((uint64_t)(epoch & 0xffffffu) << 40) | ((uint64_t)flag << 38) | (v & ((1ull << 38) - 1));
}

// Called by a full warp; returns the exclusive prefix of `agg` over tiles < tile.
__device__ __forceinline__ uint64_t warp_lookback(uint64_t* status, uint32_t tile, uint64_t agg,
                                                  uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed(&status[0], lb_pack(epoch, 2, agg));
    return 0;
  }
  if (lane == 0) st_relaxed(&status[tile], lb_pack(epoch, 1, agg));
  uint64_t prefix = 0;
  int64_t base = (int64_t)tile - 1;
  const uint32_t ep = epoch & 0xffffffu;
  for (;;) {
    const int64_t j = base - lane;
    uint64_t w = 0;
    uint32_t flag;
    for (;;) {
      if (j >= 0) {
        w = ld_relaxed(&status[j]);
        flag = ((uint32_t)(w >> 40) == ep) ? (uint32_t)((w >> 38) & 3u) : 0u;
      } else {
        w = 0;
        flag = 2;
      }
      if (!__any_sync(0xffffffffu, flag == 0)) break;
      __nanosleep(32);
    }
    const unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
    const int first = incl ? (__ffs(incl) - 1) : 32;
    uint64_t v = (lane <= first) ? (w & ((1ull << 38) - 1)) : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    prefix += v;
    if (incl) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed(&status[tile], lb_pack(epoch, 2, prefix + agg));
  return prefix;
}

}  // namespace dev
}  // namespace isf
