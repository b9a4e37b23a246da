// dlt_kernels.cuh -- the sm_100a kernels of the hot path.
//
//  compress8_kernel / decompress8_kernel : lx = 8, scalar fields (the north_star
//      configuration).  Warp tile = 4 consecutive blocks (16 KiB).  Loads are fully
//      coalesced 128-bit (one 512 B plane per warp instruction); lane (q, y) holds
//      the z-lines of x = 2q, 2q+1 at row y for the 4 blocks, so the z sweep runs in
//      registers; one padded shared-memory transposition gives lane (block, kz) a
//      whole kz-plane for the y and x sweeps.  Selection + encode run on the
//      8-lane group of each block; output offsets come from a decoupled look-back.
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
};

struct CompressArgs {
  const double* field;
  uint64_t nblocks;
  int comps;
  uint8_t* stream;
  uint64_t cap;
  uint64_t mask_off;  // byte offset of masks
  uint64_t val_off;   // byte offset of values
  uint64_t eps_q;     // floor(eps^2 * 2^64)
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
};

constexpr unsigned long long kFlagNonFinite = 1, kFlagShape = 2, kFlagOverflow = 4;

// --------------------------- helpers ---------------------------------------
template <int LX, int S, int O0, int DO, int CNT, bool INV, int N>
__device__ __forceinline__ void lines(double (&v)[N]) {
  if constexpr (CNT > 0) {
    if constexpr (INV) inv_line<LX, S, O0>(v); else fwd_line<LX, S, O0>(v);
    lines<LX, S, O0 + DO, DO, CNT - 1, INV>(v);
  }
}
template <int LX, int S, int O0, int DO1, int CNT1, int DO2, int CNT2, bool INV, int N>
__device__ __forceinline__ void lines2(double (&v)[N]) {
  if constexpr (CNT2 > 0) {
    lines<LX, S, O0, DO1, CNT1, INV>(v);
    lines2<LX, S, O0 + DO2, DO1, CNT1, DO2, CNT2 - 1, INV>(v);
  }
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

// --------------------------- lx = 8 selection -------------------------------
struct BlockSel {
  uint64_t mask;   // kept bits of this lane's 64 coefficients
  uint64_t T;      // group total of lo energies
  uint64_t hdisc;  // group hi-sum of the discarded set
  int k;           // energy scale exponent (e = a^2 * 2^(2k))
  bool nonfinite;
};

// c[i] = coefficient kz*64 + i of the block owned by this 8-lane group.
__device__ __forceinline__ BlockSel select8(const LaneGroup<8>& g, double (&c)[64], int kz,
                                            uint64_t eps_q, uint64_t* ckeys, uint16_t* cidx,
                                            unsigned long long* hist) {
  BlockSel r{0ull, 0ull, 0ull, 0, false};
  uint32_t hm = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) hm = ::max(hm, (uint32_t)__double2hiint(c[i]) & 0x7fffffffu);
  hm = g.max(hm);
  if (hm >= 0x7ff00000u) { r.nonfinite = true; return r; }
  int s;
  if (hm >= 0x00100000u) {
    s = (int)(hm >> 20) - 1022;
  } else {  // subnormal maximum or zero block (rare)
    uint64_t mb = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) { const uint64_t b = abs_bits(c[i]); mb = b > mb ? b : mb; }
    mb = g.max(mb);
    if (mb == 0) return r;  // all-zero block keeps nothing
    s = 64 - __clzll((long long)mb) - 1074;
  }
  constexpr int K = energy_K(8);
  int k = K - s;
  r.k = k;
  const bool tiny = k > 1023;  // |a| < 2^-998: pre-scale exactly by 2^(k-1023)
  if (tiny) {
    const double pre = pow2d(k - 1023);
#pragma unroll
    for (int i = 0; i < 64; ++i) c[i] = __dmul_rn(c[i], pre);
    k = 1023;
  }
  const double f = pow2d(k);
  uint64_t T = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) T += e_lo(c[i], f);
  T = g.sum(T);
  r.T = T;
  const uint64_t thr = __umul64hi(T, eps_q);
  // hi > thr <=> e > thr (thr integer); thr >= 2^50 > e means nothing is above it
  const double thrD = thr < (1ull << 50) ? (double)thr : 1125899906842624.0;
  uint64_t mH = 0, SN = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    const double t = __dmul_rn(c[i], f);
    const double e = __dmul_rn(t, t);
    if (e > thrD) mH |= 1ull << i;
    else SN += low52(__dadd_ru(e, 4503599627370496.0));
  }
  SN = g.sum(SN);
  if (SN <= thr) {
    r.mask = mH;
    r.hdisc = SN;
  } else {
    // hard block: split the non-kept side into definitely discarded (hi*512 <= thr)
    // and candidates; exact radix select over the candidates.
    const uint64_t thrn = thr >> 9;
    uint64_t mC = 0, SL = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if (!((mH >> i) & 1ull)) {
        const uint64_t h = e_hi(c[i], f);
        if (h <= thrn) SL += h; else mC |= 1ull << i;
      }
    }
    SL = g.sum(SL);
    const uint32_t nc = (uint32_t)__popcll(mC);
    uint32_t off = g.exscan(nc);
    const uint32_t ncT = g.sum(nc);
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if ((mC >> i) & 1ull) {
        ckeys[off] = abs_bits(c[i]);
        cidx[off] = (uint16_t)(kz * 64 + i);
        ++off;
      }
    }
    g.sync();
    uint64_t tstar, dsum;
    uint32_t icut;
    radix_select<8>(g, ckeys, cidx, (int)ncT, thr - SL, f, hist, tstar, icut, dsum);
    uint64_t mk = mH;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if ((mC >> i) & 1ull) {
        const uint64_t kk = abs_bits(c[i]);
        const uint32_t ii = (uint32_t)(kz * 64 + i);
        if (kk > tstar || (kk == tstar && ii < icut)) mk |= 1ull << i;
      }
    }
    r.mask = mk;
    r.hdisc = SL + dsum;
    g.sync();
  }
  if (tiny) {
    const double un = pow2d(1023 - r.k);
#pragma unroll
    for (int i = 0; i < 64; ++i) c[i] = __dmul_rn(c[i], un);
  }
  return r;
}

// --------------------------- lx = 8 compress --------------------------------
constexpr int kPS8 = 66;                     // padded plane stride (doubles): 528 B = 16 mod 128
constexpr int kGroupBytes8 = 5632;           // keys 4096 + idx 1024 + hist 512
constexpr int kWarpBytes8 = 4 * kGroupBytes8;  // >= 32 planes * 528 B
constexpr int kWarps8 = 8;

__global__ void __launch_bounds__(kWarps8 * 32, 1) compress8_kernel(CompressArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wbuf = smem + warp * kWarpBytes8;
  double* tb = reinterpret_cast<double*>(wbuf);
  const int q = lane & 3, y = lane >> 2, gb = lane >> 3, kz = lane & 7;
  const LaneGroup<8> g;
  unsigned char* gbuf = wbuf + gb * kGroupBytes8;
  uint64_t* ckeys = reinterpret_cast<uint64_t*>(gbuf);
  uint16_t* cidx = reinterpret_cast<uint16_t*>(gbuf + 4096);
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(gbuf + 5120);
  uint32_t* counts = reinterpret_cast<uint32_t*>(A.stream);
  uint64_t* masks = reinterpret_cast<uint64_t*>(A.stream + A.mask_off);
  double* vals = reinterpret_cast<double*>(A.stream + A.val_off);

  for (;;) {
    const uint32_t tile = claim_tile(A.ws.counter);
    if (tile >= A.ws.ntiles) {
      if (lane == 0 && tile == A.ws.ntiles + A.ws.total_warps - 1) *A.ws.counter = 0;
      break;
    }
    __syncwarp();
    const uint64_t blk0 = (uint64_t)tile * 4;
    double v[64];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const bool ok = blk0 + b < A.nblocks;
      const double2* src = reinterpret_cast<const double2*>(A.field + (blk0 + b) * 512) + y * 4 + q;
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        const double2 t = ok ? ldg_stream(src + z * 32) : make_double2(0.0, 0.0);
        v[b * 16 + z * 2] = t.x;
        v[b * 16 + z * 2 + 1] = t.y;
      }
    }
    // forward z sweep: lines (b, xi), stride 2
    lines2<8, 2, 0, 1, 2, 16, 4, false>(v);
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int z = 0; z < 8; ++z)
        *reinterpret_cast<double2*>(tb + (b * 8 + z) * kPS8 + y * 8 + 2 * q) =
            make_double2(v[b * 16 + z * 2], v[b * 16 + z * 2 + 1]);
    __syncwarp();
    {
      const double2* pl = reinterpret_cast<const double2*>(tb + (gb * 8 + kz) * kPS8);
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const double2 t = pl[r];
        v[2 * r] = t.x;
        v[2 * r + 1] = t.y;
      }
    }
    __syncwarp();
    lines<8, 8, 0, 1, 8, false>(v);  // y sweep (lines over y at fixed x)
    lines<8, 1, 0, 8, 8, false>(v);  // x sweep
    // v[ky*8+kx] = coefficient kz*64 + ky*8 + kx of block blk0+gb
    const BlockSel sel = select8(g, v, kz, A.eps_q, ckeys, cidx, hist);
    const uint64_t blk = blk0 + gb;
    const bool valid = blk < A.nblocks;
    if (sel.nonfinite && valid && kz == 0) atomicOr(A.ws.flags, kFlagNonFinite);
    const uint64_t mask = sel.nonfinite ? 0ull : sel.mask;
    const uint32_t nk = (uint32_t)__popcll(mask);
    const uint32_t kept_blk = g.sum(nk);
    const uint32_t off_in_blk = g.exscan(nk);
    const uint32_t k0 = __shfl_sync(0xffffffffu, kept_blk, 0), k1 = __shfl_sync(0xffffffffu, kept_blk, 8);
    const uint32_t k2 = __shfl_sync(0xffffffffu, kept_blk, 16), k3 = __shfl_sync(0xffffffffu, kept_blk, 24);
    const uint64_t agg = (uint64_t)k0 + k1 + k2 + k3;
    const uint32_t blk_excl = (gb > 0 ? k0 : 0) + (gb > 1 ? k1 : 0) + (gb > 2 ? k2 : 0);
    const uint64_t prefix = warp_lookback(A.ws.status, tile, agg, A.ws.epoch);
    const bool fits = A.val_off + 8 * (prefix + agg) <= A.cap;
    if (valid) {
      if (kz == 0) {
        counts[blk] = kept_blk;
        if (blk + 1 == A.nblocks && (A.nblocks & 1)) counts[blk + 1] = 0;  // pad to 8 B
      }
      masks[blk * 8 + kz] = mask;
      if (fits) {
        double* dst = vals + prefix + blk_excl + off_in_blk;
        int o = 0;
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if ((mask >> i) & 1ull) dst[o++] = v[i];
      }
    }
    if (!fits && lane == 0) atomicOr(A.ws.flags, kFlagOverflow);
    // per-tile coefficient energies (fixed order over the 4 blocks)
    double tot = 0.0, disc = 0.0;
    if (kz == 0 && valid && !sel.nonfinite) {
      tot = ldexp((double)sel.T, -2 * sel.k);
      disc = ldexp((double)sel.hdisc, -2 * sel.k);
    }
    const double t0 = __shfl_sync(0xffffffffu, tot, 0), t1 = __shfl_sync(0xffffffffu, tot, 8);
    const double t2 = __shfl_sync(0xffffffffu, tot, 16), t3 = __shfl_sync(0xffffffffu, tot, 24);
    const double d0 = __shfl_sync(0xffffffffu, disc, 0), d1 = __shfl_sync(0xffffffffu, disc, 8);
    const double d2 = __shfl_sync(0xffffffffu, disc, 16), d3 = __shfl_sync(0xffffffffu, disc, 24);
    if (lane == 0) {
      A.ws.partials[(uint64_t)tile * 4 + 0] = ((t0 + t1) + t2) + t3;
      A.ws.partials[(uint64_t)tile * 4 + 1] = ((d0 + d1) + d2) + d3;
    }
  }
}

// --------------------------- lx = 8 decompress ------------------------------
constexpr int kWarpBytesD8 = 32 * kPS8 * 8;  // 16896

__global__ void __launch_bounds__(kWarps8 * 32, 1) decompress8_kernel(DecompressArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* tb = reinterpret_cast<double*>(smem + warp * kWarpBytesD8);
  const int q = lane & 3, y = lane >> 2, gb = lane >> 3, kz = lane & 7;
  const LaneGroup<8> g;
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(A.stream);
  const uint64_t* masks = reinterpret_cast<const uint64_t*>(A.stream + A.mask_off);
  const double* vals = reinterpret_cast<const double*>(A.stream + A.val_off);
  const uint64_t nvals_avail = A.stream_bytes > A.val_off ? (A.stream_bytes - A.val_off) / 8 : 0;
  // GLL weights of this lane's (x, y) columns
  const double wxy0 = __dmul_rn(Wg<8>(2 * q), Wg<8>(y));
  const double wxy1 = __dmul_rn(Wg<8>(2 * q + 1), Wg<8>(y));
  double e2 = 0.0, n2 = 0.0;
  uint64_t einf = 0, uinf = 0;  // max |.| as ordered bit patterns

  for (;;) {
    const uint32_t tile = claim_tile(A.ws.counter);
    if (tile >= A.ws.ntiles) {
      if (lane == 0 && tile == A.ws.ntiles + A.ws.total_warps - 1) *A.ws.counter = 0;
      break;
    }
    __syncwarp();
    const uint64_t blk0 = (uint64_t)tile * 4;
    const uint64_t blk = blk0 + gb;
    const bool valid = blk < A.nblocks;
    const uint32_t cnt = valid ? __ldg(counts + blk) : 0u;
    uint64_t w = valid ? __ldg(reinterpret_cast<const unsigned long long*>(masks) + blk * 8 + kz) : 0ull;
    const uint32_t pc = (uint32_t)__popcll(w);
    const uint32_t bs = g.sum(pc);
    if (bs != cnt && kz == 0) atomicOr(A.ws.flags, kFlagShape);
    const uint32_t inoff = g.exscan(pc);
    const uint32_t k0 = __shfl_sync(0xffffffffu, cnt, 0), k1 = __shfl_sync(0xffffffffu, cnt, 8);
    const uint32_t k2 = __shfl_sync(0xffffffffu, cnt, 16), k3 = __shfl_sync(0xffffffffu, cnt, 24);
    const uint64_t agg = (uint64_t)k0 + k1 + k2 + k3;
    const uint32_t blk_excl = (gb > 0 ? k0 : 0) + (gb > 1 ? k1 : 0) + (gb > 2 ? k2 : 0);
    const uint64_t prefix = warp_lookback(A.ws.status, tile, agg, A.ws.epoch);
    const uint64_t boff = prefix + blk_excl + inoff;
    if (boff + pc > nvals_avail || bs != cnt) {
      if (w) atomicOr(A.ws.flags, kFlagShape);
      w = 0;
    }
    double v[64];
    {
      const double* src = vals + boff;
      int o = 0;
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = ((w >> i) & 1ull) ? __ldg(src + (o++)) : 0.0;
    }
    lines<8, 1, 0, 8, 8, true>(v);  // inverse x sweep
    lines<8, 8, 0, 1, 8, true>(v);  // inverse y sweep
    {
      double2* pl = reinterpret_cast<double2*>(tb + (gb * 8 + kz) * kPS8);
#pragma unroll
      for (int r = 0; r < 32; ++r) pl[r] = make_double2(v[2 * r], v[2 * r + 1]);
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        const double2 t = *reinterpret_cast<const double2*>(tb + (b * 8 + z) * kPS8 + y * 8 + 2 * q);
        v[b * 16 + z * 2] = t.x;
        v[b * 16 + z * 2 + 1] = t.y;
      }
    __syncwarp();
    lines2<8, 2, 0, 1, 2, 16, 4, true>(v);  // inverse z sweep
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (blk0 + b >= A.nblocks) continue;
      double2* dst = reinterpret_cast<double2*>(A.out + (blk0 + b) * 512) + y * 4 + q;
#pragma unroll
      for (int z = 0; z < 8; ++z) stg_stream(dst + z * 32, make_double2(v[b * 16 + z * 2], v[b * 16 + z * 2 + 1]));
      if (A.orig) {
        const double2* src = reinterpret_cast<const double2*>(A.orig + (blk0 + b) * 512) + y * 4 + q;
#pragma unroll
        for (int z = 0; z < 8; ++z) {
          const double2 o = ldg_stream(src + z * 32);
          const double wz = Wg<8>(z);
          const double w0 = __dmul_rn(wxy0, wz), w1 = __dmul_rn(wxy1, wz);
          const double da = __dsub_rn(o.x, v[b * 16 + z * 2]), db = __dsub_rn(o.y, v[b * 16 + z * 2 + 1]);
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
    }
  }
  if (A.orig) {
    // per-warp partials (fixed xor tree), one slot per warp
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      e2 = __dadd_rn(e2, __shfl_xor_sync(0xffffffffu, e2, o));
      n2 = __dadd_rn(n2, __shfl_xor_sync(0xffffffffu, n2, o));
      uint64_t t = __shfl_xor_sync(0xffffffffu, einf, o); einf = t > einf ? t : einf;
      t = __shfl_xor_sync(0xffffffffu, uinf, o); uinf = t > uinf ? t : uinf;
    }
    if (lane == 0) {
      const uint64_t slot = (uint64_t)blockIdx.x * kWarps8 + warp;
      A.ws.partials[slot * 4 + 0] = e2;
      A.ws.partials[slot * 4 + 1] = n2;
      A.ws.partials[slot * 4 + 2] = __longlong_as_double((long long)einf);
      A.ws.partials[slot * 4 + 3] = __longlong_as_double((long long)uinf);
    }
  }
}

// --------------------------- generic (any lx, comps) ------------------------
constexpr int kGenThreads = 128;

template <int LX>
struct GenSmem {
  static constexpr int N3 = LX * LX * LX;
  static constexpr int W = (N3 + 63) / 64;
  static constexpr size_t u_off = 0;
  static constexpr size_t key_off = u_off + sizeof(double) * N3;
  static constexpr size_t idx_off = key_off + sizeof(uint64_t) * N3;
  static constexpr size_t hist_off = ((idx_off + sizeof(uint16_t) * N3) + 15) & ~size_t(15);
  static constexpr size_t mask_off = hist_off + 64 * 8;
  static constexpr size_t misc_off = mask_off + 64 * 8;
  static constexpr size_t bytes = misc_off + 64;
};

// selection on warp 0 over the coefficients in smem u[]
template <int LX>
__device__ void select_generic(double* u, uint64_t eps_q, uint64_t* ckeys, uint16_t* cidx,
                               unsigned long long* hist, uint64_t* maskw, uint64_t& T_out,
                               uint64_t& hdisc_out, int& k_out, bool& nonfinite) {
  constexpr int N3 = LX * LX * LX;
  constexpr int W = (N3 + 63) / 64;
  constexpr int NR = (N3 + 31) / 32;
  const LaneGroup<32> g;
  const int lane = g.rank;
  for (int w = lane; w < 64; w += 32) maskw[w] = 0ull;
  T_out = 0; hdisc_out = 0; k_out = 0; nonfinite = false;
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
  constexpr int K = energy_K(LX);
  int k = K - s;
  k_out = k;
  const bool tiny = k > 1023;
  if (tiny) {
    const double pre = pow2d(k - 1023);
    for (int p = lane; p < N3; p += 32) u[p] = __dmul_rn(u[p], pre);
    k = 1023;
  }
  const double f = pow2d(k);
  uint64_t T = 0;
  for (int p = lane; p < N3; p += 32) T += e_lo(u[p], f);
  T = g.sum(T);
  T_out = T;
  const uint64_t thr = __umul64hi(T, eps_q);
  uint64_t SN = 0;
  for (int p = lane; p < N3; p += 32) { const uint64_t h = e_hi(u[p], f); if (h <= thr) SN += h; }
  SN = g.sum(SN);
  if (SN <= thr) {
    for (int r = 0; r < NR; ++r) {
      const int p = r * 32 + lane;
      const bool kept = p < N3 && e_hi(u[p], f) > thr;
      const unsigned b = __ballot_sync(0xffffffffu, kept);
      if (lane == 0) maskw[r >> 1] |= (uint64_t)b << (32 * (r & 1));
    }
    hdisc_out = SN;
  } else {
    const uint64_t thrn = thr / (uint64_t)N3;
    uint64_t SL = 0;
    uint32_t base = 0;
    for (int r = 0; r < NR; ++r) {
      const int p = r * 32 + lane;
      bool cand = false;
      if (p < N3) {
        const uint64_t h = e_hi(u[p], f);
        if (h <= thr) { if (h <= thrn) SL += h; else cand = true; }
      }
      const unsigned b = __ballot_sync(0xffffffffu, cand);
      if (cand) {
        const uint32_t o = base + __popc(b & ((1u << lane) - 1u));
        ckeys[o] = abs_bits(u[p]);
        cidx[o] = (uint16_t)p;
      }
      base += __popc(b);
    }
    SL = g.sum(SL);
    __syncwarp();
    uint64_t tstar, dsum;
    uint32_t icut;
    radix_select<32>(g, ckeys, cidx, (int)base, thr - SL, f, hist, tstar, icut, dsum);
    for (int r = 0; r < NR; ++r) {
      const int p = r * 32 + lane;
      bool kept = false;
      if (p < N3) {
        const uint64_t h = e_hi(u[p], f);
        if (h > thr) kept = true;
        else if (h > thrn) {
          const uint64_t kk = abs_bits(u[p]);
          kept = kk > tstar || (kk == tstar && (uint32_t)p < icut);
        }
      }
      const unsigned b = __ballot_sync(0xffffffffu, kept);
      if (lane == 0) maskw[r >> 1] |= (uint64_t)b << (32 * (r & 1));
    }
    hdisc_out = SL + dsum;
  }
  if (tiny) {
    const double un = pow2d(1023 - k_out);
    for (int p = lane; p < N3; p += 32) u[p] = __dmul_rn(u[p], un);
  }
  (void)W;
  __syncwarp();
}

template <int LX>
__global__ void __launch_bounds__(kGenThreads) compress_generic(CompressArgs A) {
  constexpr int N = LX, N2 = LX * LX, N3 = LX * LX * LX;
  constexpr int W = (N3 + 63) / 64;
  using L = GenSmem<LX>;
  extern __shared__ __align__(16) unsigned char smem[];
  double* u = reinterpret_cast<double*>(smem + L::u_off);
  uint64_t* ckeys = reinterpret_cast<uint64_t*>(smem + L::key_off);
  uint16_t* cidx = reinterpret_cast<uint16_t*>(smem + L::idx_off);
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(smem + L::hist_off);
  uint64_t* maskw = reinterpret_cast<uint64_t*>(smem + L::mask_off);
  uint64_t* misc = reinterpret_cast<uint64_t*>(smem + L::misc_off);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* counts = reinterpret_cast<uint32_t*>(A.stream);
  uint64_t* masks = reinterpret_cast<uint64_t*>(A.stream + A.mask_off);
  double* vals = reinterpret_cast<double*>(A.stream + A.val_off);
  for (;;) {
    __syncthreads();
    if (tid == 0) misc[0] = atomicAdd(A.ws.counter, 1u);
    __syncthreads();
    const uint32_t tile = (uint32_t)misc[0];
    if (tile >= A.ws.ntiles) {
      if (tid == 0 && tile == A.ws.ntiles + A.ws.total_warps - 1) *A.ws.counter = 0;
      break;
    }
    const uint64_t blk = tile;
    const uint64_t e = blk / A.comps, c = blk % A.comps;
    const double* src = A.field + e * (uint64_t)N3 * A.comps + c;
    for (int p = tid; p < N3; p += kGenThreads) u[p] = src[(uint64_t)p * A.comps];
    __syncthreads();
    for (int l = tid; l < N2; l += kGenThreads) fwd_line_ptr<LX>(u + l, N2);                       // z
    __syncthreads();
    for (int l = tid; l < N2; l += kGenThreads) fwd_line_ptr<LX>(u + (l / N) * N2 + (l % N), N);  // y
    __syncthreads();
    for (int l = tid; l < N2; l += kGenThreads) fwd_line_ptr<LX>(u + l * N, 1);                     // x
    __syncthreads();
    if (warp == 0) {
      uint64_t T, hd;
      int k;
      bool nf;
      select_generic<LX>(u, A.eps_q, ckeys, cidx, hist, maskw, T, hd, k, nf);
      if (nf) {
        for (int w = lane; w < W; w += 32) maskw[w] = 0ull;
        if (lane == 0) atomicOr(A.ws.flags, kFlagNonFinite);
      }
      __syncwarp();
      uint32_t nk = 0;
      for (int w = lane; w < W; w += 32) nk += __popcll(maskw[w]);
      const LaneGroup<32> g;
      nk = g.sum(nk);
      const uint64_t prefix = warp_lookback(A.ws.status, tile, nk, A.ws.epoch);
      const bool fits = A.val_off + 8 * (prefix + nk) <= A.cap;
      if (lane == 0) {
        counts[blk] = nk;
        if (blk + 1 == A.nblocks && (A.nblocks & 1)) counts[blk + 1] = 0;
        if (!fits) atomicOr(A.ws.flags, kFlagOverflow);
        A.ws.partials[blk * 4 + 0] = nf ? 0.0 : ldexp((double)T, -2 * k);
        A.ws.partials[blk * 4 + 1] = nf ? 0.0 : ldexp((double)hd, -2 * k);
        misc[1] = prefix;
        misc[2] = fits;
      }
      for (int w = lane; w < W; w += 32) masks[blk * W + w] = maskw[w];
    }
    __syncthreads();
    if (misc[2]) {
      // kept values in ascending index: rank = popcount of lower mask bits
      const uint64_t prefix = misc[1];
      for (int p = tid; p < N3; p += kGenThreads) {
        const uint64_t mw = maskw[p >> 6];
        if ((mw >> (p & 63)) & 1ull) {
          uint32_t rank = (uint32_t)__popcll(mw & ((1ull << (p & 63)) - 1ull));
          for (int w = 0; w < (p >> 6); ++w) rank += (uint32_t)__popcll(maskw[w]);
          vals[prefix + rank] = u[p];
        }
      }
    }
  }
}

template <int LX>
__global__ void __launch_bounds__(kGenThreads) decompress_generic(DecompressArgs A) {
  constexpr int N = LX, N2 = LX * LX, N3 = LX * LX * LX;
  constexpr int W = (N3 + 63) / 64;
  using L = GenSmem<LX>;
  extern __shared__ __align__(16) unsigned char smem[];
  double* u = reinterpret_cast<double*>(smem + L::u_off);
  uint64_t* maskw = reinterpret_cast<uint64_t*>(smem + L::mask_off);
  uint32_t* wpre = reinterpret_cast<uint32_t*>(smem + L::key_off);  // prefix popcounts per word
  uint64_t* misc = reinterpret_cast<uint64_t*>(smem + L::misc_off);
  double* red = reinterpret_cast<double*>(smem + L::hist_off);     // 4 warps x 4
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(A.stream);
  const uint64_t* masks = reinterpret_cast<const uint64_t*>(A.stream + A.mask_off);
  const double* vals = reinterpret_cast<const double*>(A.stream + A.val_off);
  const uint64_t nvals_avail = A.stream_bytes > A.val_off ? (A.stream_bytes - A.val_off) / 8 : 0;
  constexpr uint64_t lastmask = (N3 % 64) ? ((1ull << (N3 % 64)) - 1ull) : ~0ull;
  double e2 = 0.0, n2 = 0.0;
  uint64_t einf = 0, uinf = 0;
  for (;;) {
    __syncthreads();
    if (tid == 0) misc[0] = atomicAdd(A.ws.counter, 1u);
    __syncthreads();
    const uint32_t tile = (uint32_t)misc[0];
    if (tile >= A.ws.ntiles) {
      if (tid == 0 && tile == A.ws.ntiles + A.ws.total_warps - 1) *A.ws.counter = 0;
      break;
    }
    const uint64_t blk = tile;
    if (warp == 0) {
      const uint32_t cnt = counts[blk];
      uint32_t pc = 0;
      for (int w = lane; w < W; w += 32) {
        uint64_t mw = masks[blk * W + w];
        if (w == W - 1 && (mw & ~lastmask)) { atomicOr(A.ws.flags, kFlagShape); mw &= lastmask; }
        maskw[w] = mw;
        pc += __popcll(mw);
      }
      const LaneGroup<32> g;
      pc = g.sum(pc);
      const uint64_t prefix = warp_lookback(A.ws.status, tile, cnt, A.ws.epoch);
      bool bad = pc != cnt || prefix + cnt > nvals_avail;
      if (lane == 0) {
        if (bad) atomicOr(A.ws.flags, kFlagShape);
        misc[1] = prefix;
        misc[2] = bad;
        uint32_t run = 0;
        for (int w = 0; w < W; ++w) { wpre[w] = run; run += __popcll(maskw[w]); }
      }
    }
    __syncthreads();
    const uint64_t prefix = misc[1];
    const bool bad = misc[2] != 0;
    for (int p = tid; p < N3; p += kGenThreads) {
      const uint64_t mw = maskw[p >> 6];
      double val = 0.0;
      if (!bad && ((mw >> (p & 63)) & 1ull))
        val = vals[prefix + wpre[p >> 6] + __popcll(mw & ((1ull << (p & 63)) - 1ull))];
      u[p] = val;
    }
    __syncthreads();
    for (int l = tid; l < N2; l += kGenThreads) inv_line_ptr<LX>(u + l * N, 1);                     // x
    __syncthreads();
    for (int l = tid; l < N2; l += kGenThreads) inv_line_ptr<LX>(u + (l / N) * N2 + (l % N), N);  // y
    __syncthreads();
    for (int l = tid; l < N2; l += kGenThreads) inv_line_ptr<LX>(u + l, N2);                       // z
    __syncthreads();
    const uint64_t e = blk / A.comps, c = blk % A.comps;
    double* dst = A.out + e * (uint64_t)N3 * A.comps + c;
    const double* org = A.orig ? A.orig + e * (uint64_t)N3 * A.comps + c : nullptr;
    for (int p = tid; p < N3; p += kGenThreads) {
      const double val = u[p];
      dst[(uint64_t)p * A.comps] = val;
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
      for (int w = 0; w < kGenThreads / 32; ++w) {
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
  uint32_t ntiles;
  unsigned long long* flags;
  void* stats;              // isf_lossy_stats*
  uint64_t nblocks, field_bytes, val_off;
  int with_error;
};

constexpr int kFinThreads = 512;

__global__ void __launch_bounds__(kFinThreads) finalize_kernel(FinalizeArgs A) {
  __shared__ double s0[kFinThreads], s1[kFinThreads];
  __shared__ unsigned long long m0[kFinThreads], m1[kFinThreads];
  const int t = threadIdx.x;
  double a0 = 0.0, a1 = 0.0;
  unsigned long long x0 = 0, x1 = 0;
  for (uint64_t i = t; i < A.nparts; i += kFinThreads) {
    a0 = __dadd_rn(a0, A.partials[i * 4 + 0]);
    a1 = __dadd_rn(a1, A.partials[i * 4 + 1]);
    if (A.mode == 1) {
      unsigned long long v = (unsigned long long)__double_as_longlong(A.partials[i * 4 + 2]);
      x0 = v > x0 ? v : x0;
      v = (unsigned long long)__double_as_longlong(A.partials[i * 4 + 3]);
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
  if (t == 0) {
    double* st = reinterpret_cast<double*>(A.stats);
    uint64_t* su = reinterpret_cast<uint64_t*>(A.stats);
    const uint64_t last = A.ntiles ? ld_relaxed(A.status + (A.ntiles - 1)) : 0ull;
    const uint64_t total = last & ((1ull << 38) - 1);
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
