// isf_lossy.cu -- host side of the C ABI (include/isf_lossy.h): plans, GLL
// operators, launch configuration, error mapping, host-buffer entry points and
// the NCCL reduction.  Kernels live in dlt_kernels.cuh.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <utility>
#include <mutex>
#include <string>

#include "../../include/isf_lossy.h"
#include "dlt_warp.cuh"
#include "crc32.cuh"

namespace isf {
namespace host {
void build_operators(int lx, double* F, double* B, double* xd, double* wd);
}
}  // namespace isf

using namespace isf::dev;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = std::string(isf_lossy_error_code_name(code)) + ": " + buf;
  return code;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(ISF_E_TASK_FAILED, "%s failed: %s", #expr, cudaGetErrorString(_e));     \
  } while (0)

using isf::host::build_operators;  // gll_host.cpp (binary128 host code)

std::mutex g_init_mu;
bool g_dev_init[64] = {};

int init_device_constants(int device) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (device < 0 || device >= 64) return fail(ISF_E_INVALID_ARGUMENT, "device %d out of range", device);
  if (g_dev_init[device]) return 0;
  static double ops[kOpTableSize], ws[kWTableSize], xs[kWTableSize], bms[kWTableSize];
  for (int lx = 2; lx <= kMaxLx; ++lx) {
    double x[kMaxLx], w[kMaxLx];
    build_operators(lx, ops + op_offset(lx), ops + op_offset(lx) + lx * lx, x, w);
    for (int i = 0; i < lx; ++i) { ws[w_offset(lx) + i] = w[i]; xs[w_offset(lx) + i] = x[i]; }
    const double* Bm = ops + op_offset(lx) + lx * lx;  // B[i*lx + k]
    for (int k = 0; k < lx; ++k) {
      double m = 0.0;
      for (int i = 0; i < lx; ++i) m = std::max(m, std::fabs(Bm[i * lx + k]));
      bms[w_offset(lx) + k] = m;
    }
  }
  CUDA_TRY(cudaMemcpyToSymbol(c_bm, bms, sizeof bms));
  CUDA_TRY(cudaMemcpyToSymbol(c_ops, ops, sizeof ops));
  CUDA_TRY(cudaMemcpyToSymbol(c_w, ws, sizeof ws));
  CUDA_TRY(cudaMemcpyToSymbol(c_x, xs, sizeof xs));
  {  // lx = 8: a private copy of F and B per sweep (dlt_common.cuh, c_f8 / c_b8)
    double f8[3][64], b8[3][64];
    for (int t = 0; t < 3; ++t) {
      memcpy(f8[t], ops + op_offset(8), sizeof(double) * 64);
      memcpy(b8[t], ops + op_offset(8) + 64, sizeof(double) * 64);
    }
    CUDA_TRY(cudaMemcpyToSymbol(c_f8, f8, sizeof f8));
    CUDA_TRY(cudaMemcpyToSymbol(c_b8, b8, sizeof b8));
  }
  static isf::crc::Tables crc_tables;
  static bool crc_built = false;
  if (!crc_built) { isf::crc::build_tables(crc_tables); crc_built = true; }
  CUDA_TRY(cudaMemcpyToSymbol(isf::crc::g_tables, &crc_tables, sizeof crc_tables));
  g_dev_init[device] = true;
  return 0;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

uint64_t header_bytes(uint32_t P, uint64_t nblocks) {
  const uint64_t W = ((uint64_t)P * P * P + 63) / 64;
  return ((4 * nblocks + 15) & ~15ull) + 8 * W * nblocks;
}

}  // namespace

struct isf_lossy_plan {
  int device = 0;
  uint32_t P = 0, comps = 0;
  int sms = 0;
  uint64_t* status = nullptr;
  uint64_t* csum = nullptr;  // per-chunk kept counts (lx = 8 compress): 2 x status_cap, double buffered
  int csum_par = 0;
  uint32_t csum_hw = 0;      // most chunks any call used (both buffers are clean beyond it)
  uint64_t* rstat = nullptr;  // single-pass compress: [round][cta] epoch-tagged aggregates
  size_t rstat_cap = 0;
  int c8_mode = ISF_COMPRESS_AUTO;  // lx = 8 compress schedule (isf_lossy_plan_set_compress_mode)
  bool use_sp = false;        // the schedule of the current call
  uint64_t* density_h = nullptr;  // pinned + mapped: (kept, coefficients) of the last lx = 8 compress
  uint64_t* density_d = nullptr;
  int grid8dv = 0;            // decompress8 for vector fields (components = 3)
  size_t status_cap = 0;
  double* partials = nullptr;
  size_t partials_cap = 0;  // slots of 4 doubles
  uint64_t* toff = nullptr;  // tile offsets (lx = 8 fast path)
  size_t toff_cap = 0;
  double* vslot = nullptr;   // compress value slots (lx = 8 fast path)
  size_t vslot_cap = 0;
  uint32_t* counter = nullptr;
  unsigned long long* flags = nullptr;
  isf_lossy_stats* d_stats = nullptr;
  isf_lossy_stats* h_stats = nullptr;  // pinned
  uint32_t epoch = 0;
  int last_launches = 0;
  double F[kMaxLx * kMaxLx], B[kMaxLx * kMaxLx], x[kMaxLx], w[kMaxLx];
  // host-path staging
  void* d_in = nullptr;
  size_t d_in_cap = 0;
  void* d_out = nullptr;
  size_t d_out_cap = 0;
  void* d_aux = nullptr;
  size_t d_aux_cap = 0;
  cudaStream_t host_stream = nullptr;
  // device CRC / framing
  uint32_t* crc_chunks = nullptr;
  size_t crc_cap = 0;
  uint64_t* crc_n = nullptr;
  int grid8c = 0, grid8d = 0, grid8de = 0, gridg = 0;
  size_t smem_g = 0;
  bool use_warp = false;  // scalar lx != 8: warp-per-block decompress (dlt_warp.cuh)
};

namespace {

// ntiles: look-back descriptors; nparts: partial slots; noff: block-offset entries.
// Growth: cudaFree synchronises the device (no kernel of an earlier call still uses the
// old buffers) and the zeroing is ordered on the caller's stream s, before the kernels
// that accumulate into / look back on the new buffers.
int ensure(isf_lossy_plan* p, size_t ntiles, size_t nparts, size_t noff, cudaStream_t s) {
  if (ntiles > p->status_cap) {
    if (p->status) cudaFree(p->status);
    if (p->csum) cudaFree(p->csum);
    p->csum = nullptr;
    size_t cap = std::max<size_t>(ntiles, 1024);
    CUDA_TRY(cudaMalloc(&p->status, cap * sizeof(uint64_t)));
    CUDA_TRY(cudaMemsetAsync(p->status, 0, cap * sizeof(uint64_t), s));
    p->csum_hw = 0;
    CUDA_TRY(cudaMalloc(&p->csum, 2 * cap * sizeof(uint64_t)));
    CUDA_TRY(cudaMemsetAsync(p->csum, 0, 2 * cap * sizeof(uint64_t), s));
    p->status_cap = cap;
  }
  if (noff > p->toff_cap) {
    if (p->toff) cudaFree(p->toff);
    size_t cap = std::max<size_t>(noff, 1024);
    CUDA_TRY(cudaMalloc(&p->toff, cap * sizeof(uint64_t)));
    p->toff_cap = cap;
  }
  if (nparts > p->partials_cap) {
    if (p->partials) cudaFree(p->partials);
    size_t cap = std::max<size_t>(nparts, 1024);
    // + kFinChunks records of scratch for the two-level statistics reduction
    CUDA_TRY(cudaMalloc(&p->partials, (cap + kFinChunks) * 4 * sizeof(double)));
    p->partials_cap = cap;
  }
  return 0;
}

uint32_t next_epoch(isf_lossy_plan* p, cudaStream_t s) {
  p->epoch = (p->epoch + 1) & 0xffffffu;
  if (p->epoch == 0) {  // wrapped: clear stale descriptors
    cudaMemsetAsync(p->status, 0, p->status_cap * sizeof(uint64_t), s);
    if (p->rstat) cudaMemsetAsync(p->rstat, 0, p->rstat_cap * sizeof(uint64_t), s);
    p->epoch = 1;
  }
  return p->epoch;
}

// Launch with programmatic dependent launch: the kernel may be scheduled while its
// stream predecessor drains; every fast-path kernel starts with griddepcontrol.wait
// (dev::pdl_wait), so it reads nothing before the predecessor has completed.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// The single-pass lx = 8 schedule spins on the per-round aggregates of every CTA, so all
// CTAs must be co-resident: a cooperative launch guarantees it (or fails, e.g. when
// other work or MPS limits the SMs, and the caller falls back to the two-pass schedule).
template <typename... KArgs, typename... Args>
cudaError_t launch_coop_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

template <int LX>
int launch_compress_generic(isf_lossy_plan* p, CompressArgs a, cudaStream_t s) {
  const size_t sm = GenSmem<LX>::bytes;
  static std::once_flag attr_once[64];
  cudaError_t ae = cudaSuccess;
  std::call_once(attr_once[p->device & 63], [&] {
    ae = cudaFuncSetAttribute(compress_generic<LX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  });
  CUDA_TRY(ae);
  int occ = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, compress_generic<LX>, kGenCThreads, sm));
  occ = std::max(occ, 1);
  const uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)p->sms * occ, a.ws.ntiles ? a.ws.ntiles : 1);
  a.ws.total_warps = grid;
  compress_generic<LX><<<grid, kGenCThreads, sm, s>>>(a);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <int LX>
int launch_decompress_generic(isf_lossy_plan* p, DecompressArgs a, cudaStream_t s, uint32_t* grid_out) {
  const size_t sm = GenDSmem<LX>::bytes;
  static std::once_flag attr_once[64];
  cudaError_t ae = cudaSuccess;
  std::call_once(attr_once[p->device & 63], [&] {
    ae = cudaFuncSetAttribute(decompress_generic<LX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  });
  CUDA_TRY(ae);
  int occ = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, decompress_generic<LX>, gen_dthreads<LX>(), sm));
  occ = std::max(occ, 1);
  const uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)p->sms * occ, a.ws.ntiles ? a.ws.ntiles : 1);
  a.ws.total_warps = grid;
  *grid_out = grid;
  decompress_generic<LX><<<grid, gen_dthreads<LX>(), sm, s>>>(a);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <int LX>
int launch_decompress_w(isf_lossy_plan* p, DecompressArgs a, cudaStream_t s, uint32_t* grid_out) {
  using G = WG<LX>;
  const size_t sm = G::d_bytes * G::NWD;
  static std::once_flag attr_once[64];
  cudaError_t ae = cudaSuccess;
  std::call_once(attr_once[p->device & 63], [&] {
    ae = cudaFuncSetAttribute(decompress_w<LX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  });
  CUDA_TRY(ae);
  int occ = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, decompress_w<LX>, G::NWD * 32, sm));
  occ = std::max(occ, 1);
  const uint64_t need = (a.nblocks + G::NWD - 1) / G::NWD;
  const uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)p->sms * occ, need);
  a.ws.total_warps = grid * G::NWD;
  *grid_out = grid;
  decompress_w<LX><<<grid, G::NWD * 32, sm, s>>>(a);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <int... Ls>
struct LxList {};

template <int L0, int... Ls>
int dispatch_decompress_w(LxList<L0, Ls...>, int lx, isf_lossy_plan* p, const DecompressArgs& a, cudaStream_t s,
                          uint32_t* g) {
  if (lx == L0) return launch_decompress_w<L0>(p, a, s, g);
  if constexpr (sizeof...(Ls) > 0) return dispatch_decompress_w(LxList<Ls...>{}, lx, p, a, s, g);
  return fail(ISF_E_INVALID_ARGUMENT, "unsupported P=%d", lx);
}
using WarpLx = LxList<4, 5, 6, 10, 12>;

template <int L0, int... Ls>
int dispatch_compress_generic(LxList<L0, Ls...>, int lx, isf_lossy_plan* p, const CompressArgs& a, cudaStream_t s) {
  if (lx == L0) return launch_compress_generic<L0>(p, a, s);
  if constexpr (sizeof...(Ls) > 0) return dispatch_compress_generic(LxList<Ls...>{}, lx, p, a, s);
  return fail(ISF_E_INVALID_ARGUMENT, "unsupported P=%d", lx);
}
template <int L0, int... Ls>
int dispatch_decompress_generic(LxList<L0, Ls...>, int lx, isf_lossy_plan* p, const DecompressArgs& a,
                                cudaStream_t s, uint32_t* g) {
  if (lx == L0) return launch_decompress_generic<L0>(p, a, s, g);
  if constexpr (sizeof...(Ls) > 0) return dispatch_decompress_generic(LxList<Ls...>{}, lx, p, a, s, g);
  return fail(ISF_E_INVALID_ARGUMENT, "unsupported P=%d", lx);
}
using AllLx = LxList<2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16>;

bool use_fast8(const isf_lossy_plan* p) { return p->P == 8 && (p->comps == 1 || p->comps == 3); }

int check_plan(const isf_lossy_plan* p) {
  if (!p) return fail(ISF_E_INVALID_ARGUMENT, "null plan");
  return 0;
}

// RD(eps^2) = m 2^e with m < 2^53 an integer (truncation rule v2): the
// exact square is p + err (err = fma(eps, eps, -p)); round down when err < 0.  Near the
// subnormal range the fma error is not exact, so binary128 decides there.
void eps2_rd(double max_error, uint64_t& m, int& e) {
  double p = max_error * max_error;
  if (p < 0x1p-960) {
    const __float128 q = (__float128)max_error * (__float128)max_error;
    p = (double)q;
    if ((__float128)p > q) p = std::nextafter(p, 0.0);
  } else if (std::fma(max_error, max_error, -p) < 0.0) {
    p = std::nextafter(p, 0.0);
  }
  int ex = 0;
  const double fr = std::frexp(p, &ex);
  m = (uint64_t)std::ldexp(fr, 53);
  e = ex - 53;
}

}  // namespace

extern "C" {

const char* isf_lossy_last_error(void) { return g_last_error.c_str(); }

const char* isf_lossy_error_code_name(int status) {
  static const char* names[] = {"BadMagic", "UnsupportedVersion", "LengthMismatch", "ChecksumMismatch",
                                "SerializationFailed", "ConnectFailed", "VersionMismatch", "InvalidCapacity",
                                "ReaderGone", "WriterGone", "StagingError", "CalibrationFailed",
                                "ShapeMismatch", "UnknownCodec", "DegenerateRange", "InvalidCadence",
                                "DegenerateSamples", "TaskFailed", "ConsumerCrashed", "ConfigError",
                                "InvalidArgument"};
  if (status == 0) return "Ok";
  if (status >= 1 && status <= 21) return names[status - 1];
  return "UnknownError";
}

double isf_lossy_compression_ratio(uint64_t original_size, uint64_t compressed_size) {
  return ((double)original_size - (double)compressed_size) / (double)original_size;
}

uint64_t isf_lossy_stream_header_bytes(uint32_t P, uint32_t comps, uint64_t n_elements) {
  return header_bytes(P, n_elements * comps);
}

uint64_t isf_lossy_stream_capacity(uint32_t P, uint32_t comps, uint64_t n_elements) {
  const uint64_t B = n_elements * comps;
  return header_bytes(P, B) + 8ull * P * P * P * B;
}

int isf_lossy_plan_create(isf_lossy_plan** out, uint32_t P, uint32_t comps, int device) {
  if (!out) return fail(ISF_E_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  if (P < 2 || P > (uint32_t)kMaxLx)
    return fail(ISF_E_INVALID_ARGUMENT, "points_per_element_axis must be in [2,%d], got %u", kMaxLx, P);
  if (comps != 1 && comps != 3) return fail(ISF_E_INVALID_ARGUMENT, "components must be 1 or 3, got %u", comps);
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(ISF_E_INVALID_ARGUMENT, "device %d not present (%d devices)", device, ndev);
  DeviceGuard dg(device);
  if (int rc = init_device_constants(device)) return rc;
  auto* p = new isf_lossy_plan();
  p->device = device;
  p->P = P;
  p->comps = comps;
  CUDA_TRY(cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaMalloc(&p->counter, 64));
  CUDA_TRY(cudaMemset(p->counter, 0, 64));
  CUDA_TRY(cudaMalloc(&p->flags, 64));
  CUDA_TRY(cudaMemset(p->flags, 0, 64));
  CUDA_TRY(cudaMalloc(&p->d_stats, sizeof(isf_lossy_stats)));
  CUDA_TRY(cudaMallocHost(&p->h_stats, sizeof(isf_lossy_stats)));
  build_operators((int)P, p->F, p->B, p->x, p->w);
  {
    const char* e = getenv("ISF_LOSSY_NO_WARP");  // dev override: decompress_generic for every lx
    // the orders where it measured faster (profiles/r2/decompress_warp_sweep.json): lx 4 +70 %,
    // 5 +26 %, 6 +4 %, 10 +2 %, 12 +15 %; lx 7, 9, 11 within +-4 % keep the generic kernel
    p->use_warp = comps == 1 && (P == 4 || P == 5 || P == 6 || P == 10 || P == 12) && !(e && e[0] == '1');
  }
  if (use_fast8(p)) {
    CUDA_TRY(cudaFuncSetAttribute(compress8_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kC8Smem));
    CUDA_TRY(cudaFuncSetAttribute(decompress8_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  d8_smem<false>()));
    CUDA_TRY(cudaFuncSetAttribute(decompress8_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  d8_smem<true>()));
    CUDA_TRY(cudaFuncSetAttribute(compress8_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kC8Smem));
    if (p->comps == 3) {  // vector fields: the cp.async-gather instantiations
      CUDA_TRY(cudaFuncSetAttribute(compress8_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kC8Smem));
      CUDA_TRY(cudaFuncSetAttribute(compress8_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kC8Smem));
    }
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, compress8_kernel<true>, kC8Warps * 32, kC8Smem));
    p->grid8c = p->sms * std::max(occ, 1);
    // host-mapped density record of the auto schedule (zeroed: two-pass until a call completes)
    CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&p->density_h), 2 * sizeof(uint64_t), cudaHostAllocMapped));
    p->density_h[0] = p->density_h[1] = 0;
    CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->density_d), p->density_h, 0));
    {
      const char* e = getenv("ISF_C8_KERNEL");  // dev override of the default schedule
      if (e && strcmp(e, "singlepass") == 0) p->c8_mode = ISF_COMPRESS_SINGLE_PASS;
      if (e && strcmp(e, "twopass") == 0) p->c8_mode = ISF_COMPRESS_TWO_PASS;
    }
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, decompress8_kernel<false>, d8_warps<false>() * 32,
                                                           d8_smem<false>()));
    p->grid8d = p->sms * std::max(occ, 1);
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, decompress8_kernel<true>, d8_warps<true>() * 32,
                                                           d8_smem<true>()));
    p->grid8de = p->sms * std::max(occ, 1);
    if (p->comps == 3) {
      CUDA_TRY(cudaFuncSetAttribute(decompress8_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    d8_vec_smem()));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, decompress8_kernel<false, true>, kD8VecWarps * 32,
                                                             d8_vec_smem()));
      p->grid8dv = p->sms * std::max(occ, 1);
    }
  }
  CUDA_TRY(ensure(p, 1 << 16, 1 << 14, 1 << 16, 0) == 0 ? cudaSuccess : cudaErrorMemoryAllocation);
  // the zeroing above ran on the legacy stream: complete it before any caller stream
  // (possibly non-blocking) can use the plan
  CUDA_TRY(cudaDeviceSynchronize());
  *out = p;
  return 0;
}

int isf_lossy_plan_destroy(isf_lossy_plan* p) {
  if (!p) return 0;
  DeviceGuard dg(p->device);
  cudaFree(p->status);
  cudaFree(p->csum);
  cudaFree(p->rstat);
  cudaFree(p->partials);
  cudaFree(p->toff);
  cudaFree(p->vslot);
  cudaFree(p->counter);
  cudaFree(p->flags);
  cudaFree(p->d_stats);
  cudaFreeHost(p->h_stats);
  cudaFree(p->d_in);
  cudaFree(p->d_out);
  cudaFree(p->d_aux);
  cudaFree(p->crc_chunks);
  cudaFree(p->crc_n);
  if (p->density_h) cudaFreeHost(p->density_h);
  if (p->host_stream) cudaStreamDestroy(p->host_stream);
  delete p;
  return 0;
}

int isf_lossy_plan_operators(const isf_lossy_plan* p, double* F, double* B, double* x, double* w) {
  if (int rc = check_plan(p)) return rc;
  const int n = (int)p->P;
  if (F) memcpy(F, p->F, sizeof(double) * n * n);
  if (B) memcpy(B, p->B, sizeof(double) * n * n);
  if (x) memcpy(x, p->x, sizeof(double) * n);
  if (w) memcpy(w, p->w, sizeof(double) * n);
  return 0;
}

int isf_lossy_plan_last_launches(const isf_lossy_plan* p) { return p ? p->last_launches : -1; }

int isf_lossy_plan_set_compress_mode(isf_lossy_plan* p, int mode) {
  if (int rc = check_plan(p)) return -rc;
  if (mode != ISF_COMPRESS_TWO_PASS && mode != ISF_COMPRESS_SINGLE_PASS && mode != ISF_COMPRESS_AUTO)
    return -fail(ISF_E_INVALID_ARGUMENT, "unknown compress mode %d", mode);
  const int prev = p->c8_mode;
  p->c8_mode = mode;
  return prev;
}

int isf_lossy_compress_async(isf_lossy_plan* p, const double* d_field, uint64_t n_elements, double max_error,
                             int error_norm, void* d_stream, uint64_t capacity, isf_lossy_stats* d_stats,
                             void* cuda_stream) {
  if (int rc = check_plan(p)) return rc;
  if (!(max_error > 0.0 && max_error < 1.0))
    return fail(ISF_E_INVALID_ARGUMENT, "LossyConfig: max_error must be in (0,1), got %g", max_error);
  if (error_norm != ISF_NORM_RELATIVE_L2 && error_norm != ISF_NORM_RELATIVE_LINF)
    return fail(ISF_E_INVALID_ARGUMENT, "LossyConfig: unknown error_norm %d", error_norm);
  if (n_elements == 0) return fail(ISF_E_INVALID_ARGUMENT, "empty field (0 elements)");
  if (!d_field || !d_stream || !d_stats) return fail(ISF_E_INVALID_ARGUMENT, "null device pointer");
  if (((uintptr_t)d_field & 15) || ((uintptr_t)d_stream & 15))
    return fail(ISF_E_INVALID_ARGUMENT, "field and stream must be 16-byte aligned");
  const uint64_t B = n_elements * p->comps;
  const uint64_t hdr = header_bytes(p->P, B);
  if (capacity < hdr) return fail(ISF_E_SERIALIZATION_FAILED, "capacity %llu < stream header %llu",
                                  (unsigned long long)capacity, (unsigned long long)hdr);
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const bool fast = use_fast8(p) && error_norm == ISF_NORM_RELATIVE_L2;  // RelativeLInf: generic kernels
  if (B >= (1ull << 31)) return fail(ISF_E_INVALID_ARGUMENT, "field too large for one call");
  const uint32_t ntiles = (uint32_t)B;  // generic: one tile per block; fast: one warp per block
  const uint32_t nchunks8 = (ntiles + kOffChunk - 1) / kOffChunk;
  const size_t nparts = fast ? (size_t)p->grid8c * kC8Warps : (size_t)ntiles;
  if (int rc = ensure(p, fast ? nchunks8 : ntiles, nparts, B + 1, s)) return rc;
  CompressArgs a;
  a.field = d_field;
  a.nblocks = B;
  a.comps = (int)p->comps;
  a.stream = (uint8_t*)d_stream;
  a.cap = capacity;
  a.mask_off = (4 * B + 15) & ~15ull;
  a.val_off = hdr;
  eps2_rd(max_error, a.eps_m, a.eps_e);
  a.eps = max_error;
  a.norm = error_norm;
  a.vslot = nullptr;
  a.ws = Workspace{p->status, p->partials, p->counter, p->flags, next_epoch(p, s), ntiles, 0};
  a.ws.csum = p->csum + p->csum_par * p->status_cap;
  if (fast) p->csum_hw = std::max<uint32_t>(p->csum_hw, nchunks8);
  const uint64_t* total_ptr = nullptr;
  int launches = 2;
  uint64_t parts = ntiles;
  if (fast) {
    const uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)p->grid8c, (B + kC8Warps - 1) / kC8Warps);
    a.ws.total_warps = grid * kC8Warps;
    parts = (uint64_t)grid * kC8Warps;
    FinalizeArgs f{0, p->partials, parts, p->status, p->toff + B, ntiles, p->flags, d_stats, B,
                   B * (uint64_t)p->P * p->P * p->P * 8, hdr, 0};
    f.density = p->density_d;
    const uint64_t cap_vals = capacity > hdr ? (capacity - hdr) / 8 : 0;
    // schedule: auto = single-pass when the plan's last completed compress kept more than
    // half of the coefficients (the slot round trip then moves ~2 C bytes; read without
    // a sync from host-mapped memory the finalize writes, so it may lag a call)
    p->use_sp = p->c8_mode == ISF_COMPRESS_SINGLE_PASS;
    if (p->c8_mode == ISF_COMPRESS_AUTO && p->density_h) {
      const volatile uint64_t* dh = p->density_h;
      const uint64_t kept = dh[0], coeffs = dh[1];
      p->use_sp = coeffs > 0 && 2 * kept > coeffs;
    }
    if (p->use_sp) {
      const uint64_t W = (uint64_t)grid * kC8Warps;
      const uint32_t nrounds = (uint32_t)((B + W - 1) / W);
      const size_t need = (size_t)nrounds * grid;
      if (need > p->rstat_cap) {
        if (p->rstat) cudaFree(p->rstat);
        p->rstat = nullptr;
        p->rstat_cap = 0;
        CUDA_TRY(cudaMalloc(&p->rstat, need * sizeof(uint64_t)));
        CUDA_TRY(cudaMemsetAsync(p->rstat, 0, need * sizeof(uint64_t), s));
        p->rstat_cap = need;
      }
      Sp8Args sp{p->rstat, a.ws.epoch, nrounds, reinterpret_cast<double*>(a.stream + a.val_off), cap_vals,
                 p->toff + B, f};
      const cudaError_t le =
          p->comps == 3 ? launch_coop_pdl(compress8_kernel<true, true>, grid, kC8Warps * 32, kC8Smem, s, a, sp)
                        : launch_coop_pdl(compress8_kernel<true>, grid, kC8Warps * 32, kC8Smem, s, a, sp);
      if (le == cudaSuccess) {
        p->last_launches = 1;
        return 0;
      }
      if (le != cudaErrorCooperativeLaunchTooLarge) CUDA_TRY(le);
      (void)cudaGetLastError();  // not co-resident now: two-pass schedule below
    }
    // two-pass: per-block value slots, packed by compact8_kernel
    const size_t slot_bytes = (size_t)B * 512 * sizeof(double);
    if (slot_bytes > p->vslot_cap) {
      if (p->vslot) cudaFree(p->vslot);
      p->vslot = nullptr;
      p->vslot_cap = 0;
      CUDA_TRY(cudaMalloc(&p->vslot, slot_bytes));
      p->vslot_cap = slot_bytes;
    }
    a.vslot = p->vslot;
    if (p->comps == 3)
      CUDA_TRY(launch_pdl(compress8_kernel<false, true>, grid, kC8Warps * 32, kC8Smem, s, a, Sp8Args{}));
    else
      CUDA_TRY(launch_pdl(compress8_kernel<false>, grid, kC8Warps * 32, kC8Smem, s, a, Sp8Args{}));
    CUDA_TRY(launch_pdl(compact8_kernel, nchunks8 + 1, kCompactThreads, 0, s, a.stream, B, a.mask_off,
                        (const uint64_t*)a.ws.csum, p->csum + (p->csum_par ^ 1) * p->status_cap,
                        (const double*)p->vslot, reinterpret_cast<double*>(a.stream + a.val_off), cap_vals,
                        p->toff + B, p->csum_hw, f));  // compaction + concurrent finalize
    p->csum_par ^= 1;
    p->last_launches = 2;
    return 0;
  }
  // generic: kept values to per-block slots, then the count scan and a packing pass
  // (no per-block look-back chain)
  {
    const size_t slot_bytes = (size_t)B * p->P * p->P * p->P * sizeof(double);
    if (slot_bytes > p->vslot_cap) {
      if (p->vslot) cudaFree(p->vslot);
      p->vslot = nullptr;
      p->vslot_cap = 0;
      CUDA_TRY(cudaMalloc(&p->vslot, slot_bytes));
      p->vslot_cap = slot_bytes;
    }
    a.vslot = p->vslot;
  }
  if (int rc = dispatch_compress_generic(AllLx{}, (int)p->P, p, a, s)) return rc;
  {
    Workspace wo = a.ws;
    wo.ntiles = nchunks8;
    wo.total_warps = std::min<uint32_t>(nchunks8, (uint32_t)p->sms * 4);
    block_offsets8_kernel<<<wo.total_warps, kOffThreads, 0, s>>>(a.stream, B, p->toff, wo, FinalizeArgs{});
    CUDA_TRY(cudaGetLastError());
    const int n3 = (int)(p->P * p->P * p->P);
    compact_generic_kernel<<<p->sms * 8, 256, 0, s>>>(a.stream, B, a.mask_off, (n3 + 63) / 64, n3, p->toff, p->vslot,
                                                     reinterpret_cast<double*>(a.stream + a.val_off),
                                                     capacity > hdr ? (capacity - hdr) / 8 : 0, p->flags);
    CUDA_TRY(cudaGetLastError());
    total_ptr = p->toff + B;
    launches = 4;
  }
  FinalizeArgs f{0, p->partials, parts, p->status, total_ptr, ntiles, p->flags, d_stats, B,
                 B * (uint64_t)p->P * p->P * p->P * 8, hdr, 0};
  if (parts >= 16 * (uint64_t)kFinChunks) {  // one record per block: reduce on many SMs first
    double* scratch = p->partials + p->partials_cap * 4;
    finalize_pre_kernel<<<kFinChunks, kFinThreads, 0, s>>>(p->partials, parts, 0, scratch);
    CUDA_TRY(cudaGetLastError());
    f.partials = scratch;
    f.nparts = kFinChunks;
    ++launches;
  }
  finalize_kernel<<<1, kFinThreads, 0, s>>>(f);
  CUDA_TRY(cudaGetLastError());
  p->last_launches = launches;
  return 0;
}

static int status_to_rc_compress(const isf_lossy_stats& st) {
  if (st.status & ISF_STATUS_NONFINITE) return fail(ISF_E_INVALID_ARGUMENT, "Field: non-finite value");
  if (st.status & ISF_STATUS_OVERFLOW)
    return fail(ISF_E_SERIALIZATION_FAILED, "stream capacity too small (need %llu bytes)",
                (unsigned long long)st.stream_bytes);
  return 0;
}

int isf_lossy_compress(isf_lossy_plan* p, const double* d_field, uint64_t n_elements, double max_error,
                       int error_norm, void* d_stream, uint64_t capacity, uint64_t* stream_bytes,
                       isf_lossy_stats* stats, void* cuda_stream) {
  if (int rc = check_plan(p)) return rc;
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (int rc = isf_lossy_compress_async(p, d_field, n_elements, max_error, error_norm, d_stream, capacity,
                                        p->d_stats, cuda_stream))
    return rc;
  CUDA_TRY(cudaMemcpyAsync(p->h_stats, p->d_stats, sizeof(isf_lossy_stats), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (stats) *stats = *p->h_stats;
  if (stream_bytes) *stream_bytes = p->h_stats->stream_bytes;
  return status_to_rc_compress(*p->h_stats);
}

int isf_lossy_decompress_async(isf_lossy_plan* p, const void* d_stream, uint64_t stream_bytes, uint64_t n_elements,
                               double* d_out, const double* d_original, isf_lossy_stats* d_stats,
                               void* cuda_stream) {
  if (int rc = check_plan(p)) return rc;
  if (n_elements == 0) return fail(ISF_E_INVALID_ARGUMENT, "empty field (0 elements)");
  if (!d_stream || !d_out || !d_stats) return fail(ISF_E_INVALID_ARGUMENT, "null device pointer");
  if (((uintptr_t)d_out & 15) || ((uintptr_t)d_stream & 15) || ((uintptr_t)d_original & 15))
    return fail(ISF_E_INVALID_ARGUMENT, "stream, output and original must be 16-byte aligned");
  const uint64_t B = n_elements * p->comps;
  const uint64_t hdr = header_bytes(p->P, B);
  if (stream_bytes < hdr)
    return fail(ISF_E_SHAPE_MISMATCH, "stream of %llu bytes is shorter than its header (%llu bytes) for %llu elements",
                (unsigned long long)stream_bytes, (unsigned long long)hdr, (unsigned long long)n_elements);
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const bool fast = use_fast8(p);
  if (B >= (1ull << 31)) return fail(ISF_E_INVALID_ARGUMENT, "field too large for one call");
  const uint32_t ntiles = (uint32_t)B;
  const uint32_t nchunks8 = (ntiles + kOffChunk - 1) / kOffChunk;
  const size_t nparts = fast ? std::max<size_t>((size_t)p->grid8d * kD8Warps, (size_t)p->grid8de * kD8WarpsErr)
                             : (size_t)p->sms * 16;
  if (int rc = ensure(p, std::max<uint32_t>(nchunks8, 1), nparts, B + 1, s)) return rc;
  DecompressArgs a;
  a.stream = (const uint8_t*)d_stream;
  a.stream_bytes = stream_bytes;
  a.nblocks = B;
  a.comps = (int)p->comps;
  a.mask_off = (4 * B + 15) & ~15ull;
  a.val_off = hdr;
  a.out = d_out;
  a.orig = d_original;
  a.ws = Workspace{p->status, p->partials, p->counter, p->flags, next_epoch(p, s), ntiles, 0};
  uint32_t grid = 0, parts = 0;
  const uint64_t* total_ptr = nullptr;
  int launches = 2;
  if (fast) {
    Workspace wo = a.ws;
    wo.ntiles = nchunks8;
    wo.total_warps = std::min<uint32_t>(nchunks8, (uint32_t)p->sms * 4);
    CUDA_TRY(launch_pdl(block_offsets8_kernel, wo.total_warps, kOffThreads, 0, s, (const uint8_t*)d_stream, B, p->toff,
                        wo, FinalizeArgs{}));
    CUDA_TRY(cudaGetLastError());
    const bool vec = p->comps == 3 && !d_original;
    const int nw = d_original ? kD8WarpsErr : (vec ? kD8VecWarps : kD8Warps);
    grid = (uint32_t)std::min<uint64_t>((uint64_t)(d_original ? p->grid8de : (vec ? p->grid8dv : p->grid8d)),
                                        (B + nw - 1) / nw);
    a.ws.total_warps = grid * nw;
    parts = grid * nw;
    FinalizeArgs f{1, p->partials, d_original ? parts : 0u, p->status, p->toff + B, ntiles, p->flags, d_stats, B,
                   B * (uint64_t)p->P * p->P * p->P * 8, hdr, d_original ? 1 : 0};
    Decompress8Args a8{a, p->toff, f};
    if (d_original)  // + error report and fused finalize
      CUDA_TRY(launch_pdl(decompress8_kernel<true>, grid, d8_warps<true>() * 32, d8_smem<true>(), s, a8));
    else if (vec)
      CUDA_TRY(launch_pdl(decompress8_kernel<false, true>, grid, kD8VecWarps * 32, d8_vec_smem(), s, a8));
    else
      CUDA_TRY(launch_pdl(decompress8_kernel<false>, grid, d8_warps<false>() * 32, d8_smem<false>(), s, a8));
    CUDA_TRY(cudaGetLastError());
    p->last_launches = 2;
    return 0;
  } else {
    // value offsets from the stored counts first (the same scan as the lx = 8 path)
    Workspace wo = a.ws;
    wo.ntiles = nchunks8;
    wo.total_warps = std::min<uint32_t>(nchunks8, (uint32_t)p->sms * 4);
    block_offsets8_kernel<<<wo.total_warps, kOffThreads, 0, s>>>((const uint8_t*)d_stream, B, p->toff, wo,
                                                                  FinalizeArgs{});
    CUDA_TRY(cudaGetLastError());
    a.off = p->toff;
    total_ptr = p->toff + B;
    launches = 3;
    if (p->use_warp && !d_original) {
      if (int rc = dispatch_decompress_w(WarpLx{}, (int)p->P, p, a, s, &grid)) return rc;
    } else if (int rc = dispatch_decompress_generic(AllLx{}, (int)p->P, p, a, s, &grid)) {
      return rc;
    }
    parts = grid;
  }
  FinalizeArgs f{1, p->partials, d_original ? parts : 0u, p->status, total_ptr, ntiles, p->flags, d_stats, B,
                 B * (uint64_t)p->P * p->P * p->P * 8, hdr, d_original ? 1 : 0};
  finalize_kernel<<<1, kFinThreads, 0, s>>>(f);
  CUDA_TRY(cudaGetLastError());
  p->last_launches = launches;
  return 0;
}

int isf_lossy_decompress(isf_lossy_plan* p, const void* d_stream, uint64_t stream_bytes, uint64_t n_elements,
                         double* d_out, const double* d_original, isf_lossy_stats* stats, void* cuda_stream) {
  if (int rc = check_plan(p)) return rc;
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (int rc = isf_lossy_decompress_async(p, d_stream, stream_bytes, n_elements, d_out, d_original, p->d_stats,
                                          cuda_stream))
    return rc;
  CUDA_TRY(cudaMemcpyAsync(p->h_stats, p->d_stats, sizeof(isf_lossy_stats), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  isf_lossy_stats st = *p->h_stats;
  if (stats) *stats = st;
  if ((st.status & ISF_STATUS_SHAPE) || st.stream_bytes != stream_bytes)
    return fail(ISF_E_SHAPE_MISMATCH, "stream inconsistent with shape (%llu elements of P=%u): %llu bytes given, %llu implied",
                (unsigned long long)n_elements, p->P, (unsigned long long)stream_bytes,
                (unsigned long long)st.stream_bytes);
  return 0;
}

static int grow(void** ptr, size_t* cap, size_t need) {
  if (need <= *cap) return 0;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *cap = 0;
  CUDA_TRY(cudaMalloc(ptr, need));
  *cap = need;
  return 0;
}

int isf_lossy_compress_host(isf_lossy_plan* p, const double* h_field, uint64_t n_elements, double max_error,
                            int error_norm, void* h_stream, uint64_t capacity, uint64_t* stream_bytes,
                            isf_lossy_stats* stats) {
  if (int rc = check_plan(p)) return rc;
  if (!h_field || !h_stream) return fail(ISF_E_INVALID_ARGUMENT, "null host pointer");
  DeviceGuard dg(p->device);
  if (!p->host_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->host_stream, cudaStreamNonBlocking));
  const uint64_t fbytes = n_elements * p->comps * (uint64_t)p->P * p->P * p->P * 8;
  const uint64_t cap = std::min<uint64_t>(capacity, isf_lossy_stream_capacity(p->P, p->comps, n_elements));
  if (int rc = grow(&p->d_in, &p->d_in_cap, fbytes)) return rc;
  if (int rc = grow(&p->d_out, &p->d_out_cap, cap)) return rc;
  cudaStream_t s = p->host_stream;
  CUDA_TRY(cudaMemcpyAsync(p->d_in, h_field, fbytes, cudaMemcpyHostToDevice, s));
  uint64_t nb = 0;
  isf_lossy_stats st;
  int rc = isf_lossy_compress(p, (const double*)p->d_in, n_elements, max_error, error_norm, p->d_out, cap, &nb,
                              &st, s);
  if (stats) *stats = st;
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(h_stream, p->d_out, nb, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (stream_bytes) *stream_bytes = nb;
  return 0;
}

int isf_lossy_decompress_host(isf_lossy_plan* p, const void* h_stream, uint64_t stream_bytes, uint64_t n_elements,
                              double* h_out, const double* h_original, isf_lossy_stats* stats) {
  if (int rc = check_plan(p)) return rc;
  if (!h_stream || !h_out) return fail(ISF_E_INVALID_ARGUMENT, "null host pointer");
  DeviceGuard dg(p->device);
  if (!p->host_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->host_stream, cudaStreamNonBlocking));
  const uint64_t fbytes = n_elements * p->comps * (uint64_t)p->P * p->P * p->P * 8;
  const size_t sb = (stream_bytes + 15) & ~15ull;
  if (int rc = grow(&p->d_in, &p->d_in_cap, sb)) return rc;
  if (int rc = grow(&p->d_out, &p->d_out_cap, fbytes)) return rc;
  if (h_original) {
    if (int rc = grow(&p->d_aux, &p->d_aux_cap, fbytes)) return rc;
  }
  cudaStream_t s = p->host_stream;
  CUDA_TRY(cudaMemcpyAsync(p->d_in, h_stream, stream_bytes, cudaMemcpyHostToDevice, s));
  if (h_original) CUDA_TRY(cudaMemcpyAsync(p->d_aux, h_original, fbytes, cudaMemcpyHostToDevice, s));
  isf_lossy_stats st;
  int rc = isf_lossy_decompress(p, p->d_in, stream_bytes, n_elements, (double*)p->d_out,
                                h_original ? (const double*)p->d_aux : nullptr, &st, s);
  if (stats) *stats = st;
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(h_out, p->d_out, fbytes, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

// ---- NCCL (resolved at run time) ----
// ---------------------------------------------------------------------------
// Device CRC-32 and kind-1 framing (crc32.cuh)
// ---------------------------------------------------------------------------
namespace {
int crc_launch(isf_lossy_plan* p, const uint8_t* d, const uint64_t* n_dev, uint64_t n_max, uint32_t* out,
               uint8_t* frame_tail, cudaStream_t s) {
  const size_t nch = (size_t)((n_max + isf::crc::kChunk - 1) / isf::crc::kChunk) + 1;
  if (nch > p->crc_cap) {
    if (p->crc_chunks) cudaFree(p->crc_chunks);
    const size_t cap = std::max<size_t>(nch, 4096);
    CUDA_TRY(cudaMalloc(&p->crc_chunks, cap * sizeof(uint32_t)));
    p->crc_cap = cap;
  }
  const uint64_t warps = std::max<uint64_t>(nch, 1);
  const uint32_t grid = (uint32_t)std::min<uint64_t>((warps + 7) / 8, (uint64_t)p->sms * 8);
  isf::crc::crc_chunks_kernel<<<grid, 256, 0, s>>>(d, n_dev, n_max, p->crc_chunks);
  CUDA_TRY(cudaGetLastError());
  isf::crc::crc_final_kernel<<<1, isf::crc::kFinalThreads, 0, s>>>(p->crc_chunks, n_dev, n_max, out, frame_tail);
  CUDA_TRY(cudaGetLastError());
  return 0;
}
}  // namespace

extern "C" {

int isf_lossy_crc32(isf_lossy_plan* p, const void* d_data, uint64_t n, uint32_t* d_crc, void* cuda_stream) {
  if (int rc = check_plan(p)) return rc;
  if ((!d_data && n) || !d_crc) return fail(ISF_E_INVALID_ARGUMENT, "null data or output pointer");
  DeviceGuard dg(p->device);
  p->last_launches = 2;
  return crc_launch(p, (const uint8_t*)d_data, nullptr, n, d_crc, nullptr, (cudaStream_t)cuda_stream);
}

int isf_lossy_frame_async(isf_lossy_plan* p, void* d_frame, uint64_t frame_cap, const void* d_stream,
                          uint64_t n_elements, const isf_lossy_stats* d_stats, uint32_t elements_per_axis,
                          uint64_t step_index, double sim_time, void* cuda_stream) {
  if (int rc = check_plan(p)) return rc;
  if (!d_frame || !d_stats || !d_stream) return fail(ISF_E_INVALID_ARGUMENT, "null frame, stream or stats pointer");
  if (((uintptr_t)d_frame & 15u) != 0 || ((uintptr_t)d_stream & 15u) != 0)
    return fail(ISF_E_INVALID_ARGUMENT, "frame and stream must be 16-byte aligned");
  if (n_elements == 0) return fail(ISF_E_INVALID_ARGUMENT, "empty field (0 elements)");
  if (frame_cap < ISF_FRAME_OVERHEAD) return fail(ISF_E_LENGTH_MISMATCH, "frame capacity below %d bytes", ISF_FRAME_OVERHEAD);
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (!p->crc_n) CUDA_TRY(cudaMalloc(&p->crc_n, 64));
  const uint64_t B = n_elements * p->comps;
  if (B >= (1ull << 31)) return fail(ISF_E_INVALID_ARGUMENT, "field too large for one call");
  const uint32_t nchunks = (uint32_t)((B + kOffChunk - 1) / kOffChunk);
  if (int rc = ensure(p, std::max<uint32_t>(nchunks, 1), 1, B + 1, s)) return rc;
  // block value offsets of the stream (the same count scan as decompress)
  Workspace wo{p->status, p->partials, p->counter, p->flags, next_epoch(p, s), nchunks, 0};
  wo.total_warps = std::min<uint32_t>(nchunks, (uint32_t)p->sms * 4);
  block_offsets8_kernel<<<wo.total_warps, kOffThreads, 0, s>>>((const uint8_t*)d_stream, B, p->toff, wo,
                                                                FinalizeArgs{});
  CUDA_TRY(cudaGetLastError());
  isf::crc::spec_frame_kernel<<<p->sms * 4, 256, 0, s>>>(
      (uint8_t*)d_frame, frame_cap, (const uint8_t*)d_stream, p->toff, n_elements, elements_per_axis, p->P, p->comps,
      &d_stats->kept, step_index, sim_time, p->crc_n,
      reinterpret_cast<unsigned long long*>(const_cast<uint64_t*>(&d_stats->status)));
  CUDA_TRY(cudaGetLastError());
  if (int rc = crc_launch(p, (const uint8_t*)d_frame, p->crc_n, frame_cap - 4, nullptr, (uint8_t*)d_frame, s))
    return rc;
  p->last_launches = 4;
  return 0;
}

uint64_t isf_lossy_frame_capacity(uint32_t P, uint32_t comps, uint64_t n_elements) {
  return ISF_FRAME_OVERHEAD + 4 * n_elements + 12 * n_elements * comps * (uint64_t)P * P * P;
}

}  // extern "C"

namespace {
// isf_lossy_allreduce_n: the n records [n][12] are re-laid out in place as
//   [sum f64: err2 nrm2 disc2 tot2 x n | max f64: err_inf u_inf x n |
//    sum u64: kept blocks stream field status-lanes x n | unused x n]
// so one NCCL group of three all-reduces covers every record.  status is a bit set
// and NCCL has no OR: bit k is spread into 16-bit lane k, summed, and every non-zero
// lane folded back to its bit (exact for < 65536 ranks).
constexpr uint32_t kMaxReduceRecords = 256;
__global__ void stats_pack_kernel(uint64_t* st, uint32_t n, int unpack) {
  __shared__ uint64_t t[kMaxReduceRecords * 12];
  for (uint32_t i = threadIdx.x; i < 12 * n; i += blockDim.x) t[i] = st[i];
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) {
    uint64_t* sf = st;            // 4n
    uint64_t* mf = st + 4 * n;    // 2n
    uint64_t* su = st + 6 * n;    // 5n
    if (!unpack) {
      const uint64_t* x = t + 12 * r;
      sf[4 * r + 0] = x[0]; sf[4 * r + 1] = x[1]; sf[4 * r + 2] = x[4]; sf[4 * r + 3] = x[5];
      mf[2 * r + 0] = x[2]; mf[2 * r + 1] = x[3];
      for (int k = 0; k < 4; ++k) su[5 * r + k] = x[6 + k];
      uint64_t lanes = 0;
      for (int k = 0; k < 4; ++k) lanes |= ((x[10] >> k) & 1ull) << (16 * k);
      su[5 * r + 4] = lanes;
      st[11 * n + r] = x[11];
    } else {
      uint64_t y[12];
      const uint64_t* tf = t;
      const uint64_t* tm = t + 4 * n;
      const uint64_t* tu = t + 6 * n;
      y[0] = tf[4 * r]; y[1] = tf[4 * r + 1]; y[4] = tf[4 * r + 2]; y[5] = tf[4 * r + 3];
      y[2] = tm[2 * r]; y[3] = tm[2 * r + 1];
      for (int k = 0; k < 4; ++k) y[6 + k] = tu[5 * r + k];
      uint64_t bits = 0;
      for (int k = 0; k < 4; ++k) bits |= (((tu[5 * r + 4] >> (16 * k)) & 0xFFFFull) != 0) ? (1ull << k) : 0ull;
      y[10] = bits;
      y[11] = t[11 * n + r];
      for (int k = 0; k < 12; ++k) st[12 * r + k] = y[k];
    }
  }
}
}  // namespace

typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_group_fn)(void);

namespace {
struct NcclSyms {
  nccl_allreduce_fn ar = nullptr;
  nccl_group_fn gs = nullptr, ge = nullptr;
};
// The communicator belongs to the NCCL instance that created it (e.g. the one torch
// loaded): prefer an already-loaded libnccl (RTLD_NOLOAD), then the global scope, and
// only then load one.  Resolved once (thread safe).
const NcclSyms& nccl_syms() {
  static NcclSyms s;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_NOLOAD);
    void* src = h ? h : RTLD_DEFAULT;
    s.ar = (nccl_allreduce_fn)dlsym(src, "ncclAllReduce");
    s.gs = (nccl_group_fn)dlsym(src, "ncclGroupStart");
    s.ge = (nccl_group_fn)dlsym(src, "ncclGroupEnd");
    if (!s.ar || !s.gs || !s.ge) {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (h) {
        s.ar = (nccl_allreduce_fn)dlsym(h, "ncclAllReduce");
        s.gs = (nccl_group_fn)dlsym(h, "ncclGroupStart");
        s.ge = (nccl_group_fn)dlsym(h, "ncclGroupEnd");
      }
    }
  });
  return s;
}
}  // namespace

int isf_lossy_allreduce_n(isf_lossy_stats* d_stats, uint32_t n, void* comm, void* cuda_stream) {
  if (!d_stats || !comm) return fail(ISF_E_INVALID_ARGUMENT, "null stats or communicator");
  if (n == 0 || n > kMaxReduceRecords) return fail(ISF_E_INVALID_ARGUMENT, "record count %u not in [1, %u]", n, kMaxReduceRecords);
  const NcclSyms& N = nccl_syms();
  if (!N.ar || !N.gs || !N.ge) return fail(ISF_E_TASK_FAILED, "NCCL not found in the process");
  // ncclDataType_t: ncclUint64 = 5, ncclFloat64 = 8; ncclRedOp_t: ncclSum = 0, ncclMax = 2
  cudaStream_t s = (cudaStream_t)cuda_stream;
  uint64_t* u = reinterpret_cast<uint64_t*>(d_stats);
  double* d = reinterpret_cast<double*>(d_stats);
  stats_pack_kernel<<<1, 256, 0, s>>>(u, n, 0);
  CUDA_TRY(cudaGetLastError());
  int r = N.gs();
  r |= N.ar(d, d, 4 * (size_t)n, 8, 0, comm, s);                    // energies (sum)
  r |= N.ar(d + 4 * n, d + 4 * n, 2 * (size_t)n, 8, 2, comm, s);    // Linf terms (max)
  r |= N.ar(u + 6 * n, u + 6 * n, 5 * (size_t)n, 5, 0, comm, s);    // counts, bytes, status lanes (sum)
  r |= N.ge();
  if (r) return fail(ISF_E_TASK_FAILED, "ncclAllReduce failed (%d)", r);
  stats_pack_kernel<<<1, 256, 0, s>>>(u, n, 1);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int isf_lossy_allreduce(isf_lossy_stats* d_stats, void* comm, void* cuda_stream) {
  return isf_lossy_allreduce_n(d_stats, 1, comm, cuda_stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Synthetic in-situ producers.  Not on the timed path.
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ double Wg_node(int P, int i) { return c_x[w_offset(P) + i]; }

__global__ void tgv_kernel(double* out, uint32_t E, uint32_t ez0, uint64_t nel, int P, int which, double h) {
  const uint64_t n3 = (uint64_t)P * P * P;
  const uint64_t total = nel * n3;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = t / n3, p = t % n3;
    const uint64_t ex = e % E, ey = (e / E) % E, ez = e / ((uint64_t)E * E) + ez0;
    const int px = (int)(p % P), py = (int)((p / P) % P), pz = (int)(p / ((uint64_t)P * P));
    const double rx = (Wg_node(P, px) + 1.0) * 0.5 * h, ry = (Wg_node(P, py) + 1.0) * 0.5 * h,
                 rz = (Wg_node(P, pz) + 1.0) * 0.5 * h;
    const double x = (double)ex * h + rx, y = (double)ey * h + ry, z = (double)ez * h + rz;
    double v;
    switch (which) {
      case 0: v = cos(x) * sin(y) * sin(z); break;
      case 1: v = -sin(x) * cos(y) * sin(z); break;
      case 2: v = 0.0; break;
      default: v = (cos(2.0 * x) + cos(2.0 * y)) * (cos(2.0 * z) + 2.0) / 16.0; break;
    }
    out[t] = v;
  }
}

__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// dense stream: counts = n3, masks all ones, values = (2U-1)*amp[j]
__global__ void spectral_stream_kernel(uint8_t* stream, uint64_t nblocks, uint64_t block0, int n3, int W,
                                       uint64_t mask_off, uint64_t val_off, uint64_t seed, const double* amp) {
  uint32_t* counts = reinterpret_cast<uint32_t*>(stream);
  uint64_t* masks = reinterpret_cast<uint64_t*>(stream + mask_off);
  double* vals = reinterpret_cast<double*>(stream + val_off);
  const uint64_t lastmask = (n3 % 64) ? ((1ull << (n3 % 64)) - 1ull) : ~0ull;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nblocks * n3; t += stride) {
    const uint64_t b = t / n3;
    const uint32_t j = (uint32_t)(t % n3);
    const uint64_t gblk = block0 + b;
    uint32_t c[4] = {(uint32_t)gblk, (uint32_t)(gblk >> 32), j, 0u};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t M = ((uint64_t)c[0] << 21) | (c[1] >> 11);
    const double U2 = ldexp((double)(int64_t)(2 * M) - 9007199254740992.0, -53);
    vals[t] = __dmul_rn(U2, amp[j]);
    if (j == 0) {
      counts[b] = (uint32_t)n3;
      if (b + 1 == nblocks) for (uint64_t pb = nblocks; pb < ((nblocks + 3) & ~3ull); ++pb) counts[pb] = 0;
    }
    if (j < (uint32_t)W) masks[b * W + j] = (j == (uint32_t)W - 1) ? lastmask : ~0ull;
  }
}

}  // namespace

extern "C" {

int isf_lossy_generate_tgv(isf_lossy_plan* p, double* d_out, uint32_t E_ax, uint32_t ez0, uint32_t nz, int which,
                           double domain, void* cuda_stream) {
  if (int rc = check_plan(p)) return rc;
  if (p->comps != 1) return fail(ISF_E_INVALID_ARGUMENT, "TGV generator writes scalar fields (components=1)");
  DeviceGuard dg(p->device);
  const uint64_t nel = (uint64_t)E_ax * E_ax * nz;
  tgv_kernel<<<p->sms * 8, 256, 0, (cudaStream_t)cuda_stream>>>(d_out, E_ax, ez0, nel, (int)p->P, which,
                                                                  domain / (double)E_ax);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int isf_lossy_generate_spectral(isf_lossy_plan* p, double* d_out, uint64_t block0, uint64_t nblocks, uint64_t seed,
                                const double* h_amp, void* cuda_stream) {
  if (int rc = check_plan(p)) return rc;
  if (p->comps != 1) return fail(ISF_E_INVALID_ARGUMENT, "spectral generator writes scalar fields (components=1)");
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const int n3 = (int)(p->P * p->P * p->P), W = (n3 + 63) / 64;
  const uint64_t bytes = isf_lossy_stream_capacity(p->P, 1, nblocks);
  void* tmp = nullptr;
  double* d_amp = nullptr;
  CUDA_TRY(cudaMallocAsync(&tmp, bytes, s));
  CUDA_TRY(cudaMallocAsync((void**)&d_amp, sizeof(double) * n3, s));
  CUDA_TRY(cudaMemcpyAsync(d_amp, h_amp, sizeof(double) * n3, cudaMemcpyHostToDevice, s));
  spectral_stream_kernel<<<p->sms * 8, 256, 0, s>>>((uint8_t*)tmp, nblocks, block0, n3, W, (4 * nblocks + 15) & ~15ull,
                                                     header_bytes(p->P, nblocks), seed, d_amp);
  CUDA_TRY(cudaGetLastError());
  int rc = isf_lossy_decompress(p, tmp, bytes, nblocks, d_out, nullptr, nullptr, cuda_stream);
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(d_amp, s);
  return rc;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Solver stand-in for the async in-situ mode (cfg5): one explicit relaxation
// step dst = src + alpha * (aux - src) over n doubles (reads 2n, writes n doubles,
// the memory-bound profile of an SEM time step).  Not part of the compression path.
// ---------------------------------------------------------------------------
namespace {
__global__ void solver_standin_kernel(double* __restrict__ dst, const double* __restrict__ src,
                                      const double* __restrict__ aux, uint64_t n2, double alpha) {
  const double2* s = reinterpret_cast<const double2*>(src);
  const double2* a = reinterpret_cast<const double2*>(aux);
  double2* d = reinterpret_cast<double2*>(dst);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n2; i += (uint64_t)gridDim.x * blockDim.x) {
    const double2 x = s[i], y = a[i];
    d[i] = make_double2(__fma_rn(alpha, y.x - x.x, x.x), __fma_rn(alpha, y.y - x.y, x.y));
  }
}
}  // namespace

#ifdef ISF_PATHSTATS
extern "C" int isf_debug_pathstats(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, isf::dev::g_pathstats, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(isf::dev::g_pathstats, z, sizeof(z));
  }
  return 0;
}
#endif
extern "C" int isf_lossy_solver_standin(double* d_dst, const double* d_src, const double* d_aux, uint64_t n,
                                        double alpha, void* cuda_stream) {
  if (!d_dst || !d_src || !d_aux || (n & 1) || (((uintptr_t)d_dst | (uintptr_t)d_src | (uintptr_t)d_aux) & 15))
    return fail(ISF_E_INVALID_ARGUMENT, "solver stand-in needs 16-B aligned buffers and an even length");
  int dev = 0, sms = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  solver_standin_kernel<<<sms * 8, 512, 0, (cudaStream_t)cuda_stream>>>(d_dst, d_src, d_aux, n / 2, alpha);
  CUDA_TRY(cudaGetLastError());
  return 0;
}
