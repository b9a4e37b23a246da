// Microbenchmarks that set the design limits for the DLT kernels on B200:
// FP64 DFMA / DMMA throughput, SHFL throughput, smem 128-bit bandwidth, HBM copy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; i++) r[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) r[i] = fma(r[i], a, b);
  }
  double s = 0; for (int i = 0; i < 16; i++) s += r[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; i++) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_shfl(int* out, int iters) {
  int r[8];
  for (int i = 0; i < 8; i++) r[i] = threadIdx.x + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) r[i] = __shfl_xor_sync(0xffffffffu, r[i], (i + 1) & 31);
  }
  int s = 0; for (int i = 0; i < 8; i++) s += r[i];
  if (s == 123456789) out[0] = s;
}
__global__ void k_smem(double* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int base = threadIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      double2 v = buf[(base + i * 256 + it) & 2047];
      acc.x += v.x; acc.y -= v.y;
    }
  }
  if (acc.x == 1.2345) out[0] = acc.y;
}
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
__global__ void k_read(const double2* __restrict__ a, double* out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  double s = 0;
  for (; i < n; i += st) { double2 v = a[i]; s += v.x + v.y; }
  if (s == 1.2345) out[0] = s;
}
__global__ void k_write(double2* __restrict__ b, size_t n, int cs) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  const double2 v = make_double2(threadIdx.x, 1.0);
  if (cs) {
    for (; i < n; i += st) asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(b + i), "d"(v.x), "d"(v.y) : "memory");
  } else {
    for (; i < n; i += st) b[i] = v;
  }
}
// TMA bulk store: each warp streams 4 KiB chunks from its smem buffer
__global__ void k_bulkstore(unsigned char* __restrict__ b, size_t nbytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  unsigned char* mine = sm + warp * 4096;
  for (int i = lane; i < 512; i += 32) reinterpret_cast<double*>(mine)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const size_t nch = nbytes / 4096;
  for (size_t c = (size_t)blockIdx.x * nw + warp; c < nch; c += (size_t)gridDim.x * nw) {
    if (lane == 0) {
      unsigned sa = (unsigned)__cvta_generic_to_shared(mine);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(b + c * 4096), "r"(sa) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA bulk-load read: each warp streams 4 KiB blocks (round robin) through an S-stage ring
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t ph) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(sa), "r"(ph) : "memory");
}
template <int S>
__global__ void k_bulkread(const unsigned char* __restrict__ a, size_t nblk, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  unsigned char* mine = sm + warp * (S * 4096 + 64);
  uint64_t* bars = reinterpret_cast<uint64_t*>(mine + S * 4096);
  if (lane == 0) {
    for (int s = 0; s < S; ++s) { unsigned sa = (unsigned)__cvta_generic_to_shared(&bars[s]); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa)); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const size_t W = (size_t)gridDim.x * nw, gw = (size_t)blockIdx.x * nw + warp;
  auto issue = [&](size_t blk, int st) {
    if (lane == 0 && blk < nblk) {
      unsigned sb = (unsigned)__cvta_generic_to_shared(&bars[st]);
      unsigned sd = (unsigned)__cvta_generic_to_shared(mine + st * 4096);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(sb) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(sd), "l"(a + blk * 4096), "r"(sb) : "memory");
    }
  };
  for (int s = 0; s < S; ++s) issue(gw + s * W, s);
  double acc = 0; int st = 0; uint32_t ph = 0;
  for (size_t blk = gw; blk < nblk; blk += W) {
    mb_wait(&bars[st], (ph >> st) & 1u); ph ^= 1u << st;
    const double2* p = reinterpret_cast<const double2*>(mine + st * 4096);
#pragma unroll
    for (int z = 0; z < 8; ++z) { double2 v = p[z * 32 + lane]; acc += v.x; }
    __syncwarp();
    issue(blk + S * W, st);
    st = st + 1 == S ? 0 : st + 1;
  }
  if (acc == 1.2345) out[0] = acc;
}
// LDG read with a warp per 4 KiB block (8 x 128-bit loads per lane, all issued before use)
__global__ void k_warpread(const double2* __restrict__ a, size_t nblk, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const size_t W = (size_t)gridDim.x * nw, gw = (size_t)blockIdx.x * nw + warp;
  double acc = 0;
  for (size_t blk = gw; blk < nblk; blk += W) {
    double2 v[8];
#pragma unroll
    for (int z = 0; z < 8; ++z) v[z] = __ldcs(a + blk * 256 + z * 32 + lane);
#pragma unroll
    for (int z = 0; z < 8; ++z) acc += v[z].x;
  }
  if (acc == 1.2345) out[0] = acc;
}
int main(int argc, char** argv) {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("GPU %s SMs %d maxclk %d MHz smemPerSM %zu regsPerSM %d\n", p.name, sms, clk / 1000, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor);
  double* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const bool only_mem = argc > 1;
  for (int rep = 0; rep < (only_mem ? 0 : 2); rep++) {
    int iters = 20000, thr = 512, blocks = sms * 4;
    k_dfma<<<blocks, thr>>>(dout, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0); k_dfma<<<blocks, thr>>>(dout, iters, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)thr * blocks;
    printf("DFMA: %.2f TFLOP/s (%.1f DFMA/clk/SM at max clk)\n", fl / ms / 1e9, fl / 2 / (ms * 1e-3) / sms / (clk * 1e3));
    k_dmma<<<blocks, 256>>>(dout, 100);
    cudaEventRecord(e0); k_dmma<<<blocks, 256>>>(dout, 4000); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 8 * 4 * 8 * 4000.0 * (256 / 32) * blocks;
    printf("DMMA m8n8k4: %.2f TFLOP/s\n", fl / ms / 1e9);
    int* iout = (int*)dout;
    k_shfl<<<blocks, thr>>>(iout, 100);
    cudaEventRecord(e0); k_shfl<<<blocks, thr>>>(iout, 20000); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double sh = 8.0 * 20000 * thr / 32 * blocks;
    printf("SHFL: %.2f warp-shfl/clk/SM\n", sh / (ms * 1e-3) / sms / (clk * 1e3));
    k_smem<<<blocks, 256>>>(dout, 100);
    cudaEventRecord(e0); k_smem<<<blocks, 256>>>(dout, 20000); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double by = 8.0 * 20000 * 256 * 16 * blocks;
    printf("LDS.128: %.1f B/clk/SM\n", by / (ms * 1e-3) / sms / (clk * 1e3));
  }
  size_t n = (size_t)1 << 28; // 4 GiB of double2
  double2 *a, *b; CK(cudaMalloc(&a, n * 16 / 2)); CK(cudaMalloc(&b, n * 16 / 2)); n /= 2;
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  for (int bs : {1, 2, 4, 8}) {
    k_copy<<<sms * bs, 512>>>(a, b, n);
    cudaEventRecord(e0); for (int r = 0; r < 5; r++) k_copy<<<sms * bs, 512>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy grid=%d*SM: %.1f GB/s\n", bs, 5.0 * 2 * n * 16 / (ms * 1e6));
    k_read<<<sms * bs, 512>>>(a, dout, n);
    cudaEventRecord(e0); for (int r = 0; r < 5; r++) k_read<<<sms * bs, 512>>>(a, dout, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("read grid=%d*SM: %.1f GB/s\n", bs, 5.0 * n * 16 / (ms * 1e6));
    for (int cs = 0; cs < 2; cs++) {
      k_write<<<sms * bs, 512>>>(b, n, cs);
      cudaEventRecord(e0); for (int r = 0; r < 5; r++) k_write<<<sms * bs, 512>>>(b, n, cs); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("write%s grid=%d*SM: %.1f GB/s\n", cs ? ".cs" : "", bs, 5.0 * n * 16 / (ms * 1e6));
    }
    cudaFuncSetAttribute(k_bulkstore, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096);
    k_bulkstore<<<sms * (bs > 2 ? 2 : bs), 512, 16 * 4096>>>((unsigned char*)b, n * 16);
    cudaEventRecord(e0); for (int r = 0; r < 5; r++) k_bulkstore<<<sms * (bs > 2 ? 2 : bs), 512, 16 * 4096>>>((unsigned char*)b, n * 16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("bulkstore grid=%d*SM: %.1f GB/s\n", bs > 2 ? 2 : bs, 5.0 * n * 16 / (ms * 1e6));
  }
  {
    const size_t nblk = n * 16 / 4096;
    auto run = [&](const char* name, auto launch) {
      launch();
      cudaEventRecord(e0); for (int r = 0; r < 5; r++) launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%s: %.1f GB/s\n", name, 5.0 * n * 16 / (ms * 1e6));
      return 0;
    };
#define BR(S, NW) { const int sm_ = NW * (S * 4096 + 64); cudaFuncSetAttribute(k_bulkread<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_); \
      char nm[64]; snprintf(nm, 64, "bulkread S=%d warps=%d", S, NW); run(nm, [&] { k_bulkread<S><<<sms, NW * 32, sm_>>>((const unsigned char*)a, nblk, dout); }); }
    BR(2, 16) BR(3, 16) BR(2, 8) BR(4, 8) BR(6, 8) BR(4, 12) BR(1, 32) BR(2, 24)
    for (int nw : {8, 16, 32}) for (int bs : {1, 2, 4}) { char nm[64]; snprintf(nm, 64, "warpread warps=%d grid=%d*SM", nw, bs); run(nm, [&] { k_warpread<<<sms * bs, nw * 32>>>(a, nblk, dout); }); }
  }
  
  return 0;
}
