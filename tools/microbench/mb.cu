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
  return 0;
}
