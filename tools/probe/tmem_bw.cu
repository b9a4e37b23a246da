// Throughput of a TMEM round trip used as a register transpose: per warp
// tcgen05.st.32x32b.x32 (4 KiB) + wait::st + 2 x tcgen05.ld.16x256b.x4 (or one
// 32x32b.x32) + wait::ld.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define R8(b) "=r"(r[b]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), "=r"(r[b + 4]), "=r"(r[b + 5]), "=r"(r[b + 6]), "=r"(r[b + 7])
#define W8(b) "r"(r[b]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3]), "r"(r[b + 4]), "r"(r[b + 5]), "r"(r[b + 6]), "r"(r[b + 7])

template <int MODE>
__global__ void __launch_bounds__(512) bw(uint32_t* out, int iters) {
  __shared__ uint32_t taddr_s;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((unsigned)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t ta = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + 64 * (warp >> 2);
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; i++) r[i] = t * 32 + i;
  for (int it = 0; it < iters; it++) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        W8(0), W8(8), W8(16), W8(24));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    if (MODE == 0) {
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : R8(0), R8(8) : "r"(ta));
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : R8(16), R8(24) : "r"(ta + (16u << 16)));
    } else {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
          "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : R8(0), R8(8), R8(16), R8(24) : "r"(ta));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int i = 0; i < 32; i++) r[i] += 1;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 32; i++) s ^= r[i];
  if (s == 0x12345678u) out[0] = s;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 64);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; mode++)
    for (int nw : {4, 8, 16}) {
      const int iters = 20000;
      auto k = mode ? bw<1> : bw<0>;
      k<<<sms, nw * 32>>>(d, 100);
      cudaEventRecord(e0);
      k<<<sms, nw * 32>>>(d, iters);
      cudaEventRecord(e1);
      cudaError_t e = cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = 2.0 * 4096 * iters * nw * sms;  // st + ld
      printf("mode %s warps %2d: %s  %.1f B/clk/SM (st+ld), %.0f cycles per warp-trip\n", mode ? "32x32b" : "16x256b", nw,
             cudaGetErrorString(e), bytes / (ms * 1e-3) / sms / (clk * 1e3), (ms * 1e-3) * clk * 1e3 / iters);
    }
}
