// Probe of the tcgen05.ld thread <-> (TMEM lane, column) mapping of each shape:
// warp 0 fills lanes 0..31 x columns 0..63 with (lane << 8 | column) via 32x32b, then
// reads back with each shape and reports what every thread received.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void probe(uint32_t* out) {
  __shared__ uint32_t taddr_s;
  const int t = threadIdx.x;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"((unsigned)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t ta = taddr_s;
  if (t < 32) {
    for (int c = 0; c < 64; c += 4) {
      uint32_t a = ta + c;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"((t << 8) | c), "r"((t << 8) | (c + 1)), "r"((t << 8) | (c + 2)), "r"((t << 8) | (c + 3)));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    uint32_t r[8];
    // 16x64b.x1 : 1 reg
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[0 * 256 + t * 8 + 0] = r[0];
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[1 * 256 + t * 8 + 0] = r[0]; out[1 * 256 + t * 8 + 1] = r[1];
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[2 * 256 + t * 8 + 0] = r[0]; out[2 * 256 + t * 8 + 1] = r[1];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 4; i++) out[3 * 256 + t * 8 + i] = r[i];
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x1.b32 {%0}, [%1], 2;" : "=r"(r[0]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[4 * 256 + t * 8 + 0] = r[0];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; i++) out[5 * 256 + t * 8 + i] = r[i];
    // lane offset 16 within the warp's quadrant
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta + (16u << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 4; i++) out[6 * 256 + t * 8 + i] = r[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(ta));
}
int main() {
  uint32_t* d; cudaMalloc(&d, 8 * 256 * 4); cudaMemset(d, 0xff, 8 * 256 * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err %s\n", cudaGetErrorString(e));
  uint32_t h[8 * 256]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[] = {"16x64b.x1", "16x64b.x2", "16x128b.x1", "16x256b.x1", "16x32bx2.x1(off2)", "16x256b.x2", "16x256b.x1@lane16"};
  const int nr[] = {1, 2, 2, 4, 1, 8, 4};
  for (int s = 0; s < 7; s++) {
    printf("== %s  (thread: lane.col ...)\n", nm[s]);
    for (int t = 0; t < 32; t++) {
      printf("t%02d:", t);
      for (int i = 0; i < nr[s]; i++) { uint32_t v = h[s * 256 + t * 8 + i]; printf(" %2u.%-2u", v >> 8, v & 255); }
      printf(t % 4 == 3 ? "\n" : "  |");
    }
  }
}
