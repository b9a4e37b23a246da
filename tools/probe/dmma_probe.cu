// dmma_probe.cu -- B200 probe: (1) the rounding behaviour of mma.sync.m8n8k4.f64
// (is each output a chain of fused multiply-adds, and in which k order?) and (2)
// whether DMMA and DFMA issue on separate pipes (time of each alone vs interleaved).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_mma_once(const double* A, const double* B, const double* C, double* D, int n) {
  const int lane = threadIdx.x & 31;
  for (int t = 0; t < n; ++t) {
    const double* a = A + t * 32;  // [8][4] row major
    const double* b = B + t * 32;  // [4][8] (k, n)
    const double* c = C + t * 64;  // [8][8]
    double av = a[(lane >> 2) * 4 + (lane & 3)];
    double bv = b[(lane & 3) * 8 + (lane >> 2)];
    double d0 = c[(lane >> 2) * 8 + 2 * (lane & 3)], d1 = c[(lane >> 2) * 8 + 2 * (lane & 3) + 1];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(av), "d"(bv));
    D[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = d0;
    D[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = d1;
  }
}

// throughput: mode 0 DMMA only, 1 DFMA only, 2 both interleaved (independent chains)
__global__ void k_mix(double* out, int iters, int mode) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-9, b = 1.0 - lane * 1e-9;
  double d[8][2];
  double f[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { d[j][0] = d[j][1] = j * 1e-3; f[j] = j * 1e-3; }
  for (int i = 0; i < iters; ++i) {
    if (mode != 1) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
    }
    if (mode != 0) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = fma(f[j], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + f[j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

static double rnd(unsigned& st) {
  st = st * 1664525u + 1013904223u;
  double m = (double)(st >> 8) / 16777216.0 - 0.5;
  st = st * 1664525u + 1013904223u;
  int e = (int)(st >> 27) - 16;
  return ldexp(m, e / 2);
}

int main() {
  const int n = 4096;
  double *hA = new double[n * 32], *hB = new double[n * 32], *hC = new double[n * 64], *hD = new double[n * 64];
  unsigned st = 12345;
  for (int i = 0; i < n * 32; ++i) { hA[i] = rnd(st); hB[i] = rnd(st); }
  for (int i = 0; i < n * 64; ++i) hC[i] = (i % 3 == 0) ? 0.0 : rnd(st);
  double *A, *B, *C, *D;
  CK(cudaMalloc(&A, n * 32 * 8)); CK(cudaMalloc(&B, n * 32 * 8)); CK(cudaMalloc(&C, n * 64 * 8)); CK(cudaMalloc(&D, n * 64 * 8));
  CK(cudaMemcpy(A, hA, n * 32 * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B, hB, n * 32 * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(C, hC, n * 64 * 8, cudaMemcpyHostToDevice));
  k_mma_once<<<1, 32>>>(A, B, C, D, n);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hD, D, n * 64 * 8, cudaMemcpyDeviceToHost));
  // candidate models
  long m_fwd = 0, m_rev = 0, m_c_last = 0, m_exact = 0, m_pair = 0, tot = 0;
  for (int t = 0; t < n; ++t)
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) {
        const double* a = hA + t * 32 + r * 4;
        double bb[4];
        for (int k = 0; k < 4; ++k) bb[k] = hB[t * 32 + k * 8 + c];
        const double cc = hC[t * 64 + r * 8 + c];
        const double got = hD[t * 64 + r * 8 + c];
        double f = cc;
        for (int k = 0; k < 4; ++k) f = fma(a[k], bb[k], f);
        double g = cc;
        for (int k = 3; k >= 0; --k) g = fma(a[k], bb[k], g);
        double h = a[0] * bb[0];
        for (int k = 1; k < 4; ++k) h = fma(a[k], bb[k], h);
        h = h + cc;
        long double ex = (long double)cc;  // 64-bit mantissa: near-exact reference
        __float128 q = (__float128)cc;
        for (int k = 0; k < 4; ++k) q += (__float128)a[k] * (__float128)bb[k];
        const double e = (double)q;
        double p = fma(a[1], bb[1], a[0] * bb[0]);
        double p2 = fma(a[3], bb[3], a[2] * bb[2]);
        double pp = (p + p2) + cc;
        (void)ex;
        ++tot;
        m_fwd += got == f;
        m_rev += got == g;
        m_c_last += got == h;
        m_exact += got == e;
        m_pair += got == pp;
      }
  printf("numerics (%ld outputs): fma chain k=0..3: %ld, k=3..0: %ld, c added last: %ld, "
         "exact sum rounded once (binary128): %ld, pairwise: %ld\n", tot, m_fwd, m_rev, m_c_last, m_exact, m_pair);
  // throughput
  double* out;
  CK(cudaMalloc(&out, 4096 * 8));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  for (int warps = 4; warps <= 16; warps *= 2) {
    float ms[3];
    for (int mode = 0; mode < 3; ++mode) {
      k_mix<<<sms, warps * 32>>>(out, 10, mode);
      cudaEventRecord(e0);
      k_mix<<<sms, warps * 32>>>(out, iters, mode);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms[mode], e0, e1);
    }
    const double dmma_fl = 2.0 * 256 * 8 * (double)iters * warps * sms;  // flops
    const double dfma_fl = 2.0 * 32 * 64 * (double)iters * warps * sms;
    printf("warps/SM %2d: DMMA alone %.3f ms (%.1f TF)  DFMA alone %.3f ms (%.1f TF)  both %.3f ms (sum %.3f)\n", warps,
           ms[0], dmma_fl / ms[0] / 1e9, ms[1], dfma_fl / ms[1] / 1e9, ms[2], ms[0] + ms[1]);
  }
  return 0;
}
