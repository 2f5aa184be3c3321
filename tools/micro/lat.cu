// Dependent-chain latency microbenchmarks (one warp): cycles per operation.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp64(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
__global__ void k(double* out, long long* cyc, double seed) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = 1.0 + i * 1e-9;
  __syncwarp();
  const int N = 1024;
  double x = seed + threadIdx.x * 1e-12, y = x;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999999, 1e-9);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) y = y + 1e-9;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // MUFU.RCP64H alone
  double z = x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(z)); z = r + 1.5; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // rcp64 (approx + 2 Newton)
  double w = x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) w = rcp64(w) + 1.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // IEEE fp64 division
  double v = x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = 1.0 / v + 1.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // fp64 shuffle chain
  double s = x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1e-9;
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  // shared-memory load chain (dependent index)
  int idx = threadIdx.x;
  double acc = 0.0;
  t0 = clock64();
  for (int i = 0; i < N; ++i) { double q = sm[idx]; acc += q; idx = (idx + (q > 0.5 ? 33 : 1)) & 1023; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0);
  // FFMA chain (fp32)
  float f = (float)x;
  t0 = clock64();
  for (int i = 0; i < N; ++i) f = fmaf(f, 0.9999f, 1e-6f);
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0);
  // __syncthreads (1 warp block)
  t0 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0);
  out[threadIdx.x] = x + y + z + w + v + s + acc + f;
}
// throughput: 8 warps x independent DFMA
__global__ void kt(double* out, long long* cyc) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) {
    a0 = fma(a0, 0.9999, 1e-9); a1 = fma(a1, 0.9999, 1e-9); a2 = fma(a2, 0.9999, 1e-9); a3 = fma(a3, 0.9999, 1e-9);
    a4 = fma(a4, 0.9999, 1e-9); a5 = fma(a5, 0.9999, 1e-9); a6 = fma(a6, 0.9999, 1e-9); a7 = fma(a7, 0.9999, 1e-9);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096 * 8); cudaMalloc(&c, 64 * 8);
  k<<<1, 32>>>(o, c, 1.2345); long long h[16]; cudaMemcpy(h, c, 9 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA", "DADD", "MUFU.RCP64H", "rcp64 (approx+2 Newton)", "fp64 IEEE div", "fp64 SHFL+DADD",
                      "LDS.64 (dep)+DADD", "FFMA", "__syncthreads (1 warp)"};
  for (int i = 0; i < 9; ++i) printf("%-28s %6.1f cycles\n", nm[i], h[i] / 1024.0);
  for (int th : {256, 512, 1024}) {
    kt<<<1, th>>>(o, c); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput, %4d threads x 8 chains: %.1f DFMA/clk/SM\n", th, 8.0 * 1024 * th / h[0]);
  }
  return 0;
}
