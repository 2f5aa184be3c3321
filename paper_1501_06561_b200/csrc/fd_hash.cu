// fd_hash.cu — Hashing / OSNAP sketch:
//   B += S A,  S = s stacked count-sketch matrices of ell' = ell / s rows; row i of A
//   goes to row h_j(i) of block j with sign sigma_j(i), scaled 1/sqrt(s) (DESIGN.md
//   C28; s = 1 is Hashing, s = 4 OSNAP).  h, sigma: splitmix64 of (seed, i, j).
//
// B200 design: an HBM stream of A with fp64 bucket accumulators in shared memory.
// CTA = (64-column slice, contiguous row range), 64*s threads: thread (c, j) owns
// column c of block j's ell' buckets, so no two threads touch one accumulator and
// a warp's 32 accumulators of a row are contiguous (conflict-free).  Each CTA writes
// its fp64 partial; hash_reduce_kernel adds the partials in range order into B
// (deterministic; B is the caller's fp64 accumulator, so calls add up: mergeable).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "fd_internal.h"

namespace fdk {

namespace {

#ifndef FD_HASH_COLS
#define FD_HASH_COLS 64
#endif
#ifndef FD_HASH_CTAS
#define FD_HASH_CTAS 3
#endif
constexpr int kHashCols = FD_HASH_COLS;   // columns per CTA (a multiple of 32)
constexpr int kHashCtas = FD_HASH_CTAS;   // CTAs per SM the row ranges are sized for

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <int BATCH>
__global__ void __launch_bounds__(BATCH >= 64 ? kHashCols : 512) hash_kernel(const float* __restrict__ A, int64_t n, int64_t ld, int64_t d,
                                                   int ell, int s, uint64_t seed, int64_t row0, int64_t rows_per_range,
                                                   double* __restrict__ partials) {
  static_assert(32 % BATCH == 0 || BATCH % 32 == 0, "hash batches (32 rows) and load batches nest");
  extern __shared__ double hacc[];   // [ell][64]: block j's bucket h at row j * lb + h
  const int lb = ell / s;
  const int c = threadIdx.x % kHashCols, j = threadIdx.x / kHashCols;
  const int64_t col = (int64_t)blockIdx.x * kHashCols + c;
  for (int e = threadIdx.x; e < ell * kHashCols; e += blockDim.x) hacc[e] = 0.0;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_range;
  const int nrows = (int)max((int64_t)0, min(n, r0 + rows_per_range) - r0);
  const bool cv = col < d;
  double* my = hacc + (size_t)j * lb * kHashCols + c;
  const int lane = threadIdx.x & 31;
  // rows of this range through a running pointer (32-bit steps); BATCH-row load batches
  // with the next batch loaded while this one accumulates
  const float* pa = A + r0 * ld + (cv ? col : 0);
  float cur[BATCH], nxt[BATCH];
#pragma unroll
  for (int q = 0; q < BATCH; ++q) cur[q] = (q < nrows && cv) ? __ldg(pa + (int64_t)q * ld) : 0.f;
  constexpr int NC = BATCH >= 32 ? BATCH / 32 : 1;   // hash groups of 32 rows per load batch
  int code[NC];
#pragma unroll
  for (int t = 0; t < NC; ++t) code[t] = 0;
  for (int k = 0; k < nrows; k += BATCH) {
    if ((k & 31) == 0) {
      // lane l hashes row kh + l for this warp's block j (the hash depends on the row and
      // block only, so a row's bucket is warp-uniform); broadcast by shuffles below
#pragma unroll
      for (int t = 0; t < NC; ++t) {
        const int kh = k + 32 * t;
        code[t] = 0;
        if (kh + lane < nrows) {
          const uint64_t i = (uint64_t)(row0 + r0 + kh + lane);
          const uint64_t x = mix64(seed ^ (i * (uint64_t)s + (uint64_t)j) * 0xD1B54A32D192ED03ull);
          const uint32_t h = (uint32_t)(((uint64_t)(uint32_t)(x >> 32) * (uint64_t)lb) >> 32);   // multiply-shift range
          code[t] = (int)(h << 1) | (int)(x & 1ull);
        }
      }
    }
    pa += BATCH * ld;
    if (k + 2 * BATCH <= nrows && cv) {      // full next batch: no per-row predicates
      const float* p = pa;
#pragma unroll
      for (int q = 0; q < BATCH; ++q) { nxt[q] = __ldg(p); p += ld; }
    } else {
#pragma unroll
      for (int q = 0; q < BATCH; ++q) nxt[q] = (k + BATCH + q < nrows && cv) ? __ldg(pa + (int64_t)q * ld) : 0.f;
    }
    const int base = k & 31;
    const int nb = min(BATCH, nrows - k);
    if (nb == BATCH) {
#pragma unroll
      for (int q = 0; q < BATCH; ++q) {
        const int cd = __shfl_sync(0xffffffffu, code[q / 32], (base + q) & 31);
        my[(cd >> 1) * kHashCols] += (cd & 1) ? -(double)cur[q] : (double)cur[q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < BATCH; ++q) {
        const int cd = __shfl_sync(0xffffffffu, code[q / 32], (base + q) & 31);
        if (q < nb) my[(cd >> 1) * kHashCols] += (cd & 1) ? -(double)cur[q] : (double)cur[q];
      }
    }
#pragma unroll
    for (int q = 0; q < BATCH; ++q) cur[q] = nxt[q];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ell * kHashCols; e += blockDim.x) {
    const int b = e / kHashCols, cc = e % kHashCols;
    const int64_t col2 = (int64_t)blockIdx.x * kHashCols + cc;
    if (col2 < d) partials[((size_t)blockIdx.y * ell + b) * d + col2] = hacc[e];
  }
}

__global__ void hash_reduce_kernel(const double* __restrict__ partials, int R, int ell, int64_t d, double scale,
                                   double* __restrict__ B) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ne = (int64_t)ell * d;
  if (e >= ne) return;
  double acc = 0.0;
  for (int r = 0; r < R; ++r) acc += partials[(size_t)r * ne + e];
  B[e] += acc * scale;
}

}  // namespace

// row ranges per column slice: one wave of 3 CTAs per SM (64 KiB of fp64 buckets each at ell = 128)
int hash_ranges(int64_t d) {
  const int nslices = (int)((d + kHashCols - 1) / kHashCols);
  return std::max(1, (kHashCtas * kNumSMs) / nslices);
}

bool hash_supported(int ell, int s) {
  return s >= 1 && s <= 8 && ell >= s && ell % s == 0 && (size_t)ell * kHashCols * sizeof(double) <= 200 * 1024;
}

cudaError_t launch_hash(const float* A, int64_t n, int64_t ld, int64_t d, int ell, int s, uint64_t seed, int64_t row0,
                        double* partials, double* B, cudaStream_t st) {
  const int nslices = (int)((d + kHashCols - 1) / kHashCols);
  const int R = hash_ranges(d);
  const int64_t rpr = (n + R - 1) / R;
  const int smem = ell * kHashCols * (int)sizeof(double);
  // load batch: 64 rows for s = 1 (64 threads per CTA, 2 warps: more loads in flight per
  // thread; c4 Hashing 24.6 / 17.6 / 15.1 ms at 16 / 32 / 64 rows), 16 rows otherwise (at
  // 32, s = 4 needs 128 registers and 2 instead of 3 CTAs fit per SM: c4 OSNAP 35.6 -> 39.0
  // ms).  FD_HASH_BATCH=16|32|64 overrides (A/B only).
  static const int env_batch = [] { const char* e = getenv("FD_HASH_BATCH"); return e ? atoi(e) : 0; }();
  int batch = (env_batch == 16 || env_batch == 32 || env_batch == 64) ? env_batch : (s <= 1 ? 64 : 16);
  if (batch == 64 && s > 1) batch = 32;   // the 64-row kernel is built for 64-thread CTAs
  auto kern = (batch == 64) ? hash_kernel<64> : (batch == 32) ? hash_kernel<32> : hash_kernel<16>;
  static AttrOnce once[3];
  if (smem > 48 * 1024) {
    if (cudaError_t e = once[batch / 32].ensure(kern, smem); e != cudaSuccess) return e;
  }
  if (n > 0) {
    kern<<<dim3((unsigned)nslices, (unsigned)R), kHashCols * s, smem, st>>>(A, n, ld, d, ell, s, seed, row0,
                                                                          rpr, partials);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t ne = (int64_t)ell * d;
    hash_reduce_kernel<<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(partials, R, ell, d, 1.0 / sqrt((double)s), B);
  }
  return cudaGetLastError();
}

}  // namespace fdk
