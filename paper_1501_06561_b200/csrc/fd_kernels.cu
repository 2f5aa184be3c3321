// fd_kernels.cu — sm_100a kernels of the Frequent Directions hot path.
//
// One ReduceRank (Alg. 1 lines "svd(B_[i]) ... B_[i] <- S'V^T")
// of a batch of independent shard buffers is three kernels:
//   gram_kernel   G = Bf Bf^T                         (buffer Gram, fp32)
//   eig_kernel    G = U diag(lambda) U^T; delta = lambda_ell; rule -> w_j;
//                 Wt = diag(w) U[:, :ell-1]^T         (one CTA per problem)
//   recon_kernel  B' = Wt Bf   (= S'V^T since V^T = S^-1 U^T Bf)
// plus ingest_kernel (rows of A -> shard buffers, ||a||^2 in fp64) and the
// cov-err evaluator (fp64 A^T A, M = A^T A - B^T B, Lanczos).
//
// The eigen-solver is Householder tridiagonalisation (LAPACK ssytd2 order,
// fp32, packed lower triangle resident in shared memory), multisection
// bisection on Sturm counts for the top ell eigenvalues, fp64 inverse
// iteration (with modified Gram-Schmidt inside eigenvalue clusters) for the
// ell-1 retained eigenvectors, and a fp32 Householder back-transform.
#include <cuda_runtime.h>
#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <float.h>
#include <math.h>
#include <stdint.h>

#include "fd_internal.h"

namespace fdk {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ============================================================================
// ingest: rows of A (user layout, any ld / alignment) -> shard buffer (ldb),
// fp64 sum of squares, non-finite detection.  One CTA per shard-round.
// ============================================================================
__global__ void __launch_bounds__(256) ingest_kernel(const Ingest* __restrict__ desc, Params p,
                                                     int* __restrict__ nonfinite) {
  const Ingest D = desc[blockIdx.x];
  const int64_t d = p.d, ldb = p.ldb;
  double acc = 0.0;
  int bad = 0;
  const bool vec = ((D.ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(D.src) & 15) == 0) && ((d & 3) == 0);
  if (vec) {
    const int64_t nq = d >> 2;
    const int64_t total = (int64_t)D.nrows * nq;
    for (int64_t q = threadIdx.x; q < total; q += blockDim.x) {
      const int64_t r = q / nq, c = q - r * nq;
      float4 v = __ldcs(reinterpret_cast<const float4*>(D.src + r * D.ld) + c);
      bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
      acc += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
      reinterpret_cast<float4*>(D.dst + r * ldb)[c] = v;
    }
  } else {
    const int64_t total = (int64_t)D.nrows * ldb;
    for (int64_t q = threadIdx.x; q < total; q += blockDim.x) {
      const int64_t r = q / ldb, c = q - r * ldb;
      float v = 0.f;
      if (c < d) {
        v = D.src[r * D.ld + c];
        bad |= !isfinite(v);
        acc += (double)v * v;
      }
      D.dst[r * ldb + c] = v;
    }
  }
  __shared__ double red[8];
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    D.stats->frob += s;
    if (bad) atomicOr(nonfinite, 1);
  }
}

cudaError_t launch_ingest(const Ingest* dev_desc, int count, const Params& p, int* nonfinite, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  ingest_kernel<<<count, 256, 0, s>>>(dev_desc, p, nonfinite);
  return cudaGetLastError();
}

// ============================================================================
// Gram: G = Bf Bf^T for Bf = [src0 (rows0); src1 (rows1)] in precision T
// (fp32 rows are exact in fp64), 64x64 lower-triangular output tiles, both
// triangles written.
// ============================================================================
__device__ __forceinline__ const float* prob_row(const Prob& P, int r, int64_t ldb) {
  if (r < P.rows0) return P.src0 + (int64_t)r * ldb;
  r -= P.rows0;
  if (r < P.rows1) return P.src1 + (int64_t)r * P.ld1;
  return nullptr;
}

__device__ __forceinline__ void tri_index(int t, int& ti, int& tj) {
  int i = (int)((sqrtf(8.f * (float)t + 1.f) - 1.f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  ti = i;
  tj = t - i * (i + 1) / 2;
}

template <typename T>
__global__ void __launch_bounds__(256) gram_kernel(const Prob* __restrict__ probs, Params p) {
  const Prob P = probs[blockIdx.y];
  const int N = P.rows0 + P.rows1;
  int ti, tj;
  tri_index(blockIdx.x, ti, tj);
  if (ti * 64 >= N) return;
  __shared__ __align__(16) T As[16][68];
  __shared__ __align__(16) T Bs[16][68];
  const int lr = threadIdx.x >> 2, lk = (threadIdx.x & 3) * 4;
  const float* arow = (ti * 64 + lr < N) ? prob_row(P, ti * 64 + lr, p.ldb) : nullptr;
  const float* brow = (tj * 64 + lr < N) ? prob_row(P, tj * 64 + lr, p.ldb) : nullptr;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t k0 = 0; k0 < p.ldb; k0 += 16) {
    const bool kin = (k0 + lk) < p.ldb;
    const float4 av = (arow && kin) ? *reinterpret_cast<const float4*>(arow + k0 + lk) : z4;
    const float4 bv = (brow && kin) ? *reinterpret_cast<const float4*>(brow + k0 + lk) : z4;
    As[lk + 0][lr] = av.x; As[lk + 1][lr] = av.y; As[lk + 2][lr] = av.z; As[lk + 3][lr] = av.w;
    Bs[lk + 0][lr] = bv.x; Bs[lk + 1][lr] = bv.y; Bs[lk + 2][lr] = bv.z; Bs[lk + 3][lr] = bv.w;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      T a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = As[k][ty * 4 + q]; b[q] = Bs[k][tx * 4 + q]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  T* G = static_cast<T*>(P.G);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = ti * 64 + ty * 4 + i, c = tj * 64 + tx * 4 + j;
      if (r < N && c < N) {
        G[(int64_t)r * p.ldg + c] = acc[i][j];
        G[(int64_t)c * p.ldg + r] = acc[i][j];
      }
    }
}

cudaError_t launch_gram(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s) {
  if (count <= 0 || nmax <= 0) return cudaSuccess;
  const int nt = (nmax + 63) / 64;
  dim3 grid(nt * (nt + 1) / 2, count);
  if (p.f64) gram_kernel<double><<<grid, 256, 0, s>>>(dev_probs, p);
  else gram_kernel<float><<<grid, 256, 0, s>>>(dev_probs, p);
  return cudaGetLastError();
}

// ============================================================================
// Reconstruct: dst[j] = sum_r Wt[j][r] Bf[r] (j < ell-1) accumulated in T,
// stored fp32; dst[ell-1] = 0.
// ============================================================================
template <typename T>
__global__ void __launch_bounds__(256) recon_kernel(const Prob* __restrict__ probs, Params p) {
  const Prob P = probs[blockIdx.z];
  const int N = P.rows0 + P.rows1;
  const int c0 = blockIdx.x * 64, j0 = blockIdx.y * 64;
  if (j0 >= p.ell) return;
  __shared__ __align__(16) T Ws[16][68];  // Ws[k][jj] = Wt[j0+jj][r0+k]
  __shared__ __align__(16) T Bs[16][68];  // Bs[k][cc] = Bf[r0+k][c0+cc]
  const T* Wt = static_cast<const T*>(P.Wt);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int wj = threadIdx.x >> 2, wk = (threadIdx.x & 3) * 4;    // Wt loader: 64 rows x 16
  const int bk = threadIdx.x >> 4, bc = (threadIdx.x & 15) * 4;   // Bf loader: 16 rows x 64
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const int jrow = j0 + wj;
  for (int r0 = 0; r0 < N; r0 += 16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = r0 + wk + q;
      Ws[wk + q][wj] = (jrow < p.ret && r < N) ? Wt[(int64_t)jrow * p.ldg + r] : T(0);
    }
    float4 bv = z4;
    const int r = r0 + bk;
    if (r < N && c0 + bc < p.ldb) bv = *reinterpret_cast<const float4*>(prob_row(P, r, p.ldb) + c0 + bc);
    Bs[bk][bc + 0] = bv.x; Bs[bk][bc + 1] = bv.y; Bs[bk][bc + 2] = bv.z; Bs[bk][bc + 3] = bv.w;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      T a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = Ws[k][ty * 4 + q]; b[q] = Bs[k][tx * 4 + q]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int j = j0 + ty * 4 + i;
    if (j >= p.ell) continue;
    const int c = c0 + tx * 4;
    if (c >= p.ldb) continue;
    float4 o = z4;
    if (j < p.ret) o = make_float4((float)acc[i][0], (float)acc[i][1], (float)acc[i][2], (float)acc[i][3]);
    *reinterpret_cast<float4*>(P.dst + (int64_t)j * p.ldb + c) = o;
  }
}

// cp.async helpers of the pipelined reconstruct
namespace {
__device__ __forceinline__ void cp_async16(float* dst, const float* src, int bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }
}  // namespace

// Default fp32 reconstruct: CTA tile 128 (j) x 256 (n), thread tile 16 x 8 (rows ty + 8 i,
// columns 4 lane + 128 h), 256 threads / 255 registers, one CTA per SM, 4-stage
// cp.async pipeline (BK = 32); A keeps its [j][k] layout in shared memory and is
// read as broadcast k-pairs, B rows as conflict-free float4 runs.
#ifndef FD_RC2_BK
#define FD_RC2_BK 32
#endif
#ifndef FD_RC2_STAGES
#define FD_RC2_STAGES 4
#endif
constexpr int kRc2BK = FD_RC2_BK, kRc2Stages = FD_RC2_STAGES, kRc2ALd = kRc2BK + 4;
constexpr int kRc2BLd = 256;
constexpr int kRc2StageFloats = 128 * kRc2ALd + kRc2BK * kRc2BLd;

__global__ void __launch_bounds__(256, 1) recon_pipe2_kernel(const Prob* __restrict__ probs, Params p) {
  const Prob P = probs[blockIdx.z];
  const int N = P.rows0 + P.rows1;
  const int n0 = blockIdx.x * 256, j0 = blockIdx.y * 128;
  const int jrows = p.ret;
  if (j0 >= p.ell) return;
  extern __shared__ __align__(16) float rsm[];
  const float* Wt = static_cast<const float*>(P.Wt);
  const int tid = threadIdx.x, lane = tid & 31, ty = tid >> 5;
  const int nk = (N + kRc2BK - 1) / kRc2BK;
  auto issue = [&](int kt) {
    float* As = rsm + (kt % kRc2Stages) * kRc2StageFloats;
    float* Bs = As + 128 * kRc2ALd;
    const int k0 = kt * kRc2BK;
    constexpr int kQ = kRc2BK / 4;            // 16-byte chunks per A row
#pragma unroll
    for (int h = 0; h < 128 * kQ / 256; ++h) {
      const int e = tid + 256 * h, m = e / kQ, kq = 4 * (e % kQ), k = k0 + kq, j = j0 + m;
      const int bytes = (j < jrows && k < N) ? 4 * min(4, N - k) : 0;
      const float* src = bytes ? Wt + (int64_t)j * p.ldg + k : Wt;
      cp_async16(As + m * kRc2ALd + kq, src, bytes);
    }
#pragma unroll
    for (int h = 0; h < kRc2BK / 4; ++h) {
      const int kr = (tid >> 6) + 4 * h, nq = 4 * (tid & 63), k = k0 + kr, n = n0 + nq;
      const bool ok = k < N && n < p.ldb;
      const float* src = ok ? prob_row(P, k, p.ldb) + n : Wt;
      cp_async16(Bs + kr * kRc2BLd + nq, src, ok ? 16 : 0);
    }
  };
  // column pairs (2q, 2q+1) of the thread tile: packed FFMA2 (fma.rn.f32x2) with the
  // A value as a broadcast scalar operand -- half the FMA instructions of FFMA, same
  // flops and the same rounding (one fma per element)
  float2 acc[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = make_float2(0.f, 0.f);
#pragma unroll
  for (int st = 0; st < kRc2Stages - 1; ++st) {
    if (st < nk) issue(st);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<kRc2Stages - 2>();
    __syncthreads();
    if (kt + kRc2Stages - 1 < nk) issue(kt + kRc2Stages - 1);
    cp_async_commit();
    const float* As = rsm + (kt % kRc2Stages) * kRc2StageFloats;
    const float* Bs = As + 128 * kRc2ALd;
#pragma unroll
    for (int kk = 0; kk < kRc2BK; kk += 2) {
      float2 a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = *reinterpret_cast<const float2*>(&As[(ty + 8 * i) * kRc2ALd + kk]);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float4 b0 = *reinterpret_cast<const float4*>(&Bs[(kk + u) * kRc2BLd + 4 * lane]);
        const float4 b1 = *reinterpret_cast<const float4*>(&Bs[(kk + u) * kRc2BLd + 128 + 4 * lane]);
        const float2 bb[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                              make_float2(b1.z, b1.w)};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float av = u ? a[i].y : a[i].x;
          const float2 a2 = make_float2(av, av);
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[i][q] = __ffma2_rn(a2, bb[q], acc[i][q]);
        }
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int j = j0 + ty + 8 * i;
    if (j >= p.ell) continue;
    float* dst = P.dst + (int64_t)j * p.ldb + n0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 128 * h + 4 * lane;
      if (n0 + c >= p.ldb) continue;
      const float4 o = (j < jrows) ? make_float4(acc[i][2 * h].x, acc[i][2 * h].y, acc[i][2 * h + 1].x, acc[i][2 * h + 1].y)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(dst + c) = o;
    }
  }
}

cudaError_t launch_recon(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  (void)nmax;
  if (!p.f64) {   // ldg and ldb are multiples of 4 by construction (fd_api.cpp derive)
    constexpr int dyn = kRc2Stages * kRc2StageFloats * (int)sizeof(float);
    static AttrOnce once;
    if (cudaError_t e = once.ensure(recon_pipe2_kernel, dyn); e != cudaSuccess) return e;
    dim3 grid((unsigned)((p.ldb + 255) / 256), (unsigned)((p.ell + 127) / 128), count);
    recon_pipe2_kernel<<<grid, 256, dyn, s>>>(dev_probs, p);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((p.ldb + 63) / 64), (unsigned)((p.ell + 63) / 64), count);
  recon_kernel<double><<<grid, 256, 0, s>>>(dev_probs, p);
  return cudaGetLastError();
}

// ============================================================================
// Eigen-solver + ReduceRank rule (one CTA per problem, persistent over
// problems), precision T, max size NM.
// ============================================================================
constexpr int kNW = kEigThreads / 32;  // 16 warps
#ifndef FD_EIG_CTAS
#define FD_EIG_CTAS 3
#endif
constexpr int kEigPreCtasPerSM = FD_EIG_CTAS;     // resident CTAs of the lean (tridiagonal-input) variant
constexpr int kPreZst = 132;          // lean variant: fp32 inverse-iteration scratch stride (>= 129 vectors)
constexpr int kSmallCl = 8;             // clusters up to this size: warp MGS; larger: block CGS2
#ifndef FD_INV_ITERS
#define FD_INV_ITERS 2
#endif
constexpr int kInvIters = FD_INV_ITERS;
#ifndef FD_BISECT_LOOSE
#define FD_BISECT_LOOSE 1
#endif
#ifndef FD_INV_F32
#define FD_INV_F32 1
#endif
#ifndef FD_EIG_DISCARD
#define FD_EIG_DISCARD 1
#endif
#ifndef FD_SOLVE_BATCH
#define FD_SOLVE_BATCH 4
#endif
constexpr int kSB = FD_SOLVE_BATCH;   // rows per load batch of the twisted solves  // inverse-iteration sweeps (2: same parity as 3)

// fp64 reciprocal: fp32 estimate + two Newton steps (each squares the ~6e-8
// relative error of the estimate), cheaper than the IEEE division.
__device__ __forceinline__ float rcp_rt(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_d(double x) {
  if (!(fabs(x) > 1e-30 && fabs(x) < 1e30)) return 1.0 / x;   // outside the fp32 estimate's range
  double r = (double)__frcp_rn((float)x);
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}
__device__ __forceinline__ double rcp_rt(double x) { return rcp_d(x); }
// fp64 scratch per CTA slot (stride zld): LDL^T factors and Z (element-major
// [i][j], zld x zld each), a Rayleigh-Ritz copy region, then, for problems above
// kMaxNS, the packed matrix (global / L2 instead of shared memory).
__host__ __device__ inline size_t slot_doubles(int zld) {
  return (size_t)4 * zld * zld + (zld > kMaxNS ? ((size_t)zld * (zld + 1) / 2 + 1) / 2 : 0);
}

size_t eig_scratch_bytes(int zld) {
  return (size_t)kNumSMs * kEigPreCtasPerSM * slot_doubles(zld) * sizeof(double);
}

template <typename T, int NM, bool GAPK, bool PRE = false>
struct EigCfg {
  static_assert(NM % 32 == 0, "NM must be a multiple of 32");
  // packed matrix in smem unless GAPK (global) or PRE (tridiagonal form precomputed by
  // trd_kernel: neither the packed matrix nor the Householder workspaces are needed)
  static constexpr int kPk = (GAPK || PRE) ? 0 : NM * (NM + 1) / 2;
  static constexpr int kPart = PRE ? 0 : kNW * NM + 32 * (NM + 1);  // ppart[16][NM] + colpart[32][NM+1]
  static constexpr int kVec = 13;                 // vector arrays of NM
  static constexpr size_t kT = (size_t)kPk + kPart + kVec * NM + 64;  // elements of T
  // block-CGS scratch (cpart [warps][NM+1] + chq [NM], doubles): aliases the Householder
  // workspaces (ppart / colpart, idle during the eigenvectors) unless PRE has none
  static constexpr int kNWc = (PRE ? 256 : kEigThreads) / 32;
  static constexpr size_t kCgs = (size_t)(kNWc * (NM + 1) + NM) * sizeof(double);
  static_assert(PRE || (size_t)kPart * sizeof(T) >= kCgs, "CGS scratch must fit the SYMV workspaces");
  static constexpr size_t kBytes = kT * sizeof(T) + (4 * NM + kNWc * 32) * sizeof(int) + 2 * NM * sizeof(double) + 16 +
                                   (PRE ? kCgs : 0);
};

__device__ __forceinline__ int pk_off(int c, int N) { return c * N - (c * (c - 1)) / 2; }

template <typename T>
__device__ __forceinline__ T wsum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = wsum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T s = T(0);
#pragma unroll
  for (int w = 0; w < kNW; ++w) s += red[w];
  __syncthreads();
  return s;
}

__device__ __forceinline__ float fast_div(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double fast_div(double a, double b) { return a / b; }

// number of eigenvalues of the tridiagonal (d, e2) strictly less than x
// (Sturm count with the LAPACK xSTEBZ pivot guard)
template <typename T>
__device__ __forceinline__ int sturm_count(const T* __restrict__ dd, const T* __restrict__ e2, int N, T x, T pivmin) {
  T q = dd[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  int cnt = q < T(0);
#pragma unroll 4
  for (int i = 1; i < N; ++i) {
    q = (dd[i] - x) - fast_div(e2[i - 1], q);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < T(0);
  }
  return cnt;
}

template <typename T> struct Lim;
template <> struct Lim<float> {
  static __device__ float eps() { return FLT_EPSILON; }
  static __device__ float tiny() { return FLT_MIN; }
  static __device__ float big() { return FLT_MAX; }
  static constexpr float bits = 27.f;
  static constexpr float btol = 4e-9f;    // bisection: absolute width / (gu - gl)
  static constexpr float gspan = 30.f;    // coarse geometric points down to gu 2^-gspan
  using V2 = float2;
};
template <> struct Lim<double> {
  static __device__ double eps() { return DBL_EPSILON; }
  static __device__ double tiny() { return DBL_MIN; }
  static __device__ double big() { return DBL_MAX; }
  static constexpr float bits = 56.f;
  static constexpr double btol = 1e-17;
  static constexpr double gspan = 60.0;
  using V2 = double2;
};

// Sturm counts (number of eigenvalues < x) of the tridiagonal packed as
// de[i] = (d_i, e_{i-1}^2): one point, or two interleaved points sharing the loads.
template <typename T, typename V2>
__device__ __forceinline__ int sturm1(const V2* __restrict__ de, int N, T x, T pivmin) {
  T q = de[0].x - x;
  if (fabs(q) < pivmin) q = -pivmin;
  int cnt = q < T(0);
#pragma unroll 4
  for (int i = 1; i < N; ++i) {
    const V2 v = de[i];
    q = (v.x - x) - fast_div(v.y, q);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < T(0);
  }
  return cnt;
}
template <typename T, typename V2>
__device__ __forceinline__ void sturm2(const V2* __restrict__ de, int N, T x0, T x1, T pivmin, int& c0, int& c1) {
  T q0 = de[0].x - x0, q1 = de[0].x - x1;
  if (fabs(q0) < pivmin) q0 = -pivmin;
  if (fabs(q1) < pivmin) q1 = -pivmin;
  int n0 = q0 < T(0), n1 = q1 < T(0);
#pragma unroll 4
  for (int i = 1; i < N; ++i) {
    const V2 v = de[i];
    q0 = (v.x - x0) - fast_div(v.y, q0);
    q1 = (v.x - x1) - fast_div(v.y, q1);
    if (fabs(q0) < pivmin) q0 = -pivmin;
    if (fabs(q1) < pivmin) q1 = -pivmin;
    n0 += q0 < T(0);
    n1 += q1 < T(0);
  }
  c0 = n0;
  c1 = n1;
}

// coarse bisection points: family 0 linear over (gl, gu), family 1 geometric below gu
template <typename T>
__device__ __forceinline__ T coarse_pt(int t, int fam, int H, T gl, T gu) {
  if (fam == 0) return gl + (gu - gl) * (T)(t + 1) / (T)(H + 1);
  return gu * (T)exp2((double)(-Lim<T>::gspan * (double)(H - t) / (double)H));
}

// PRE = true: the lean variant for the tridiagonal-kernel path (p.pretrd): 256
// threads, small shared memory, several CTAs (problems) per SM.
// Large clusters (> kSmallCl members) of the inverse iteration: panels of 8 members,
// block Gram-Schmidt twice against the earlier members + warp MGS inside the panel (see
// the call site).  Out of line so its registers do not perturb the solver loop's.
template <int NM, int kNT, typename ZT>
__device__
#ifdef FD_PANEL_INLINE
__forceinline__
#else
__noinline__
#endif
void panel_cgs(ZT* __restrict__ Zs, int kMaxN, double* __restrict__ pscl,
                                       double* __restrict__ cpart, const int* __restrict__ cstart,
                                       const int* __restrict__ clen, int ncl, int N) {
  constexpr int kNW = kNT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int c = 0; c < ncl; ++c) {
      const int j0 = cstart[c], nc = clen[c];
      if (nc <= kSmallCl) continue;
      const int rpw = (N + kNW - 1) / kNW;   // rows per warp (<= 32 for every instantiation)
      double* cp = cpart;                    // [kNW][32][8] partial dots
      double* hq = cpart + kNW * 256;        // [32][8] projection coefficients
      for (int p0 = j0; p0 < j0 + nc; p0 += 8) {
        const int pb = min(8, j0 + nc - p0);
        __syncthreads();   // previous panel finished; pscl stable
        for (int i = tid; i < N; i += kNT)
          for (int m = 0; m < pb; ++m) Zs[(size_t)i * kMaxN + p0 + m] *= pscl[p0 + m];
        __syncthreads();
        const int kq = p0 - j0;
        for (int pass = 0; pass < 2 && kq > 0; ++pass) {
          for (int q0 = 0; q0 < kq; q0 += 32) {
            const int nq = min(32, kq - q0);
            {
              const int ia = warp * rpw, ir = ia + lane;
              const int q = j0 + q0 + lane;
              for (int mh = 0; mh < 8; mh += 4) {   // half a panel at a time (register pressure)
                double pv[4];
#pragma unroll
                for (int m = 0; m < 4; ++m)
                  pv[m] = (lane < rpw && ir < N && mh + m < pb) ? Zs[(size_t)ir * kMaxN + p0 + mh + m] : 0.0;
                double h[4] = {0.0, 0.0, 0.0, 0.0};
                for (int r = 0; r < rpw; r += 4) {
                  double zq[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u) {
                    const int i = ia + r + u;
                    zq[u] = (r + u < rpw && i < N && lane < nq) ? Zs[(size_t)i * kMaxN + q] : 0.0;
                  }
#pragma unroll
                  for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                      h[m] = fma(zq[u], __shfl_sync(0xffffffffu, pv[m], (r + u) & 31), h[m]);
                }
#pragma unroll
                for (int m = 0; m < 4; ++m) cp[(warp * 32 + lane) * 8 + mh + m] = h[m];
              }
            }
            __syncthreads();
            if (tid < 256) {
              double sum = 0.0;
              for (int w = 0; w < kNW; ++w) sum += cp[w * 256 + tid];
              hq[tid] = sum;
            }
            __syncthreads();
            for (int i = tid; i < N; i += kNT) {
              ZT* zi = Zs + (size_t)i * kMaxN;
              double z[8];
#pragma unroll
              for (int m = 0; m < 8; ++m) z[m] = (m < pb) ? zi[p0 + m] : 0.0;
              int l = 0;
              for (; l + 4 <= nq; l += 4) {
                double zl[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) zl[u] = zi[j0 + q0 + l + u];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                  for (int m = 0; m < 8; ++m) z[m] = fma(-hq[(l + u) * 8 + m], zl[u], z[m]);
              }
              for (; l < nq; ++l) {
                const double zl = zi[j0 + q0 + l];
#pragma unroll
                for (int m = 0; m < 8; ++m) z[m] = fma(-hq[l * 8 + m], zl, z[m]);
              }
#pragma unroll
              for (int m = 0; m < 8; ++m)
                if (m < pb) zi[p0 + m] = z[m];
            }
            __syncthreads();
          }
        }
        if (warp == 0) {   // the panel itself: MGS twice, normalise (registers)
          for (int k = p0; k < p0 + pb; ++k) {
            ZT* zk = Zs + k;
            double zr[NM / 32];
#pragma unroll
            for (int t = 0; t < NM / 32; ++t) {
              const int i = 32 * t + lane;
              zr[t] = (i < N) ? zk[(size_t)i * kMaxN] : 0.0;
            }
            for (int pass = 0; pass < 2; ++pass)
              for (int q = p0; q < k; ++q) {
                const ZT* zq = Zs + q;
                double zqr[NM / 32];
                double hh = 0.0;
#pragma unroll
                for (int t = 0; t < NM / 32; ++t) {
                  const int i = 32 * t + lane;
                  zqr[t] = (i < N) ? zq[(size_t)i * kMaxN] : 0.0;
                  hh = fma(zqr[t], zr[t], hh);
                }
                hh = warp_sum_d(hh);
#pragma unroll
                for (int t = 0; t < NM / 32; ++t) zr[t] = fma(-hh, zqr[t], zr[t]);
              }
            double n2 = 0.0;
#pragma unroll
            for (int t = 0; t < NM / 32; ++t) n2 = fma(zr[t], zr[t], n2);
            n2 = warp_sum_d(n2);
            const double inv = (n2 > 0.0) ? 1.0 / sqrt(n2) : 0.0;
#pragma unroll
            for (int t = 0; t < NM / 32; ++t) {
              const int i = 32 * t + lane;
              if (i < N) zk[(size_t)i * kMaxN] = zr[t] * inv;
            }
            __syncwarp();
          }
        }
        __syncthreads();
        if (tid < pb) pscl[p0 + tid] = 1.0;
      }
    }
    
}

template <typename T, int NM, bool GAPK, bool PRE = false, bool BIG = false>
__global__ void __launch_bounds__(PRE ? 256 : kEigThreads, PRE ? kEigPreCtasPerSM : 1)
eig_kernel(const Prob* __restrict__ probs, int count, Params p, double* __restrict__ scratch) {
  using C = EigCfg<T, NM, GAPK, PRE>;
  constexpr int kNT = PRE ? 256 : kEigThreads;   // threads
  constexpr int kNW = kNT / 32;                  // warps
  constexpr int kCpStride = NM + 1;
  constexpr int NT = NM / 32;   // row blocks (lane <-> row 32t + lane)
  constexpr int NK = NM / kNW;  // columns per warp (warp <-> column warp + 16k)
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const int kMaxN = p.zld;        // scratch stride (runtime)
  double* slot = scratch + (size_t)blockIdx.x * slot_doubles(kMaxN);   // one slot per resident CTA
  T* Apk = GAPK ? reinterpret_cast<T*>(slot + (size_t)4 * kMaxN * kMaxN) : sm;
  T* ppart = sm + C::kPk;         // [kNW][NM]  per-warp row partials of the SYMV
  T* colpart = ppart + kNW * NM;  // [32][NM+1] per-lane column partials (padded: no bank conflicts)
  T* vbuf0 = sm + C::kPk + C::kPart;    // v / w of the current and previous Householder step
  T* wbuf0 = vbuf0 + NM;
  T* vbuf1 = wbuf0 + NM;
  T* wbuf1 = vbuf1 + NM;
  T* dd = wbuf1 + NM;
  T* ee = dd + NM;
  T* e2 = ee + NM;
  T* tau = e2 + NM;
  T* lam = tau + NM;
  T* wgt = lam + NM;
  T* spv = wgt + NM;
  T* pvec = spv + NM;   // per-vector normalisation scale of the inverse iteration
  T* red = pvec + 2 * NM;
  int* cstart = reinterpret_cast<int*>(red + 64);
  int* clen = cstart + NM;
  int* cid = clen + NM;                       // Rayleigh-Ritz cluster list
  int* ord = cid + NM;                        // Ritz-vector order
  int* ccnt = ord + NM;                       // [kNT] coarse bisection counts
  constexpr size_t kOffD = C::kT * sizeof(T) + (4 * NM + kNT) * sizeof(int);
  double* pscl = reinterpret_cast<double*>(smraw + kOffD + 8 - (kOffD & 7));  // per-vector scale (fp64)
  double* lamd = pscl + NM;   // fp64 shifts of the inverse iteration (refined inside large clusters)
  double* cpart = PRE ? pscl + 2 * NM : reinterpret_cast<double*>(ppart);  // [kNW][kCpStride] block-CGS dots
  __shared__ int s_ncl, s_jx, s_nrr;
  __shared__ T s_gl, s_gu, s_a1, s_a2;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // element-major (coalesced across threads): LF[i][j] (multipliers), Zs[i][j] (vectors),
  // row stride zst.  The lean variant stores them in fp32 with stride kPreZst (its <= 129
  // vectors): 444 resident slots x 2 x 256 x 132 x 4 B = 120 MB stay in L2, where the fp64
  // full-stride layout (2 MB per slot) streamed from HBM (round-1 ncu: 18x the algorithmic
  // bytes).  The recurrences themselves run in fp64 registers; the Gram (3xTF32) and the
  // tridiagonal form (fp32) already carry errors far above fp32 rounding of the vectors.
  using ZT = typename std::conditional<PRE, float, double>::type;
  const int zst = PRE ? kPreZst : kMaxN;
  ZT* LF = reinterpret_cast<ZT*>(slot);
  ZT* Zs = reinterpret_cast<ZT*>(slot + (size_t)kMaxN * kMaxN);
  double* RD = slot + (size_t)2 * kMaxN * kMaxN;

  for (int pi = blockIdx.x; pi < count; pi += gridDim.x) {
    const Prob P = probs[pi];
    const int N = P.rows0 + P.rows1;
    const int ell = p.ell;
    long long t_ph0 = clock64();
    const T* G = static_cast<const T*>(P.G);
    T* Wt = static_cast<T*>(P.Wt);
    if (PRE || p.pretrd) {
      // ---------------- tridiagonal form from trd_kernel (fd_trd.cu) ----------------
      // packed Householder vectors, then d / e / tau at round_up(N(N+1)/2, 4)
      const float* V = reinterpret_cast<const float*>(P.G);
      const int npk = N * (N + 1) / 2;
      const int offd = (npk + 3) / 4 * 4;
      (void)npk;  // the reflectors stay in global memory for bt_kernel (fd_bt.cu)
      for (int r = tid; r < N; r += blockDim.x) {
        dd[r] = (T)V[offd + r];
        ee[r] = (T)V[offd + N + r];
        tau[r] = (T)V[offd + 2 * N + r];
      }
      __syncthreads();
      if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[1] += t_ - t_ph0; t_ph0 = t_; }
    } else if constexpr (!PRE) {
    // ---------------- load lower triangle (packed, column-major) ----------------
    for (int c = warp; c < N; c += kNW) {
      const int oc = pk_off(c, N);
      for (int r = c + lane; r < N; r += 32) Apk[oc + r - c] = G[(int64_t)r * p.ldg + c];
    }
    for (int r = tid; r < NM; r += blockDim.x) { vbuf1[r] = T(0); wbuf1[r] = T(0); }
    __syncthreads();
    if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[1] += t_ - t_ph0; t_ph0 = t_; }
    // ---------------- Householder tridiagonalisation (lower, xSYTD2 order) ----------------
    // One fused shared-memory pass per step: the pending rank-2 update of step i-1
    // is applied while the SYMV of step i is accumulated from the pre-update values;
    // p = A^(i) v is then recovered exactly with the rank-2 correction
    //   A^(i) v = A^(i-1) v - v_{i-1} (w_{i-1}^T v) - w_{i-1} (v_{i-1}^T v).
    T* vc = vbuf0; T* wc = wbuf0;   // step i
    T* vp = vbuf1; T* wp = wbuf1;   // step i-1 (zero before the first step)
    for (int i = 0; i < N - 2; ++i) {
      const int oi = pk_off(i, N);
      // (a) warp 0: apply update i-1 to column i, build the reflector of column i
      if (warp == 0) {
        const T vpi = vp[i], wpi = wp[i];
        T sig = T(0);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int R = 32 * t + lane;
          if (R >= i && R < N) {
            T a = Apk[oi + R - i];
            a = fma(-vp[R], wpi, a);
            a = fma(-wp[R], vpi, a);
            Apk[oi + R - i] = a;
            if (R >= i + 2) sig = fma(a, a, sig);
          }
        }
        sig = wsum(sig);
        __syncwarp();
        const T alpha = Apk[oi + 1];
        T t_, beta, scale;
        if (sig == T(0)) {
          t_ = T(0); beta = alpha; scale = T(0);
        } else {
          const T nrm = sqrt(fma(alpha, alpha, sig));
          beta = (alpha <= T(0)) ? nrm : -nrm;
          t_ = (beta - alpha) / beta;
          scale = T(1) / (alpha - beta);
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int R = 32 * t + lane;
          T v = T(0);
          if (R == i + 1) v = T(1);
          else if (R >= i + 2 && R < N) {
            v = Apk[oi + R - i] * scale;
            Apk[oi + R - i] = v;
          }
          vc[R] = v;
        }
        if (lane == 0) { tau[i] = t_; dd[i] = Apk[oi]; ee[i] = beta; }
      }
      __syncthreads();
      const T t_ = tau[i];
      // (b) fused pass over the trailing matrix (columns >= i+1)
      T racc[NT];
      T vr[NT], vpr[NT], wpr[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        racc[t] = T(0);
        vr[t] = vc[32 * t + lane];
        vpr[t] = vp[32 * t + lane];
        wpr[t] = wp[32 * t + lane];
      }
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const int Cc = warp + kNW * k;
        if (Cc <= i || Cc >= N) continue;  // warp-uniform
        const int base = pk_off(Cc, N) - Cc;
        const T vcc = vc[Cc], vpc = vp[Cc], wpc = wp[Cc];
        // all loads of the column first (no store->load ordering stalls), then compute, then store
        T a[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int R = 32 * t + lane;
          a[t] = (32 * t + 31 >= Cc && R >= Cc && R < N) ? Apk[base + R] : T(0);
        }
        T csum = T(0);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int R = 32 * t + lane;
          racc[t] = fma(a[t], vcc, racc[t]);
          if (R > Cc) csum = fma(a[t], vr[t], csum);
          a[t] = fma(-vpr[t], wpc, a[t]);
          a[t] = fma(-wpr[t], vpc, a[t]);
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (32 * t + 31 < Cc) continue;  // warp-uniform
          const int R = 32 * t + lane;
          if (R >= Cc && R < N) Apk[base + R] = a[t];
        }
        colpart[lane * (NM + 1) + Cc] = csum;
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) ppart[warp * NM + 32 * t + lane] = racc[t];
      __syncthreads();
      // (c) raw = A^(i-1) v (partials), a1 = w_{i-1}.v, a2 = v_{i-1}.v, S0 = raw.v in ONE block
      //     reduction; p = tau (raw - v_{i-1} a1 - w_{i-1} a2), K = p.v = tau (S0 - 2 a1 a2),
      //     w = p - tau/2 K v.
      T raw = T(0), vR = T(0), vpR = T(0), wpR = T(0);
      if (tid > i && tid < N) {
#pragma unroll
        for (int w2 = 0; w2 < kNW; ++w2) raw += ppart[w2 * NM + tid];
#pragma unroll 8
        for (int l = 0; l < 32; ++l) raw += colpart[l * (NM + 1) + tid];
        vR = vc[tid]; vpR = vp[tid]; wpR = wp[tid];
      }
      T r3[3] = {raw * vR, wpR * vR, vpR * vR};
#pragma unroll
      for (int q = 0; q < 3; ++q) r3[q] = wsum(r3[q]);
      if (lane == 0) { red[warp] = r3[0]; red[16 + warp] = r3[1]; red[32 + warp] = r3[2]; }
      __syncthreads();
      T S0 = T(0), a1 = T(0), a2 = T(0);
#pragma unroll
      for (int w2 = 0; w2 < kNW; ++w2) { S0 += red[w2]; a1 += red[16 + w2]; a2 += red[32 + w2]; }
      const T K = t_ * (S0 - T(2) * a1 * a2);
      if (tid < NM) {
        T wv = T(0);
        if (tid > i && tid < N) {
          const T pr = t_ * (raw - vpR * a1 - wpR * a2);
          wv = fma(T(-0.5) * t_ * K, vR, pr);
        }
        wc[tid] = wv;
      }
      __syncthreads();
      // rotate step buffers
      T* tv = vp; vp = vc; vc = tv;
      T* tw = wp; wp = wc; wc = tw;
    }
    // pending update of the last step on the trailing 2 x 2 block, then the last entries
    if (tid == 0) {
      if (N >= 2) {
        const int a = N - 2, b = N - 1;
        const int oa = pk_off(a, N), ob = pk_off(b, N);
        T aa = Apk[oa], ba = Apk[oa + 1], bb = Apk[ob];
        aa -= T(2) * vp[a] * wp[a];
        ba -= vp[b] * wp[a] + wp[b] * vp[a];
        bb -= T(2) * vp[b] * wp[b];
        dd[a] = aa; ee[a] = ba; dd[b] = bb; tau[a] = T(0);
      } else if (N == 1) {
        dd[0] = Apk[0];
      }
      if (N >= 1) { ee[N - 1] = T(0); tau[N - 1] = T(0); }
    }
    __syncthreads();
    }  // !p.pretrd
    if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[2] += t_ - t_ph0; t_ph0 = t_; }
    // ---------------- eigenvalues: multisection bisection ----------------
    const int K = min(max(p.tdel, p.ret), N);   // top-K eigenvalues needed (lambda_tdel = delta)
    const int J = min(p.ret, N);                // retained eigenvectors
    // iSVD's weights jump between J-1 (kept) and J (dropped): a cluster straddling
    // that boundary needs its members beyond J, so a margin of eigenvalues is found
    // (and any rule whose weights drop from unchanged to 0 at J: alpha-FD with m = 1,
    // the paper-literal Fast alpha-FD when ell - m >= R)
    const int KC = (p.rule == RULE_ISVD || ell - p.m >= p.ret) ? min(N, max(K, J) + 16) : K;
    T glo = Lim<T>::big(), ghi = -Lim<T>::big(), emax2 = T(0);
    for (int i = tid; i < N; i += blockDim.x) {
      const T em = (i > 0) ? fabs(ee[i - 1]) : T(0);
      const T ep = (i < N - 1) ? fabs(ee[i]) : T(0);
      glo = fmin(glo, dd[i] - em - ep);
      ghi = fmax(ghi, dd[i] + em + ep);
      e2[i] = (i < N - 1) ? ee[i] * ee[i] : T(0);
      emax2 = fmax(emax2, e2[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      glo = fmin(glo, __shfl_xor_sync(0xffffffffu, glo, o));
      ghi = fmax(ghi, __shfl_xor_sync(0xffffffffu, ghi, o));
      emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
    }
    if (lane == 0) { red[warp] = glo; red[16 + warp] = ghi; red[32 + warp] = emax2; }
    __syncthreads();
    if (tid == 0) {
      T a = Lim<T>::big(), b = -Lim<T>::big(), e = T(0);
      for (int w = 0; w < kNW; ++w) { a = fmin(a, red[w]); b = fmax(b, red[16 + w]); e = fmax(e, red[32 + w]); }
      const T bn = fmax(fabs(a), fabs(b));
      const T slack = T(2) * Lim<T>::eps() * bn * (T)N + Lim<T>::tiny();
      s_gl = a - slack; s_gu = b + slack;
      red[48] = fmax(Lim<T>::tiny(), Lim<T>::tiny() * e);   // pivmin
      red[49] = bn;
    }
    __syncthreads();
    const T pivmin = red[48];
    const T bnorm = red[49];
    if (N > 0) {
      using V2 = typename Lim<T>::V2;
      V2* de = reinterpret_cast<V2*>(vbuf0);   // (d_i, e_{i-1}^2): Householder buffers are idle here
      for (int i = tid; i < N; i += kNT) {
        V2 v;
        v.x = dd[i];
        v.y = (i > 0) ? e2[i - 1] : T(0);
        de[i] = v;
      }
      __syncthreads();
      // coarse pass: one Sturm count per thread, kNT/2 linear and kNT/2 geometric points
      constexpr int H = kNT / 2;
      const T gl = s_gl, gu = s_gu;
      ccnt[tid] = sturm1<T, V2>(de, N, coarse_pt<T>(tid % H, tid / H, H, gl, gu), pivmin);
      __syncthreads();
      int kp = 1;
      while (kp < KC) kp <<= 1;
      int g = kNT / kp;  // threads per eigenvalue (power of two), 2 points each
      if (g > 32) g = 32;
      if (g < 1) g = 1;
      const int j = tid / g, sub = tid % g;
      const unsigned gmask = (g == 32) ? 0xffffffffu : (((1u << g) - 1u) << ((lane / g) * g));
      const int base = (lane / g) * g;
      T lo = gl, hi = gu;
      if (j < KC) {  // initial bracket from the coarse counts (non-decreasing in each family)
        const int target = N - j;   // lambda_j (descending index j) is the target-th smallest
        for (int fam = 0; fam < 2; ++fam) {
          int a0 = -1, b0 = H;
          while (b0 - a0 > 1) {
            const int mid = (a0 + b0) >> 1;
            if (ccnt[fam * H + mid] >= target) b0 = mid; else a0 = mid;
          }
          if (a0 >= 0) lo = fmax(lo, coarse_pt<T>(a0, fam, H, gl, gu));
          if (b0 < H) hi = fmin(hi, coarse_pt<T>(b0, fam, H, gl, gu));
        }
        hi = fmax(hi, lo);
      }
      // stream rounds of the lean variant: eigenvalues to ~eps32 ||T|| absolute (the fp32
      // tridiagonalisation's own backward error; FD_BISECT_LOOSE); merges (eigenvalue
      // ranges of 1e5-1e6) and the other variants keep the tight absolute width
      const T tol = (gu - gl) * ((PRE && FD_BISECT_LOOSE && !p.merge && sizeof(T) == 4) ? (T)6e-8f : (T)Lim<T>::btol);
      const int P = 2 * g;
      for (int it = 0; it < 96; ++it) {
        // converged: absolute width tol, or a few ulps of the endpoints (fp resolution)
        const bool need = (j < KC) && (hi - lo > fmax(tol, T(4) * Lim<T>::eps() * fmax(fabs(lo), fabs(hi))));
        if (!__syncthreads_or(need)) break;
        const T step = (hi - lo) / (T)(P + 1);
        int c0 = 0, c1 = 0;
        if (need) sturm2<T, V2>(de, N, lo + step * (T)(sub + 1), lo + step * (T)(sub + g + 1), pivmin, c0, c1);
        const unsigned m0 = __ballot_sync(0xffffffffu, need && c0 >= N - j) & gmask;
        const unsigned m1 = __ballot_sync(0xffffffffu, need && c1 >= N - j) & gmask;
        int ss = P;   // first point at or above lambda_j (points 0..g-1 = x0 of sub, g..2g-1 = x1)
        if (m0) ss = __ffs(m0) - 1 - base;
        else if (m1) ss = __ffs(m1) - 1 - base + g;
        if (need) {
          const T nlo = (ss == 0) ? lo : lo + step * (T)ss;
          const T nhi = (ss == P) ? hi : lo + step * (T)(ss + 1);
          lo = nlo;
          hi = fmax(nhi, nlo);
        }
      }
      if (sub == 0 && j < KC) lam[j] = fmax(T(0.5) * (lo + hi), T(0));  // clamp (reading C8)
    }
    __syncthreads();
    if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[3] += t_ - t_ph0; t_ph0 = t_; }
    // ---------------- ReduceRank rule ----------------
    // s_a1 = delta; s_a2 = 1 when ReduceRank-SS moves sigma_{ell-1}^2;
    // red[50] = Delta after this step (Compensative FD final step)
    if (tid == 0) {
      T dl = (p.tdel <= N) ? lam[p.tdel - 1] : T(0);
      T moved = T(0);
      if (p.rule == RULE_SS) {
        // delta = sigma_{ell-1}^2; the direction of sigma_ell (position ell-1) takes it
        // and is kept in output row ell-2 (swap, so the kept set stays 0..ell-2).
        // Reading C26: sigma_ell = 0 (buffer rank <= ell-1) -> lossless, nothing moves.
        const T tol = (sizeof(T) == 8) ? T(1e-12) : T(1e-5);
        dl = T(0);
        if (ell <= N && lam[ell - 1] > tol * lam[0]) {
          dl = lam[ell - 2];
          const T x = lam[ell - 2];
          lam[ell - 2] = lam[ell - 1];
          lam[ell - 1] = x;
          moved = T(1);
        }
      }
      s_a1 = dl;
      s_a2 = moved;
      if (p.comp) {
        double dt = (double)dl;
        if (P.stats) dt += P.child0 ? (P.child0->delta + P.child1->delta) : P.stats->delta;
        red[50] = (T)dt;
      }
    }
    __syncthreads();
    const T delta = s_a1;
    if (tid < J) {
      const T l = lam[tid];
      T sp2;
      if (p.rule == RULE_SS) sp2 = (s_a2 != T(0) && tid == ell - 2) ? l + delta : l;
      else if (p.rule == RULE_ISVD || tid < ell - p.m) sp2 = l;
      else sp2 = fmax(l - delta, T(0));
      if (p.comp && l > T(0)) sp2 += red[50];   // reading C27: sigma_j = 0 gets nothing
      spv[tid] = sp2;
      wgt[tid] = (l > T(0)) ? sqrt(sp2 / l) : T(0);
    }
    for (int j = J + tid; j < KC; j += blockDim.x) wgt[j] = T(0);
    __syncthreads();
    if (tid == 0) {
      double tr = 0.0, sp = 0.0;
      for (int i = 0; i < N; ++i) tr += (double)dd[i];
      for (int j = 0; j < J; ++j) sp += (double)spv[j];
      if (P.stats) {
        Stats st;
        if (P.child0) {
          const Stats a = *P.child0, b = *P.child1;
          st.frob = a.frob + b.frob; st.delta = a.delta + b.delta;
          st.removed = a.removed + b.removed; st.shrinks = a.shrinks + b.shrinks;
        } else {
          st = *P.stats;
        }
        st.delta += (double)delta;
        st.removed += tr - sp;
        st.shrinks += 1.0;
        *P.stats = st;
      }
      // Clusters of close eigenvalues among 0..KC-1 (consecutive gaps <= ctol).
      // Members of a cluster are computed together and orthonormalised.  Only the
      // clusters that contain a retained vector (< J) are kept; JX = end of the
      // last one.  A cluster is marked for Rayleigh-Ritz when the rule's weight is
      // discontinuous inside it (alpha-FD boundary ell-m, iSVD boundary J).
      const T ctol = T(1e-5) * bnorm;
      const int bnd = (p.rule == RULE_ISVD) ? J : ((p.m < ell) ? ell - p.m : -1);
      int ncl = 0, jx = 0;
      for (int j = 0; j < KC; ++j) {
        const bool cont = (j > 0) && (lam[j - 1] - lam[j] <= ctol);
        if (!cont) {
          if (j >= J) break;
          cstart[ncl] = j; clen[ncl] = 0; ++ncl;
        }
        clen[ncl - 1]++;
        jx = j + 1;
      }
      int nrr = 0;
      for (int c = 0; c < ncl; ++c) {
        const int a = cstart[c], b = cstart[c] + clen[c];
        if (bnd > a && bnd < b) cid[nrr++] = c;   // Rayleigh-Ritz list
      }
      s_ncl = ncl; s_jx = jx; s_nrr = nrr;
    }
    __syncthreads();
    // fp64 shifts.  The fp32 Sturm counts resolve an eigenvalue only to ~eps32 ||T||, hence
    // ctol; when ||T|| is dominated by a few large eigenvalues (merged sketches, the
    // c3 pixel data's mean direction) the whole noise band falls inside ctol and the
    // clusters reach 100+ members, whose block Gram-Schmidt dominates the solve.  Members
    // of clusters larger than kSmallCl are re-bisected with fp64 Sturm counts inside
    // lambda_j +- 2 ctol to ~1e-13 ||T|| and the clusters are rebuilt at 1e-10 ||T||
    // (inverse-iteration vectors are accurate to ~(shift error) / gap).
    for (int j = tid; j < s_jx; j += blockDim.x) lamd[j] = (double)lam[j];
#ifndef FD_NO_REFINE
    if constexpr (sizeof(T) == 4) {
      bool big = false;
      for (int c = 0; c < s_ncl; ++c) big |= clen[c] > kSmallCl;
      if (big) {
        // members of the large clusters -> ccnt[0..nbig) (the coarse counts are dead here)
        __shared__ int s_nbig;
        if (tid == 0) {
          int nb = 0;
          for (int c = 0; c < s_ncl; ++c)
            if (clen[c] > kSmallCl)
              for (int j = cstart[c]; j < cstart[c] + clen[c]; ++j) ccnt[nb++] = j;
          s_nbig = nb;
        }
        __syncthreads();
        const int nbig = s_nbig;
        // multisection: g threads per member (aligned lane groups), 2 interleaved points
        // each -> 2g + 1 sub-intervals per step, counts exchanged by ballot
        int g = 1;
        while (g < 8 && 2 * g * nbig <= (int)blockDim.x) g <<= 1;
        const int mi = tid / g, sub = tid % g;
        const unsigned gmask = (g == 32) ? 0xffffffffu : (((1u << g) - 1u) << ((lane / g) * g));
        const int base = (lane / g) * g;
        const double ctol = 1e-5 * (double)bnorm, pv = 1e-290, stop = 1e-12 * (double)bnorm;
        const int j = (mi < nbig) ? ccnt[mi] : 0;
        const int target = N - j;   // lambda_j is the target-th smallest
        double lo = (double)lam[j] - 2.0 * ctol, hi = (double)lam[j] + 2.0 * ctol;
        bool ok = mi < nbig;
        auto cnt2 = [&](double x0, double x1, int& c0, int& c1) {
          double q0 = (double)dd[0] - x0, q1 = (double)dd[0] - x1;
          if (fabs(q0) < pv) q0 = -pv;
          if (fabs(q1) < pv) q1 = -pv;
          int n0 = q0 < 0.0, n1 = q1 < 0.0;
          for (int i = 1; i < N; ++i) {
            const double di = (double)dd[i], ei = (double)e2[i - 1];
            q0 = (di - x0) - ei * rcp_d(q0);
            q1 = (di - x1) - ei * rcp_d(q1);
            if (fabs(q0) < pv) q0 = -pv;
            if (fabs(q1) < pv) q1 = -pv;
            n0 += q0 < 0.0;
            n1 += q1 < 0.0;
          }
          c0 = n0;
          c1 = n1;
        };
        {   // the bracket must hold lambda_j, else keep the fp32 value
          int clo = 0, chi = N;
          if (ok) cnt2(lo, hi, clo, chi);
          ok = ok && clo < target && chi >= target;
        }
        const int P = 2 * g;
        for (int it = 0; it < 64; ++it) {
          const bool need = ok && (hi - lo > stop);
          if (!__syncthreads_or(need)) break;
          const double step = (hi - lo) / (double)(P + 1);
          int c0 = 0, c1 = 0;
          if (need) cnt2(lo + step * (double)(sub + 1), lo + step * (double)(sub + g + 1), c0, c1);
          const unsigned m0 = __ballot_sync(0xffffffffu, need && c0 >= target) & gmask;
          const unsigned m1 = __ballot_sync(0xffffffffu, need && c1 >= target) & gmask;
          int ss = P;   // first point at or above lambda_j
          if (m0) ss = __ffs(m0) - 1 - base;
          else if (m1) ss = __ffs(m1) - 1 - base + g;
          if (need) {
            const double nlo = (ss == 0) ? lo : lo + step * (double)ss;
            const double nhi = (ss == P) ? hi : lo + step * (double)(ss + 1);
            lo = nlo;
            hi = fmax(nhi, nlo);
          }
        }
        if (ok && sub == 0) lamd[j] = fmax(0.5 * (lo + hi), 0.0);
        __syncthreads();
        if (tid == 0) {   // rebuild the clusters (same rules) on the fp64 shifts
          const double ctol2 = 1e-10 * (double)bnorm;
          const int bnd = (p.rule == RULE_ISVD) ? J : ((p.m < ell) ? ell - p.m : -1);
          const int jx0 = s_jx;
          int ncl = 0, jx = 0;
          for (int j = 0; j < jx0; ++j) {
            const bool cont = (j > 0) && (lamd[j - 1] - lamd[j] <= ctol2);
            if (!cont) {
              if (j >= J) break;
              cstart[ncl] = j; clen[ncl] = 0; ++ncl;
            }
            clen[ncl - 1]++;
            jx = j + 1;
          }
          int nrr = 0;
          for (int c = 0; c < ncl; ++c) {
            const int a = cstart[c], b = cstart[c] + clen[c];
            if (bnd > a && bnd < b) cid[nrr++] = c;
          }
          s_ncl = ncl; s_jx = jx; s_nrr = nrr;
        }
      }
    }
#endif
    __syncthreads();
    if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[4] += t_ - t_ph0; t_ph0 = t_; }
    // ---------------- eigenvectors of T: fp64 inverse iteration ----------------
    // One thread per vector j < JX (3 iterations, shift lam[j]); after every
    // iteration the members of each multi-member cluster are orthonormalised by
    // one warp (modified Gram-Schmidt, twice), so a member converges inside the
    // complement of the earlier ones.  Scratch is element-major (z[i * zst + j]):
    // the per-thread recurrences are coalesced across threads.
    const int ncl = s_ncl;
    const int JX = s_jx;
    int* vact = ccnt;   // coarse bisection counts are dead here: per-vector "needed" flags
    for (int j = tid; j < JX; j += blockDim.x) {   // singletons with zero weight are not needed
      bool a = wgt[j] != T(0);
      if (!a) {
        int c = 0;
        while (c + 1 < ncl && cstart[c + 1] <= j) ++c;
        a = clen[c] > 1;
      }
      vact[j] = a;
      pscl[j] = 1.0;
    }
    __syncthreads();
    {
      // recurrence precision of the twisted solves (FD_INV_F32: fp32 A/B)
      using RT = typename std::conditional<PRE && FD_INV_F32, float, double>::type;
      const RT tiny = (sizeof(RT) == 4) ? (RT)(1.2e-7 * (double)bnorm + 1e-30) : (RT)(2.3e-16 * (double)bnorm + 1e-300);
      long long t_iv = clock64();
      // Twisted solves: vector j is solved by the lane pair (2j', 2j'+1); the even
      // lane eliminates rows 0..m-1 top-down (T - mu I = L D+ L^T part), the odd lane
      // rows N-1..m+1 bottom-up (U D- U^T part); they meet at the twist m = N/2
      // (gamma_m = a_m - l_{m-1} e_{m-1} - u_m e_m) and back-substitute outwards.
      // Same arithmetic as one LDL^T solve, half the sequential chain.
      const int side = tid & 1;
      const unsigned pmask = 3u << (lane & ~1);
      const int m = N >> 1;
      for (int it = 0; it < kInvIters; ++it) {
        for (int j = tid >> 1; j < JX; j += blockDim.x >> 1) {
          if (!vact[j]) continue;
          ZT* lf = LF + j;   // lf[i * zst]: l_i (i < m), u_i (i >= m)
          ZT* z = Zs + j;    // z[i * zst]
          const RT sc = (RT)pscl[j];
          const RT mu = (RT)lamd[j];
          auto rhs = [&](int i, RT zi) -> RT {
            return (it == 0) ? (RT)(1.0 + 0.5 * (double)(((i + 1) * 7919 + (j + 3) * 104729) % 211) / 211.0) : zi * sc;
          };
          // Both lanes run ONE instruction stream (no divergence): step k of a side is
          // row i = i0 + dir k; the coupling to the previous row of its elimination
          // order is e[ec] with ec = i - 1 (top) / i (bottom), stored multiplier lf[ec].
          const int cnt = side ? (N - 1 - m) : m;     // rows of this side (<= m)
          const int dir = side ? -1 : 1, ist = side ? N - 1 : 0;
          RT rd = 0, w = 0, eprev = 0;
          for (int k0 = 0; k0 < m; k0 += kSB) {
            RT zb[kSB];
            if (it > 0) {
#pragma unroll
              for (int q = 0; q < kSB; ++q) zb[q] = (k0 + q < cnt) ? z[(size_t)(ist + dir * (k0 + q)) * zst] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < kSB; ++q) {
              const int k = k0 + q;
              if (k < cnt) {
                const int i = ist + dir * k;
                const RT bi = rhs(i, zb[q]);
                RT dpi;
                if (k == 0) {
                  dpi = (RT)dd[i] - mu;
                  w = bi;
                } else {
                  const RT li = eprev * rd;
                  lf[(size_t)(i - 1 + side) * zst] = li;
                  dpi = ((RT)dd[i] - mu) - li * eprev;
                  w = bi - li * w;
                }
                if (fabs(dpi) < tiny) dpi = (dpi < (RT)0) ? -tiny : tiny;
                rd = rcp_rt(dpi);
                zb[q] = w * rd;
                eprev = (RT)ee[i - side];
              }
            }
#pragma unroll
            for (int q = 0; q < kSB; ++q)
              if (k0 + q < cnt) z[(size_t)(ist + dir * (k0 + q)) * zst] = zb[q];
          }
          RT tS = 0, wS = 0;   // this side's term of the twist row
          if (cnt > 0) {
            const RT l = eprev * rd;   // l_{m-1} (top) / u_m (bottom)
            lf[(size_t)(m - 1 + side) * zst] = l;
            tS = l * eprev;
            wS = l * w;
          }
          // twist row m (both lanes, identical arithmetic)
          const RT tO = __shfl_xor_sync(pmask, tS, 1), wO = __shfl_xor_sync(pmask, wS, 1);
          const RT tA = side ? tO : tS, tB = side ? tS : tO;
          const RT wA = side ? wO : wS, wB = side ? wS : wO;
          RT gm = (((RT)dd[m] - mu) - tA) - tB;
          if (fabs(gm) < tiny) gm = (gm < (RT)0) ? -tiny : tiny;
          const RT bm = rhs(m, (it > 0) ? (RT)z[(size_t)m * zst] : (RT)0);
          const RT zm = ((bm - wA) - wB) * rcp_rt(gm);
          __syncwarp(pmask);   // both lanes read z[m] before it is overwritten
          if (side == 0) z[(size_t)m * zst] = zm;
          double nr = side ? 0.0 : (double)zm * (double)zm;
          // back-substitution outwards from m: top i = m-1..0 (l_i = lf[i]),
          // bottom i = m+1..N-1 (u_{i-1} = lf[i-1])
          RT next = zm;
          const int bst = side ? m + 1 : m - 1, bdir = side ? 1 : -1;
          for (int k0 = 0; k0 < m; k0 += kSB) {
            RT zb[kSB], lb[kSB];
#pragma unroll
            for (int q = 0; q < kSB; ++q) {
              const int i = bst + bdir * (k0 + q);
              const bool ok = k0 + q < cnt;
              zb[q] = ok ? z[(size_t)i * zst] : 0.0;
              lb[q] = ok ? lf[(size_t)(i - side) * zst] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < kSB; ++q) {
              if (k0 + q < cnt) {
                next = zb[q] - lb[q] * next;
                zb[q] = next;
                nr += (double)next * (double)next;
              }
            }
#pragma unroll
            for (int q = 0; q < kSB; ++q)
              if (k0 + q < cnt) z[(size_t)(bst + bdir * (k0 + q)) * zst] = zb[q];
          }
          nr += __shfl_xor_sync(pmask, nr, 1);
          if (side == 0) pscl[j] = (nr > 0.0) ? 1.0 / sqrt(nr) : 0.0;
        }
        __syncthreads();
        if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[16] += t_ - t_iv; t_iv = t_; }
        // clusters of 2..kSmallCl members: one warp each, modified Gram-Schmidt
        // (normalise, orthogonalise twice, renormalise)
        for (int c = warp; c < ncl; c += kNW) {
          const int j0 = cstart[c], j1 = cstart[c] + clen[c];
          if (j1 - j0 < 2 || j1 - j0 > kSmallCl) continue;
          for (int k = j0; k < j1; ++k) {
            ZT* zk = Zs + k;
            double zr[NM / 32];
            const double s0 = pscl[k];
#pragma unroll
            for (int t = 0; t < NM / 32; ++t) {
              const int i = 32 * t + lane;
              zr[t] = (i < N) ? zk[(size_t)i * zst] * s0 : 0.0;
            }
            for (int pass = 0; pass < 2; ++pass)
              for (int q = j0; q < k; ++q) {
                const ZT* zq = Zs + q;
                double zqr[NM / 32];
                double h = 0.0;
#pragma unroll
                for (int t = 0; t < NM / 32; ++t) {
                  const int i = 32 * t + lane;
                  zqr[t] = (i < N) ? zq[(size_t)i * zst] : 0.0;
                  h = fma(zqr[t], zr[t], h);
                }
                h = warp_sum_d(h);
#pragma unroll
                for (int t = 0; t < NM / 32; ++t) zr[t] = fma(-h, zqr[t], zr[t]);
              }
            double n2 = 0.0;
#pragma unroll
            for (int t = 0; t < NM / 32; ++t) n2 = fma(zr[t], zr[t], n2);
            n2 = warp_sum_d(n2);
            const double inv = (n2 > 0.0) ? 1.0 / sqrt(n2) : 0.0;
#pragma unroll
            for (int t = 0; t < NM / 32; ++t) {
              const int i = 32 * t + lane;
              if (i < N) zk[(size_t)i * zst] = zr[t] * inv;
            }
            __syncwarp();
            if (lane == 0) pscl[k] = 1.0;
          }
        }
        if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[17] += t_ - t_iv; t_iv = t_; }
        // larger clusters (wide-spread Grams put many small eigenvalues within ctol,
        // e.g. at merge levels): the whole CTA, one cluster at a time, in panels of 8
        // members.  Per panel: two passes of block Gram-Schmidt against the cluster's
        // earlier (orthonormal) members in chunks of 32 -- dots: warp w takes rows
        // w*rpw.., lane = earlier member (contiguous in the element-major scratch), the
        // panel's values of a row broadcast by shuffle from the lane holding that row;
        // update: a thread per row -- then one warp orthonormalises the panel itself
        // (modified Gram-Schmidt twice, registers).
        if constexpr (BIG) {   // merge launches: panels of 8 (block CGS2 + warp MGS)
          panel_cgs<NM, kNT, ZT>(Zs, zst, pscl, cpart, cstart, clen, ncl, N);
          __syncthreads();
        } else {
          double* chq = cpart + kNW * kCpStride;   // [NM] projection coefficients
        // larger clusters (wide-spread Grams put many small eigenvalues within ctol,
        // e.g. at merge levels): the whole CTA, one cluster at a time, classical
        // Gram-Schmidt twice per member.  Dots: warp w sweeps its rows, lane = earlier
        // member (row segments of a cluster are contiguous in the element-major
        // scratch -> coalesced); update: thread per row.
        for (int c = 0; c < ncl; ++c) {
          const int j0 = cstart[c], nc = clen[c];
          if (nc <= kSmallCl) continue;
          const int rpw = (N + kNW - 1) / kNW;   // rows per warp
          for (int k = j0; k < j0 + nc; ++k) {
            ZT* zk = Zs + k;
            const double s0 = pscl[k];
            __syncthreads();   // previous member finished; pscl stable
            for (int i = tid; i < N; i += kNT) zk[(size_t)i * zst] *= s0;
            for (int pass = 0; pass < 2 && k > j0; ++pass) {
              __syncthreads();
              for (int q0 = 0; q0 < k - j0; q0 += 32) {
                const int q = j0 + q0 + lane;
                double h = 0.0;
                if (q < k) {
                  const int ia = warp * rpw, ib = min(N, ia + rpw);
                  int i = ia;
                  for (; i + 8 <= ib; i += 8) {   // 8 independent load pairs in flight
                    double za[8], zb[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                      za[u] = Zs[(size_t)(i + u) * zst + q];
                      zb[u] = zk[(size_t)(i + u) * zst];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) h = fma(za[u], zb[u], h);
                  }
                  for (; i < ib; ++i) h = fma((double)Zs[(size_t)i * zst + q], (double)zk[(size_t)i * zst], h);
                }
                cpart[warp * kCpStride + q0 + lane] = h;
              }
              __syncthreads();
              for (int q = tid; q < k - j0; q += kNT) {
                double h = 0.0;
                for (int w = 0; w < kNW; ++w) h += cpart[w * kCpStride + q];
                chq[q] = h;
              }
              __syncthreads();
              for (int i = tid; i < N; i += kNT) {
                double zi = zk[(size_t)i * zst];
                const ZT* zrow = Zs + (size_t)i * zst + j0;
                const int nq = k - j0;
                int q = 0;
                for (; q + 8 <= nq; q += 8) {   // 8 independent loads in flight
                  double zr8[8];
#pragma unroll
                  for (int u = 0; u < 8; ++u) zr8[u] = zrow[q + u];
#pragma unroll
                  for (int u = 0; u < 8; ++u) zi = fma(-chq[q + u], zr8[u], zi);
                }
                for (; q < nq; ++q) zi = fma(-chq[q], (double)zrow[q], zi);
                zk[(size_t)i * zst] = zi;
              }
            }
            __syncthreads();
            double n2 = 0.0;
            for (int i = tid; i < N; i += kNT) { const double x = zk[(size_t)i * zst]; n2 = fma(x, x, n2); }
            n2 = warp_sum_d(n2);
            if (lane == 0) cpart[warp] = n2;
            __syncthreads();
            double tot = 0.0;
            for (int w = 0; w < kNW; ++w) tot += cpart[w];
            const double inv = (tot > 0.0) ? 1.0 / sqrt(tot) : 0.0;
            for (int i = tid; i < N; i += kNT) zk[(size_t)i * zst] *= inv;
            if (tid == 0) pscl[k] = 1.0;
          }
        }
        __syncthreads();
        }
        if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[18] += t_ - t_iv; t_iv = t_; }
      }
      for (int j = tid; j < JX; j += blockDim.x)
        if (vact[j]) pvec[j] = (T)pscl[j];   // normalisation folded into the back-transform
    }
    // Rayleigh-Ritz inside the (rare) clusters that straddle a rule discontinuity:
    // H = Z_c^T T Z_c (fp64), cyclic Jacobi on H, Z_c <- Z_c Q (eigenvalues descending).
    for (int r = 0; r < s_nrr; ++r) {
      const int c = cid[r];
      const int j0 = cstart[c], nc = clen[c];
      double* H = slot;                 // nc x nc (ld nc), over the dead multipliers
      double* Q = RD;                   // nc x nc (ld nc)
      double* Zc = slot + (size_t)3 * kMaxN * kMaxN;   // copy of Z_c (N x nc), 4th scratch region
      for (int x = tid; x < nc * nc; x += blockDim.x) {
        const int a = x / nc, b = x % nc;
        const ZT* za = Zs + j0 + a;
        const ZT* zb = Zs + j0 + b;
        double h = 0.0;
        for (int i = 0; i < N; ++i) {
          double tz = (double)dd[i] * zb[(size_t)i * zst];
          if (i > 0) tz += (double)ee[i - 1] * zb[(size_t)(i - 1) * zst];
          if (i < N - 1) tz += (double)ee[i] * zb[(size_t)(i + 1) * zst];
          h = fma((double)za[(size_t)i * zst], tz, h);
        }
        H[a * nc + b] = h;
        Q[a * nc + b] = (a == b) ? 1.0 : 0.0;
      }
      for (int x = tid; x < N * nc; x += blockDim.x) {
        const int i = x / nc, a = x % nc;
        Zc[(size_t)i * nc + a] = Zs[(size_t)i * zst + j0 + a];
      }
      __syncthreads();
      if (warp == 0) {
        for (int sweep = 0; sweep < 30; ++sweep) {
          int rot = 0;
          for (int a = 0; a < nc - 1; ++a)
            for (int b = a + 1; b < nc; ++b) {
              const double hab = H[a * nc + b], haa = H[a * nc + a], hbb = H[b * nc + b];
              if (fabs(hab) <= 1e-15 * sqrt(fabs(haa * hbb)) + 1e-300) continue;
              ++rot;
              const double th = (hbb - haa) / (2.0 * hab);
              const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
              const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
              __syncwarp();
              for (int k = lane; k < nc; k += 32) {
                if (k == a || k == b) continue;
                const double hka = H[k * nc + a], hkb = H[k * nc + b];
                const double na = cs * hka - sn * hkb, nb = sn * hka + cs * hkb;
                H[k * nc + a] = na; H[a * nc + k] = na;
                H[k * nc + b] = nb; H[b * nc + k] = nb;
              }
              for (int k = lane; k < nc; k += 32) {
                const double qa = Q[k * nc + a], qb = Q[k * nc + b];
                Q[k * nc + a] = cs * qa - sn * qb;
                Q[k * nc + b] = sn * qa + cs * qb;
              }
              __syncwarp();
              if (lane == 0) {
                H[a * nc + a] = haa - t * hab;
                H[b * nc + b] = hbb + t * hab;
                H[a * nc + b] = 0.0;
                H[b * nc + a] = 0.0;
              }
              __syncwarp();
            }
          if (rot == 0) break;
        }
        // order of the Ritz vectors: descending Ritz value (stable)
        if (lane == 0) {
          for (int a = 0; a < nc; ++a) ord[a] = a;
          for (int a = 1; a < nc; ++a) {
            const int x = ord[a];
            int b = a - 1;
            while (b >= 0 && H[ord[b] * (nc + 1)] < H[x * (nc + 1)]) {
              ord[b + 1] = ord[b];
              --b;
            }
            ord[b + 1] = x;
          }
        }
      }
      __syncthreads();
      for (int x = tid; x < N * nc; x += blockDim.x) {
        const int i = x / nc, k = x % nc;
        const int col = ord[k];
        double s = 0.0;
        for (int a = 0; a < nc; ++a) s = fma(Zc[(size_t)i * nc + a], Q[a * nc + col], s);
        Zs[(size_t)i * zst + j0 + k] = s;
      }
      __syncthreads();
    }
    __syncthreads();
    if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[5] += t_ - t_ph0; t_ph0 = t_; }
    if (PRE || p.pretrd) {
      // ---------------- hand Z to bt_kernel (fd_bt.cu) ----------------
      // Wt scratch <- Z row-major [r][j] (ld 128; normalised, fp32; 0 for unused j);
      // w_j after the tridiagonal data in the Gram scratch
      {  // thread -> fixed column j; 8 independent row loads in flight per batch
        const int j = tid & 127, rs = blockDim.x >> 7;
        const bool a = (j < J) && (wgt[j] != T(0));
        const double sc = a ? (double)pvec[j] : 0.0;
        for (int r0 = tid >> 7; r0 < N; r0 += 8 * rs) {
          double v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int r = r0 + q * rs;
            v[q] = (a && r < N) ? Zs[(size_t)r * zst + j] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int r = r0 + q * rs;
            if (r < N) Wt[r * 128 + j] = (T)(v[q] * sc);
          }
        }
      }
      {
        float* wout = reinterpret_cast<float*>(P.G) + (N * (N + 1) / 2 + 3) / 4 * 4 + 3 * N;
        for (int j = tid; j < J; j += blockDim.x) wout[j] = (float)wgt[j];
      }
    } else if constexpr (!PRE)
    // ---------------- back-transform U = H_0 ... H_{N-3} Z ; Wt = diag(w) U^T ----------------
    // warp-owned vectors held in registers (lane <-> rows 32t + lane), 4 per warp per chunk
    for (int c0 = 0; c0 < J; c0 += 4 * kNW) {
      T z[4][NT];
      bool act[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = c0 + warp + kNW * q;
        act[q] = (j < J) && (wgt[j] != T(0));
        const ZT* zg = Zs + (act[q] ? j : 0);
        const double zs = act[q] ? (double)pvec[j] : 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int R = 32 * t + lane;
          z[q][t] = (act[q] && R < N) ? (T)(zg[(size_t)R * zst] * zs) : T(0);
        }
      }
      const bool any = act[0] || act[1] || act[2] || act[3];
      if (any) {
        // reflector i's entries are register-prefetched during reflector i+1 (the
        // packed matrix sits in global / L2 scratch for N > kMaxNS: one L2 round trip
        // per reflector otherwise serialises the loop)
        auto vload = [&](int i, T (&v)[NT]) {
          const int base = pk_off(i, N) - i;
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int R = 32 * t + lane;
            v[t] = (R == i + 1) ? T(1) : ((R > i + 1 && R < N) ? Apk[base + R] : T(0));
          }
        };
        T vn[NT];
        if (N >= 3) vload(N - 3, vn);
        for (int i = N - 3; i >= 0; --i) {
          T v[NT];
#pragma unroll
          for (int t = 0; t < NT; ++t) v[t] = vn[t];
          if (i > 0) vload(i - 1, vn);
          const T ti = tau[i];
          if (ti == T(0)) continue;
          T s[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (32 * t + 31 < i + 1) continue;  // warp-uniform
#pragma unroll
            for (int q = 0; q < 4; ++q) s[q] = fma(v[t], z[q][t], s[q]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) s[q] = wsum(s[q]) * ti;
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (32 * t + 31 < i + 1) continue;
#pragma unroll
            for (int q = 0; q < 4; ++q) z[q][t] = fma(-s[q], v[t], z[q][t]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = c0 + warp + kNW * q;
        if (j >= J) continue;
        const T wj = act[q] ? wgt[j] : T(0);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int R = 32 * t + lane;
          if (R < N) Wt[(int64_t)j * p.ldg + R] = wj * z[q][t];
        }
      }
    }
    // rows J..ell-2 of Wt (only when N < ell-1) are zero
    for (int j = J + warp; j < p.ret; j += kNW)
      for (int r = lane; r < p.ldg; r += 32) Wt[(int64_t)j * p.ldg + r] = T(0);
    __syncthreads();
#if FD_EIG_DISCARD
    if (PRE) {
      // the inverse-iteration scratch of this problem is dead (the next problem of this
      // slot writes before it reads): drop its dirty L2 lines instead of writing them back
      const size_t nl = ((size_t)N * zst * sizeof(ZT) + 127) / 128;
      char* b0 = reinterpret_cast<char*>(LF);
      char* b1 = reinterpret_cast<char*>(Zs);
      for (size_t l = tid; l < nl; l += blockDim.x) {
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(b0 + l * 128) : "memory");
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(b1 + l * 128) : "memory");
      }
    }
#endif
    if (p.dbg && blockIdx.x == 0 && tid == 0) {
      p.dbg[6] += clock64() - t_ph0;
      int mx = 0;
      for (int c = 0; c < s_ncl; ++c) mx = max(mx, clen[c]);
      p.dbg[7] += s_ncl; p.dbg[8] = max((long long)mx, p.dbg[8]); p.dbg[9] = N; p.dbg[10] += 1;
    }
  }
}

template <typename T, int NM, bool GAPK, bool PRE = false, bool BIG = false>
static cudaError_t launch_eig_t(const Prob* dev_probs, int count, const Params& p, double* scratch, cudaStream_t s) {
  using C = EigCfg<T, NM, GAPK, PRE>;
  static AttrOnce once;
  if (cudaError_t e = once.ensure(eig_kernel<T, NM, GAPK, PRE, BIG>, (int)C::kBytes); e != cudaSuccess) return e;
  const int slots = kNumSMs * (PRE ? kEigPreCtasPerSM : 1);
  const int grid = count < slots ? count : slots;
  eig_kernel<T, NM, GAPK, PRE, BIG><<<grid, PRE ? 256 : kEigThreads, C::kBytes, s>>>(dev_probs, count, p, scratch);
  return cudaGetLastError();
}

cudaError_t launch_eig(const Prob* dev_probs, int count, const Params& p, double* scratch, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (p.f64) return launch_eig_t<double, kMaxN64, false>(dev_probs, count, p, scratch, s);
  if (p.pretrd) {
    // merge levels (p.merge) carry the large eigenvalue clusters: the panel variant;
    // stream rounds keep the member-wise variant (its register allocation is the
    // solver loop's)
    if (p.merge) return launch_eig_t<float, kMaxNS, false, true, true>(dev_probs, count, p, scratch, s);
    return launch_eig_t<float, kMaxNS, false, true>(dev_probs, count, p, scratch, s);
  }
  if (p.zld <= kMaxNS) return launch_eig_t<float, kMaxNS, false>(dev_probs, count, p, scratch, s);
  // above kMaxNS (c3 ell = 200 merges, N = 398): wide spectra put 100+ eigenvalues in
  // one cluster -> the panel block CGS2 (BIG)
  return launch_eig_t<float, kMaxN, true, false, true>(dev_probs, count, p, scratch, s);
}

__global__ void sub_btb_kernel(double* __restrict__ M, const double* __restrict__ AtA, const float* __restrict__ B,
                               int ell, int64_t d) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (j >= d) return;
  double s = 0.0;
  for (int r = 0; r < ell; ++r) s = fma((double)B[(int64_t)r * d + i], (double)B[(int64_t)r * d + j], s);
  M[i * d + j] = AtA[i * d + j] - s;
}

cudaError_t launch_sub_btb(double* M, const double* AtA, const float* B, int ell, int64_t d, cudaStream_t s) {
  dim3 grid((unsigned)((d + 255) / 256), (unsigned)d);
  sub_btb_kernel<<<grid, 256, 0, s>>>(M, AtA, B, ell, d);
  return cudaGetLastError();
}


}  // namespace fdk
