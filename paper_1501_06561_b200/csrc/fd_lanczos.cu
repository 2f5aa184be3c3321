// fd_lanczos.cu — the evaluator's extreme eigenvalues (cov-err, PAPER.md:57 [Sec. 1];
// proj-err denominator) by Lanczos with full re-orthogonalisation
// (reading C11: FD residuals have lambda_2 / lambda_1 ~ 0.99996, so power iteration
// would need ~1e5 matvecs).
//
// B200 design: one persistent grid, one CTA per SM (cooperative launch, so every CTA
// is resident and the grid barrier is safe), five grid barriers per Lanczos step:
//   M   z = M q_j (warp per row; q_j = z_{j-1} / beta_j formed on the fly; each CTA also
//       stores its rows of q_j into Q)
//   D1  h_i = q_i^T z, i <= j (warp per dot across the grid); alpha_j = h_j
//   U1  z -= Q h (CTA = 32 rows x 8 slices of i, smem reduction)
//   D2, U2  the second Gram-Schmidt pass (CGS2); U2 leaves per-CTA partials of ||z||^2
// and every CTA sums the partials in CTA order, so beta_{j+1} (and the stop decision)
// is bit-identical on every CTA.  M (d x d fp64, 8 MB at d = 1024) and Q stay in L2;
// the single-CTA round-1 kernel was bound by one SM's L2 bandwidth (80 ms at d = 1024).
// The extreme Ritz values then come from fp64 bisection on the k x k tridiagonal (CTA 0).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fd_internal.h"

namespace cg = cooperative_groups;

namespace fdk {

namespace {

constexpr int kLzThreads = 256;
constexpr int kLzMaxCtas = 1024;   // partials slots in the work array

__device__ __forceinline__ double lz_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ int lz_sturm_count(const double* a, const double* b, int k, double x) {
  int cnt = 0;
  double q = a[0] - x;
  const double piv = 1e-300;
  if (fabs(q) < piv) q = -piv;
  cnt += q < 0.0;
  for (int i = 1; i < k; ++i) {
    q = (a[i] - x) - b[i] * b[i] / q;
    if (fabs(q) < piv) q = -piv;
    cnt += q < 0.0;
  }
  return cnt;
}

// bisection for the eigenvalue with `target` eigenvalues below-or-at it (1 = smallest,
// k = largest) of the k x k tridiagonal (alpha, beta[1..k-1])
__device__ double lz_bisect(const double* alpha, const double* beta, int k, int target) {
  double gl = 1e308, gu = -1e308;
  for (int i = 0; i < k; ++i) {
    const double em = (i > 0) ? fabs(beta[i]) : 0.0;
    const double ep = (i + 1 < k) ? fabs(beta[i + 1]) : 0.0;
    gl = fmin(gl, alpha[i] - em - ep);
    gu = fmax(gu, alpha[i] + em + ep);
  }
  double lo = gl - 1e-12 * fabs(gl) - 1e-300, hi = gu + 1e-12 * fabs(gu) + 1e-300;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (lz_sturm_count(alpha, beta, k, mid) >= target) hi = mid;
    else lo = mid;
  }
  return 0.5 * (lo + hi);
}

// z -= Q[0..j] h over this CTA's 32-row groups; returns this thread's share of ||z||^2
__device__ double lz_update(double* __restrict__ z, const double* __restrict__ Q, const double* __restrict__ h, int j,
                            int64_t d, double (*s_part)[33]) {
  const int tid = threadIdx.x, rr = tid & 31, sl = tid >> 5;   // row in group, slice of i
  double nrm = 0.0;
  for (int64_t g = (int64_t)blockIdx.x * 32; g < d; g += (int64_t)gridDim.x * 32) {
    const int64_t r = g + rr;
    double acc = 0.0;
    if (r < d) {
      int i = sl;
      for (; i + 24 <= j; i += 32) {   // four independent loads in flight
        const double a0 = Q[(int64_t)i * d + r], a1 = Q[(int64_t)(i + 8) * d + r];
        const double a2 = Q[(int64_t)(i + 16) * d + r], a3 = Q[(int64_t)(i + 24) * d + r];
        acc = fma(h[i], a0, acc);
        acc = fma(h[i + 8], a1, acc);
        acc = fma(h[i + 16], a2, acc);
        acc = fma(h[i + 24], a3, acc);
      }
      for (; i <= j; i += 8) acc = fma(h[i], Q[(int64_t)i * d + r], acc);
    }
    s_part[sl][rr] = acc;
    __syncthreads();
    if (sl == 0 && r < d) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += s_part[q][rr];
      const double zr = z[r] - s;
      z[r] = zr;
      nrm = fma(zr, zr, nrm);
    }
    __syncthreads();
  }
  return nrm;
}

// h[i] = Q[i]^T z, i <= j: one warp per dot across the grid
__device__ void lz_dots(const double* __restrict__ z, const double* __restrict__ Q, double* __restrict__ h, int j,
                        int64_t d) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), nw = gridDim.x * (blockDim.x >> 5);
  for (int i = gw; i <= j; i += nw) {
    const double* qi = Q + (int64_t)i * d;
    double s = 0.0;
    for (int64_t c = lane; c < d; c += 32) s = fma(qi[c], z[c], s);
    s = lz_warp_sum(s);
    if (lane == 0) h[i] = s;
  }
}

}  // namespace

size_t lanczos_work_doubles(int64_t d, int kmax) { return (size_t)(3 * kmax + 2) + 2 * (size_t)d + kLzMaxCtas + 64; }

// work layout (doubles): alpha[kmax] | beta[kmax+1] | z0[d] | z1[d] | h[kmax] | part[kLzMaxCtas] | misc[64]
__global__ void __launch_bounds__(kLzThreads, 1) lanczos_grid_kernel(const double* __restrict__ M, int64_t d,
                                                                     int kmax, double* __restrict__ Q,
                                                                     double* __restrict__ work,
                                                                     double* __restrict__ out2, int ntop,
                                                                     double* __restrict__ top) {
  cg::grid_group grid = cg::this_grid();
  double* alpha = work;
  double* beta = alpha + kmax;       // beta[j] couples q_{j-1}, q_j (beta[0] unused)
  double* zb[2] = {beta + kmax + 1, beta + kmax + 1 + d};
  double* h = zb[1] + d;
  double* part = h + kmax;
  __shared__ double s_part[8][33];
  __shared__ double s_red[kLzThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwb = blockDim.x >> 5;
  const int gw = blockIdx.x * nwb + warp, nwg = gridDim.x * nwb;

  // q_0 = v / ||v|| (every CTA forms ||v||^2 itself, same order: identical values)
  double ss = 0.0;
  for (int64_t i = tid; i < d; i += blockDim.x) {
    const double v = 1.0 + 0.001 * (double)((i * 7919) % 101);
    ss = fma(v, v, ss);
  }
  ss = lz_warp_sum(ss);
  if (lane == 0) s_red[warp] = ss;
  __syncthreads();
  ss = 0.0;
  for (int w = 0; w < nwb; ++w) ss += s_red[w];
  __syncthreads();
  double ib = 1.0 / sqrt(ss);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + tid; i < d; i += (int64_t)gridDim.x * blockDim.x)
    zb[1][i] = 1.0 + 0.001 * (double)((i * 7919) % 101);   // "z_{-1}": q_0 = z_{-1} * ib
  grid.sync();

  double amax = 0.0;
  int k = kmax;
  for (int j = 0; j < kmax; ++j) {
    const double* zp = zb[(j + 1) & 1];   // previous z (q_j = zp * ib)
    double* z = zb[j & 1];
    double* qj = Q + (int64_t)j * d;
    // ---- M: z = M q_j; this CTA's rows of q_j into Q ----
    for (int64_t r = gw; r < d; r += nwg) {
      const double* Mr = M + r * d;
      double s = 0.0;
      for (int64_t c = lane; c < d; c += 32) s = fma(Mr[c], zp[c] * ib, s);
      s = lz_warp_sum(s);
      if (lane == 0) z[r] = s;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + tid; i < d; i += (int64_t)gridDim.x * blockDim.x)
      qj[i] = zp[i] * ib;
    grid.sync();
    // ---- CGS2 against q_0..q_j ----
    lz_dots(z, Q, h, j, d);
    grid.sync();
    const double a = h[j];   // alpha_j = q_j^T (M q_j)
    lz_update(z, Q, h, j, d, s_part);
    grid.sync();
    lz_dots(z, Q, h, j, d);
    grid.sync();
    double nrm = lz_update(z, Q, h, j, d, s_part);
    nrm = lz_warp_sum(nrm);
    if (lane == 0) s_red[warp] = nrm;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < nwb; ++w) s += s_red[w];
      part[blockIdx.x] = s;
    }
    grid.sync();
    double b2 = 0.0;
    for (int c = 0; c < (int)gridDim.x; ++c) b2 += part[c];   // CTA order: identical on every CTA
    const double b = sqrt(b2);
    amax = fmax(amax, fabs(a));
    if (blockIdx.x == 0 && tid == 0) {
      alpha[j] = a;
      beta[j + 1] = b;
    }
    if (j + 1 == kmax || b <= 1e-12 * amax) {
      k = j + 1;
      break;
    }
    ib = 1.0 / b;
    // part[] is rewritten only after two more grid barriers: no hazard with this read
  }
  if (blockIdx.x != 0) return;
  __syncthreads();
  // top-ntop Ritz values (descending) for the proj-err denominator: thread 2 + t
  // bisects the (k - t)-th smallest; t >= k (Krylov space exhausted) -> 0
  if (tid >= 2 && tid < 2 + ntop) {
    const int t = tid - 2;
    top[t] = (t >= k) ? 0.0 : lz_bisect(alpha, beta, k, k - t);
  }
  if (tid < 2) out2[tid] = lz_bisect(alpha, beta, k, tid == 0 ? k : 1);   // largest, smallest
}

cudaError_t launch_lanczos(const double* M, int64_t d, int kmax, double* Q, double* work, double* out2,
                           cudaStream_t s, int ntop, double* top) {
  if (ntop > kLzThreads - 2) return cudaErrorInvalidValue;
  int dev = 0, nsm = 0, per_sm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lanczos_grid_kernel, kLzThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int grid = nsm < kLzMaxCtas ? nsm : kLzMaxCtas;   // one CTA per SM, all resident
  void* args[] = {(void*)&M, (void*)&d, (void*)&kmax, (void*)&Q, (void*)&work, (void*)&out2, (void*)&ntop, (void*)&top};
  return cudaLaunchCooperativeKernel((const void*)lanczos_grid_kernel, dim3(grid), dim3(kLzThreads), args, 0, s);
}

}  // namespace fdk
