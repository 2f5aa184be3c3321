// fd_eval.cu — proj-err evaluator kernels:
//   proj-err(A, B) = ||A - pi_{B_k}(A)||_F^2 / ||A - A_k||_F^2   (PAPER.md:62-66,
//   k = 10 in the paper's experiments).
// B_k is the span of the top-k right singular vectors of B: from B B^T = U S^2 U^T
// (fp64 Gram, one-CTA parallel-ordering Jacobi), v_j = B^T u_j / s_j.  With V_k
// orthonormal, ||A - A V_k V_k^T||_F^2 = ||A||_F^2 - sum_j v_j^T (A^T A) v_j (the
// quadratic forms run on the evaluator's fp64 A^T A), and ||A - A_k||_F^2 =
// ||A||_F^2 - sum_{j<=k} lambda_j(A^T A) (Lanczos top-k Ritz values, fd_kernels.cu).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fd_internal.h"

namespace fdk {

namespace {

__device__ __forceinline__ double wsum_e(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// G[i][j] = sum_c B[i][c] B[j][c] (fp64), one warp per entry
__global__ void bbt_kernel(const float* __restrict__ B, int ell, int64_t d, double* __restrict__ G) {
  const int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= (int64_t)ell * ell) return;
  const int i = (int)(e / ell), j = (int)(e % ell);
  double s = 0.0;
  for (int64_t c = lane; c < d; c += 32) s = fma((double)B[(int64_t)i * d + c], (double)B[(int64_t)j * d + c], s);
  s = wsum_e(s);
  if (lane == 0) G[e] = s;
}

// Cyclic two-sided Jacobi on the n x n symmetric G (global, overwritten), one CTA.
// Parallel ordering (circle method): round r of a sweep rotates the n'/2 disjoint
// pairs {(n'-1, r)} U {((r+i) mod (n'-1), (r-i) mod (n'-1)) : 0 < i < n'/2}
// (n' = n rounded up to even; the padding index is skipped), i.e. G <- J^T G J with
// J a product of disjoint Givens rotations: columns first, then rows.  V (column j =
// eigenvector j) accumulates J.  w = diag(G); ord = indices by w descending (ties:
// lower index first).
__global__ void __launch_bounds__(1024, 1) jacobi_kernel(double* __restrict__ G, int n, double* __restrict__ V,
                                                         double* __restrict__ w, int* __restrict__ ord,
                                                         int* __restrict__ sweeps_out) {
  extern __shared__ double jsm[];
  const int np = (n + 1) & ~1, npair = np / 2;
  double* cs = jsm;                 // [npair]
  double* sn = cs + npair;          // [npair]
  int* pp = reinterpret_cast<int*>(sn + npair);
  int* qq = pp + npair;
  __shared__ int s_rot;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int x = tid; x < n * n; x += nt) V[x] = ((x / n) == (x % n)) ? 1.0 : 0.0;
  __syncthreads();
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int r = 0; r < np - 1; ++r) {
      for (int i = tid; i < npair; i += nt) {
        int p, q;
        if (i == 0) { p = np - 1; q = r; }
        else { p = (r + i) % (np - 1); q = (r - i + (np - 1)) % (np - 1); }
        if (p > q) { const int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = G[(int64_t)p * n + q], app = G[(int64_t)p * n + p], aqq = G[(int64_t)q * n + q];
          // rotate unless |apq| is at the fp64 noise level of its diagonal (a threshold
          // below eps would keep rotating noise until the sweep cap)
          if (apq != 0.0 && fabs(apq) > 1e-15 * sqrt(fabs(app) * fabs(aqq))) {
            const double th = (aqq - app) / (2.0 * apq);
            const double t = (fabs(th) > 1e150) ? 0.5 / th : ((th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0)));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
            s_rot = 1;
          }
        }
        pp[i] = p; qq[i] = (q < n) ? q : -1; cs[i] = c; sn[i] = s;
      }
      __syncthreads();
      // columns: G[:, p], G[:, q] and V[:, p], V[:, q]
      for (int x = tid; x < npair * n; x += nt) {
        const int i = x / n, k = x - i * n;
        const int p = pp[i], q = qq[i];
        if (q < 0 || sn[i] == 0.0) continue;
        const double c = cs[i], s = sn[i];
        const double gp = G[(int64_t)k * n + p], gq = G[(int64_t)k * n + q];
        G[(int64_t)k * n + p] = c * gp - s * gq;
        G[(int64_t)k * n + q] = s * gp + c * gq;
        const double vp = V[(int64_t)k * n + p], vq = V[(int64_t)k * n + q];
        V[(int64_t)k * n + p] = c * vp - s * vq;
        V[(int64_t)k * n + q] = s * vp + c * vq;
      }
      __syncthreads();
      // rows: G[p, :], G[q, :]
      for (int x = tid; x < npair * n; x += nt) {
        const int i = x / n, k = x - i * n;
        const int p = pp[i], q = qq[i];
        if (q < 0 || sn[i] == 0.0) continue;
        const double c = cs[i], s = sn[i];
        const double gp = G[(int64_t)p * n + k], gq = G[(int64_t)q * n + k];
        G[(int64_t)p * n + k] = c * gp - s * gq;
        G[(int64_t)q * n + k] = s * gp + c * gq;
      }
      __syncthreads();
      // the rotated pair is exactly decoupled (as in the oracle's Jacobi)
      for (int i = tid; i < npair; i += nt) {
        const int p = pp[i], q = qq[i];
        if (q < 0 || sn[i] == 0.0) continue;
        G[(int64_t)p * n + q] = 0.0;
        G[(int64_t)q * n + p] = 0.0;
      }
      __syncthreads();
    }
    if (!s_rot) break;
    __syncthreads();
  }
  for (int i = tid; i < n; i += nt) w[i] = G[(int64_t)i * n + i];
  __syncthreads();
  for (int i = tid; i < n; i += nt) {
    const double wi = w[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += (w[j] > wi) || (w[j] == wi && j < i);
    ord[rank] = i;
  }
  if (tid == 0) *sweeps_out = sweep;
}

// q[t] = v^T M v with v = B^T u_j / s_j, j = ord[t] (0 if s_j^2 <= 1e-12 s_1^2:
// B has rank < t+1 and B_k is spanned by the nonzero ones).  One CTA per t < k.
__global__ void __launch_bounds__(256) proj_quad_kernel(const float* __restrict__ B, int ell, int64_t d,
                                                        const double* __restrict__ V, const double* __restrict__ w,
                                                        const int* __restrict__ ord, const double* __restrict__ M,
                                                        double* __restrict__ vbuf, double* __restrict__ q) {
  __shared__ double red[8];
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* v = vbuf + (int64_t)t * d;
  const double wmax = w[ord[0]];
  const int j = (t < ell) ? ord[t] : -1;
  const bool live = (j >= 0) && (w[j] > 1e-12 * wmax) && (w[j] > 0.0);
  if (!live) {
    if (tid == 0) q[t] = 0.0;
    return;
  }
  const double inv = 1.0 / sqrt(w[j]);
  for (int64_t c = tid; c < d; c += blockDim.x) {
    double x = 0.0;
    for (int i = 0; i < ell; ++i) x = fma((double)B[(int64_t)i * d + c], V[(int64_t)i * ell + j], x);
    v[c] = x * inv;
  }
  __syncthreads();
  double acc = 0.0;
  for (int64_t r = warp; r < d; r += blockDim.x >> 5) {
    double s = 0.0;
    for (int64_t c = lane; c < d; c += 32) s = fma(M[r * d + c], v[c], s);
    s = wsum_e(s);
    acc = fma(v[r], s, acc);
  }
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int x = 0; x < (int)(blockDim.x >> 5); ++x) s += red[x];
    q[t] = s;
  }
}

}  // namespace

cudaError_t launch_proj_parts(const float* B, int ell, int64_t d, int k, const double* AtA, double* G, double* V,
                              double* w, int* ord, int* sweeps, double* vbuf, double* q, cudaStream_t s) {
  const int64_t ne = (int64_t)ell * ell;
  bbt_kernel<<<(unsigned)((ne + 7) / 8), 256, 0, s>>>(B, ell, d, G);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int npair = ((ell + 1) & ~1) / 2;
  const size_t smem = (size_t)npair * (2 * sizeof(double) + 2 * sizeof(int));
  jacobi_kernel<<<1, 1024, smem, s>>>(G, ell, V, w, ord, sweeps);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  proj_quad_kernel<<<k, 256, 0, s>>>(B, ell, d, V, w, ord, AtA, vbuf, q);
  return cudaGetLastError();
}

}  // namespace fdk
