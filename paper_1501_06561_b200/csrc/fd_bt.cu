// fd_bt.cu — blocked back-transform of the eigenvectors of one ReduceRank:
// U_J = Q Z_J with Q = H_0 H_1 ... H_{N-3} the Householder reflectors of the
// tridiagonalisation (trd_kernel, fd_trd.cu), then Wt = diag(w) U_J^T, the
// weights of the reconstruct B' = Wt Bf = S'V^T ("B_[i] <- S'V^T", Alg. 1,
// PAPER.md:238; w_j = sigma'_j / sigma_j per the ReduceRank rule).
//
// Compact WY form (LAPACK xLARFT 'F','C'): a block of nb = 32 consecutive
// reflectors is Q_b = I - V_b T_b V_b^T with T_b upper triangular, so
// Z <- Q_b Z = Z - V_b (T_b (V_b^T Z)) is two GEMM-shaped products, applied from
// the last block to the first.  One CTA per problem (persistent), Z resident in
// shared memory (fp32), V_b streamed from the reflectors trd_kernel left in the
// problem's Gram scratch; register-blocked FP32 SIMT products (FP32-accurate,
// like the rest of the eigensolver).
//
// In:  P.G  = packed reflectors (column i rows i+2..N-1 at pk_off(i,N) + r - i),
//             tau at off = round_up(N(N+1)/2, 4) + 2N, w_j at off + N;
//      P.Wt = Z row-major [r][j], ld 128 (normalised eigenvectors of T, 0 if unused).
// Out: P.Wt rows j < J (ld ldg): w_j U[:, j]^T; rows J..ell-2: 0.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fd_internal.h"

namespace fdk {

namespace {

constexpr int kBtThreads = 512;    // two groups of 8 warps split the row range of each product
constexpr int kNbBt = 32;          // reflectors per block
constexpr int kZld = 132;          // Z row stride (floats): J <= 128, padded
constexpr int kVld = kMaxNS + 1;    // V_b column stride (column-major, odd: conflict-free)

__device__ __forceinline__ int pk_off_b(int c, int N) { return c * N - (c * (c - 1)) / 2; }

}  // namespace

__global__ void __launch_bounds__(kBtThreads, 1) bt_kernel(const Prob* __restrict__ probs, int count, Params p) {
  extern __shared__ __align__(16) float sm[];
  float* Zs = sm;                                  // [kMaxNS][kZld]
  float* Vb = Zs + kMaxNS * kZld;                   // [32][kVld]   Vb[c][r] = v_{i0+c}[r]
  float* W1 = Vb + kNbBt * kVld;                   // [32][128]
  float* W2 = W1 + kNbBt * 128;                    // [32][128]  (also group 1's partial W1)
  float* S = W2 + kNbBt * 128;                     // [32][33]  V^T V
  float* Tm = S + kNbBt * 33;                      // [32][33]  T
  float* tau = Tm + kNbBt * 33;                    // [32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp >> 3, wg8 = warp & 7;       // row-range group, warp within group
  const int ell = p.ell;

  for (int pi = blockIdx.x; pi < count; pi += gridDim.x) {
    const Prob P = probs[pi];
    const int N = P.rows0 + P.rows1;
    const int J = min(ell - 1, N);
    const int Jp = (J + 3) & ~3;                   // columns updated (multiple of 4, <= 128)
    const float* V = static_cast<const float*>(P.G);
    const float* taug = V + (N * (N + 1) / 2 + 3) / 4 * 4 + 2 * N;
    const float* wg = taug + N;
    float* Wt = static_cast<float*>(P.Wt);
    // Z [r][j] (ld 128) -> Zs
    for (int x = tid; x < N * 32; x += kBtThreads) {
      const int r = x >> 5, j4 = 4 * (x & 31);
      *reinterpret_cast<float4*>(&Zs[r * kZld + j4]) = *reinterpret_cast<const float4*>(Wt + (int64_t)r * 128 + j4);
    }
    __syncthreads();
    const int nref = N - 2;                        // reflectors 0..N-3
    const int nblk = (nref + kNbBt - 1) / kNbBt;
    for (int b = nblk - 1; b >= 0; --b) {
      const int i0 = b * kNbBt, nb = min(kNbBt, nref - i0);
      const int r0 = i0 + 1;                       // rows < r0 of the block's vectors are 0
      // ---- V_b (rows r0..N-1) and tau ----
      for (int x = tid; x < kNbBt * (N - r0); x += kBtThreads) {
        const int c = x / (N - r0), r = r0 + (x - c * (N - r0));
        float v = 0.f;
        if (c < nb && taug[i0 + c] != 0.f) {   // tau = 0: identity reflector -> zero column
          const int i = i0 + c;
          v = (r == i + 1) ? 1.f : ((r > i + 1) ? V[pk_off_b(i, N) + r - i] : 0.f);
        }
        Vb[c * kVld + r] = v;
      }
      if (tid < kNbBt) {
        const float t = (tid < nb) ? taug[i0 + tid] : 0.f;
        tau[tid] = (t != 0.f) ? t : 1.f;   // zero columns of V_b: any nonzero tau (no effect)
      }
      __syncthreads();
      // ---- W1 = V_b^T Z and S = V_b^T V_b (one pass over the rows; group g takes
      //      rows r0 + g, r0 + g + 2, ...; group 1's partials go to W2 / Tm) ----
      {
        const int cb = 4 * wg8, jb = 4 * lane;
        float acc[4][4] = {};
        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 2
        for (int r = r0 + grp; r < N; r += 2) {
          const float4 zz = *reinterpret_cast<const float4*>(&Zs[r * kZld + jb]);
          const float vl = Vb[lane * kVld + r];
          float va[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) va[a] = Vb[(cb + a) * kVld + r];
          const float za[4] = {zz.x, zz.y, zz.z, zz.w};
#pragma unroll
          for (int a = 0; a < 4; ++a) {
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[a][q] = fmaf(va[a], za[q], acc[a][q]);
            sacc[a] = fmaf(va[a], vl, sacc[a]);
          }
        }
        float* Wd = grp ? W2 : W1;
        float* Sd = grp ? Tm : S;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          *reinterpret_cast<float4*>(&Wd[(cb + a) * 128 + jb]) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
          Sd[(cb + a) * 33 + lane] = sacc[a];
        }
      }
      __syncthreads();
      for (int x = tid; x < kNbBt * 128; x += kBtThreads) W1[x] += W2[x];
      for (int x = tid; x < kNbBt * 32; x += kBtThreads) {
        const int a = x >> 5, c = x & 31;
        S[a * 33 + c] += Tm[a * 33 + c];
      }
      __syncthreads();
      // ---- T = U^-1, U = diag(1/tau) + strict_upper(V_b^T V_b): the xLARFT forward
      //      recurrence T[0:c,c] = -tau_c T[0:c,0:c] S[0:c,c] is exactly this inverse
      //      (induction on c).  Recursive doubling: for block size h = 1, 2, .., 16 the
      //      off-diagonal block of each 2h x 2h diagonal block is -T11 U12 T22. ----
      for (int x = tid; x < kNbBt * 32; x += kBtThreads) {
        const int a = x >> 5, c = x & 31;
        Tm[a * 33 + c] = (a == c) ? tau[a] : 0.f;
      }
      __syncthreads();
      for (int h = 1; h < kNbBt; h <<= 1) {
        const int npair = kNbBt / (2 * h), nent = npair * h * h;
        // Y = U12 T22 (U12 = S block, rows 2mh.., cols (2m+1)h..)
        for (int x = tid; x < nent; x += kBtThreads) {
          const int m = x / (h * h), e = x - m * h * h, i = e / h, j = e - (e / h) * h;
          const int r1 = 2 * m * h, c2 = (2 * m + 1) * h;
          float y = 0.f;
          for (int k = 0; k < h; ++k) y = fmaf(S[(r1 + i) * 33 + c2 + k], Tm[(c2 + k) * 33 + c2 + j], y);
          W2[x] = y;
        }
        __syncthreads();
        // X = -T11 Y
        for (int x = tid; x < nent; x += kBtThreads) {
          const int m = x / (h * h), e = x - m * h * h, i = e / h, j = e - (e / h) * h;
          const int r1 = 2 * m * h, c2 = (2 * m + 1) * h;
          float t = 0.f;
          for (int k = 0; k < h; ++k) t = fmaf(Tm[(r1 + i) * 33 + r1 + k], W2[m * h * h + k * h + j], t);
          Tm[(r1 + i) * 33 + c2 + j] = -t;
        }
        __syncthreads();
      }
      // ---- W2 = T W1 (T upper triangular; group 0) ----
      if (grp == 0) {
        const int cb = 4 * wg8, jb = 4 * lane;
        float acc[4][4] = {};
        {
          for (int k = cb; k < kNbBt; ++k) {
            const float4 ww = *reinterpret_cast<const float4*>(&W1[k * 128 + jb]);
            const float wa[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const float t = Tm[(cb + a) * 33 + k];
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[a][q] = fmaf(t, wa[q], acc[a][q]);
            }
          }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
          *reinterpret_cast<float4*>(&W2[(cb + a) * 128 + jb]) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
      }
      __syncthreads();
      // ---- Z[r0:N, :] -= V_b W2 : thread = 4 rows x 4 columns per 32-row group ----
      {
        const int rq = warp, jb = 4 * lane;   // 16 warps x 4 rows per 64-row sweep
        if (jb < Jp) {  // columns >= Jp of Z are zero
          for (int rbase = r0 + 4 * rq; rbase < N; rbase += 4 * (kBtThreads / 32)) {
            float acc[4][4] = {};
#pragma unroll 4
            for (int k = 0; k < nb; ++k) {
              const float4 ww = *reinterpret_cast<const float4*>(&W2[k * 128 + jb]);
              const float wa[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                const int r = rbase + a;
                const float v = (r < N) ? Vb[k * kVld + r] : 0.f;
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[a][q] = fmaf(v, wa[q], acc[a][q]);
              }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const int r = rbase + a;
              if (r < N) {
                float4 z = *reinterpret_cast<float4*>(&Zs[r * kZld + jb]);
                z.x -= acc[a][0]; z.y -= acc[a][1]; z.z -= acc[a][2]; z.w -= acc[a][3];
                *reinterpret_cast<float4*>(&Zs[r * kZld + jb]) = z;
              }
            }
          }
        }
      }
      __syncthreads();
    }
    // ---- Wt[j][r] = w_j U[r][j], transposed through per-warp 32 x 33 smem tiles ----
    {
      float* tile = Vb + warp * 32 * 33;   // V_b / W1 / W2 are free now (16 x 4.1 KB)
      const int ntr = (N + 31) / 32, ntj = (J + 31) / 32;
      for (int t = warp; t < ntr * ntj; t += kBtThreads / 32) {
        const int rt = t / ntj, jt = t - rt * ntj;
        const int j = 32 * jt + lane;
        for (int k = 0; k < 32; ++k) {
          const int r = 32 * rt + k;
          tile[lane * 33 + k] = (r < N && j < J) ? Zs[r * kZld + j] : 0.f;
        }
        __syncwarp();
        for (int k = 0; k < 32; ++k) {
          const int jj = 32 * jt + k, r = 32 * rt + lane;
          if (jj < J && r < N) Wt[(int64_t)jj * p.ldg + r] = wg[jj] * tile[k * 33 + lane];
        }
        __syncwarp();
      }
    }
    __syncthreads();
  }
}

size_t bt_smem_bytes() {
  return sizeof(float) * ((size_t)kMaxNS * kZld + (size_t)kNbBt * kVld + 2 * kNbBt * 128 + 2 * kNbBt * 33 + kNbBt);
}

bool bt_supported(int nmax, const Params& p) { return p.pretrd && nmax <= kMaxNS && p.ell - 1 <= 128; }

cudaError_t launch_bt(const Prob* dev_probs, int count, const Params& p, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int dyn = (int)bt_smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(bt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = count < kNumSMs ? count : kNumSMs;
  bt_kernel<<<grid, kBtThreads, dyn, s>>>(dev_probs, count, p);
  return cudaGetLastError();
}

}  // namespace fdk
