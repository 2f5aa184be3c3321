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

constexpr int kBtThreads = 256;
constexpr int kNbBt = 32;          // reflectors per block
constexpr int kZld = 132;          // Z row stride (floats): J <= 128, padded

__device__ __forceinline__ int pk_off_b(int c, int N) { return c * N - (c * (c - 1)) / 2; }

}  // namespace

__global__ void __launch_bounds__(kBtThreads, 1) bt_kernel(const Prob* __restrict__ probs, int count, Params p) {
  extern __shared__ __align__(16) float sm[];
  float* Zs = sm;                                  // [kMaxN][kZld]
  float* Vb = Zs + kMaxN * kZld;                   // [kMaxN][32]   Vb[r][c] = v_{i0+c}[r]
  float* W1 = Vb + kMaxN * kNbBt;                  // [32][128]
  float* W2 = W1 + kNbBt * 128;                    // [32][128]
  float* S = W2 + kNbBt * 128;                     // [32][33]  V^T V
  float* Tm = S + kNbBt * 33;                      // [32][33]  T
  float* tau = Tm + kNbBt * 33;                    // [32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
        if (c < nb) {
          const int i = i0 + c;
          v = (r == i + 1) ? 1.f : ((r > i + 1) ? V[pk_off_b(i, N) + r - i] : 0.f);
        }
        Vb[r * kNbBt + c] = v;
      }
      if (tid < kNbBt) tau[tid] = (tid < nb) ? taug[i0 + tid] : 0.f;
      __syncthreads();
      // ---- W1 = V_b^T Z and S = V_b^T V_b (one pass over the rows) ----
      {
        // thread: 4 reflectors (c-block = warp) x {4 columns of Z (lane), 1 column of V_b (lane)}
        const int cb = 4 * warp, jb = 4 * lane;
        float acc[4][4] = {};
        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int r = r0; r < N; ++r) {
          const float4 vv = *reinterpret_cast<const float4*>(&Vb[r * kNbBt + cb]);
          const float4 zz = *reinterpret_cast<const float4*>(&Zs[r * kZld + jb]);
          const float vl = Vb[r * kNbBt + lane];
          const float va[4] = {vv.x, vv.y, vv.z, vv.w}, za[4] = {zz.x, zz.y, zz.z, zz.w};
#pragma unroll
          for (int a = 0; a < 4; ++a) {
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[a][q] = fmaf(va[a], za[q], acc[a][q]);
            sacc[a] = fmaf(va[a], vl, sacc[a]);
          }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          *reinterpret_cast<float4*>(&W1[(cb + a) * 128 + jb]) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
          S[(cb + a) * 33 + lane] = sacc[a];
        }
      }
      __syncthreads();
      // ---- T (xLARFT forward, columnwise): T[c][c] = tau_c,
      //      T[0:c, c] = -tau_c T[0:c, 0:c] S[0:c, c]  (lane = row of T) ----
      if (warp == 0) {
        for (int c = 0; c < kNbBt; ++c) {
          float t = 0.f;
          if (lane < c) {
            for (int k = lane; k < c; ++k) t = fmaf(Tm[lane * 33 + k], S[k * 33 + c], t);
            t *= -tau[c];
          } else if (lane == c) {
            t = tau[c];
          }
          __syncwarp();
          if (lane <= c) Tm[lane * 33 + c] = t;
          else Tm[lane * 33 + c] = 0.f;
          __syncwarp();
        }
      }
      __syncthreads();
      // ---- W2 = T W1 (T upper triangular) ----
      {
        const int cb = 4 * warp, jb = 4 * lane;
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
        const int rq = warp, jb = 4 * lane;
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
                const float v = (r < N) ? Vb[r * kNbBt + k] : 0.f;
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
      float* tile = Vb + warp * 32 * 33;   // V_b / W1 are free now (8 x 4.1 KB)
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
  return sizeof(float) * ((size_t)kMaxN * kZld + (size_t)kMaxN * kNbBt + 2 * kNbBt * 128 + 2 * kNbBt * 33 + kNbBt);
}

bool bt_supported(int nmax, const Params& p) { return p.pretrd && nmax <= kMaxN && p.ell - 1 <= 128; }

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
