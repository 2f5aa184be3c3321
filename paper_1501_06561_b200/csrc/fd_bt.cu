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
// problem's Gram scratch (register-prefetched one block ahead); register-blocked
// FP32 SIMT products (FP32-accurate, like the rest of the eigensolver).  Per block,
// one warp group forms V_b^T Z while the other forms V_b^T V_b and T.
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

constexpr int kBtThreads = 512;    // 16 warps: two groups of 8 overlap V^T Z with V^T V -> T
constexpr int kNbBt = 32;          // reflectors per block
constexpr int kZld = 132;          // Z row stride (floats): J <= 128, padded
constexpr int kVt = 36;            // V_b^T row stride: VbT[r][c] (16-byte aligned rows)

__device__ __forceinline__ int pk_off_b(int c, int N) { return c * N - (c * (c - 1)) / 2; }

__device__ __forceinline__ void bar_group1() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// the 16 V_b entries one thread stages for block (i0, nb): column c = 2 warp + cc,
// rows r0 + lane + 32 t (v_{i+1} = 1 implicit, rows above it 0, tau = 0 -> zero column)
__device__ __forceinline__ void vb_fetch(float (&pf)[16], const float* __restrict__ V, const float* __restrict__ taug,
                                         int i0, int nb, int N, int warp, int lane) {
  const int r0 = i0 + 1;
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const int c = 2 * warp + cc, i = i0 + c;
    const bool live = (c < nb) && (taug[i] != 0.f);
    const int base = pk_off_b(i, N) - i;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int r = r0 + lane + 32 * t;
      float v = 0.f;
      if (live && r < N) v = (r == i + 1) ? 1.f : ((r > i + 1) ? V[base + r] : 0.f);
      pf[8 * cc + t] = v;
    }
  }
}

}  // namespace

__global__ void __launch_bounds__(kBtThreads, 1) bt_kernel(const Prob* __restrict__ probs, int count, Params p) {
  extern __shared__ __align__(16) float sm[];
  float* Zs = sm;                                  // [kMaxNS][kZld]
  float* VbT = Zs + kMaxNS * kZld;                 // [kMaxNS][kVt]  VbT[r][c] = v_{i0+c}[r]
  float* W1 = VbT + kMaxNS * kVt;                  // [32][128]  V^T Z
  float* W2 = W1 + kNbBt * 128;                    // [32][128]  T V^T Z
  float* S = W2 + kNbBt * 128;                     // [32][33]   V^T V
  float* Tm = S + kNbBt * 33;                      // [32][33]   T
  float* Yb = Tm + kNbBt * 33;                     // [256]      recursive-doubling scratch
  float* tau = Yb + 256;                           // [32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp >> 3, wg8 = warp & 7;

  for (int pi = blockIdx.x; pi < count; pi += gridDim.x) {
    const Prob P = probs[pi];
    const int N = P.rows0 + P.rows1;
    const int J = min(p.ret, N);
    const int Jp = (J + 3) & ~3;                   // columns updated (multiple of 4, <= 128)
    const float* V = static_cast<const float*>(P.G);
    const float* taug = V + (N * (N + 1) / 2 + 3) / 4 * 4 + 2 * N;
    const float* wg = taug + N;
    float* Wt = static_cast<float*>(P.Wt);
    // Z [r][j] (ld 128) -> Zs
    {  // 4 independent 16-byte loads in flight per thread
      const int j4 = 4 * (tid & 31);
      for (int r0 = tid >> 5; r0 < N; r0 += 4 * (kBtThreads / 32)) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = r0 + u * (kBtThreads / 32);
          v[u] = (r < N) ? *reinterpret_cast<const float4*>(Wt + (int64_t)r * 128 + j4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = r0 + u * (kBtThreads / 32);
          if (r < N) *reinterpret_cast<float4*>(&Zs[r * kZld + j4]) = v[u];
        }
      }
    }
    const int nref = N - 2;                        // reflectors 0..N-3
    const int nblk = nref > 0 ? (nref + kNbBt - 1) / kNbBt : 0;
    float pf[16];
    float tpf = 0.f;
    if (nblk > 0) {
      const int i0 = (nblk - 1) * kNbBt;
      vb_fetch(pf, V, taug, i0, min(kNbBt, nref - i0), N, warp, lane);
      if (tid < kNbBt) tpf = (tid < nref - i0) ? taug[i0 + tid] : 0.f;
    }
    for (int b = nblk - 1; b >= 0; --b) {
      const int i0 = b * kNbBt, nb = min(kNbBt, nref - i0);
      const int r0 = i0 + 1;                       // rows < r0 of the block's vectors are 0
      // ---- stage V_b^T and tau (prefetched), then prefetch the next block ----
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int r = r0 + lane + 32 * t;
          if (r < N) VbT[r * kVt + 2 * warp + cc] = pf[8 * cc + t];
        }
      if (tid < kNbBt) tau[tid] = (tpf != 0.f) ? tpf : 1.f;   // zero columns: any nonzero tau
      __syncthreads();
      if (b > 0) {
        const int i0n = (b - 1) * kNbBt;
        vb_fetch(pf, V, taug, i0n, kNbBt, N, warp, lane);
        if (tid < kNbBt) tpf = taug[i0n + tid];
      }
      if (grp == 0) {
        // ---- W1 = V_b^T Z: warp (h, g) takes reflectors 8g..8g+7 x columns 4 lane..+3
        // over row half h (thread tile 8 x 4: one Z float4 and two broadcast V_b float4s
        // per 16 FFMA2, where a 4 x 4 tile over all rows spent 5 shared-memory wavefronts
        // per 8 FFMA2 and was bound by them); half 0 -> W1, half 1 -> W2 (summed below) ----
        const int g8 = wg8 & 3, hh = wg8 >> 2, cb = 8 * g8, jb = 4 * lane;
        const int rm = r0 + ((N - r0) >> 1);
        const int ra = hh ? rm : r0, rb = hh ? N : rm;
        float2 acc[8][2];   // column pairs on packed FFMA2, the V entries as broadcast scalars
#pragma unroll
        for (int a = 0; a < 8; ++a) acc[a][0] = acc[a][1] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int r = ra; r < rb; ++r) {
          const float4 zz = *reinterpret_cast<const float4*>(&Zs[r * kZld + jb]);
          const float4 v0 = *reinterpret_cast<const float4*>(&VbT[r * kVt + cb]);
          const float4 v1 = *reinterpret_cast<const float4*>(&VbT[r * kVt + cb + 4]);
          const float2 z01 = make_float2(zz.x, zz.y), z23 = make_float2(zz.z, zz.w);
          const float va[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            acc[a][0] = __ffma2_rn(make_float2(va[a], va[a]), z01, acc[a][0]);
            acc[a][1] = __ffma2_rn(make_float2(va[a], va[a]), z23, acc[a][1]);
          }
        }
        float* Wh = hh ? W2 : W1;
#pragma unroll
        for (int a = 0; a < 8; ++a)
          *reinterpret_cast<float4*>(&Wh[(cb + a) * 128 + jb]) = make_float4(acc[a][0].x, acc[a][0].y, acc[a][1].x, acc[a][1].y);
      } else {
        // ---- S = V_b^T V_b (thread: row a, columns c4..c4+3), then T = U^-1 ----
        const int t = tid - 256, a = t >> 3, c4 = 4 * (t & 7);
        float sa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int r = r0; r < N; ++r) {
          const float va = VbT[r * kVt + a];
          const float4 vv = *reinterpret_cast<const float4*>(&VbT[r * kVt + c4]);
          sa[0] = fmaf(va, vv.x, sa[0]); sa[1] = fmaf(va, vv.y, sa[1]);
          sa[2] = fmaf(va, vv.z, sa[2]); sa[3] = fmaf(va, vv.w, sa[3]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          S[a * 33 + c4 + q] = sa[q];
          Tm[a * 33 + c4 + q] = (a == c4 + q) ? tau[a] : 0.f;
        }
        bar_group1();
        // U = diag(1/tau) + strict_upper(V_b^T V_b); the xLARFT forward recurrence
        // T[0:c,c] = -tau_c T[0:c,0:c] S[0:c,c] is exactly T = U^-1 (induction on c).
        // Recursive doubling: for h = 1, 2, .., 16 the off-diagonal block of each
        // 2h x 2h diagonal block is -T11 U12 T22 (16 h entries, one per thread).
#pragma unroll
        for (int lh = 0; lh < 5; ++lh) {
          const int h = 1 << lh;
          const bool on = t < 16 * h;
          const int m = t >> (2 * lh), e = t & (h * h - 1), i = e >> lh, j = e & (h - 1);
          const int r1 = 2 * m * h, c2 = r1 + h;
          if (on) {
            float y = 0.f;
            for (int k = 0; k < h; ++k) y = fmaf(S[(r1 + i) * 33 + c2 + k], Tm[(c2 + k) * 33 + c2 + j], y);
            Yb[t] = y;
          }
          bar_group1();
          if (on) {
            float x = 0.f;
            for (int k = 0; k < h; ++k) x = fmaf(Tm[(r1 + i) * 33 + r1 + k], Yb[(m << (2 * lh)) + k * h + j], x);
            Tm[(r1 + i) * 33 + c2 + j] = -x;
          }
          bar_group1();
        }
      }
      __syncthreads();
      // W1 = sum of the two row-half partials (fixed order: half 0 + half 1)
      for (int e = tid; e < kNbBt * 128 / 4; e += kBtThreads) {
        float4 a = reinterpret_cast<float4*>(W1)[e];
        const float4 b2 = reinterpret_cast<const float4*>(W2)[e];
        a.x += b2.x; a.y += b2.y; a.z += b2.z; a.w += b2.w;
        reinterpret_cast<float4*>(W1)[e] = a;
      }
      __syncthreads();
      // ---- W2 = T W1 (T upper triangular; thread: 2 reflectors x 4 columns) ----
      {
        const int a0 = 2 * warp, jb = 4 * lane;
        float acc[2][4] = {};
        for (int k = a0; k < kNbBt; ++k) {
          const float4 ww = *reinterpret_cast<const float4*>(&W1[k * 128 + jb]);
          const float t0 = Tm[a0 * 33 + k], t1 = (k > a0) ? Tm[(a0 + 1) * 33 + k] : 0.f;
          acc[0][0] = fmaf(t0, ww.x, acc[0][0]); acc[0][1] = fmaf(t0, ww.y, acc[0][1]);
          acc[0][2] = fmaf(t0, ww.z, acc[0][2]); acc[0][3] = fmaf(t0, ww.w, acc[0][3]);
          acc[1][0] = fmaf(t1, ww.x, acc[1][0]); acc[1][1] = fmaf(t1, ww.y, acc[1][1]);
          acc[1][2] = fmaf(t1, ww.z, acc[1][2]); acc[1][3] = fmaf(t1, ww.w, acc[1][3]);
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
          *reinterpret_cast<float4*>(&W2[(a0 + a) * 128 + jb]) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
      }
      __syncthreads();
      // ---- Z[r0:N, :] -= V_b W2 : thread = 8 rows x 4 columns, warp = 8 rows ----
      {
        const int jb = 4 * lane;
        if (jb < Jp) {  // columns >= Jp of Z are zero
          for (int rbase = r0 + 8 * warp; rbase < N; rbase += 8 * (kBtThreads / 32)) {
            float2 acc[8][2];
#pragma unroll
            for (int a = 0; a < 8; ++a) acc[a][0] = acc[a][1] = make_float2(0.f, 0.f);
#pragma unroll 4
            for (int k = 0; k < kNbBt; ++k) {
              const float4 w4 = *reinterpret_cast<const float4*>(&W2[k * 128 + jb]);
              const float2 w01 = make_float2(w4.x, w4.y), w23 = make_float2(w4.z, w4.w);
#pragma unroll
              for (int a = 0; a < 8; ++a) {
                const float v = VbT[(rbase + a) * kVt + k];   // rows >= N: never stored
                acc[a][0] = __ffma2_rn(make_float2(v, v), w01, acc[a][0]);
                acc[a][1] = __ffma2_rn(make_float2(v, v), w23, acc[a][1]);
              }
            }
#pragma unroll
            for (int a = 0; a < 8; ++a) {
              const int r = rbase + a;
              if (r < N) {
                float4 z = *reinterpret_cast<float4*>(&Zs[r * kZld + jb]);
                z.x -= acc[a][0].x; z.y -= acc[a][0].y; z.z -= acc[a][1].x; z.w -= acc[a][1].y;
                *reinterpret_cast<float4*>(&Zs[r * kZld + jb]) = z;
              }
            }
          }
        }
      }
      __syncthreads();
    }
    __syncthreads();
    // ---- Wt[j][r] = w_j U[r][j], transposed through per-warp 32 x 33 smem tiles ----
    {
      float* tile = VbT + warp * 32 * 33;   // V_b^T / W1 / W2 are free now
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
  return sizeof(float) * ((size_t)kMaxNS * kZld + (size_t)kMaxNS * kVt + 2 * kNbBt * 128 + 2 * kNbBt * 33 + 256 + kNbBt);
}

bool bt_supported(int nmax, const Params& p) { return p.pretrd && nmax <= kMaxNS && p.ret <= 128; }

cudaError_t launch_bt(const Prob* dev_probs, int count, const Params& p, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int dyn = (int)bt_smem_bytes();
  static AttrOnce once;
  if (cudaError_t e = once.ensure(bt_kernel, dyn); e != cudaSuccess) return e;
  const int grid = count < kNumSMs ? count : kNumSMs;
  bt_kernel<<<grid, kBtThreads, dyn, s>>>(dev_probs, count, p);
  return cudaGetLastError();
}

}  // namespace fdk
