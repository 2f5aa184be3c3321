// fd_bt_tc.cu — the back-transform of one ReduceRank's eigenvectors on the 5th-gen
// tensor cores: U_J = Q Z_J with Q = H_0 H_1 ... H_{N-3} the Householder reflectors
// of the tridiagonalisation (trd_kernel, fd_trd.cu), then Wt = diag(w) U_J^T, the
// weights of the reconstruct B' = Wt Bf = S'V^T ("B_[i] <- S'V^T", Alg. 1,
// PAPER.md:238; w_j = sigma'_j / sigma_j per the ReduceRank rule).
//
// Compact WY (LAPACK xLARFT 'F','C'): a block of nb = 32 consecutive reflectors is
// Q_b = I - V_b T_b V_b^T (T_b upper triangular), applied from the last block to the
// first: Z <- Z - V_b (T_b (V_b^T Z)).  Both products run as tcgen05.mma kind::tf32
// with the 3xTF32 split (x = hi + lo, hi = tf32_rna(x); a.b ~ hi.hi + hi.lo + lo.hi):
//   W1^T = Z^T V_b      M = 128 (columns j of Z), N = 32, K = rows r in 32-row chunks
//   Z   += V_b (-W2)    M = 128 (rows r, two halves), N = 128 (j), K = 32
// with W2^T = W1^T T_b^T formed in registers (SIMT, 32 x 32 upper triangular).  Z stays
// resident in TMEM as the fp32 accumulator of the second product for the whole
// problem (256 lanes x 128 columns = columns 0..255); each block stages Z^T chunks
// TMEM -> registers -> hi/lo K-major SW128 tiles for the first.  T_b comes from
// S = V_b^T V_b (a third product riding on the W1 chunks) by recursive doubling.
//
// Accuracy: the tensor core's fp32 accumulation truncates (~0.5 ulp per MMA step),
// shrinking the columns of U by ~1e-6; they are renormalised exactly (U is
// orthonormal in exact arithmetic) before the weights are applied, so the
// reconstructed rows carry no systematic shrink.
//
// In:  P.G  = packed reflectors (column i rows i+2..N-1 at pk_off(i,N) + r - i),
//             tau at off = round_up(N(N+1)/2, 4) + 2N, w_j at off + 3N;
//      P.Wt = Z row-major [r][j], ld 128 (normalised eigenvectors of T, 0 if unused).
// Out: P.Wt rows j < J (ld ldg): w_j U[:, j]^T; rows J..ret-1: 0.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fd_internal.h"
#include "fd_tc.cuh"

namespace fdk {

namespace {

constexpr int kBtcThreads = 256;
constexpr int kNb = 32;                    // reflectors per block
constexpr int kTileV = 256 * 128;          // V_b [r][c]: 256 rows x 128 B (K-major for the update, K = c)
constexpr int kTileT = 32 * 128;           // V_b^T chunk [c][r]: 32 rows x 128 B (K-major for W1, K = r)
constexpr int kTileZ = 128 * 128;          // Z^T chunk [j][r]: 128 rows x 128 B
constexpr int kTileW = 128 * 128;          // (-W2)^T [j][c]: 128 rows x 128 B
constexpr int kVfLd = 33;                  // fp32 copy of V_b [r][c] (for S)
constexpr int kUld = 129;                  // final U staging [r][j]
// dynamic shared memory (from a 1024-byte aligned base); every tile is 1024-aligned
constexpr int kOffVh = 0;
constexpr int kOffVl = kOffVh + kTileV;
constexpr int kOffZ = kOffVl + kTileV;                 // [buf 0..1][hi, lo]
constexpr int kOffT = kOffZ + 4 * kTileZ;              // [buf 0..1][hi, lo]
constexpr int kOffWh = kOffT + 4 * kTileT;
constexpr int kOffWl = kOffWh + kTileW;
constexpr int kOffVf = kOffWl + kTileW;
constexpr int kOffS = kOffVf + 256 * kVfLd * 4;        // S (32 x 33), T (32 x 36), Yb (256), tau (32)
constexpr int kSmem = kOffS + (32 * 33 + 32 * 36 + 256 + 32) * 4;
static_assert(256 * kUld * 4 <= kOffVf, "final U staging reuses the tile regions");

__device__ __forceinline__ int pk_off_c(int c, int N) { return c * N - (c * (c - 1)) / 2; }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
      :
      : "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void cta_sync() {
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

}  // namespace

__global__ void __launch_bounds__(kBtcThreads, 1) bt_tc_kernel(const Prob* __restrict__ probs, int count, Params p) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t mbar[2];   // [0]: W1 products, [1]: Z updates
  __shared__ uint32_t s_tmem;
  __shared__ float s_scl[128];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q4 = warp & 3, hw = warp >> 2;     // TMEM lane quarter; row half (Z) / column half
  if (warp == 0) tc::tmem_alloc(&s_tmem, 512);
  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::fence_mbar_init();
  }
  cta_sync();
  const uint32_t tbase = s_tmem;
  const uint32_t lanes = tbase + ((uint32_t)(32 * q4) << 16);
  uint32_t ph0 = 0, ph1 = 0;
  float* Vf = reinterpret_cast<float*>(sm + kOffVf);
  float* S = reinterpret_cast<float*>(sm + kOffS);
  float* Tm = S + 32 * 33;
  float* Yb = Tm + 32 * 36;
  float* tau = Yb + 256;
  const uint32_t idW1 = tc::idesc_tf32(128, 32, 0, 0);
  const uint32_t idUp = tc::idesc_tf32(128, 128, 0, 0);
  const uint32_t smb = tc::smem_u32(sm);

  for (int pi = blockIdx.x; pi < count; pi += gridDim.x) {
    const Prob P = probs[pi];
    const int N = P.rows0 + P.rows1;
    const int J = min(p.ret, N);
    const float* V = static_cast<const float*>(P.G);
    const int offd = (N * (N + 1) / 2 + 3) / 4 * 4;
    const float* taug = V + offd + 2 * N;
    const float* wg = taug + N;
    float* Wt = static_cast<float*>(P.Wt);
    // ---- Z (Wt [r][j], ld 128) -> TMEM: row r = 128 hw + 32 q4 + lane at lane 32 q4 + lane,
    //      columns 128 hw + j ----
    {
      const int r = 128 * hw + 32 * q4 + lane;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 16) {
        float v[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 x = (r < N) ? *reinterpret_cast<const float4*>(Wt + (int64_t)r * 128 + c0 + 4 * q)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
          v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
        }
        tmem_st16(lanes + 128 * hw + c0, v);
      }
      tmem_wait_st();
    }
    cta_sync();
    const int nref = N - 2;
    const int nblk = nref > 0 ? (nref + kNb - 1) / kNb : 0;
    for (int b = nblk - 1; b >= 0; --b) {
      const int i0 = b * kNb, nb = min(kNb, nref - i0), r0 = i0 + 1;
      if (b < nblk - 1) {   // the previous block's Z update read V_b / W2 and wrote D_Z
        tc::mbar_wait(&mbar[1], ph1);
        ph1 ^= 1;
        tc::fence_after_sync();
      }
      // ---- stage V_b: thread = row r (v_{i+1} = 1 implicit, rows <= i zero, tau = 0 -> 0 column) ----
      {
        const int r = tid;
        float v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int i = i0 + c;
          float x = 0.f;
          if (c < nb && r < N && r > i && taug[i] != 0.f) x = (r == i + 1) ? 1.f : V[pk_off_c(i, N) + r - i];
          v[c] = x;
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) Vf[r * kVfLd + c] = v[c];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float4 h, l;
          tc::split_tf32(v[4 * g], h.x, l.x);
          tc::split_tf32(v[4 * g + 1], h.y, l.y);
          tc::split_tf32(v[4 * g + 2], h.z, l.z);
          tc::split_tf32(v[4 * g + 3], h.w, l.w);
          const uint32_t o = tc::sw128_off(r, 4 * g);
          *reinterpret_cast<float4*>(sm + kOffVh + o) = h;
          *reinterpret_cast<float4*>(sm + kOffVl + o) = l;
        }
      }
      if (tid < kNb) {
        const float t = (tid < nb) ? taug[i0 + tid] : 0.f;
        tau[tid] = (t != 0.f) ? t : 1.f;   // zero columns: any nonzero tau
      }
      __syncthreads();
      // ---- W1^T = Z^T V_b and S = V_b^T V_b: 32-row chunks of K staged in pairs (Z^T from
      //      TMEM, V_b^T from Vf); S rides along as an M = 128 product whose A operand is the
      //      32-row V_b^T chunk (rows 32..127 read whatever follows: their outputs are ignored) ----
      const int qa = r0 >> 5, qb = (N - 1) >> 5;
      for (int q0 = qa; q0 <= qb; q0 += 2) {
#pragma unroll 1
        for (int u = 0; u < 2; ++u) {
          const int q = q0 + u;
          if (q > qb) break;
          unsigned char* zh = sm + kOffZ + (2 * u) * kTileZ;
          unsigned char* zl = zh + kTileZ;
          if (q4 == (q & 3)) {   // TMEM rows 32q.. live in lane quarter q % 4, half q / 4
            const int h = q >> 2;
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 16) {
              float z[16];
              tc::tmem_ld16(lanes + 128 * h + 64 * hw + c0, z);
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                float zhv, zlv;
                tc::split_tf32(z[e], zhv, zlv);
                const uint32_t o = tc::sw128_off(64 * hw + c0 + e, lane);   // row j, k = r - 32q
                *reinterpret_cast<float*>(zh + o) = zhv;
                *reinterpret_cast<float*>(zl + o) = zlv;
              }
            }
          } else if (q4 == ((q + 2) & 3)) {   // two other warps: V_b^T chunk [c][r]
            unsigned char* th = sm + kOffT + (2 * u) * kTileT;
            unsigned char* tl = th + kTileT;
#pragma unroll 4
            for (int c = 16 * hw; c < 16 * hw + 16; ++c) {
              float x = Vf[(32 * q + lane) * kVfLd + c], xh, xl;
              tc::split_tf32(x, xh, xl);
              const uint32_t o = tc::sw128_off(c, lane);
              *reinterpret_cast<float*>(th + o) = xh;
              *reinterpret_cast<float*>(tl + o) = xl;
            }
          }
        }
        tc::fence_async_smem();
        cta_sync();
        if (tid == 0) {
          for (int u = 0; u < 2; ++u) {
            const int q = q0 + u;
            if (q > qb) break;
            const uint32_t zh = smb + kOffZ + (2 * u) * kTileZ, zl = zh + kTileZ;
            const uint32_t th = smb + kOffT + (2 * u) * kTileT, tl = th + kTileT;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const uint32_t ko = ks * 32;
              const uint32_t acc = (q > qa || ks > 0) ? 1u : 0u;
              tc::mma_tf32(tbase + 256, tc::desc_k_sw128(zh + ko), tc::desc_k_sw128(th + ko), idW1, acc);
              tc::mma_tf32(tbase + 256, tc::desc_k_sw128(zh + ko), tc::desc_k_sw128(tl + ko), idW1, 1u);
              tc::mma_tf32(tbase + 256, tc::desc_k_sw128(zl + ko), tc::desc_k_sw128(th + ko), idW1, 1u);
              tc::mma_tf32(tbase + 288, tc::desc_k_sw128(th + ko), tc::desc_k_sw128(th + ko), idW1, acc);
              tc::mma_tf32(tbase + 288, tc::desc_k_sw128(th + ko), tc::desc_k_sw128(tl + ko), idW1, 1u);
              tc::mma_tf32(tbase + 288, tc::desc_k_sw128(tl + ko), tc::desc_k_sw128(th + ko), idW1, 1u);
            }
          }
          tc::commit(&mbar[0]);
        }
        tc::mbar_wait(&mbar[0], ph0);   // the staging buffers are reused by the next pair
        ph0 ^= 1;
        tc::fence_after_sync();
      }
      // ---- T = (diag(1/tau) + strict_upper(S))^-1 by recursive doubling (S from TMEM lanes 0..31) ----
      if (warp == 0) {
        float t0[16], t1[16];
        tc::tmem_ld16(lanes + 288, t0);
        tc::tmem_ld16(lanes + 304, t1);
#pragma unroll
        for (int k = 0; k < 16; ++k) { S[lane * 33 + k] = t0[k]; S[lane * 33 + 16 + k] = t1[k]; }
      }
      for (int e = tid; e < 32 * 32; e += kBtcThreads) {
        const int a = e >> 5, c = e & 31;
        Tm[a * 36 + c] = (a == c) ? tau[a] : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int lh = 0; lh < 5; ++lh) {   // off-diagonal block of each 2h x 2h block: -T11 U12 T22
        const int h = 1 << lh, t = tid;
        const bool on = t < 16 * h;
        const int m = t >> (2 * lh), e = t & (h * h - 1), i = e >> lh, j = e & (h - 1);
        const int r1 = 2 * m * h, c2 = r1 + h;
        if (on) {
          float y = 0.f;
          for (int k = 0; k < h; ++k) y = fmaf(S[(r1 + i) * 33 + c2 + k], Tm[(c2 + k) * 36 + c2 + j], y);
          Yb[t] = y;
        }
        __syncthreads();
        if (on) {
          float x = 0.f;
          for (int k = 0; k < h; ++k) x = fmaf(Tm[(r1 + i) * 36 + r1 + k], Yb[(m << (2 * lh)) + k * h + j], x);
          Tm[(r1 + i) * 36 + c2 + j] = -x;
        }
        __syncthreads();
      }
      // ---- (-W2)^T [j][c] = -sum_k T[c][k] W1^T[j][k] (lane j, this warp's 16 columns c) ----
      {
        const int j = 32 * q4 + lane;
        float w1[32];
        {
          float t0[16], t1[16];
          tc::tmem_ld16(lanes + 256, t0);
          tc::tmem_ld16(lanes + 272, t1);
#pragma unroll
          for (int k = 0; k < 16; ++k) { w1[k] = t0[k]; w1[16 + k] = t1[k]; }
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = 16 * hw + 4 * g + e;
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < 32; k += 4) {   // T upper: zeros below; rows are 16-byte aligned (ld 36)
              const float4 t4 = *reinterpret_cast<const float4*>(&Tm[c * 36 + k]);
              acc = fmaf(t4.x, w1[k], acc);
              acc = fmaf(t4.y, w1[k + 1], acc);
              acc = fmaf(t4.z, w1[k + 2], acc);
              acc = fmaf(t4.w, w1[k + 3], acc);
            }
            o[e] = -acc;
          }
          float4 h, l;
          tc::split_tf32(o[0], h.x, l.x);
          tc::split_tf32(o[1], h.y, l.y);
          tc::split_tf32(o[2], h.z, l.z);
          tc::split_tf32(o[3], h.w, l.w);
          const uint32_t off = tc::sw128_off(j, 16 * hw + 4 * g);
          *reinterpret_cast<float4*>(sm + kOffWh + off) = h;
          *reinterpret_cast<float4*>(sm + kOffWl + off) = l;
        }
      }
      tc::fence_async_smem();
      cta_sync();
      // ---- Z[r][j] += sum_c V_b[r][c] (-W2)[c][j]: two 128-row halves ----
      if (tid == 0) {
        const uint32_t wh = smb + kOffWh, wl = smb + kOffWl;
        for (int h = 0; h < 2 && 128 * h < N; ++h) {
          const uint32_t vh = smb + kOffVh + h * 16384, vl = smb + kOffVl + h * 16384;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t ko = ks * 32;
            tc::mma_tf32(tbase + 128 * h, tc::desc_k_sw128(vh + ko), tc::desc_k_sw128(wh + ko), idUp, 1u);
            tc::mma_tf32(tbase + 128 * h, tc::desc_k_sw128(vh + ko), tc::desc_k_sw128(wl + ko), idUp, 1u);
            tc::mma_tf32(tbase + 128 * h, tc::desc_k_sw128(vl + ko), tc::desc_k_sw128(wh + ko), idUp, 1u);
          }
        }
        tc::commit(&mbar[1]);
      }
    }
    if (nblk > 0) {
      tc::mbar_wait(&mbar[1], ph1);
      ph1 ^= 1;
      tc::fence_after_sync();
    }
    __syncthreads();
    // ---- U -> shared [r][j] (ld kUld); exact column norms; Wt[j][r] = w_j U[r][j] / ||U_j|| ----
    float* Us = reinterpret_cast<float*>(sm);
    {
      const int r = 128 * hw + 32 * q4 + lane;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 16) {
        float v[16];
        tc::tmem_ld16(lanes + 128 * hw + c0, v);
#pragma unroll
        for (int e = 0; e < 16; ++e) Us[r * kUld + c0 + e] = v[e];
      }
    }
    __syncthreads();
    if (tid < 128) {
      const int j = tid;
      float sc = 0.f;
      if (j < J) {
        double s2 = 0.0;
        for (int r = 0; r < N; ++r) {
          const double x = Us[r * kUld + j];
          s2 = fma(x, x, s2);
        }
        sc = (s2 > 0.0) ? (float)((double)wg[j] / sqrt(s2)) : 0.f;
      }
      s_scl[j] = sc;
    }
    __syncthreads();
    for (int e = tid; e < J * N; e += kBtcThreads) {
      const int j = e / N, r = e - j * N;
      Wt[(int64_t)j * p.ldg + r] = s_scl[j] * Us[r * kUld + j];
    }
    for (int e = tid; e < (p.ret - J) * N; e += kBtcThreads) {   // rows J..ret-1 (N < ell-1)
      const int j = J + e / N, r = e % N;
      Wt[(int64_t)j * p.ldg + r] = 0.f;
    }
    cta_sync();
  }
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

bool bt_tc_supported(int nmax, const Params& p) { return p.pretrd && nmax <= 256 && p.ret <= 128; }

cudaError_t launch_bt_tc(const Prob* dev_probs, int count, const Params& p, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  constexpr int dyn = kSmem + 1024;
  static AttrOnce once;
  if (cudaError_t e = once.ensure(bt_tc_kernel, dyn); e != cudaSuccess) return e;
  const int grid = count < kNumSMs ? count : kNumSMs;
  bt_tc_kernel<<<grid, kBtcThreads, dyn, s>>>(dev_probs, count, p);
  return cudaGetLastError();
}

}  // namespace fdk
