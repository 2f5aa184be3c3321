// fd_trd.cu — register-resident Householder tridiagonalisation of the buffer
// Gram G (fp32), the first stage of the symmetric eigensolve of one ReduceRank
// ("[U,S,V] = svd(B_[i])", Alg. 1; svd via G = B B^T = U S^2 U^T).
//
// Algorithm: LAPACK xSYTD2 order (lower): for i = 0..N-3, the reflector
// H_i = I - tau_i v_i v_i^T annihilates column i below the subdiagonal,
// p = tau A v, w = p - (tau/2)(p^T v) v, A <- A - v w^T - w v^T.
//
// B200 design: the N x N matrix (N <= NM) is tiled in 32 x 32 tiles.  Each of the
// NB(NB-1)/2 strictly-lower tiles (NB = NM/32) lives in the REGISTERS of one warp
// (each lane an 8-row x 4-column block, 32 registers); the NB diagonal tiles live
// in shared memory, two per warp, stored full (both triangles, updated with an
// exactly symmetric formula) so their SYMV contribution is a column sum only.
// NM = 256: 28 + 4 = 32 warps.  Every step is register FMA work: the SYMV
// partials (column sums lane-local over 8 rows + a 2-level shuffle
// reduce-scatter; row sums over 4 columns + a 3-level reduce-scatter) and the
// rank-2 update, with only v / w / p and the partial sums going through shared
// memory.
//
// Output (overwrites the problem's G scratch, which is fully read first):
//   packed Householder vectors V (column-major packed lower, column i rows
//   i+2..N-1 at pk_off(i,N) + r - i; v_{i+1} = 1 implicit), then at
//   off = round_up(N(N+1)/2, 4): d[N], e[N], tau[N].
#include <cuda_runtime.h>
#include <stdint.h>

#include "fd_internal.h"

namespace fdk {

namespace {

__device__ __forceinline__ int pk_off_t(int c, int N) { return c * N - (c * (c - 1)) / 2; }

template <int NM>
struct TrdCfg {
  static constexpr int NB = NM / 32;
  static constexpr int kOff = NB * (NB - 1) / 2;       // strictly-lower tiles (registers)
  static constexpr int kUnits = kOff + NB;
  static constexpr int kW0 = (kUnits + 1) / 2;
  static constexpr int kWarps = kW0 > 16 ? 16 : (kW0 < 2 ? 2 : kW0);
  static constexpr int kThreads = kWarps * 32;
  // warps whose second register block is free hold the diagonal tiles (<= 2 each)
  static constexpr int kFree = (2 * kWarps - kOff) < kWarps ? (2 * kWarps - kOff) : kWarps;
  static_assert(2 * kWarps >= kOff, "not enough register slots");
  static_assert(2 * kFree >= NB, "not enough diagonal slots");
  static_assert(kThreads >= NM, "P4 needs a thread per row");
  static_assert(NB <= 8, "the alpha / sigma reductions assume at most 8 row blocks");
};

// sub-column cc (0..3) of a lane block row
__device__ __forceinline__ float pick4(const float (&x)[4], int cc) {
  return (cc == 0) ? x[0] : (cc == 1) ? x[1] : (cc == 2) ? x[2] : x[3];
}

// SYMV column sums of a lane block: sum over the 8 rows, reduce-scatter over the
// 4 row groups (lanes ^16, ^8); lane (rg, cg) returns column 4cg + rg.
__device__ __forceinline__ float col_sums(const float (&a)[8][4], const float (&vr)[8], int lane) {
  float cs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float vk = vr[k];
#pragma unroll
    for (int c = 0; c < 4; ++c) cs[c] = fmaf(a[k][c], vk, cs[c]);
  }
  const bool hb = (lane >> 4) & 1;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const float snd = hb ? cs[q] : cs[q + 2];
    const float kp = hb ? cs[q + 2] : cs[q];
    cs[q] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
  }
  const bool lb = (lane >> 3) & 1;
  const float snd = lb ? cs[0] : cs[1];
  const float kp = lb ? cs[1] : cs[0];
  return kp + __shfl_xor_sync(0xffffffffu, snd, 8);
}

// SYMV row sums: sum over the 4 columns, reduce-scatter over the 8 column groups
// (lanes ^4, ^2, ^1); lane (rg, cg) returns row 8rg + cg.
__device__ __forceinline__ float row_sums(const float (&a)[8][4], const float (&vc)[4], int lane) {
  float rs[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float x = a[k][0] * vc[0];
    x = fmaf(a[k][1], vc[1], x);
    x = fmaf(a[k][2], vc[2], x);
    x = fmaf(a[k][3], vc[3], x);
    rs[k] = x;
  }
  const bool b2 = (lane >> 2) & 1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float snd = b2 ? rs[q] : rs[q + 4];
    const float kp = b2 ? rs[q + 4] : rs[q];
    rs[q] = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
  }
  const bool b1 = (lane >> 1) & 1;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const float snd = b1 ? rs[q] : rs[q + 2];
    const float kp = b1 ? rs[q + 2] : rs[q];
    rs[q] = kp + __shfl_xor_sync(0xffffffffu, snd, 2);
  }
  const bool b0 = lane & 1;
  const float snd = b0 ? rs[0] : rs[1];
  const float kp = b0 ? rs[1] : rs[0];
  return kp + __shfl_xor_sync(0xffffffffu, snd, 1);
}

}  // namespace

size_t trd_out_floats(int N) { return (size_t)((N * (N + 1) / 2 + 3) / 4 * 4) + 3 * (size_t)N; }

// Per-tile helpers (lane block rows r0..r0+7, cols c0..c0+3).
// rank-2 update A -= v w^T + w v^T with w = p - alpha v (previous step)
template <bool DIAG>
__device__ __forceinline__ void tile_update(float (&t)[8][4], int r0, int c0, float alpha,
                                            const float* s_v, const float* s_p) {
  float vc[4], wc[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) { vc[c] = s_v[c0 + c]; wc[c] = fmaf(-alpha, vc[c], s_p[c0 + c]); }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float vr = s_v[r0 + k], wr = fmaf(-alpha, vr, s_p[r0 + k]);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (DIAG) t[k][c] -= vr * wc[c] + wr * vc[c];   // exactly symmetric
      else t[k][c] = fmaf(-wr, vc[c], fmaf(-vr, wc[c], t[k][c]));
    }
  }
}

template <int NM>
__global__ void __launch_bounds__(TrdCfg<NM>::kThreads, 1)
trd_kernel(const Prob* __restrict__ probs, int count, Params p) {
  using C = TrdCfg<NM>;
  constexpr int NB = C::NB, W = C::kWarps;
  extern __shared__ __align__(16) float s_dyn[];    // diagonal tiles (full): s_dg[NB][32][32]
  float (*s_dg)[32][32] = reinterpret_cast<float (*)[32][32]>(s_dyn);
  __shared__ __align__(16) float s_v[NM];      // v of the previous step (materialised in P4)
  __shared__ __align__(16) float s_p[NM];      // p = tau A v of the previous step
  __shared__ __align__(16) float s_col[NM];    // column i, rows >= i (rows < i of its blocks: 0)
  __shared__ __align__(16) float s_col2[NM];   // column N-1 (final step)
  __shared__ __align__(16) float s_ctb[NB][NB][32];  // SYMV contributions [block][slot][row]
  __shared__ float s_sig[NB];                  // per-block partial sum of squares of column i
  __shared__ float s_apart[NB];                // per-warp partials of p^T v
  __shared__ float s_d[NM], s_e[NM], s_tau[NM];
  __shared__ float s_tprev;                    // tau of the previous step

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rg = lane >> 3, cg = lane & 7;     // lane block: rows 8rg..8rg+7, cols 4cg..4cg+3
  // register tiles: off-diagonal tile t -> warp t (slot 0) / warp t - W (slot 1)
  int oI[2], oJ[2];
  bool ov[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int t = warp + q * W;
    ov[q] = t < C::kOff;
    int J = 0, base = 0;
    if (ov[q]) while (t >= base + (NB - 1 - J)) { base += NB - 1 - J; ++J; }
    oJ[q] = J;
    oI[q] = J + 1 + (t - base);
  }
  // diagonal tiles on the warps with a free second block: D -> warp W - kFree + D % kFree
  int dT[2];
  int nd = 0;
  for (int D = 0; D < NB; ++D)
    if (warp == W - C::kFree + D % C::kFree) dT[nd++] = D;

  for (int pi = blockIdx.x; pi < count; pi += gridDim.x) {
    const Prob P = probs[pi];
    const int N = P.rows0 + P.rows1;
    float* G = static_cast<float*>(P.G);
    // ---------------- load (zero outside N) ----------------
    float a0[8][4], a1[8][4];
    auto load_blk = [&](int TI, int TJ, float (&t)[8][4]) {
      const int c0 = 32 * TJ + 4 * cg;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = 32 * TI + 8 * rg + k;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < N && c0 < N) x = *reinterpret_cast<const float4*>(G + (int64_t)r * p.ldg + c0);
        t[k][0] = x.x;
        t[k][1] = (c0 + 1 < N) ? x.y : 0.f;
        t[k][2] = (c0 + 2 < N) ? x.z : 0.f;
        t[k][3] = (c0 + 3 < N) ? x.w : 0.f;
      }
    };
    if (ov[0]) load_blk(oI[0], oJ[0], a0);
    if (ov[1]) load_blk(oI[1], oJ[1], a1);
    for (int q = 0; q < nd; ++q) {
      load_blk(dT[q], dT[q], a1);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        *reinterpret_cast<float4*>(&s_dg[dT[q]][8 * rg + k][4 * cg]) = make_float4(a1[k][0], a1[k][1], a1[k][2], a1[k][3]);
    }
    for (int r = tid; r < NM; r += blockDim.x) { s_p[r] = 0.f; s_v[r] = 0.f; }
    if (tid < NB) s_apart[tid] = 0.f;
    if (tid == 0) s_tprev = 0.f;
    __syncthreads();  // G fully read before V overwrites it
    // diagonal tiles: mirror the lower triangle (the tensor-core Gram is symmetric
    // only up to accumulation order; the symmetric update needs exact symmetry)
    for (int q = 0; q < nd; ++q) {
      const int D = dT[q];
      for (int e = lane; e < 32 * 32; e += 32) {
        const int r = e >> 5, c = e & 31;
        if (r < c) s_dg[D][r][c] = s_dg[D][c][r];
      }
    }
    __syncthreads();
    float* Vout = G;
    const int offd = (N * (N + 1) / 2 + 3) / 4 * 4;
    long long t_ph = clock64(), t_st = t_ph;

    for (int i = 0; i <= N - 2; ++i) {
      const int ci = i >> 5, cc = i & 3, cgi = (i & 31) >> 2;
      const int cn = (N - 1) >> 5, ccn = (N - 1) & 3, cgn = ((N - 1) & 31) >> 2;
      const bool last = (i == N - 2);
      // ---- P1: pending rank-2 update of step i-1, publish column i ----
      {
        float alpha = 0.f;
        if (i > 0) {
          // NB <= 8 partials: every group of 8 lanes reduces its own copy (3 levels)
          float x = ((lane & 7) < NB) ? s_apart[lane & 7] : 0.f;
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          alpha = 0.5f * s_tprev * x;
        }
        // publication of column i (rows >= i; rows < i -> 0) + partial sum of squares (rows >= i+2)
        auto publish = [&](const float (&t)[8][4], int TI, int TJ) {
          const int r0 = 32 * TI + 8 * rg;
          if (TJ == ci) {
            float sq = 0.f;
            if (cg == cgi) {
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float x = pick4(t[k], cc);
                const int r = r0 + k;
                s_col[r] = (r >= i) ? x : 0.f;
                if (r >= i + 2) sq = fmaf(x, x, sq);
              }
            }
            sq += __shfl_xor_sync(0xffffffffu, sq, 8);
            sq += __shfl_xor_sync(0xffffffffu, sq, 16);
            if (lane == cgi) s_sig[TI] = sq;
          }
          if (last && TJ == cn && cg == cgn) {
#pragma unroll
            for (int k = 0; k < 8; ++k) s_col2[r0 + k] = pick4(t[k], ccn);
          }
        };
        if (ov[0] && 32 * oJ[0] + 31 >= i) {
          if (i > 0) tile_update<false>(a0, 32 * oI[0] + 8 * rg, 32 * oJ[0] + 4 * cg, alpha, s_v, s_p);
          publish(a0, oI[0], oJ[0]);
        }
        if (ov[1] && 32 * oJ[1] + 31 >= i) {
          if (i > 0) tile_update<false>(a1, 32 * oI[1] + 8 * rg, 32 * oJ[1] + 4 * cg, alpha, s_v, s_p);
          publish(a1, oI[1], oJ[1]);
        }
        for (int q = 0; q < nd; ++q) {
          const int D = dT[q];
          if (32 * D + 31 < i) continue;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 x = *reinterpret_cast<const float4*>(&s_dg[D][8 * rg + k][4 * cg]);
            a1[k][0] = x.x; a1[k][1] = x.y; a1[k][2] = x.z; a1[k][3] = x.w;
          }
          if (i > 0) {
            tile_update<true>(a1, 32 * D + 8 * rg, 32 * D + 4 * cg, alpha, s_v, s_p);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              *reinterpret_cast<float4*>(&s_dg[D][8 * rg + k][4 * cg]) = make_float4(a1[k][0], a1[k][1], a1[k][2], a1[k][3]);
          }
          publish(a1, D, D);
        }
      }
      __syncthreads();
      if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[11] += t_ - t_ph; t_ph = t_; }
      if (last) break;
      // ---- P3: the reflector of column i (every warp, identical arithmetic); SYMV of the
      //      unscaled x (x_r = col_r for r >= i+2, x_{i+1} = alpha - beta, v = x * scale) ----
      float tau_i, scale, amb;
      {
        float x = ((lane & 7) >= ci && (lane & 7) < NB) ? s_sig[lane & 7] : 0.f;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        const float sig = x;
        const float al = s_col[i + 1];
        float beta;
        if (sig == 0.f) {
          tau_i = 0.f; beta = al; scale = 0.f; amb = 0.f;
        } else {
          const float nrm = sqrtf(fmaf(al, al, sig));
          beta = (al <= 0.f) ? nrm : -nrm;
          amb = al - beta;
          tau_i = __fdividef(-amb, beta);
          scale = __fdividef(1.f, amb);
        }
        if (warp == W - 1) {  // output of the reflector (off the critical path)
          const int base = pk_off_t(i, N) - i;
          for (int r = i + 2 + lane; r < N; r += 32) Vout[base + r] = s_col[r] * scale;
          if (lane == 0) { s_d[i] = s_col[i]; s_e[i] = beta; s_tau[i] = tau_i; }
        }
      }
      auto symv = [&](const float (&t)[8][4], int TI, int TJ) {
        const int r0 = 32 * TI + 8 * rg, c0 = 32 * TJ + 4 * cg;
        float xr[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int r = r0 + k;
          const float x = s_col[r];
          xr[k] = (r == i + 1) ? amb : ((r == i) ? 0.f : x);
        }
        s_ctb[TJ][TI][4 * cg + rg] = col_sums(t, xr, lane);
        if (TI != TJ) {
          float xc[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int r = c0 + c;
            const float x = s_col[r];
            xc[c] = (r == i + 1) ? amb : ((r == i) ? 0.f : x);
          }
          s_ctb[TI][TJ][8 * rg + cg] = row_sums(t, xc, lane);
        }
      };
      if (ov[0] && 32 * oJ[0] + 31 > i) symv(a0, oI[0], oJ[0]);
      if (ov[1] && 32 * oJ[1] + 31 > i) symv(a1, oI[1], oJ[1]);
      for (int q = 0; q < nd; ++q) {
        const int D = dT[q];
        if (32 * D + 31 <= i) continue;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 x = *reinterpret_cast<const float4*>(&s_dg[D][8 * rg + k][4 * cg]);
          a1[k][0] = x.x; a1[k][1] = x.y; a1[k][2] = x.z; a1[k][3] = x.w;
        }
        symv(a1, D, D);
      }
      __syncthreads();
      if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[12] += t_ - t_ph; t_ph = t_; }
      // ---- P4 (warps owning rows): y = scale * (A x), p = tau y (rows > i), v = scale x ----
      if (warp < NB) {
        const int r = tid;
        float y = 0.f;
        const int b = r >> 5, rr = r & 31;
        if (r > i && r < N) {
#pragma unroll
          for (int sl = 0; sl < NB; ++sl) {
            const int tc = sl < b ? sl : b;
            if (32 * tc + 31 > i) y += s_ctb[b][sl][rr];
          }
        }
        const float x = (b >= ci) ? s_col[r] : 0.f;
        const float vr = (r == i + 1) ? 1.f : ((r >= i + 2 && r < N) ? x * scale : 0.f);
        const float pr = tau_i * scale * y;
        s_p[r] = pr;
        s_v[r] = vr;
        float pv = pr * vr;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
        if (lane == 0) s_apart[warp] = pv;
        if (tid == 0) s_tprev = tau_i;
      }
      __syncthreads();
      if (p.dbg && blockIdx.x == 0 && tid == 0) {
        const long long t_ = clock64();
        p.dbg[13] += t_ - t_ph; t_ph = t_; p.dbg[14] += 1;
        p.dbg[20 + min(3, i / 64)] += t_ - t_st; t_st = t_;
      }
    }
    // ---------------- last entries, outputs ----------------
    if (tid == 0) {
      if (N >= 2) {
        s_d[N - 2] = s_col[N - 2];
        s_e[N - 2] = s_col[N - 1];
        s_d[N - 1] = s_col2[N - 1];
        s_tau[N - 2] = 0.f;
      }
      s_e[N - 1] = 0.f;
      s_tau[N - 1] = 0.f;
    }
    __syncthreads();
    for (int r = tid; r < N; r += blockDim.x) {
      Vout[offd + r] = s_d[r];
      Vout[offd + N + r] = s_e[r];
      Vout[offd + 2 * N + r] = s_tau[r];
    }
    __syncthreads();
  }
}

template <int NM>
static cudaError_t launch_trd_t(const Prob* dev_probs, int count, const Params& p, cudaStream_t s) {
  constexpr int dyn = TrdCfg<NM>::NB * 32 * 32 * (int)sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(trd_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = count < kNumSMs ? count : kNumSMs;
  trd_kernel<NM><<<grid, TrdCfg<NM>::kThreads, dyn, s>>>(dev_probs, count, p);
  return cudaGetLastError();
}

bool trd_supported(int nmax, const Params& p) { return !p.f64 && nmax > 32 && nmax <= 256 && p.ell - 1 <= 128; }

cudaError_t launch_trd(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (nmax <= 64) return launch_trd_t<64>(dev_probs, count, p, s);
  if (nmax <= 128) return launch_trd_t<128>(dev_probs, count, p, s);
  if (nmax <= 192) return launch_trd_t<192>(dev_probs, count, p, s);
  return launch_trd_t<256>(dev_probs, count, p, s);
}

}  // namespace fdk
