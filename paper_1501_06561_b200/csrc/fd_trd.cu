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
  // resident CTAs per SM (the tail variant runs several problems per SM)
  static constexpr int kMinBlocks = (NM <= 128) ? 3 : 1;
};

constexpr int kTrdTail = 128;   // trailing size handed from the head to the tail stage

// sub-column cc (0..3) of a lane block row
__device__ __forceinline__ float pick4(const float (&x)[4], int cc) {
  return (cc == 0) ? x[0] : (cc == 1) ? x[1] : (cc == 2) ? x[2] : x[3];
}

// SYMV column sums of a lane block: sum over the 8 rows, reduce-scatter over the
// 4 row groups (lanes ^16, ^8); lane (rg, cg) returns column 4cg + rg.  Also the
// lane-local part of x_I^T T x_J (its 8 x 4 block) in dot.
__device__ __forceinline__ float col_sums(const float (&a)[8][4], const float (&vr)[8], const float (&vc)[4],
                                          int lane, float& dot) {
  float cs[4];
  {   // column pairs on packed FFMA2 (the row values as broadcast scalars)
    float2 c01 = make_float2(0.f, 0.f), c23 = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float2 vk = make_float2(vr[k], vr[k]);
      c01 = __ffma2_rn(make_float2(a[k][0], a[k][1]), vk, c01);
      c23 = __ffma2_rn(make_float2(a[k][2], a[k][3]), vk, c23);
    }
    cs[0] = c01.x; cs[1] = c01.y; cs[2] = c23.x; cs[3] = c23.y;
  }
  dot = fmaf(cs[3], vc[3], fmaf(cs[2], vc[2], fmaf(cs[1], vc[1], cs[0] * vc[0])));
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
  const float2 v01 = make_float2(vc[0], vc[1]), v23 = make_float2(vc[2], vc[3]);
#pragma unroll
  for (int k = 0; k < 8; ++k) {   // (a0 v0 + a2 v2) + (a1 v1 + a3 v3): FMUL2 + FFMA2 + FADD
    const float2 x = __ffma2_rn(make_float2(a[k][2], a[k][3]), v23, __fmul2_rn(make_float2(a[k][0], a[k][1]), v01));
    rs[k] = x.x + x.y;
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
// rank-2 update A -= v w^T + w v^T (pending step)
template <bool DIAG>
__device__ __forceinline__ void tile_update(float (&t)[8][4], int r0, int c0, const float* s_v, const float* s_w) {
  const float4 v4 = *reinterpret_cast<const float4*>(s_v + c0), w4 = *reinterpret_cast<const float4*>(s_w + c0);
  const float vc[4] = {v4.x, v4.y, v4.z, v4.w}, wc[4] = {w4.x, w4.y, w4.z, w4.w};
  const float4 va = *reinterpret_cast<const float4*>(s_v + r0), vb = *reinterpret_cast<const float4*>(s_v + r0 + 4);
  const float4 wa = *reinterpret_cast<const float4*>(s_w + r0), wb = *reinterpret_cast<const float4*>(s_w + r0 + 4);
  const float vrs[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
  const float wrs[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float vr = vrs[k], wr = wrs[k];
    if (DIAG) {   // exactly symmetric: round(round(v_r w_c) + round(w_r v_c)), no contraction
#pragma unroll
      for (int c = 0; c < 4; c += 2) {
        const float2 s2 = __fadd2_rn(__fmul2_rn(make_float2(vr, vr), make_float2(wc[c], wc[c + 1])),
                                     __fmul2_rn(make_float2(wr, wr), make_float2(vc[c], vc[c + 1])));
        const float2 x = __fadd2_rn(make_float2(t[k][c], t[k][c + 1]), make_float2(-s2.x, -s2.y));
        t[k][c] = x.x;
        t[k][c + 1] = x.y;
      }
    } else {   // column pairs on packed FFMA2, the row values as broadcast scalars
#pragma unroll
      for (int c = 0; c < 4; c += 2) {
        float2 x = make_float2(t[k][c], t[k][c + 1]);
        x = __ffma2_rn(make_float2(-vr, -vr), make_float2(wc[c], wc[c + 1]), x);
        x = __ffma2_rn(make_float2(-wr, -wr), make_float2(vc[c], vc[c + 1]), x);
        t[k][c] = x.x;
        t[k][c + 1] = x.y;
      }
    }
  }
}

// Staging (mode): the latency-bound steps of a large problem run at one CTA per SM,
// its last kTrdTail steps at several.  mode 0: the whole reduction.  mode 1 (head,
// NM > kTrdTail): steps 0 .. N-kTrdTail-1, then the trailing matrix
// A^(N-kTrdTail-1)[N-kTrdTail:, N-kTrdTail:] (lower triangle, row-major, ld kTrdTail)
// goes to the problem's Wt scratch (free until eig_kernel).  mode 2 (tail,
// NM == kTrdTail): the remaining steps from that matrix (from G when N <= kTrdTail).
// Householder vectors and d / e / tau keep the global (problem) indexing.
template <int NM>
__global__ void __launch_bounds__(TrdCfg<NM>::kThreads, TrdCfg<NM>::kMinBlocks)
trd_kernel(const Prob* __restrict__ probs, int count, Params p, int mode) {
  using C = TrdCfg<NM>;
  constexpr int NB = C::NB, W = C::kWarps;
  extern __shared__ __align__(16) float s_dyn[];    // diagonal tiles (full): s_dg[NB][32][32]
  float (*s_dg)[32][32] = reinterpret_cast<float (*)[32][32]>(s_dyn);
  __shared__ __align__(16) float s_v[NM];      // v of the pending update (step s-1)
  __shared__ __align__(16) float s_w[NM];      // w = p - alpha v of the pending update
  __shared__ __align__(16) float s_x[NM];      // x~_s: column s of A^(s-1), rows >= s+1 (else 0)
  __shared__ __align__(16) float s_nxt[NM];    // look-ahead: column s+1 of A^(s-1)
  __shared__ __align__(16) float s_ctb[NB][NB][32];  // SYMV contributions [block][slot][row]
  __shared__ __align__(16) float s_sq[NM];     // squares of the column entries that enter sigma
  __shared__ __align__(16) float s_xax[(W + 3) / 4 * 4];  // per-warp partials of x^T A x (zero-padded)
  __shared__ float s_d[NM], s_e[NM], s_tau[NM];
  __shared__ float s_corner, s_dlast;          // A[N-1][N-1] (look-ahead / updated)

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
  const int fw = warp - (W - C::kFree);
  const int dT[2] = {fw, fw + C::kFree};
  const int nd = (fw < 0) ? 0 : (fw < NB) + (fw + C::kFree < NB);

  if (tid < (W + 3) / 4 * 4) s_xax[tid] = 0.f;   // padding stays zero
  for (int pi = blockIdx.x; pi < count; pi += gridDim.x) {
    const Prob P = probs[pi];
    const int NG = P.rows0 + P.rows1;            // problem size (global indexing)
    // this launch's steps: global s0 + local 0 .. send-1 on the local N x N matrix
    int s0 = 0, send;
    if (mode == 1) {
      send = NG - kTrdTail;                      // local == global (s0 = 0)
      if (send <= 0) continue;                   // the tail stage does all of it
    } else {
      if (mode == 2) s0 = NG > kTrdTail ? NG - kTrdTail : 0;
      send = NG - s0 - 2;
    }
    const int N = NG - s0;
    float* Vout = static_cast<float*>(P.G);       // packed reflectors + d / e / tau (global)
    const float* G = (s0 > 0) ? static_cast<const float*>(P.Wt) : static_cast<const float*>(P.G);
    const int64_t ldin = (s0 > 0) ? kTrdTail : p.ldg;
    // ---------------- load (zero outside N) ----------------
    float a0[8][4], a1[8][4];
    auto load_blk = [&](int TI, int TJ, float (&t)[8][4]) {
      const int c0 = 32 * TJ + 4 * cg;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = 32 * TI + 8 * rg + k;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < N && c0 < N) x = *reinterpret_cast<const float4*>(G + (int64_t)r * ldin + c0);
        t[k][0] = x.x;
        t[k][1] = (c0 + 1 < N) ? x.y : 0.f;
        t[k][2] = (c0 + 2 < N) ? x.z : 0.f;
        t[k][3] = (c0 + 3 < N) ? x.w : 0.f;
      }
    };
    if (ov[0]) load_blk(oI[0], oJ[0], a0);
    if (ov[1]) load_blk(oI[1], oJ[1], a1);
    _Pragma("unroll") for (int q = 0; q < 2; ++q) {
      if (q >= nd) break;
      load_blk(dT[q], dT[q], a1);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        *reinterpret_cast<float4*>(&s_dg[dT[q]][8 * rg + k][4 * cg]) = make_float4(a1[k][0], a1[k][1], a1[k][2], a1[k][3]);
    }
    // column 0 straight from G (the lower triangle the tiles hold): d_0, x~_0 (rows >= 1)
    // and the partial sums of squares of its rows >= 2, per 32-row block
    if (warp < NB) {
      const int r = tid;
      const float c = (r < N) ? G[(int64_t)r * ldin] : 0.f;
      s_x[r] = (r >= 1) ? c : 0.f;
      if (r == 0) s_d[0] = c;
      s_sq[r] = (r >= 2 && r < N) ? c * c : 0.f;
      s_v[r] = 0.f;
      s_w[r] = 0.f;
      if (r == N - 1) s_dlast = G[(int64_t)r * ldin + r];
    }
    __syncthreads();  // G fully read before V overwrites it
    // diagonal tiles: mirror the lower triangle (the tensor-core Gram is symmetric
    // only up to accumulation order; the symmetric update needs exact symmetry)
    _Pragma("unroll") for (int q = 0; q < 2; ++q) {
      if (q >= nd) break;
      const int D = dT[q];
      for (int e = lane; e < 32 * 32; e += 32) {
        const int r = e >> 5, c = e & 31;
        if (r < c) s_dg[D][r][c] = s_dg[D][c][r];
      }
    }
    __syncthreads();
    const int offd = (NG * (NG + 1) / 2 + 3) / 4 * 4;
    long long t_ph = clock64(), t_st = t_ph;
    const int cn = (N - 1) >> 5, ccn = (N - 1) & 3;

    // Step s: reflector H_s of column s.  Invariant at the top of phase A(s): the
    // tiles hold A^(s-2) with the rank-2 update of step s-1 pending (s_v, s_w);
    // s_x = x~_s = column s of A^(s-1) on rows >= s+1 (else 0); s_sq = the squares of its
    // entries on rows >= s+2 (sigma of the reflector, reduced by the row warps in phase A,
    // off the critical path: the SYMV does not need the reflector).  The Householder x_s
    // differs from x~_s only in row s+1 (alpha - beta instead of alpha): the SYMV
    // runs on x~_s and phase B adds delta * A[:, s+1] (the look-ahead column).
    for (int s = 0; s < send; ++s) {
      const int cs1 = (s + 1) >> 5, cc1 = (s + 1) & 3, cg1 = ((s + 1) & 31) >> 2;
      const bool last = (s == N - 3);
      float tau_s, scale, amb, beta_s, al;
      // ---- phase A: pending update (s-1), reflector s, SYMV y = A^(s-1) x_s,
      //      look-ahead column s+1 of A^(s-1), tile partials of x^T A x ----
      {
        if (s > 0) {
          if (ov[0] && 32 * oJ[0] + 31 > s) tile_update<false>(a0, 32 * oI[0] + 8 * rg, 32 * oJ[0] + 4 * cg, s_v, s_w);
          if (ov[1] && 32 * oJ[1] + 31 > s) tile_update<false>(a1, 32 * oI[1] + 8 * rg, 32 * oJ[1] + 4 * cg, s_v, s_w);
        }
        if (warp < NB) {  // reflector (the row warps of phase B, identical arithmetic)
          float x = 0.f;
#pragma unroll
          for (int t = 0; t < NB; ++t) x += s_sq[32 * t + lane];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          const float sig = x;
          al = s_x[s + 1];
          float beta;
          if (sig == 0.f) {
            tau_s = 0.f; beta = al; scale = 0.f; amb = 0.f;
          } else {
            const float nrm = sqrtf(fmaf(al, al, sig));
            beta = (al <= 0.f) ? nrm : -nrm;
            amb = al - beta;
            tau_s = __fdividef(-amb, beta);
            scale = __fdividef(1.f, amb);
          }
          beta_s = beta;
        }
        float xax = 0.f;
        auto publish_symv = [&](const float (&t)[8][4], int TI, int TJ) {
          const int r0 = 32 * TI + 8 * rg, c0 = 32 * TJ + 4 * cg;
          if (TJ == cs1 && cg == cg1) {
            *reinterpret_cast<float4*>(&s_nxt[r0]) = make_float4(pick4(t[0], cc1), pick4(t[1], cc1), pick4(t[2], cc1), pick4(t[3], cc1));
            *reinterpret_cast<float4*>(&s_nxt[r0 + 4]) = make_float4(pick4(t[4], cc1), pick4(t[5], cc1), pick4(t[6], cc1), pick4(t[7], cc1));
          }
          if (last && TI == cn && TJ == cn && cg == (((N - 1) & 31) >> 2)) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (r0 + k == N - 1) s_corner = pick4(t[k], ccn);
          }
          const float4 ra = *reinterpret_cast<const float4*>(&s_x[r0]);
          const float4 rb = *reinterpret_cast<const float4*>(&s_x[r0 + 4]);
          const float4 cv = *reinterpret_cast<const float4*>(&s_x[c0]);
          const float xr[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
          const float xc[4] = {cv.x, cv.y, cv.z, cv.w};
          float dot;
          s_ctb[TJ][TI][4 * cg + rg] = col_sums(t, xr, xc, lane, dot);
          xax = fmaf(TI != TJ ? 2.f : 1.f, dot, xax);
          if (TI != TJ) s_ctb[TI][TJ][8 * rg + cg] = row_sums(t, xc, lane);
        };
        if (ov[0] && 32 * oJ[0] + 31 > s) publish_symv(a0, oI[0], oJ[0]);
        if (ov[1] && 32 * oJ[1] + 31 > s) publish_symv(a1, oI[1], oJ[1]);
        _Pragma("unroll") for (int q = 0; q < 2; ++q) {
          if (q >= nd) break;
          const int D = dT[q];
          if (32 * D + 31 <= s) continue;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 x = *reinterpret_cast<const float4*>(&s_dg[D][8 * rg + k][4 * cg]);
            a1[k][0] = x.x; a1[k][1] = x.y; a1[k][2] = x.z; a1[k][3] = x.w;
          }
          if (s > 0) {
            tile_update<true>(a1, 32 * D + 8 * rg, 32 * D + 4 * cg, s_v, s_w);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              *reinterpret_cast<float4*>(&s_dg[D][8 * rg + k][4 * cg]) = make_float4(a1[k][0], a1[k][1], a1[k][2], a1[k][3]);
          }
          publish_symv(a1, D, D);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) xax += __shfl_xor_sync(0xffffffffu, xax, o);
        if (lane == 0) s_xax[warp] = xax;
      }
      __syncthreads();
      if (p.dbg && blockIdx.x == 0 && tid == 0) { const long long t_ = clock64(); p.dbg[11] += t_ - t_ph; t_ph = t_; }
      // ---- phase B (a thread per row): p = tau A v, w = p - alpha v with
      //      alpha = (tau/2) p^T v = (tau^2 scale^2 / 2) x^T A x; column s+1 of A^(s) ----
      if (warp < NB) {
        const int r = tid, b = r >> 5, rr = r & 31;
        float yp[NB], y1p[NB];
#pragma unroll
        for (int sl = 0; sl < NB; ++sl) {
          const int tc = sl < b ? sl : b;
          yp[sl] = (r > s && r < N && 32 * tc + 31 > s) ? s_ctb[b][sl][rr] : 0.f;
          const int tc1 = sl < cs1 ? sl : cs1;
          y1p[sl] = (32 * tc1 + 31 > s) ? s_ctb[cs1][sl][(s + 1) & 31] : 0.f;
        }
#pragma unroll
        for (int h = 1; h < NB; h *= 2)
#pragma unroll
          for (int sl = 0; sl + h < NB; sl += 2 * h) { yp[sl] += yp[sl + h]; y1p[sl] += y1p[sl + h]; }
        const float yt = yp[0], yt1 = y1p[0];       // (A x~)_r, (A x~)_{s+1}
        float xp[(W + 3) / 4 * 4];
#pragma unroll
        for (int q = 0; q < (W + 3) / 4; ++q) {
          const float4 t4 = *reinterpret_cast<const float4*>(&s_xax[4 * q]);
          xp[4 * q] = t4.x; xp[4 * q + 1] = t4.y; xp[4 * q + 2] = t4.z; xp[4 * q + 3] = t4.w;
        }
        constexpr int XP = (W + 3) / 4 * 4;
#pragma unroll
        for (int h = 1; h < XP; h *= 2)
#pragma unroll
          for (int q = 0; q + h < XP; q += 2 * h) xp[q] += xp[q + h];
        // x = x~ + delta e_{s+1}:  A x = A x~ + delta A[:, s+1],
        // x^T A x = x~^T A x~ + delta (2 (A x~)_{s+1} + delta A[s+1][s+1])
        const float dl = amb - al;
        const float nx = s_nxt[r], a11 = s_nxt[s + 1];
        const float y = fmaf(dl, nx, yt), y1 = fmaf(dl, a11, yt1);
        const float xax = fmaf(dl, fmaf(dl, a11, 2.f * yt1), xp[0]);
        const float alpha = 0.5f * (tau_s * scale) * (tau_s * scale) * xax;
        const float xt = s_x[r];
        const float vr = (r == s + 1) ? 1.f : ((r >= s + 2 && r < N) ? xt * scale : 0.f);
        const float ts = tau_s * scale;
        const float wr = (r > s && r < N) ? fmaf(-alpha, vr, ts * y) : 0.f;
        const float w1 = fmaf(ts, y1, -alpha);              // w_{s+1} (v_{s+1} = 1)
        const float col = (r >= s + 1 && r < N) ? nx - vr * w1 - wr : 0.f;   // column s+1 of A^(s)
        s_v[r] = vr;
        s_w[r] = wr;
        s_x[r] = (r >= s + 2) ? col : 0.f;
        if (r >= s + 2 && r < N) Vout[pk_off_t(s0 + s, NG) - s + r] = vr;   // Householder vector s0 + s
        if (r == s) { s_e[s] = beta_s; s_tau[s] = tau_s; }
        if (r == s + 1) s_d[s + 1] = col;
        s_sq[r] = (r >= s + 3 && r < N) ? col * col : 0.f;
        if (last && r == N - 1) s_dlast = s_corner - 2.f * vr * wr;
      }
      __syncthreads();
      if (p.dbg && blockIdx.x == 0 && tid == 0) {
        const long long t_ = clock64();
        p.dbg[12] += t_ - t_ph; t_ph = t_; p.dbg[14] += 1;
        p.dbg[20 + min(3, s / 64)] += t_ - t_st; t_st = t_;
      }
    }
    if (mode == 1) {
      // ---------------- head: hand the trailing matrix A^(send-1)[send:, send:] to the tail ----------------
      float* T = static_cast<float*>(P.Wt);
      auto put_blk = [&](const float (&t)[8][4], int TI, int TJ) {   // lower entries r >= c >= send
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int r = 32 * TI + 8 * rg + k;
          if (r < send || r >= N) continue;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int cc = 32 * TJ + 4 * cg + c;
            if (cc >= send && cc <= r) T[(int64_t)(r - send) * kTrdTail + (cc - send)] = t[k][c];
          }
        }
      };
      if (ov[0] && 32 * oJ[0] + 31 >= send) {
        tile_update<false>(a0, 32 * oI[0] + 8 * rg, 32 * oJ[0] + 4 * cg, s_v, s_w);
        put_blk(a0, oI[0], oJ[0]);
      }
      if (ov[1] && 32 * oJ[1] + 31 >= send) {
        tile_update<false>(a1, 32 * oI[1] + 8 * rg, 32 * oJ[1] + 4 * cg, s_v, s_w);
        put_blk(a1, oI[1], oJ[1]);
      }
      _Pragma("unroll") for (int q = 0; q < 2; ++q) {
        if (q >= nd) break;
        const int D = dT[q];
        if (32 * D + 31 < send) continue;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 x = *reinterpret_cast<const float4*>(&s_dg[D][8 * rg + k][4 * cg]);
          a1[k][0] = x.x; a1[k][1] = x.y; a1[k][2] = x.z; a1[k][3] = x.w;
        }
        tile_update<true>(a1, 32 * D + 8 * rg, 32 * D + 4 * cg, s_v, s_w);
        put_blk(a1, D, D);
      }
      for (int r = tid; r < send; r += blockDim.x) {
        Vout[offd + r] = s_d[r];
        Vout[offd + NG + r] = s_e[r];
        Vout[offd + 2 * NG + r] = s_tau[r];
      }
      __syncthreads();
      continue;
    }
    // ---------------- last entries, outputs ----------------
    if (tid == 0) {
      if (N >= 2) {
        s_e[N - 2] = s_x[N - 1];
        s_d[N - 1] = s_dlast;
        s_tau[N - 2] = 0.f;
      }
      s_e[N - 1] = 0.f;
      s_tau[N - 1] = 0.f;
    }
    __syncthreads();
    for (int r = tid; r < N; r += blockDim.x) {
      Vout[offd + s0 + r] = s_d[r];
      Vout[offd + NG + s0 + r] = s_e[r];
      Vout[offd + 2 * NG + s0 + r] = s_tau[r];
    }
    __syncthreads();
  }
}

template <int NM>
static cudaError_t launch_trd_t(const Prob* dev_probs, int count, const Params& p, int mode, cudaStream_t s) {
  constexpr int dyn = TrdCfg<NM>::NB * 32 * 32 * (int)sizeof(float);
  static AttrOnce once;
  if (cudaError_t e = once.ensure(trd_kernel<NM>, dyn); e != cudaSuccess) return e;
  const int slots = kNumSMs * TrdCfg<NM>::kMinBlocks;
  const int grid = count < slots ? count : slots;
  trd_kernel<NM><<<grid, TrdCfg<NM>::kThreads, dyn, s>>>(dev_probs, count, p, mode);
  return cudaGetLastError();
}

bool trd_supported(int nmax, const Params& p) { return !p.f64 && nmax > 32 && nmax <= 256 && p.ret <= 128; }

cudaError_t launch_trd(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (nmax <= 64) return launch_trd_t<64>(dev_probs, count, p, 0, s);
  if (nmax <= kTrdTail) return launch_trd_t<kTrdTail>(dev_probs, count, p, 0, s);
  // head at one CTA per SM, then the last kTrdTail steps of every problem at
  // TrdCfg<kTrdTail>::kMinBlocks CTAs per SM (requires Wt slots of >= kTrdTail^2 floats:
  // wt_rows >= 128 and ldg >= nmax > kTrdTail)
  cudaError_t e = (nmax <= 192) ? launch_trd_t<192>(dev_probs, count, p, 1, s) : launch_trd_t<256>(dev_probs, count, p, 1, s);
  if (e != cudaSuccess) return e;
  return launch_trd_t<kTrdTail>(dev_probs, count, p, 2, s);
}

}  // namespace fdk
