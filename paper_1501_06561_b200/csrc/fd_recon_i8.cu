// fd_recon_i8.cu — the reconstruct of ReduceRank, "B <- S'V^T" (Alg. 1
// [Sec. 2.3]), as B' = W Bf with W = diag(sigma'/sigma) U^T (ret x N, from eig/bt) and
// Bf the N x d buffer, on the tensor cores with exact integer accumulation.
//
// Why integers: a tf32 (3xTF32) reconstruct accumulates in fp32 with truncation, a
// one-sided bias of ~1e-6 per ReduceRank that compounds through the retained rows
// (c2 ell = 100 cov-err bias 2.1e-3).  Here every product is an int8 x int8
// digit product summed exactly in int32 TMEM accumulators, and the only roundings are the
// round-to-nearest quantisations (zero-mean):
//   W row j:     scaled by 2^(22 - eW_j) (eW_j = frexp exponent of max_k |W_jk|), rounded
//                to |qW| <= 2^22, three balanced base-256 digits (w2 w1 w0);
//   Bf column c: scaled by 2^(30 - eB_c) over the buffer's N rows, |qB| <= 2^30, four
//                digits (b3 b2 b1 b0);
//   sum_k qW qB = 2^40 G5 + 2^32 G4 + 2^24 G3 + 2^16 G2 (+ dropped weights <= 2^8:
//                <= 2^-29 of the largest product), G5 = w2 b3, G4 = w2 b2 + w1 b3,
//                G3 = w2 b1 + w1 b2 + w0 b3, G2 = w2 b0 + w1 b1 + w0 b2 (|G| <= 32768 N).
// Output B'[j][c] = (((G5 2^24 + G4 2^16) + (G3 2^8 + G2)) in fp32) 2^(eW_j + eB_c - 36).
// Relative to the row / column maxima the error is ~2^-22 (W) and ~2^-30 (Bf) per term,
// random in sign; the fp32 SIMT reconstruct rounds each of its N fp32 FMAs instead.
//
// Structure: one persistent CTA per SM (256 threads), problems strided over the grid.
// Per problem W's three digit planes (K-major, SWIZZLE_128B, up to 2 K-atoms of 128
// rows) stay in shared memory; the d columns are processed in tiles of 64: all threads
// load the N x 64 fp32 tile (coalesced rows), reduce the column maxima, write the four
// digit planes of the tile (K-major SW128) into one of two buffers; thread 0 issues the
// 9 int8 MMAs (M = 128, N = 64, K = 32) per K-step into one of two TMEM accumulator
// sets (4 x 64 columns each) and commits; while they run, all 8 warps drain the previous
// tile (warp w: TMEM lanes 32 (w % 4).., columns 32 (w / 4)..) and store it.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fd_internal.h"
#include "fd_tc.cuh"

namespace fdk {

namespace {

constexpr int kRiThreads = 256;
constexpr int kRiNT = 64;                    // columns per tile (MMA N)
constexpr int kRiMaxN = 256;                 // buffer rows (K) supported
constexpr int kRiAtom = 128 * 128;           // one K-atom (128 K-bytes) of a 128-row plane: 16 KB
constexpr int kRiWPlanes = 3, kRiBPlanes = 4;
constexpr int kRiW = kRiWPlanes * 2 * kRiAtom;              // W planes: 96 KB
constexpr int kRiBAtom = kRiNT * 128;                       // one K-atom of a 64-row plane: 8 KB
constexpr int kRiB = kRiBPlanes * 2 * kRiBAtom;             // one B buffer: 64 KB
constexpr int kRiSmem = kRiW + 2 * kRiB + 1024;

__device__ __forceinline__ int frexp_e(float m) {
  if (!(m > 0.f)) return 0;
  int e;
  frexpf(m, &e);
  return e;
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
      :
      : "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// byte offset of K-byte k of row r in a K-major SW128 plane of R rows (2 K-atoms of 128 B)
__device__ __forceinline__ uint32_t ri_off(int r, int k, int atom_bytes) {
  return (uint32_t)((k >> 7) * atom_bytes + r * 128 + ((((k >> 4) & 7) ^ (r & 7)) << 4) + (k & 15));
}

__device__ __forceinline__ const float* prob_row_f(const Prob& P, int r, int64_t ldb) {
  if (r < P.rows0) return P.src0 + (int64_t)r * ldb;
  r -= P.rows0;
  if (r < P.rows1) return P.src1 + (int64_t)r * P.ld1;
  return nullptr;
}

// Balanced base-256 digits by one add and one xor: with u = q + 0x808080, the bytes of
// u ^ 0x808080 are the digits d0, d1, d2 in [-128, 127] (int8) and the signed top digit
// d3 (|q| <= 2^30: |d3| <= 64); for |q| <= 2^22 byte 2 is the signed top digit d2.
__device__ __forceinline__ uint32_t digit_word(float x, float sc) {
  const uint32_t u = (uint32_t)__float2int_rn(x * sc) + 0x808080u;
  return u ^ 0x808080u;
}

// 4 digit words (elements e0..e3) -> plane words: byte p of each element, in order
__device__ __forceinline__ void bytes_t4(uint32_t e0, uint32_t e1, uint32_t e2, uint32_t e3, uint32_t (&pl)[4]) {
  const uint32_t t0 = __byte_perm(e0, e1, 0x5140), t1 = __byte_perm(e2, e3, 0x5140);
  const uint32_t t2 = __byte_perm(e0, e1, 0x7362), t3 = __byte_perm(e2, e3, 0x7362);
  pl[0] = __byte_perm(t0, t1, 0x5410);
  pl[1] = __byte_perm(t0, t1, 0x7632);
  pl[2] = __byte_perm(t2, t3, 0x5410);
  pl[3] = __byte_perm(t2, t3, 0x7632);
}

}  // namespace

__global__ void __launch_bounds__(kRiThreads, 1) recon_i8_kernel(const Prob* __restrict__ probs, int count, Params p) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  unsigned char* wpl = sm;                    // [plane][atom][128 rows x 128 B]
  unsigned char* bpl = sm + kRiW;             // [buffer][plane][atom][64 rows x 128 B]
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t s_tmem;
  __shared__ float s_fw[128];                 // W row factors 2^(eW - 18)
  __shared__ float s_fb[2][kRiNT];            // column factors 2^(eB - 18) of the two B buffers
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tc::tmem_alloc(&s_tmem, 512);
  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = s_tmem;
  const uint32_t idesc = idesc_i8(128, kRiNT);
  uint32_t uses[2] = {0, 0};
  int u = 0;                                   // running tile counter (buffer / accumulator parity)
  const int ntile = (int)((p.ldb + kRiNT - 1) / kRiNT);
  // B tile mapping: thread (column group cg: columns 4cg..4cg+3, row group rg: rows 16rg..16rg+15)
  const int cg = tid >> 4, rg = tid & 15;

  // drain of a tile (problem P, columns n0..): accumulator set b, column factors s_fb[b]
  auto drain = [&](const Prob& P, int n0, int b) {
    tc::mbar_wait(&mbar[b], uses[b] & 1);
    ++uses[b];
    tc::fence_after_sync();
    const int j = 32 * (warp & 3) + lane, ch = warp >> 2;   // row, column half (32 columns)
    const uint32_t la = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * b + 32u * ch;
    const float fw = s_fw[j];
    float* dst = P.dst + (int64_t)j * p.ldb + n0 + 32 * ch;
#pragma unroll 1
    for (int c0 = 0; c0 < 32; c0 += 16) {
      float g5[16], g4[16], g3[16], g2[16];
      tc::tmem_ld16(la + c0, g5);
      tc::tmem_ld16(la + 64 + c0, g4);
      tc::tmem_ld16(la + 128 + c0, g3);
      tc::tmem_ld16(la + 192 + c0, g2);
      float o[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float x = fmaf((float)__float_as_int(g5[q]), 16777216.f, (float)__float_as_int(g4[q]) * 65536.f) +
                        fmaf((float)__float_as_int(g3[q]), 256.f, (float)__float_as_int(g2[q]));
        o[q] = (x * fw) * s_fb[b][32 * ch + c0 + q];
      }
      if (j < p.ell) {
        const int64_t nv = p.ldb - (n0 + 32 * ch + c0);
        if (nv >= 16) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float4*>(dst + c0 + 4 * q) = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (q < nv) dst[c0 + q] = o[q];
        }
      }
    }
  };

  // Bf[16rg .. 16rg+15][n0 + 4cg .. +3] -> registers (0 outside N / ldb)
  auto load_tile = [&](const Prob& P, int N, int n0, float4 (&R)[16]) {
    const int col = n0 + 4 * cg;
    const bool cok = col < p.ldb;              // ldb % 4 == 0: all 4 columns valid or none
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = 16 * rg + i;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (cok && r < N) {
        const float* row = (r < P.rows0) ? P.src0 + (int64_t)r * p.ldb : P.src1 + (int64_t)(r - P.rows0) * P.ld1;
        x = *reinterpret_cast<const float4*>(row + col);
      }
      R[i] = x;
    }
  };

  float4 R[16];
  for (int pi = blockIdx.x; pi < count; pi += gridDim.x) {
    const Prob P = probs[pi];
    const int N = P.rows0 + P.rows1;
    const int nks = (N + 31) / 32;             // K-steps of 32 (zero-padded planes)
    load_tile(P, N, 0, R);
    // ---- W (ret x N, ld ldg) -> three digit planes; 2 threads per row: a max pass,
    //      then a quantising pass over the (L2-resident) row in 16-value chunks ----
    {
      const float* Wt = static_cast<const float*>(P.Wt);
      const int j = tid >> 1, hh = tid & 1;     // row, K half (128 values)
      const bool live = j < p.ret;
      const float* wr = Wt + (int64_t)j * p.ldg + 128 * hh;
      auto ld4 = [&](int k) {                   // 4 values at K index 128 hh + k (0 outside)
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        const int kk = 128 * hh + k;
        if (live && kk < N) x = *reinterpret_cast<const float4*>(wr + k);
        if (kk + 1 >= N) x.y = 0.f;
        if (kk + 2 >= N) x.z = 0.f;
        if (kk + 3 >= N) x.w = 0.f;
        return x;
      };
      float mx = 0.f;
#pragma unroll 8
      for (int q = 0; q < 32; ++q) {
        const float4 x = ld4(4 * q);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      const int ew = frexp_e(mx);
      if (hh == 0) s_fw[j] = ldexpf(1.f, ew - 18);
      const float sc = ldexpf(1.f, 22 - ew);
#pragma unroll 2
      for (int c16 = 0; c16 < 8; ++c16) {      // 16-byte K chunks of this half
        uint32_t w[4][4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const float4 x = ld4(16 * c16 + 4 * g);
          uint32_t pl[4];
          bytes_t4(digit_word(x.x, sc), digit_word(x.y, sc), digit_word(x.z, sc), digit_word(x.w, sc), pl);
#pragma unroll
          for (int q = 0; q < kRiWPlanes; ++q) w[q][g] = pl[q];
        }
        const uint32_t off = ri_off(j, 128 * hh + 16 * c16, kRiAtom);
#pragma unroll
        for (int q = 0; q < kRiWPlanes; ++q)
          *reinterpret_cast<uint4*>(wpl + q * 2 * kRiAtom + off) = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
      }
    }
    // ---- column tiles: quantise tile t (registers R) -> MMAs(t) -> prefetch t + 1 -> drain t - 1 ----
    for (int t = 0; t < ntile; ++t, ++u) {
      const int b = u & 1, n0 = t * kRiNT;
      unsigned char* bb = bpl + b * kRiB;
      {
        float cm[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) cm[c] = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          cm[0] = fmaxf(cm[0], fabsf(R[i].x)); cm[1] = fmaxf(cm[1], fabsf(R[i].y));
          cm[2] = fmaxf(cm[2], fabsf(R[i].z)); cm[3] = fmaxf(cm[3], fabsf(R[i].w));
        }
#pragma unroll
        for (int o = 1; o < 16; o <<= 1)
#pragma unroll
          for (int c = 0; c < 4; ++c) cm[c] = fmaxf(cm[c], __shfl_xor_sync(0xffffffffu, cm[c], o));
        float sc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) sc[c] = ldexpf(1.f, 30 - frexp_e(cm[c]));
        __syncthreads();   // every warp is past the drain of tile u - 2 (its reads of s_fb[b])
        if (rg == 0) {
#pragma unroll
          for (int c = 0; c < 4; ++c) s_fb[b][4 * cg + c] = ldexpf(1.f, frexp_e(cm[c]) - 18);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t w[4][4];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float* v0 = reinterpret_cast<const float*>(&R[4 * g]);
            const float* v1 = reinterpret_cast<const float*>(&R[4 * g + 1]);
            const float* v2 = reinterpret_cast<const float*>(&R[4 * g + 2]);
            const float* v3 = reinterpret_cast<const float*>(&R[4 * g + 3]);
            uint32_t pl[4];
            bytes_t4(digit_word(v0[c], sc[c]), digit_word(v1[c], sc[c]), digit_word(v2[c], sc[c]),
                     digit_word(v3[c], sc[c]), pl);
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q][g] = pl[q];
          }
          const uint32_t off = ri_off(4 * cg + c, 16 * rg, kRiBAtom);
#pragma unroll
          for (int q = 0; q < kRiBPlanes; ++q)
            *reinterpret_cast<uint4*>(bb + q * 2 * kRiBAtom + off) = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
        }
      }
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncthreads();
      tc::fence_after_sync();
      if (tid == 0) {
        const uint32_t wa = tc::smem_u32(wpl), ba = tc::smem_u32(bb);
        const uint32_t tb = tbase + 256u * b;
        for (int s = 0; s < nks; ++s) {
          const uint32_t ko = (uint32_t)((s >> 2) * kRiAtom + (s & 3) * 32);
          const uint32_t kb = (uint32_t)((s >> 2) * kRiBAtom + (s & 3) * 32);
          auto A_ = [&](int q) { return tc::desc_k_sw128(wa + q * 2 * kRiAtom + ko); };
          auto B_ = [&](int q) { return tc::desc_k_sw128(ba + q * 2 * kRiBAtom + kb); };
          const uint32_t a0 = s > 0 ? 1u : 0u;
          mma_i8(tb, A_(2), B_(3), idesc, a0);          // 2^40
          mma_i8(tb + 64, A_(2), B_(2), idesc, a0);     // 2^32
          mma_i8(tb + 64, A_(1), B_(3), idesc, 1u);
          mma_i8(tb + 128, A_(2), B_(1), idesc, a0);    // 2^24
          mma_i8(tb + 128, A_(1), B_(2), idesc, 1u);
          mma_i8(tb + 128, A_(0), B_(3), idesc, 1u);
          mma_i8(tb + 192, A_(2), B_(0), idesc, a0);    // 2^16
          mma_i8(tb + 192, A_(1), B_(1), idesc, 1u);
          mma_i8(tb + 192, A_(0), B_(2), idesc, 1u);
        }
        tc::commit(&mbar[b]);
      }
      __syncwarp();
      if (t + 1 < ntile) load_tile(P, N, n0 + kRiNT, R);   // in flight during the drain
      if (t > 0) drain(P, n0 - kRiNT, b ^ 1);
      tc::fence_before_sync();
    }
    // last tile of this problem (its W planes are overwritten by the next problem)
    drain(P, (ntile - 1) * kRiNT, (u - 1) & 1);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

// Used where it beats the FP32 SIMT reconstruct: its cost is set by the 128-row MMA tile
// and the 256-row quantisation pass, so it needs the retained rows to fill M (c4: ret = 127,
// N = 256: 55 vs 90 ms per pass); at c3 ell = 100 (ret = 99, N = 200) SIMT is faster
// (3.1 vs 3.8 ms), at ell = 50 more so (3.0 vs 3.7 ms).
bool recon_i8_supported(int nmax, const Params& p) {
  return !p.f64 && p.ret >= 112 && p.ret <= 128 && nmax >= 224 && nmax <= kRiMaxN && (p.ldg % 4) == 0 &&
         (p.ldb % 4) == 0;
}

cudaError_t launch_recon_i8(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s) {
  (void)nmax;
  if (count <= 0) return cudaSuccess;
  static AttrOnce once;
  if (cudaError_t e = once.ensure(recon_i8_kernel, kRiSmem); e != cudaSuccess) return e;
  const int grid = count < kNumSMs ? count : kNumSMs;
  recon_i8_kernel<<<grid, kRiThreads, kRiSmem, s>>>(dev_probs, count, p);
  return cudaGetLastError();
}

}  // namespace fdk
