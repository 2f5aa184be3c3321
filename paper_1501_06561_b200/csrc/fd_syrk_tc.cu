// fd_syrk_tc.cu — the evaluator's A^T A (cov-err M = A^T A - B^T B, PAPER.md:57
// [Sec. 1], 570-571 [Sec. 4]; proj-err) on the tensor cores:
// tcgen05.mma kind::i8 with exact int32 accumulation on fixed-point slices of A.
//
// Numerics (reading E3).  Rows are processed in chunks; inside a chunk
// column j of A is scaled by 2^(30 - e_j) (e_j: frexp exponent of max_i |a_ij| over the
// chunk) and rounded to an integer q_ij, |q| <= 2^30.  q is split exactly into balanced
// base-256 digits q = d3 2^24 + d2 2^16 + d1 2^8 + d0 (d0..d2 in [-128, 127], |d3| <= 64),
// and q_i q_j is summed as the digit products of weight 2^48 ... 2^16:
//   G6 = d3 d3,  G5 = d3 d2 + d2 d3,  G4 = d3 d1 + d2 d2 + d1 d3,
//   G3 = d3 d0 + d2 d1 + d1 d2 + d0 d3,  G2 = d2 d0 + d1 d1 + d0 d2
// (the dropped weights 2^8, 2^0 are <= 2^23 + 2^14 in q^2 units, 2^-37 of the product,
// and the one with a sign bias, d0 d0 >= 0, is 2^-46).  G2 must stay: its d1 d1 >= 0
// biased the diagonal (||A||_F^2) by ~5e-9 relative when dropped.  Per row and entry the
// error is <= ~2^-29 cmax_i cmax_j (the rounding of q), zero-mean.  Each weight is one
// int32 TMEM accumulator of a 128 x 64 tile (5 x 64 columns) fed by 1-4 int8 MMAs; int32
// sums are exact while a CTA accumulates at most kMaxKb K-blocks of 64 rows (|G2|, |G3|
// <= 49152 per row, 49152 * 680 * 64 < 2^31).  The drain forms
// (G6 2^48 + G5 2^40 + G4 2^32 + G3 2^24 + G2 2^16) 2^(e_i + e_j - 60) in fp64 and adds
// it to the CTA's own fp64 partial tile; partials are summed in split order at the end.
//
// Kernels per row chunk: colmax (max |a| per column, non-finite flag) -> quantise
// (fp32 -> four int8 digit planes, written as the UMMA K-major SWIZZLE_64B smem image of
// each (64-row K-block, 128-column block): one 32 KB bulk copy per operand per K-block) ->
// syrk_i8 (one CTA per (128 x 64 tile of the lower block triangle, K split);
// cp.async.bulk producer thread, single-thread MMA issue, 4-stage mbarrier pipeline,
// TMEM drain by warps 0-3).  Then one finish kernel: AtA += sum over splits (both
// triangles).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fd_internal.h"
#include "fd_tc.cuh"

namespace fdk {

namespace {

constexpr int kQB = 128;                 // columns per column block (tile edge)
constexpr int kKB = 64;                  // rows per K-block (64 int8 = one SWIZZLE_64B row)
constexpr int kND = 4;                   // digit planes
constexpr int kPlaneBytes = kQB * kKB;   // one digit plane of a (K-block, column block): 8 KB
constexpr int kBlkBytes = kND * kPlaneBytes;
constexpr int kStages = 4;
constexpr int kTN = 64;                  // tile columns (N of the MMA)
constexpr int kNG = 5;                   // accumulators (weights 2^48 .. 2^16)
constexpr int kMaxKb = 680;              // K-blocks per CTA between drains (int32 exactness)
constexpr int kSyThreads = 128;
constexpr int kSyTargetCtas = 148;

__device__ __forceinline__ int e_of_max(uint32_t bits) {   // max |a| = f 2^e, f in [0.5, 1)
  if (bits == 0u) return 0;
  int e;
  frexpf(__uint_as_float(bits), &e);
  return e;
}

__global__ void __launch_bounds__(256) colmax_kernel(const float* __restrict__ A, int64_t nr, int64_t ld, int64_t d,
                                                     uint32_t* __restrict__ cmax, int* __restrict__ nanflag) {
  const int64_t c = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  uint32_t m = 0u;
  bool bad = false;
  if (c < d) {
    for (int64_t r = (int64_t)blockIdx.y * 8 + (threadIdx.x >> 5); r < nr; r += (int64_t)gridDim.y * 8) {
      const float x = __ldcs(A + r * ld + c);
      bad |= !isfinite(x);
      const uint32_t b = __float_as_uint(fabsf(x));
      m = (b > m && isfinite(x)) ? b : m;
    }
  }
  __shared__ uint32_t s_m[8][32];
  s_m[threadIdx.x >> 5][threadIdx.x & 31] = m;
  bad = __syncthreads_or(bad);
  if (threadIdx.x < 32 && c < d) {
    uint32_t t = 0u;
#pragma unroll
    for (int w = 0; w < 8; ++w) t = max(t, s_m[w][threadIdx.x]);
    atomicMax(cmax + c, t);
  }
  if (bad && threadIdx.x == 0) atomicOr(nanflag, 1);
}

// one CTA per (64-row K-block kb, column block cb) -> 4 digit planes of the K-major
// SWIZZLE_64B image: row m (= column cb*128 + m of A) at byte m*64, its 16-byte chunk c
// (rows 16c..16c+15 of the K-block) at position c ^ ((m >> 1) & 3)
__global__ void __launch_bounds__(256) quant_kernel(const float* __restrict__ A, int64_t nr, int64_t ld, int64_t d,
                                                    const uint32_t* __restrict__ cmax, int ncb,
                                                    unsigned char* __restrict__ planes) {
  __shared__ float s_t[kKB][kQB + 1];
  __shared__ float s_sc[kQB];
  const int kb = blockIdx.x, cb = blockIdx.y, tid = threadIdx.x;
  const int64_t r0 = (int64_t)kb * kKB, c0 = (int64_t)cb * kQB;
  if (tid < kQB) {
    const int64_t c = c0 + tid;
    s_sc[tid] = (c < d) ? ldexpf(1.0f, 30 - e_of_max(cmax[c])) : 0.f;
  }
  // load: 32 lanes x float4 along a row (128 columns), 8 rows per pass
  const bool vec = ((ld & 3) == 0) && (c0 + kQB <= d);
  for (int rr = tid >> 5; rr < kKB; rr += 8) {
    const int64_t r = r0 + rr;
    const int cc = 4 * (tid & 31);
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < nr) {
      const float* src = A + r * ld + c0 + cc;
      if (vec) {
        x = __ldcs(reinterpret_cast<const float4*>(src));
      } else {
        if (c0 + cc < d) x.x = src[0];
        if (c0 + cc + 1 < d) x.y = src[1];
        if (c0 + cc + 2 < d) x.z = src[2];
        if (c0 + cc + 3 < d) x.w = src[3];
      }
    }
    s_t[rr][cc] = x.x; s_t[rr][cc + 1] = x.y; s_t[rr][cc + 2] = x.z; s_t[rr][cc + 3] = x.w;
  }
  __syncthreads();
  unsigned char* dst = planes + ((size_t)kb * ncb + cb) * kBlkBytes;
  for (int u = tid; u < kQB * 4; u += 256) {   // (m, 16-row chunk kc)
    const int m = u >> 2, kc = u & 3;
    const float sc = s_sc[m];
    uint32_t w[kND][4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint32_t b[kND] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float a = s_t[16 * kc + 4 * g + e][m];
        int q = __float2int_rn(a * sc);          // exact power-of-two scaling, |q| <= 2^30
#pragma unroll
        for (int p = 0; p < kND - 1; ++p) {
          const int dg = (int)(int8_t)(q & 0xff);
          b[p] |= (uint32_t)(dg & 0xff) << (8 * e);
          q = (q - dg) >> 8;
        }
        b[kND - 1] |= (uint32_t)(q & 0xff) << (8 * e);   // |d3| <= 64
      }
#pragma unroll
      for (int p = 0; p < kND; ++p) w[p][g] = b[p];
    }
    const uint32_t off = (uint32_t)m * 64u + ((uint32_t)((kc ^ (m >> 1)) & 3) << 4);
#pragma unroll
    for (int p = 0; p < kND; ++p)
      *reinterpret_cast<uint4*>(dst + p * kPlaneBytes + off) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
  }
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_64B (8-row atoms of 64-byte rows, SBO = 512 B)
__device__ __forceinline__ uint64_t desc_k_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;   // SWIZZLE_64B
  return d;
}

__device__ __forceinline__ uint32_t idesc_i8(int M, int N) {
  uint32_t d = 0;
  d |= 2u << 4;    // c_format = S32
  d |= 1u << 7;    // a_format = signed int8
  d |= 1u << 10;   // b_format = signed int8
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
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

__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :
               : "r"(tc::smem_u32(mbar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :
      : "r"(tc::smem_u32(dst)), "l"(src), "r"(bytes), "r"(tc::smem_u32(mbar))
      : "memory");
}

struct SyrkGeo {
  int ncb, ntiles, nsplit, nkb;   // 128-column blocks, 128 x 64 tiles, K splits, K-blocks of the chunk
};

// tile t -> (I, J): rows = 128-column block I, cols = 64-column block J <= 2I + 1
__device__ __forceinline__ void tile_ij(int t, int& I, int& J) {
  I = 0;
  while ((I + 1) * (I + 2) <= t) ++I;
  J = t - I * (I + 1);
}

__global__ void __launch_bounds__(kSyThreads, 1) syrk_i8_kernel(const unsigned char* __restrict__ planes, SyrkGeo g,
                                                                const uint32_t* __restrict__ cmax, int64_t d,
                                                                double* __restrict__ part) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], done;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = blockIdx.x / g.nsplit, sp = blockIdx.x % g.nsplit;
  int I, J;
  tile_ij(t, I, J);
  const int Jb = J >> 1, Jh = J & 1;           // 128-column block holding the tile's columns, half
  const bool diag = (Jb == I);                 // B rows are rows of the A block: no second copy
  const int per = (g.nkb + g.nsplit - 1) / g.nsplit;
  const int kb0 = sp * per, kb1 = min(g.nkb, kb0 + per);
  const int nk = kb1 - kb0;
  if (warp == 0) tc::tmem_alloc(&s_tmem, 512);
  if (tid == 0) {
    for (int q = 0; q < kStages; ++q) { tc::mbar_init(&full[q], 1); tc::mbar_init(&empty[q], 1); }
    tc::mbar_init(&done, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = s_tmem;
  constexpr int kHalf = kTN * kKB;             // 4 KB: rows 64h.. of a plane
  constexpr int kStage = kBlkBytes + kND * kHalf;   // A block (32 KB) + B half planes (16 KB)
  const uint32_t bytes = diag ? kBlkBytes : kStage;
  auto stA = [&](int q) { return sm + (size_t)q * kStage; };
  auto src = [&](int kb, int cb) { return planes + ((size_t)kb * g.ncb + cb) * kBlkBytes; };
  if (nk > 0) {
    if (warp == 0 && lane == 0) {
      // producer: stage q = k % kStages, refilled once the MMAs of K-block k - kStages committed
      for (int k = 0; k < nk; ++k) {
        const int q = k % kStages;
        if (k >= kStages) tc::mbar_wait(&empty[q], ((k - kStages) / kStages) & 1);
        mbar_expect_tx(&full[q], bytes);
        bulk_g2s(stA(q), src(kb0 + k, I), kBlkBytes, &full[q]);
        if (!diag) {
          const unsigned char* sb = src(kb0 + k, Jb) + Jh * kHalf;
#pragma unroll
          for (int p = 0; p < kND; ++p) bulk_g2s(stA(q) + kBlkBytes + p * kHalf, sb + p * kPlaneBytes, kHalf, &full[q]);
        }
      }
    } else if (warp == 1 && lane == 0) {
      const uint32_t id = idesc_i8(128, kTN);
      for (int k = 0; k < nk; ++k) {
        const int q = k % kStages;
        tc::mbar_wait(&full[q], (k / kStages) & 1);
        tc::fence_after_sync();
        const uint32_t a = tc::smem_u32(stA(q));
        const uint32_t b = diag ? a + Jh * kHalf : a + kBlkBytes;
        const uint32_t bstride = diag ? kPlaneBytes : kHalf;
#pragma unroll
        for (int ks = 0; ks < kKB / 32; ++ks) {
          const uint32_t ko = ks * 32, acc = (k > 0 || ks > 0) ? 1u : 0u;
          auto A_ = [&](int p) { return desc_k_sw64(a + p * kPlaneBytes + ko); };
          auto B_ = [&](int p) { return desc_k_sw64(b + p * bstride + ko); };
          mma_i8(tbase, A_(3), B_(3), id, acc);                 // 2^48
          mma_i8(tbase + 64, A_(3), B_(2), id, acc);            // 2^40
          mma_i8(tbase + 64, A_(2), B_(3), id, 1u);
          mma_i8(tbase + 128, A_(3), B_(1), id, acc);           // 2^32
          mma_i8(tbase + 128, A_(2), B_(2), id, 1u);
          mma_i8(tbase + 128, A_(1), B_(3), id, 1u);
          mma_i8(tbase + 192, A_(3), B_(0), id, acc);           // 2^24
          mma_i8(tbase + 192, A_(2), B_(1), id, 1u);
          mma_i8(tbase + 192, A_(1), B_(2), id, 1u);
          mma_i8(tbase + 192, A_(0), B_(3), id, 1u);
          mma_i8(tbase + 256, A_(2), B_(0), id, acc);           // 2^16
          mma_i8(tbase + 256, A_(1), B_(1), id, 1u);
          mma_i8(tbase + 256, A_(0), B_(2), id, 1u);
        }
        tc::commit(&empty[q]);
      }
      tc::commit(&done);
    }
    __syncwarp();
    tc::mbar_wait(&done, 0);
    tc::fence_after_sync();
    // drain: warp w holds TMEM lanes 32w.. = tile rows (columns I*128 + m of A)
    const int m = 32 * warp + lane;
    const int64_t gi = (int64_t)I * kQB + m;
    const int ei = (gi < d) ? e_of_max(cmax[gi]) - 30 : 0;
    double* pt = part + ((size_t)t * g.nsplit + sp) * (kQB * kTN) + (size_t)m * kTN;
    const uint32_t lanebase = tbase + ((uint32_t)(32 * warp) << 16);
    for (int c0 = 0; c0 < kTN; c0 += 16) {
      float v[kNG][16];
#pragma unroll
      for (int gg = 0; gg < kNG; ++gg) tc::tmem_ld16(lanebase + 64 * gg + c0, v[gg]);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int64_t gj = (int64_t)J * kTN + c0 + q;
        const int ej = (gj < d) ? e_of_max(cmax[gj]) - 30 : 0;
        const double x = ((((double)__float_as_int(v[0][q]) * 281474976710656.0 +     // 2^48
                            (double)__float_as_int(v[1][q]) * 1099511627776.0) +      // 2^40
                           (double)__float_as_int(v[2][q]) * 4294967296.0) +          // 2^32
                          (double)__float_as_int(v[3][q]) * 16777216.0) +             // 2^24
                         (double)__float_as_int(v[4][q]) * 65536.0;                   // 2^16
        pt[c0 + q] += ldexp(x, ei + ej);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

// AtA[i][j] (+)= sum over splits of part[tile][split][m][n], lower entries j <= i, mirrored
__global__ void syrk_i8_finish_kernel(const double* __restrict__ part, SyrkGeo g, int64_t d, double* __restrict__ AtA,
                                      const int* __restrict__ nanflag) {
  int I, J;
  tile_ij(blockIdx.x, I, J);
  const bool bad = *nanflag != 0;
  for (int e = threadIdx.x; e < kQB * kTN; e += blockDim.x) {
    const int m = e / kTN, n = e % kTN;
    const int64_t i = (int64_t)I * kQB + m, j = (int64_t)J * kTN + n;
    if (i >= d || j >= d || j > i) continue;
    double s = 0.0;
    for (int sp = 0; sp < g.nsplit; ++sp) s += part[((size_t)blockIdx.x * g.nsplit + sp) * (kQB * kTN) + e];
    if (bad) s = __longlong_as_double(0x7ff8000000000000ll);
    AtA[i * d + j] += s;
    if (i != j) AtA[j * d + i] += s;
  }
}

SyrkGeo syrk_geo(int64_t d, int64_t nrows) {
  SyrkGeo g{};
  g.ncb = (int)((d + kQB - 1) / kQB);
  g.ntiles = g.ncb * (g.ncb + 1);              // sum over I of 2(I + 1)
  g.nsplit = kSyTargetCtas / g.ntiles;
  if (g.nsplit < 1) g.nsplit = 1;
  g.nkb = (int)((nrows + kKB - 1) / kKB);
  return g;
}

// rows per chunk (a multiple of kKB): every CTA accumulates <= kMaxKb K-blocks, and the
// digit planes of a chunk stay under kPlaneCap bytes
constexpr int64_t kPlaneCap = (int64_t)512 << 20;
int64_t syrk_chunk_rows(int64_t d) {
  const SyrkGeo g = syrk_geo(d, 0);
  const int64_t by_k = (int64_t)g.nsplit * kMaxKb * kKB;
  int64_t by_mem = kPlaneCap / ((int64_t)g.ncb * kND * kQB) / kKB * kKB;   // kND * kQB bytes per row
  if (by_mem < kKB) by_mem = kKB;
  return by_k < by_mem ? by_k : by_mem;
}

}  // namespace

size_t syrk_tc_workspace_bytes(int64_t n, int64_t d) {
  const int64_t rows = n < syrk_chunk_rows(d) ? n : syrk_chunk_rows(d);
  const SyrkGeo g = syrk_geo(d, rows);
  size_t b = (size_t)g.nkb * g.ncb * kBlkBytes;                          // digit planes of one chunk
  b = (b + 255) / 256 * 256 + (size_t)g.ntiles * g.nsplit * kQB * kTN * sizeof(double);   // partial tiles
  b = (b + 255) / 256 * 256 + (size_t)g.ncb * kQB * sizeof(uint32_t) + 256;             // column maxima + flag
  return b;
}

cudaError_t launch_syrk_tc(const float* A, int64_t n, int64_t ld, int64_t d, double* AtA, void* ws, size_t ws_bytes,
                           cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (ws_bytes < syrk_tc_workspace_bytes(n, d)) return cudaErrorInvalidValue;
  const int64_t crows = syrk_chunk_rows(d);
  const SyrkGeo gmax = syrk_geo(d, n < crows ? n : crows);
  unsigned char* planes = static_cast<unsigned char*>(ws);
  size_t off = ((size_t)gmax.nkb * gmax.ncb * kBlkBytes + 255) / 256 * 256;
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + off);
  const size_t part_bytes = (size_t)gmax.ntiles * gmax.nsplit * kQB * kTN * sizeof(double);
  off = (off + part_bytes + 255) / 256 * 256;
  uint32_t* cmax = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + off);
  int* nanflag = reinterpret_cast<int*>(cmax + gmax.ncb * kQB);
  static AttrOnce once;
  const int smem = kStages * (kBlkBytes + kND * kTN * kKB) + 1024;
  if (cudaError_t e = once.ensure(syrk_i8_kernel, smem); e != cudaSuccess) return e;
  cudaError_t e = cudaMemsetAsync(part, 0, part_bytes, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(nanflag, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  for (int64_t r0 = 0; r0 < n; r0 += crows) {
    const int64_t nr = (n - r0) < crows ? (n - r0) : crows;
    SyrkGeo g = syrk_geo(d, nr);
    g.nsplit = gmax.nsplit;   // partial layout (tile, split) is fixed across chunks
    const float* Ac = A + r0 * ld;
    e = cudaMemsetAsync(cmax, 0, (size_t)g.ncb * kQB * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    const int ry = (int)((nr + 8 * 64 - 1) / (8 * 64));
    colmax_kernel<<<dim3((unsigned)((d + 31) / 32), (unsigned)(ry < 1024 ? ry : 1024)), 256, 0, s>>>(Ac, nr, ld, d,
                                                                                                    cmax, nanflag);
    quant_kernel<<<dim3((unsigned)g.nkb, (unsigned)g.ncb), 256, 0, s>>>(Ac, nr, ld, d, cmax, g.ncb, planes);
    syrk_i8_kernel<<<g.ntiles * g.nsplit, kSyThreads, smem, s>>>(planes, g, cmax, d, part);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  syrk_i8_finish_kernel<<<gmax.ntiles, 256, 0, s>>>(part, gmax, d, AtA, nanflag);
  return cudaGetLastError();
}

}  // namespace fdk
