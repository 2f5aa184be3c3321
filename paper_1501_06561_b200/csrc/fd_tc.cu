// fd_tc.cu — the buffer Gram of one ReduceRank on the tensor cores (tcgen05,
// kind::tf32) with an FP32-accurate 3xTF32 split (x = hi + lo, hi = tf32(x);
// a.b ~ hi.hi + hi.lo + lo.hi, fp32 accumulation in TMEM).  SURVEY §8(a) row a2:
//   gram:  G = Bf Bf^T                (buffer Gram; "svd(B_[i])", Alg. 1)
// (the reconstruct, row a5, is fd_recon_i8.cu: int8 digit planes, exact accumulation)
//
// One CTA per problem (persistent over the launch's problems), 256 threads:
// all threads stream 32-column K-chunks of the operands from global memory into
// registers, split them into hi / lo and store them into double-buffered,
// 128-byte-swizzled shared-memory tiles; one elected thread issues the MMAs and
// commits them to an mbarrier that releases the buffer; warps 0-3 read the
// accumulators back with tcgen05.ld for the epilogue.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fd_internal.h"
#include "fd_tc.cuh"

namespace fdk {

namespace {

#ifndef FD_TC_THREADS
#define FD_TC_THREADS 512
#endif
constexpr int kTcThreads = FD_TC_THREADS;   // staging threads, all in the epilogue (c4 gram: 256 -> 512 threads 42.6 -> 39.3 ms)
constexpr int kTile = 256 * 128;   // bytes of one 256-row x 32-value SW128 tile
constexpr int kAccs = 4;           // K-split accumulators of the NP = 128 Gram (4 x 128 TMEM columns)

__device__ __forceinline__ double warp_sum_d_tc(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ const float* row_ptr(const Prob& P, int r, int64_t ldb) {
  if (r < P.rows0) return P.src0 + (int64_t)r * ldb;
  r -= P.rows0;
  return P.src1 + (int64_t)r * P.ld1;
}

// load 32-column K-chunk kc of rows [0, NP) of Bf (zero outside N / ldb) into registers
template <int NP>
__device__ __forceinline__ void gram_load(const Prob& P, int N, int64_t ldb, int kc, float4 (&x)[NP * 8 / kTcThreads]) {
  constexpr int NI = NP * 8 / kTcThreads;
#pragma unroll
  for (int j = 0; j < NI; ++j) {
    const int it = threadIdx.x + kTcThreads * j;
    const int r = it >> 3, c4 = it & 7;
    const int64_t col = (int64_t)kc * 32 + 4 * c4;
    x[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < N && col < ldb) x[j] = __ldg(reinterpret_cast<const float4*>(row_ptr(P, r, ldb) + col));
  }
}

template <int NP>
__device__ __forceinline__ void gram_store(unsigned char* hi, unsigned char* lo, const float4 (&x)[NP * 8 / kTcThreads]) {
  constexpr int NI = NP * 8 / kTcThreads;
#pragma unroll
  for (int j = 0; j < NI; ++j) {
    const int it = threadIdx.x + kTcThreads * j;
    const int r = it >> 3, c4 = it & 7;
    const uint32_t off = tc::sw128_off(r, 4 * c4);
    float4 h, l;
    tc::split_tf32(x[j].x, h.x, l.x);
    tc::split_tf32(x[j].y, h.y, l.y);
    tc::split_tf32(x[j].z, h.z, l.z);
    tc::split_tf32(x[j].w, h.w, l.w);
    *reinterpret_cast<float4*>(hi + off) = h;
    *reinterpret_cast<float4*>(lo + off) = l;
  }
}

}  // namespace

// G (fp32, ldg) = Bf Bf^T for every problem, N <= NP (NP = 128: one 128x128 tile;
// NP = 256: tiles rows [0,128) x cols [0,128) and rows [128,256) x cols [0,256)).
// Written: the lower block triangle (rows >= 128 x all cols, rows < 128 x cols < 128);
// entries are symmetric up to accumulation order (readers use the lower triangle).
template <int NP>
__global__ void __launch_bounds__(kTcThreads, 1) gram_tc_kernel(const Prob* __restrict__ probs, int count, Params p) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t s_tmem;
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
  uint32_t uses[2] = {0, 0};   // completed commits per buffer (phase tracking)
  const uint32_t id0 = tc::idesc_tf32(128, 128, 0, 0);
  const uint32_t id1 = tc::idesc_tf32(128, 256, 0, 0);
  constexpr int NI = NP * 8 / kTcThreads;

  __shared__ double s_fr[kTcThreads / 32];
  for (int pi = blockIdx.x; pi < count; pi += gridDim.x) {
    const Prob P = probs[pi];
    const int N = P.rows0 + P.rows1;
    const int nk = (int)((p.ldb + 31) / 32);
    // new rows read in place from A (Prob.acc1): ||a||^2 in fp64 and the non-finite
    // check ride on the staging loads (the ingest pass of row 1 of SURVEY 8(a))
    double fr = 0.0;
    bool bad = false;
    auto acc_rows = [&](const float4 (&v)[NI]) {
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int r = (threadIdx.x + kTcThreads * j) >> 3;
        if (r >= P.rows0) {   // zero outside N
          bad |= !(isfinite(v[j].x) && isfinite(v[j].y) && isfinite(v[j].z) && isfinite(v[j].w));
          fr += (double)v[j].x * v[j].x + (double)v[j].y * v[j].y + (double)v[j].z * v[j].z + (double)v[j].w * v[j].w;
        }
      }
    };
    float4 x[NI];
    gram_load<NP>(P, N, p.ldb, 0, x);
    if (P.acc1) acc_rows(x);
    gram_store<NP>(sm, sm + kTile, x);
    tc::fence_async_smem();
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
      const int b = kc & 1;
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t hi = tc::smem_u32(sm + (2 * b) * kTile), lo = tc::smem_u32(sm + (2 * b + 1) * kTile);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          // NP = 128: K-chunks rotate over kAccs accumulators (TMEM columns 128 a), summed
          // in fp32 registers by the epilogue: each accumulates 1/kAccs of the K range, so
          // the truncating fp32 accumulation of the MMAs (~0.5 ulp of the running sum per
          // step) biases the Gram kAccs^2 times less per accumulator, kAccs times less in total
          const uint32_t acc = ((NP == 128 ? kc >= kAccs : kc > 0) || ks > 0) ? 1u : 0u;
          const uint32_t ta = (NP == 128) ? tbase + 128u * (uint32_t)(kc % kAccs) : tbase;
          const uint32_t ko = ks * 32;  // 8 tf32 = 32 bytes along K
          // tile 0: rows [0,128) x cols [0,128)
          tc::mma_tf32(ta, tc::desc_k_sw128(hi + ko), tc::desc_k_sw128(hi + ko), id0, acc);
          tc::mma_tf32(ta, tc::desc_k_sw128(hi + ko), tc::desc_k_sw128(lo + ko), id0, 1u);
          tc::mma_tf32(ta, tc::desc_k_sw128(lo + ko), tc::desc_k_sw128(hi + ko), id0, 1u);
          if (NP == 256) {  // tile 1: rows [128,256) x cols [0,256), TMEM columns [128, 384)
            tc::mma_tf32(tbase + 128, tc::desc_k_sw128(hi + 16384 + ko), tc::desc_k_sw128(hi + ko), id1, acc);
            tc::mma_tf32(tbase + 128, tc::desc_k_sw128(hi + 16384 + ko), tc::desc_k_sw128(lo + ko), id1, 1u);
            tc::mma_tf32(tbase + 128, tc::desc_k_sw128(lo + 16384 + ko), tc::desc_k_sw128(hi + ko), id1, 1u);
          }
        }
        tc::commit(&mbar[b]);
      }
      if (kc + 1 < nk) {
        gram_load<NP>(P, N, p.ldb, kc + 1, x);
        if (P.acc1) acc_rows(x);
        const int nb = b ^ 1;
        if (kc >= 1) {  // buffer nb was read by the MMAs of chunk kc-1
          tc::mbar_wait(&mbar[nb], uses[nb] & 1);
          ++uses[nb];
        }
        gram_store<NP>(sm + (2 * nb) * kTile, sm + (2 * nb + 1) * kTile, x);
        tc::fence_async_smem();
      }
      __syncthreads();
    }
    // all MMAs of this problem: the last commit (and, if nk > 1, the one before it)
    {
      const int bl = (nk - 1) & 1;
      if (nk >= 2) { tc::mbar_wait(&mbar[bl ^ 1], uses[bl ^ 1] & 1); ++uses[bl ^ 1]; }
      tc::mbar_wait(&mbar[bl], uses[bl] & 1);
      ++uses[bl];
    }
    tc::fence_after_sync();
    if (P.acc1) {   // fixed-order reduction: lanes, then warps (deterministic)
      fr = warp_sum_d_tc(fr);
      if (lane == 0) s_fr[warp] = fr;
      bad = __syncthreads_or(bad);
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kTcThreads / 32; ++w) t += s_fr[w];
        P.stats->frob += t;
        if (bad && p.nonfinite) atomicOr(p.nonfinite, 1);
      }
    }
    // epilogue: warp w reads TMEM lanes 32 (w % 4).. (= tile rows); the warp groups
    // w / 4 split the 16-column chunks
    {
      constexpr int kNG = kTcThreads / 128;
      const int wq = warp & 3, wg = warp >> 2;
      float* G = static_cast<float*>(P.G);
      const int m = 32 * wq + lane;
      const uint32_t lanebase = tbase + ((uint32_t)(32 * wq) << 16);
#pragma unroll 1
      for (int t = 0; t < (NP == 256 ? 2 : 1); ++t) {
        const int row = 128 * t + m;
        const int ncols = (t == 0) ? 128 : 256;
        for (int c0 = 16 * wg; c0 < ncols; c0 += 16 * kNG) {
          float v[16];
          tc::tmem_ld16(lanebase + (t == 0 ? 0 : 128) + c0, v);
          if (NP == 128) {
            for (int a = 1; a < kAccs && a < nk; ++a) {
              float u[16];
              tc::tmem_ld16(lanebase + 128 * a + c0, u);
#pragma unroll
              for (int q = 0; q < 16; ++q) v[q] += u[q];
            }
          }
          if (row < N) {
            float* dst = G + (int64_t)row * p.ldg + c0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (c0 + 4 * q + 4 <= p.ldg) *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
  }
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

template <int NP>
static cudaError_t launch_gram_tc_t(const Prob* dev_probs, int count, const Params& p, cudaStream_t s) {
  constexpr int dyn = 4 * kTile + 1024;
  static AttrOnce once;
  if (cudaError_t e = once.ensure(gram_tc_kernel<NP>, dyn); e != cudaSuccess) return e;
  const int grid = count < kNumSMs ? count : kNumSMs;
  gram_tc_kernel<NP><<<grid, kTcThreads, dyn, s>>>(dev_probs, count, p);
  return cudaGetLastError();
}

bool gram_tc_supported(int nmax, const Params& p) { return !p.f64 && nmax >= 1 && nmax <= 256 && (p.ldg % 4) == 0; }

cudaError_t launch_gram_tc(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (nmax <= 128) return launch_gram_tc_t<128>(dev_probs, count, p, s);
  return launch_gram_tc_t<256>(dev_probs, count, p, s);
}

}  // namespace fdk
