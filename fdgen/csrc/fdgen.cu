/*
 * fdgen.cu — host and device drivers for the synthetic input generators.
 * See fdgen_core.h for the arithmetic contract (bit-identical host/device).
 * This library is input plumbing only; it contains none of the FD method.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include "fdgen_core.h"

#define FDG_MAXK 128
#define FDG_ROWS_PER_CTA 8

/* -------- per-row coefficient vector (S_i for noisy/image, g_i for drift) -------- */
FDG_HD void fdg_coeffs(const fdg_params* p, uint64_t i, double* c) {
  uint32_t tag = (p->kind == FDG_DRIFT) ? FDG_TAG_G : FDG_TAG_S;
  for (int t = 0; t < p->k; t += 2) {
    double z0, z1;
    fdg_normal2((uint32_t)(t >> 1), (uint32_t)i, (uint32_t)(i >> 32), tag, p->key0, p->key1, &z0, &z1);
    c[t] = z0;
    if (t + 1 < p->k) c[t + 1] = z1;
  }
}

/* signal part x_ij = sum_t c_t * F[t][j] in fixed order t = 0..k-1 */
FDG_HD double fdg_signal(const double* F, int k, int64_t d, int64_t j, const double* c) {
  double x = 0.0;
  for (int t = 0; t < k; ++t) x = FD_ADD(x, FD_MUL(c[t], F[(int64_t)t * d + j]));
  return x;
}

FDG_HD int fdg_drift_block(const fdg_params* p, uint64_t i) {
  int64_t b = (int64_t)i / p->block_rows;
  if (b >= p->nblocks) b = p->nblocks - 1;
  return (int)b;
}

FDG_HD double fdg_drift_scale(const fdg_params* p, int blk) {
  double s = 1.0;
  int r = blk % p->cycle;
  for (int q = 0; q < r; ++q) s = FD_MUL(s, p->growth);
  return s;
}

FDG_HD int fdg_is_e_row(const fdg_params* p, uint64_t i) {
  return p->period > 0 && (((int64_t)i + 1) % p->period) == 0;
}

/* Final element value given the signal x and noise z. */
FDG_HD float fdg_finish(const fdg_params* p, double x, double z) {
  if (p->kind == FDG_NOISY_LOWRANK) {
    return (float)FD_ADD(x, FD_DIV(z, p->noise_scale));
  } else { /* FDG_IMAGE_LIKE */
    double y = FD_DIV(FD_SUB(x, p->xmin), FD_SUB(p->xmax, p->xmin));
    y = FD_ADD(FD_MUL(255.0, y), FD_MUL(p->noise_scale, z));
#if defined(__CUDA_ARCH__)
    y = rint(y);
#else
    y = nearbyint(y);
#endif
    if (y < 0.0) y = 0.0;
    if (y > 255.0) y = 255.0;
    return (float)FD_DIV(y, 255.0);
  }
}

/* ============================== host ============================== */
extern "C" int fdg_host_rows(const fdg_params* p, int64_t row0, int64_t nrows, float* out, int64_t ld) {
  if (!p || !out || p->k > FDG_MAXK || p->k < 1 || ld < p->d) return -1;
  double c[FDG_MAXK];
  const int64_t d = p->d;
  for (int64_t r = 0; r < nrows; ++r) {
    uint64_t i = (uint64_t)(row0 + r);
    float* o = out + r * ld;
    if (p->kind == FDG_DRIFT) {
      if (fdg_is_e_row(p, i)) {
        for (int64_t j = 0; j < d; ++j) o[j] = (float)p->e[j];
        continue;
      }
      int blk = fdg_drift_block(p, i);
      double sc = fdg_drift_scale(p, blk);
      fdg_coeffs(p, i, c);
      const double* V = p->DU + (int64_t)blk * p->k * d;
      for (int64_t j = 0; j < d; ++j) o[j] = (float)FD_MUL(fdg_signal(V, p->k, d, j, c), sc);
      continue;
    }
    fdg_coeffs(p, i, c);
    for (int64_t j = 0; j < d; j += 2) {
      double z0, z1;
      fdg_normal2((uint32_t)(j >> 1), (uint32_t)i, (uint32_t)(i >> 32), FDG_TAG_N, p->key0, p->key1, &z0, &z1);
      o[j] = fdg_finish(p, fdg_signal(p->DU, p->k, d, j, c), z0);
      if (j + 1 < d) o[j + 1] = fdg_finish(p, fdg_signal(p->DU, p->k, d, j + 1, c), z1);
    }
  }
  return 0;
}

/* min / max of the signal part (image-like workload's global rescaling). */
extern "C" int fdg_host_minmax(const fdg_params* p, int64_t row0, int64_t nrows, double* mn, double* mx) {
  if (!p || p->k > FDG_MAXK) return -1;
  double c[FDG_MAXK];
  double lo = 1e300, hi = -1e300;
  for (int64_t r = 0; r < nrows; ++r) {
    fdg_coeffs(p, (uint64_t)(row0 + r), c);
    for (int64_t j = 0; j < p->d; ++j) {
      double x = fdg_signal(p->DU, p->k, p->d, j, c);
      lo = x < lo ? x : lo;
      hi = x > hi ? x : hi;
    }
  }
  *mn = lo; *mx = hi;
  return 0;
}

/* ============================== device ============================== */
__global__ void __launch_bounds__(256) fdg_rows_kernel(fdg_params p, int64_t row0, int64_t nrows,
                                                       float* __restrict__ out, int64_t ld) {
  __shared__ double coef[FDG_ROWS_PER_CTA][FDG_MAXK];
  __shared__ double scale[FDG_ROWS_PER_CTA];
  __shared__ int blkid[FDG_ROWS_PER_CTA];
  const int64_t rbase = (int64_t)blockIdx.x * FDG_ROWS_PER_CTA;
  const int nr = (int)min((int64_t)FDG_ROWS_PER_CTA, nrows - rbase);
  const int64_t d = p.d;
  /* coefficients: one (row, pair) per thread */
  const int npairs = (p.k + 1) / 2;
  for (int q = threadIdx.x; q < nr * npairs; q += blockDim.x) {
    int r = q / npairs, t2 = q % npairs;
    uint64_t i = (uint64_t)(row0 + rbase + r);
    uint32_t tag = (p.kind == FDG_DRIFT) ? FDG_TAG_G : FDG_TAG_S;
    double z0, z1;
    fdg_normal2((uint32_t)t2, (uint32_t)i, (uint32_t)(i >> 32), tag, p.key0, p.key1, &z0, &z1);
    coef[r][2 * t2] = z0;
    if (2 * t2 + 1 < p.k) coef[r][2 * t2 + 1] = z1;
  }
  if (threadIdx.x < nr && p.kind == FDG_DRIFT) {
    uint64_t i = (uint64_t)(row0 + rbase + threadIdx.x);
    int b = fdg_drift_block(&p, i);
    blkid[threadIdx.x] = b;
    scale[threadIdx.x] = fdg_drift_scale(&p, b);
  }
  __syncthreads();
  for (int64_t j = 2 * (int64_t)threadIdx.x; j < d; j += 2 * blockDim.x) {
    const bool has2 = (j + 1 < d);
    if (p.kind == FDG_DRIFT) {
      for (int r = 0; r < nr; ++r) {
        uint64_t i = (uint64_t)(row0 + rbase + r);
        float* o = out + (rbase + r) * ld;
        if (fdg_is_e_row(&p, i)) {
          o[j] = (float)p.e[j];
          if (has2) o[j + 1] = (float)p.e[j + 1];
          continue;
        }
        const double* V = p.DU + (int64_t)blkid[r] * p.k * d;
        o[j] = (float)FD_MUL(fdg_signal(V, p.k, d, j, coef[r]), scale[r]);
        if (has2) o[j + 1] = (float)FD_MUL(fdg_signal(V, p.k, d, j + 1, coef[r]), scale[r]);
      }
      continue;
    }
    double x0[FDG_ROWS_PER_CTA], x1[FDG_ROWS_PER_CTA];
#pragma unroll
    for (int r = 0; r < FDG_ROWS_PER_CTA; ++r) { x0[r] = 0.0; x1[r] = 0.0; }
    for (int t = 0; t < p.k; ++t) {
      double f0 = p.DU[(int64_t)t * d + j];
      double f1 = has2 ? p.DU[(int64_t)t * d + j + 1] : 0.0;
#pragma unroll
      for (int r = 0; r < FDG_ROWS_PER_CTA; ++r) {
        x0[r] = FD_ADD(x0[r], FD_MUL(coef[r][t], f0));
        x1[r] = FD_ADD(x1[r], FD_MUL(coef[r][t], f1));
      }
    }
#pragma unroll
    for (int r = 0; r < FDG_ROWS_PER_CTA; ++r) {
      if (r >= nr) break;
      uint64_t i = (uint64_t)(row0 + rbase + r);
      double z0, z1;
      fdg_normal2((uint32_t)(j >> 1), (uint32_t)i, (uint32_t)(i >> 32), FDG_TAG_N, p.key0, p.key1, &z0, &z1);
      float* o = out + (rbase + r) * ld;
      o[j] = fdg_finish(&p, x0[r], z0);
      if (has2) o[j + 1] = fdg_finish(&p, x1[r], z1);
    }
  }
}

__global__ void __launch_bounds__(256) fdg_minmax_kernel(fdg_params p, int64_t row0, int64_t nrows,
                                                         unsigned long long* mnmx) {
  /* min/max of the signal; exact (order-independent).  Stored as ordered-integer keys. */
  __shared__ double coef[FDG_MAXK];
  double lo = 1e300, hi = -1e300;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    uint64_t i = (uint64_t)(row0 + r);
    __syncthreads();
    for (int t2 = threadIdx.x; t2 < (p.k + 1) / 2; t2 += blockDim.x) {
      double z0, z1;
      fdg_normal2((uint32_t)t2, (uint32_t)i, (uint32_t)(i >> 32), FDG_TAG_S, p.key0, p.key1, &z0, &z1);
      coef[2 * t2] = z0;
      if (2 * t2 + 1 < p.k) coef[2 * t2 + 1] = z1;
    }
    __syncthreads();
    for (int64_t j = threadIdx.x; j < p.d; j += blockDim.x) {
      double x = fdg_signal(p.DU, p.k, p.d, j, coef);
      lo = fmin(lo, x);
      hi = fmax(hi, x);
    }
  }
  /* map doubles to monotone unsigned keys */
  auto key = [](double v) -> unsigned long long {
    unsigned long long u = (unsigned long long)__double_as_longlong(v);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
  };
  atomicMin(&mnmx[0], key(lo));
  atomicMax(&mnmx[1], key(hi));
}

extern "C" int fdg_dev_rows(const fdg_params* p, int64_t row0, int64_t nrows, float* out, int64_t ld, void* stream) {
  if (!p || !out || p->k > FDG_MAXK || p->k < 1 || ld < p->d) return -1;
  if (nrows <= 0) return 0;
  int64_t grid = (nrows + FDG_ROWS_PER_CTA - 1) / FDG_ROWS_PER_CTA;
  fdg_rows_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(*p, row0, nrows, out, ld);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

/* mnmx: device buffer of 2 unsigned long long, initialised by the caller to {~0, 0}. */
extern "C" int fdg_dev_minmax(const fdg_params* p, int64_t row0, int64_t nrows, unsigned long long* mnmx, void* stream) {
  if (!p || p->k > FDG_MAXK) return -1;
  fdg_minmax_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(*p, row0, nrows, mnmx);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" double fdg_key_to_double(unsigned long long k) {
  unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  double v;
  memcpy(&v, &u, 8);
  return v;
}
