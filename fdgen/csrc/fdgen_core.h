/*
 * fdgen_core.h — seeded, counter-based synthetic input generators.
 *
 * This module produces the INPUT rows A for both the CPU oracle and the GPU
 * path. It holds none of the sketching method's arithmetic: it only draws
 * Gaussian variates and forms the synthetic rows of the workloads named in
 * BASELINE.json (DESIGN.md §"Input recipe").
 *
 * Bit-exactness: every function here is compiled twice — once for the host
 * (gcc, -ffp-contract=off) and once for sm_100a (all fp64 products/sums go
 * through FD_MUL/FD_ADD, which are __dmul_rn/__dadd_rn on the device, so no
 * FMA contraction happens on either side).  The only operations used are
 * IEEE-754 correctly-rounded +, -, *, /, sqrt and integer arithmetic, hence
 * the host and device generators produce identical fp32 bytes for every row.
 *
 * Gaussian variates: Philox4x32-10 (counter-based) -> two 53-bit uniforms ->
 * Box-Muller with a hand-written log / sin / cos built from the operations
 * above (no libm, whose last-ulp behaviour differs between glibc and CUDA).
 */
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define FDG_HD __host__ __device__ __forceinline__
#else
#define FDG_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define FD_MUL(a, b) __dmul_rn((a), (b))
#define FD_ADD(a, b) __dadd_rn((a), (b))
#define FD_SUB(a, b) __dsub_rn((a), (b))
#define FD_DIV(a, b) __ddiv_rn((a), (b))
#define FD_SQRT(a) __dsqrt_rn(a)
#else
#include <math.h>
#define FD_MUL(a, b) ((a) * (b))
#define FD_ADD(a, b) ((a) + (b))
#define FD_SUB(a, b) ((a) - (b))
#define FD_DIV(a, b) ((a) / (b))
#define FD_SQRT(a) sqrt(a)
#endif

/* ---------------- Philox4x32-10 ---------------- */
typedef struct { uint32_t v[4]; } fdg_u4;

FDG_HD void fdg_mulhilo(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  *lo = (uint32_t)p;
}

FDG_HD fdg_u4 fdg_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                         uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    fdg_mulhilo(0xD2511F53u, c0, &hi0, &lo0);
    fdg_mulhilo(0xCD9E8D57u, c2, &hi1, &lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  fdg_u4 out;
  out.v[0] = c0; out.v[1] = c1; out.v[2] = c2; out.v[3] = c3;
  return out;
}

/* 53-bit uniform in [0,1) from two 32-bit words (exact: k * 2^-53). */
FDG_HD double fdg_u53(uint32_t a, uint32_t b) {
  uint64_t k = ((uint64_t)(a >> 5) << 26) | (uint64_t)(b >> 6);
  return (double)k * 1.1102230246251565e-16; /* 2^-53, exact */
}

/* ---------------- log / sin / cos from +,-,*,/ only ---------------- */
/* ln(u) for u in (0, 1]: u = m * 2^e (exact bit split), m in [sqrt(.5), sqrt(2)),
 * ln m = 2 atanh(s), s = (m-1)/(m+1), |s| <= 0.1716; odd series to s^23. */
FDG_HD double fdg_log(double u) {
  union { double d; uint64_t i; } x;
  x.d = u;
  int e = (int)((x.i >> 52) & 0x7FF) - 1023;
  x.i = (x.i & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull; /* m in [1,2) */
  double m = x.d;
  if (m > 1.4142135623730951) { m = FD_MUL(m, 0.5); e += 1; }
  double s = FD_DIV(FD_SUB(m, 1.0), FD_ADD(m, 1.0));
  double s2 = FD_MUL(s, s);
  double p = 1.0 / 23.0;
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 21.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 19.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 17.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 15.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 13.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 11.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 9.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 7.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 5.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0 / 3.0);
  p = FD_ADD(FD_MUL(p, s2), 1.0);
  double lnm = FD_MUL(FD_MUL(2.0, s), p);
  return FD_ADD(FD_MUL((double)e, 0.69314718055994531), lnm);
}

/* sin and cos of x in [0, pi/4] by Taylor series (error < 1e-17). */
FDG_HD void fdg_sincos_small(double x, double* sn, double* cs) {
  double x2 = FD_MUL(x, x);
  double s = 1.0 / 355687428096000.0;            /* 1/17! */
  s = FD_SUB(1.0 / 1307674368000.0, FD_MUL(s, x2)); /* 1/15! */
  s = FD_SUB(1.0 / 6227020800.0, FD_MUL(s, x2));    /* 1/13! */
  s = FD_SUB(1.0 / 39916800.0, FD_MUL(s, x2));      /* 1/11! */
  s = FD_SUB(1.0 / 362880.0, FD_MUL(s, x2));        /* 1/9!  */
  s = FD_SUB(1.0 / 5040.0, FD_MUL(s, x2));          /* 1/7!  */
  s = FD_SUB(1.0 / 120.0, FD_MUL(s, x2));           /* 1/5!  */
  s = FD_SUB(1.0 / 6.0, FD_MUL(s, x2));             /* 1/3!  */
  s = FD_SUB(1.0, FD_MUL(s, x2));
  *sn = FD_MUL(s, x);
  double c = 1.0 / 6402373705728000.0;           /* 1/18! */
  c = FD_SUB(1.0 / 20922789888000.0, FD_MUL(c, x2)); /* 1/16! */
  c = FD_SUB(1.0 / 87178291200.0, FD_MUL(c, x2));    /* 1/14! */
  c = FD_SUB(1.0 / 479001600.0, FD_MUL(c, x2));      /* 1/12! */
  c = FD_SUB(1.0 / 3628800.0, FD_MUL(c, x2));        /* 1/10! */
  c = FD_SUB(1.0 / 40320.0, FD_MUL(c, x2));          /* 1/8!  */
  c = FD_SUB(1.0 / 720.0, FD_MUL(c, x2));            /* 1/6!  */
  c = FD_SUB(1.0 / 24.0, FD_MUL(c, x2));             /* 1/4!  */
  c = FD_SUB(0.5, FD_MUL(c, x2));                    /* 1/2!  */
  *cs = FD_SUB(1.0, FD_MUL(c, x2));
}

/* sin(2 pi v), cos(2 pi v) for v in [0, 1): octant reduction is exact. */
FDG_HD void fdg_sincos2pi(double v, double* sn, double* cs) {
  double x = FD_MUL(v, 8.0); /* exact */
  int oct = (int)x;          /* 0..7 */
  double f = FD_SUB(x, (double)oct); /* exact, in [0,1) */
  const double pi4 = 0.78539816339744831;
  double a, b; /* a = sin, b = cos of the reduced angle */
  if (oct & 1) {
    fdg_sincos_small(FD_MUL(FD_SUB(1.0, f), pi4), &a, &b);
    double t = a; a = b; b = t; /* angle = (oct+1)*pi/4 - g  -> swap */
  } else {
    fdg_sincos_small(FD_MUL(f, pi4), &a, &b);
  }
  /* Now (a, b) = (sin, cos) of phi = f*pi/4 + (oct&1 ? ... ) within the quadrant.
   * Rotate by the quadrant q = oct/2: (s,c) -> q=0:(s,c) 1:(c,-s) 2:(-s,-c) 3:(-c,s). */
  int q = oct >> 1;
  double s, c;
  if (q == 0) { s = a; c = b; }
  else if (q == 1) { s = b; c = -a; }
  else if (q == 2) { s = -a; c = -b; }
  else { s = -b; c = a; }
  *sn = s; *cs = c;
}

/* Two independent N(0,1) variates for counter (c0..c3) under key (k0,k1). */
FDG_HD void fdg_normal2(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                        uint32_t k0, uint32_t k1, double* z0, double* z1) {
  fdg_u4 r = fdg_philox(c0, c1, c2, c3, k0, k1);
  double u1 = FD_SUB(1.0, fdg_u53(r.v[0], r.v[1])); /* (0, 1] */
  double u2 = fdg_u53(r.v[2], r.v[3]);              /* [0, 1) */
  double rad = FD_SQRT(FD_MUL(-2.0, fdg_log(u1)));
  double sn, cs;
  fdg_sincos2pi(u2, &sn, &cs);
  *z0 = FD_MUL(rad, cs);
  *z1 = FD_MUL(rad, sn);
}

/* Stream tags (counter word 3) so different random objects never share draws. */
#define FDG_TAG_S 0x53u      /* signal coefficients S (n x k)          */
#define FDG_TAG_N 0x4Eu      /* dense noise N (n x d)                  */
#define FDG_TAG_G 0x47u      /* drifting-subspace coefficients g (n x 8) */

/* Normal variate number j (0-based) of row i for object `tag`.
 * Variates come in pairs: pair p = j/2 of row i uses counter (p, i_lo, i_hi, tag). */
FDG_HD double fdg_normal_at(uint64_t i, uint32_t j, uint32_t tag, uint32_t k0, uint32_t k1) {
  double z0, z1;
  fdg_normal2(j >> 1, (uint32_t)i, (uint32_t)(i >> 32), tag, k0, k1, &z0, &z1);
  return (j & 1) ? z1 : z0;
}

/* ---------------- workload kinds ---------------- */
enum {
  FDG_NOISY_LOWRANK = 0, /* A = S * DU + N / zeta           (configs 1, 2, 4) */
  FDG_IMAGE_LIKE = 1,    /* clip(rint(255*minmax(S*DU) + sigma*N), 0, 255)/255 (config 3) */
  FDG_DRIFT = 2          /* drifting 8-dim subspaces + fixed direction  (config 5) */
};

/* Parameters shared by host and device.  Small fp64 factor matrices (DU, V, e)
 * are computed once on the host by fdgen/__init__.py and passed by pointer. */
typedef struct {
  int kind;
  int64_t d;
  int k;              /* signal rank (noisy/image) or subspace dim (drift)    */
  uint32_t key0, key1;
  double noise_scale; /* noisy: divide N by zeta -> stores zeta; image: sigma */
  const double* DU;   /* noisy/image: k x d (row t scaled by D_t); drift: nblk x k x d */
  const double* e;    /* drift: fixed direction (d)                         */
  double xmin, xmax;  /* image: global min / max of S*DU                    */
  int64_t block_rows; /* drift: rows per block                              */
  int64_t period;     /* drift: every `period`-th row is e                  */
  int nblocks;        /* drift: number of subspaces                        */
  double growth;      /* drift: block scale = growth^(j mod cycle)         */
  int cycle;
} fdg_params;
