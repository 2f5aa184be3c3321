// fd_perrow.cu — persistent per-row Frequent Directions kernel:
// Alg. 1's row loop for the per-row variants FD,
// alpha-FD (Alg. 2), iSVD, SpaceSaving Directions
// (Alg. 3) and Compensative FD's lazy stream,
// one thread-block cluster per shard stream, every row of an append call in one
// launch, the sketch state in fp64.
//
// Row step.  After every step the state rows b_1..b_k are mutually orthogonal
// (B' = diag(w) U^T Bf has orthogonal rows: u_j^T G u_i = lambda_j delta_ij), so the
// Gram of [B; a] is the arrowhead
//       H = [[ D, z ], [ z^T, rho ]],  D = diag(||b_j||^2), z_j = b_j . a, rho = ||a||^2
// (the neglected b_i . b_j, i != j, are fp64 rounding, ~1e-16 ||B||^2).  Its
// eigenvalues are the roots of the secular equation
//       f(lambda) = lambda - rho - sum_j z_j^2 / (lambda - d_j) = 0,
// one in each interval between consecutive poles (interlacing), after deflating
// z_j ~ 0 and coincident poles (Givens).  Eigenvectors come from Loewner's formula
// (Gu-Eisenstat): z^_i^2 = -prod_m (d_i - lambda_m) / prod_{j != i} (d_i - d_j) is the
// z for which the computed lambdas are exact, and u_m ~ [z^/(lambda_m - D); 1], so the
// vectors are numerically orthogonal.  When the buffer is full (k + 1 = ell) the
// variant's ReduceRank rule picks delta and sigma'^2 exactly as the batched path
// (eig_kernel) and the oracle do; otherwise (the first ell - 1 rows; Compensative
// FD's pending row) the step only rotates: B' = U^T Bf keeps every row (B'^T B' =
// Bf^T Bf; the oracle keeps those rows unrotated: the same covariance).
//
// Work split: CTA r of a cluster of C owns the column slice [r dc, (r+1) dc) of the
// state (fp64, resident in shared memory for the whole call).  Per row: (1) the
// slice's partial dots b_j . a, ||b_j||^2, ||a||^2 (thread tile 8 rows x 4 columns,
// 16-lane reduce-scatter); (2) cluster barrier, every CTA sums the C partial vectors
// from distributed shared memory in the same order (bit-identical inputs, so every
// CTA takes the same decisions); (3) the secular roots are split over the cluster
// (warp per root, lanes over the terms) and gathered after a second barrier; (4)
// Loewner vectors and the rule, redundantly in every CTA; (5) the slice's
// reconstruct B'[:, slice] = W^T [B; a][:, slice] (fp64 register tiles 8 x 4) into
// the other state buffer.  fp64 throughout.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>
#include <stdint.h>

#include "fd_internal.h"

namespace cg = cooperative_groups;

namespace fdk {

namespace {

constexpr int kPrThreads = 256;
constexpr int kPrMaxCluster = 16;         // CTAs per stream (column slices of the state)
constexpr int kPrMaxRows = 128;           // state rows the register tiles cover (16 groups x 8)
constexpr int kPrColsPass = 64;           // columns per tile pass (16 lanes x 4)
constexpr int kPL = 2 * kPrMaxRows + 2;   // partial vector: c[128], nrm[128], ||a||^2
constexpr unsigned kFull = 0xffffffffu;

struct PrLayout {
  int ellp;       // state rows allocated (ell rounded up to 8)
  int dcp;        // state row stride (doubles), multiple of 4, >= dc
  int ws;         // WtT row stride (doubles): ellp + 2
  size_t S0, S1, arow, part, full, rp, rt, dsort, zsort, dpol, z2, zhat, lam, wout, scl, sclo, rc, rs, WtT, ints,
      total;
};

__host__ __device__ inline size_t pr_align(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline PrLayout pr_layout(int ell, int dc) {
  PrLayout L;
  L.ellp = (ell + 7) / 8 * 8;
  L.dcp = (dc + 3) / 4 * 4;
  L.ws = L.ellp + 2;
  const size_t v = (size_t)(ell + 2) * 8;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = pr_align(off + bytes); return o; };
  L.S0 = take((size_t)L.ellp * L.dcp * 8);
  L.S1 = take((size_t)L.ellp * L.dcp * 8);
  L.arow = take((size_t)L.dcp * 8);
  L.part = take((size_t)2 * kPL * 8);     // double-buffered across rows (DSMEM readers)
  L.full = take((size_t)kPL * 8);
  L.rp = take(v);                          // roots: nearer pole p and offset tau (lambda = p + tau)
  L.rt = take(v);
  L.dsort = take(v);                       // arrowhead diagonal, sorted (coordinate order)
  L.zsort = take(v);
  L.dpol = take(v);                        // non-deflated poles (secular equation)
  L.z2 = take(v);
  L.zhat = take(v);                        // Loewner z^
  L.lam = take(v);                         // eigenvalue of each eigen slot
  L.wout = take(v);                        // rule weight of each output row
  L.scl = take(v);                         // pre-scale of each state row (CFD pending shrink)
  L.sclo = take(v);                        // final scale of each output column (weight / norm)
  L.rc = take(v);                          // Givens deflations
  L.rs = take(v);
  L.WtT = take((size_t)(ell + 1) * L.ws * 8);   // rows: Bf rows (state rows, then a); cols: outputs
  L.ints = take((size_t)9 * (ell + 2) * 4 + 32 * 4);
  L.total = off;
  return L;
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// 1/x in fp64: the hardware approximation (rcp.approx.ftz.f64) + two Newton steps
// (quadratic: ~2^-20 -> 2^-40 -> full precision); x is never 0 here (the poles and
// roots are separated by the deflation tolerance).
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// sum over the LW lanes of a lane group (xor butterfly: every lane gets the same bits)
template <int LW>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
  for (int o = LW / 2; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
template <int LW>
__device__ __forceinline__ void gsum2(double& a, double& b) {
#pragma unroll
  for (int o = LW / 2; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(kFull, a, o), y = __shfl_xor_sync(kFull, b, o);
    a += x;
    b += y;
  }
}

// Secular roots, one per group of LW lanes (the lanes split the terms).  Poles
// dp[0..K-1] strictly decreasing, z2 = z^2 > 0, tip rho, zn = ||z||.  Root m lies in
// (dp[m], dp[m-1]) (dp[-1] = +inf, dp[K] = -inf); groups with has == false idle.
// Returns lambda = p + tau with p the nearer pole (tau then carries the root's
// distance to it to full relative accuracy).  Safeguarded Newton on
// g(tau) = tau f(p + tau), which has no pole at tau = 0, started from the root of the
// model with the other poles frozen; bisection on the bracket (sign of f) whenever a
// step leaves it.  The whole warp iterates until its last group has converged.
template <int LW>
__device__ int secular_roots(int m, bool has, int K, const double* dp, const double* z2, double rho, double zn,
                             int gl, double& p_out, double& t_out) {
  int ip = 0;
  double p = 0.0, lo = 0.0, hi = 0.0;
  const bool interior = has && m > 0 && m < K;
  const double mid = interior ? 0.5 * (dp[m] + dp[m - 1]) : 0.0;
  double sm = 0.0;
  if (interior)
    for (int i = gl; i < K; i += LW) sm = fma(z2[i], rcp64(mid - dp[i]), sm);
  sm = gsum<LW>(sm);
  if (has) {
    if (m == 0) {
      ip = 0; p = dp[0]; lo = 0.0;
      hi = (fmax(rho - p, 0.0) + zn) * (1.0 + 8.0 * DBL_EPSILON) + DBL_MIN;
    } else if (m == K) {
      ip = K - 1; p = dp[K - 1]; hi = 0.0;
      lo = -(fmax(p - rho, 0.0) + zn) * (1.0 + 8.0 * DBL_EPSILON) - DBL_MIN;
    } else if (mid - rho - sm >= 0.0) {
      ip = m; p = dp[m]; lo = 0.0; hi = mid - p;
    } else {
      ip = m - 1; p = dp[m - 1]; lo = mid - p; hi = 0.0;
    }
  }
  double s0 = 0.0;
  if (has)
    for (int i = gl; i < K; i += LW)
      if (i != ip) s0 = fma(z2[i], rcp64(p - dp[i]), s0);
  s0 = gsum<LW>(s0);
  double t = 0.0;
  bool done = !has;
  double zp = 0.0;
  if (has) {
    zp = z2[ip];
    const double B = p - rho - s0;          // f(p + t) ~ t + B - zp / t
    const double disc = sqrt(B * B + 4.0 * zp);
    if (hi > 0.0) t = (B <= 0.0) ? 0.5 * (disc - B) : 2.0 * zp / (B + disc);
    else t = (B >= 0.0) ? -0.5 * (B + disc) : -2.0 * zp / (disc - B);
    if (!(t > lo && t < hi)) t = 0.5 * (lo + hi);
  }
  int it = 0;
  for (; it < 80; ++it) {
    if (!__any_sync(kFull, !done)) break;
    double s1 = 0.0, s2 = 0.0, s1b = 0.0, s2b = 0.0;
    if (!done) {
      int i = gl;
      for (; i + LW < K; i += 2 * LW) {     // two independent reciprocal chains per step
        const double ra = (i == ip) ? 0.0 : rcp64(t - (dp[i] - p));
        const double rb = (i + LW == ip) ? 0.0 : rcp64(t - (dp[i + LW] - p));
        const double qa = z2[i] * ra, qb = z2[i + LW] * rb;
        s1 += qa;
        s2 = fma(qa, ra, s2);
        s1b += qb;
        s2b = fma(qb, rb, s2b);
      }
      if (i < K && i != ip) {
        const double r = rcp64(t - (dp[i] - p));
        const double q = z2[i] * r;
        s1 += q;
        s2 = fma(q, r, s2);
      }
      s1 += s1b;
      s2 += s2b;
    }
    gsum2<LW>(s1, s2);
    if (done) continue;
    const double f = (p + t - rho) - zp * rcp64(t) - s1;
    if (f == 0.0) { done = true; continue; }   // t is a root
    if (f < 0.0) lo = t; else hi = t;
    const double g = t * (p + t - rho) - zp - t * s1;
    const double gp = (p + 2.0 * t - rho) - s1 + t * s2;
    const double dt = g * rcp64(gp);
    const double tn = t - dt;
    if (fabs(dt) <= 2.0 * DBL_EPSILON * fabs(t)) {   // converged (a last step may round onto the bracket)
      if (tn > lo && tn < hi) t = tn;
      done = true;
      continue;
    }
    t = (tn > lo && tn < hi) ? tn : 0.5 * (lo + hi);
    if (hi - lo <= 4.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) done = true;
  }
  p_out = p;
  t_out = t;
  return it;
}

// the roots of one CTA (m = crank, crank + C, ...), LW lanes per root
template <int LW>
__device__ int cta_roots(int K, int C, int crank, const double* dp, const double* z2, double rho, double zn,
                         double* rp, double* rt) {
  int iters = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int G = 32 / LW;                          // groups per warp
  const int nloc = (K + 1 - crank + C - 1) / C;       // roots this CTA owns
  const int grp = warp * G + lane / LW;
  for (int base = 0; base < nloc; base += (kPrThreads / 32) * G) {
    if (base + warp * G >= nloc) break;               // warp-uniform
    const int li = base + grp;
    const bool has = li < nloc;
    const int m = crank + C * li;
    double pp, tt;
    iters += secular_roots<LW>(has ? m : 0, has, K, dp, z2, rho, zn, lane % LW, pp, tt);
    if (has && lane % LW == 0) { rp[m] = pp; rt[m] = tt; }
  }
  return iters;
}

// block-wide sum of one double per thread (kPrThreads), result in every thread
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = wsum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kPrThreads / 32; ++w) s += red[w];
  return s;
}

}  // namespace

size_t perrow_smem_bytes(int ell, int64_t d, int C) {
  const int dc = (int)((d + C - 1) / C);
  return pr_layout(ell, dc).total;
}

// Cluster size of a per-row stream: enough CTAs that the state slice fits in shared
// memory and the per-row reconstruct (~ell^2 dc fp64 FMAs per CTA) stays short.
// Clusters above 8 CTAs are a non-portable size (opted into at launch); a 16-CTA
// cluster fits in one B200 GPC.
int perrow_cluster(int ell, int64_t d) {
  const double work = (double)ell * ell * (double)d;
  int C = 1;
  while (C < kPrMaxCluster && (work / C > 32768.0 || perrow_smem_bytes(ell, d, C) > kPrSmemMax)) C *= 2;
  if (perrow_smem_bytes(ell, d, C) > kPrSmemMax) return 0;
  return C;
}

bool perrow_supported(int ell, int64_t d, const Params& p) {
  return ell >= 2 && ell < kPrMaxRows && p.ret == ell - 1 && p.tdel == ell && perrow_cluster(ell, d) > 0;
}

__global__ void __launch_bounds__(kPrThreads, 1)
perrow_kernel(const RowJob* __restrict__ jobs, Params p, int C, int lazy, int* __restrict__ nonfinite) {
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const RowJob J = jobs[blockIdx.x / C];
  const int ell = p.ell, d = (int)p.d;
  const int dc = (d + C - 1) / C;
  const int c0 = crank * dc, c1 = min(d, c0 + dc), ncol = max(0, c1 - c0);
  const PrLayout Lo = pr_layout(ell, dc);
  extern __shared__ __align__(16) unsigned char smem[];
  auto D_ = [&](size_t o) { return reinterpret_cast<double*>(smem + o); };
  double* Sbuf[2] = {D_(Lo.S0), D_(Lo.S1)};
  double *arow = D_(Lo.arow), *part = D_(Lo.part), *full = D_(Lo.full), *rp = D_(Lo.rp), *rt = D_(Lo.rt);
  double *dsort = D_(Lo.dsort), *zsort = D_(Lo.zsort), *dpol = D_(Lo.dpol), *z2 = D_(Lo.z2), *zhat = D_(Lo.zhat);
  double *lam = D_(Lo.lam), *wout = D_(Lo.wout), *scl = D_(Lo.scl), *sclo = D_(Lo.sclo), *rc = D_(Lo.rc);
  double *rs = D_(Lo.rs), *WtT = D_(Lo.WtT);
  int* ib = reinterpret_cast<int*>(smem + Lo.ints);
  const int E = ell + 2;
  int* perm = ib;              // sorted coordinate -> state row
  int* dflag = ib + E;         // coordinate deflated?
  int* pidx = ib + 2 * E;      // coordinate -> pole index (non-deflated) or -1
  int* coord = ib + 3 * E;     // pole index -> coordinate
  int* slot_src = ib + 4 * E;  // eigen slot -> root m (>= 0) or ~coordinate (deflated)
  int* order = ib + 5 * E;     // sorted position -> eigen slot
  int* out_src = ib + 6 * E;   // output row -> eigen slot
  int* rot_a = ib + 7 * E;     // Givens deflation pairs (coordinates)
  int* rot_b = ib + 8 * E;
  int* misc = ib + 9 * E;      // [0] K  [1] nrot  [4..11] / [12..19] per-warp ballot counts
  __shared__ double s_red[kPrThreads / 32];
  __shared__ double s_stat[4];  // frob, delta, removed, shrinks of this call (CTA-local copy)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cgp = lane & 15, rg = (lane >> 4) + 2 * warp;   // tile: rows 8 rg .. +7, cols 4 cgp .. +3
  const int lds = Lo.dcp, ws = Lo.ws;

  // ---- load the state slice (fp64, persistent across calls) ----
  int k = J.k_in;
  int cur = 0;
  for (int e = tid; e < Lo.ellp * lds; e += kPrThreads) {
    const int r = e / lds, c = e - r * lds;
    Sbuf[0][e] = (r < k && c < ncol) ? J.state[(int64_t)r * p.ldb + c0 + c] : 0.0;
    Sbuf[1][e] = 0.0;
  }
  if (tid < 4) s_stat[tid] = 0.0;
  for (int e = tid; e < 2 * kPL; e += kPrThreads) part[e] = 0.0;
  if (tid < 32) misc[tid] = 0;
  __syncthreads();
  if (C > 1) cluster.sync();

  const double eps = DBL_EPSILON;
  int bad = 0;
  float pre = 0.f;                      // prefetched element (column c0 + tid) of the next row
  if (J.nrows > 0 && tid < ncol) pre = J.src[c0 + tid];

  const bool tr = p.dbg && blockIdx.x == 0 && tid == 0;   // phase clocks (FD_DEBUG_EIG)
  long long t_ph = tr ? clock64() : 0;
  auto phase = [&](int i) {
    if (tr) { const long long c = clock64(); p.dbg[i] += c - t_ph; t_ph = c; }
  };
  for (int64_t t = 0; t < J.nrows; ++t) {
    const double* S = Sbuf[cur];
    double* Sn = Sbuf[cur ^ 1];
    double* pt = part + (t & 1) * kPL;
    // ---- the row's slice (fp64) into shared memory; prefetch the next row ----
    if (tid < lds) arow[tid] = (tid < ncol) ? (double)pre : 0.0;
    for (int c = tid + kPrThreads; c < lds; c += kPrThreads)
      arow[c] = (c < ncol) ? (double)J.src[t * J.ld + c0 + c] : 0.0;
    if (tid < ncol) bad |= !isfinite(pre);
    if (t + 1 < J.nrows && tid < ncol) pre = J.src[(t + 1) * J.ld + c0 + tid];
    __syncthreads();
    // ---- (1) slice partials: c_j = b_j . a, n_j = ||b_j||^2, ||a||^2 ----
    {
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = 0.0;
      if (8 * rg < k) {
        for (int cb = 0; cb < lds; cb += kPrColsPass) {
          const int c = cb + 4 * cgp;
          if (c >= lds) break;
          const double2 a01 = *reinterpret_cast<const double2*>(arow + c);
          const double2 a23 = *reinterpret_cast<const double2*>(arow + c + 2);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const double* row = S + (8 * rg + q) * lds + c;
            const double2 b01 = *reinterpret_cast<const double2*>(row);
            const double2 b23 = *reinterpret_cast<const double2*>(row + 2);
            v[q] = fma(b01.x, a01.x, fma(b01.y, a01.y, fma(b23.x, a23.x, fma(b23.y, a23.y, v[q]))));
            v[8 + q] = fma(b01.x, b01.x, fma(b01.y, b01.y, fma(b23.x, b23.x, fma(b23.y, b23.y, v[8 + q]))));
          }
        }
      }
      // reduce-scatter over the 16 column lanes: lane cgp ends with value cgp's total
#pragma unroll
      for (int lvl = 0; lvl < 4; ++lvl) {
        const int half = 8 >> lvl;
        const bool up = (cgp >> (3 - lvl)) & 1;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < half) {
            const double snd = up ? v[q] : v[q + half];
            const double kp = up ? v[q + half] : v[q];
            v[q] = kp + __shfl_xor_sync(kFull, snd, half);
          }
        }
      }
      if (8 * rg < kPrMaxRows) pt[(cgp < 8 ? 0 : kPrMaxRows) + 8 * rg + (cgp & 7)] = v[0];
      if (warp == 0) {
        double na = 0.0;
        for (int c = lane; c < lds; c += 32) na = fma(arow[c], arow[c], na);
        na = wsum(na);
        if (lane == 0) pt[2 * kPrMaxRows] = na;
      }
    }
    phase(0);
    // ---- (2) cluster-wide sums, fixed order (identical in every CTA) ----
    if (C > 1) cluster.sync(); else __syncthreads();
    phase(1);
    for (int e = tid; e <= 2 * kPrMaxRows; e += kPrThreads) {
      const bool used = (e < k) || (e >= kPrMaxRows && e < kPrMaxRows + k) || e == 2 * kPrMaxRows;
      double v[kPrMaxCluster];
#pragma unroll
      for (int r = 0; r < kPrMaxCluster; ++r)
        v[r] = (used && r < C) ? (r == crank ? pt : cluster.map_shared_rank(pt, r))[e] : 0.0;
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < kPrMaxCluster; ++r) s += v[r];
      full[e] = s;
    }
    __syncthreads();
    const double rho = full[2 * kPrMaxRows];
    if (tid == 0) s_stat[0] += rho;
    phase(2);
    // ---- (3) Compensative FD: ReduceRank of the full pending buffer first (C27).  Its
    //      Gram is diag(||b_j||^2); the FD rule gives every state row a weight ----
    if (tid <= ell) scl[tid] = 1.0;
    const bool full_pend = lazy && (k == ell);
    if (full_pend) {
      if (tid < k) {
        const double dv = fmax(full[kPrMaxRows + tid], 0.0);
        int rk = 0;
        for (int j = 0; j < k; ++j) {
          const double dj = fmax(full[kPrMaxRows + j], 0.0);
          rk += (dj > dv) || (dj == dv && j < tid);
        }
        order[rk] = tid;
        lam[rk] = dv;
      }
      __syncthreads();
      const double delta = lam[ell - 1];
      double rem = 0.0;
      if (tid < ell) {
        const double lj = lam[tid];
        double sp2 = 0.0;
        if (tid < ell - 1) sp2 = (tid < ell - p.m) ? lj : fmax(lj - delta, 0.0);
        rem = lj - sp2;
        scl[order[tid]] = (lj > 0.0) ? sqrt(sp2) / sqrt(lj) : 0.0;
      }
      rem = block_sum(rem, s_red);
      if (tid == 0) { s_stat[1] += delta; s_stat[2] += rem; s_stat[3] += 1.0; }
    }
    __syncthreads();
    // the pending shrink frees the slot of the smallest direction (slot semantics, C6):
    // that row leaves the arrowhead; kc state coordinates + the new row remain
    const int drop = full_pend ? order[ell - 1] : -1;
    const int kc = full_pend ? k - 1 : k;
    const int n = kc + 1;
    const bool shrink = !lazy && (n == ell);
    // ---- (4) arrowhead coordinates: D' = scl^2 D sorted descending (ties by row).  The
    //      state rows come out of the previous step sorted (sigma'^2 descending), so the
    //      rank sort only runs when rounding (or CFD's pending shrink) broke the order ----
    {
      int unsorted = full_pend;
      if (!full_pend && tid > 0 && tid < k)
        unsorted = fmax(full[kPrMaxRows + tid - 1], 0.0) < fmax(full[kPrMaxRows + tid], 0.0);
      unsorted = __syncthreads_or(unsorted);
      if (tid < k && tid != drop) {
        const double sc = scl[tid];
        const double dv = sc * sc * fmax(full[kPrMaxRows + tid], 0.0);
        int rk = tid;
        if (unsorted) {
          rk = 0;
          for (int j = 0; j < k; ++j) {
            if (j == drop) continue;
            const double sj = scl[j];
            const double dj = sj * sj * fmax(full[kPrMaxRows + j], 0.0);
            rk += (dj > dv) || (dj == dv && j < tid);
          }
        }
        perm[rk] = tid;
        dsort[rk] = dv;
        zsort[rk] = sc * full[tid];
      }
    }
    __syncthreads();
    double zz = 0.0;
    if (tid < kc) zz = zsort[tid] * zsort[tid];
    zz = block_sum(zz, s_red);
    const double znorm = sqrt(zz);
    const double tol = 8.0 * eps * (fmax((kc > 0) ? dsort[0] : 0.0, rho) + znorm);
    // deflation (|z| <= tol); coincident poles: parallel detection, serial resolution (rare)
    int dfl = (tid < kc) ? (fabs(zsort[tid]) <= tol) : 0;
    if (tid < kc) dflag[tid] = dfl;
    __syncthreads();
    int close = 0;
    if (tid < kc && !dfl && tid > 0) {
      int j = tid - 1;
      while (j >= 0 && dflag[j]) --j;
      close = (j >= 0) && (dsort[j] - dsort[tid] <= tol);
    }
    if (__syncthreads_or(close)) {
      if (tid == 0) {
        int prev = -1, nrot = 0;
        for (int i = 0; i < kc; ++i) {
          if (dflag[i]) continue;
          if (prev >= 0 && dsort[prev] - dsort[i] <= tol) {
            const double zp = zsort[prev], zi = zsort[i];
            const double r = hypot(zp, zi);
            rc[nrot] = zp / r;
            rs[nrot] = zi / r;
            rot_a[nrot] = prev;
            rot_b[nrot] = i;
            ++nrot;
            zsort[prev] = r;
            zsort[i] = 0.0;
            dflag[i] = 1;
          } else {
            prev = i;
          }
        }
        misc[1] = nrot;
      }
      __syncthreads();
      dfl = (tid < kc) ? dflag[tid] : 0;
    } else if (tid == 0) {
      misc[1] = 0;
    }
    // pole index / deflated index of every coordinate (ballot prefix counts)
    {
      const unsigned live = __ballot_sync(kFull, tid < kc && !dfl);
      const unsigned dead = __ballot_sync(kFull, tid < kc && dfl);
      if (lane == 0) { ib[9 * E + 4 + warp] = __popc(live); ib[9 * E + 12 + warp] = __popc(dead); }
      __syncthreads();
      int ol = 0, od = 0;
      for (int w = 0; w < warp; ++w) { ol += ib[9 * E + 4 + w]; od += ib[9 * E + 12 + w]; }
      const unsigned lt = (1u << lane) - 1u;
      const int q = ol + __popc(live & lt), qd = od + __popc(dead & lt);
      if (tid < kc) {
        if (!dfl) {
          pidx[tid] = q;
          coord[q] = tid;
          dpol[q] = dsort[tid];
          z2[q] = zsort[tid] * zsort[tid];
        } else {
          pidx[tid] = -1 - qd;          // deflated: -1 - (its index among the deflated)
        }
      }
      if (tid == 0) {
        int K = 0;
        for (int w = 0; w < kPrThreads / 32; ++w) K += ib[9 * E + 4 + w];
        misc[0] = K;
      }
    }
    __syncthreads();
    const int K = misc[0];
    const int nrot = misc[1];
    phase(3);
    // ---- (5) secular roots, split over the cluster: root m -> CTA m % C ----
    {
      const int nroots = K + 1;
      if (K == 0) {
        if (tid == 0) { rp[0] = rho; rt[0] = 0.0; }
      } else {
        double zs = 0.0;
        if (tid < K) zs = z2[tid];
        zs = block_sum(zs, s_red);
        const double zn = sqrt(zs);
        int its;
        if (K <= 16) its = cta_roots<4>(K, C, crank, dpol, z2, rho, zn, rp, rt);
        else if (K <= 32) its = cta_roots<8>(K, C, crank, dpol, z2, rho, zn, rp, rt);
        else if (K <= 64) its = cta_roots<16>(K, C, crank, dpol, z2, rho, zn, rp, rt);
        else its = cta_roots<32>(K, C, crank, dpol, z2, rho, zn, rp, rt);
        if (tr) { p.dbg[10] += its; p.dbg[11] = max(p.dbg[11], (long long)its); p.dbg[12] += K; }
      }
      phase(4);
      if (C > 1) {
        cluster.sync();
        if (K > 0)
          for (int m = tid; m < nroots; m += kPrThreads) {
            const int own = m % C;
            if (own != crank) {
              rp[m] = cluster.map_shared_rank(rp, own)[m];
              rt[m] = cluster.map_shared_rank(rt, own)[m];
            }
          }
      }
      __syncthreads();
    }
    phase(5);
    // ---- (6) Loewner z^_q = sign(z_q) sqrt(-(d_q - l_q)(d_q - l_K) prod_{m != q} (d_q - l_m)/(d_q - d_m)) ----
    {   // two threads per pole (even / odd m), combined by one shuffle
      const int q = tid >> 1, h = tid & 1;
      double prod = 1.0;
      if (q < K) {
        const double di = dpol[q];
        if (h == 0) prod = -((di - rp[q]) - rt[q]) * ((di - rp[K]) - rt[K]);
        for (int m = h; m < K; m += 2)
          if (m != q) prod *= ((di - rp[m]) - rt[m]) * rcp64(di - dpol[m]);
      }
      prod *= __shfl_xor_sync(kFull, prod, 1);
      if (q < K && h == 0) zhat[q] = copysign(sqrt(fmax(prod, 0.0)), zsort[coord[q]]);
    }
    // eigen slots: roots 0..K (descending by interlacing), then the deflated coordinates
    // (descending: a subsequence of the sorted diagonal)
    if (tid <= K) { slot_src[tid] = tid; lam[tid] = fmax(rp[tid] + rt[tid], 0.0); }
    if (tid < kc && pidx[tid] < 0) {
      const int qd = -1 - pidx[tid];
      slot_src[K + 1 + qd] = ~tid;
      lam[K + 1 + qd] = fmax(dsort[tid], 0.0);
    }
    __syncthreads();
    // merge of the two descending lists by binary search (ties: roots first)
    if (tid < n) {
      const int nd = n - (K + 1);
      const double lv = lam[tid];
      int rk;
      if (tid <= K) {            // roots: + #deflated strictly greater
        int lo = 0, hi = nd;
        while (lo < hi) { const int md = (lo + hi) >> 1; if (lam[K + 1 + md] > lv) lo = md + 1; else hi = md; }
        rk = tid + lo;
      } else {                   // deflated: + #roots >= value
        int lo = 0, hi = K + 1;
        while (lo < hi) { const int md = (lo + hi) >> 1; if (lam[md] >= lv) lo = md + 1; else hi = md; }
        rk = (tid - (K + 1)) + lo;
      }
      order[rk] = tid;
    }
    __syncthreads();
    // ---- (7) the ReduceRank rule ----
    int kept = n;
    if (!shrink) {
      if (tid < n) { out_src[tid] = order[tid]; wout[tid] = 1.0; }
    } else {
      kept = ell - 1;
      const double l0 = lam[order[0]], lm1 = lam[order[ell - 1]];
      double delta = lm1;
      int src_last = -1;
      if (p.rule == RULE_SS) {
        delta = 0.0;
        if (lm1 > 1e-12 * l0) { delta = lam[order[ell - 2]]; src_last = ell - 1; }
      }
      double rem = 0.0;
      if (tid < n) {
        const int j = tid;
        const double lj = lam[order[j]];
        double sp2;
        if (p.rule == RULE_SS) {
          if (src_last >= 0) sp2 = (j < ell - 2) ? lj : (j == ell - 1 ? lj + delta : 0.0);
          else sp2 = (j < ell - 1) ? lj : 0.0;
        } else if (j >= ell - 1) {
          sp2 = 0.0;
        } else if (p.rule == RULE_ISVD || j < ell - p.m) {
          sp2 = lj;
        } else {
          sp2 = fmax(lj - delta, 0.0);
        }
        rem = lj - sp2;
        int orow = j;
        if (src_last >= 0) orow = (j == ell - 1) ? ell - 2 : (j == ell - 2 ? -1 : j);
        if (orow >= 0 && orow < kept) {
          out_src[orow] = order[j];
          wout[orow] = (lj > 0.0) ? sqrt(sp2) / sqrt(lj) : 0.0;
        }
      }
      rem = block_sum(rem, s_red);
      if (tid == 0) { s_stat[1] += delta; s_stat[2] += rem; s_stat[3] += 1.0; }
    }
    __syncthreads();
    phase(6);
    // ---- (8) W^T (rows: Bf rows = state rows, then the new row k; cols: outputs), two
    //      threads per output column (coordinates split by parity), fused column norms;
    //      CFD's pending-shrink weights scale the state rows ----
    {
      const int j = tid >> 1, h = tid & 1;
      double nn = 0.0;
      if (j < kept) {
        const int src = slot_src[out_src[j]];
        if (src >= 0) {
          const double pm = rp[src], tm = rt[src];
          for (int ci = h; ci < kc; ci += 2) {
            const int q = pidx[ci];
            double x = 0.0;
            if (q >= 0) x = zhat[q] * rcp64(tm - (dpol[q] - pm));   // z^_q / (lambda_m - d_q)
            nn = fma(x, x, nn);
            const int row = perm[ci];
            WtT[row * ws + j] = x * scl[row];
          }
          if (h == 0) { WtT[k * ws + j] = 1.0; nn += 1.0; }
        } else {
          const int c0d = ~src;
          for (int ci = h; ci < kc; ci += 2) {
            const int row = perm[ci];
            WtT[row * ws + j] = (ci == c0d) ? scl[row] : 0.0;
          }
          if (h == 0) { WtT[k * ws + j] = 0.0; nn = 1.0; }
        }
        if (h == 0 && drop >= 0) WtT[drop * ws + j] = 0.0;
      }
      nn += __shfl_xor_sync(kFull, nn, 1);
      __syncwarp();
      if (j < kept && h == 0) {
        // Givens deflations, reverse order (rows perm[a], perm[b]; scl is 1 outside CFD's
        // pending shrink, and then the rotated pair shares ... scl applied per row above)
        for (int r = nrot - 1; r >= 0; --r) {
          const int ra = perm[rot_a[r]], rb = perm[rot_b[r]];
          const double sa = scl[ra], sb = scl[rb];
          const double xa = (sa != 0.0) ? WtT[ra * ws + j] / sa : 0.0;
          const double xb = (sb != 0.0) ? WtT[rb * ws + j] / sb : 0.0;
          const double c = rc[r], sn = rs[r];
          WtT[ra * ws + j] = (c * xa - sn * xb) * sa;
          WtT[rb * ws + j] = (sn * xa + c * xb) * sb;
        }
        sclo[j] = (nn > 0.0) ? wout[j] / sqrt(nn) : 0.0;
      }
    }
    __syncthreads();
    phase(7);
    // ---- (9) reconstruct the slice: Sn[j][c] = sclo_j sum_r WtT[r][j] Bf[r][c] ----
    for (int cb = 0; cb < lds; cb += kPrColsPass) {
      const int c = cb + 4 * cgp;
      if (c >= lds || 8 * rg >= Lo.ellp) continue;
      double acc[8][4];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int h = 0; h < 4; ++h) acc[q][h] = 0.0;
      if (8 * rg < kept) {
        for (int r = 0; r <= k; ++r) {
          const double* br = (r < k) ? (S + r * lds + c) : (arow + c);
          const double2 b01 = *reinterpret_cast<const double2*>(br);
          const double2 b23 = *reinterpret_cast<const double2*>(br + 2);
          const double* wr = WtT + r * ws + 8 * rg;
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) {
            const double2 w = *reinterpret_cast<const double2*>(wr + 2 * q2);
            acc[2 * q2][0] = fma(w.x, b01.x, acc[2 * q2][0]);
            acc[2 * q2][1] = fma(w.x, b01.y, acc[2 * q2][1]);
            acc[2 * q2][2] = fma(w.x, b23.x, acc[2 * q2][2]);
            acc[2 * q2][3] = fma(w.x, b23.y, acc[2 * q2][3]);
            acc[2 * q2 + 1][0] = fma(w.y, b01.x, acc[2 * q2 + 1][0]);
            acc[2 * q2 + 1][1] = fma(w.y, b01.y, acc[2 * q2 + 1][1]);
            acc[2 * q2 + 1][2] = fma(w.y, b23.x, acc[2 * q2 + 1][2]);
            acc[2 * q2 + 1][3] = fma(w.y, b23.y, acc[2 * q2 + 1][3]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = 8 * rg + q;
        const double sc = (j < kept) ? sclo[j] : 0.0;
        double* o = Sn + j * lds + c;
        *reinterpret_cast<double2*>(o) = make_double2(sc * acc[q][0], sc * acc[q][1]);
        *reinterpret_cast<double2*>(o + 2) = make_double2(sc * acc[q][2], sc * acc[q][3]);
      }
    }
    __syncthreads();
    phase(8);
    if (tr) p.dbg[9] += 1;
    k = kept;
    cur ^= 1;
  }
  // ---- write back: fp64 state, its fp32 copy (the shard buffer fd_sketch reads), stats ----
  const double* S = Sbuf[cur];
  for (int e = tid; e < ell * lds; e += kPrThreads) {
    const int r = e / lds, c = e - r * lds;
    if (c >= ncol) continue;
    const double v = (r < k) ? S[e] : 0.0;
    J.state[(int64_t)r * p.ldb + c0 + c] = v;
    J.dst[(int64_t)r * p.ldb + c0 + c] = (float)v;
  }
  if (crank == C - 1)   // padding columns d..ldb-1 of the fp32 rows stay zero
    for (int e = tid; e < ell * (int)(p.ldb - d); e += kPrThreads) {
      const int r = e / (int)(p.ldb - d), c = d + e % (int)(p.ldb - d);
      J.dst[(int64_t)r * p.ldb + c] = 0.f;
    }
  bad = __syncthreads_or(bad);
  if (tid == 0) {
    if (bad) atomicOr(nonfinite, 1);
    if (crank == 0) {
      J.stats->frob += s_stat[0];
      J.stats->delta += s_stat[1];
      J.stats->removed += s_stat[2];
      J.stats->shrinks += s_stat[3];
    }
  }
  if (C > 1) cluster.sync();   // no CTA exits while a peer may still read its shared memory
}

cudaError_t launch_perrow(const RowJob* dev_jobs, int count, const Params& p, int lazy, int* nonfinite,
                          cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  int C = perrow_cluster(p.ell, p.d);
  if (C <= 0) return cudaErrorInvalidValue;
  int dev = 0;
  cudaGetDevice(&dev);
  static AttrOnce np;   // per device, like the smem attribute
  if (dev >= 64 || !((np.done >> dev) & 1ull)) {
    if (cudaError_t e = cudaFuncSetAttribute(perrow_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        e != cudaSuccess)
      return e;
    if (dev < 64) np.done |= 1ull << dev;
  }
  static AttrOnce once;
  if (cudaError_t e = once.ensure(perrow_kernel, (int)kPrSmemMax); e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kPrThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // the streams are dependent chains that all run for the whole call: every cluster must
  // be resident at once.  Clusters of 16 fit about one per GPC, so with many streams the
  // cluster shrinks (more column work per CTA) until all of them are co-resident.
  for (;;) {
    at[0].val.clusterDim.x = (unsigned)C;
    cfg.gridDim = dim3((unsigned)(count * C));
    cfg.dynamicSmemBytes = perrow_smem_bytes(p.ell, p.d, C);
    if (C == 1 || perrow_smem_bytes(p.ell, p.d, C / 2) > kPrSmemMax) break;
    int active = 0;
    if (cudaOccupancyMaxActiveClusters(&active, perrow_kernel, &cfg) != cudaSuccess) {
      cudaGetLastError();
      break;
    }
    if (active >= count) break;
    C /= 2;
  }
  return cudaLaunchKernelEx(&cfg, perrow_kernel, dev_jobs, p, C, lazy, nonfinite);
}

}  // namespace fdk
