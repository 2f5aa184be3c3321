// fd_internal.h — device-side descriptors and kernel launchers of libfd.
// Internal to the CUDA path (never included by the oracle).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fdk {

constexpr int kNumSMs = 148;
constexpr int kMaxN = 416;          // largest buffer Gram (eigen-problem) size (fp32 path; c3 ell=200 -> 400)
constexpr int kMaxNS = 256;         // largest size whose packed matrix / eigenvector block is smem-resident
constexpr int kMaxN64 = 160;        // largest problem run in fp64 (per-row chains)
constexpr int kEigThreads = 512;

enum Rule : int { RULE_FD = 0, RULE_ISVD = 1, RULE_SS = 3 };   // SS: ReduceRank-SS (Alg. 3)

// Per-shard / per-node statistics, fp64 (device).
struct Stats {
  double frob;     // sum ||a_i||^2
  double delta;    // Delta = sum delta_i
  double removed;  // sum (lambda_j - sigma'_j^2)
  double shrinks;  // number of ReduceRanks
};

// One ReduceRank problem: buffer Bf = [src0 rows0; src1 rows1] (ld = ldb each),
// Gram size N = rows0 + rows1 (<= kMaxN).  Output: dst rows 0..ell-1 (row ell-1 = 0).
struct Prob {
  const float* src0;
  const float* src1;
  int rows0, rows1;
  float* dst;
  void* G;       // N x N (ldg), element type float or double (Params.f64)
  void* Wt;      // (ell-1) x N (ldg), same element type
  Stats* stats;  // accumulates delta / removed / shrinks of this ReduceRank
  const Stats* child0;  // merges: stats = child0 + child1 before accumulating
  const Stats* child1;
  int64_t ld1;   // row stride of src1 (floats): Params.ldb, or the caller's ld when src1 is A itself
  int acc1;      // 1: src1 rows are new stream rows read in place from A (no ingest copy) --
                 // the Gram adds their fp64 sum of squares to stats->frob and flags non-finite values
};

// One shard stream's rows of an append call for the persistent per-row kernel
// (fd_perrow.cu): rows src[0 .. nrows) (stride ld) in stream order, the fp64 state
// (ell rows, stride Params.ldb doubles) carried across calls, its fp32 copy for
// fd_sketch's final ReduceRank (the shard buffer), and the shard's statistics.
struct RowJob {
  const float* src;
  int64_t ld;
  int64_t nrows;
  double* state;
  float* dst;
  Stats* stats;
  int k_in;       // rows in the state at entry (occupancy)
  int pad;
};
constexpr size_t kPrSmemMax = 225 * 1024;

// Ingest of one shard in one round: copy nrows rows of the user's A into the
// shard buffer (row stride ldb, zero-padded to ldb columns), accumulate ||a||^2.
struct Ingest {
  const float* src;
  int64_t ld;
  float* dst;
  int nrows;
  int pad;
  Stats* stats;
};

struct Params {
  int64_t d;     // true row length
  int64_t ldb;   // internal row stride (d rounded up to 4)
  int ldg;       // Gram / Wt row stride (= max problem size)
  int ell;
  int rule;
  int m;         // alpha-FD: number of trailing values that shrink
  int ret;       // rows kept by a ReduceRank: ell-1, or R of the paper-literal Fast alpha-FD
  int tdel;      // delta = lambda_tdel (1-based): ell, or t of the paper-literal Fast alpha-FD
  int comp;      // 1: Compensative FD final step, sigma_hat^2 = sigma'^2 + Delta on ret = ell rows
  int merge;     // 1: a merge level (large eigenvalue clusters expected: eig panel variant)
  int f64;       // 1: Gram / eigen / reconstruct accumulate in fp64 (per-row chains)
  int pretrd;    // 1: the Gram scratch already holds the tridiagonal form (trd_kernel)
  int zld;       // eig_kernel fp64 scratch stride (>= every problem size of the handle)
  long long* dbg;  // optional phase clock trace of problem 0 (FD_DEBUG_EIG), else null
  int* nonfinite;  // sticky device flag (Prob.acc1 rows)
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the current device
// only: remember, per kernel launcher, the device ordinals it was set on.
struct AttrOnce {
  unsigned long long done = 0;   // bit per device ordinal (< 64)
  int bytes[64] = {};
  template <typename K>
  cudaError_t ensure(K kernel, int nbytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 64 && ((done >> dev) & 1ull) && bytes[dev] >= nbytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, nbytes);
    if (e == cudaSuccess && dev < 64) { done |= 1ull << dev; bytes[dev] = nbytes; }
    return e;
  }
};

// All launchers return cudaGetLastError() after enqueueing.
cudaError_t launch_ingest(const Ingest* dev_desc, int count, const Params& p, int* nonfinite, cudaStream_t s);
cudaError_t launch_gram(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s);
cudaError_t launch_eig(const Prob* dev_probs, int count, const Params& p, double* scratch, cudaStream_t s);
cudaError_t launch_recon(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s);
size_t eig_scratch_bytes(int zld);   // device scratch the eig kernel needs (all CTA slots)
// Register-resident Householder tridiagonalisation (fd_trd.cu): overwrites each
// problem's Gram scratch with the packed reflectors + d / e / tau.
bool trd_supported(int nmax, const Params& p);
// tcgen05 3xTF32 GEMMs (fd_tc.cu)
bool gram_tc_supported(int nmax, const Params& p);
cudaError_t launch_gram_tc(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s);
// reconstruct B' = Wt Bf on tcgen05 kind::i8 (fd_recon_i8.cu: int8 digit planes of row- /
// column-scaled fixed point, exact int32 accumulation); N <= 256, ret <= 128
bool recon_i8_supported(int nmax, const Params& p);
cudaError_t launch_recon_i8(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s);
cudaError_t launch_trd(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s);
// Blocked (compact WY) back-transform + Wt = diag(w) U^T (fd_bt.cu), after eig when p.pretrd.
cudaError_t launch_bt(const Prob* dev_probs, int count, const Params& p, cudaStream_t s);

// Persistent per-row kernel (fd_perrow.cu): every row of an append call,
// one thread-block cluster per shard stream, fp64 state, arrowhead eigen-updates.
bool perrow_supported(int ell, int64_t d, const Params& p);
int perrow_cluster(int ell, int64_t d);
size_t perrow_smem_bytes(int ell, int64_t d, int C);
cudaError_t launch_perrow(const RowJob* dev_jobs, int count, const Params& p, int lazy, int* nonfinite,
                          cudaStream_t s);

// Evaluator.
// AtA += A^T A on the tensor cores (fd_syrk_tc.cu: int8 digit planes of column-scaled
// fixed-point A, tcgen05 kind::i8, exact int32 accumulation, fp64 drains); workspace
// syrk_tc_workspace_bytes(n, d) (required)
size_t syrk_tc_workspace_bytes(int64_t n, int64_t d);
cudaError_t launch_syrk_tc(const float* A, int64_t n, int64_t ld, int64_t d, double* AtA, void* ws, size_t ws_bytes,
                           cudaStream_t s);
cudaError_t launch_sub_btb(double* M, const double* AtA, const float* B, int ell, int64_t d, cudaStream_t s);
// Lanczos (fd_lanczos.cu): one cooperative grid, full re-orthogonalisation; work holds
// lanczos_work_doubles(d, kmax) doubles, Q (kmax + 1) x d
size_t lanczos_work_doubles(int64_t d, int kmax);
cudaError_t launch_lanczos(const double* M, int64_t d, int kmax, double* Q, double* work, double* out2,
                           cudaStream_t s, int ntop = 0, double* top = nullptr);
// Hashing / OSNAP (fd_hash.cu): B (ell x d fp64) += S A; partials: hash_ranges(d) * ell * d doubles
int hash_ranges(int64_t d);
bool hash_supported(int ell, int s);
cudaError_t launch_hash(const float* A, int64_t n, int64_t ld, int64_t d, int ell, int s, uint64_t seed, int64_t row0,
                        double* partials, double* B, cudaStream_t st);
// proj-err parts (fd_eval.cu): G = B B^T, Jacobi -> (V, w, ord), q[t] = v_t^T AtA v_t
cudaError_t launch_proj_parts(const float* B, int ell, int64_t d, int k, const double* AtA, double* G, double* V,
                              double* w, int* ord, int* sweeps, double* vbuf, double* q, cudaStream_t s);

}  // namespace fdk
