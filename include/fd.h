/*
 * fd.h — C ABI of the B200-native Frequent Directions library (libfd.so).
 *
 * The library sketches an n x d fp32 row stream A into an ell x d sketch B with
 * the Frequent Directions family of arXiv:1501.06561 and evaluates
 * cov-err = ||A^T A - B^T B||_2 / ||A||_F^2.  Citations are to the paper text
 * (PAPER.md = the paper's LaTeX, line numbers) and to the readings C1..C20 of
 * DESIGN.md where the paper is silent or garbled.
 *
 *  - Alg. 1 (Generic FD): rows are inserted into zero rows
 *    of B; when none is left, [U,S,V] = svd(B), S' = ReduceRank(S), B = S'V^T.
 *  - ReduceRank rules: FD, Fast FD, iSVD
 *    (PAPER.md:248), alpha-FD / Alg. 2.
 *  - cov-err: PAPER.md:57.
 *
 * Conventions (apply to every function):
 *  - All matrices are row-major fp32 unless stated; `ld` is the row stride in
 *    ELEMENTS (ld >= d).
 *  - Pointers marked [device] are CUDA device pointers owned by the caller;
 *    pointers marked [host] are host pointers.  The library never allocates
 *    device memory: every device scratch comes from the caller's workspace
 *    (`ws`, `ws_bytes`), sized by the matching *_workspace_bytes() call.
 *  - Work is enqueued on the caller's CUDA stream (`cuda_stream`, a
 *    cudaStream_t; NULL = legacy default stream) and is stream-ordered and
 *    asynchronous unless the function returns host scalars (then it
 *    synchronises that stream before returning).
 *  - A handle is used by one host thread at a time; distinct handles may run
 *    concurrently.  Nothing throws across the ABI; every function returns an
 *    fd_status and fd_last_error() gives a thread-local message.
 */
#ifndef FD_H_
#define FD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fd_handle fd_handle; /* opaque */

typedef enum {
  FD_OK = 0,
  FD_ERR_INVALID_ARG = -1, /* NULL pointer, d < 1, ell < 2, alpha outside (0,1], n < 0 ...    */
  FD_ERR_SHAPE = -2,       /* ld < d, merging sketches of different (d, ell, variant)          */
  FD_ERR_ALIGNMENT = -3,   /* reserved: misaligned rows are accepted (scalar ingest path)       */
  FD_ERR_WORKSPACE = -4,   /* ws NULL or ws_bytes smaller than *_workspace_bytes()             */
  FD_ERR_NONFINITE = -5,   /* a non-finite input value was seen (sticky; see fd_append_rows)   */
  FD_ERR_ZERO_NORM = -6,   /* ||A||_F^2 = 0: cov-err undefined                   */
  FD_ERR_CUDA = -7,        /* a CUDA launch / copy failed (message in fd_last_error)           */
  FD_ERR_UNSUPPORTED = -8, /* eigen-problem size 2*ell (batched) or ell (per-row) above FD_MAX_N */
  FD_ERR_STATE = -9        /* handle refuses work after a sticky error                          */
} fd_status;

/* Variants.  "Per-row" = Alg. 1 verbatim: buffer capacity L = ell, one
 * ReduceRank per row once full.  "Fast"/batched = buffer capacity L = 2*ell,
 * one ReduceRank per ell+1 rows (PAPER.md:256 with the paper's buffer size
 * ell' = 2*ell, reading C1).  In every variant delta = sigma_ell^2 (the ell-th
 * largest squared singular value of the buffer, 1-based) and exactly ell-1
 * rows are kept after each ReduceRank (slot semantics, reading C6). */
typedef enum {
  FD_FD = 0,            /* FD rule sigma'^2 = max(sigma^2 - delta, 0), per-row   */
  FD_FAST_FD = 1,       /* FD rule, 2*ell buffer (C1)                             */
  FD_ALPHA_FD = 2,      /* Alg. 2: only the last m = max(1, round(alpha*ell)) values shrink,
                           per-row (C5)                                       */
  FD_FAST_ALPHA_FD = 3, /* Alg. 2 rule on the 2*ell buffer (C3)                                  */
  FD_ISVD = 4,          /* sigma'_j = sigma_j for j < ell, sigma'_ell = 0, per-row */
  FD_FAST_ISVD = 5,     /* iSVD rule on the 2*ell buffer                                         */
  FD_FAST_ALPHA_FD_PAPER = 6, /* paper-literal Fast alpha-FD: ell-row buffer,
                           delta = sigma_t^2 with t = ell - max(1, ceil(alpha*ell/2)); the last
                           m = max(1, round(alpha*ell)) values shrink; rows j <= max(ell-m, t-1)
                           are kept (C25).  Output: ell rows, rows >= that count 0 */
  FD_SSD = 7,           /* SpaceSaving Directions: Alg. 1 with ReduceRank-SS (Alg. 3):
                           delta = sigma_{ell-1}^2, sigma_{ell-1} -> 0, sigma_ell -> sqrt(sigma_ell^2 + delta);
                           per-row (C26) */
  FD_CFD = 8            /* Compensative FD: FD per-row, the final step returns
                           sqrt(sigma'^2 + Delta) on all ell directions; ReduceRank runs when a row
                           arrives at a full buffer (C27).  fd_merge: UNSUPPORTED */
} fd_variant;

/* Largest eigen-problem (buffer Gram) size supported by this build. */
#define FD_MAX_N 416

typedef struct {
  int64_t d;        /* row length (columns of A), >= 1                                     */
  int32_t ell;      /* sketch rows, >= 2; buffer Gram size is ell (per-row) or 2*ell       */
  int32_t variant;  /* fd_variant                                                          */
  double alpha;     /* alpha-FD parameter in (0,1]; ignored by the other variants          */
  int32_t n_shards; /* P >= 1 independent row streams (reading C10): every append call's  *
                     * rows are split into P contiguous ranges; fd_sketch merges the P    *
                     * shard sketches by a recursive-halving pairwise tree.               */
  int32_t device;   /* CUDA device ordinal the workspace lives on                          */
} fd_config;

typedef struct {
  int64_t rows_seen;   /* rows appended so far                                         */
  int64_t n_shrinks;   /* ReduceRank calls (row shrinks + final + merges)              */
  double frob_sq;      /* ||A||_F^2 of the rows seen (fp64 accumulation)               */
  double delta_total;  /* Delta = sum_i delta_i, incl. final and merges */
  double removed_mass; /* sum over ReduceRanks of sum_j (lambda_j - sigma'_j^2);       *
                        * equals ||A||_F^2 - ||B||_F^2 (Lemma 3)      */
  int32_t nonfinite;   /* 1 if a non-finite input was seen                             */
} fd_stats;

/* Bytes of device workspace fd_create needs for this config (0 on invalid config). */
size_t fd_workspace_bytes(const fd_config* cfg);

/* Create a handle.  ws [device] must stay valid until fd_destroy; ws_bytes >=
 * fd_workspace_bytes(cfg).  cuda_stream: the stream all work is enqueued on.
 * Errors: INVALID_ARG (cfg NULL/out NULL, d < 1, ell < 2, n_shards < 1, alpha
 * outside (0,1] for the alpha variants, unknown variant), UNSUPPORTED (Gram size
 * > FD_MAX_N), WORKSPACE, CUDA. */
fd_status fd_create(const fd_config* cfg, void* ws, size_t ws_bytes, void* cuda_stream, fd_handle** out);

/* Append n_rows rows (row-major, row stride ld elements) to the stream.
 * rows [device]: read asynchronously — must stay valid until the stream
 * passes this call.  The rows are split into n_shards contiguous ranges
 * (sizes floor(n/P) + (s < n mod P)) and each range is streamed, in order,
 * into its shard (Alg. 1 row loop).  Asynchronous.
 * Non-finite values set a sticky device flag, reported as FD_ERR_NONFINITE
 * by the next synchronising call; after that the handle returns FD_ERR_STATE.
 * Errors: INVALID_ARG (n_rows < 0, rows NULL with n_rows > 0), SHAPE (ld < d),
 * STATE, CUDA. */
fd_status fd_append_rows(fd_handle* h, const float* rows, int64_t n_rows, int64_t ld);

/* Append n_rows rows that live in HOST memory (row stride ld elements;
 * host_rows should be page-locked for the copies to overlap).  Same semantics
 * and shard split as fd_append_rows (Alg. 1 row loop; reading
 * C10): each lockstep round's rows are copied host -> device into `stage`
 * [device] (one 2-D copy per run of equally sized shard chunks, on an internal
 * copy stream) while the previous round computes.  stage_bytes >=
 * fd_host_stage_bytes(cfg, ld).  host_rows must stay valid and unmodified until
 * the handle's stream passes this call.  Errors: as fd_append_rows, plus
 * WORKSPACE (stage too small). */
size_t fd_host_stage_bytes(const fd_config* cfg, int64_t ld);
fd_status fd_append_rows_host(fd_handle* h, const float* host_rows, int64_t n_rows, int64_t ld, void* stage,
                              size_t stage_bytes);

/* Snapshot sketch (non-destructive; appends may continue, reading C9): every
 * shard's buffer gets one more ReduceRank (Alg. 1 "return B = B_[n]" with the
 * final shrink of C9), then the P shard sketches are merged pairwise
 * (merge(X,Y) = ReduceRank([X;Y]), C10).  B_out [device]: ell x d, ld = d;
 * rows are orthogonal with non-increasing norms and row ell-1 is zero.
 * st [host]: NULL -> asynchronous; non-NULL -> synchronises and fills stats. */
fd_status fd_sketch(fd_handle* h, float* B_out, fd_stats* st);

/* Merge `count` sketches (count x ell x d, [device], each ell x d with ld = d,
 * e.g. the all-gathered per-GPU sketches) with the same recursive-halving tree
 * and this handle's rule; B_out [device] ell x d.  st [host] optional: only
 * the merge's own delta / removed / shrinks are reported (add the inputs'
 * stats yourself).  Errors: INVALID_ARG (count < 1), STATE, CUDA. */
fd_status fd_merge(fd_handle* h, const float* sketches, int32_t count, float* B_out, fd_stats* st);

/* Copy shard `shard`'s canonical sketch (one final ReduceRank of its buffer,
 * no merging) into B_out [device] (ell x d).  For sampled parity checks of
 * large runs.  Synchronises. */
fd_status fd_shard_sketch(fd_handle* h, int32_t shard, float* B_out);

/* Reset the stream state (empty sketch, zero statistics, sticky flag cleared)
 * keeping the workspace; stream-ordered.  Used to run a fresh pass with the
 * same handle. */
fd_status fd_reset(fd_handle* h);

/* Live per-kernel timing (for the bench's roofline).  enable != 0 records a
 * CUDA event pair (on the handle's stream) around every kernel launch.
 * fd_profile_read synchronises, writes per-kernel totals
 * {ingest, gram, eig, recon, trd, bt} (ms[k], launches[k], k < max_kernels)
 * since the last read, and returns the number of kernel kinds (6). */
fd_status fd_profile(fd_handle* h, int32_t enable);
int32_t fd_profile_read(fd_handle* h, double* ms, int64_t* launches, int32_t max_kernels);

/* Release the handle (the workspace belongs to the caller). */
fd_status fd_destroy(fd_handle* h);

/* ---------------- covariance-error evaluator ---------------- */

/* Workspace bytes for the evaluator functions at dimension d. */
size_t fd_cov_workspace_bytes(int64_t d);

/* Scratch bytes fd_cov_gram_partial needs at (n, d): the int8 digit planes of one row
 * chunk (<= 512 MiB), the per-CTA fp64 partial tiles and the column maxima. */
size_t fd_cov_gram_workspace_bytes(int64_t n, int64_t d);

/* AtA [device] (d x d fp64, row-major, full symmetric) += A^T A for the n rows
 * of A [device] (fp32, ld) on the tensor cores (tcgen05 kind::i8; reading E3):
 * per row chunk, column j is scaled by 2^(22 - e_j) (e_j = frexp exponent of the chunk's
 * max |a_ij|) and rounded to an integer of <= 23 bits, split exactly into three int8
 * digits; the digit products of weight 2^32, 2^24, 2^16 accumulate exactly in int32 TMEM
 * accumulators and drain to fp64.  Error vs the exact fp64 A^T A: <= ~2^-22 of
 * max|a_i| max|a_j| per row and term (~1e-11 of ||A||_F^2 in ||.||_2 on c4).  Fixed
 * reduction order (deterministic).  A non-finite input makes AtA NaN.  ws [device]:
 * fd_cov_gram_workspace_bytes(n, d) bytes (required: WORKSPACE otherwise).
 * Asynchronous. */
fd_status fd_cov_gram_partial(const float* A, int64_t n, int64_t ld, int64_t d, double* AtA,
                              void* ws, size_t ws_bytes, void* cuda_stream);

/* err = ||AtA - B^T B||_2 / frob_sq with B [device] (ell x d fp32, ld = d),
 * AtA [device] as produced by fd_cov_gram_partial (summed over ranks),
 * frob_sq = ||A||_F^2 [host scalar].  The extreme eigenvalues of the d x d
 * fp64 difference M are found by Lanczos with full re-orthogonalisation
 * (min(d, 512) steps).  Outputs [host]: err, lam_max and lam_min of M divided by
 * frob_sq (M is PSD for every variant, Lemma 1; lam_min is a check).
 * Synchronises.  Errors: ZERO_NORM (frob_sq <= 0), WORKSPACE, CUDA. */
fd_status fd_cov_err_from_gram(const double* AtA, const float* B, int32_t ell, int64_t d, double frob_sq,
                               double* err, double* lam_max, double* lam_min,
                               void* ws, size_t ws_bytes, void* cuda_stream);

/* frob_sq [host] = trace(AtA) = ||A||_F^2 (PAPER.md:57's denominator) of AtA
 * [device] (d x d fp64 from fd_cov_gram_partial, summed over ranks): the d
 * diagonal entries are copied to the host and summed in index order.
 * Synchronises the stream.  Errors: INVALID_ARG, CUDA. */
fd_status fd_cov_frob_from_gram(const double* AtA, int64_t d, double* frob_sq, void* cuda_stream);

/* Single-GPU convenience: AtA from A, then fd_cov_err_from_gram with
 * frob_sq = trace(A^T A).  A, B [device]. */
fd_status fd_cov_err(const float* A, int64_t n, int64_t ld, const float* B, int32_t ell, int64_t d,
                     double* err, double* lam_max, double* lam_min,
                     void* ws, size_t ws_bytes, void* cuda_stream);

/* ---- proj-err -------------------------------------------
 * proj-err(A, B) = ||A - pi_{B_k}(A)||_F^2 / ||A - A_k||_F^2   (the
 * paper uses k = 10).  B_k = span of the top-k right singular
 * vectors of B (fewer if rank B < k: singular values with s^2 <= 1e-12 s_1^2 are
 * dropped), found from B B^T = U S^2 U^T (fp64, parallel-ordering Jacobi) as
 * v_j = B^T u_j / s_j.  Numerator = frob_sq - sum_j v_j^T AtA v_j; denominator =
 * frob_sq - sum_{j<=k} lambda_j(AtA) with the top-k eigenvalues as Lanczos Ritz
 * values (min(d, 512) steps, full re-orthogonalisation; a top-k eigenvalue of
 * exact multiplicity > 1 is found once: DESIGN.md reading E2). */

/* Workspace bytes for fd_proj_err_from_gram / fd_proj_err (d, ell, k as passed). */
size_t fd_proj_workspace_bytes(int64_t d, int32_t ell, int32_t k);

/* proj-err of B [device] (ell x d fp32, ld = d) from AtA [device] (d x d fp64 as
 * produced by fd_cov_gram_partial, summed over ranks) and frob_sq = ||A||_F^2
 * [host].  Outputs [host]: proj_err, num = ||A - pi_{B_k}(A)||_F^2 and
 * den = ||A - A_k||_F^2 (either may be NULL except proj_err).  1 <= k <= d.
 * Synchronises.  Errors: INVALID_ARG, ZERO_NORM (frob_sq <= 0, or den <= 1e-8 frob_sq:
 * numerically rank A <= k, below the A^T A error of fd_cov_gram_partial), WORKSPACE, CUDA. */
fd_status fd_proj_err_from_gram(const double* AtA, const float* B, int32_t ell, int64_t d, double frob_sq,
                                int32_t k, double* proj_err, double* num, double* den,
                                void* ws, size_t ws_bytes, void* cuda_stream);

/* Single-GPU convenience: AtA from A [device] (fp32, ld), frob_sq = trace(A^T A),
 * then fd_proj_err_from_gram.  ws must hold fd_proj_workspace_bytes + round_up(d*d*8, 256)
 * + fd_cov_gram_workspace_bytes(n, d). */
fd_status fd_proj_err(const float* A, int64_t n, int64_t ld, const float* B, int32_t ell, int64_t d, int32_t k,
                      double* proj_err, void* ws, size_t ws_bytes, void* cuda_stream);

/* ---- Hashing / OSNAP -------------------------------------
 * B = S A with S = s stacked count-sketch matrices of ell/s rows each (PAPER.md:198-201:
 * "exactly 1 non-zero element per column ... -1 or +1", OSNAP "stacks s instances";
 * s = 1 is Hashing, the paper uses s = 4): row i of the stream is added to row
 * h_j(i) of block j with sign sigma_j(i), scaled 1/sqrt(s) (C28).  h and
 * sigma come from splitmix64 of (seed, i, j) with i the row's GLOBAL stream index. */

/* Workspace bytes of fd_hash_sketch at dimension d and ell. */
size_t fd_hash_workspace_bytes(int64_t d, int32_t ell);

/* B_acc [device] (ell x d fp64, row-major, caller-owned) += S A for the n rows of
 * A [device] (fp32, ld >= d), which are rows row0 .. row0+n-1 of the stream.  B is
 * linear in A, so successive calls (or ranks, by an all-reduce sum) add up.  Fixed
 * summation order (deterministic).  1 <= s <= 8, s | ell, ell * 512 B <= 200 KiB.
 * Asynchronous.  Errors: INVALID_ARG, SHAPE (ld < d), UNSUPPORTED, WORKSPACE, CUDA. */
fd_status fd_hash_sketch(const float* A, int64_t n, int64_t ld, int64_t d, int32_t ell, int32_t s, uint64_t seed,
                         int64_t row0, double* B_acc, void* ws, size_t ws_bytes, void* cuda_stream);

/* Thread-local message for the last error on this thread ("" if none). */
const char* fd_last_error(void);

/* Library version string. */
const char* fd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FD_H_ */
