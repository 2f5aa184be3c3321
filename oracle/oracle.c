/*
 * oracle.c — plain, slow, obviously-correct fp64 CPU oracle for the Frequent
 * Directions family (FD, Fast FD, alpha-FD, iSVD) and the covariance-error
 * evaluator of arXiv:1501.06561.
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` leg may load or call this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1501_06561_b200/), and neither includes the other.
 *
 * What it follows (PAPER.md = /root/reference/PAPER.md, line numbers):
 *   Alg. 1 (Generic FD), PAPER.md:227-243:
 *       insert a_i into a zero row; if no zero row: [U,S,V] = svd(B);
 *       S' = ReduceRank(S); B = S' V^T.
 *     svd(B) is computed from the eigen-decomposition of the Gram B B^T
 *     (B = U S V^T  =>  B B^T = U S^2 U^T and S' V^T = diag(S'/S) U^T B),
 *     with a cyclic two-sided Jacobi eigensolver in fp64.
 *   iSVD rule:      sigma'_j = sigma_j (j < ell), sigma'_ell = 0.
 *   FD rule:        sigma'_j = sqrt(sigma_j^2 - delta), delta = sigma_ell^2.
 *   Fast FD:        delta = sigma_{ell'/2}^2 in an ell'-row buffer,
 *                                 sigma'_j = max(0, sqrt(sigma_j^2 - delta)).
 *                                 Here ell' = L = 2*ell (reading C1 of DESIGN.md).
 *   alpha-FD (Alg. 2): delta = sigma_ell^2; only the last
 *                                 alpha*ell values shrink (m = max(1, round(alpha*ell)),
 *                                 reading C5).
 *   Delta = sum_i delta_i.
 *   paper-literal Fast alpha-FD: delta = sigma_t^2, t = ell - ceil(alpha ell/2),
 *                                 ell-row buffer (reading C25).
 *   SpaceSaving Directions (Alg. 3): delta = sigma_{ell-1}^2,
 *                                 S' = diag(sigma_1..sigma_{ell-2}, 0, sqrt(sigma_ell^2 + delta)).
 *   Compensative FD: FD, final step sigma_hat = sqrt(sigma'^2 + Delta).
 *   proj-err.
 *   cov-err = ||A^T A - B^T B||_2 / ||A||_F^2.
 * Slot semantics (reading C6), final ReduceRank (C9), shard ranges and the
 * recursive-halving merge tree (C10) are the DESIGN.md readings.
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"): SPEC hand examples of
 * each rule, Jacobi vs the 2x2 closed form and vs numpy eigh, the covariance-form
 * brute force on tiny inputs, Lemma 1 / Lemma 3 identities, the FD bounds,
 * exactness when rank(A) <= ell-1, cov-err closed forms, merge symmetry.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_RULE_FD 0   /* alpha-FD with alpha given; FD is alpha = 1 */
#define ORC_RULE_ISVD 1
#define ORC_RULE_CFD 4  /* Compensative FD: FD rule + compensated final step */
#define ORC_RULE_SS 3   /* SpaceSaving Directions, ReduceRank-SS (Alg. 3)  */
#define ORC_RULE_FD_T 2 /* paper-literal Fast alpha-FD: delta = sigma_t^2,
                           t = ell - ceil(alpha ell / 2), buffer of ell rows */

/* ------------------------------------------------------------------------ */
/* Symmetric eigen-decomposition: cyclic two-sided Jacobi (fp64).            */
/* A: n x n row-major symmetric (overwritten); V: n x n, column j = vector j. */
/* Returns number of sweeps, or -1 if not converged in 100 sweeps.           */
/* ------------------------------------------------------------------------ */
int oracle_jacobi_eig(double* A, int n, double* w, double* V) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) V[(size_t)i * n + j] = (i == j) ? 1.0 : 0.0;
  int sweep;
  for (sweep = 0; sweep < 100; ++sweep) {
    long rotations = 0;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        double apq = A[(size_t)p * n + q];
        double app = A[(size_t)p * n + p];
        double aqq = A[(size_t)q * n + q];
        if (apq == 0.0) continue;
        if (fabs(apq) <= 1e-17 * sqrt(fabs(app) * fabs(aqq))) continue;
        double theta = (aqq - app) / (2.0 * apq);
        double t;
        if (fabs(theta) > 1e150) t = 0.5 / theta;
        else t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0);
        double s = t * c;
        for (int k = 0; k < n; ++k) {
          if (k == p || k == q) continue;
          double akp = A[(size_t)k * n + p], akq = A[(size_t)k * n + q];
          double nkp = c * akp - s * akq;
          double nkq = s * akp + c * akq;
          A[(size_t)k * n + p] = nkp; A[(size_t)p * n + k] = nkp;
          A[(size_t)k * n + q] = nkq; A[(size_t)q * n + k] = nkq;
        }
        A[(size_t)p * n + p] = app - t * apq;
        A[(size_t)q * n + q] = aqq + t * apq;
        A[(size_t)p * n + q] = 0.0;
        A[(size_t)q * n + p] = 0.0;
        for (int k = 0; k < n; ++k) {
          double vkp = V[(size_t)k * n + p], vkq = V[(size_t)k * n + q];
          V[(size_t)k * n + p] = c * vkp - s * vkq;
          V[(size_t)k * n + q] = s * vkp + c * vkq;
        }
        rotations++;
      }
    }
    if (rotations == 0) break;
  }
  for (int i = 0; i < n; ++i) w[i] = A[(size_t)i * n + i];
  return sweep < 100 ? sweep : -1;
}

/* order[0..n) = indices sorted by w descending, ties by lower index (stable). */
static void sort_desc(const double* w, int n, int* order) {
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 1; i < n; ++i) { /* insertion sort: stable, n <= 1024 */
    int x = order[i];
    int j = i - 1;
    while (j >= 0 && w[order[j]] < w[x]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = x;
  }
}

/* ------------------------------------------------------------------------ */
/* ReduceRank on an L x d buffer (Alg. 1 lines "svd ... B = S'V^T").         */
/* ------------------------------------------------------------------------ */
typedef struct {
  double frob_sq;      /* sum of ||a_i||^2 of rows seen                    */
  double delta_total;  /* Delta = sum_i delta_i             */
  double removed;      /* sum over shrinks of sum_j (lambda_j - sigma'_j^2) */
  int64_t n_shrinks;
  int64_t rows_seen;
} orc_stats;

typedef struct {
  int L, ell, rule, m;
  int t;   /* delta = lambda_t (1-based): ell for every rule but ORC_RULE_FD_T     */
  double comp;  /* >= 0: Compensative FD final step with this Delta */
  int R;   /* rows kept after a ReduceRank (slot semantics, C6): ell-1, or R_t    */
  int64_t d;
  double *G, *V, *lam, *w, *Bn;
  int* order;
} orc_work;

/* Paper-literal Fast alpha-FD: "delta_i = sigma_t^2 for
 * t = ell - ell alpha/2", "only changing the last alpha ell singular values:
 * sigma'_j^2 = max(sigma_j^2 - delta_i, 0)".  Integer reading (C25):
 * t = ell - max(1, ceil(alpha ell / 2)), m = max(1, round(alpha ell)) (C5); the
 * rows that can stay nonzero are j <= max(ell - m, t - 1), which are kept. */
static void fd_t_indices(int ell, double alpha, int* t, int* R) {
  int h = (int)ceil(alpha * (double)ell / 2.0 - 1e-9);
  if (h < 1) h = 1;
  int m = (int)llround(alpha * ell);
  if (m < 1) m = 1;
  *t = ell - h;
  *R = (ell - m > *t - 1) ? ell - m : *t - 1;
}

static int work_init(orc_work* W, int L, int64_t d, int ell, int rule, int m) {
  W->L = L; W->d = d; W->ell = ell; W->rule = rule; W->m = m;
  W->t = ell; W->R = ell - 1; W->comp = -1.0;
  W->G = malloc(sizeof(double) * L * L);
  W->V = malloc(sizeof(double) * L * L);
  W->lam = malloc(sizeof(double) * L);
  W->w = malloc(sizeof(double) * L);
  W->Bn = malloc(sizeof(double) * (size_t)L * d);
  W->order = malloc(sizeof(int) * L);
  return (W->G && W->V && W->lam && W->w && W->Bn && W->order) ? 0 : -1;
}

static void work_free(orc_work* W) {
  free(W->G); free(W->V); free(W->lam); free(W->w); free(W->Bn); free(W->order);
}

/* Bf: L x d (fp64, row-major), all L rows used (free slots are zero rows).
 * On return rows 0..ell-2 hold S'V^T (descending), rows ell-1..L-1 are zero. */
static int reduce_rank(orc_work* W, double* Bf, orc_stats* st) {
  const int L = W->L, ell = W->ell;
  const int64_t d = W->d;
  /* G = Bf Bf^T */
  for (int i = 0; i < L; ++i)
    for (int j = 0; j <= i; ++j) {
      const double* a = Bf + (size_t)i * d;
      const double* b = Bf + (size_t)j * d;
      double s = 0.0;
      for (int64_t k = 0; k < d; ++k) s += a[k] * b[k];
      W->G[(size_t)i * L + j] = s;
      W->G[(size_t)j * L + i] = s;
    }
  if (oracle_jacobi_eig(W->G, L, W->lam, W->V) < 0) return -1;
  sort_desc(W->lam, L, W->order);
  double lam_sorted[1024];
  double* lams = (L <= 1024) ? lam_sorted : malloc(sizeof(double) * L);
  for (int j = 0; j < L; ++j) {
    double v = W->lam[W->order[j]];
    lams[j] = v > 0.0 ? v : 0.0; /* clamp (reading C8) */
  }
  /* delta = lambda_t (1-based), i.e. sigma_t^2: t = ell except the paper-literal
   * Fast alpha-FD */
  double delta = (W->t <= L) ? lams[W->t - 1] : 0.0;
  double removed = 0.0;
  int src_last = -1;   /* SS: output row ell-2 takes direction ell-1 (0-based) */
  if (W->rule == ORC_RULE_SS) {
    /* ReduceRank-SS: delta = sigma_{ell-1}^2; return diag(sigma_1..sigma_{ell-2}, 0,
     * sqrt(sigma_ell^2 + delta)).  Slot semantics: the direction of sigma_ell is kept
     * in row ell-2 (0-based), row ell-1 is the free slot.  Reading C26: if sigma_ell = 0
     * (buffer rank <= ell-1; sigma_ell^2 <= 1e-12 sigma_1^2, the fp64 eigensolver's
     * resolution) the step is lossless (delta = 0, nothing moves). */
    delta = 0.0;
    if (ell <= L && lams[ell - 1] > 1e-12 * lams[0]) { delta = lams[ell - 2]; src_last = ell - 1; }
  }
  double sp2s[1024];
  double* sp2v = (L <= 1024) ? sp2s : malloc(sizeof(double) * L);
  for (int j = 0; j < L; ++j) {
    double sp2; /* sigma'_j^2 for 0-based j */
    if (W->rule == ORC_RULE_SS) {
      if (src_last >= 0) sp2 = (j < ell - 2) ? lams[j] : (j == ell - 1 ? lams[j] + delta : 0.0);
      else sp2 = (j < ell - 1) ? lams[j] : 0.0;
    }
    else if (j >= W->R) sp2 = 0.0; /* rows R.. are freed; sigma'_ell = 0 in every rule */
    else if (W->rule == ORC_RULE_ISVD) sp2 = lams[j];
    else if (j < ell - W->m) sp2 = lams[j]; /* alpha-FD: first ell-m unchanged */
    else sp2 = (lams[j] - delta > 0.0) ? lams[j] - delta : 0.0;
    removed += lams[j] - sp2;
    sp2v[j] = sp2;
  }
  /* Compensative FD, final step: sigma_hat_j = sqrt(sigma'_j^2 + Delta)
   * for every one of the ell directions, Delta including this step's delta.  A
   * direction with sigma_j = 0 has no defined v_j here and gets nothing (reading C27). */
  int nout = (W->rule == ORC_RULE_SS) ? ell - 1 : W->R;
  if (W->comp >= 0.0) {
    const double Dt = W->comp + delta;
    nout = ell;
    for (int j = 0; j < ell && j < L; ++j) {
      const double add = (lams[j] > 0.0) ? Dt : 0.0;
      removed -= add;
      sp2v[j] += add;
    }
  }
  for (int j = 0; j < L; ++j) W->w[j] = (lams[j] > 0.0) ? sqrt(sp2v[j]) / sqrt(lams[j]) : 0.0;
  /* B'_j = w_j * u_j^T Bf  (u_j = column order[j] of V) */
  memset(W->Bn, 0, sizeof(double) * (size_t)L * d);
  for (int j = 0; j < nout && j < L; ++j) {
    const int sj = (src_last >= 0 && j == ell - 2) ? src_last : j;
    double wj = W->w[sj];
    if (wj == 0.0) continue;
    int c = W->order[sj];
    double* out = W->Bn + (size_t)j * d;
    for (int r = 0; r < L; ++r) {
      double coef = wj * W->V[(size_t)r * L + c];
      if (coef == 0.0) continue;
      const double* in = Bf + (size_t)r * d;
      for (int64_t k = 0; k < d; ++k) out[k] += coef * in[k];
    }
  }
  if (sp2v != sp2s) free(sp2v);
  memcpy(Bf, W->Bn, sizeof(double) * (size_t)L * d);
  st->delta_total += delta;
  st->removed += removed;
  st->n_shrinks += 1;
  if (lams != lam_sorted) free(lams);
  return 0;
}

/* Exported for rule-level tests: apply ReduceRank to a given buffer. */
int oracle_reduce_rank(double* Bf, int L, int64_t d, int ell, int rule, int m, double* stats3) {
  orc_work W;
  if (work_init(&W, L, d, ell, rule, m)) return -2;
  orc_stats st = {0};
  int rc = reduce_rank(&W, Bf, &st);
  work_free(&W);
  if (stats3) { stats3[0] = st.delta_total; stats3[1] = st.removed; stats3[2] = (double)st.n_shrinks; }
  return rc;
}

/* Rule-level entry for the paper-literal Fast alpha-FD: delta = lambda_t, rows
 * 0..R-1 kept (t, R as fd_t_indices gives them for (ell, alpha)). */
int oracle_reduce_rank_t(double* Bf, int L, int64_t d, int ell, double alpha, double* stats3) {
  orc_work W;
  int m = (int)llround(alpha * ell);
  if (m < 1) m = 1;
  if (work_init(&W, L, d, ell, ORC_RULE_FD_T, m)) return -2;
  fd_t_indices(ell, alpha, &W.t, &W.R);
  orc_stats st = {0};
  int rc = reduce_rank(&W, Bf, &st);
  work_free(&W);
  if (stats3) { stats3[0] = st.delta_total; stats3[1] = st.removed; stats3[2] = (double)st.n_shrinks; }
  return rc;
}

/* ------------------------------------------------------------------------ */
/* One shard: Alg. 1 row loop with slot semantics, then a final ReduceRank.   */
/* rows: pointers to the shard's row segments (one per append call).          */
/* ------------------------------------------------------------------------ */
typedef struct {
  const float* A; int64_t lda, d;
  const int64_t* seg_start; const int64_t* seg_len; int nseg;
  int L, ell, rule, m, t, R;
  int comp_final;  /* Compensative FD with P = 1: the shard's final ReduceRank compensates */
  int lazy;        /* Compensative FD: ReduceRank when a row arrives at a full buffer, so the
                      final step (C9) is the last full-buffer SVD (reading C27) */
  double* B_out;   /* ell x d */
  orc_stats st;
  int rc;
} orc_shard_job;

static void run_shard(orc_shard_job* J) {
  orc_work W;
  if (work_init(&W, J->L, J->d, J->ell, J->rule, J->m)) { J->rc = -2; return; }
  W.t = J->t; W.R = J->R;
  const int64_t d = J->d;
  double* Bf = calloc((size_t)J->L * d, sizeof(double));
  memset(&J->st, 0, sizeof(J->st));
  int occ = 0;
  J->rc = 0;
  for (int s = 0; s < J->nseg && J->rc == 0; ++s) {
    for (int64_t r = 0; r < J->seg_len[s]; ++r) {
      const float* a = J->A + (J->seg_start[s] + r) * J->lda;
      if (J->lazy && occ == J->L) {
        if (reduce_rank(&W, Bf, &J->st)) { J->rc = -1; break; }
        occ = J->R;
      }
      double* slot = Bf + (size_t)occ * d;
      double nrm = 0.0;
      for (int64_t k = 0; k < d; ++k) { slot[k] = (double)a[k]; nrm += slot[k] * slot[k]; }
      J->st.frob_sq += nrm;
      J->st.rows_seen += 1;
      occ += 1;
      if (!J->lazy && occ == J->L) {
        if (reduce_rank(&W, Bf, &J->st)) { J->rc = -1; break; }
        occ = J->R;
      }
    }
  }
  if (J->comp_final) W.comp = J->st.delta_total;
  if (J->rc == 0 && reduce_rank(&W, Bf, &J->st)) J->rc = -1; /* final ReduceRank (C9) */
  memcpy(J->B_out, Bf, sizeof(double) * (size_t)J->ell * d);
  free(Bf);
  work_free(&W);
}

typedef struct {
  orc_shard_job* jobs; int njobs; int next; pthread_mutex_t mu;
} orc_pool;

static void* pool_worker(void* arg) {
  orc_pool* P = (orc_pool*)arg;
  for (;;) {
    pthread_mutex_lock(&P->mu);
    int j = P->next++;
    pthread_mutex_unlock(&P->mu);
    if (j >= P->njobs) break;
    run_shard(&P->jobs[j]);
  }
  return NULL;
}

/* merge(X, Y) = ReduceRank([X; Y]) with L = 2 ell (reading C10). */
static int merge2(const double* X, const double* Y, int64_t d, int ell, int rule, int m, int t, int R,
                  double comp, double* out, orc_stats* st) {
  orc_work W;
  if (work_init(&W, 2 * ell, d, ell, rule, m)) return -2;
  W.t = t; W.R = R; W.comp = comp;
  double* Bf = malloc(sizeof(double) * (size_t)2 * ell * d);
  memcpy(Bf, X, sizeof(double) * (size_t)ell * d);
  memcpy(Bf + (size_t)ell * d, Y, sizeof(double) * (size_t)ell * d);
  int rc = reduce_rank(&W, Bf, st);
  memcpy(out, Bf, sizeof(double) * (size_t)ell * d);
  free(Bf);
  work_free(&W);
  return rc;
}

/* Recursive-halving tree over sketches [lo, hi): left half has ceil((hi-lo)/2). */
/* comp_root: Compensative FD -- the root merge (the last ReduceRank of the DAG) is
 * the compensated final step, with Delta = everything accumulated before it. */
static int merge_tree(double* S, int lo, int hi, int64_t d, int ell, int rule, int m, int t, int R,
                      int comp_root, double* out, orc_stats* st) {
  size_t sz = (size_t)ell * d;
  if (hi - lo == 1) { memcpy(out, S + (size_t)lo * sz, sizeof(double) * sz); return 0; }
  int mid = lo + (hi - lo + 1) / 2;
  double* X = malloc(sizeof(double) * sz);
  double* Y = malloc(sizeof(double) * sz);
  int rc = merge_tree(S, lo, mid, d, ell, rule, m, t, R, 0, X, st);
  if (!rc) rc = merge_tree(S, mid, hi, d, ell, rule, m, t, R, 0, Y, st);
  if (!rc) rc = merge2(X, Y, d, ell, rule, m, t, R, comp_root ? st->delta_total : -1.0, out, st);
  free(X); free(Y);
  return rc;
}

/* rule ORC_RULE_FD_T: alpha = the variant's alpha (t, R from fd_t_indices);
 * other rules: alpha unused beyond m. */
int oracle_merge(const double* sketches, int count, int64_t d, int ell, int rule, int m, double alpha,
                 double* B_out, double* stats5) {
  if (count < 1 || rule == ORC_RULE_CFD) return -3;   /* CFD: no merge of finished sketches (C27) */
  int t = ell, R = ell - 1;
  if (rule == ORC_RULE_FD_T) fd_t_indices(ell, alpha, &t, &R);
  orc_stats st = {0};
  double* S = malloc(sizeof(double) * (size_t)count * ell * d);
  memcpy(S, sketches, sizeof(double) * (size_t)count * ell * d);
  int rc = merge_tree(S, 0, count, d, ell, rule, m, t, R, 0, B_out, &st);
  free(S);
  if (stats5) { stats5[0] = 0; stats5[1] = st.delta_total; stats5[2] = st.removed; stats5[3] = (double)st.n_shrinks; stats5[4] = 0; }
  return rc;
}

/*
 * Full sketch of A (n x d fp32, leading dim lda) with P shards.
 * appends: nappend sizes (sum = n) of the successive fd_append_rows calls
 * (NULL -> one call with all n rows).  Each call's rows are split into P
 * contiguous ranges, sizes floor(n_c/P) + (s < n_c mod P).
 * L = buffer capacity (ell: per-row mode, 2*ell: batched mode).
 * Outputs: B_out (ell x d), optionally shard_out (P x ell x d), stats5 =
 * {frob_sq, Delta, removed, n_shrinks, rows_seen}.
 */
int oracle_sketch(const float* A, int64_t n, int64_t lda, int64_t d, int ell, int rule,
                  double alpha, int L, int P, const int64_t* appends, int nappend,
                  int nthreads, double* B_out, double* shard_out, double* stats5) {
  if (ell < 2 || P < 1 || d < 1 || L < ell || lda < d) return -3;
  int m = ell;
  int tt = ell, RR = ell - 1;
  if (rule == ORC_RULE_FD_T) {
    if (!(alpha > 0.0 && alpha <= 1.0) || L != ell) return -3;
    m = (int)llround(alpha * ell);
    if (m < 1) m = 1;
    fd_t_indices(ell, alpha, &tt, &RR);
  }
  if (rule == ORC_RULE_FD) {
    if (!(alpha > 0.0 && alpha <= 1.0)) return -3;
    m = (int)llround(alpha * ell);
    if (m < 1) m = 1;
  }
  int64_t one[1] = {n};
  if (!appends) { appends = one; nappend = 1; }
  orc_shard_job* jobs = calloc(P, sizeof(orc_shard_job));
  int64_t* starts = malloc(sizeof(int64_t) * P * nappend);
  int64_t* lens = malloc(sizeof(int64_t) * P * nappend);
  double* S = malloc(sizeof(double) * (size_t)P * ell * d);
  int64_t base = 0;
  for (int c = 0; c < nappend; ++c) {
    int64_t nc = appends[c], q = nc / P, r = nc % P, off = base;
    for (int s = 0; s < P; ++s) {
      int64_t len = q + (s < r ? 1 : 0);
      starts[(size_t)s * nappend + c] = off;
      lens[(size_t)s * nappend + c] = len;
      off += len;
    }
    base += nc;
  }
  for (int s = 0; s < P; ++s) {
    orc_shard_job* J = &jobs[s];
    J->A = A; J->lda = lda; J->d = d;
    J->seg_start = starts + (size_t)s * nappend; J->seg_len = lens + (size_t)s * nappend; J->nseg = nappend;
    J->L = L; J->ell = ell; J->rule = rule; J->m = m; J->t = tt; J->R = RR;
    J->comp_final = (rule == ORC_RULE_CFD && P == 1);
    J->lazy = (rule == ORC_RULE_CFD);
    J->B_out = S + (size_t)s * ell * d;
  }
  if (nthreads < 1) nthreads = 1;
  if (nthreads > P) nthreads = P;
  orc_pool pool = {jobs, P, 0};
  pthread_mutex_init(&pool.mu, NULL);
  pthread_t* th = malloc(sizeof(pthread_t) * nthreads);
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, pool_worker, &pool);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&pool.mu);
  free(th);
  orc_stats tot = {0};
  int rc = 0;
  for (int s = 0; s < P; ++s) {
    if (jobs[s].rc) rc = jobs[s].rc;
    tot.frob_sq += jobs[s].st.frob_sq; tot.delta_total += jobs[s].st.delta_total;
    tot.removed += jobs[s].st.removed; tot.n_shrinks += jobs[s].st.n_shrinks;
    tot.rows_seen += jobs[s].st.rows_seen;
  }
  if (shard_out) memcpy(shard_out, S, sizeof(double) * (size_t)P * ell * d);
  if (!rc && B_out) rc = merge_tree(S, 0, P, d, ell, rule, m, tt, RR, rule == ORC_RULE_CFD, B_out, &tot);
  if (stats5) {
    stats5[0] = tot.frob_sq; stats5[1] = tot.delta_total; stats5[2] = tot.removed;
    stats5[3] = (double)tot.n_shrinks; stats5[4] = (double)tot.rows_seen;
  }
  free(jobs); free(starts); free(lens); free(S);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Evaluator: cov-err = ||A^T A - B^T B||_2 / ||A||_F^2.        */
/* ------------------------------------------------------------------------ */
typedef struct {
  const float* A; int64_t lda, d, r0, r1;
  double* C;   /* d x d partial (upper triangle used) */
  double frob;
} orc_gram_job;

static void* gram_worker(void* arg) {
  orc_gram_job* J = (orc_gram_job*)arg;
  const int64_t d = J->d;
  double* row = malloc(sizeof(double) * d);
  J->frob = 0.0;
  for (int64_t r = J->r0; r < J->r1; ++r) {
    const float* a = J->A + r * J->lda;
    for (int64_t k = 0; k < d; ++k) { row[k] = (double)a[k]; J->frob += row[k] * row[k]; }
    for (int64_t i = 0; i < d; ++i) {
      double ai = row[i];
      if (ai == 0.0) continue;
      double* Ci = J->C + i * d;
      for (int64_t j = i; j < d; ++j) Ci[j] += ai * row[j];
    }
  }
  free(row);
  return NULL;
}

/* AtA (d x d, full symmetric) = A^T A in fp64; returns ||A||_F^2 via frob. */
int oracle_gram(const float* A, int64_t n, int64_t lda, int64_t d, int nthreads, double* AtA, double* frob) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > n && n > 0) nthreads = (int)n;
  if (n == 0) nthreads = 1;
  orc_gram_job* jobs = calloc(nthreads, sizeof(orc_gram_job));
  pthread_t* th = malloc(sizeof(pthread_t) * nthreads);
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].A = A; jobs[t].lda = lda; jobs[t].d = d;
    jobs[t].r0 = n * t / nthreads; jobs[t].r1 = n * (t + 1) / nthreads;
    jobs[t].C = calloc((size_t)d * d, sizeof(double));
    pthread_create(&th[t], NULL, gram_worker, &jobs[t]);
  }
  memset(AtA, 0, sizeof(double) * (size_t)d * d);
  double f = 0.0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    for (int64_t i = 0; i < d; ++i)
      for (int64_t j = i; j < d; ++j) AtA[i * d + j] += jobs[t].C[i * d + j];
    f += jobs[t].frob;
    free(jobs[t].C);
  }
  for (int64_t i = 0; i < d; ++i)
    for (int64_t j = 0; j < i; ++j) AtA[i * d + j] = AtA[j * d + i];
  *frob = f;
  free(jobs); free(th);
  return 0;
}

/* Lanczos with full (twice-iterated Gram-Schmidt) re-orthogonalisation on a
 * d x d symmetric M; the k x k tridiagonal is diagonalised by Jacobi.
 * Returns the extreme Ritz values. */
int oracle_lanczos_extremes(const double* M, int64_t d, int kmax, double* lmax, double* lmin) {
  int k = (int)(kmax < d ? kmax : d);
  double* Q = calloc((size_t)(k + 1) * d, sizeof(double));
  double* alpha = calloc(k, sizeof(double));
  double* beta = calloc(k + 1, sizeof(double));
  double* z = malloc(sizeof(double) * d);
  /* deterministic start vector */
  double nrm = 0.0;
  for (int64_t i = 0; i < d; ++i) { Q[i] = 1.0 + 0.001 * (double)((i * 7919) % 101); nrm += Q[i] * Q[i]; }
  nrm = sqrt(nrm);
  for (int64_t i = 0; i < d; ++i) Q[i] /= nrm;
  int steps = 0;
  for (int j = 0; j < k; ++j) {
    const double* q = Q + (size_t)j * d;
    for (int64_t r = 0; r < d; ++r) {
      double s = 0.0;
      const double* Mr = M + r * d;
      for (int64_t c = 0; c < d; ++c) s += Mr[c] * q[c];
      z[r] = s;
    }
    double a = 0.0;
    for (int64_t r = 0; r < d; ++r) a += q[r] * z[r];
    alpha[j] = a;
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i <= j; ++i) {
        const double* qi = Q + (size_t)i * d;
        double h = 0.0;
        for (int64_t r = 0; r < d; ++r) h += qi[r] * z[r];
        for (int64_t r = 0; r < d; ++r) z[r] -= h * qi[r];
      }
    double b = 0.0;
    for (int64_t r = 0; r < d; ++r) b += z[r] * z[r];
    b = sqrt(b);
    steps = j + 1;
    beta[j + 1] = b;
    if (b <= 1e-13 * (fabs(a) + 1e-300) || j + 1 == k) break;
    double* qn = Q + (size_t)(j + 1) * d;
    for (int64_t r = 0; r < d; ++r) qn[r] = z[r] / b;
  }
  double* T = calloc((size_t)steps * steps, sizeof(double));
  double* V = malloc(sizeof(double) * steps * steps);
  double* w = malloc(sizeof(double) * steps);
  for (int i = 0; i < steps; ++i) {
    T[(size_t)i * steps + i] = alpha[i];
    if (i + 1 < steps) { T[(size_t)i * steps + i + 1] = beta[i + 1]; T[(size_t)(i + 1) * steps + i] = beta[i + 1]; }
  }
  int rc = oracle_jacobi_eig(T, steps, w, V) < 0 ? -1 : 0;
  double hi = -1e308, lo = 1e308;
  for (int i = 0; i < steps; ++i) { if (w[i] > hi) hi = w[i]; if (w[i] < lo) lo = w[i]; }
  *lmax = hi; *lmin = lo;
  free(Q); free(alpha); free(beta); free(z); free(T); free(V); free(w);
  return rc;
}

/* Extreme eigenvalues of symmetric M (d x d): full Jacobi when d <= jacobi_max,
 * otherwise Lanczos (kmax steps).  M is not modified. */
int oracle_sym_extremes(const double* M, int64_t d, int jacobi_max, int kmax, double* lmax, double* lmin) {
  if (d <= jacobi_max) {
    double* Mc = malloc(sizeof(double) * d * d);
    double* V = malloc(sizeof(double) * d * d);
    double* w = malloc(sizeof(double) * d);
    memcpy(Mc, M, sizeof(double) * d * d);
    int rc = oracle_jacobi_eig(Mc, (int)d, w, V) < 0 ? -1 : 0;
    double hi = -1e308, lo = 1e308;
    for (int64_t i = 0; i < d; ++i) { if (w[i] > hi) hi = w[i]; if (w[i] < lo) lo = w[i]; }
    *lmax = hi; *lmin = lo;
    free(Mc); free(V); free(w);
    return rc;
  }
  return oracle_lanczos_extremes(M, d, kmax, lmax, lmin);
}

/* cov-err of sketch B (ell x d, fp64) for A (n x d fp32).
 * out4 = {err, lambda_max(M)/frob, lambda_min(M)/frob, frob} with M = A^T A - B^T B;
 * err = max(|lambda_max|, |lambda_min|) / frob = ||M||_2 / ||A||_F^2. */
int oracle_cov_err(const float* A, int64_t n, int64_t lda, int64_t d, const double* B, int ell,
                   int nthreads, int jacobi_max, int kmax, double* out4) {
  double* M = malloc(sizeof(double) * d * d);
  double frob = 0.0;
  oracle_gram(A, n, lda, d, nthreads, M, &frob);
  for (int r = 0; r < ell; ++r) {
    const double* b = B + (size_t)r * d;
    for (int64_t i = 0; i < d; ++i) {
      if (b[i] == 0.0) continue;
      for (int64_t j = 0; j < d; ++j) M[i * d + j] -= b[i] * b[j];
    }
  }
  if (frob <= 0.0) { free(M); return -4; }
  double lmax, lmin;
  int rc = oracle_sym_extremes(M, d, jacobi_max, kmax, &lmax, &lmin);
  double nrm = fabs(lmax) > fabs(lmin) ? fabs(lmax) : fabs(lmin);
  out4[0] = nrm / frob; out4[1] = lmax / frob; out4[2] = lmin / frob; out4[3] = frob;
  free(M);
  return rc;
}

/* Ritz values of Lanczos (full re-orthogonalisation, as oracle_lanczos_extremes)
 * on symmetric M, the top `ntop` of them descending into top[].  Returns the
 * number of Lanczos steps, or -1. */
static int lanczos_top(const double* M, int64_t d, int kmax, int ntop, double* top) {
  int k = (int)(kmax < d ? kmax : d);
  double* Q = calloc((size_t)(k + 1) * d, sizeof(double));
  double* alpha = calloc(k, sizeof(double));
  double* beta = calloc(k + 1, sizeof(double));
  double* z = malloc(sizeof(double) * d);
  double nrm = 0.0;
  for (int64_t i = 0; i < d; ++i) { Q[i] = 1.0 + 0.001 * (double)((i * 7919) % 101); nrm += Q[i] * Q[i]; }
  nrm = sqrt(nrm);
  for (int64_t i = 0; i < d; ++i) Q[i] /= nrm;
  int steps = 0;
  for (int j = 0; j < k; ++j) {
    const double* q = Q + (size_t)j * d;
    for (int64_t r = 0; r < d; ++r) {
      double s = 0.0;
      for (int64_t c = 0; c < d; ++c) s += M[r * d + c] * q[c];
      z[r] = s;
    }
    double a = 0.0;
    for (int64_t r = 0; r < d; ++r) a += q[r] * z[r];
    alpha[j] = a;
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i <= j; ++i) {
        const double* qi = Q + (size_t)i * d;
        double h = 0.0;
        for (int64_t r = 0; r < d; ++r) h += qi[r] * z[r];
        for (int64_t r = 0; r < d; ++r) z[r] -= h * qi[r];
      }
    double b = 0.0;
    for (int64_t r = 0; r < d; ++r) b += z[r] * z[r];
    b = sqrt(b);
    steps = j + 1;
    beta[j + 1] = b;
    if (b <= 1e-13 * (fabs(a) + 1e-300) || j + 1 == k) break;
    double* qn = Q + (size_t)(j + 1) * d;
    for (int64_t r = 0; r < d; ++r) qn[r] = z[r] / b;
  }
  double* T = calloc((size_t)steps * steps, sizeof(double));
  double* V = malloc(sizeof(double) * steps * steps);
  double* w = malloc(sizeof(double) * steps);
  int* ord = malloc(sizeof(int) * steps);
  for (int i = 0; i < steps; ++i) {
    T[(size_t)i * steps + i] = alpha[i];
    if (i + 1 < steps) { T[(size_t)i * steps + i + 1] = beta[i + 1]; T[(size_t)(i + 1) * steps + i] = beta[i + 1]; }
  }
  int rc = oracle_jacobi_eig(T, steps, w, V) < 0 ? -1 : steps;
  sort_desc(w, steps, ord);
  for (int t = 0; t < ntop; ++t) top[t] = (t < steps) ? w[ord[t]] : 0.0;
  free(Q); free(alpha); free(beta); free(z); free(T); free(V); free(w); free(ord);
  return rc;
}

/* proj-err (k = 10 in the experiments):
 *   proj-err(A, B) = ||A - pi_{B_k}(A)||_F^2 / ||A - A_k||_F^2.
 * B_k = span of the top-k right singular vectors of B ("the best rank k subspace
 * described by B"), from the Jacobi eigen-decomposition of B B^T = U S^2 U^T:
 * v_j = B^T u_j / s_j for the top min(k, rank B) values (s_j^2 > 1e-12 s_1^2).
 * With V_k orthonormal, ||A - A V_k V_k^T||_F^2 = ||A||_F^2 - sum_j v_j^T (A^T A) v_j,
 * and ||A - A_k||_F^2 = ||A||_F^2 - sum_{j<=k} lambda_j(A^T A) (Eckart-Young), the
 * top-k eigenvalues by full Jacobi when d <= jacobi_max, else Lanczos Ritz values.
 * B: ell x d fp64 row-major.  out4 = {proj_err, numerator, denominator, frob}.
 * Returns 0, -4 (||A||_F = 0), -5 (||A - A_k||_F = 0: undefined), -1. */
int oracle_proj_err(const float* A, int64_t n, int64_t lda, int64_t d, const double* B, int ell, int k,
                    int nthreads, int jacobi_max, int kmax, double* out4) {
  double* M = malloc(sizeof(double) * d * d);
  double frob = 0.0;
  oracle_gram(A, n, lda, d, nthreads, M, &frob);
  if (frob <= 0.0) { free(M); return -4; }
  /* B B^T and its eigen-decomposition */
  double* G = malloc(sizeof(double) * ell * ell);
  double* U = malloc(sizeof(double) * ell * ell);
  double* s2 = malloc(sizeof(double) * ell);
  int* ord = malloc(sizeof(int) * ell);
  for (int i = 0; i < ell; ++i)
    for (int j = 0; j < ell; ++j) {
      double s = 0.0;
      for (int64_t c = 0; c < d; ++c) s += B[(size_t)i * d + c] * B[(size_t)j * d + c];
      G[(size_t)i * ell + j] = s;
    }
  int rc = oracle_jacobi_eig(G, ell, s2, U) < 0 ? -1 : 0;
  sort_desc(s2, ell, ord);
  double captured = 0.0;
  double* v = malloc(sizeof(double) * d);
  const double smax = ell > 0 ? s2[ord[0]] : 0.0;
  for (int t = 0; t < k && t < ell; ++t) {
    const int j = ord[t];
    if (!(s2[j] > 1e-12 * smax) || s2[j] <= 0.0) break;
    const double inv = 1.0 / sqrt(s2[j]);
    for (int64_t c = 0; c < d; ++c) {
      double x = 0.0;
      for (int i = 0; i < ell; ++i) x += B[(size_t)i * d + c] * U[(size_t)i * ell + j];
      v[c] = x * inv;
    }
    double q = 0.0;
    for (int64_t r = 0; r < d; ++r) {
      double mv = 0.0;
      for (int64_t c = 0; c < d; ++c) mv += M[r * d + c] * v[c];
      q += v[r] * mv;
    }
    captured += q;
  }
  /* top-k eigenvalues of A^T A */
  double* top = calloc(k > 0 ? k : 1, sizeof(double));
  if (d <= jacobi_max) {
    double* Mc = malloc(sizeof(double) * d * d);
    double* W = malloc(sizeof(double) * d * d);
    double* w = malloc(sizeof(double) * d);
    int* o2 = malloc(sizeof(int) * d);
    memcpy(Mc, M, sizeof(double) * d * d);
    if (oracle_jacobi_eig(Mc, (int)d, w, W) < 0) rc = -1;
    sort_desc(w, (int)d, o2);
    for (int t = 0; t < k; ++t) top[t] = (t < d) ? w[o2[t]] : 0.0;
    free(Mc); free(W); free(w); free(o2);
  } else if (lanczos_top(M, d, kmax, k, top) < 0) {
    rc = -1;
  }
  double best = 0.0;
  for (int t = 0; t < k; ++t) best += top[t];
  const double num = frob - captured, den = frob - best;
  out4[0] = (den > 0.0) ? num / den : 0.0;
  out4[1] = num; out4[2] = den; out4[3] = frob;
  if (rc == 0 && !(den > 0.0)) rc = -5;
  free(M); free(G); free(U); free(s2); free(ord); free(v); free(top);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Hashing / OSNAP.                    */
/* B = S A, S = s stacked count-sketch matrices of ell' = ell / s rows each:   */
/* row i of A is added to row h_j(i) of block j with sign sigma_j(i), scaled   */
/* 1/sqrt(s) (reading C28; s = 1 is Hashing, s = 4 OSNAP).  h and sigma come   */
/* from a counter-based generator (splitmix64 of (seed, i, j)), which the CUDA */
/* path implements separately.                                                 */
/* ------------------------------------------------------------------------ */
static uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* B (ell x d fp64) += S A for rows row0 .. row0 + n - 1 of the stream. */
int oracle_hash_sketch(const float* A, int64_t n, int64_t lda, int64_t d, int ell, int s, uint64_t seed,
                       int64_t row0, double* B) {
  if (s < 1 || ell < s || ell % s != 0) return -3;
  const int lb = ell / s;
  const double scale = 1.0 / sqrt((double)s);
  for (int64_t r = 0; r < n; ++r) {
    const uint64_t i = (uint64_t)(row0 + r);
    const float* a = A + r * lda;
    for (int j = 0; j < s; ++j) {
      const uint64_t x = orc_splitmix64(seed ^ (i * (uint64_t)s + (uint64_t)j) * 0xD1B54A32D192ED03ull);
      const int h = (int)(((uint64_t)(uint32_t)(x >> 32) * (uint64_t)lb) >> 32);   /* multiply-shift into [0, lb) */
      const double sg = (x & 1ull) ? -scale : scale;
      double* b = B + (size_t)(j * lb + h) * d;
      for (int64_t c = 0; c < d; ++c) b[c] += sg * (double)a[c];
    }
  }
  return 0;
}
