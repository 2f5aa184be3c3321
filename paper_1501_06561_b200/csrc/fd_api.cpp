// fd_api.cpp — C ABI of libfd (include/fd.h): handle, workspace carving, the
// lockstep round scheduler over shard streams, the merge tree and the
// evaluator entry points.  All arithmetic runs in the kernels of fd_kernels.cu.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "fd.h"
#include "fd_internal.h"

using fdk::Ingest;
using fdk::Params;
using fdk::Prob;
using fdk::Stats;

namespace {

thread_local std::string g_err;

fd_status fail(fd_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

fd_status cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return FD_ERR_CUDA;
}

#define FD_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e__ = (call);                           \
    if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
  } while (0)

constexpr size_t kAlign = 256;
constexpr int kMergeMax = 64;                 // fd_merge: max sketches per call
constexpr size_t kArenaHalf = 8u << 20;       // descriptor arena half (bytes)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Every handle entry point runs on the handle's device and restores the caller's.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DevGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

struct Layout {
  size_t buf0, buf1, nodes, G, Wt, stats, flag, eig, arena, state, total;
  int nnodes, nslots;
};

struct Derived {
  int64_t d, ldb;
  int ell, L, P, rule, m, ldg, nmax;
  int R;         // rows kept by a ReduceRank (ell-1; paper-literal Fast alpha-FD: max(ell-m, t-1))
  int t;         // delta = lambda_t (ell; paper-literal Fast alpha-FD: ell - ceil(alpha ell/2))
  bool cfd;      // Compensative FD: lazy ReduceRank + compensated final step (reading C27)
  bool perrow;   // Alg. 1 per-row chain (buffer L = ell)
  bool prk;      // per-row chain on the persistent per-row kernel (fd_perrow.cu, fp64 state)
  size_t gbytes; // element size of the Gram / Wt scratch
};

// Precision of a ReduceRank of size N: per-row chains run one
// dependent ReduceRank per row, so the sketch is built in fp64 there (fp32
// eigenvalue noise on rank-deficient buffers would be clamped at 0 and
// accumulate as a bias); batched buffers run in fp32.
bool use_f64(const Derived& D, int N) { return D.perrow && N <= fdk::kMaxN64; }

bool derive(const fd_config* c, Derived* D, std::string* why) {
  if (!c) { *why = "cfg is NULL"; return false; }
  if (c->d < 1) { *why = "d < 1"; return false; }
  if (c->ell < 2) { *why = "ell < 2"; return false; }
  if (c->n_shards < 1) { *why = "n_shards < 1"; return false; }
  if (c->variant < FD_FD || c->variant > FD_CFD) { *why = "unknown variant"; return false; }
  const bool literal = (c->variant == FD_FAST_ALPHA_FD_PAPER);
  const bool batched = (c->variant == FD_FAST_FD || c->variant == FD_FAST_ALPHA_FD || c->variant == FD_FAST_ISVD);
  const bool isvd = (c->variant == FD_ISVD || c->variant == FD_FAST_ISVD);
  const bool alpha_v = (c->variant == FD_ALPHA_FD || c->variant == FD_FAST_ALPHA_FD || literal);
  D->d = c->d;
  D->ldb = (c->d + 3) / 4 * 4;
  D->ell = c->ell;
  D->L = batched ? 2 * c->ell : c->ell;
  D->P = c->n_shards;
  D->rule = isvd ? fdk::RULE_ISVD : (c->variant == FD_SSD ? fdk::RULE_SS : fdk::RULE_FD);
  D->cfd = (c->variant == FD_CFD);
  D->m = c->ell;
  if (alpha_v) {
    if (!(c->alpha > 0.0 && c->alpha <= 1.0)) { *why = "alpha must be in (0,1]"; return false; }
    // m = max(1, round(alpha*ell)) (reading C5; round half away from zero)
    D->m = std::max(1, (int)(c->alpha * c->ell + 0.5));
  }
  D->R = c->ell - 1;
  D->t = c->ell;
  if (literal) {
    // paper-literal Fast alpha-FD (C25): an ell-row buffer,
    // delta = lambda_t, t = ell - max(1, ceil(alpha ell / 2)); rows j <= max(ell-m, t-1)
    // can stay nonzero and are kept, the others are free slots
    int h = (int)std::ceil(c->alpha * (double)c->ell / 2.0 - 1e-9);
    h = std::max(1, h);
    D->t = c->ell - h;
    D->R = std::max(c->ell - D->m, D->t - 1);
  }
  D->perrow = !batched && !literal;
  D->gbytes = D->perrow ? sizeof(double) : sizeof(float);
  D->nmax = std::max(D->L, 2 * D->R);
  if (c->n_shards == 1) D->nmax = D->L;  // merges only via fd_merge (checked there)
  D->ldg = (std::max(D->nmax, 2 * D->R) + 3) / 4 * 4;
  {
    Params q{};
    q.d = D->d; q.ell = D->ell; q.ret = D->R; q.tdel = D->t;
    D->prk = D->perrow && fdk::perrow_supported(D->ell, D->d, q);
  }
  return true;
}

// rows of a Wt slot: ell-1 weight rows (+1), or the N x 128 eigenvector block
// eig_kernel hands to bt_kernel (fd_bt.cu) in the tridiagonal-kernel path
size_t wt_rows(const Derived& D) { return (size_t)std::max(D.ell, 128); }

Layout layout(const Derived& D) {
  Layout Lo;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, kAlign); return o; };
  const size_t bufb = (size_t)D.P * D.L * D.ldb * sizeof(float);
  Lo.nnodes = std::max(2 * D.P - 1, 2 * kMergeMax - 1);
  Lo.nslots = std::max(D.P, kMergeMax);
  Lo.buf0 = take(bufb);
  Lo.buf1 = take(bufb);
  Lo.nodes = take((size_t)Lo.nnodes * D.ell * D.ldb * sizeof(float));
  Lo.G = take((size_t)Lo.nslots * D.ldg * D.ldg * D.gbytes);
  Lo.Wt = take((size_t)Lo.nslots * wt_rows(D) * D.ldg * D.gbytes);

  Lo.stats = take((size_t)(D.P + Lo.nnodes) * sizeof(Stats));
  Lo.flag = take(sizeof(int) * 4);
  Lo.eig = take(fdk::eig_scratch_bytes(D.ldg));
  Lo.arena = take(2 * kArenaHalf);
  Lo.state = D.prk ? take((size_t)D.P * D.ell * D.ldb * sizeof(double)) : 0;   // fp64 per-row state
  Lo.total = off;
  return Lo;
}

}  // namespace

struct fd_handle {
  fd_config cfg;
  Derived D;
  Params prm;
  Layout Lo;
  char* ws;
  cudaStream_t stream;
  int device;
  float* buf[2];
  float* nodes;
  char* G;
  char* Wt;
  Stats* stats;       // [P] shard stats, then [nnodes] node stats
  int* flag;
  double* eig;
  double* state;      // fp64 per-row state (D.prk): P x ell x ldb
  char* arena;        // device descriptor arena (2 halves)
  char* host_arena;   // pinned host mirror
  cudaEvent_t ev[2];
  cudaStream_t copy_stream;     // host-input staging (fd_append_rows_host)
  cudaEvent_t ev_copied[2], ev_consumed[2];
  cudaEvent_t ev_copied_desc;   // descriptor uploads on the copy stream (host-input path)
  int half;
  size_t half_used;
  size_t max_pitch;   // cudaDevAttrMaxPitch: larger 2-D copy pitches fall back to 1-D copies
  std::vector<int> occ, cur;
  int64_t rows_seen;
  bool dead;
  bool ingest_copy;   // FD_INGEST_COPY set: always copy new rows into the buffers (A/B checks)
  bool legacy_trd;    // FD_LEGACY_TRD set: tridiagonalise inside eig_kernel (A/B checks)
  bool simt_gemm;     // FD_SIMT_GEMM set: FP32 SIMT Gram / reconstruct instead of tcgen05 (A/B checks)
  bool simt_gram, simt_recon;  // per-GEMM variants (FD_SIMT_GRAM, FD_SIMT_RECON: the FP32 SIMT kernels, A/B only)
  // live profiling: event pairs around launches
  bool prof;
  struct Rec { int kind; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
};

namespace {

Stats* node_stats(fd_handle* h, int node) { return h->stats + h->D.P + node; }
float* node_buf(fd_handle* h, int node) { return h->nodes + (size_t)node * h->D.ell * h->D.ldb; }
float* shard_buf(fd_handle* h, int s, int which) { return h->buf[which] + (size_t)s * h->D.L * h->D.ldb; }

// Copy a block of descriptors to the device arena; returns the device pointer.
template <typename T>
fd_status push_desc(fd_handle* h, const std::vector<T>& v, const T** out, cudaStream_t sx = nullptr) {
  if (!sx) sx = h->stream;   // the host-input path uploads on the copy stream (append_impl)
  const size_t bytes = align_up(v.size() * sizeof(T), 64);
  if (bytes > kArenaHalf) return fail(FD_ERR_INVALID_ARG, "descriptor batch larger than arena");
  if (h->half_used + bytes > kArenaHalf) {
    // switch halves: the other half's previous H2D copies (either stream) must be done
    // before its pinned host mirror is overwritten
    FD_CUDA(cudaEventRecord(h->ev[h->half], h->stream));
    FD_CUDA(cudaEventRecord(h->ev_copied_desc, h->copy_stream));
    h->half ^= 1;
    FD_CUDA(cudaEventSynchronize(h->ev[h->half]));
    FD_CUDA(cudaEventSynchronize(h->ev_copied_desc));
    h->half_used = 0;
  }
  char* hp = h->host_arena + (size_t)h->half * kArenaHalf + h->half_used;
  char* dp = h->arena + (size_t)h->half * kArenaHalf + h->half_used;
  memcpy(hp, v.data(), v.size() * sizeof(T));
  FD_CUDA(cudaMemcpyAsync(dp, hp, v.size() * sizeof(T), cudaMemcpyHostToDevice, sx));
  h->half_used += bytes;
  *out = reinterpret_cast<const T*>(dp);
  return FD_OK;
}

enum { K_INGEST = 0, K_GRAM = 1, K_EIG = 2, K_RECON = 3, K_TRD = 4, K_BT = 5, K_PERROW = 6, K_COUNT = 7 };

cudaEvent_t get_event(fd_handle* h) {
  if (!h->pool.empty()) {
    cudaEvent_t e = h->pool.back();
    h->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// launch `f` on the handle's stream, bracketed by an event pair when profiling
template <typename F>
cudaError_t timed(fd_handle* h, int kind, F f) {
  if (!h->prof) return f();
  fd_handle::Rec r{kind, get_event(h), get_event(h)};
  cudaEventRecord(r.a, h->stream);
  cudaError_t e = f();
  cudaEventRecord(r.b, h->stream);
  h->recs.push_back(r);
  return e;
}

fd_status run_reduce(fd_handle* h, const std::vector<Prob>& probs, bool comp = false, bool merge = false,
                     const Prob* pushed = nullptr) {
  if (probs.empty()) return FD_OK;
  int nmax = 0;
  for (const Prob& p : probs) nmax = std::max(nmax, p.rows0 + p.rows1);
  const Prob* dp = pushed;
  if (!dp) {
    fd_status s = push_desc(h, probs, &dp);
    if (s != FD_OK) return s;
  }
  fd_status s = FD_OK;
  const int n = (int)probs.size();
  Params prm = h->prm;
  prm.merge = merge ? 1 : 0;
  if (comp) {   // Compensative FD final step: all ell directions get sigma'^2 + Delta
    prm.comp = 1;
    prm.ret = h->D.ell;
  }
  prm.f64 = use_f64(h->D, nmax) ? 1 : 0;
  prm.pretrd = (!h->legacy_trd && fdk::trd_supported(nmax, prm)) ? 1 : 0;
  cudaError_t e;
  const bool tc_gram = !h->simt_gram && fdk::gram_tc_supported(nmax, prm);
  if ((e = timed(h, K_GRAM, [&] {
         return tc_gram ? fdk::launch_gram_tc(dp, n, nmax, prm, h->stream) : fdk::launch_gram(dp, n, nmax, prm, h->stream);
       })) != cudaSuccess)
    return cuda_fail(e, "gram");
  if (prm.pretrd &&
      (e = timed(h, K_TRD, [&] { return fdk::launch_trd(dp, n, nmax, prm, h->stream); })) != cudaSuccess)
    return cuda_fail(e, "trd");
  if ((e = timed(h, K_EIG, [&] { return fdk::launch_eig(dp, n, prm, h->eig, h->stream); })) != cudaSuccess)
    return cuda_fail(e, "eig");
  if (prm.pretrd && (e = timed(h, K_BT, [&] { return fdk::launch_bt(dp, n, prm, h->stream); })) != cudaSuccess)
    return cuda_fail(e, "bt");
  const bool tc_recon = !h->simt_recon && fdk::recon_i8_supported(nmax, prm);
  if ((e = timed(h, K_RECON, [&] {
         return tc_recon ? fdk::launch_recon_i8(dp, n, nmax, prm, h->stream) : fdk::launch_recon(dp, n, nmax, prm, h->stream);
       })) != cudaSuccess)
    return cuda_fail(e, "recon");
  return FD_OK;
}

Prob make_prob(fd_handle* h, int slot, const float* s0, int r0, const float* s1, int r1, float* dst, Stats* st,
               const Stats* c0 = nullptr, const Stats* c1 = nullptr) {
  Prob p;
  p.src0 = s0; p.rows0 = r0;
  p.src1 = s1; p.rows1 = r1;
  p.dst = dst;
  p.G = h->G + (size_t)slot * h->D.ldg * h->D.ldg * h->D.gbytes;
  p.Wt = h->Wt + (size_t)slot * wt_rows(h->D) * h->D.ldg * h->D.gbytes;

  p.stats = st;
  p.child0 = c0; p.child1 = c1;
  p.ld1 = h->D.ldb;
  p.acc1 = 0;
  return p;
}

// Recursive-halving tree over leaves [lo, hi) (left half = ceil).  Appends
// internal nodes to `plan` as (left, right, node) and returns the root id.
struct Merge { int a, b, node, height; };
int build_tree(int lo, int hi, int* next_id, std::vector<Merge>* plan, std::vector<int>* height) {
  if (hi - lo == 1) return lo;
  const int mid = lo + (hi - lo + 1) / 2;
  const int a = build_tree(lo, mid, next_id, plan, height);
  const int b = build_tree(mid, hi, next_id, plan, height);
  const int id = (*next_id)++;
  const int hgt = std::max((*height)[a], (*height)[b]) + 1;
  if ((int)height->size() <= id) height->resize(id + 1, 0);
  (*height)[id] = hgt;
  plan->push_back({a, b, id, hgt});
  return id;
}

// Merge the `count` leaves already in node slots 0..count-1 (node stats set).
fd_status run_tree(fd_handle* h, int count, int* root, bool comp = false) {
  if (count == 1) { *root = 0; return FD_OK; }
  if (2 * h->D.R > fdk::kMaxN)
    return fail(FD_ERR_UNSUPPORTED, "merge Gram size 2*ell-2 exceeds FD_MAX_N");
  std::vector<Merge> plan;
  std::vector<int> height(count, 0);
  int next = count;
  *root = build_tree(0, count, &next, &plan, &height);
  int maxh = 0;
  for (const Merge& m : plan) maxh = std::max(maxh, m.height);
  const int R = h->D.R;
  for (int lvl = 1; lvl <= maxh; ++lvl) {
    std::vector<Prob> probs;
    for (const Merge& m : plan) {
      if (m.height != lvl) continue;
      const int slot = (int)probs.size();
      // [X; Y] without their zero last rows: Gram size 2R = 2*ell-2 (same nonzero spectrum)
      probs.push_back(make_prob(h, slot, node_buf(h, m.a), R, node_buf(h, m.b), R, node_buf(h, m.node),
                                node_stats(h, m.node), node_stats(h, m.a), node_stats(h, m.b)));
    }
    fd_status s = run_reduce(h, probs, comp && lvl == maxh, true);   // CFD: the root is the final step
    if (s != FD_OK) return s;
  }
  return FD_OK;
}

fd_status check_flag(fd_handle* h) {
  int flag = 0;
  FD_CUDA(cudaMemcpyAsync(&flag, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  FD_CUDA(cudaStreamSynchronize(h->stream));
  if (flag) {
    h->dead = true;
    return fail(FD_ERR_NONFINITE, "non-finite value in the appended rows");
  }
  return FD_OK;
}

fd_status read_stats(fd_handle* h, const Stats* dev, fd_stats* st) {
  Stats s;
  int flag = 0;
  FD_CUDA(cudaMemcpyAsync(&s, dev, sizeof(Stats), cudaMemcpyDeviceToHost, h->stream));
  FD_CUDA(cudaMemcpyAsync(&flag, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  FD_CUDA(cudaStreamSynchronize(h->stream));
  st->rows_seen = h->rows_seen;
  st->n_shrinks = (int64_t)(s.shrinks + 0.5);
  st->frob_sq = s.frob;
  st->delta_total = s.delta;
  st->removed_mass = s.removed;
  st->nonfinite = flag;
  if (flag) {
    h->dead = true;
    return fail(FD_ERR_NONFINITE, "non-finite value in the appended rows");
  }
  return FD_OK;
}

// Final ReduceRank of shards [s0, s1) into node slots (non-destructive snapshot).
fd_status finalize_shards(fd_handle* h, int s0, int s1, bool comp = false) {
  // leaf node stats start as copies of the shard stats
  FD_CUDA(cudaMemcpyAsync(node_stats(h, s0), h->stats + s0, sizeof(Stats) * (s1 - s0), cudaMemcpyDeviceToDevice,
                          h->stream));
  std::vector<Prob> probs;
  for (int s = s0; s < s1; ++s) {
    probs.push_back(make_prob(h, (int)probs.size(), shard_buf(h, s, h->cur[s]), h->occ[s], nullptr, 0,
                              node_buf(h, s), node_stats(h, s)));
  }
  return run_reduce(h, probs, comp);
}

}  // namespace

extern "C" {

size_t fd_workspace_bytes(const fd_config* cfg) {
  Derived D;
  std::string why;
  if (!derive(cfg, &D, &why)) return 0;
  return layout(D).total;
}

fd_status fd_create(const fd_config* cfg, void* ws, size_t ws_bytes, void* cuda_stream, fd_handle** out) {
  if (!out) return fail(FD_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  Derived D;
  std::string why;
  if (!derive(cfg, &D, &why)) return fail(FD_ERR_INVALID_ARG, why);
  if (D.L > fdk::kMaxN) return fail(FD_ERR_UNSUPPORTED, "buffer Gram size exceeds FD_MAX_N");
  if (D.P > 1 && 2 * D.R > fdk::kMaxN) return fail(FD_ERR_UNSUPPORTED, "merge Gram size exceeds FD_MAX_N");
  Layout Lo = layout(D);
  if (!ws || ws_bytes < Lo.total) return fail(FD_ERR_WORKSPACE, "workspace too small");
  fd_handle* h = new fd_handle();
  h->cfg = *cfg;
  h->D = D;
  h->Lo = Lo;
  h->ws = static_cast<char*>(ws);
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  h->device = cfg->device;
  h->prm.nonfinite = nullptr;   // set below with the flag
  h->prm.d = D.d; h->prm.ldb = D.ldb; h->prm.ldg = D.ldg; h->prm.ell = D.ell; h->prm.rule = D.rule; h->prm.m = D.m;
  h->prm.ret = D.R; h->prm.tdel = D.t; h->prm.comp = 0; h->prm.merge = 0;
  h->prm.f64 = 0;
  h->prm.pretrd = 0;
  h->prm.zld = D.ldg;
  h->legacy_trd = getenv("FD_LEGACY_TRD") != nullptr;
  h->ingest_copy = getenv("FD_INGEST_COPY") != nullptr;
  h->simt_gemm = getenv("FD_SIMT_GEMM") != nullptr;
  h->simt_gram = h->simt_gemm || getenv("FD_SIMT_GRAM") != nullptr;
  // FP32 SIMT reconstruct instead of the int8 tensor-core one (A/B checks)
  h->simt_recon = h->simt_gemm || getenv("FD_SIMT_RECON") != nullptr;
  h->prm.dbg = nullptr;
  if (getenv("FD_DEBUG_EIG")) {
    void* dbgp = nullptr;
    if (cudaMalloc(&dbgp, 32 * sizeof(long long)) == cudaSuccess) {
      cudaMemset(dbgp, 0, 32 * sizeof(long long));
      h->prm.dbg = static_cast<long long*>(dbgp);
    }
  }
  h->buf[0] = reinterpret_cast<float*>(h->ws + Lo.buf0);
  h->buf[1] = reinterpret_cast<float*>(h->ws + Lo.buf1);
  h->nodes = reinterpret_cast<float*>(h->ws + Lo.nodes);
  h->G = h->ws + Lo.G;
  h->Wt = h->ws + Lo.Wt;

  h->stats = reinterpret_cast<Stats*>(h->ws + Lo.stats);
  h->flag = reinterpret_cast<int*>(h->ws + Lo.flag);
  h->prm.nonfinite = h->flag;
  h->eig = reinterpret_cast<double*>(h->ws + Lo.eig);
  h->state = D.prk ? reinterpret_cast<double*>(h->ws + Lo.state) : nullptr;
  h->arena = h->ws + Lo.arena;
  h->half = 0;
  h->half_used = 0;
  h->occ.assign(D.P, 0);
  h->cur.assign(D.P, 0);
  h->rows_seen = 0;
  h->dead = false;
  h->prof = false;
  DevGuard guard(h->device);
  int pitch = 0;
  cudaError_t e = cudaDeviceGetAttribute(&pitch, cudaDevAttrMaxPitch, h->device);
  h->max_pitch = pitch > 0 ? (size_t)pitch : ((size_t)1 << 31);
  if (e == cudaSuccess) e = cudaMallocHost(&h->host_arena, 2 * kArenaHalf);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev[0], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev[1], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&h->ev_copied[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_consumed[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_consumed[k], h->stream);
  }
  if (e == cudaSuccess) {
    e = cudaEventCreateWithFlags(&h->ev_copied_desc, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_copied_desc, h->copy_stream);
  }
  if (e == cudaSuccess) e = cudaEventRecord(h->ev[0], h->stream);
  if (e == cudaSuccess) e = cudaEventRecord(h->ev[1], h->stream);
  // zero the shard buffers' statistics and the flag
  if (e == cudaSuccess) e = cudaMemsetAsync(h->stats, 0, sizeof(Stats) * (D.P + Lo.nnodes), h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->flag, 0, sizeof(int) * 4, h->stream);
  if (e != cudaSuccess) {
    fd_status st = cuda_fail(e, "fd_create");
    delete h;
    return st;
  }
  *out = h;
  return FD_OK;
}

// Rows a per-row chain keeps in its state after n more rows (slot semantics, C6):
// Alg. 1 reduces when the buffer fills (occupancy ell -> ell-1); Compensative FD
// reduces lazily, when the next row arrives at a full buffer (reading C27).
static int perrow_occ_after(const Derived& D, int occ, int64_t n) {
  if (n <= 0) return occ;
  if (D.cfd) return (int)std::min<int64_t>((int64_t)occ + n, D.L);
  return (int)std::min<int64_t>((int64_t)occ + n, D.L - 1);
}

// Rows per shard per staging round of a host-input per-row append.
static int64_t perrow_stage_rows(const Derived& D) { return std::max<int64_t>(D.L, 16384 / D.P); }

// Per-row variants on the persistent per-row kernel: one launch per call (device
// rows) or per staged chunk (host rows, double-buffered copies on the copy stream).
static fd_status append_perrow(fd_handle* h, const float* rows, int64_t n_rows, int64_t ld, bool host, float* stage,
                               size_t stage_bytes) {
  const int P = h->D.P;
  const int64_t q = n_rows / P, r = n_rows % P;
  std::vector<int64_t> start(P), rem(P);
  int64_t off = 0;
  for (int s = 0; s < P; ++s) {
    start[s] = off;
    rem[s] = q + (s < r ? 1 : 0);
    off += rem[s];
  }
  const int64_t CH = host ? perrow_stage_rows(h->D) : std::numeric_limits<int64_t>::max();
  const size_t slot_floats = (size_t)P * (size_t)std::min<int64_t>(CH, std::max<int64_t>(q + 1, 1)) * ld;
  if (host && (!stage || stage_bytes < 2 * (size_t)P * CH * ld * sizeof(float)))
    return fail(FD_ERR_WORKSPACE, "host staging buffer smaller than fd_host_stage_bytes()");
  (void)slot_floats;
  std::vector<fdk::RowJob> jobs;
  for (int round = 0;; ++round) {
    jobs.clear();
    const int slot = round & 1;
    float* base = host ? stage + (size_t)slot * P * CH * ld : nullptr;
    if (host) FD_CUDA(cudaStreamWaitEvent(h->copy_stream, h->ev_consumed[slot], 0));
    for (int s = 0; s < P; ++s) {
      if (rem[s] == 0) continue;
      const int64_t c = std::min(CH, rem[s]);
      fdk::RowJob J{};
      if (host) {
        float* dstp = base + (size_t)s * CH * ld;
        FD_CUDA(cudaMemcpyAsync(dstp, rows + start[s] * ld, (size_t)c * ld * sizeof(float), cudaMemcpyHostToDevice,
                                h->copy_stream));
        J.src = dstp;
      } else {
        J.src = rows + start[s] * ld;
      }
      J.ld = ld;
      J.nrows = c;
      J.state = h->state + (size_t)s * h->D.ell * h->D.ldb;
      J.dst = shard_buf(h, s, h->cur[s]);
      J.stats = h->stats + s;
      J.k_in = h->occ[s];
      jobs.push_back(J);
      h->occ[s] = perrow_occ_after(h->D, h->occ[s], c);
      start[s] += c;
      rem[s] -= c;
    }
    if (jobs.empty()) break;
    if (host) {
      FD_CUDA(cudaEventRecord(h->ev_copied[slot], h->copy_stream));
      FD_CUDA(cudaStreamWaitEvent(h->stream, h->ev_copied[slot], 0));
    }
    const fdk::RowJob* dj = nullptr;
    fd_status st = push_desc(h, jobs, &dj);
    if (st != FD_OK) return st;
    const int nj = (int)jobs.size();
    cudaError_t e = timed(h, K_PERROW, [&] { return fdk::launch_perrow(dj, nj, h->prm, h->D.cfd ? 1 : 0, h->flag, h->stream); });
    if (e != cudaSuccess) return cuda_fail(e, "perrow");
    if (host) FD_CUDA(cudaEventRecord(h->ev_consumed[slot], h->stream));
  }
  h->rows_seen += n_rows;
  return FD_OK;
}

// Round loop shared by the device- and host-input appends.  Every call's rows are
// split into P contiguous ranges (reading C10); each round ingests the next
// min(L - occ, remaining) rows of every shard, then runs one batched ReduceRank
// over the shards whose buffer filled.  For host input the rows of round k are
// staged to the device (one 2-D copy per run of equally sized, equally spaced
// shard chunks) on the copy stream while round k-1 computes.
static fd_status append_impl(fd_handle* h, const float* rows, int64_t n_rows, int64_t ld, bool host, float* stage,
                             size_t stage_bytes) {
  if (!h) return fail(FD_ERR_INVALID_ARG, "handle is NULL");
  if (h->dead) return fail(FD_ERR_STATE, "handle refuses work after a sticky error");
  if (n_rows < 0) return fail(FD_ERR_INVALID_ARG, "n_rows < 0");
  if (n_rows == 0) return FD_OK;
  if (!rows) return fail(FD_ERR_INVALID_ARG, "rows is NULL");
  if (ld < h->D.d) return fail(FD_ERR_SHAPE, "ld < d");
  DevGuard guard(h->device);
  if (h->D.prk) return append_perrow(h, rows, n_rows, ld, host, stage, stage_bytes);
  const int P = h->D.P, L = h->D.L, ell = h->D.ell;
  const size_t slot_floats = (size_t)P * L * ld;
  if (host && (!stage || stage_bytes < 2 * slot_floats * sizeof(float)))
    return fail(FD_ERR_WORKSPACE, "host staging buffer smaller than fd_host_stage_bytes()");
  const int64_t q = n_rows / P, r = n_rows % P;
  std::vector<int64_t> start(P), rem(P);
  int64_t off = 0;
  for (int s = 0; s < P; ++s) {
    start[s] = off;
    rem[s] = q + (s < r ? 1 : 0);
    off += rem[s];
  }
  // plan of one round: (shard, first row, count)
  struct Chunk { int s; int64_t row; int c; };
  auto plan_round = [&](std::vector<int>& occ, std::vector<int64_t>& st, std::vector<int64_t>& rm,
                        std::vector<Chunk>& out) {
    out.clear();
    for (int s = 0; s < P; ++s) {
      if (rm[s] == 0) continue;
      const int c = (int)std::min<int64_t>(L - occ[s], rm[s]);
      out.push_back({s, st[s], c});
      st[s] += c;
      rm[s] -= c;
      occ[s] += c;
      if (occ[s] == L && (!h->D.cfd || rm[s] > 0)) occ[s] = h->D.R;
    }
  };
  // host staging: copy the chunks of a round into stage slot k (chunk i at i * maxc * ld)
  auto stage_round = [&](const std::vector<Chunk>& ch, int slot) -> fd_status {
    int maxc = 0;
    for (const Chunk& c : ch) maxc = std::max(maxc, c.c);
    float* base = stage + (size_t)slot * slot_floats;
    FD_CUDA(cudaStreamWaitEvent(h->copy_stream, h->ev_consumed[slot], 0));
    size_t i = 0;
    while (i < ch.size()) {
      size_t j = i + 1;
      const int64_t delta = (j < ch.size()) ? ch[j].row - ch[i].row : 0;
      while (j < ch.size() && ch[j].c == ch[i].c && ch[j].row - ch[j - 1].row == delta) ++j;
      const size_t cnt = j - i;
      const size_t width = (size_t)ch[i].c * ld * sizeof(float);
      const size_t spitch = (cnt > 1) ? (size_t)delta * ld * sizeof(float) : width;
      const size_t dpitch = (size_t)maxc * ld * sizeof(float);
      if (cnt > 1 && (spitch > h->max_pitch || dpitch > h->max_pitch)) {
        // pitches beyond the device's 2-D copy limit: one 1-D copy per chunk
        for (size_t k = i; k < j; ++k)
          FD_CUDA(cudaMemcpyAsync(base + k * (size_t)maxc * ld, rows + ch[k].row * ld, width, cudaMemcpyHostToDevice,
                                  h->copy_stream));
      } else {
        FD_CUDA(cudaMemcpy2DAsync(base + i * (size_t)maxc * ld, dpitch, rows + ch[i].row * ld, spitch, width, cnt,
                                  cudaMemcpyHostToDevice, h->copy_stream));
      }
      i = j;
    }
    FD_CUDA(cudaEventRecord(h->ev_copied[slot], h->copy_stream));
    return FD_OK;
  };
  if (h->D.cfd) {   // Compensative FD, lazy ReduceRank: buffers the previous call left full
    std::vector<Prob> pre;
    for (int s = 0; s < P; ++s) {
      if (h->occ[s] == L && rem[s] > 0) {
        pre.push_back(make_prob(h, (int)pre.size(), shard_buf(h, s, h->cur[s]), L, nullptr, 0,
                                shard_buf(h, s, h->cur[s] ^ 1), h->stats + s));
        h->cur[s] ^= 1;
        h->occ[s] = h->D.R;
      }
    }
    fd_status e = run_reduce(h, pre);
    if (e != FD_OK) return e;
  }
  std::vector<int> pocc = h->occ;   // planning copies (host staging runs one round ahead)
  std::vector<int64_t> pst = start, prm = rem;
  std::vector<Chunk> cur_ch, next_ch;
  int round = 0;
  if (host) {
    plan_round(pocc, pst, prm, cur_ch);
    if (!cur_ch.empty()) { fd_status e0 = stage_round(cur_ch, 0); if (e0 != FD_OK) return e0; }
  }
  // Rows that complete a buffer are read in place by the round's Gram and reconstruct
  // (Prob.src1 = the rows themselves, ld1 = ld; the tcgen05 Gram accumulates their
  // ||a||^2 and non-finite flag): only rows that stay in a buffer past this call are
  // copied by ingest_kernel.  Needs 16-byte rows (ld % 4 == 0, aligned base, d == ldb)
  // and the tcgen05 Gram; Compensative FD keeps full buffers across calls (lazy
  // ReduceRank, reading C27) and always copies.
  const bool direct = !h->D.cfd && !h->simt_gram && !use_f64(h->D, L) &&
                      fdk::gram_tc_supported(L, h->prm) && (ld % 4) == 0 && h->D.d == h->D.ldb &&
                      (reinterpret_cast<uintptr_t>(host ? stage : rows) % 16) == 0 && !h->ingest_copy;
  std::vector<Ingest> ing;
  std::vector<Prob> probs;
  ing.reserve(P);
  probs.reserve(P);
  for (;;) {
    ing.clear();
    probs.clear();
    int maxc = 0;
    if (host) for (const Chunk& c : cur_ch) maxc = std::max(maxc, c.c);
    int ci = 0;
    for (int s = 0; s < P; ++s) {
      if (rem[s] == 0) continue;
      const int c = (int)std::min<int64_t>(L - h->occ[s], rem[s]);
      const float* src = host ? stage + (size_t)(round & 1) * slot_floats + (size_t)ci * maxc * ld : rows + start[s] * ld;
      ++ci;
      start[s] += c;
      rem[s] -= c;
      const int occ0 = h->occ[s];
      h->occ[s] += c;
      const bool full = h->occ[s] == L && (!h->D.cfd || rem[s] > 0);   // CFD: lazy (reading C27)
      if (full && direct) {   // [buffer rows 0..occ0) ; the c new rows in place
        const int slot = (int)probs.size();
        Prob pr = make_prob(h, slot, shard_buf(h, s, h->cur[s]), occ0, src, c, shard_buf(h, s, h->cur[s] ^ 1),
                            h->stats + s);
        pr.ld1 = ld;
        pr.acc1 = 1;
        probs.push_back(pr);
        h->cur[s] ^= 1;
        h->occ[s] = h->D.R;
        continue;
      }
      Ingest g;
      g.src = src;
      g.ld = ld;
      g.dst = shard_buf(h, s, h->cur[s]) + (size_t)occ0 * h->D.ldb;
      g.nrows = c;
      g.pad = 0;
      g.stats = h->stats + s;
      ing.push_back(g);
      if (full) {
        const int slot = (int)probs.size();
        probs.push_back(make_prob(h, slot, shard_buf(h, s, h->cur[s]), L, nullptr, 0, shard_buf(h, s, h->cur[s] ^ 1),
                                  h->stats + s));
        h->cur[s] ^= 1;
        h->occ[s] = h->D.R;
      }
    }
    if (ing.empty() && probs.empty()) break;
    // this round's descriptors go to the device before the next round's staging copy is
    // enqueued: host -> device copies share the copy engine in issue order, and a small
    // descriptor upload queued behind a ~1 GB staging copy would hold the round back
    // (host input: on the copy stream, behind this round's staging copy and ahead of the
    // next one; the compute stream waits for both)
    fd_status st = FD_OK;
    const Ingest* di = nullptr;
    const Prob* dp = nullptr;
    cudaStream_t ds = host ? h->copy_stream : h->stream;
    if (!ing.empty() && (st = push_desc(h, ing, &di, ds)) != FD_OK) return st;
    if (!probs.empty() && (st = push_desc(h, probs, &dp, ds)) != FD_OK) return st;
    if (host) {
      FD_CUDA(cudaEventRecord(h->ev_copied_desc, h->copy_stream));   // staging of this round + descriptors
      FD_CUDA(cudaStreamWaitEvent(h->stream, h->ev_copied_desc, 0));
      // stage the next round while this one computes
      plan_round(pocc, pst, prm, next_ch);
      if (!next_ch.empty()) { fd_status e1 = stage_round(next_ch, (round + 1) & 1); if (e1 != FD_OK) return e1; }
    }
    if (!ing.empty()) {
      const int ni = (int)ing.size();
      cudaError_t e = timed(h, K_INGEST, [&] { return fdk::launch_ingest(di, ni, h->prm, h->flag, h->stream); });
      if (e != cudaSuccess) return cuda_fail(e, "ingest");
    }
    st = run_reduce(h, probs, false, false, dp);
    if (st != FD_OK) return st;
    // the staged rows were read by the ingest and (in place) by the round's Gram / reconstruct
    if (host) FD_CUDA(cudaEventRecord(h->ev_consumed[round & 1], h->stream));
    if (host) cur_ch.swap(next_ch);
    ++round;
  }
  h->rows_seen += n_rows;
  return FD_OK;
}

fd_status fd_append_rows(fd_handle* h, const float* rows, int64_t n_rows, int64_t ld) {
  return append_impl(h, rows, n_rows, ld, false, nullptr, 0);
}

size_t fd_host_stage_bytes(const fd_config* cfg, int64_t ld) {
  Derived D;
  std::string why;
  if (!derive(cfg, &D, &why) || ld < D.d) return 0;
  if (D.prk) return 2 * (size_t)D.P * perrow_stage_rows(D) * ld * sizeof(float);
  return 2 * (size_t)D.P * D.L * ld * sizeof(float);
}

fd_status fd_append_rows_host(fd_handle* h, const float* host_rows, int64_t n_rows, int64_t ld, void* stage,
                              size_t stage_bytes) {
  return append_impl(h, host_rows, n_rows, ld, true, static_cast<float*>(stage), stage_bytes);
}

fd_status fd_sketch(fd_handle* h, float* B_out, fd_stats* st) {
  if (!h || !B_out) return fail(FD_ERR_INVALID_ARG, "NULL argument");
  if (h->dead) return fail(FD_ERR_STATE, "handle refuses work after a sticky error");
  DevGuard guard(h->device);
  const bool cfd = h->D.cfd;
  fd_status s = finalize_shards(h, 0, h->D.P, cfd && h->D.P == 1);
  if (s != FD_OK) return s;
  int root = 0;
  s = run_tree(h, h->D.P, &root, cfd);
  if (s != FD_OK) return s;
  FD_CUDA(cudaMemcpy2DAsync(B_out, h->D.d * sizeof(float), node_buf(h, root), h->D.ldb * sizeof(float),
                            h->D.d * sizeof(float), h->D.ell, cudaMemcpyDeviceToDevice, h->stream));
  if (st) return read_stats(h, node_stats(h, root), st);
  return FD_OK;
}

fd_status fd_merge(fd_handle* h, const float* sketches, int32_t count, float* B_out, fd_stats* st) {
  if (!h || !sketches || !B_out) return fail(FD_ERR_INVALID_ARG, "NULL argument");
  if (h->dead) return fail(FD_ERR_STATE, "handle refuses work after a sticky error");
  if (count < 1 || count > kMergeMax) return fail(FD_ERR_INVALID_ARG, "count must be in [1, 64]");
  if (h->D.cfd)
    return fail(FD_ERR_UNSUPPORTED, "Compensative FD sketches are final (compensated); merge the handle's shards via fd_sketch");
  DevGuard guard(h->device);
  const int ell = h->D.ell;
  FD_CUDA(cudaMemcpy2DAsync(node_buf(h, 0), h->D.ldb * sizeof(float), sketches, h->D.d * sizeof(float),
                            h->D.d * sizeof(float), (size_t)count * ell, cudaMemcpyDeviceToDevice, h->stream));
  if (h->D.ldb != h->D.d) {
    // zero the padding columns of the copied rows
    FD_CUDA(cudaMemset2DAsync(node_buf(h, 0) + h->D.d, h->D.ldb * sizeof(float), 0,
                              (h->D.ldb - h->D.d) * sizeof(float), (size_t)count * ell, h->stream));
  }
  FD_CUDA(cudaMemsetAsync(node_stats(h, 0), 0, sizeof(Stats) * (2 * count - 1), h->stream));
  int root = 0;
  fd_status s = run_tree(h, count, &root);
  if (s != FD_OK) return s;
  FD_CUDA(cudaMemcpy2DAsync(B_out, h->D.d * sizeof(float), node_buf(h, root), h->D.ldb * sizeof(float),
                            h->D.d * sizeof(float), ell, cudaMemcpyDeviceToDevice, h->stream));
  if (st) {
    s = read_stats(h, node_stats(h, root), st);
    st->frob_sq = 0.0;
    st->rows_seen = 0;
    return s;
  }
  return FD_OK;
}

fd_status fd_shard_sketch(fd_handle* h, int32_t shard, float* B_out) {
  if (!h || !B_out) return fail(FD_ERR_INVALID_ARG, "NULL argument");
  if (shard < 0 || shard >= h->D.P) return fail(FD_ERR_INVALID_ARG, "shard out of range");
  if (h->dead) return fail(FD_ERR_STATE, "handle refuses work after a sticky error");
  DevGuard guard(h->device);
  fd_status s = finalize_shards(h, shard, shard + 1);
  if (s != FD_OK) return s;
  FD_CUDA(cudaMemcpy2DAsync(B_out, h->D.d * sizeof(float), node_buf(h, shard), h->D.ldb * sizeof(float),
                            h->D.d * sizeof(float), h->D.ell, cudaMemcpyDeviceToDevice, h->stream));
  return check_flag(h);
}

fd_status fd_reset(fd_handle* h) {
  if (!h) return fail(FD_ERR_INVALID_ARG, "handle is NULL");
  DevGuard guard(h->device);
  std::fill(h->occ.begin(), h->occ.end(), 0);
  std::fill(h->cur.begin(), h->cur.end(), 0);
  h->rows_seen = 0;
  h->dead = false;
  FD_CUDA(cudaMemsetAsync(h->stats, 0, sizeof(Stats) * (h->D.P + h->Lo.nnodes), h->stream));
  FD_CUDA(cudaMemsetAsync(h->flag, 0, sizeof(int) * 4, h->stream));
  return FD_OK;
}

fd_status fd_profile(fd_handle* h, int32_t enable) {
  if (!h) return fail(FD_ERR_INVALID_ARG, "handle is NULL");
  h->prof = enable != 0;
  return FD_OK;
}

int32_t fd_profile_read(fd_handle* h, double* ms, int64_t* launches, int32_t max_kernels) {
  if (!h) return 0;
  cudaStreamSynchronize(h->stream);
  double acc[K_COUNT] = {};
  int64_t cnt[K_COUNT] = {};
  for (auto& r : h->recs) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) acc[r.kind] += t;
    cnt[r.kind] += 1;
    h->pool.push_back(r.a);
    h->pool.push_back(r.b);
  }
  h->recs.clear();
  for (int k = 0; k < K_COUNT && k < max_kernels; ++k) {
    if (ms) ms[k] = acc[k];
    if (launches) launches[k] = cnt[k];
  }
  return K_COUNT;
}

fd_status fd_destroy(fd_handle* h) {
  if (!h) return FD_OK;
  DevGuard guard(h->device);
  cudaStreamSynchronize(h->stream);
  for (auto& r : h->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : h->pool) cudaEventDestroy(e);
  cudaEventDestroy(h->ev[0]);
  cudaEventDestroy(h->ev[1]);
  for (int k = 0; k < 2; ++k) { cudaEventDestroy(h->ev_copied[k]); cudaEventDestroy(h->ev_consumed[k]); }
  cudaEventDestroy(h->ev_copied_desc);
  cudaStreamDestroy(h->copy_stream);
  cudaFreeHost(h->host_arena);
  delete h;
  return FD_OK;
}

// ---------------------------------------------------------------------------
// Evaluator
// ---------------------------------------------------------------------------
static int lanczos_k(int64_t d) { return (int)std::min<int64_t>(d, 512); }

// bytes of fd_cov_gram_partial's scratch at any n (one row chunk at most)
static size_t syrk_part_max(int64_t d) { return fdk::syrk_tc_workspace_bytes(INT64_MAX / 4, d); }

// evaluator workspace: [M][Q][work][out] (fd_cov_err_from_gram), then fd_cov_err's AtA,
// then the SYRK row-chunk partials
static size_t cov_base_bytes(int64_t d) {
  const int k = lanczos_k(d);
  size_t off = 0;
  off = align_up(off + (size_t)d * d * sizeof(double), kAlign);                 // M
  off = align_up(off + (size_t)(k + 1) * d * sizeof(double), kAlign);           // Q
  off = align_up(off + (size_t)fdk::lanczos_work_doubles(d, k) * sizeof(double), kAlign);  // work
  off = align_up(off + 4 * sizeof(double), kAlign);                             // out
  return off;
}

size_t fd_cov_workspace_bytes(int64_t d) {
  if (d < 1) return 0;
  return cov_base_bytes(d) + align_up((size_t)d * d * sizeof(double), kAlign) + align_up(syrk_part_max(d), kAlign);
}

size_t fd_cov_gram_workspace_bytes(int64_t n, int64_t d) {
  if (d < 1 || n < 0) return 0;
  return fdk::syrk_tc_workspace_bytes(n, d);
}

fd_status fd_cov_gram_partial(const float* A, int64_t n, int64_t ld, int64_t d, double* AtA, void* ws,
                              size_t ws_bytes, void* cuda_stream) {
  if (!AtA || (n > 0 && !A) || d < 1 || n < 0) return fail(FD_ERR_INVALID_ARG, "bad argument");
  if (ld < d) return fail(FD_ERR_SHAPE, "ld < d");
  if (n == 0) return FD_OK;
  if (!ws || ws_bytes < fdk::syrk_tc_workspace_bytes(n, d)) return fail(FD_ERR_WORKSPACE, "gram workspace too small");
  cudaError_t e = fdk::launch_syrk_tc(A, n, ld, d, AtA, ws, ws_bytes, static_cast<cudaStream_t>(cuda_stream));
  if (e != cudaSuccess) return cuda_fail(e, "syrk");
  return FD_OK;
}

fd_status fd_cov_err_from_gram(const double* AtA, const float* B, int32_t ell, int64_t d, double frob_sq,
                               double* err, double* lam_max, double* lam_min, void* ws, size_t ws_bytes,
                               void* cuda_stream) {
  if (!AtA || !B || !err || ell < 1 || d < 1) return fail(FD_ERR_INVALID_ARG, "bad argument");
  if (!(frob_sq > 0.0)) return fail(FD_ERR_ZERO_NORM, "||A||_F^2 = 0: cov-err undefined");
  if (!ws || ws_bytes < fd_cov_workspace_bytes(d)) return fail(FD_ERR_WORKSPACE, "evaluator workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  const int k = lanczos_k(d);
  char* w = static_cast<char*>(ws);
  size_t off = 0;
  double* M = reinterpret_cast<double*>(w + off); off = align_up(off + (size_t)d * d * sizeof(double), kAlign);
  double* Q = reinterpret_cast<double*>(w + off); off = align_up(off + (size_t)(k + 1) * d * sizeof(double), kAlign);
  double* work = reinterpret_cast<double*>(w + off); off = align_up(off + (size_t)fdk::lanczos_work_doubles(d, k) * sizeof(double), kAlign);
  double* out = reinterpret_cast<double*>(w + off);
  cudaError_t e = fdk::launch_sub_btb(M, AtA, B, ell, d, s);
  if (e != cudaSuccess) return cuda_fail(e, "sub_btb");
  e = fdk::launch_lanczos(M, d, k, Q, work, out, s);
  if (e != cudaSuccess) return cuda_fail(e, "lanczos");
  double ex[2];
  e = cudaMemcpyAsync(ex, out, sizeof(ex), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "lanczos result");
  const double nrm = std::max(std::fabs(ex[0]), std::fabs(ex[1]));
  *err = nrm / frob_sq;
  if (lam_max) *lam_max = ex[0] / frob_sq;
  if (lam_min) *lam_min = ex[1] / frob_sq;
  return FD_OK;
}

fd_status fd_cov_frob_from_gram(const double* AtA, int64_t d, double* frob_sq, void* cuda_stream) {
  if (!AtA || !frob_sq || d < 1) return fail(FD_ERR_INVALID_ARG, "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  std::vector<double> diag(d);
  cudaError_t e = cudaMemcpy2DAsync(diag.data(), sizeof(double), AtA, (d + 1) * sizeof(double), sizeof(double), d,
                                    cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "trace");
  double frob = 0.0;
  for (double x : diag) frob += x;
  *frob_sq = frob;
  return FD_OK;
}

fd_status fd_cov_err(const float* A, int64_t n, int64_t ld, const float* B, int32_t ell, int64_t d, double* err,
                     double* lam_max, double* lam_min, void* ws, size_t ws_bytes, void* cuda_stream) {
  if (!ws || ws_bytes < fd_cov_workspace_bytes(d)) return fail(FD_ERR_WORKSPACE, "evaluator workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  const size_t base = cov_base_bytes(d), atab = align_up((size_t)d * d * sizeof(double), kAlign);
  double* AtA = reinterpret_cast<double*>(static_cast<char*>(ws) + base);
  cudaError_t e = cudaMemsetAsync(AtA, 0, (size_t)d * d * sizeof(double), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  fd_status st = fd_cov_gram_partial(A, n, ld, d, AtA, static_cast<char*>(ws) + base + atab, ws_bytes - base - atab,
                                     cuda_stream);
  if (st != FD_OK) return st;
  double frob = 0.0;
  st = fd_cov_frob_from_gram(AtA, d, &frob, cuda_stream);
  if (st != FD_OK) return st;
  return fd_cov_err_from_gram(AtA, B, ell, d, frob, err, lam_max, lam_min, ws, ws_bytes, cuda_stream);
}

// ---- proj-err (fd_eval.cu) ----
namespace {
struct ProjLayout {
  size_t G, V, w, ord, sweeps, vbuf, q, Q, work, out, top, total;
};
ProjLayout proj_layout(int64_t d, int32_t ell, int32_t k) {
  ProjLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, kAlign); return o; };
  const int kl = lanczos_k(d);
  L.G = take((size_t)ell * ell * sizeof(double));
  L.V = take((size_t)ell * ell * sizeof(double));
  L.w = take((size_t)ell * sizeof(double));
  L.ord = take((size_t)ell * sizeof(int));
  L.sweeps = take(sizeof(int));
  L.vbuf = take((size_t)k * d * sizeof(double));
  L.q = take((size_t)k * sizeof(double));
  L.Q = take((size_t)(kl + 1) * d * sizeof(double));
  L.work = take((size_t)fdk::lanczos_work_doubles(d, kl) * sizeof(double));
  L.out = take(2 * sizeof(double));
  L.top = take((size_t)k * sizeof(double));
  L.total = off;
  return L;
}
}  // namespace

size_t fd_proj_workspace_bytes(int64_t d, int32_t ell, int32_t k) {
  if (d < 1 || ell < 1 || k < 1) return 0;
  return proj_layout(d, ell, k).total;
}

fd_status fd_proj_err_from_gram(const double* AtA, const float* B, int32_t ell, int64_t d, double frob_sq, int32_t k,
                                double* proj_err, double* num, double* den, void* ws, size_t ws_bytes,
                                void* cuda_stream) {
  if (!AtA || !B || !proj_err || ell < 1 || d < 1 || k < 1 || k > d) return fail(FD_ERR_INVALID_ARG, "bad argument");
  if (!(frob_sq > 0.0)) return fail(FD_ERR_ZERO_NORM, "||A||_F^2 = 0: proj-err undefined");
  const ProjLayout L = proj_layout(d, ell, k);
  if (!ws || ws_bytes < L.total) return fail(FD_ERR_WORKSPACE, "proj-err workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  char* w = static_cast<char*>(ws);
  auto D = [&](size_t o) { return reinterpret_cast<double*>(w + o); };
  cudaError_t e = fdk::launch_proj_parts(B, ell, d, k, AtA, D(L.G), D(L.V), D(L.w), reinterpret_cast<int*>(w + L.ord),
                                         reinterpret_cast<int*>(w + L.sweeps), D(L.vbuf), D(L.q), s);
  if (e != cudaSuccess) return cuda_fail(e, "proj-err parts");
  e = fdk::launch_lanczos(AtA, d, lanczos_k(d), D(L.Q), D(L.work), D(L.out), s, k, D(L.top));
  if (e != cudaSuccess) return cuda_fail(e, "lanczos top-k");
  std::vector<double> q(k), top(k);
  e = cudaMemcpyAsync(q.data(), D(L.q), k * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(top.data(), D(L.top), k * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "proj-err result");
  double cap = 0.0, best = 0.0;
  for (int t = 0; t < k; ++t) { cap += q[t]; best += top[t]; }
  const double nu = frob_sq - cap, de = frob_sq - best;
  if (num) *num = nu;
  if (den) *den = de;
  // numerically rank A <= k: the tensor-core A^T A carries ~2^-30 relative error per row
  // (reading E3), so a tail below 1e-8 ||A||_F^2 is indistinguishable from zero
  if (!(de > 1e-8 * frob_sq)) return fail(FD_ERR_ZERO_NORM, "||A - A_k||_F^2 ~ 0 (rank A <= k): proj-err undefined");
  *proj_err = nu / de;
  return FD_OK;
}

fd_status fd_proj_err(const float* A, int64_t n, int64_t ld, const float* B, int32_t ell, int64_t d, int32_t k,
                      double* proj_err, void* ws, size_t ws_bytes, void* cuda_stream) {
  if (!A || !B || !proj_err || d < 1 || ell < 1 || k < 1) return fail(FD_ERR_INVALID_ARG, "bad argument");
  const size_t pb = fd_proj_workspace_bytes(d, ell, k);
  const size_t ab = align_up((size_t)d * d * sizeof(double), kAlign);
  const size_t gb = fd_cov_gram_workspace_bytes(n, d);
  if (!ws || ws_bytes < pb + ab + gb) return fail(FD_ERR_WORKSPACE, "proj-err workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  double* AtA = reinterpret_cast<double*>(static_cast<char*>(ws) + pb);
  cudaError_t e = cudaMemsetAsync(AtA, 0, (size_t)d * d * sizeof(double), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  fd_status st = fd_cov_gram_partial(A, n, ld, d, AtA, static_cast<char*>(ws) + pb + ab, gb, cuda_stream);
  if (st != FD_OK) return st;
  double frob = 0.0;
  st = fd_cov_frob_from_gram(AtA, d, &frob, cuda_stream);
  if (st != FD_OK) return st;
  return fd_proj_err_from_gram(AtA, B, ell, d, frob, k, proj_err, nullptr, nullptr, ws, pb, cuda_stream);
}

size_t fd_hash_workspace_bytes(int64_t d, int32_t ell) {
  if (d < 1 || ell < 1) return 0;
  return (size_t)fdk::hash_ranges(d) * (size_t)ell * (size_t)d * sizeof(double);
}

fd_status fd_hash_sketch(const float* A, int64_t n, int64_t ld, int64_t d, int32_t ell, int32_t s, uint64_t seed,
                         int64_t row0, double* B_acc, void* ws, size_t ws_bytes, void* cuda_stream) {
  if (!B_acc || (n > 0 && !A) || n < 0 || d < 1 || ell < 1 || row0 < 0) return fail(FD_ERR_INVALID_ARG, "bad argument");
  if (ld < d) return fail(FD_ERR_SHAPE, "ld < d");
  if (!fdk::hash_supported(ell, s)) return fail(FD_ERR_UNSUPPORTED, "hash sketch: need 1 <= s <= 8, s | ell, ell <= 400");
  if (n == 0) return FD_OK;
  if (!ws || ws_bytes < fd_hash_workspace_bytes(d, ell)) return fail(FD_ERR_WORKSPACE, "hash workspace too small");
  cudaError_t e = fdk::launch_hash(A, n, ld, d, ell, s, seed, row0, static_cast<double*>(ws), B_acc,
                                   static_cast<cudaStream_t>(cuda_stream));
  if (e != cudaSuccess) return cuda_fail(e, "hash sketch");
  return FD_OK;
}

const char* fd_last_error(void) { return g_err.c_str(); }

// debug: copy the phase trace (32 x int64, CTA 0 of the eig / trd kernels; FD_DEBUG_EIG set)
int32_t fd_debug_eig_trace(fd_handle* h, long long* out16) {
  if (!h || !h->prm.dbg) return -1;
  cudaStreamSynchronize(h->stream);
  cudaMemcpy(out16, h->prm.dbg, 32 * sizeof(long long), cudaMemcpyDeviceToHost);
  return 0;
}

const char* fd_version(void) { return "fd-b200 0.1 (sm_100a)"; }

}  // extern "C"
