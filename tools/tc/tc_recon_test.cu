// Standalone check of recon_tc_kernel (tcgen05 3xTF32, MN-major B) against fp64 CPU.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "fd_internal.h"
namespace fdk { cudaError_t launch_recon_tc(const Prob*, int, int, const Params&, cudaStream_t); }
using namespace fdk;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)
int main(int argc, char** argv) {
  int N = atoi(argv[1]), d = atoi(argv[2]), ell = atoi(argv[3]), nprob = atoi(argv[4]);
  int64_t ldb = (d + 3) / 4 * 4; int ldg = (N + 3) / 4 * 4;
  std::vector<float> A((size_t)nprob * N * ldb, 0.f), W((size_t)nprob * ell * ldg, 0.f);
  srand(2);
  for (auto& x : A) x = (float)(rand() / (double)RAND_MAX - 0.5);
  for (int p = 0; p < nprob; ++p) for (int r = 0; r < N; ++r) for (int c = d; c < ldb; ++c) A[((size_t)p * N + r) * ldb + c] = 0.f;
  for (int p = 0; p < nprob; ++p) for (int j = 0; j < ell - 1; ++j) for (int k = 0; k < ldg; ++k)
    W[((size_t)p * ell + j) * ldg + k] = (k < N) ? (float)(rand() / (double)RAND_MAX - 0.5) : 777.f;
  float *dA, *dW, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dW, W.size() * 4)); CK(cudaMalloc(&dD, (size_t)nprob * ell * ldb * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0xFF, (size_t)nprob * ell * ldb * 4));
  std::vector<Prob> pr(nprob);
  for (int p = 0; p < nprob; ++p) {
    pr[p] = Prob{}; pr[p].src0 = dA + (size_t)p * N * ldb; pr[p].rows0 = N / 2; pr[p].src1 = dA + ((size_t)p * N + N / 2) * ldb; pr[p].rows1 = N - N / 2;
    pr[p].dst = dD + (size_t)p * ell * ldb; pr[p].Wt = dW + (size_t)p * ell * ldg;
  }
  Prob* dP; CK(cudaMalloc(&dP, nprob * sizeof(Prob))); CK(cudaMemcpy(dP, pr.data(), nprob * sizeof(Prob), cudaMemcpyHostToDevice));
  Params prm{}; prm.d = d; prm.ldb = ldb; prm.ldg = ldg; prm.ell = ell;
  CK(launch_recon_tc(dP, nprob, N, prm, 0)); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); for (int it = 0; it < 5; ++it) CK(launch_recon_tc(dP, nprob, N, prm, 0)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<float> D((size_t)nprob * ell * ldb); CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxv = 0; int bad = 0;
  for (int p = 0; p < nprob; ++p) for (int j = 0; j < ell; ++j) for (int c = 0; c < ldb; ++c) {
    double s = 0;
    if (j < ell - 1) for (int k = 0; k < N; ++k) s += (double)W[((size_t)p * ell + j) * ldg + k] * A[((size_t)p * N + k) * ldb + c];
    double g = D[((size_t)p * ell + j) * ldb + c];
    if (!(fabs(g - s) <= 1e-3 * (1 + fabs(s)))) { if (bad < 5) printf("  bad p=%d j=%d c=%d gpu=%g ref=%g\n", p, j, c, g, s); ++bad; }
    maxerr = fmax(maxerr, fabs(g - s)); maxv = fmax(maxv, fabs(s));
  }
  printf("N=%d d=%d ell=%d nprob=%d: max|D|=%.4g max abs err %.3e (rel %.3e) bad=%d  %.3f ms/launch\n", N, d, ell, nprob, maxv, maxerr, maxerr / maxv, bad, ms / 5);
  return bad ? 2 : 0;
}
