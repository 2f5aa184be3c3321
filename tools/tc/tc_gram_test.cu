// Standalone check of gram_tc_kernel (tcgen05 3xTF32) against an fp64 CPU Gram.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "fd_internal.h"
namespace fdk {
cudaError_t launch_gram_tc(const Prob* dev_probs, int count, int nmax, const Params& p, cudaStream_t s);
}
using namespace fdk;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)
int main(int argc, char** argv) {
  int N = argc > 1 ? atoi(argv[1]) : 256, d = argc > 2 ? atoi(argv[2]) : 1024, nprob = argc > 3 ? atoi(argv[3]) : 4;
  int split = argc > 4 ? atoi(argv[4]) : N / 2;  // rows0
  int64_t ldb = (d + 3) / 4 * 4; int ldg = (N + 3) / 4 * 4;
  std::vector<float> A((size_t)nprob * N * ldb, 0.f);
  srand(1);
  for (int p = 0; p < nprob; ++p) for (int r = 0; r < N; ++r) for (int c = 0; c < d; ++c)
    A[((size_t)p * N + r) * ldb + c] = (float)((rand() / (double)RAND_MAX - 0.5) * (1.0 + 3.0 * (c % 7 == 0)) * (r < 10 ? 30.0 : 1.0));
  float *dA, *dG; CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dG, (size_t)nprob * ldg * ldg * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice)); CK(cudaMemset(dG, 0, (size_t)nprob * ldg * ldg * 4));
  std::vector<Prob> pr(nprob);
  for (int p = 0; p < nprob; ++p) {
    pr[p].src0 = dA + (size_t)p * N * ldb; pr[p].rows0 = split;
    pr[p].src1 = dA + ((size_t)p * N + split) * ldb; pr[p].rows1 = N - split;
    pr[p].dst = nullptr; pr[p].G = dG + (size_t)p * ldg * ldg; pr[p].Wt = nullptr; pr[p].stats = nullptr; pr[p].child0 = pr[p].child1 = nullptr;
  }
  Prob* dP; CK(cudaMalloc(&dP, nprob * sizeof(Prob))); CK(cudaMemcpy(dP, pr.data(), nprob * sizeof(Prob), cudaMemcpyHostToDevice));
  Params prm{}; prm.d = d; prm.ldb = ldb; prm.ldg = ldg; prm.ell = N / 2;
  CK(launch_gram_tc(dP, nprob, N, prm, 0)); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); for (int it = 0; it < 5; ++it) CK(launch_gram_tc(dP, nprob, N, prm, 0)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<float> G((size_t)nprob * ldg * ldg); CK(cudaMemcpy(G.data(), dG, G.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxg = 0, maxerr32 = 0;
  for (int p = 0; p < nprob; ++p) for (int r = 0; r < N; ++r) for (int c = 0; c < N; ++c) {
    if (r < 128 && c >= 128) continue;
    double s = 0; float s32 = 0;
    const float* a = &A[((size_t)p * N + r) * ldb]; const float* b = &A[((size_t)p * N + c) * ldb];
    for (int k = 0; k < d; ++k) { s += (double)a[k] * b[k]; s32 += a[k] * b[k]; }
    double g = G[(size_t)p * ldg * ldg + (size_t)r * ldg + c];
    maxerr = fmax(maxerr, fabs(g - s)); maxg = fmax(maxg, fabs(s)); maxerr32 = fmax(maxerr32, fabs(s32 - s));
  }
  double flops = 2.0 * nprob * (N <= 128 ? 128.0 * 128 : 128.0 * 128 + 128.0 * 256) * ldb * 3;
  printf("N=%d d=%d nprob=%d: max|G|=%.4g  max abs err %.3e (rel %.3e)  [fp32 naive err %.3e]  %.3f ms/launch  %.1f TFLOP/s (3xTF32 incl.)\n",
         N, d, nprob, maxg, maxerr, maxerr / maxg, maxerr32, ms / 5, flops / (ms / 5 * 1e-3) / 1e12);
  return maxerr / maxg < 1e-5 ? 0 : 2;
}
