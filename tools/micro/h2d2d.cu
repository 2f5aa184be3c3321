// H2D bandwidth of the fd_append_rows_host staging pattern: one cudaMemcpy2DAsync of
// `chunks` chunks of 129 rows x 4 KB taken at a shard stride of 3543 rows (c4, P = 2368),
// against one contiguous copy of the same bytes (pinned host memory, CUDA events).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t chunks = 592, rows = 129, stride = 3543, ld = 1024;
  const size_t w = rows * ld * 4, sp = stride * ld * 4;
  char* h; char* d;
  if (cudaMallocHost(&h, chunks * sp) != cudaSuccess) { printf("pin failed\n"); return 1; }
  for (size_t i = 0; i < chunks * sp; i += 4096) h[i] = 1;
  cudaMalloc(&d, chunks * w);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) cudaMemcpyAsync(d, h, chunks * w, cudaMemcpyHostToDevice);
  cudaEventRecord(a);
  for (int rep = 0; rep < 5; ++rep) cudaMemcpyAsync(d, h, chunks * w, cudaMemcpyHostToDevice);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf("contiguous: %.1f GB/s\n", 5.0 * chunks * w / (ms * 1e-3) / 1e9);
  for (int rep = 0; rep < 2; ++rep) cudaMemcpy2DAsync(d, w, h, sp, w, chunks, cudaMemcpyHostToDevice);
  cudaEventRecord(a);
  for (int rep = 0; rep < 5; ++rep) cudaMemcpy2DAsync(d, w, h, sp, w, chunks, cudaMemcpyHostToDevice);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf("2-D (%zu x %zu KB, pitch %.1f MB): %.1f GB/s\n", chunks, w >> 10, sp / 1e6, 5.0 * chunks * w / (ms * 1e-3) / 1e9);
  // per-chunk 1-D copies
  cudaEventRecord(a);
  for (int rep = 0; rep < 5; ++rep)
    for (size_t c = 0; c < chunks; ++c) cudaMemcpyAsync(d + c * w, h + c * sp, w, cudaMemcpyHostToDevice);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf("1-D per chunk: %.1f GB/s\n", 5.0 * chunks * w / (ms * 1e-3) / 1e9);
  return 0;
}
