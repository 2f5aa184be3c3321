// How does tcgen05.mma kind::tf32 read an fp32 operand whose low 13 mantissa bits are
// set: truncation (ignore them), round-to-nearest, or full fp32?  A = [x_r, 0..] per
// row r, B = [1, 0, ..] so D[r][0] = conv(x_r) * 1.  If the hardware truncates, the
// Gram's 3xTF32 "hi" operand can be the raw fp32 value (TMA-staged, no SIMT pass) and
// lo = x - trunc(x).   nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_1501_06561_b200/csrc
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fd_tc.cuh"

using namespace fdk;

__global__ void k(const float* xs, float* out) {
  extern __shared__ unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  unsigned char* A = sm;            // 128 rows x 32 values
  unsigned char* B = sm + 16384;    // 128 rows x 32 values
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    const int r = e / 32, c = e % 32;
    *reinterpret_cast<float*>(A + tc::sw128_off(r, c)) = (c == 0) ? xs[r] : 0.f;
    *reinterpret_cast<float*>(B + tc::sw128_off(r, c)) = (c == 0 && r == 0) ? 1.f : 0.f;
  }
  if (warp == 0) tc::tmem_alloc(&s_tmem, 128);
  if (tid == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    const uint32_t id = tc::idesc_tf32(128, 128, 0, 0);
    tc::mma_tf32(s_tmem, tc::desc_k_sw128(tc::smem_u32(A)), tc::desc_k_sw128(tc::smem_u32(B)), id, 0u);
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  float v[16];
  tc::tmem_ld16(s_tmem + ((uint32_t)(32 * (warp & 3)) << 16), v);
  out[32 * (warp & 3) + (tid & 31)] = v[0];
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(s_tmem, 128);
}

static float bits(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t ubits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

int main() {
  float h[128];
  // 1 + mantissa patterns in the 13 dropped bits: tie, above half, below half, all set
  const uint32_t lows[8] = {0x0, 0x1000, 0x1001, 0x0FFF, 0x1FFF, 0x0001, 0x1800, 0x0800};
  for (int r = 0; r < 128; ++r) {
    const uint32_t keep = (uint32_t)(r % 16) << 13;   // varies the kept lsb (ties to even vs away)
    h[r] = bits(0x3F800000u | keep | lows[r % 8]);
    if (r >= 64) h[r] = -h[r];
  }
  float *dx, *dout;
  cudaMalloc(&dx, sizeof h); cudaMalloc(&dout, sizeof h);
  cudaMemcpy(dx, h, sizeof h, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  k<<<1, 128, 40000>>>(dx, dout);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  float o[128];
  cudaMemcpy(o, dout, sizeof o, cudaMemcpyDeviceToHost);
  int ntr = 0, nrn = 0, nfull = 0;
  for (int r = 0; r < 128; ++r) {
    const uint32_t u = ubits(h[r]);
    const float tr = bits(u & ~0x1FFFu);
    uint32_t rn = u & ~0x1FFFu;   // round to nearest even on 13 bits
    const uint32_t low = u & 0x1FFF;
    if (low > 0x1000 || (low == 0x1000 && ((u >> 13) & 1))) rn += 0x2000;
    const uint32_t ra = (u + 0x1000) & ~0x1FFFu;   // round half away
    ntr += (o[r] == tr);
    nrn += (o[r] == bits(rn));
    nfull += (o[r] == h[r]);
    if (r < 16) printf("x=%08x out=%08x trunc=%08x rne=%08x rna=%08x\n", u, ubits(o[r]), ubits(tr), rn, ra);
  }
  printf("tf32 operand conversion: trunc %d/128, rne %d/128, full fp32 %d/128\n", ntr, nrn, nfull);
  return 0;
}
