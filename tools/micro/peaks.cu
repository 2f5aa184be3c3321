// Peak microbenchmarks for the roofline denominators: FP32 FFMA,
// FP64 DFMA and tcgen05 kind::tf32 dense MMA throughput on all 148 SMs, timed with
// CUDA events.  Output: one JSON object (TFLOP/s, measured at the clock the run saw).
#include <cstdio>
#include <cuda_runtime.h>
#include "fd_tc.cuh"
using namespace fdk;

template <typename T>
__global__ void __launch_bounds__(1024) fma_kernel(T* out, int iters) {
  T a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = (T)(threadIdx.x + j);
  const T b = (T)0.999999, c = (T)1e-7;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  T s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == (T)-1) out[0] = s;
}

// packed fp32 FMA (FFMA2, fma.rn.f32x2): 8 independent float2 chains per thread
__global__ void __launch_bounds__(1024) fma2_kernel(float* out, int iters) {
  unsigned long long a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 v = make_float2((float)(threadIdx.x + j), (float)(threadIdx.x - j));
    a[j] = *reinterpret_cast<const unsigned long long*>(&v);
  }
  const float2 bf = make_float2(0.999999f, 0.999998f), cf = make_float2(1e-7f, 2e-7f);
  const unsigned long long b = *reinterpret_cast<const unsigned long long*>(&bf);
  const unsigned long long c = *reinterpret_cast<const unsigned long long*>(&cf);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(b), "l"(c));
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 v = *reinterpret_cast<const float2*>(&a[j]);
    s += v.x + v.y;
  }
  if (s == -1.f) out[0] = s;
}

// one CTA per SM; one thread issues M=128 x N=256 x K=8 tf32 MMAs back to back from
// resident SW128 smem tiles into TMEM, committing every 32 MMAs to an mbarrier
__global__ void __launch_bounds__(128, 1) tf32_kernel(int iters, int* sink) {
  extern __shared__ unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 + 256) * 32; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.5f;
  if (warp == 0) tc::tmem_alloc(&s_tmem, 512);
  if (tid == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tb = s_tmem;
  if (tid == 0) {
    const uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 128 * 128);
    const uint32_t id = tc::idesc_tf32(128, 256, 0, 0);
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const uint32_t ko = (q & 3) * 32;
        tc::mma_tf32(tb + (q & 1) * 256, tc::desc_k_sw128(a + ko), tc::desc_k_sw128(b + ko), id, 1u);
      }
      tc::commit(&mbar);
      tc::mbar_wait(&mbar, ph);
      ph ^= 1;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tb, 512);
  if (tid == 0 && iters < 0) sink[0] = 1;
}

// same for kind::i8 (s8 x s8 -> s32), M = 128, N = NN, K = 32 bytes per MMA
template <int NN>
__global__ void __launch_bounds__(128, 1) i8_kernel(int iters, int* sink) {
  extern __shared__ unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 + 256) * 32; i += blockDim.x) reinterpret_cast<int*>(sm)[i] = 0x01010101;
  if (warp == 0) tc::tmem_alloc(&s_tmem, 512);
  if (tid == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tb = s_tmem;
  if (tid == 0) {
    const uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 128 * 128);
    const uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const uint32_t ko = (q & 3) * 32;
        const uint64_t ad = tc::desc_k_sw128(a + ko), bd = tc::desc_k_sw128(b + ko);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
            :
            : "r"(tb + (q & 1) * 256), "l"(ad), "l"(bd), "r"(id), "r"(1u));
      }
      tc::commit(&mbar);
      tc::mbar_wait(&mbar, ph);
      ph ^= 1;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tb, 512);
  if (tid == 0 && iters < 0) sink[0] = 1;
}

template <int NN>
double time_i8(int sms, int smem, void* out, cudaEvent_t e0, cudaEvent_t e1) {
  cudaFuncSetAttribute(i8_kernel<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  i8_kernel<NN><<<sms, 128, smem>>>(16, (int*)out);
  const int ti = 4096;
  float ms;
  cudaEventRecord(e0);
  i8_kernel<NN><<<sms, 128, smem>>>(ti, (int*)out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  return 2.0 * 128 * NN * 32 * 32.0 * ti * sms / (ms * 1e-3) / 1e12;
}

int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  void* out;
  cudaMalloc(&out, 64);
  const int sms = 148;
  // FFMA: 8 resident 1024-thread... use 2 x 1024 threads per SM
  const int it = 1 << 16;
  fma_kernel<float><<<sms * 2, 1024>>>((float*)out, 16);
  cudaEventRecord(e0);
  fma_kernel<float><<<sms * 2, 1024>>>((float*)out, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double ffma = 2.0 * 8 * it * (double)sms * 2 * 1024 / (ms * 1e-3) / 1e12;
  fma2_kernel<<<sms * 2, 1024>>>((float*)out, 16);
  cudaEventRecord(e0);
  fma2_kernel<<<sms * 2, 1024>>>((float*)out, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double ffma2 = 4.0 * 8 * it * (double)sms * 2 * 1024 / (ms * 1e-3) / 1e12;
  fma_kernel<double><<<sms * 2, 1024>>>((double*)out, 16);
  cudaEventRecord(e0);
  fma_kernel<double><<<sms * 2, 1024>>>((double*)out, it / 8);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma = 2.0 * 8 * (it / 8) * (double)sms * 2 * 1024 / (ms * 1e-3) / 1e12;
  const int smem = (128 + 256) * 128 + 1024;
  cudaFuncSetAttribute(tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tf32_kernel<<<sms, 128, smem>>>(16, (int*)out);
  const int ti = 4096;
  cudaEventRecord(e0);
  tf32_kernel<<<sms, 128, smem>>>(ti, (int*)out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double tf32 = 2.0 * 128 * 256 * 8 * 32.0 * ti * sms / (ms * 1e-3) / 1e12;
  const double i8_256 = time_i8<256>(sms, smem, out, e0, e1);
  const double i8_64 = time_i8<64>(sms, smem, out, e0, e1);
  cudaError_t err = cudaGetLastError();
  printf("{\"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"dfma_tflops\": %.2f, \"tf32_tcgen05_tflops\": %.2f, \"tf32x3_tflops\": %.2f, "
         "\"i8_tcgen05_tops\": %.1f, \"i8_tcgen05_n64_tops\": %.1f, "
         "\"error\": \"%s\", \"how\": \"tools/micro/peaks.cu: 296x1024 threads x 8 independent FMA chains (FFMA, FFMA2 = fma.rn.f32x2, DFMA); "
         "148 CTAs each issuing back-to-back tcgen05.mma.kind::tf32 M128 N256 K8 / kind::i8 M128 N256|N64 K32 from resident smem tiles, CUDA events\"}\n",
         ffma, ffma2, dfma, tf32, tf32 / 3.0, i8_256, i8_64, cudaGetErrorString(err));
  return 0;
}
