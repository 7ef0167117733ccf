// Microbenchmark: raw tcgen05.mma kind::tf32 throughput for the SVM kernel's
// operand layout (K-major, SWIZZLE_NONE core matrices), M=128 x N=256 x K=8,
// one CTA per SM issuing back-to-back MMAs on a resident smem stage.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2301_13441_b200/csrc/sm100.cuh"
using namespace cmlb::sm100;

template <int LAYOUT>  // 0: no swizzle core matrices (as svm.cu)
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f;
  if (threadIdx.x == 0) { bar_init(&done, 1); bar_fence_init(); }
  if (warp == 0) tmem_alloc(&slot, 256);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t base = smem_addr(smem);
    const uint32_t abig = base, asmall = base + 16384, bbig = base + 32768, bsmall = bbig + 32768;
    constexpr uint32_t idesc = idesc_tf32(128, 256);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k8 = 0; k8 < 4; ++k8) {
        const uint32_t ao = k8 * 2 * (128 * 16), bo = k8 * 2 * (256 * 16);
        const uint64_t ab = desc_kmajor(abig + ao, 128 * 16, 128), as = desc_kmajor(asmall + ao, 128 * 16, 128);
        const uint64_t bb = desc_kmajor(bbig + bo, 256 * 16, 128), bs = desc_kmajor(bsmall + bo, 256 * 16, 128);
        mma_tf32(tmem, ab, bb, idesc, (it | k8) != 0);
        mma_tf32(tmem, as, bb, idesc, 1u);
        mma_tf32(tmem, ab, bs, idesc, 1u);
      }
    }
    mma_commit(&done);
    bar_wait(&done, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_free(tmem, 256); }
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d; cudaMalloc(&d, sms * 8);
  const int smem = 96 * 1024;
  cudaFuncSetAttribute(mma_rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  mma_rate<0><<<sms, 128, smem>>>(100, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_rate<0><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c[256]; cudaMemcpy(c, d, sms * 8, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * 256 * 8 * 12.0 * iters * sms;
  printf("{\"layout\": \"kmajor_noswizzle\", \"ms\": %.3f, \"tflops\": %.1f, \"cycles_per_stage\": %.1f, \"err\": \"%s\"}\n",
         ms, flops / (ms / 1e3) / 1e12, (double)c[0] / iters, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
