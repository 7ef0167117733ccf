// Microbenchmark: tcgen05.mma kind::i8 (u8 x s8 -> s32) throughput for the
// forest MMA variant's operand layout (K-major, SWIZZLE_NONE core matrices),
// M=128 x N=256 x K=32 per instruction, 8 instructions per tree (K = 256).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2301_13441_b200/csrc/sm100.cuh"
using namespace cmlb::sm100;

__global__ void __launch_bounds__(128, 1) mma_rate_i8(int iters, int wait_each, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  if (threadIdx.x == 0) { bar_init(&done, 1); bar_fence_init(); }
  if (warp == 0) tmem_alloc(&slot, 256);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t base = smem_addr(smem);
    const uint32_t A = base, B = base + 32768;
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int s = 0; s < 8; ++s) {
        const uint64_t ad = desc_kmajor(A + s * 2 * (128 * 16), 128 * 16, 128);
        const uint64_t bd = desc_kmajor(B + s * 2 * (256 * 16), 256 * 16, 128);
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(s) : "memory");
      }
      if (wait_each) {  // the forest kernel's per-tree commit + wait
        mma_commit(&done);
        bar_wait(&done, it & 1);
      }
    }
    if (!wait_each) { mma_commit(&done); bar_wait(&done, 0); }
    cycles[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_free(tmem, 256); }
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d; cudaMalloc(&d, sms * 8);
  const int smem = 96 * 1024;
  cudaFuncSetAttribute(mma_rate_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int wait_each = 0; wait_each < 2; ++wait_each) {
    const int iters = 1000;
    mma_rate_i8<<<sms, 128, smem>>>(10, wait_each, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_rate_i8<<<sms, 128, smem>>>(iters, wait_each, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c[256]; cudaMemcpy(c, d, sms * 8, cudaMemcpyDeviceToHost);
    const double ops = 2.0 * 128 * 256 * 256 * (double)iters * sms;
    printf("{\"kind\": \"i8\", \"wait_each_tree\": %d, \"ms\": %.3f, \"tops\": %.1f, \"cycles_per_tree\": %.1f, \"err\": \"%s\"}\n",
           wait_each, ms, ops / (ms / 1e3) / 1e12, (double)c[0] / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
