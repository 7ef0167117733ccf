// Does tcgen05.mma kind::tf32 truncate or round the low 13 mantissa bits of
// its fp32 operands?  A = 1 + 3*2^-12 (not a tf32 value), B = 1: D = 1 under
// truncation, 1 + 2^-10 under round-to-nearest.  Also A = 1 + 2^-11 + 2^-13
// (just above the half-ulp: RN rounds up).  Single 128x16x8 MMA.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2301_13441_b200/csrc/sm100.cuh"
using namespace cmlb::sm100;

__global__ void probe(float aval, float* out) {
  __shared__ __align__(128) float A[128 * 8];   // K-major core matrices: [2 chunks][128 rows][4]
  __shared__ __align__(128) float B[16 * 8];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 8; i += blockDim.x) A[i] = 0.0f;
  for (int i = t; i < 16 * 8; i += blockDim.x) B[i] = 0.0f;
  __syncthreads();
  if (t == 0) {
    A[0] = aval;   // row 0, k = 0
    B[0] = 1.0f;   // col 0, k = 0
    bar_init(&done, 1);
    bar_fence_init();
  }
  if (warp == 0) tmem_alloc(&slot, 32);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint64_t ad = desc_kmajor(smem_addr(A), 128 * 16, 128);
    const uint64_t bd = desc_kmajor(smem_addr(B), 16 * 16, 128);
    mma_tf32(slot, ad, bd, idesc_tf32(128, 16), 0u);
    mma_commit(&done);
    bar_wait(&done, 0);
  }
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    uint32_t r[32];
    tmem_ld32(slot, r);
    if (t == 0) out[0] = __uint_as_float(r[0]);
  }
  __syncthreads();
  if (warp == 0) tmem_free(slot, 32);
}

int main() {
  float* d; cudaMalloc(&d, 4);
  const float vals[3] = {1.0f + 3.0f / 4096.0f, 1.0f + 1.0f / 2048.0f + 1.0f / 8192.0f, -(1.0f + 3.0f / 4096.0f)};
  for (float v : vals) {
    probe<<<1, 128>>>(v, d);
    float h = 0; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("{\"a\": %.9g, \"d\": %.9g, \"trunc\": %.9g, \"err\": \"%s\"}\n", v, h,
           (double)__builtin_bit_cast(float, __builtin_bit_cast(unsigned, v) & 0xFFFFE000u),
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
