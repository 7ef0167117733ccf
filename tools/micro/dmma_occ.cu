// DMMA (mma.sync m8n8k4 f64) rate versus warps per SM and independent
// accumulators per warp: is the SVM certifying tier (16 warps/SM, 8
// accumulators per warp, ~31% of the DMMA rate) short of parallelism?
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_occ dmma_occ.cu && ./dmma_occ
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int ACC>
__global__ void dmma_rate(unsigned long long* cycles, double* sink, float seed) {
  double acc[ACC][2];
  double a = seed * (threadIdx.x + 1), b = seed * 0.5;
#pragma unroll
  for (int u = 0; u < ACC; ++u) acc[u][0] = acc[u][1] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < ACC; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[u][0]), "+d"(acc[u][1]) : "d"(a), "d"(b));
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  double s = 0;
#pragma unroll
  for (int u = 0; u < ACC; ++u) s += acc[u][0] + acc[u][1];
  if (s == 1.2345) sink[0] = s;
}

template <int ACC>
static void run(int sms, int threads, double* dsink) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  dmma_rate<ACC><<<sms, threads>>>(cyc, dsink, 1.0f);
  dmma_rate<ACC><<<sms, threads>>>(cyc, dsink, 1.0f);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(sms);
  cudaMemcpy(h.data(), cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  const double fma = (double)(threads / 32) * ITERS * ACC * 256 / (double)h[sms / 2];
  printf("{\"warps_per_sm\": %d, \"acc_per_warp\": %d, \"dmma_fma_per_sm_clk\": %.2f}\n", threads / 32, ACC, fma);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* dsink;
  cudaMalloc(&dsink, 8);
  for (int t : {128, 256, 512, 1024}) {
    run<2>(sms, t, dsink);
    run<4>(sms, t, dsink);
    run<8>(sms, t, dsink);
    run<16>(sms, t, dsink);
  }
  return 0;
}
