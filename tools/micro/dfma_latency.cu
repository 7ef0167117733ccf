// Dependent-chain latency of float64 FMA (DFMA) and float32 FMA (FFMA) on one
// warp: the float64 linear recompute (linear_exact_whole_kernel) is one
// 784-long DFMA chain per output, so its time is this latency x 784.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dfma_latency dfma_latency.cu && ./dfma_latency
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void chain_f64(double* out, long long* cyc, double a, double b) {
  double acc = threadIdx.x;
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) acc = fma(acc, a, b);
  const long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void chain_f32(float* out, long long* cyc, float a, float b) {
  float acc = threadIdx.x;
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) acc = fmaf(acc, a, b);
  const long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* od;
  float* of;
  long long* c;
  cudaMalloc(&od, 32 * sizeof(double));
  cudaMalloc(&of, 32 * sizeof(float));
  cudaMalloc(&c, sizeof(long long));
  long long h = 0;
  chain_f64<<<1, 32>>>(od, c, 0.999, 1e-3);
  chain_f64<<<1, 32>>>(od, c, 0.999, 1e-3);
  cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"dfma_chain_cycles_per_op\": %.2f, ", (double)h / N);
  chain_f32<<<1, 32>>>(of, c, 0.999f, 1e-3f);
  chain_f32<<<1, 32>>>(of, c, 0.999f, 1e-3f);
  cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("\"ffma_chain_cycles_per_op\": %.2f}\n", (double)h / N);
  return 0;
}
