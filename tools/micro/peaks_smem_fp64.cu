// Microbenchmarks for the rooflines the forest and exact paths are bound by
// (measure, don't assume):
//
//  * shared-memory load wavefronts per SM per clock: 32-bit loads with
//    conflict-free lane addresses, broadcast (all lanes one word), 64-bit
//    conflict-free loads (2 wavefronts each), and random addresses inside a
//    256-word table (the deep-level pattern of the row-parallel tree walk);
//  * float64 add / FMA and float32 -> float64 conversion instructions per SM
//    per clock (the ensemble accumulators and the exact recompute paths).
//
// Each CTA times its own loop with clock64(); rates are per SM per clock with
// one CTA per SM.  Prints one JSON object (tools/peaks_micro.sh saves it).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o peaks_smem_fp64 peaks_smem_fp64.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int THREADS = 1024;
constexpr int ITERS = 4096;
constexpr int UNROLL = 8;

// MODE 0: lane-distinct banks (conflict-free); 1: broadcast; 2: 64-bit conflict-free;
// 3: random words in a 256-word table (per-lane xorshift)
template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) smem_rate(unsigned long long* cycles, uint32_t* sink) {
  __shared__ __align__(16) uint32_t tab[8192];
  for (int i = threadIdx.x; i < 8192; i += THREADS) tab[i] = (uint32_t)i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t acc = 0, st = 0x9E3779B9u ^ (threadIdx.x * 7919u) ^ (blockIdx.x * 104729u);
  uint32_t idx[UNROLL];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) idx[u] = (uint32_t)((warp * UNROLL + u) * 32 % 4096);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (MODE == 0) {
        acc ^= tab[(idx[u] + lane) & 8191];
        idx[u] += 32 * 17;
      } else if (MODE == 1) {
        acc ^= tab[idx[u] & 8191];
        idx[u] += 33;
      } else if (MODE == 2) {
        const uint2 v = reinterpret_cast<const uint2*>(tab)[(idx[u] + lane) & 4095];
        acc ^= v.x ^ v.y;
        idx[u] += 32 * 17;
      } else {
        st ^= st << 13; st ^= st >> 17; st ^= st << 5;
        acc ^= tab[(idx[u] & 7936) + (st & 255)];
        idx[u] += 256;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 0x12345678u) sink[0] = acc;
}

// MODE 0: DADD, 1: DFMA, 2: F2F.F64.F32 (+ a cheap FADD to vary the source), 3: FFMA with
// immediate operands, 4: FFMA with register operands, 5: FFMA2 (packed fp32x2) register form
template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) fp_rate(unsigned long long* cycles, double* sink, float seed) {
  double d[UNROLL];
  float f[UNROLL], g[UNROLL], h[UNROLL];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    d[u] = seed * (u + 1 + threadIdx.x);
    f[u] = seed + u;
    g[u] = seed * 0.9999f - u * 1e-7f;
    h[u] = seed * 1e-9f + u;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (MODE == 0) d[u] = d[u] + 1.0000001;
      else if (MODE == 1) d[u] = fma(d[u], 0.9999999, 1e-9);
      else if (MODE == 2) d[u] += (double)__int_as_float(0x3f800000 | ((it * UNROLL + u) & 0x7fffff));
      else if (MODE == 3) f[u] = fmaf(f[u], 0.9999999f, 1e-9f);
      else if (MODE == 4) f[u] = fmaf(f[u], g[u], h[u]);  // independent chains, register operands
      else {  // FFMA2: chains (f[u], h[u]) x (g[u], g[u]) + (f[u], h[u])
        unsigned long long a, b, r;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(f[u]), "f"(h[u]));
        asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(g[u]));
        asm("fma.rn.f32x2 %0, %1, %2, %1;" : "=l"(r) : "l"(a), "l"(b));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(f[u]), "=f"(h[u]) : "l"(r));
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  double s = 0;
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) s += d[u] + f[u] + h[u];
  if (s == 1.2345) sink[0] = s;
}

// FP64 tensor-core MMA (mma.sync m8n8k4 f64, DMMA): 8 independent accumulator
// tiles per warp, each instruction 8 x 8 x 4 = 256 FMAs
__global__ void __launch_bounds__(THREADS, 1) dmma_rate(unsigned long long* cycles, double* sink, float seed) {
  double acc[8][2];
  double a = seed * (threadIdx.x + 1), b = seed * 0.5;
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u][0] = acc[u][1] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[u][0]), "+d"(acc[u][1]) : "d"(a), "d"(b));
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += acc[u][0] + acc[u][1];
  if (s == 1.2345) sink[0] = s;
}

template <typename K, typename... A>
static double per_sm_clk(K kern, int sms, double ops_per_cta, A... args) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  kern<<<sms, THREADS>>>(cyc, args...);  // warm
  kern<<<sms, THREADS>>>(cyc, args...);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(sms);
  cudaMemcpy(h.data(), cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(cyc);
  std::sort(h.begin(), h.end());
  return ops_per_cta / (double)h[sms / 2];  // median CTA
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceProp p{};
  cudaGetDeviceProperties(&p, dev);
  uint32_t* sink;
  double* dsink;
  cudaMalloc(&sink, 64);
  cudaMalloc(&dsink, 64);
  const double warp_instr = (double)(THREADS / 32) * ITERS * UNROLL;
  const double thread_ops = (double)THREADS * ITERS * UNROLL;
  const double cf = per_sm_clk(smem_rate<0>, sms, warp_instr, sink);
  const double bc = per_sm_clk(smem_rate<1>, sms, warp_instr, sink);
  const double v2 = per_sm_clk(smem_rate<2>, sms, warp_instr, sink);
  const double rnd = per_sm_clk(smem_rate<3>, sms, warp_instr, sink);
  const double dadd = per_sm_clk(fp_rate<0>, sms, thread_ops, dsink, 1.0f);
  const double dfma = per_sm_clk(fp_rate<1>, sms, thread_ops, dsink, 1.0f);
  const double f2f = per_sm_clk(fp_rate<2>, sms, thread_ops, dsink, 1.0f);
  const double ffma = per_sm_clk(fp_rate<3>, sms, thread_ops, dsink, 1.0f);
  const double ffma_reg = per_sm_clk(fp_rate<4>, sms, thread_ops, dsink, 1.0f);
  const double ffma2 = per_sm_clk(fp_rate<5>, sms, thread_ops, dsink, 1.0f);  // thread instructions (2 FMAs each)
  // DMMA: per warp-instruction 256 FMAs -> FMAs per SM per clock
  const double dmma_fma = per_sm_clk(dmma_rate, sms, (double)(THREADS / 32) * ITERS * 8 * 256, dsink, 1.0f);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_attr_mhz\": %.0f,\n", p.name, sms, clk_khz / 1e3);
  printf(" \"smem_lds32_conflict_free_warp_instr_per_sm_clk\": %.4f,\n", cf);
  printf(" \"smem_lds32_broadcast_warp_instr_per_sm_clk\": %.4f,\n", bc);
  printf(" \"smem_lds64_conflict_free_warp_instr_per_sm_clk\": %.4f,\n", v2);
  printf(" \"smem_lds32_random256_warp_instr_per_sm_clk\": %.4f,\n", rnd);
  printf(" \"dadd_per_sm_clk\": %.2f, \"dfma_per_sm_clk\": %.2f, \"f2f_f64_f32_plus_dadd_per_sm_clk\": %.2f, "
         "\"ffma_per_sm_clk\": %.2f, \"ffma_reg_per_sm_clk\": %.2f, \"ffma2_instr_per_sm_clk\": %.2f,\n",
         dadd, dfma, f2f, ffma, ffma_reg, ffma2);
  printf(" \"dmma_fp64_fma_per_sm_clk\": %.2f, \"dmma_fp64_tflops_at_max_clock\": %.2f,\n", dmma_fma,
         dmma_fma * 2 * sms * 1965e6 / 1e12);
  printf(" \"fp64_fma_tflops_at_max_clock\": %.2f}\n", dfma * 2 * sms * 1965e6 / 1e12);
  return cudaDeviceSynchronize() != cudaSuccess;
}
