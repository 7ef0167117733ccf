// Linear operator representation: matmul(X, coef^T) -> add(intercept) -> tail
// (pkg/src/mlower/convert.py:230-252) in one kernel.
//
// Exactness: the reference accumulates float64 products in ascending k
// (kernels.py:95-100: acc += a64[:, k] * b64[k, :]).  A product of two
// float32 values is exact in float64, so fma(x, w, acc) rounds exactly like
// the reference's separate multiply and add; the logit is rounded once to
// float32 and the intercept added in float32 (kernels.py:162-166).  B200 has
// full-rate-enough FP64 (unlike B300) for this to stay near the HBM roof:
// 1M x 784 x 10 -> 7.8 GFMA vs 3.1 GB of X.
//
// Layout: 128 threads, 2 rows per thread, K staged in chunks of 16 features.
// X chunk in shared memory as xs[k][row] with an odd row stride (conflict-free
// for both the coalesced fill and the per-row reads); the weight chunk as
// float64 ws[k][c], read as warp-wide broadcasts.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"

#include <atomic>
static std::atomic<int64_t> g_linear_queued{-1};  // cmlb_debug_linear_queued

namespace cmlb {

struct LinearArgs {
  const float* x;
  int64_t n_rows, ldx;
  void* y;
  const float* w;        // [C][F]
  const float* b;        // [C]
  const double* classes;
  const cmlb_column_op* pro;  // fused preprocessing (nullable)
  const float* wnorm;         // [C] |w_c|_2 rounded up (certified path)
  int F, C, tail, out_dt, sparse;
  int32_t* queue;             // certified path: rows left to the float64 recompute
  int32_t* queue_len;
};

constexpr int LNT = 128;

// numpy pairwise_sum for n <= 128 (softmax denominator over classes), plus
// the reduction's +0.0 start.
template <int CM>
__device__ __forceinline__ double pw_small(const double (&e)[CM], int n) {
  double res = 0.0;
  if (n < 8) {
#pragma unroll
    for (int i = 0; i < CM; ++i)
      if (i < n) res += e[i];
    return 0.0 + res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = (j < CM) ? e[j] : 0.0;
  const int m = n - n % 8;
#pragma unroll
  for (int i = 8; i < CM; ++i)
    if (i < m) r[i % 8] += e[i];
  res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
  for (int i = 0; i < CM; ++i)
    if (i >= m && i < n) res += e[i];
  return 0.0 + res;
}

// X is streamed in K-chunks of 16 features: each thread holds its share of
// chunk c+1 in registers (float4 loads, coalesced across the row) while the
// CTA computes on chunk c from shared memory, so HBM latency overlaps the FP64
// FMA chains.  The chunk is stored transposed (xs[k][row], odd stride) so the
// per-row reads are conflict-free; W is read as broadcast double2 pairs.
template <int CM, int LRPT, int LKC>
__global__ void __launch_bounds__(LNT) linear_kernel(const LinearArgs a) {
  constexpr int LROWS = LNT * LRPT;
  constexpr int LXS = LROWS + 1;       // odd stride
  constexpr int CE = (CM + 1) / 2 * 2;  // classes padded to pairs
  constexpr int NV = LROWS * LKC / 4 / LNT;  // float4 per thread per chunk
  static_assert(LKC == 16 && NV * LNT * 4 == LROWS * LKC, "chunk shape");
  __shared__ float xs[LKC * LXS];
  __shared__ __align__(16) double ws[LKC * CE];
  const int tid = threadIdx.x;
  const int64_t tile = (int64_t)blockIdx.x * LROWS;
  const int F = a.F, C = a.C;
  const bool vec = (a.ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);

  double acc[LRPT][CM];
#pragma unroll
  for (int k = 0; k < LRPT; ++k)
#pragma unroll
    for (int c = 0; c < CM; ++c) acc[k][c] = 0.0;

  float4 pre[NV];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int idx = tid + LNT * i;
      const int r = idx >> 2, part = idx & 3;
      const int64_t row = tile + r;
      const int k = k0 + part * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < a.n_rows) {
        const float* src = a.x + row * a.ldx + k;
        if (a.pro) {
          const float* rp = a.x + row * a.ldx;
          if (k < F) v.x = load_col(a.pro, rp, k);
          if (k + 1 < F) v.y = load_col(a.pro, rp, k + 1);
          if (k + 2 < F) v.z = load_col(a.pro, rp, k + 2);
          if (k + 3 < F) v.w = load_col(a.pro, rp, k + 3);
        } else if (vec && k + 4 <= F) {
          v = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          if (k < F) v.x = __ldg(src);
          if (k + 1 < F) v.y = __ldg(src + 1);
          if (k + 2 < F) v.z = __ldg(src + 2);
          if (k + 3 < F) v.w = __ldg(src + 3);
        }
      }
      pre[i] = v;
    }
  };
  auto store_chunk = [&](int k0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int idx = tid + LNT * i;
      const int r = idx >> 2, part = idx & 3;
      float* dst = xs + (part * 4) * LXS + r;
      dst[0] = pre[i].x;
      dst[LXS] = pre[i].y;
      dst[2 * LXS] = pre[i].z;
      dst[3 * LXS] = pre[i].w;
    }
    for (int i = tid; i < LKC * CE; i += LNT) {
      const int kk = i / CE, c = i % CE;
      ws[i] = (k0 + kk < F && c < C) ? (double)__ldg(a.w + (int64_t)c * F + k0 + kk) : 0.0;
    }
  };

  load_chunk(0);
  for (int k0 = 0; k0 < F; k0 += LKC) {
    __syncthreads();  // previous chunk consumed
    store_chunk(k0);
    __syncthreads();
    if (k0 + LKC < F) load_chunk(k0 + LKC);  // in flight during the FMAs below
    const int kc = min(LKC, F - k0);
    for (int kk = 0; kk < kc; ++kk) {
      double xv[LRPT];
#pragma unroll
      for (int k = 0; k < LRPT; ++k) xv[k] = (double)xs[kk * LXS + tid + k * LNT];
      const double2* w2 = reinterpret_cast<const double2*>(ws + kk * CE);
#pragma unroll
      for (int c2 = 0; c2 < CE / 2; ++c2) {
        const double2 wv = w2[c2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 2 * c2 + h;
          if (c < CM) {
            const double wc = h ? wv.y : wv.x;
            if (c < C && !(a.sparse && wc == 0.0)) {
#pragma unroll
              for (int k = 0; k < LRPT; ++k) acc[k][c] = fma(xv[k], wc, acc[k][c]);
            }
          }
        }
      }
    }
  }

#pragma unroll
  for (int k = 0; k < LRPT; ++k) {
    const int64_t row = tile + tid + k * LNT;
    if (row >= a.n_rows) continue;
    float z[CM];
#pragma unroll
    for (int c = 0; c < CM; ++c) z[c] = c < C ? __fadd_rn(__double2float_rn(acc[k][c]), __ldg(a.b + c)) : 0.0f;
    switch (a.tail) {
      case CMLB_LIN_VALUES:
#pragma unroll
        for (int c = 0; c < CM; ++c)
          if (c < C) store_out(a.y, row * C + c, a.out_dt, (double)z[c]);
        break;
      case CMLB_LIN_ARGMAX:
        store_out(a.y, row, a.out_dt, a.classes[first_max<CM>(z, C)]);
        break;
      case CMLB_LIN_SOFTMAX_ARGMAX: {
        // kernels.py:227-233: float64 softmax (max-shifted), rounded to float32
        double m = (double)z[0];
        bool nan = false;
#pragma unroll
        for (int c = 0; c < CM; ++c)
          if (c < C) {
            nan |= z[c] != z[c];
            m = fmax(m, (double)z[c]);
          }
        if (nan) m = __longlong_as_double(0x7ff8000000000000LL);
        double e[CM];
#pragma unroll
        for (int c = 0; c < CM; ++c) e[c] = c < C ? exp((double)z[c] - m) : 0.0;
        const double s = pw_small<CM>(e, C);
        float p[CM];
#pragma unroll
        for (int c = 0; c < CM; ++c) p[c] = __double2float_rn(e[c] / s);
        store_out(a.y, row, a.out_dt, a.classes[first_max<CM>(p, C)]);
        break;
      }
      case CMLB_LIN_SIGMOID: {
        const float p = __double2float_rn(ref_sigmoid((double)z[0]));
        store_out(a.y, row, a.out_dt, a.classes[p > 0.5f ? 1 : 0]);
        break;
      }
      default:  // SIGN
        store_out(a.y, row, a.out_dt, a.classes[z[0] > 0.0f ? 1 : 0]);
        break;
    }
  }
}

using LinFn = void (*)(const LinearArgs);


// (kernel, rows per CTA) by output count
static LinFn linear_for(int C, int* rows) {
  *rows = LNT * 2;
  if (C <= 1) return linear_kernel<1, 2, 16>;
  if (C <= 2) return linear_kernel<2, 2, 16>;
  if (C <= 4) return linear_kernel<4, 2, 16>;
  if (C <= 8) return linear_kernel<8, 2, 16>;
  if (C <= 10) return linear_kernel<10, 2, 16>;
  if (C <= 16) return linear_kernel<16, 2, 16>;
  *rows = LNT;
  if (C <= 32) return linear_kernel<32, 1, 16>;
  if (C <= 64) return linear_kernel<64, 1, 16>;
  return nullptr;
}


// ---------------------------------------------------------------------------
// Certified float32 path for the class tails (ARGMAX / SIGMOID / SIGN).
//
// The class needs only the ORDER of the reference's float32 logits (or the
// sign of one), not their bits.  Logits are accumulated in float32 FFMA
// chains (half the bytes of ws, full-rate FP32) with a rigorous bound: a
// sequential chain of n fused multiply-adds errs by at most n u sum|x_k w_k|
// <= n u |x| |w_c| (u = 2^-24, Cauchy-Schwarz), plus the reference's two
// float32 roundings (logit, + b).  When the top logit beats every other by
// more than twice that bound (or the sign is clear of the sigmoid's rounding
// window), the reference class is certain.  Otherwise -- or on any
// non-finite value -- the thread recomputes its row in float64 exactly as the
// reference does (ascending k, kernels.py:95-100, CSR zero-skip) and takes the
// reference tail.  X is read once from HBM either way.
// ---------------------------------------------------------------------------

template <int CM>
__device__ void exact_row_tail(const LinearArgs& a, int64_t row) {
  double acc[CM];
#pragma unroll
  for (int c = 0; c < CM; ++c) acc[c] = 0.0;
  const float* src = a.x + row * a.ldx;
  for (int k = 0; k < a.F; ++k) {
    const double xv = (double)load_col(a.pro, src, k);
#pragma unroll
    for (int c = 0; c < CM; ++c) {
      if (c < a.C) {
        const double wc = (double)__ldg(a.w + (int64_t)c * a.F + k);
        if (!(a.sparse && wc == 0.0)) acc[c] = fma(xv, wc, acc[c]);
      }
    }
  }
  float z[CM];
#pragma unroll
  for (int c = 0; c < CM; ++c) z[c] = c < a.C ? __fadd_rn(__double2float_rn(acc[c]), __ldg(a.b + c)) : 0.0f;
  if (a.tail == CMLB_LIN_ARGMAX) {
    store_out(a.y, row, a.out_dt, a.classes[first_max<CM>(z, a.C)]);
  } else if (a.tail == CMLB_LIN_SIGMOID) {
    const float p = __double2float_rn(ref_sigmoid((double)z[0]));
    store_out(a.y, row, a.out_dt, a.classes[p > 0.5f ? 1 : 0]);
  } else {
    store_out(a.y, row, a.out_dt, a.classes[z[0] > 0.0f ? 1 : 0]);
  }
}

template <int CM, int LRPT, int LKC>
__global__ void __launch_bounds__(LNT) linear_cert_kernel(const LinearArgs a) {
  constexpr int LROWS = LNT * LRPT;
  constexpr int LXS = LROWS + 1;
  constexpr int CE = (CM + 3) / 4 * 4;
  constexpr int NV = LROWS * LKC / 4 / LNT;
  static_assert(LKC == 16 && NV * LNT * 4 == LROWS * LKC, "chunk shape");
  __shared__ float xs[LKC * LXS];
  __shared__ __align__(16) float ws[LKC * CE];
  const int tid = threadIdx.x;
  const int64_t tile = (int64_t)blockIdx.x * LROWS;
  const int F = a.F, C = a.C;
  const bool vec = (a.ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);

  float acc[LRPT][CM], nx[LRPT];
#pragma unroll
  for (int k = 0; k < LRPT; ++k) {
    nx[k] = 0.0f;
#pragma unroll
    for (int c = 0; c < CM; ++c) acc[k][c] = 0.0f;
  }

  float4 pre[NV];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int idx = tid + LNT * i;
      const int r = idx >> 2, part = idx & 3;
      const int64_t row = tile + r;
      const int k = k0 + part * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < a.n_rows) {
        const float* rp = a.x + row * a.ldx;
        if (a.pro) {
          if (k < F) v.x = load_col(a.pro, rp, k);
          if (k + 1 < F) v.y = load_col(a.pro, rp, k + 1);
          if (k + 2 < F) v.z = load_col(a.pro, rp, k + 2);
          if (k + 3 < F) v.w = load_col(a.pro, rp, k + 3);
        } else if (vec && k + 4 <= F) {
          v = __ldg(reinterpret_cast<const float4*>(rp + k));
        } else {
          if (k < F) v.x = __ldg(rp + k);
          if (k + 1 < F) v.y = __ldg(rp + k + 1);
          if (k + 2 < F) v.z = __ldg(rp + k + 2);
          if (k + 3 < F) v.w = __ldg(rp + k + 3);
        }
      }
      pre[i] = v;
    }
  };
  auto store_chunk = [&](int k0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int idx = tid + LNT * i;
      const int r = idx >> 2, part = idx & 3;
      float* dst = xs + (part * 4) * LXS + r;
      dst[0] = pre[i].x;
      dst[LXS] = pre[i].y;
      dst[2 * LXS] = pre[i].z;
      dst[3 * LXS] = pre[i].w;
    }
    for (int i = tid; i < LKC * CE; i += LNT) {
      const int kk = i / CE, c = i % CE;
      ws[i] = (k0 + kk < F && c < C) ? __ldg(a.w + (int64_t)c * F + k0 + kk) : 0.0f;
    }
  };

  load_chunk(0);
  for (int k0 = 0; k0 < F; k0 += LKC) {
    __syncthreads();
    store_chunk(k0);
    __syncthreads();
    if (k0 + LKC < F) load_chunk(k0 + LKC);
    const int kc = min(LKC, F - k0);
    for (int kk = 0; kk < kc; ++kk) {
      float xv[LRPT];
#pragma unroll
      for (int k = 0; k < LRPT; ++k) {
        xv[k] = xs[kk * LXS + tid + k * LNT];
        nx[k] = fmaf(xv[k], xv[k], nx[k]);
      }
      const float4* w4 = reinterpret_cast<const float4*>(ws + kk * CE);
#pragma unroll
      for (int c4 = 0; c4 < CE / 4; ++c4) {
        const float4 wv = w4[c4];
        const float wq[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int c = 4 * c4 + h;
          if (c < CM) {
#pragma unroll
            for (int k = 0; k < LRPT; ++k) acc[k][c] = fmaf(xv[k], wq[h], acc[k][c]);
          }
        }
      }
    }
  }

  // n u |x| |w|: |x| from its own float32 chain (relative error <= F u,
  // covered by the 1.0625 factor for F < 2^20)
  const float nu = (float)(F + 2) * 5.9604644775390625e-08f;
#pragma unroll
  for (int k = 0; k < LRPT; ++k) {
    const int64_t row = tile + tid + k * LNT;
    if (row >= a.n_rows) continue;
    const float xn = sqrtf(nx[k]) * 1.0625f;
    float z[CM], e[CM];
    bool ok = true;
#pragma unroll
    for (int c = 0; c < CM; ++c) {
      if (c < C) {
        z[c] = __fadd_rn(acc[k][c], __ldg(a.b + c));
        // chain bound + the reference's rounding of the logit and of + b
        e[c] = nu * xn * __ldg(a.wnorm + c) + 2.4e-7f * (fabsf(acc[k][c]) + fabsf(z[c]));
        ok = ok && (z[c] - z[c] == 0.0f) && (e[c] < 3.0e38f);  // finite
      } else {
        z[c] = 0.0f;
        e[c] = 0.0f;
      }
    }
    if (ok) {
      if (a.tail == CMLB_LIN_ARGMAX) {
        const int t = first_max<CM>(z, C);
#pragma unroll
        for (int c = 0; c < CM; ++c)
          if (c < C && c != t) ok = ok && (z[t] - z[c] > 2.0f * (e[t] + e[c]));
        if (ok) store_out(a.y, row, a.out_dt, a.classes[t]);
      } else if (a.tail == CMLB_LIN_SIGMOID) {
        // sigmoid(z) rounds above 0.5 for z > 2^-23: demand 2^-21
        if (z[0] - 2.0f * e[0] > 4.76837158203125e-07f) store_out(a.y, row, a.out_dt, a.classes[1]);
        else if (z[0] + 2.0f * e[0] < 0.0f) store_out(a.y, row, a.out_dt, a.classes[0]);
        else ok = false;
      } else {  // SIGN
        if (z[0] - 2.0f * e[0] > 0.0f) store_out(a.y, row, a.out_dt, a.classes[1]);
        else if (z[0] + 2.0f * e[0] < 0.0f) store_out(a.y, row, a.out_dt, a.classes[0]);
        else ok = false;
      }
    }
    if (!ok) a.queue[atomicAdd(a.queue_len, 1)] = (int32_t)row;
  }
}

// Persistent: RPW queued rows per warp (two when C <= 16: one per half-warp),
// float64 in the reference's order -- lane c of a row's lane group runs output
// c's ascending-k FMA chain (kernels.py:95-100); x arrives 32 features at a
// time by coalesced loads, converted once and shuffled within the group.
template <int CM>
__global__ void __launch_bounds__(LNT) linear_exact_rows_kernel(const LinearArgs a) {
  constexpr int RPW = CM <= 16 ? 2 : 1;
  constexpr int GL = 32 / RPW;                      // lanes per row group
  const int nq = *a.queue_len;
  const int lane = threadIdx.x & 31;
  const int slot = lane / GL, c = lane % GL;
  const int64_t gw = ((int64_t)blockIdx.x * LNT + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * LNT) >> 5;
  const int F = a.F, C = a.C;
  for (int64_t i0 = gw * RPW; i0 < nq; i0 += nw * RPW) {
    const int64_t qi = i0 + slot;
    const bool live = qi < nq;
    const int64_t row = live ? a.queue[qi] : a.queue[i0];
    const float* src = a.x + row * a.ldx;
    double acc = 0.0;
    const float* wr = a.w + (int64_t)(c < C ? c : 0) * F;
    for (int k0 = 0; k0 < F; k0 += 32) {
      const int kn = min(32, F - k0);
      double xl[RPW == 2 ? 2 : 1];
#pragma unroll
      for (int h = 0; h < RPW; ++h) {
        const int k = k0 + h * GL + c;
        xl[h] = k < k0 + kn ? (double)load_col(a.pro, src, k) : 0.0;
      }
      float wv[32];  // this lane's coefficients for the 32 features, loaded up front
      if (kn == 32 && c < C && ((reinterpret_cast<uintptr_t>(wr + k0) & 15) == 0)) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(wr + k0 + j));
          wv[j] = q.x; wv[j + 1] = q.y; wv[j + 2] = q.z; wv[j + 3] = q.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) wv[j] = (j < kn && c < C) ? __ldg(wr + k0 + j) : 0.0f;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double xv = __shfl_sync(0xffffffffu, xl[j / GL], slot * GL + (j % GL));
        if (j < kn && c < C && !(a.sparse && wv[j] == 0.0f)) acc = fma(xv, (double)wv[j], acc);
      }
    }
    float zl = c < C ? __fadd_rn(__double2float_rn(acc), __ldg(a.b + c)) : 0.0f;
    float z[CM];
#pragma unroll
    for (int q = 0; q < CM; ++q) z[q] = __shfl_sync(0xffffffffu, zl, slot * GL + (q % GL));
    if (c == 0 && live) {
      if (a.tail == CMLB_LIN_ARGMAX) {
        store_out(a.y, row, a.out_dt, a.classes[first_max<CM>(z, C)]);
      } else if (a.tail == CMLB_LIN_SIGMOID) {
        const float p = __double2float_rn(ref_sigmoid((double)z[0]));
        store_out(a.y, row, a.out_dt, a.classes[p > 0.5f ? 1 : 0]);
      } else {
        store_out(a.y, row, a.out_dt, a.classes[z[0] > 0.0f ? 1 : 0]);
      }
    }
  }
}

// Certified class decision for one row from its float32 logit accumulators
// (sequential FMA chains) and sum of squares: store the label, or queue the
// row for the float64 recompute when the n u |x| |w| bound cannot settle it.
template <int CM>
__device__ __forceinline__ void cert_finish(const LinearArgs& a, int64_t row, const float (&acc)[CM], float nxr,
                                            const float* eblk = nullptr, int kc = 0) {
  const int C = a.C;
  const float nu = (float)(a.F + 2) * 5.9604644775390625e-08f;
  // block a-posteriori bound (eblk, see linear_tile_kernel): u' KC / (1 - KC u')
  // x (sum_b |s_b| + |x| |w_c|), inflated by 1/16 for the float32 evaluation of
  // the bound itself, plus n 2^-149 for underflow in the chain
  const float ku = (float)(kc + 1) * 5.9604644775390625e-08f * 1.0625f;
  const float xn = sqrtf(nxr) * 1.0625f;
  float z[CM], e[CM];
  bool ok = true;
#pragma unroll
  for (int c = 0; c < CM; ++c) {
    if (c < C) {
      z[c] = __fadd_rn(acc[c], __ldg(a.b + c));
      const float chain = eblk ? ku * (eblk[c] + xn * __ldg(a.wnorm + c)) + 1e-37f : nu * xn * __ldg(a.wnorm + c);
      e[c] = chain + 2.4e-7f * (fabsf(acc[c]) + fabsf(z[c]));
      ok = ok && (z[c] - z[c] == 0.0f) && (e[c] < 3.0e38f);
    } else {
      z[c] = 0.0f;
      e[c] = 0.0f;
    }
  }
  if (ok) {
    if (a.tail == CMLB_LIN_ARGMAX) {
      const int t = first_max<CM>(z, C);
      float zt = z[0], et = e[0];
#pragma unroll
      for (int c = 1; c < CM; ++c)
        if (c == t) { zt = z[c]; et = e[c]; }
#pragma unroll
      for (int c = 0; c < CM; ++c)
        if (c < C && c != t) ok = ok && (zt - z[c] > 2.0f * (et + e[c]));
      if (ok) store_out(a.y, row, a.out_dt, a.classes[t]);
    } else if (a.tail == CMLB_LIN_SIGMOID) {
      if (z[0] - 2.0f * e[0] > 4.76837158203125e-07f) store_out(a.y, row, a.out_dt, a.classes[1]);
      else if (z[0] + 2.0f * e[0] < 0.0f) store_out(a.y, row, a.out_dt, a.classes[0]);
      else ok = false;
    } else {
      if (z[0] - 2.0f * e[0] > 0.0f) store_out(a.y, row, a.out_dt, a.classes[1]);
      else if (z[0] + 2.0f * e[0] < 0.0f) store_out(a.y, row, a.out_dt, a.classes[0]);
      else ok = false;
    }
  }
  if (!ok) a.queue[atomicAdd(a.queue_len, 1)] = (int32_t)row;
}

// Thread-per-row certified kernel (the default for class tails, F % 4 == 0):
// each thread streams its rows' features straight from HBM with float4 loads
// (16 features in flight per row, double-buffered in registers; a warp's 32
// rows share their cache lines through L1) and multiplies them against W,
// which sits in shared memory k-major so the CM coefficients of feature k are
// one broadcast read for the whole warp.  Every logit is a sequential float32
// FMA chain (the n u |x| |w| bound of linear_cert_kernel applies verbatim);
// FP32 work is 7,840 FMA per 784-feature row against 3,136 B of HBM reads, so
// the kernel is HBM-bound.
// (1024-thread blocks sharing one W copy measured slower: 64-register cap)
constexpr int LR_NT = 128;

template <int CM, int RPT>
__global__ void __launch_bounds__(LR_NT, 4) linear_rows_kernel(const LinearArgs a) {
  constexpr int CE = (CM + 3) & ~3;
  extern __shared__ __align__(16) float wkm[];   // [F][CE]
  const int F = a.F, C = a.C;
  for (int i = threadIdx.x; i < F * CE; i += LR_NT) {
    const int k = i / CE, c = i - k * CE;
    wkm[i] = c < C ? __ldg(a.w + (int64_t)c * F + k) : 0.0f;
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * LR_NT * RPT + threadIdx.x;
  const float* rp[RPT];
  bool live[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int64_t row = base + r * LR_NT;
    live[r] = row < a.n_rows;
    rp[r] = a.x + (live[r] ? row : 0) * a.ldx;
  }
  float acc[RPT][CM], nx[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    nx[r] = 0.0f;
#pragma unroll
    for (int c = 0; c < CM; ++c) acc[r][c] = 0.0f;
  }
  constexpr int U = 2;  // float4 per row per step (8 features), double-buffered
  float4 cur[RPT][U], nxt[RPT][U];
  auto load = [&](float4 (&dst)[RPT][U], int k0) {
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + 4 * u;
        dst[r][u] = (k < F) ? __ldg(reinterpret_cast<const float4*>(rp[r] + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
  };
  load(cur, 0);
  for (int k0 = 0; k0 < F; k0 += 4 * U) {
    if (k0 + 4 * U < F) load(nxt, k0 + 4 * U);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + 4 * u;
      if (k >= F) break;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4* w4 = reinterpret_cast<const float4*>(wkm + (k + e) * CE);
        float xv[RPT];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          xv[r] = e == 0 ? cur[r][u].x : e == 1 ? cur[r][u].y : e == 2 ? cur[r][u].z : cur[r][u].w;
          nx[r] = fmaf(xv[r], xv[r], nx[r]);
        }
#pragma unroll
        for (int c4 = 0; c4 < CE / 4; ++c4) {
          const float4 w = w4[c4];
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            if (4 * c4 + 0 < CM) acc[r][4 * c4 + 0] = fmaf(xv[r], w.x, acc[r][4 * c4 + 0]);
            if (4 * c4 + 1 < CM) acc[r][4 * c4 + 1] = fmaf(xv[r], w.y, acc[r][4 * c4 + 1]);
            if (4 * c4 + 2 < CM) acc[r][4 * c4 + 2] = fmaf(xv[r], w.z, acc[r][4 * c4 + 2]);
            if (4 * c4 + 3 < CM) acc[r][4 * c4 + 3] = fmaf(xv[r], w.w, acc[r][4 * c4 + 3]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int u = 0; u < U; ++u) cur[r][u] = nxt[r][u];
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r)
    if (live[r]) cert_finish<CM>(a, base + r * LR_NT, acc[r], nx[r]);
}

// Tiled variant of the thread-per-row kernel: a CTA owns NT * RPT consecutive rows
// (RPT per thread, so each W broadcast read feeds RPT rows)
// and streams them through shared memory in KC-feature slices with cp.async
// (16-byte pieces; consecutive lanes fetch one row's contiguous slice, so
// every request covers whole sectors) in an ST-deep ring; the CTA's warps
// share one copy of W.  The 16-byte pieces land XOR-swizzled by row so the
// thread-per-row float4 reads of a quarter warp (8 rows) hit eight distinct
// 16-byte bank groups.  Arithmetic and the certificate are the rows kernel's.
// Stage W ([C][F] float32, F % 4 == 0, 16-byte aligned) into shared memory
// k-major as T [F][ldw] (zero for c >= C), with float4 loads issued eight at
// a time so the copy costs a few L2 round trips, not one per element.
template <typename T, int NTH>
__device__ __forceinline__ void stage_w_kmajor(T* dst, int ldw, const float* w, int C, int F) {
  const int n4 = C * F / 4;
  for (int i0 = threadIdx.x; i0 < n4; i0 += NTH * 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * NTH;
      v[u] = i < n4 ? __ldg(reinterpret_cast<const float4*>(w) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * NTH;
      if (i < n4) {
        const int c = (4 * i) / F, k = 4 * i - c * F;
        dst[(k + 0) * ldw + c] = (T)v[u].x;
        dst[(k + 1) * ldw + c] = (T)v[u].y;
        dst[(k + 2) * ldw + c] = (T)v[u].z;
        dst[(k + 3) * ldw + c] = (T)v[u].w;
      }
    }
  }
  for (int i = threadIdx.x; i < F * (ldw - C); i += NTH) {   // padding columns
    const int k = i / (ldw - C), c = C + i % (ldw - C);
    dst[k * ldw + c] = (T)0;
  }
}

// a0 = fma(x, w0, a0), a1 = fma(x, w1, a1) as one FFMA2 (sm_100 packed fp32;
// ptxas folds the packing moves and the broadcast of x into the operands)
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x, float w0, float w1) {
  unsigned long long xp, wp, ap, rp;
  asm("mov.b64 %0, {%1, %1};" : "=l"(xp) : "f"(x));
  asm("mov.b64 %0, {%1, %2};" : "=l"(wp) : "f"(w0), "f"(w1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(ap) : "f"(a0), "f"(a1));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rp) : "l"(xp), "l"(wp), "l"(ap));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(rp));
}

// (n0, n1) += (v.x^2, v.y^2) then += (v.z^2, v.w^2): one FFMA2 per feature pair
__device__ __forceinline__ void ffma2_pair(float& n0, float& n1, const float4& v) {
  unsigned long long lo, hi, ap, rp;
  asm("mov.b64 %0, {%1, %2};" : "=l"(lo) : "f"(v.x), "f"(v.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(hi) : "f"(v.z), "f"(v.w));
  asm("mov.b64 %0, {%1, %2};" : "=l"(ap) : "f"(n0), "f"(n1));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(rp) : "l"(lo), "l"(ap));
  asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(ap) : "l"(hi), "l"(rp));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(n0), "=f"(n1) : "l"(ap));
}

template <int KC>
__device__ __forceinline__ int lt_swz(int r, int p) {
  if constexpr (KC == 32) return p ^ (r & 7);        // 128-byte rows
  else return p ^ ((r >> 1) & 3);                     // 64-byte rows: two rows per line
}

template <int CM, int NT, int KC, int ST, int RPT>
__global__ void __launch_bounds__(NT, 1) linear_tile_kernel(const LinearArgs a) {
  static_assert(KC == 16 || KC == 32, "slice width");
  constexpr int CE = (CM + 3) & ~3, PC = KC / 4;      // 16-byte pieces per row slice
  constexpr int TR = NT * RPT;                        // rows per tile; thread rows tid + k NT
  extern __shared__ __align__(16) float lsm[];
  float* xt = lsm;                                   // [ST][TR][KC], swizzled
  float* wkm = lsm + ST * TR * KC;                   // [F][CE]
  const int F = a.F, C = a.C, tid = threadIdx.x;
  const int nk = (F + KC - 1) / KC;
  // persistent: this CTA's row tiles are blockIdx.x + i * gridDim.x; the
  // slice stream (tile i, slice kc) runs through the ring without draining
  // between tiles
  const int64_t ntiles = (a.n_rows + TR - 1) / TR;
  const int64_t total = ntiles > blockIdx.x ? ((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * nk : 0;
  // issue cursor: this thread's RPT * PC pieces keep their row and column
  // within a slice, so their source pointers are set once per tile
  int64_t iss_row0 = (int64_t)blockIdx.x * TR;
  int iss_kc = 0;
  int64_t iss_g = 0;
  constexpr int NP = RPT * PC;
  const float* isrc[NP];
  uint32_t idst[NP];
  bool irow[NP];
  const uint32_t xt_s = (uint32_t)__cvta_generic_to_shared(xt);
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const int c = tid + j * NT, r = c / PC, p = c % PC;
    idst[j] = xt_s + (uint32_t)(r * KC + (lt_swz<KC>(r, p) << 2)) * 4u;
  }
  auto set_tile = [&]() {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int c = tid + j * NT, r = c / PC, p = c % PC;
      irow[j] = iss_row0 + r < a.n_rows;
      isrc[j] = a.x + (irow[j] ? iss_row0 + r : 0) * a.ldx + 4 * p;
    }
  };
  set_tile();
  auto issue = [&]() {
    if (iss_g < total) {
      const uint32_t boff = (uint32_t)(iss_g % ST) * (TR * KC * 4);
      const int k0 = iss_kc * KC;
      const bool full = k0 + KC <= F;
      if (full && iss_row0 + TR <= a.n_rows) {  // whole slice of a whole tile: no zero fill
#pragma unroll
        for (int j = 0; j < NP; ++j)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(idst[j] + boff), "l"(isrc[j] + k0)
                       : "memory");
      } else {
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const int p = (tid + j * NT) % PC;
          const bool ok = irow[j] && (full || k0 + 4 * p < F);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(idst[j] + boff),
                       "l"(ok ? isrc[j] + k0 : a.x), "r"(ok ? 16 : 0) : "memory");
        }
      }
      if (++iss_kc == nk) {
        iss_kc = 0;
        iss_row0 += (int64_t)gridDim.x * TR;
        set_tile();
      }
    }
    ++iss_g;
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) issue();
  stage_w_kmajor<float, NT>(wkm, CE, a.w, C, F);
  // eb: sum over slices of |partial logit| at each slice end, for the block
  // a-posteriori bound of cert_finish (a chain's rounding error is at most
  // u' sum_k |s_k|, and within a slice |s_k| <= |s at the slice start| + that
  // slice's sum |x_j w_j|); ~20x tighter than n u |x| |w| on random rows
  float acc[RPT][CM], nx[RPT], nx2[RPT], eb[RPT][CM];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    nx[q] = nx2[q] = 0.0f;
#pragma unroll
    for (int c = 0; c < CM; ++c) acc[q][c] = eb[q][c] = 0.0f;
  }
  int64_t row0 = (int64_t)blockIdx.x * TR;
  int kc = 0;
  for (int64_t g = 0; g < total; ++g) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 2) : "memory");
    __syncthreads();               // slice g visible to all; slice g-1's buffer is free
    issue();
    const float* xb = xt + (int)(g % ST) * (TR * KC);
    const int k0 = kc * KC;
    const int kn = min(KC, F - k0);
#pragma unroll
    for (int p = 0; p < PC; ++p) {
      if (4 * p >= kn) break;
      float4 v[RPT];
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * NT;
        v[q] = *reinterpret_cast<const float4*>(xb + r * KC + (lt_swz<KC>(r, p) << 2));
      }
      // |x|^2 as two interleaved chains (features 4p, 4p+2 and 4p+1, 4p+3): two
      // FFMA2 per float4 instead of four FFMA
#pragma unroll
      for (int q = 0; q < RPT; ++q) ffma2_pair(nx[q], nx2[q], v[q]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float xv[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) xv[q] = e == 0 ? v[q].x : e == 1 ? v[q].y : e == 2 ? v[q].z : v[q].w;
        const float4* w4 = reinterpret_cast<const float4*>(wkm + (k0 + 4 * p + e) * CE);
#pragma unroll
        for (int c4 = 0; c4 < CE / 4; ++c4) {
          const float4 w = w4[c4];
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            // two outputs per FFMA2 (x broadcast): the same IEEE fma chains,
            // half the FMA-pipe instructions
            if (4 * c4 + 1 < CM) ffma2(acc[q][4 * c4 + 0], acc[q][4 * c4 + 1], xv[q], w.x, w.y);
            else if (4 * c4 + 0 < CM) acc[q][4 * c4 + 0] = fmaf(xv[q], w.x, acc[q][4 * c4 + 0]);
            if (4 * c4 + 3 < CM) ffma2(acc[q][4 * c4 + 2], acc[q][4 * c4 + 3], xv[q], w.z, w.w);
            else if (4 * c4 + 2 < CM) acc[q][4 * c4 + 2] = fmaf(xv[q], w.z, acc[q][4 * c4 + 2]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
      for (int c = 0; c < CM; ++c) eb[q][c] += fabsf(acc[q][c]);
    if (++kc == nk) {
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int64_t row = row0 + tid + q * NT;
        if (row < a.n_rows) cert_finish<CM>(a, row, acc[q], nx[q] + nx2[q], eb[q], KC);
        nx[q] = nx2[q] = 0.0f;
#pragma unroll
        for (int c = 0; c < CM; ++c) acc[q][c] = eb[q][c] = 0.0f;
      }
      kc = 0;
      row0 += (int64_t)gridDim.x * TR;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

struct TileCfg { int nt, kc, st, rpt, per_sm; };
static const TileCfg kTileCfg[] = {{128, 32, 4, 1, 2}, {128, 16, 4, 2, 2}, {128, 16, 4, 4, 1}, {64, 16, 4, 4, 2}, {128, 16, 3, 2, 2},
                                   {256, 16, 4, 2, 1}, {128, 32, 4, 2, 1}, {128, 16, 6, 2, 1}, {256, 16, 5, 2, 1},
                                   {256, 16, 6, 1, 1}};
constexpr int N_TILE_CFG = sizeof(kTileCfg) / sizeof(kTileCfg[0]);

template <int CM>
static LinFn tile_fn(int cfg) {
  switch (cfg) {
    case 0: return linear_tile_kernel<CM, 128, 32, 4, 1>;
    case 1: return linear_tile_kernel<CM, 128, 16, 4, 2>;
    case 2: return linear_tile_kernel<CM, 128, 16, 4, 4>;
    case 3: return linear_tile_kernel<CM, 64, 16, 4, 4>;
    case 5: return linear_tile_kernel<CM, 256, 16, 4, 2>;
    case 6: return linear_tile_kernel<CM, 128, 32, 4, 2>;
    case 7: return linear_tile_kernel<CM, 128, 16, 6, 2>;
    case 8: return linear_tile_kernel<CM, 256, 16, 5, 2>;
    case 9: return linear_tile_kernel<CM, 256, 16, 6, 1>;
    default: return linear_tile_kernel<CM, 128, 16, 3, 2>;
  }
}

// Float64 recompute of the queued rows (C <= 16, no prologue, float4-aligned
// rows), one thread per (row, output): thread (r, c) runs output c's
// ascending-k FMA chain of row r (kernels.py:95-100) -- the same arithmetic
// as linear_exact_rows_kernel.  A CTA takes LX_R queued rows x 16 output
// slots; W sits in shared memory as float64 [F][16] (a half warp reads 128
// contiguous bytes per feature), and the rows stream through a cp.async ring
// of 32-feature slices (a half warp's x value is one broadcast read).  Many
// short independent chains per SM keep the float64 pipe fed.
constexpr int LX_R = 16, LX_ST = 4, LX_NT = LX_R * 16;

__global__ void __launch_bounds__(LX_NT) linear_exact_lanes_kernel(const LinearArgs a) {
  extern __shared__ __align__(16) double wq[];        // [F][16], the float64 slice, then the x ring [LX_ST][LX_R][32]
  const int nq = *a.queue_len;
  const int64_t first = (int64_t)blockIdx.x * LX_R;
  if (first >= nq) return;
  const int F = a.F, C = a.C, tid = threadIdx.x;
  stage_w_kmajor<double, LX_NT>(wq, 16, a.w, C, F);
  double* xd = wq + F * 16;                                  // [LX_R][32] the current slice in float64
  float* ring = reinterpret_cast<float*>(xd + LX_R * 32);
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const int r = tid >> 4, c = tid & 15;
  const int nk = (F + 31) / 32;
  __syncthreads();
  for (int64_t qb = first; qb < nq; qb += (int64_t)gridDim.x * LX_R) {
    const int64_t qi = qb + r;
    const bool live = qi < nq;
    const int64_t row = a.queue[live ? qi : qb];
    // pieces: thread t < LX_R * 8 fetches row t / 8's piece t % 8 of each slice
    const int pr = tid >> 3, pp = tid & 7;
    const int64_t prow = tid < LX_R * 8 ? a.queue[qb + pr < nq ? qb + pr : qb] : 0;
    const float* psrc = a.x + prow * a.ldx + 4 * pp;
    auto issue = [&](int kc) {
      if (kc < nk && tid < LX_R * 8) {
        const int k0 = kc * 32;
        const bool ok = k0 + 4 * pp < F;
        const uint32_t d = ring_s + (uint32_t)(((kc % LX_ST) * LX_R + pr) * 32 + 4 * pp) * 4u;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(ok ? psrc + k0 : a.x),
                     "r"(ok ? 16 : 0) : "memory");
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
#pragma unroll
    for (int s2 = 0; s2 < LX_ST - 1; ++s2) issue(s2);
    double acc = 0.0;
    const bool act = c < C;
    for (int kc = 0; kc < nk; ++kc) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(LX_ST - 2) : "memory");
      __syncthreads();
      issue(kc + LX_ST - 1);
      // the slice in float64, converted once (each x value feeds 16 output lanes)
      const float* xsl = ring + (kc % LX_ST) * LX_R * 32;
      for (int i = tid; i < LX_R * 32; i += LX_NT) xd[i] = (double)xsl[i];
      __syncthreads();
      const double* xs = xd + r * 32;
      const int k0 = kc * 32, kn = min(32, F - k0);
      const double* wk = wq + k0 * 16 + c;
      if (a.sparse) {  // CSR weights: only nonzero terms enter the sum (kernels.py:103-126)
        for (int j = 0; j < kn; ++j) {
          const double w = wk[j * 16];
          if (act && w != 0.0) acc = fma(xs[j], w, acc);
        }
      } else if (kn == 32) {
#pragma unroll 8
        for (int j = 0; j < 32; ++j) acc = fma(xs[j], wk[j * 16], acc);  // padded lanes: w = 0
      } else {
        for (int j = 0; j < kn; ++j) acc = fma(xs[j], wk[j * 16], acc);
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();               // ring free before the next batch's prologue
    const float zl = act ? __fadd_rn(__double2float_rn(acc), __ldg(a.b + c)) : 0.0f;
    float z[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) z[q] = __shfl_sync(0xffffffffu, zl, (tid & 16) + q);
    if (c == 0 && live) {
      if (a.tail == CMLB_LIN_ARGMAX) {
        store_out(a.y, row, a.out_dt, a.classes[first_max<16>(z, C)]);
      } else if (a.tail == CMLB_LIN_SIGMOID) {
        const float pz = __double2float_rn(ref_sigmoid((double)z[0]));
        store_out(a.y, row, a.out_dt, a.classes[pz > 0.5f ? 1 : 0]);
      } else {
        store_out(a.y, row, a.out_dt, a.classes[z[0] > 0.0f ? 1 : 0]);
      }
    }
  }
}

// Whole-row form of linear_exact_lanes_kernel for the few rows the block
// bound leaves (~0.03% of LR 784x10): the CTA's 16 queued rows are loaded and
// converted to float64 once (row stride F + 1 doubles: the two rows a warp
// reads sit in different banks), then each thread runs its output's
// ascending-k FMA chain with no barrier inside the chain (the ring form pays
// two barriers per 32 features).  W float64 [F][16] + rows [16][F + 1] must
// fit shared memory (F <= 880); larger F takes the ring form.
__global__ void __launch_bounds__(LX_NT) linear_exact_whole_kernel(const LinearArgs a) {
  extern __shared__ __align__(16) double wq[];   // [F][16] then the rows [LX_R][F + 1]
  const int nq = *a.queue_len;
  const int64_t first = (int64_t)blockIdx.x * LX_R;
  if (first >= nq) return;
  const int F = a.F, C = a.C, tid = threadIdx.x, FP = F + 1;
  stage_w_kmajor<double, LX_NT>(wq, 16, a.w, C, F);
  double* xd = wq + F * 16;
  const int r = tid >> 4, c = tid & 15;
  const bool act = c < C;
  const int f4 = F / 4;  // F % 4 == 0, rows 16-byte aligned (host)
  for (int64_t qb = first; qb < nq; qb += (int64_t)gridDim.x * LX_R) {
    const int64_t qi = qb + r;
    const bool live = qi < nq;
    const int64_t row = a.queue[live ? qi : qb];
    // rows -> float64 shared memory, float4 loads, four in flight per thread
    for (int i0 = tid; i0 < LX_R * f4; i0 += 4 * LX_NT) {
      float4 v[4];
      int64_t rr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * LX_NT;
        if (i < LX_R * f4) {
          const int lr = i / f4;
          rr[u] = a.queue[qb + lr < nq ? qb + lr : qb];
          v[u] = __ldg(reinterpret_cast<const float4*>(a.x + rr[u] * a.ldx) + (i - lr * f4));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * LX_NT;
        if (i < LX_R * f4) {
          const int lr = i / f4, k = 4 * (i - lr * f4);
          double* d = xd + lr * FP + k;
          d[0] = (double)v[u].x; d[1] = (double)v[u].y; d[2] = (double)v[u].z; d[3] = (double)v[u].w;
        }
      }
    }
    __syncthreads();
    const double* xs = xd + r * FP;
    const double* wk = wq + c;
    double acc = 0.0;
    if (a.sparse) {  // CSR weights: only nonzero terms enter the sum (kernels.py:103-126)
      for (int k = 0; k < F; ++k) {
        const double w = wk[k * 16];
        if (act && w != 0.0) acc = fma(xs[k], w, acc);
      }
    } else {
#pragma unroll 8
      for (int k = 0; k < F; ++k) acc = fma(xs[k], wk[k * 16], acc);  // padded lanes: w = 0
    }
    __syncthreads();  // rows consumed before the next batch overwrites them
    const float zl = act ? __fadd_rn(__double2float_rn(acc), __ldg(a.b + c)) : 0.0f;
    float z[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) z[q] = __shfl_sync(0xffffffffu, zl, (tid & 16) + q);
    if (c == 0 && live) {
      if (a.tail == CMLB_LIN_ARGMAX) {
        store_out(a.y, row, a.out_dt, a.classes[first_max<16>(z, C)]);
      } else if (a.tail == CMLB_LIN_SIGMOID) {
        const float pz = __double2float_rn(ref_sigmoid((double)z[0]));
        store_out(a.y, row, a.out_dt, a.classes[pz > 0.5f ? 1 : 0]);
      } else {
        store_out(a.y, row, a.out_dt, a.classes[z[0] > 0.0f ? 1 : 0]);
      }
    }
  }
}

static LinFn linear_cert_for(int C, LinFn* fixup) {
  if (C <= 1) { *fixup = linear_exact_rows_kernel<1>; return linear_cert_kernel<1, 2, 16>; }
  if (C <= 2) { *fixup = linear_exact_rows_kernel<2>; return linear_cert_kernel<2, 2, 16>; }
  if (C <= 4) { *fixup = linear_exact_rows_kernel<4>; return linear_cert_kernel<4, 2, 16>; }
  if (C <= 8) { *fixup = linear_exact_rows_kernel<8>; return linear_cert_kernel<8, 2, 16>; }
  if (C <= 12) { *fixup = linear_exact_rows_kernel<12>; return linear_cert_kernel<12, 2, 16>; }
  if (C <= 16) { *fixup = linear_exact_rows_kernel<16>; return linear_cert_kernel<16, 2, 16>; }
  if (C <= 32) { *fixup = linear_exact_rows_kernel<32>; return linear_cert_kernel<32, 1, 16>; }
  return nullptr;
}

}  // namespace cmlb

struct cmlb_linear {
  int device = 0, F = 0, C = 0, tail = 0, out_dt = 4, sparse = 0, n_inputs = 0;
  float* wnorm = nullptr;
  float* w = nullptr;
  float* b = nullptr;
  double* classes = nullptr;
  cmlb_column_op* pro = nullptr;
  ~cmlb_linear() { cudaFree(w); cudaFree(b); cudaFree(classes); cudaFree(pro); cudaFree(wnorm); }
};

extern "C" {

int cmlb_linear_create(const cmlb_linear_desc* d, int device, cmlb_linear** out) {
  using namespace cmlb;
  if (!out || !d) return fail(CMLB_E_VALIDATION, "null linear descriptor/handle");
  *out = nullptr;
  if (d->n_features < 1 || d->n_outputs < 1) return fail(CMLB_E_VALIDATION, "empty linear model");
  int cm = 0;
  if (!linear_for(d->n_outputs, &cm)) return fail(CMLB_E_UNRESOLVED, "more than 64 linear outputs");
  if (!out_dtype_ok(d->out_dtype)) return fail(CMLB_E_VALIDATION, "bad out_dtype");
  if (d->tail != CMLB_LIN_VALUES && d->n_classes < (d->n_outputs == 1 ? 2 : d->n_outputs))
    return fail(CMLB_E_VALIDATION, "class table does not match the tail");
  DeviceGuard guard(device);
  std::unique_ptr<cmlb_linear> m(new cmlb_linear());
  m->device = device; m->F = d->n_features; m->C = d->n_outputs; m->tail = d->tail;
  m->out_dt = d->out_dtype; m->sparse = d->sparse_coef ? 1 : 0;
  const size_t nw = (size_t)m->F * m->C;
  CMLB_CUDA(cudaMalloc(&m->w, nw * sizeof(float)));
  CMLB_CUDA(cudaMemcpy(m->w, d->coef, nw * sizeof(float), cudaMemcpyHostToDevice));
  CMLB_CUDA(cudaMalloc(&m->b, m->C * sizeof(float)));
  CMLB_CUDA(cudaMemcpy(m->b, d->intercept, m->C * sizeof(float), cudaMemcpyHostToDevice));
  const int nc = d->n_classes > 0 ? d->n_classes : 1;
  CMLB_CUDA(cudaMalloc(&m->classes, nc * sizeof(double)));
  if (d->n_classes > 0)
    CMLB_CUDA(cudaMemcpy(m->classes, d->classes, nc * sizeof(double), cudaMemcpyHostToDevice));
  {
    std::vector<float> wn(m->C);
    for (int c = 0; c < m->C; ++c) {
      double s2 = 0.0;
      for (int k = 0; k < m->F; ++k) s2 += (double)d->coef[(size_t)c * m->F + k] * d->coef[(size_t)c * m->F + k];
      wn[c] = (float)(std::sqrt(s2) * (1.0 + 1e-6));
    }
    CMLB_CUDA(cudaMalloc(&m->wnorm, m->C * sizeof(float)));
    CMLB_CUDA(cudaMemcpy(m->wnorm, wn.data(), m->C * sizeof(float), cudaMemcpyHostToDevice));
  }
  m->n_inputs = m->F;
  if (d->prologue) {
    if (d->n_inputs <= 0) return fail(CMLB_E_VALIDATION, "prologue needs n_inputs > 0");
    for (int k = 0; k < m->F; ++k) {
      const cmlb_column_op& o = d->prologue[k];
      if (o.src < 0 || o.src >= d->n_inputs || o.op < CMLB_COL_COPY || o.op > CMLB_COL_EQUAL)
        return fail(CMLB_E_VALIDATION, "bad prologue column op");
    }
    m->n_inputs = d->n_inputs;
    CMLB_CUDA(cudaMalloc(&m->pro, (size_t)m->F * sizeof(cmlb_column_op)));
    CMLB_CUDA(cudaMemcpy(m->pro, d->prologue, (size_t)m->F * sizeof(cmlb_column_op), cudaMemcpyHostToDevice));
  }
  *out = m.release();
  return CMLB_OK;
}

int cmlb_linear_run(const cmlb_linear* m, const float* x, int64_t n_rows, int64_t ldx, void* y,
                    void* stream) {
  using namespace cmlb;
  if (!m) return fail(CMLB_E_VALIDATION, "null linear model");
  if (n_rows < 0 || ldx < m->n_inputs) return fail(CMLB_E_INPUT, "bad input extents");
  if (n_rows == 0) return CMLB_OK;
  DeviceGuard guard(m->device);
  LinearArgs a{};
  a.pro = m->pro;
  a.x = x; a.n_rows = n_rows; a.ldx = ldx; a.y = y; a.w = m->w; a.b = m->b; a.classes = m->classes;
  a.F = m->F; a.C = m->C; a.tail = m->tail; a.out_dt = m->out_dt; a.sparse = m->sparse;
  a.wnorm = m->wnorm;
  keep_pool(m->device);
  int rows = 0;
  LinFn k = linear_for(m->C, &rows);
  // class tails: certified float32 logits (exact float64 recompute of the
  // rare rows whose class the bound cannot settle); CMLB_LINEAR_EXACT=1 forces
  // the float64 kernel everywhere
  static const bool force_exact = [] {
    const char* e = std::getenv("CMLB_LINEAR_EXACT");
    return e && e[0] == '1';
  }();
  LinFn fixup = nullptr;
  if (!force_exact && m->tail != CMLB_LIN_VALUES && m->tail != CMLB_LIN_SOFTMAX_ARGMAX) {
    if (LinFn kc = linear_cert_for(m->C, &fixup)) {
      k = kc;
      rows = m->C <= 16 ? 2 * LNT : LNT;
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  void* scratch = nullptr;
  if (fixup) {
    if (n_rows > INT32_MAX) return fail(CMLB_E_INPUT, "linear batch exceeds 2^31 rows");
    CMLB_CUDA(cudaMallocAsync(&scratch, (size_t)(n_rows + 4) * sizeof(int32_t), s));
    a.queue_len = static_cast<int32_t*>(scratch);
    a.queue = a.queue_len + 4;
    CMLB_CUDA(cudaMemsetAsync(a.queue_len, 0, sizeof(int32_t), s));
  }
  // thread-per-row certified kernel when rows are float4-aligned and W fits
  const int cm = m->C <= 2 ? 2 : m->C <= 4 ? 4 : m->C <= 8 ? 8 : m->C <= 10 ? 10 : m->C <= 12 ? 12 : 16;
  const size_t wbytes = (size_t)m->F * ((cm + 3) & ~3) * 4;
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (ldx % 4) == 0 && (m->F % 4) == 0;
  if (fixup && !m->pro && m->C <= 16 && aligned && wbytes <= 100 * 1024) {
    static const int lin_impl = [] {
      const char* e = std::getenv("CMLB_LINEAR_IMPL");   // 0: rows kernel; n >= 1: tile config n - 1
      return e ? std::atoi(e) : 2;
    }();
    if (lin_impl >= 1) {
      const int cfg = std::min(lin_impl - 1, N_TILE_CFG - 1);
      LinFn kt = cm == 2 ? tile_fn<2>(cfg) : cm == 4 ? tile_fn<4>(cfg) : cm == 8 ? tile_fn<8>(cfg)
               : cm == 10 ? tile_fn<10>(cfg) : cm == 12 ? tile_fn<12>(cfg) : tile_fn<16>(cfg);
      const TileCfg tc = kTileCfg[cfg];
      const size_t sb = (size_t)tc.st * tc.nt * tc.rpt * tc.kc * 4 + wbytes;
      CMLB_CUDA(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
      int occ = 0;   // persistent grid: as many CTAs per SM as registers / shared memory allow
      CMLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kt, tc.nt, sb));
      const int64_t g = std::min<int64_t>(ceil_div(n_rows, (int64_t)tc.nt * tc.rpt),
                                          (int64_t)num_sms(m->device) * std::max(occ, 1));
      kt<<<(unsigned)g, tc.nt, sb, s>>>(a);
    } else {
      LinFn kr = cm == 2 ? linear_rows_kernel<2, 2> : cm == 4 ? linear_rows_kernel<4, 2> : cm == 8 ? linear_rows_kernel<8, 2>
               : cm == 10 ? linear_rows_kernel<10, 2> : cm == 12 ? linear_rows_kernel<12, 2> : linear_rows_kernel<16, 2>;
      const int rpt = 2;
      CMLB_CUDA(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wbytes));
      kr<<<(unsigned)ceil_div(n_rows, (int64_t)LR_NT * rpt), LR_NT, wbytes, s>>>(a);
    }
  } else {
    const int64_t grid = ceil_div(n_rows, rows);
    k<<<(unsigned)grid, LNT, 0, s>>>(a);
  }
  note_launch();
  CMLB_CUDA(cudaGetLastError());
  if (fixup) {
    static const bool old_fix = std::getenv("CMLB_LINEAR_FIXUP_WARP") != nullptr;
    const size_t xb = (size_t)m->F * 16 * 8 + (size_t)LX_R * 32 * 8 + (size_t)LX_ST * LX_R * 32 * 4;
    const size_t xw = (size_t)m->F * 16 * 8 + (size_t)LX_R * (m->F + 1) * 8;
    if (!old_fix && m->C <= 16 && !m->pro && aligned && xw <= 220 * 1024 && !std::getenv("CMLB_LINEAR_RING")) {
      CMLB_CUDA(cudaFuncSetAttribute(linear_exact_whole_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xw));
      // persistent: one CTA per SM (at ~0.03% queued rows, a handful are busy)
      const int g = (int)std::min<int64_t>(ceil_div(n_rows, (int64_t)LX_R), (int64_t)num_sms(m->device));
      linear_exact_whole_kernel<<<g, LX_NT, xw, s>>>(a);
    } else if (!old_fix && m->C <= 16 && !m->pro && aligned && xb <= 200 * 1024) {
      CMLB_CUDA(cudaFuncSetAttribute(linear_exact_lanes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xb));
      int per_sm = 0;
      CMLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, linear_exact_lanes_kernel, LX_NT, xb));
      const int g = (int)std::min<int64_t>(ceil_div(n_rows, (int64_t)LX_R), (int64_t)num_sms(m->device) * std::max(per_sm, 1));
      linear_exact_lanes_kernel<<<g, LX_NT, xb, s>>>(a);
    } else {
      const int g = (int)std::min<int64_t>(ceil_div(n_rows, LNT), (int64_t)num_sms(m->device) * 4);
      fixup<<<g, LNT, 0, s>>>(a);
    }
    note_launch();
    CMLB_CUDA(cudaGetLastError());
    static const bool qstat = std::getenv("CMLB_LINEAR_QSTAT") != nullptr;  // measurement knob
    if (qstat) {
      int32_t q = 0;
      CMLB_CUDA(cudaMemcpyAsync(&q, a.queue_len, sizeof(q), cudaMemcpyDeviceToHost, s));
      CMLB_CUDA(cudaStreamSynchronize(s));
      g_linear_queued.store(q);
    }
    CMLB_CUDA(cudaFreeAsync(scratch, s));
  }
  return CMLB_OK;
}

int64_t cmlb_debug_linear_queued(void) { return g_linear_queued.load(); }

void cmlb_linear_destroy(cmlb_linear* m) { delete m; }

}  // extern "C"
