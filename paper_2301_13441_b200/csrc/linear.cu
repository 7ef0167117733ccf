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

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace cmlb {

struct LinearArgs {
  const float* x;
  int64_t n_rows, ldx;
  void* y;
  const float* w;        // [C][F]
  const float* b;        // [C]
  const double* classes;
  const cmlb_column_op* pro;  // fused preprocessing (nullable)
  int F, C, tail, out_dt, sparse;
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

}  // namespace cmlb

struct cmlb_linear {
  int device = 0, F = 0, C = 0, tail = 0, out_dt = 4, sparse = 0, n_inputs = 0;
  float* w = nullptr;
  float* b = nullptr;
  double* classes = nullptr;
  cmlb_column_op* pro = nullptr;
  ~cmlb_linear() { cudaFree(w); cudaFree(b); cudaFree(classes); cudaFree(pro); }
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
  int rows = 0;
  LinFn k = linear_for(m->C, &rows);
  const int64_t grid = ceil_div(n_rows, rows);
  k<<<(unsigned)grid, LNT, 0, (cudaStream_t)stream>>>(a);
  note_launch();
  CMLB_CUDA(cudaGetLastError());
  return CMLB_OK;
}

void cmlb_linear_destroy(cmlb_linear* m) { delete m; }

}  // extern "C"
